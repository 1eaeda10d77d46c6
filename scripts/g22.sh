cd /root/repo
bash scripts/g_full.sh
bash scripts/launch_rank.sh rmat 8 0
TOOLS=memcheck bash scripts/sanitize.sh
