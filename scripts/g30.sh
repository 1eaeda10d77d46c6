cd /root/repo
bash scripts/g_full.sh
bash scripts/launch_list.sh rmat
bash scripts/launch_rank.sh rmat 8 0
