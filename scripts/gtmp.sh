cd /root/repo
bash scripts/final_check.sh
TOOLS="memcheck" bash scripts/sanitize.sh
