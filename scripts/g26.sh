cd /root/repo
bash scripts/esc_diag.sh
timeout 600 python scripts/cfg_time.py rmat rect --reps 5 > gpurun_out/cfg_time.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rmat or rect or general or r02 or counters" > gpurun_out/pytest_g26.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g26.log
bash scripts/launch_list.sh rmat
