cd /root/repo
: > gpurun_out/pos_ab.log
for v in 0 1; do echo "TSG_ESC_POS=$v" >> gpurun_out/pos_ab.log; TSG_ESC_POS=$v timeout 600 python scripts/cfg_time.py rmat rect --reps 5 >> gpurun_out/pos_ab.log 2>&1; done
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rmat or rect or general or r02 or counters or summary or corpus" > gpurun_out/pytest_pos.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pos.log
bash scripts/launch_list.sh rmat
