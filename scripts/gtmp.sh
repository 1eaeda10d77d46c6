cd /root/repo
timeout 1500 python scripts/emulate_ranks.py rmat rect > gpurun_out/emulated_ranks2.md 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "multi or distributed or summary or light or fem27" > gpurun_out/pytest_g39.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g39.log
