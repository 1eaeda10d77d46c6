cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "summary or r02" > gpurun_out/pytest_g31.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g31.log
timeout 1200 python scripts/emulate_ranks.py rmat > gpurun_out/emulated_ranks.md 2>&1
