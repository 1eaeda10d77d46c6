cd /root/repo
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python scripts/emulate_ranks.py rmat fem27 amg rect > gpurun_out/emulated_ranks.md 2>&1
