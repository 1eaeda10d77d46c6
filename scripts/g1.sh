mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/cfg_time.py > gpurun_out/cfg_time.log 2>&1; echo "rc=$?" >> gpurun_out/cfg_time.log
timeout 600 python bench.py --config rmat --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rmat.log 2>&1; echo "rc=$?" >> gpurun_out/bench_rmat.log
