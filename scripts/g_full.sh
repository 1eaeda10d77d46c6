#!/bin/bash
# full GPU tests, per-config device times, rank emulation
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/cfg_time.py > gpurun_out/cfg_time.log 2>&1
[ -n "$EMU" ] && timeout 900 python scripts/emulate_ranks.py rmat fem27 amg > gpurun_out/emulated_ranks.md 2>&1
true
