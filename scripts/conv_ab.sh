#!/bin/bash
# conversion variants (TSG_CONV_MINB resident blocks of convert_fast_kernel); then the GPU tests
mkdir -p gpurun_out
: > gpurun_out/conv_ab.log
for mb in 4 3; do
  TSG_NVCC_FLAGS="-DTSG_CONV_MINB=$mb" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/conv_ab.log 2>&1
  echo "CONV_MINB=$mb" >> gpurun_out/conv_ab.log
  timeout 600 python scripts/cfg_time.py rmat rect fem27 --reps 5 >> gpurun_out/conv_ab.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/conv_ab.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
bash scripts/launch_list.sh rmat
