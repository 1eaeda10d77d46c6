#!/bin/bash
# general-path copy: TSG_ESC_COPY_U staged entries per lane in flight
mkdir -p gpurun_out
: > gpurun_out/esccopy_ab.log
for u in 4 8; do
  TSG_NVCC_FLAGS="-DTSG_ESC_COPY_U=$u" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esccopy_ab.log 2>&1
  echo "ESC_COPY_U=$u" >> gpurun_out/esccopy_ab.log
  timeout 600 python scripts/cfg_time.py rmat rect --reps 5 >> gpurun_out/esccopy_ab.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esccopy_ab.log 2>&1
