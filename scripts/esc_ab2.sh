#!/bin/bash
# esc_kernel variants: TSG_ESC_ROT (rotated 16-byte vectors of the blocked layout)
mkdir -p gpurun_out
: > gpurun_out/esc_ab2.log
for v in ${VARIANTS:-"-DTSG_ESC_ROT=1" "-DTSG_ESC_ROT=0"}; do
  TSG_NVCC_FLAGS="$v" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esc_ab2.log 2>&1
  echo "VARIANT $v" >> gpurun_out/esc_ab2.log
  timeout 600 python scripts/cfg_time.py rmat rect --reps 5 >> gpurun_out/esc_ab2.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esc_ab2.log 2>&1
