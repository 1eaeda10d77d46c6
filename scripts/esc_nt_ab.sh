#!/bin/bash
# esc_kernel CTA size A/B: 256 threads (IPT <= 16) vs 512 threads (IPT <= 8)
mkdir -p gpurun_out
: > gpurun_out/esc_nt.log
for nt in 256 512; do
  TSG_NVCC_FLAGS="-DTSG_ESC_NT=$nt" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esc_nt.log 2>&1
  echo "TSG_ESC_NT=$nt" >> gpurun_out/esc_nt.log
  timeout 600 python scripts/cfg_time.py rmat rect --reps 3 >> gpurun_out/esc_nt.log 2>&1
  if [ $nt = 512 ]; then
    timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "general or rect or config_full_size or r02 or conversion" > gpurun_out/pytest_nt512.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_nt512.log
  fi
done
