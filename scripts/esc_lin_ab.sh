#!/bin/bash
# build_table range searches: binary steps down to TSG_ESC_LIN entries, then one linear round
mkdir -p gpurun_out
: > gpurun_out/lin_ab.log
for l in 0 4 8 16; do
  TSG_NVCC_FLAGS="-DTSG_ESC_LIN=$l" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/lin_ab.log 2>&1
  echo "TSG_ESC_LIN=$l" >> gpurun_out/lin_ab.log
  timeout 600 python scripts/cfg_time.py rmat rect --reps 5 >> gpurun_out/lin_ab.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/lin_ab.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rmat or rect or general or counters or corpus" > gpurun_out/pytest_lin.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_lin.log
