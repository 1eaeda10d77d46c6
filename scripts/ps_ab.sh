#!/bin/bash
# pair statistics: A tiles per lane (TSG_PS_TILES)
mkdir -p gpurun_out
: > gpurun_out/ps_ab.log
for t in 1 2 4; do
  TSG_NVCC_FLAGS="-DTSG_PS_TILES=$t" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/ps_ab.log 2>&1
  echo "PS_TILES=$t" >> gpurun_out/ps_ab.log
  timeout 600 python scripts/cfg_time.py rmat rect --reps 5 >> gpurun_out/ps_ab.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/ps_ab.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rmat or rect or general or counters or summary or corpus or golden" > gpurun_out/pytest_ps.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ps.log
