#!/bin/bash
# light-pass variants: TSG_PANEL_PREFETCH (double-buffered chunk gathers) x TSG_PANEL_KB (resident blocks)
mkdir -p gpurun_out
: > gpurun_out/panel_ab.log
for v in "0 4" "1 3" "0 3" ${EXTRA_VARIANTS}; do
  set -- $v
  TSG_NVCC_FLAGS="-DTSG_PANEL_PREFETCH=$1 -DTSG_PANEL_KB=$2" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/panel_ab.log 2>&1
  echo "PREFETCH=$1 KB=$2" >> gpurun_out/panel_ab.log
  timeout 600 python scripts/cfg_time.py fem27 poisson amg --reps 7 >> gpurun_out/panel_ab.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/panel_ab.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "light or fem27 or poisson or amg or golden or corpus or chain or config" > gpurun_out/pytest_panel.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_panel.log
