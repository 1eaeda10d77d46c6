#!/bin/bash
# esc_kernel leaf statistics (build-time -DTSG_ESC_DIAG), then the normal build back
mkdir -p gpurun_out
TSG_NVCC_FLAGS="-DTSG_ESC_DIAG" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" > gpurun_out/esc_diag.log 2>&1
for c in ${CFGS:-rmat rect}; do timeout 600 python scripts/one_call.py $c >> gpurun_out/esc_diag.log 2>&1; done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esc_diag.log 2>&1
