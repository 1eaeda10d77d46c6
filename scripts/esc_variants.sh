#!/bin/bash
# A/B of general-path (esc_kernel) variants on the device-resident configs,
# then the general-path parity tests.  Usage: esc_variants.sh [configs]
mkdir -p gpurun_out
CFGS=${CFGS:-"rmat rect"}
: > gpurun_out/esc_variants.log
for v in ${VARIANTS:-3 4}; do
  echo "TSG_ESC_MINB=$v" >> gpurun_out/esc_variants.log
  TSG_ESC_MINB=$v timeout 600 python scripts/cfg_time.py $CFGS --reps 3 >> gpurun_out/esc_variants.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "${TESTK:-general or rect or config_full_size or chain or r02 or conversion}" > gpurun_out/pytest_esc.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_esc.log
