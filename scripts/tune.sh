#!/bin/bash
# Sweep build-time kernel variants (env-selected) on the bench config.
mkdir -p gpurun_out
: > gpurun_out/tune.log
for v in ${VARIANTS:-"2 5"}; do
  set -- $v
  echo "TSG_NUMERIC_BATCH=$1 TSG_NUMERIC_MINB=$2" >> gpurun_out/tune.log
  TSG_NUMERIC_BATCH=$1 TSG_NUMERIC_MINB=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} >> gpurun_out/tune.log 2>&1
done
