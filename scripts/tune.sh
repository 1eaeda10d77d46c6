#!/bin/bash
# Sweep build-time kernel variants (env-selected) on the bench config.
mkdir -p gpurun_out
: > gpurun_out/tune.log
for nb in ${NBS:-2 4 8}; do
  for cb in ${CBS:-4 8 16}; do
    echo "NUMERIC_BATCH=$nb COUNT_BATCH=$cb" >> gpurun_out/tune.log
    TSG_NUMERIC_BATCH=$nb TSG_COUNT_BATCH=$cb timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} >> gpurun_out/tune.log 2>&1
  done
done
