#!/bin/bash
# Bench every BASELINE config (device-resident step, phase times), no CPU legs.
mkdir -p gpurun_out
: > gpurun_out/bench_all.log
for c in ${CONFIGS:-fem27 poisson amg rect rmat}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/bench_all.log 2>&1
done
