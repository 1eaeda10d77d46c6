#!/bin/bash
# Round profile of a bench config: the ncu launch list of the bench command
# (per-launch device times, cold + serialised) and one --set full capture of
# every kernel of a single call (scripts/one_call.py).
# Usage: profile_round.sh <tag> <config>
TAG=${1:-r01}; CFG=${2:-fem27}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --config ${CFG} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -o gpurun_out/prof_${TAG} -f python scripts/one_call.py ${CFG} > gpurun_out/ncu_full_${TAG}.log 2>&1
