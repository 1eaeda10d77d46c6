#!/bin/bash
# Round profile of the bench workload: ncu launch list (per-launch device
# times, cold + serialised) and one --set full capture of every kernel of
# one step.  Usage: profile_round.sh <tag> [bench args]
TAG=${1:-r01}; shift
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_launch_${TAG}.log 2>&1
# one step after one warm-up: skip the warm-up's launches
N=$(grep -c '"gpu__time_duration.sum"' gpurun_out/launches_${TAG}.csv)
PER=$((N / 3))
timeout 1200 ncu --set full --clock-control none --import-source on -s ${PER} -c ${PER} \
  -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ncu_full_${TAG}.log 2>&1
