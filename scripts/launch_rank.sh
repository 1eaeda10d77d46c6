#!/bin/bash
# per-kernel device times of one warm call of rank p's panel of an N-GPU run
mkdir -p gpurun_out
CFG=${1:-rmat}; N=${2:-8}; P=${3:-0}
ONE_CALL_WARM=1 ONE_CALL_PANEL=$N,$P timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_rank_${CFG}_${N}_${P}.csv python scripts/one_call.py $CFG > gpurun_out/launch_rank_${CFG}.log 2>&1
python scripts/launches.py gpurun_out/launches_rank_${CFG}_${N}_${P}.csv > gpurun_out/launches_rank_${CFG}_${N}_${P}.txt 2>&1
