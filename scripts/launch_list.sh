#!/bin/bash
# per-kernel device times of one warm call of a config (ncu launch list)
mkdir -p gpurun_out
CFG=${1:-rmat}
ONE_CALL_WARM=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_one_${CFG}.csv python scripts/one_call.py $CFG > gpurun_out/launch_one_${CFG}.log 2>&1
python scripts/launches.py gpurun_out/launches_one_${CFG}.csv > gpurun_out/launches_one_${CFG}.txt 2>&1
