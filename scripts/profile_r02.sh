#!/bin/bash
# Round-2 profile of one bench config, summarised ON the box (the raw .ncu-rep
# of a large config exceeds gpurun's 64 MiB return limit):
#   launches_<tag>.csv      ncu launch list of the bench command (cold, serialised)
#   ncu_full_<tag>.json     --set full of every kernel of one device-output call
#                           (scripts/one_call.py), scripts/ncu_json.py summary
#   src_<tag>.csv / mix     source-level SASS page + opcode mix of the top kernel
# Usage: profile_r02.sh <tag> <config> <top-kernel-regex>
TAG=${1:-r02_rmat}; CFG=${2:-rmat}; KRE=${3:-esc_kernel}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --config ${CFG} --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch_${TAG}.log
timeout 1500 ncu --set full --clock-control none -o /tmp/prof_${TAG} -f python scripts/one_call.py ${CFG} > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full_${TAG}.log
python scripts/ncu_json.py /tmp/prof_${TAG}.ncu-rep gpurun_out/ncu_full_${TAG}.json "ncu --set full --clock-control none of scripts/one_call.py ${CFG}" > /dev/null 2>> gpurun_out/ncu_full_${TAG}.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KRE}" -c 1 -o /tmp/top_${TAG} -f python scripts/one_call.py ${CFG} >> gpurun_out/ncu_full_${TAG}.log 2>&1
python scripts/ncu_summary.py /tmp/top_${TAG}.ncu-rep > gpurun_out/top_${TAG}.txt 2>&1
ncu -i /tmp/top_${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}.csv 2>/dev/null
ls -la /tmp/top_${TAG}.ncu-rep >> gpurun_out/ncu_full_${TAG}.log
sz=$(stat -c %s /tmp/top_${TAG}.ncu-rep); [ "$sz" -lt 40000000 ] && cp /tmp/top_${TAG}.ncu-rep gpurun_out/
