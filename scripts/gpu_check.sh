#!/bin/bash
# One gpurun session: parity tests, smoke, a short bench, ncu launch list +
# one full capture of the top kernel.  Usage: gpu_check.sh [tag] [kernel-regex]
TAG=${1:-r1}
KREGEX=${2:-numeric_tc}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
      python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX}" -s ${NSKIP:-2} -c ${NCAP:-1} \
      -o gpurun_out/prof_${TAG} -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
fi
# compute-sanitizer memcheck / racecheck / synccheck over the parity corpus
# (summaries: gpurun_out/sanitizer_<tool>.txt, kept as profiles/r02_sanitizer_*)
[ -n "$SANITIZE" ] && bash scripts/sanitize.sh
true
