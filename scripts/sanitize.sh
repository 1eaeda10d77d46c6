#!/bin/bash
# compute-sanitizer over scripts/sanitize_corpus.py (memcheck, racecheck,
# synccheck); summaries to gpurun_out/sanitizer_<tool>.txt
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck}; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
    python scripts/sanitize_corpus.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer_$tool.txt
done
