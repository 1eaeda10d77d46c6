#!/bin/bash
# tcgen05 light pass: parity on the light configs + timing against mma.sync
mkdir -p gpurun_out
timeout 600 python scripts/diag_rmat.py > gpurun_out/diag_rmat.log 2>&1
TSG_TC05=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "poisson or fem27 or golden or acceptance_corpus or device_output or fp16" > gpurun_out/pytest_tc05.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_tc05.log
for v in 0 1; do echo "TSG_TC05=$v" >> gpurun_out/tc05_time.log; TSG_TC05=$v timeout 300 python scripts/cfg_time.py fem27 poisson amg --reps 5 >> gpurun_out/tc05_time.log 2>&1; done
