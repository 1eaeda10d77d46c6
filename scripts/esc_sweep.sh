#!/bin/bash
# esc_kernel: work-unit target sweep + a source-level ncu capture of the kernel
mkdir -p gpurun_out
: > gpurun_out/esc_sweep.log
for t in 2560 3072 3584 4000; do
  echo "TSG_ESC_TARGET=$t" >> gpurun_out/esc_sweep.log
  TSG_ESC_TARGET=$t timeout 300 python scripts/cfg_time.py rmat rect --reps 3 >> gpurun_out/esc_sweep.log 2>&1
done
ONE_CALL_WARM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:esc_kernel -c 1 -o /tmp/p_esc -f \
    python scripts/one_call.py rmat > gpurun_out/ncu_esc.log 2>&1
python scripts/ncu_summary.py /tmp/p_esc.ncu-rep > gpurun_out/top_esc.txt 2>&1
python scripts/ncu_json.py /tmp/p_esc.ncu-rep gpurun_out/ncu_esc.json "ncu --set full --clock-control none, esc_kernel of scripts/one_call.py rmat (warm)" > /dev/null 2>&1
cp /tmp/p_esc.ncu-rep gpurun_out/p_esc.ncu-rep
