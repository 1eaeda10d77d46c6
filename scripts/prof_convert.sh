#!/bin/bash
# ncu --set full (with source) of the R-MAT conversion and pair-statistics
# kernels of one warm call; summaries on the box
mkdir -p gpurun_out
KRE=${KRE:-"convert_fast|convert_hub|tiles_compact|esc_njt|esc_pairstats|esc_colhist|esc_brow"}
ONE_CALL_WARM=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KRE" -c 14 \
  -o /tmp/p_conv -f python scripts/one_call.py ${CFG:-rmat} > gpurun_out/ncu_conv.log 2>&1
python scripts/ncu_json.py /tmp/p_conv.ncu-rep gpurun_out/ncu_conv.json "ncu --set full --clock-control none, conversion + pair statistics of scripts/one_call.py rmat (warm)" >> gpurun_out/ncu_conv.log 2>&1
python scripts/ncu_summary.py /tmp/p_conv.ncu-rep > gpurun_out/top_conv.txt 2>&1
ls -la /tmp/p_conv.ncu-rep >> gpurun_out/ncu_conv.log
sz=$(stat -c %s /tmp/p_conv.ncu-rep); [ "$sz" -lt 40000000 ] && cp /tmp/p_conv.ncu-rep gpurun_out/
