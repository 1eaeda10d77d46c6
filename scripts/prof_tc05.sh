#!/bin/bash
mkdir -p gpurun_out
timeout 900 python scripts/emulate_ranks.py rmat fem27 amg > gpurun_out/emulated_ranks.md 2>&1
ONE_CALL_WARM=1 TSG_TC05=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc05 -c 1 -o /tmp/p_tc05 -f \
    python scripts/one_call.py fem27 > gpurun_out/ncu_r02_fem27_tc05.log 2>&1
python scripts/ncu_json.py /tmp/p_tc05.ncu-rep gpurun_out/ncu_r02_fem27_tc05.json "ncu --set full --clock-control none, tc05_panel_kernel of scripts/one_call.py fem27 (TSG_TC05=1, second call)" > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/p_tc05.ncu-rep > gpurun_out/top_r02_fem27_tc05.txt 2>&1
cp /tmp/p_tc05.ncu-rep gpurun_out/p_r02_fem27_tc05.ncu-rep
