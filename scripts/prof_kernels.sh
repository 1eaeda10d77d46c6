#!/bin/bash
# ncu --set full of the numeric kernels (summaries on the box):
#   fem27 panel_numeric (mma.sync), fem27 tc05 (tcgen05), rmat esc_kernel
mkdir -p gpurun_out
timeout 600 python scripts/diag_rmat.py > gpurun_out/diag_rmat.log 2>&1
prof() {  # tag config regex env
  env $4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$3" -c 1 -o /tmp/p_$1 -f \
    python scripts/one_call.py $2 > gpurun_out/ncu_$1.log 2>&1
  python scripts/ncu_json.py /tmp/p_$1.ncu-rep gpurun_out/ncu_$1.json "ncu --set full --clock-control none, $3 of scripts/one_call.py $2 ($4)" > /dev/null 2>&1
  python scripts/ncu_summary.py /tmp/p_$1.ncu-rep > gpurun_out/top_$1.txt 2>&1
  sz=$(stat -c %s /tmp/p_$1.ncu-rep); [ "$sz" -lt 30000000 ] && cp /tmp/p_$1.ncu-rep gpurun_out/
}
prof r02_fem27_panel fem27 panel_numeric TSG_TC05=0
prof r02_fem27_tc05 fem27 tc05_panel TSG_TC05=1
prof r02_rmat_esc rmat esc_kernel TSG_TC05=0
