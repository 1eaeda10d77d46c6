cd /root/repo
mkdir -p gpurun_out
for p in 0 1 7; do
  ONE_CALL_WARM=1 ONE_CALL_PANEL=8,$p ONE_CALL_BSUM=8 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_bsum_rank$p.csv python scripts/one_call.py rmat > gpurun_out/launch_bsum_rank$p.log 2>&1
  python scripts/launches.py gpurun_out/launches_bsum_rank$p.csv > gpurun_out/launches_bsum_rank$p.txt 2>&1
done
