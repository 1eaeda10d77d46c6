cd /root/repo
: > gpurun_out/copy16_ab.log
for v in "-DTSG_ESC_COPY_U=8 -DTSG_COPY_U=8" "-DTSG_ESC_COPY_U=16 -DTSG_COPY_U=16"; do
  TSG_NVCC_FLAGS="$v" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/copy16_ab.log 2>&1
  echo "VARIANT $v" >> gpurun_out/copy16_ab.log
  timeout 600 python scripts/cfg_time.py rmat fem27 --reps 5 >> gpurun_out/copy16_ab.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/copy16_ab.log 2>&1
