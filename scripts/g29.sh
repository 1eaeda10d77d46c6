cd /root/repo
VARIANTS='-DTSG_ESC_R8=0 -DTSG_ESC_R8=1 -DTSG_ESC_R8=1@-DTSG_ESC_ROT=0' 
mkdir -p gpurun_out; : > gpurun_out/esc_ab2.log
for v in "-DTSG_ESC_R8=0" "-DTSG_ESC_R8=1" "-DTSG_ESC_R8=1 -DTSG_ESC_ROT=0"; do
  TSG_NVCC_FLAGS="$v" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esc_ab2.log 2>&1
  echo "VARIANT $v" >> gpurun_out/esc_ab2.log
  timeout 600 python scripts/cfg_time.py rmat rect --reps 5 >> gpurun_out/esc_ab2.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/esc_ab2.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "rmat or rect or general or r02 or counters or corpus" > gpurun_out/pytest_g29.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_g29.log
