cd /root/repo
: > gpurun_out/kb_ab.log
for kb in 4 5 6; do
  TSG_NVCC_FLAGS="-DTSG_PANEL_KB=$kb" python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/kb_ab.log 2>&1
  echo "PANEL_KB=$kb" >> gpurun_out/kb_ab.log
  timeout 600 python scripts/cfg_time.py fem27 poisson amg --reps 7 >> gpurun_out/kb_ab.log 2>&1
done
python -c "from paper_2009_14600_b200 import _build; _build.build(force=True)" >> gpurun_out/kb_ab.log 2>&1
