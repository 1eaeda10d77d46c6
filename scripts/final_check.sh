#!/bin/bash
# round-end evidence: GPU tests, smoke, the default bench line, FEM27's bench
# line and its light-pass ncu capture
cd /root/repo
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --config fem27 --no-cpu-baseline > gpurun_out/bench_fem27.log 2>&1
ONE_CALL_WARM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:panel_numeric -c 1 \
  -o /tmp/p_fem27 -f python scripts/one_call.py fem27 > gpurun_out/ncu_fem27.log 2>&1
python scripts/ncu_json.py /tmp/p_fem27.ncu-rep gpurun_out/ncu_r02_fem27_panel.json "ncu --set full --clock-control none, panel_numeric_kernel of scripts/one_call.py fem27 (warm)" > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/p_fem27.ncu-rep > gpurun_out/top_r02_fem27_panel.txt 2>&1
