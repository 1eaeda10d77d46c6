"""Per-call diagnostics on the GPU: phase times, counters and wall time of
single spGEMM calls for a config (each chain stage separately)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2009_14600_b200 import workloads as W  # noqa: E402
from paper_2009_14600_b200.tilemul import Context  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "amg"
ctx = Context(device=0)
mats = [M.to_device("cuda") for M in W.make(cfg)]
if len(mats) == 1:
    stages = [(mats[0], mats[0])]
elif len(mats) == 2:
    stages = [(mats[0], mats[1])]
else:
    RA = ctx.spgemm(mats[0], mats[1], out="device").C
    stages = [(mats[0], mats[1]), (RA, mats[2])]
for i, (A, B) in enumerate(stages):
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ctx.spgemm(A, B, out="device", phase_timing=True)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
    ph = {k: round(ctx.last_phase_ms(k), 3) for k in
          ("convert", "task_list", "sort", "counting", "multiply", "compaction", "total", "numeric_kernel", "assemble_kernel")}
    st = {k: r.stats[k] for k in ("tiles_a", "tiles_b", "raw_pairs", "filtered_pairs", "segments", "counted_elements", "nnz_c")}
    print(json.dumps({"config": cfg, "stage": i, "wall_ms": round(wall, 3), "phase_ms": ph, "stats": st}), flush=True)

if len(mats) == 3:
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ctx.spgemm_chain(mats, out="device", phase_timing=True)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        st = r.stats
        print(json.dumps({"config": cfg, "chain_rep": rep, "wall_ms": round(wall, 3),
                          "multiply_s": st["multiply"], "total_s": st["total"],
                          "numeric_kernel_last": ctx.last_phase_ms("numeric_kernel")}), flush=True)
