"""Summarise an ncu report (run here, no GPU): key metrics + SASS opcode mix."""
import csv, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units, vals = rows[0], rows[1], rows[2:]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sectors_srcunit_tex_op_read.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]
for v in vals:
    for k in keys:
        if k in h:
            i = h.index(k)
            print(f"  {k:70s} {v[i]} {units[i]}")
    print()
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(src.splitlines()))
if len(r) > 2:
    hh = r[1]
    ia, isrc, iw = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
    c, w = Counter(), Counter()
    for x in r[2:]:
        if len(x) <= ia or not x[ia]:
            continue
        op = x[isrc].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        o = o.split(".")[0]
        c[o] += int(float(x[ia]))
        w[o] += int(float(x[iw] or 0))
    tot, tw = sum(c.values()), max(1, sum(w.values()))
    print("  opcode mix (inst share / stall-sample share):")
    for o, n in c.most_common(16):
        print(f"    {o:10s} {n:12d} {100*n/tot:5.1f}%  {100*w[o]/tw:5.1f}%")
