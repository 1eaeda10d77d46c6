"""Summarise an ncu --set full report as JSON (profiles/rNN_ncu_full_*.json):
per kernel launch -- duration, DRAM bytes (the roofline `traffic` source),
instructions, occupancy, issue, L1/L2 hit rates, tensor-pipe activity.

usage: python scripts/ncu_json.py <report.ncu-rep> <out.json> "<source text>"
"""
import csv
import json
import re
import subprocess
import sys

rep, out, source = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h, units = rows[0], rows[1]
keys = {
    "duration_us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "inst_executed": ("smsp__inst_executed.sum", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "l1tex_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
}
scale_bytes = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
res = {"source": source, "kernels": {}}
for v in rows[2:]:
    name = v[h.index("Kernel Name")]
    name = name.split("(")[0].replace("void ", "").replace("tsg::<unnamed>::", "").replace("<unnamed>::", "").strip()
    name = name.replace("unnamed>::", "").replace("tsg::", "")
    if name.startswith("cub::"):
        name = name.split("<")[0]
    d = {}
    for k, (m, sc) in keys.items():
        if m not in h:
            continue
        i = h.index(m)
        try:
            x = float(v[i].replace(",", ""))
        except ValueError:
            continue
        if sc is None:
            x *= scale_bytes.get(units[i], 1)
        elif units[i] == "ns" and k == "duration_us":
            x *= 1e-3
        elif units[i] == "us" and k == "duration_us":
            pass
        elif units[i] == "ms" and k == "duration_us":
            x *= 1e3
        d[k] = round(x, 3)
    if name in res["kernels"]:
        n = 2
        while f"{name}#{n}" in res["kernels"]:
            n += 1
        name = f"{name}#{n}"
    res["kernels"][name] = d
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
