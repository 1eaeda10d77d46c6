"""Per-source-line instruction counts: ncu SASS page x nvdisasm line info.

usage: python scripts/ncu_lines.py <report.ncu-rep> <kernel-substring> <object.o> [topN]
"""
import csv, re, subprocess, sys, tempfile, os, glob
from collections import Counter

rep, kname, obj = sys.argv[1], sys.argv[2], sys.argv[3]
# "ncu-regex::mangled-substring" when the two names differ (template kernels)
kname, dname = (kname.split("::", 1) + [None])[:2] if "::" in kname else (kname, kname)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
# match on the mangled name so one template instance is selected
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name-base", "mangled", "--kernel-name", f"regex:{dname}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
ia, iaddr, iw = h.index("Instructions Executed"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
execs = {}
base = None
for r in rows[2:]:
    if len(r) > ia and r[ia] and r[ia] != "Instructions Executed":
        a = int(r[iaddr], 16)
        base = a if base is None else base
        execs[a - base] = (int(float(r[ia])), int(float(r[iw] or 0)))
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
dis = ""
for cub in sorted(glob.glob(os.path.join(d, "*.cubin"))):  # the cubin holding the kernel
    dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    if dname in dis:
        break
lines, cur, infn = {}, None, False
for ln in dis.splitlines():
    if ln.startswith("//---------------------"):
        infn = dname in ln
    if not infn:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if "//## File" in ln and m:
        cur = (m.group(1), int(m.group(2)))
    m2 = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m2 and cur is not None:
        lines[int(m2.group(1), 16)] = cur
c, w = Counter(), Counter()
for a, (n, s) in execs.items():
    c[lines.get(a, -1)] += n
    w[lines.get(a, -1)] += s
tot, tw = sum(c.values()), max(1, sum(w.values()))
srcs = {}
for l, n in c.most_common(top):
    txt, tag = "?", "?"
    if l != -1:
        f, ln_ = l
        if f not in srcs:
            srcs[f] = open(f).read().splitlines() if os.path.exists(f) else []
        txt = srcs[f][ln_ - 1].strip()[:64] if 0 < ln_ <= len(srcs[f]) else "?"
        tag = f"{os.path.basename(f)[:14]}:{ln_}"
    print(f"{n:11d} {100*n/tot:5.1f}% stall {100*w[l]/tw:5.1f}%  {tag:20s} {txt}")
print("total", tot)
