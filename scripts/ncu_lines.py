"""Per-source-line instruction counts: ncu SASS page x nvdisasm line info.

usage: python scripts/ncu_lines.py <report.ncu-rep> <kernel-substring> <object.o> [topN]
"""
import csv, re, subprocess, sys, tempfile, os, glob
from collections import Counter

rep, kname, obj = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-name", f"regex:{kname}"], capture_output=True, text=True).stdout
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
cub = glob.glob(os.path.join(d, "*.cubin"))[0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
lines, cur, infn = {}, None, False
for ln in dis.splitlines():
    if ln.startswith("//---------------------"):
        infn = kname in ln
    if not infn:
        continue
    m = re.search(r'line (\d+)', ln)
    if "//## File" in ln and m:
        cur = int(m.group(1))
    m2 = re.match(r'\s+/\*([0-9a-f]{4,})\*/', ln)
    if m2 and cur is not None:
        lines[int(m2.group(1), 16)] = cur
c, w = Counter(), Counter()
for a, (n, s) in execs.items():
    c[lines.get(a, -1)] += n
    w[lines.get(a, -1)] += s
tot, tw = sum(c.values()), max(1, sum(w.values()))
path = re.search(r'File "([^"]+)"', dis)
srcl = open(path.group(1)).read().splitlines() if path else []
for l, n in c.most_common(top):
    txt = srcl[l - 1].strip()[:70] if 0 < l <= len(srcl) else "?"
    print(f"{n:11d} {100*n/tot:5.1f}% stall {100*w[l]/tw:5.1f}%  L{l:4d} {txt}")
print("total", tot)
