"""Per-kernel device times from an ncu launch-list CSV (gpu__time_duration.sum)."""
import csv, re, sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 14 and r[0].isdigit()]
    tot = 0.0
    print(f)
    for r in rows:
        n = re.sub(r"\(.*", "", r[4]).replace("void ", "").replace("tsg::<unnamed>::", "")[:60]
        t = float(r[14]) / 1000
        tot += t
        print(f"  {n:60s} {t:8.1f}")
    print("  total", round(tot, 1))
