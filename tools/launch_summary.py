"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
reps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.reader(open(path)))
start = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[start]
iN, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[start + 1:]:
    n = r[iN].split("(")[0][:60]
    tot[n] += float(r[iV].replace(",", ""))
    cnt[n] += 1
T = sum(tot.values()) / reps / 1e6
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
    print(f"{k:60s} {cnt[k]:4d} {v / 1e6 / reps:9.3f} ms/step {100 * v / 1e6 / reps / T:5.1f}%")
print(f"{'total':60s}      {T:9.3f} ms/step")
