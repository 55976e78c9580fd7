"""Summarise an ncu report (--page details --csv) per kernel: the metrics the
profiles/ tables quote. Usage: python tools/ncu_details.py report.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "DRAM Throughput",
        "Memory Throughput", "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction", "Issued Ipc Active",
        "Branch Efficiency", "Avg. Active Threads Per Warp", "L2 Hit Rate", "L1/TEX Hit Rate", "Local Memory Spilling"]

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
seen = {}
for r in rows:
    name = r["Kernel Name"].split("(")[0]
    if pat and not pat.search(name):
        continue
    key = (r["ID"], name)
    seen.setdefault(key, {})
    m = r["Metric Name"]
    if m in WANT and m not in seen[key]:
        seen[key][m] = f'{r["Metric Value"]} {r["Metric Unit"]}'.strip()
for (i, name), d in seen.items():
    print(f"[{i}] {name}")
    for m in WANT:
        if m in d:
            print(f"    {m:40s} {d[m]}")
