"""Stall-sample shares of a kernel's SASS from an ncu report: by subroutine
(regions ending in RET) and the hottest instructions.
Usage: python tools/ncu_sass_hot.py report.ncu-rep kernel_name [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source", "sass",
                      "--launch-count", "1"] + (["--kernel-name-base", "demangled"] if False else []), capture_output=True, text=True).stdout
lines = out.splitlines()
i = next(j for j, l in enumerate(lines) if l.startswith('"Address"'))
rows = [r for r in csv.DictReader(io.StringIO("\n".join(lines[i:]))) if r.get("Address", "").startswith("0x")]
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[S] or 0) for r in rows)
print(f"{kern}: {len(rows)} SASS instructions, {tot:.0f} stall samples")
# regions: split after RET / EXIT-terminated subroutines
regs, cur, start = [], 0.0, 0
for j, r in enumerate(rows):
    cur += float(r[S] or 0)
    if "RET" in r["Source"].split()[0:2] or j == len(rows) - 1:
        regs.append((start, j, cur))
        cur, start = 0.0, j + 1
print("regions (instruction index range, share):")
for a, b, s in regs:
    print(f"  [{a:5d}-{b:5d}] {100 * s / tot:5.1f}%  first: {rows[a]['Source'].strip()[:60]}")
hot = sorted(range(len(rows)), key=lambda j: -float(rows[j][S] or 0))[:top]
print("hottest instructions:")
for j in hot:
    r = rows[j]
    print(f"  {j:5d} {100 * float(r[S] or 0) / tot:5.2f}%  thr {r['Avg. Threads Executed']:>5s}  {r['Source'].strip()[:70]}")
