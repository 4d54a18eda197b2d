"""Summarise an ncu report's SASS source page: top stalled instructions and
samples per 'region' (split at BAR.SYNC / barrier waits).  Usage:
python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = rows[2:]
iS, iW, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[iW] or 0) for r in data)
print("total samples", tot)
for k, r in enumerate(data):
    r.append(k)
for r in sorted(data, key=lambda r: -float(r[iW] or 0))[:n]:
    print(f"{r[-1]:5d} {float(r[iW]):9.0f} {100*float(r[iW])/tot:5.1f}% {r[iE]:>10s}  {r[iS][:90]}")
# regions between BAR.SYNC
print("--- samples between BAR.SYNC boundaries")
acc, start = 0.0, 0
for k, r in enumerate(data):
    acc += float(r[iW] or 0)
    if "BAR.SYNC" in r[iS] or k == len(data) - 1:
        if acc > 0.01 * tot:
            print(f"lines {start:5d}-{k:5d}: {100*acc/tot:5.1f}%")
        acc, start = 0.0, k + 1
