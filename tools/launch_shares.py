"""Per-kernel launch counts, total time and share of an ncu launch list
(--metrics gpu__time_duration.sum --csv).  Usage:
python tools/launch_shares.py launches.csv "header comment" > profiles/X.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[iu], 1e-6)
    k = r[ik].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
    agg[k][0] += 1
    agg[k][1] += float(r[iv].replace(",", "")) * scale
tot = sum(v[1] for v in agg.values())
if len(sys.argv) > 2:
    print("#", sys.argv[2])
print("# (per-launch times are cold-cache and serialised: compare SHARES)")
print("# kernel, launches, total ms, share")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {v[0]:5d} {v[1]:10.3f} {100 * v[1] / tot:6.2f}%")
