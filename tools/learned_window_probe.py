"""The whole-window driver (Simulation::step_window) with the LEARNED backend
at a BASELINE config: per-window timings (regroup, train, netsim, ...) and
samples trained.  Usage: python tools/learned_window_probe.py [c4] [windows]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_11727_b200 as ecco  # noqa: E402
from paper_2512_11727_b200 import scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
wins = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spg = float(sys.argv[3]) if len(sys.argv) > 3 else 16.0 / 0.06
spec = int(sys.argv[4]) if len(sys.argv) > 4 else 2
sc = scenarios.config(cfg, windows=wins, seed=1, local_acc=0.0)  # fresh learned models join
sim = ecco.Simulation(json.dumps(sc), backend=ecco.LEARNED, math=ecco.TC_BF16, full_matrix=1,
                      steps_per_gpu_s=spg, spec_depth=spec)
out = {"config": cfg, "windows": wins, "steps_per_gpu_s": spg, "spec_depth": spec, "gpu": []}
while True:
    t = time.perf_counter()
    if not sim.step_window():
        break
    d = {k: round(v, 3) for k, v in sim.last_timings().items()}
    d["wall_ms"] = round((time.perf_counter() - t) * 1e3, 3)
    d["samples"] = sim.last_samples()
    out["gpu"].append(d)
summ = json.loads(sim.summary_json())
out["summary_keys"] = list(summ)[:12]
print(json.dumps(out, indent=1))
