"""Parametric window driver vs the unmodified reference library at a
BASELINE config (default c4): per-window wall time (GPU driver: total,
regroup, train, replay) and the reference's Simulation::step_window, plus
trace identity.  Usage: python tools/param_window_probe.py [c4] [windows]"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2512_11727_b200 as ecco  # noqa: E402
from paper_2512_11727_b200 import scenarios  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
wins = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sc = json.dumps(scenarios.config(cfg, windows=wins, seed=1))
sim = ecco.Simulation(sc, backend=ecco.PARAMETRIC)
out = {"config": cfg, "windows": wins, "gpu": []}
while True:
    t = time.perf_counter()
    if not sim.step_window():
        break
    d = sim.last_timings()
    d["wall_ms"] = (time.perf_counter() - t) * 1e3
    out["gpu"].append(d)
gpu_trace = sim.trace_csv()
sim.close()
R = oracle.ref()
ref_s = np.zeros(16)
n = C.c_int()
R.ref_time_windows(sc.encode(), 16, ref_s, C.byref(n))
out["reference_window_ms"] = [x * 1e3 for x in ref_s[:n.value]]
tcap = 1 << 28
tb, sb = C.create_string_buffer(tcap), C.create_string_buffer(1 << 20)
tl, sl = C.c_size_t(), C.c_size_t()
R.ref_run_scenario(sc.encode(), -1, tb, tcap, C.byref(tl), sb, 1 << 20, C.byref(sl))
out["trace_identical"] = gpu_trace == tb.raw[:tl.value].decode()
out["trace_bytes"] = len(gpu_trace)
print(json.dumps(out, indent=1))
