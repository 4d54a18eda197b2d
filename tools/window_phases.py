"""Host wall-clock phases of the product's window (GroupRetrainer.window) at a
bench config: the initial pass, every extension call (its depth, the chain
launch + batched member evaluation, the host replay in between), the join.

  python tools/window_phases.py [c2|c3|c4] [windows]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2512_11727_b200 as ecco  # noqa: E402
from paper_2512_11727_b200 import window as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wins = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = bench.Workload(cfg)


class Args:
    math = "bf16"


r = bench.make_retrainer(Args(), wl, 0, 1, None, 0)
log = []
orig_train = r.ctx.train_prepared
orig_alloc = W.allocate_trajectories


def timed_train(p, gpu_s, depth, window=0, micro_base=None, out=None):
    t = time.perf_counter()
    res = orig_train(p, gpu_s, depth, window=window, micro_base=micro_base, out=out)
    log.append(("train", depth, (time.perf_counter() - t) * 1e3))
    return res


def timed_alloc(*a, **k):
    t = time.perf_counter()
    res = orig_alloc(*a, **k)
    log.append(("replay", 0, (time.perf_counter() - t) * 1e3))
    return res


r.ctx.train_prepared = timed_train
W.allocate_trajectories = timed_alloc
out = []
for w in range(wins):
    log.clear()
    t = time.perf_counter()
    r.window(w + 1, reserve_sms=bench.RESERVE_SMS)
    r.ctx.synchronize()
    tot = (time.perf_counter() - t) * 1e3
    out.append({"window_ms": round(tot, 3),
                "train_calls": [(d, round(ms, 3)) for k, d, ms in log if k == "train"],
                "replay_ms": round(sum(ms for k, _, ms in log if k == "replay"), 3),
                "replays": sum(1 for k, _, _ in log if k == "replay"),
                "max_micro": int(r.stats["max_micro_windows"])})
print(json.dumps({"config": cfg, "windows": out}, indent=1))
