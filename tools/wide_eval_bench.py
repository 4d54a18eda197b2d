"""Times the fused evaluation at the detection-head shape (k_eval_wide):
the dense camera x group matrix (ecco_eval_matrix_dev) of N cameras x G
groups, CUDA events on the context stream, and the member evaluations of
one serial-chain call (pairs mode: every snapshot on its group's members).

    python tools/wide_eval_bench.py [N G reps]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_11727_b200 as ecco  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
G = int(sys.argv[2]) if len(sys.argv) > 2 else 64
REPS = int(sys.argv[3]) if len(sys.argv) > 3 else 3
F, H, C, S = 1024, 1024, 96, 64

ctx = ecco.Context(backend=ecco.LEARNED, math=ecco.TC_BF16, max_cameras=N, max_jobs=G, max_depth=2,
                   feat_dim=F, hidden_dim=H, num_classes=C, minibatch=128, ring_frames=64,
                   eval_samples=S)
rng = np.random.default_rng(0)
ctx.set_cameras(np.round(rng.random((N, 2)), 1), np.full(N, 8.192e6))
ctx.generate_frames(1)
ids = list(range(G))
ctx.seed_models(ids)
out = torch.empty((N, G), dtype=torch.float64, device="cuda")
cams = np.arange(N, dtype=np.int32)
st = torch.cuda.ExternalStream(ctx.stream)
ctx.eval_matrix_dev(ids, out.data_ptr(), cams=cams)  # warm-up (shadows, attributes)
ctx.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ctx.profile(True)
with torch.cuda.stream(st):
    e0.record(st)
for _ in range(REPS):
    ctx.eval_matrix_dev(ids, out.data_ptr(), cams=cams)
with torch.cuda.stream(st):
    e1.record(st)
ctx.synchronize()
ms = e0.elapsed_time(e1) / REPS
kst = ctx.kernel_stat(ecco.KSTAT_EVAL_MATRIX)
ctx.profile(False)
flops = 2.0 * N * G * S * (F * H + H * C)
res = {"N": N, "G": G, "ms_per_matrix": ms, "tflops": flops / ms / 1e9,
       "kernel": {"launches": kst[0], "ms": kst[1], "tflops": kst[2] / kst[1] / 1e9 if kst[1] else None},
       "sm_clock_note": "CUDA events on the context stream, after one warm-up call"}
# pairs mode: 20-member groups, every camera under its own group (the
# member evaluations of one micro-window of every group)
members = [list(range((g * 20) % N, (g * 20) % N + 20)) for g in range(min(G, N // 20))]
jj = ids[:len(members)]
ctx.eval_jobs(jj, members)
ctx.synchronize()
t = time.perf_counter()
for _ in range(REPS):
    ctx.eval_jobs(jj, members)
ctx.synchronize()
pms = (time.perf_counter() - t) * 1e3 / REPS
pflops = 2.0 * sum(len(m) for m in members) * S * (F * H + H * C)
res["pairs"] = {"groups": len(members), "ms_wall": pms, "tflops_wall": pflops / pms / 1e9}
print(json.dumps(res))
