"""The fused chain's latency regime in isolation: ONE group (20 members,
C4 shape F512-H256-C16, B = 128, 16 SGD steps per micro-window) trained
`depth` micro-windows in one ecco_train_trajectories call, as the exact
replay's extension chains run.  Prints the CUDA-event time per chain launch
and per call.  With an instrumented build (tools/chain_trace.py on) and
ECCO_CHAIN_TRACE=0 the per-phase clock64 trace of CTA 0 is printed too.

  python tools/single_chain.py [depth] [reps] [c4|c5] [tc|ffma]

c5: the detection-head shape F1024-H1024-C96 (the wide fused chain,
wide_kernels.cu; members evaluated on the general tensor-core path)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_11727_b200 as ecco  # noqa: E402


def main():
    depth = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    shape = sys.argv[3] if len(sys.argv) > 3 else "c4"
    math = ecco.FFMA_EXACT if len(sys.argv) > 4 and sys.argv[4] == "ffma" else ecco.TC_BF16
    dims = (dict(feat_dim=512, hidden_dim=256, num_classes=16) if shape == "c4" else
            dict(feat_dim=1024, hidden_dim=1024, num_classes=96))
    N, per = 400, 20
    ctx = ecco.Context(backend=ecco.LEARNED, math=math, max_cameras=N, max_jobs=4,
                       max_depth=64, steps_per_gpu_s=16.0, minibatch=128, ring_frames=512,
                       eval_samples=64, **dims)
    scenes = np.array([[0.1 * (c // per % 10), 0.1 * (c // per // 10)] for c in range(N)])
    ctx.set_cameras(scenes, np.full(N, 8.192e6))
    ctx.generate_frames(0)
    ctx.seed_models([0])
    mem = list(range(per))
    p = ctx.prepare_trajectories([0], [(30.0, 1080.0, 1.0)], [mem], [[1.0 / per] * per], [mem])
    acc = np.zeros((1, depth + 1))
    stream = torch.cuda.ExternalStream(ctx.stream)
    ctx.train_prepared(p, 1.0, depth, window=1, out=acc)
    ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
    for k in range(reps):
        ctx.train_prepared(p, 1.0, depth, window=2 + k, out=acc)
    with torch.cuda.stream(stream):
        e1.record(stream)
    e1.synchronize()
    n, ms, fl, by = ctx.kernel_stat(ecco.KSTAT_TRAIN_STEP)
    n2, ms2, _, _ = ctx.kernel_stat(ecco.KSTAT_EVAL_PAIRS)
    other = {k: ctx.kernel_stat(getattr(ecco, "KSTAT_" + k))[:2]
             for k in ("EVAL_MATRIX", "TRAIN_DW1", "TRAIN_HEAD")}
    print(json.dumps({"shape": shape, "math": "ffma" if math == ecco.FFMA_EXACT else "tc", "other_kernels": other, "depth": depth, "ms_per_call": e0.elapsed_time(e1) / reps,
                      "ms_per_micro_window": e0.elapsed_time(e1) / reps / depth,
                      "chain_launch_ms": ms / max(n, 1), "chain_launches": n,
                      "eval_launch_ms": ms2 / max(n2, 1), "us_per_sgd_step": ms / max(n, 1) / 16 * 1e3}))


if __name__ == "__main__":
    main()
