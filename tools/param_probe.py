"""The parametric backend's kernels at C4 size, one launch family at a time,
for ncu captures and CUDA-event timing (K1 k_p_eval_matrix, K2
k_p_trajectories, K3 k_p_profile):

  python tools/param_probe.py [k1|k2|k3|all] [reps]

K1: 10,000 scenes x 500 models (K = 3 clusters, D = 2), as bench.py's
parametric leg.  K2: 500 jobs' speculative chains (depth 4, 20 sources
each).  K3: 1,000 cameras' profile tables (1,000 budget levels x 20 configs,
the C4 window-0 grid on a tenth of the cameras).  Prints the mean CUDA-event
time per launch and the FP64 instruction-level work estimate."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_11727_b200 as ecco  # noqa: E402


def timed(ctx, fn, reps):
    stream = torch.cuda.ExternalStream(ctx.stream)
    fn()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
    for _ in range(reps):
        fn()
    with torch.cuda.stream(stream):
        e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    rng = np.random.default_rng(7)
    out = {}
    N, G, K, D = 10000, 500, 3, 2
    scenes = np.round(rng.random((N, D)), 2)
    ctx = ecco.Context(backend=ecco.PARAMETRIC, max_jobs=G, max_cameras=N, max_clusters=8,
                       max_depth=8)
    ctx.set_cameras(scenes, np.full(N, 8.192e6))
    ids = list(range(G))
    cl = np.zeros((G, 8, D))
    cl[:, :K] = np.round(rng.random((G, K, D)), 2)
    pr = np.zeros((G, 8))
    pr[:, :K] = rng.random((G, K))
    ctx.put_models(ids, np.full(G, K, np.int32), cl.reshape(G, -1), pr, cl[:, :K].mean(1),
                   np.full(G, D, np.int32))
    if which in ("k1", "all"):
        dM = torch.empty((N, G), dtype=torch.float64, device="cuda")
        ms = timed(ctx, lambda: ctx.eval_matrix_dev(ids, dM.data_ptr(), scenes=scenes), reps)
        out["k1_eval_matrix"] = {"pairs": N * G, "ms": ms, "out_bytes": N * G * 8,
                                 "hbm_gbs_on_output": N * G * 8 / ms / 1e6}
    if which in ("k2", "all"):
        per = N // G
        # every job's members share one cluster scene (C4 layout): train_step
        # finds / adds one cluster per distinct scene
        ctx2 = ecco.Context(backend=ecco.PARAMETRIC, max_jobs=G, max_cameras=N, max_clusters=8,
                            max_depth=8)
        sc2 = np.repeat(np.round(rng.random((G, D)), 2), per, axis=0)
        ctx2.set_cameras(sc2, np.full(N, 8.192e6))
        ctx2.seed_models(ids, scenes=sc2[::per], device_acc=np.full(G, 0.2))
        members = [list(range(g * per, (g + 1) * per)) for g in ids]
        fr = [[1.0 / per] * per for _ in ids]
        p = ctx2.prepare_trajectories(ids, [(15.0 * per, 720.0, 1.0)] * G, members, fr, members)
        acc = np.zeros((G, 5))
        ms = timed(ctx2, lambda: ctx2.train_prepared(p, 0.06, 4, out=acc), reps)
        out["k2_trajectories"] = {"jobs": G, "depth": 4, "sources": per, "ms_per_call": ms}
    if which in ("k3", "all"):
        n = 1000
        levels = np.arange(1, 1001) * 0.06
        fps = np.repeat([1.0, 2.0, 5.0, 10.0, 15.0], 4)
        res = np.tile([360.0, 480.0, 720.0, 960.0], 5)
        cams = np.arange(n, dtype=np.int32)
        ms = timed(ctx, lambda: ctx.profile_tables(cams, levels, fps, res, 60.0), reps)
        out["k3_profile"] = {"cameras": n, "levels": len(levels), "grid": len(fps),
                             "probe_slots": n * len(levels) * len(fps), "ms_per_call": ms}
    ctx.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
