"""A/B timing of the learned trajectories alone, for tuning:

  python tools/chain_bench.py [reps] [c4|c5]

c4 (default): the fused SGD chain at the C4 shape (500 groups x 20 members,
F512-H256-C16, B = 128, 2 micro-windows x 16 steps); prints the median / min
CUDA-event time of the chain kernel per launch (ECCO_KSTAT_TRAIN_STEP).
c5: the detection-head shape (F1024-H1024-C96) through the general
tensor-core path; prints the per-window time of every kernel family.
Both print the median SM clock sampled meanwhile."""
import os
import statistics
import subprocess
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2512_11727_b200 as ecco  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c4"
    dims = dict(bench.DIMS)
    if cfg == "c5":
        dims.update(bench.DET_DIMS)
    wl = bench.Workload(cfg, 0, 1)
    ctx = ecco.Context(backend=ecco.LEARNED, device=0, math=ecco.TC_BF16, max_cameras=wl.N,
                       max_jobs=len(wl.local), max_depth=bench.DEPTH,
                       steps_per_gpu_s=float(bench.STEPS), **dims)
    ctx.set_cameras(wl.scenes, wl.tp)
    ctx.generate_frames(0)
    ctx.seed_models(wl.local)
    prep = ctx.prepare_trajectories(
        wl.local, [bench.BATCH] * len(wl.local), [wl.members(g) for g in wl.local],
        [[1.0 / wl.per] * wl.per for _ in wl.local], [wl.members(g) for g in wl.local])
    acc = np.zeros((len(wl.local), bench.DEPTH + 1))
    for w in range(3):
        ctx.train_prepared(prep, bench.GPU_S, bench.DEPTH, window=w + 1, out=acc)
    clocks, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits",
                                  "-i", "0"], capture_output=True, text=True).stdout.strip()
            if out.isdigit():
                clocks.append(int(out))
            stop.wait(0.2)

    th = threading.Thread(target=sample)
    th.start()
    fams = ["TRAIN_STEP", "TRAIN_DW1", "TRAIN_HEAD", "EVAL_MATRIX", "EVAL_PAIRS"]
    per, fam = [], {f: [] for f in fams}
    for k in range(reps):
        ctx.profile(True)
        ctx.train_prepared(prep, bench.GPU_S, bench.DEPTH, window=10 + k, out=acc)
        n, ms = ctx.kernel_stat(ecco.KSTAT_TRAIN_STEP)[:2]
        for f in fams:
            fam[f].append(ctx.kernel_stat(getattr(ecco, "KSTAT_" + f))[1])
        ctx.profile(False)
        per.append(ms / max(n, 1))
    stop.set()
    th.join()
    clk = statistics.median(clocks) if clocks else 0
    if cfg == "c4":
        print(f"chain ms/launch: median {statistics.median(per):.4f} min {min(per):.4f} "
              f"(reps {reps}, sm clock median {clk} MHz)")
    else:
        parts = " ".join(f"{f} {statistics.median(v):.2f}" for f, v in fam.items())
        tot = statistics.median([sum(v[i] for v in fam.values()) for i in range(reps)])
        print(f"c5 ms/window: total {tot:.2f} | {parts} (reps {reps}, sm clock median {clk} MHz)")


if __name__ == "__main__":
    main()
