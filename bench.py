"""Benchmark of the B200 group-retraining path (BASELINE.json `metric`:
group-retrain samples/s and regroup latency per window).

One step = one retraining window of the hot path over the workload's
synthetic camera streams, through the product's group-sharded window
(paper_2512_11727_b200/window.py):

  regroup   the camera x group evaluation matrix -- every camera's S labelled
            eval frames scored under every group model (ecco_eval_matrix_dev,
            the ModelEvalFn batch of grouping.cpp:33) -- all-gathered across
            ranks, then the warp-reduced argmax/threshold per camera
            (ecco_route_matrix_ids_dev, group_request's join rule);
  retrain   every group's speculative chain of DEPTH micro-windows x STEPS SGD
            steps of B sampled frames (ecco_train_trajectories, the
            allocator's TrainingBackend probes of gpu_allocator.cpp:125-135),
            the trajectories all-gathered, the reference's greedy
            (WindowAllocation, ecco_allocate_trajectories) replayed over every
            group with W = W_PER_GROUP x G micro-windows -- chains the greedy
            exhausts are committed and extended (exact replay, no frozen
            accuracies) -- and each group's granted prefix committed.

Keys: `value` = COMMITTED samples (granted micro-windows x steps x B) of the
whole window / max-over-ranks device time of the window (regroup + retrain),
the north star's "per-window regroup+retrain"; `retrain_samples_per_s` =
the same samples / train-phase time; `regroup_ms_per_window`
= regroup latency.  `e2e` = the same window through the public API with the
frames ingested from pinned host memory every window and the assignments /
accuracies read back, phase by phase.  Groups are placed on ranks by cost
(shard.Placement); cameras are replicated (frames regenerated per rank).

`--impl reference` times the CPU restatement of the same train phase
(oracle/, the reference itself has no learned trainer: SURVEY.md 0) on this
box's cores.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# BASELINE.json configs -> (cameras, groups)
CONFIGS = {
    "c2": (100, 10),
    "c3": (1000, 50),
    "c4": (10000, 500),
    "c5": (10000, 500),  # detection head (DET_DIMS), allocator marginal-gain probes only
}
DIMS = dict(feat_dim=512, hidden_dim=256, num_classes=16, minibatch=128, ring_frames=512,
            eval_samples=64)
W_PER_GROUP = 2       # allocator budget W = 2 x groups micro-windows (C4: W = 1000)
DEPTH = 1             # speculative chain every group trains up front: the initial pass.  The
                      # ECCO greedy's fairness bonus goes to the minimum-accuracy group, which on
                      # these streams absorbs most of the remaining budget; its chain is extended
                      # by depth doubling (window.py), the other groups' chains are never wasted
MAX_DEPTH = 64        # deepest extension chain (snapshots: groups x MAX_DEPTH x params in HBM)
RESERVE_SMS = int(os.environ.get("ECCO_RESERVE_SMS", "12"))  # SMs the overlapped
# regroup matrix leaves to the serial extension chains (and the e2e ingest's fetch CTAs)
STEPS = 16            # SGD steps per micro-window
# configs[4]: the detection-head variant (larger per-group model and frame
# features).  Its window is the allocator's marginal-gain probing (every
# group's speculative chain + member evaluations, as configs[4] states); the
# full camera x group matrix at this shape (k_eval_wide, 7.3e14 FLOP) is
# timed beside it as the line's `regroup_matrix` leg.
DET_DIMS = dict(feat_dim=1024, hidden_dim=1024, num_classes=96)
MATRIX = True         # the regroup matrix is part of the step (False for c5)
GPU_S = 1.0           # GPU-seconds per micro-window; steps = floor(GPU_S * STEPS)
BATCH = (30.0, 1080.0, 1.0)  # delivered fps, resolution, quality: sufficiency 1
THROUGHPUT = 8.192e6  # CameraState.gpu_pixel_throughput default


def flops_per_sample(F, H, C):
    """fwd + bwd of the F->H->C MLP per training sample."""
    return 4.0 * F * H + 6.0 * H * C


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _red_device():
    import torch
    nccl = os.environ.get("ECCO_DIST_BACKEND", "nccl") == "nccl"
    return torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")


def reduce_max(dist, values):
    """Max over ranks (device times: the slowest rank bounds the job)."""
    if dist is None:
        return list(values)
    import torch
    t = torch.tensor(values, dtype=torch.float64, device=_red_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def reduce_sum(dist, value):
    if dist is None:
        return value
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=_red_device())
    dist.all_reduce(t)
    return t.item()


# ------------------------------------------------------------------ workload --

class Workload:
    """Cameras and groups of a config: group g = cameras [g*per, (g+1)*per)
    (one spatial cluster, scenes on a 0.1 grid per cluster)."""

    def __init__(self, config):
        self.config = config
        self.N, self.G = CONFIGS[config]
        self.per = self.N // self.G
        side = 10
        self.scenes = np.array([[0.1 * ((c // self.per) % side), 0.1 * ((c // self.per // side) % side)]
                                for c in range(self.N)], np.float64)
        self.tp = np.full(self.N, THROUGHPUT)
        self.groups = [list(range(g * self.per, (g + 1) * self.per)) for g in range(self.G)]

    def members(self, g):
        return self.groups[g]


def make_retrainer(args, wl, rank, world, dist, device, emulate=False):
    import paper_2512_11727_b200 as ecco
    from paper_2512_11727_b200.window import GroupRetrainer
    math = ecco.FFMA_EXACT if args.math == "ffma" else ecco.TC_BF16
    cls = EmulatedRank0 if emulate else GroupRetrainer
    return cls(wl.scenes, wl.tp, wl.groups, rank=rank, world=world, dist=dist, device=device,
               math=math, depth=DEPTH, gpu_s=GPU_S, batch=BATCH, steps_per_gpu_s=float(STEPS),
               micro_windows=W_PER_GROUP * wl.G, max_depth=MAX_DEPTH, dims=DIMS)


# ----------------------------------------------------------------- B200 arm --

def run_b200(args, rank, world, local_rank):
    import torch
    import paper_2512_11727_b200 as ecco

    # ECCO_DIST_BACKEND=gloo (testing only) runs N ranks on however many GPUs
    # the box has, gathering through host memory; the product path is NCCL
    backend = os.environ.get("ECCO_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    wl = Workload(args.config)
    retr = make_retrainer(args, wl, rank, world, dist, local_rank)
    ctx, stream = retr.ctx, retr.stream
    ev = {k: torch.cuda.Event(enable_timing=True) for k in ("a", "b", "c")}
    acc = {"regroup": 0.0, "retrain": 0.0, "committed": 0, "speculative": 0, "extensions": 0,
           "max_micro": 0}

    def mark_b():
        with torch.cuda.stream(stream):
            ev["b"].record(stream)

    def step(w, timed=False, mid=None):
        # the window in the reference's order -- retrain, then the window-end
        # regroup over the trained models -- with the regroup matrix of the
        # groups the greedy leaves alone overlapped with its serial extension
        # chains (GroupRetrainer.window); "retrain" = start -> the schedule
        # committed, "regroup" = -> the join rule done (what the window still
        # waits for after the retrain)
        if timed:
            with torch.cuda.stream(stream):
                ev["a"].record(stream)
        if MATRIX:
            retr.window(w, mid=mid, reserve_sms=RESERVE_SMS, mark=mark_b if timed else None)
        else:
            retr.retrain(w, mid=mid)
            if timed:
                mark_b()
        if timed:
            with torch.cuda.stream(stream):
                ev["c"].record(stream)
            ev["c"].synchronize()
            acc["retrain"] += ev["a"].elapsed_time(ev["b"])
            acc["regroup"] += ev["b"].elapsed_time(ev["c"])
            acc["committed"] += retr.stats["committed_samples"]
            acc["speculative"] += retr.stats["speculative_samples"]
            acc["extensions"] += retr.stats["extensions"]
            acc["max_micro"] = max(acc["max_micro"], retr.stats["max_micro_windows"])

    def barrier():
        torch.cuda.synchronize()
        ctx.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for w in range(args.warmup):
        step(w + 1)
    barrier()
    clocks = Clocks(local_rank)
    clocks.start()
    ctx.profile(True)
    l0 = ctx.launches
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        t0.record(stream)
    for k in range(args.steps):
        step(args.warmup + 1 + k, timed=True)
    with torch.cuda.stream(stream):
        t1.record(stream)
    barrier()
    launches = ctx.launches - l0
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    # ECCO_KSTAT_TRAIN_STEP is the fused SGD chain where it applies
    # (train_kernels.cu: tensor-core math, B = 128, C = 16, F a power of two
    # <= 512, H = 256 / 512; wide_kernels.cu: the detection head F = 1024,
    # C = 96, H = 512 / 1024), else the unfused forward; DW1 / HEAD are the
    # unfused tensor-core / FFMA kernels (other shapes, --math ffma)
    F, H = DIMS["feat_dim"], DIMS["hidden_dim"]
    chain = (args.math != "ffma" and DIMS["minibatch"] == 128 and
             ((DIMS["num_classes"] == 16 and F <= 512 and F % 128 == 0 and F & (F - 1) == 0
               and H in (256, 512)) or
              (DIMS["num_classes"] == 96 and F == 1024 and H in (512, 1024))))
    kst = {name: ctx.kernel_stat(getattr(ecco, "KSTAT_" + stat)) for name, stat in
           (("EVAL_MATRIX", "EVAL_MATRIX"), ("EVAL_PAIRS", "EVAL_PAIRS"),
            ("TRAIN_CHAIN" if chain else "TRAIN_FWD", "TRAIN_STEP"), ("TRAIN_DW1", "TRAIN_DW1"),
            ("TRAIN_HEAD", "TRAIN_HEAD"))}
    ctx.profile(False)
    ms, regroup_ms, retrain_ms = reduce_max(dist, [ms, acc["regroup"], acc["retrain"]])
    samples = acc["committed"]  # every rank replays the same schedule: already global
    probes = None
    if not args.no_probes:
        try:
            probes = probe_leg(retr, torch, dist)
        except Exception as e:  # reported, never fatal for the headline line
            probes = {"error": repr(e)}
    regroup = None
    if not MATRIX and not args.no_regroup:
        try:
            regroup = regroup_leg(retr, torch, dist, peaks()[0])
        except Exception as e:  # reported, never fatal for the headline line
            regroup = {"error": repr(e)}
    parity = None
    if not args.no_parity:
        try:
            parity = parity_spot_check(args, retr, wl)
        except Exception as e:  # reported, never fatal for the headline line
            parity = {"error": repr(e)}

    # ---- e2e: same window through the public API, frames from pinned host memory
    e2e = None if args.no_e2e else run_e2e(args, retr, wl, torch, dist)

    if rank == 0:
        pk, pk_kind = peaks()
        roof = roofline(kst, pk, pk_kind, args, fused=chain, window_ms=ms)
        steps = args.steps
        line = {
            "metric": "group-retrain samples/s (per-window regroup + retrain)",
            "value": samples / (ms / 1e3),
            "unit": "samples/s",
            "retrain_samples_per_s": samples / (retrain_ms / 1e3),
            "regroup_ms_per_window": regroup_ms / steps,
            "retrain_ms_per_window": retrain_ms / steps,
            "n_gpus": world,
            "steps": steps,
            "warmup": args.warmup,
            "ms_per_step": ms / steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            # operand type of the tensor-core contractions (fp32 accumulation
            # and fp32 masters throughout): the fused chain and the evaluation
            # kernels run kind::f16 bf16; shapes outside the chain train with
            # a bf16 forward and a tf32 dW1; --math ffma is fp32 on CUDA cores
            "dtype": ("f32" if args.math == "ffma" else "bf16" if chain
                      else "bf16+tf32" if DIMS["minibatch"] % 128 == 0 and H % 256 == 0 else "tf32"),
            "data": "synthetic (counter-RNG camera streams, random-init group MLPs)",
            "config": {
                "workload": f"{args.config}: {wl.N} cameras / {wl.G} groups, learned classifier "
                            f"F{DIMS['feat_dim']}-H{DIMS['hidden_dim']}-C{DIMS['num_classes']}, "
                            f"B={DIMS['minibatch']}, S={DIMS['eval_samples']} eval frames/camera, "
                            f"R={DIMS['ring_frames']} ring frames/camera, {STEPS} SGD steps per "
                            f"micro-window, W = {W_PER_GROUP} x groups micro-windows (ECCO policy, "
                            f"exact replay: speculative depth {DEPTH}, extensions up to {MAX_DEPTH}), "
                            + ("full camera x group matrix" if MATRIX else
                               "marginal-gain probes only (no regroup matrix)"),
                "cameras": wl.N, "groups": wl.G, "groups_per_rank": len(retr.local),
                "parallelism": f"groups placed on {world} rank(s) by cost; eval matrix + "
                               "trajectory all-gather",
                "l2": "inputs larger than L2 (frames "
                      f"{wl.N * (DIMS['ring_frames'] + DIMS['eval_samples']) * DIMS['feat_dim'] * 2 / 2**30:.1f} GiB)",
            },
            "samples": {"committed_per_window": samples / steps,
                        "speculative_per_window": acc["speculative"] / steps,
                        "chain_extensions_per_window": acc["extensions"] / steps,
                        "max_micro_windows_one_group": acc["max_micro"],
                        "note": "value counts COMMITTED samples (the replayed schedule's granted "
                                "micro-windows); speculative = trained (chains + extensions)"},
            "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": e2e,
            "roofline": roof[0],
            "rooflines": roof[1],
            "kernels": {k: {"launches": v[0], "ms": v[1], "tflops": (v[2] / v[1] / 1e9) if v[1] else None}
                        for k, v in kst.items()},
            "parity": parity,
            "probes": probes,
        }
        if regroup is not None:
            line["regroup_matrix"] = regroup
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_sample(wl.N, wl.G)
            try:
                line["cpu_baseline_blas"] = cpu_blas(wl.N, wl.G)
            except Exception as e:
                line["cpu_baseline_blas"] = {"error": repr(e)}
        if world == 1 and not args.no_scaling:
            try:
                line["scaling_emulation"] = scaling_emulation(args, ms / steps)
            except Exception as e:  # reported, never fatal for the headline line
                line["scaling_emulation"] = {"error": repr(e)}
        if world == 1 and not args.no_parametric:
            try:
                line["parametric"] = parametric_leg(args)
            except Exception as e:  # reported, never fatal for the headline line
                line["parametric"] = {"error": repr(e)}
        print(json.dumps(line), flush=True)
    retr.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


PROBE_DEPTH = 2


def probe_leg(retr, torch, dist, reps=5):
    """The allocator's marginal-gain probes as concurrent batched kernels
    (the north star's third subsystem): every group's speculative chain of
    PROBE_DEPTH micro-windows in ONE ecco_train_trajectories call (the
    evaluate / train / evaluate probes of WindowAllocation::run_micro,
    gpu_allocator.cpp:125-135, for all groups at once), nothing committed.
    This is the throughput regime of the fused SGD chain (every group's
    cluster busy); the window's exact schedule above is the latency regime
    (the ECCO greedy serialises most of the budget on one group)."""
    if not retr.local:
        return None
    ctx = retr.ctx
    acc = np.zeros((len(retr.local), PROBE_DEPTH + 1))
    ctx.train_prepared(retr.prep, retr.gpu_s, PROBE_DEPTH, window=77, out=acc)
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(retr.stream):
        e0.record(retr.stream)
    for k in range(reps):
        ctx.train_prepared(retr.prep, retr.gpu_s, PROBE_DEPTH, window=78 + k, out=acc)
    with torch.cuda.stream(retr.stream):
        e1.record(retr.stream)
    e1.synchronize()
    ms = reduce_max(dist, [e0.elapsed_time(e1) / reps])[0]
    samples = reduce_sum(dist, float(PROBE_DEPTH * int(retr.steps[retr.local].sum()) * retr.B))
    return {"value": samples / (ms / 1e3), "unit": "samples/s", "ms_per_call": ms,
            "depth": PROBE_DEPTH, "groups": int(retr.G),
            "how": f"every group's {PROBE_DEPTH}-micro-window speculative chain in one "
                   "ecco_train_trajectories call (member evaluations included, nothing "
                   "committed), CUDA events on the context stream, max over ranks"}


def regroup_leg(retr, torch, dist, pk, reps=2):
    """configs[4]'s window is the allocator's marginal-gain probing; its
    window-end regroup -- the full camera x group matrix at the
    detection-head shape (k_eval_wide: X streamed beside the model), the
    all-gather and group_request's join rule -- is timed here on its own
    (CUDA events on the context stream, max over ranks; the kernel's own
    device time from the context's per-family events)."""
    if not retr.local:
        return None
    ctx = retr.ctx
    retr.regroup()
    ctx.synchronize()
    ctx.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(retr.stream):
        e0.record(retr.stream)
    for _ in range(reps):
        retr.regroup()
    with torch.cuda.stream(retr.stream):
        e1.record(retr.stream)
    e1.synchronize()
    ctx.synchronize()
    import paper_2512_11727_b200 as ecco
    n, kms, fl, by = ctx.kernel_stat(ecco.KSTAT_EVAL_MATRIX)
    ctx.profile(False)
    ms = reduce_max(dist, [e0.elapsed_time(e1) / reps])[0]
    tf = fl / kms / 1e9 if kms else None
    peak = pk.get("bf16_tflops_sustained", pk["bf16_tflops"])
    return {"ms_per_regroup": ms, "kernel_ms": kms / max(n, 1), "launches_per_regroup": n / reps,
            "flops": fl / max(n, 1), "achieved_tflops": tf, "peak_tflops": peak,
            "frac": tf / peak if tf else None,
            "how": "full camera x group matrix (every camera's S eval frames under every local "
                   "group), all-gather and join rule, CUDA events on the context stream"}


def parity_spot_check(args, retr, wl, n_cams=64):
    """The production-grid regroup matrix against the oracle-exact path: one
    more regroup on the bench's grid (C4: ~34 super tiles per CTA pair), its
    rows for a seeded sample of cameras compared with an FFMA_EXACT context
    (bit-exact to the fp32 oracle) holding the same committed weights and the
    same frames.  Reports count differences (of S) and the agreement of the
    join decision (argmax, lowest group id on ties)."""
    import torch
    import paper_2512_11727_b200 as ecco
    if not MATRIX or args.math == "ffma" or not retr.local:
        return None
    retr.regroup()
    retr.ctx.synchronize()
    rng = np.random.default_rng(1234)
    cams = np.sort(rng.choice(wl.N, min(n_cams, wl.N), replace=False)).astype(np.int32)
    tc = retr.M_local[torch.from_numpy(cams).long().to(retr.dev), :len(retr.local)].cpu().numpy()
    ff = ecco.Context(backend=ecco.LEARNED, device=retr.dev.index, math=ecco.FFMA_EXACT,
                      max_cameras=wl.N, max_jobs=len(retr.local), max_depth=2,
                      steps_per_gpu_s=float(STEPS), **DIMS)
    ff.set_cameras(wl.scenes, wl.tp)
    ff.generate_frames(0)
    ff.seed_models(retr.local)
    for g in retr.local:
        ff.set_weights(g, *retr.ctx.get_weights(g))
    ex = ff.eval_matrix(retr.local, cams=cams)
    ff.close()
    S = DIMS["eval_samples"]
    d = np.abs(tc - ex) * S
    ids = np.array(retr.local)
    # join rule per camera over these groups (no threshold): max, lowest id
    pick = lambda M: ids[np.argmax(M, axis=1)]  # local ids ascending: first max = lowest id
    return {"cameras": int(len(cams)), "groups": int(len(ids)),
            "max_count_diff": float(d.max()), "mean_count_diff": float(d.mean()),
            "pairs_equal": float((d == 0).mean()),
            "join_agreement": float((pick(tc) == pick(ex)).mean()),
            "how": "rows of the production-grid k_eval_pair matrix (bf16 tensor cores) vs an "
                   "FFMA_EXACT context (bit-exact to the fp32 oracle) with the same weights and "
                   "frames; counts of S = %d eval frames" % S}


def kernel_roofline(name, stat, pk, pk_kind, args, traffic=None, fused=True):
    """Roofline of one kernel family from its CUDA-event stats (launches, ms,
    algorithmic flops, algorithmic bytes), against the pipe the family runs
    on: under TC math the fused chain / evaluation kernels and the general
    bf16 forward run bf16 kind::f16 MMAs (held to the SUSTAINED bf16 peak of
    MEASURED_PEAKS.json, the kernels run back to back inside a long step;
    burst beside it), the general dW1 runs kind::tf32 (half that rate), and
    the general head (TRAIN_HEAD, and EVAL_PAIRS where the fused evaluation
    does not apply) is fp32 FFMA on the CUDA cores; --math ffma is all FFMA."""
    n, ms, fl, by = stat
    if not n or not ms:
        return None
    achieved = fl / (ms / 1e3) / 1e12
    ffma = 148 * 128 * 2 * 1.965e9 / 1e12
    if args.math == "ffma" or name == "TRAIN_HEAD" or (name == "EVAL_PAIRS" and not fused):
        peak = burst = ffma
        bound, how = "fp32", "fp32 FFMA spec (148 SM x 128 lanes x 2 x 1.965 GHz), CUDA cores"
    else:
        peak, burst = pk.get("bf16_tflops_sustained", pk["bf16_tflops"]), pk["bf16_tflops"]
        bound = "tensor"
        how = (f"{pk_kind} bf16 dense sustained {peak} TFLOP/s (burst {burst}): the kernel runs "
               "kind::f16 bf16 MMAs back to back inside a long step")
        if name == "TRAIN_DW1":
            peak, burst = peak / 2, burst / 2
            how = (f"half the {pk_kind} bf16 dense peak ({peak:.1f} sustained, {burst:.1f} burst): "
                   "kind::tf32 MMAs")
    gbs = by / (ms / 1e3) / 1e9
    out = {"kernel": name, "bound": bound, "achieved": achieved, "peak": peak,
           "unit": "TFLOP/s", "frac": achieved / peak, "frac_burst": achieved / burst,
           "peak_source": how, "avg_launch_ms": ms / n, "launches": n, "traffic": traffic,
           "algorithmic_gbs": gbs, "hbm_frac": gbs / pk["hbm_gbs"]}
    if name == "TRAIN_CHAIN" and args.math != "ffma":
        # (the fraction is of the whole GPU: the window's chains are one
        # group's dependent SGD steps on one cluster -- DESIGN.md 4 / 8)
        out["regime"] = ("latency: the exact schedule's serial chain runs one group's dependent "
                         "SGD steps on ONE cluster (C4: 4 SMs, ~6.3 us per step, the step's "
                         "tail bound by the shared-memory port; C5: 16 SMs, ~19 us per step, "
                         "bound by the fp32 master's read-modify-write through L2) beside the "
                         "regroup matrix; the throughput regime is the `probes` leg")
    return out


def roofline(kst, pk, pk_kind, args, fused=True, window_ms=None):
    """The dominant kernel's roofline (the headline `roofline` key) and every
    kernel family's.  Dominant = the family carrying most of the window's
    algorithmic work (FLOPs): at C4 the regroup matrix (~8.7e13 FLOP per
    window) against the retrain's ~1.1e12 -- the retrain's fused-chain
    launches take as much device time, but they are one group's serial
    chain running BESIDE the matrix on the reserved SMs (latency-bound by
    construction: its number is reported in `rooflines`, with each family's
    share of the window's device time)."""
    name = max(kst.items(), key=lambda kv: kv[1][2])[0]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            key = args.config if args.math == "bf16" else f"{args.config}_{args.math}"
            traffic = json.load(open(tpath)).get(key, {}).get(name)
        except (OSError, ValueError, AttributeError):
            traffic = None
    head = kernel_roofline(name, kst[name], pk, pk_kind, args, traffic, fused)
    if head is not None:
        head["selected_by"] = "largest algorithmic FLOPs of the window"
    every = {k: kernel_roofline(k, v, pk, pk_kind, args, fused=fused) for k, v in kst.items() if v[0]}
    if window_ms:
        for k, v in every.items():
            if v is not None:
                v["device_ms_share_of_window"] = kst[k][1] / window_ms
    return head, every


def run_e2e(args, retr, wl, torch, dist):
    """The same window through the public API with host buffers: every
    window's frames are ingested from pinned host memory and its results
    read back.  Pipelined as the product runs it: window k+1's
    eval sets stream in on the copy stream during window k; window k's drawn
    ring rows (ecco_stage_sampled_frames: only the rows its SGD steps draw,
    marked on the device, read zero-copy over PCIe) stream in during window
    k's own regroup and become current before its chains; chains the replay
    extends top their rows up (ecco_fetch_sampled_frames).  Host wall clock
    per phase: regroup = window start -> assignments on the host; retrain =
    -> trajectories replayed and the schedule committed."""
    import paper_2512_11727_b200 as ecco
    ctx = retr.ctx
    R, S, F = DIMS["ring_frames"], DIMS["eval_samples"], DIMS["feat_dim"]
    fr = torch.empty((wl.N, R, F), dtype=torch.int16, pin_memory=True)
    lb = torch.empty((wl.N, R), dtype=torch.int32, pin_memory=True)
    evf = torch.empty((wl.N, S, F), dtype=torch.int16, pin_memory=True)
    evl = torch.empty((wl.N, S), dtype=torch.int32, pin_memory=True)
    f, l, e, el = ctx.read_frames(wl.N)
    fr.numpy().view(np.uint16)[...] = f
    lb.numpy()[...] = l
    evf.numpy().view(np.uint16)[...] = e
    evl.numpy()[...] = el
    del f, l, e, el
    best_host = torch.empty(wl.N, dtype=torch.int32, pin_memory=True)
    steps = max(16, args.steps)  # amortises the pipeline fill (window 0's upload is not overlapped)
    ctx.reserve_ingest()  # setup: the back buffers' device memory is allocated before the clock
    retr.set_host_frames(fr.data_ptr())
    prep = retr.prep

    def stage_eval():
        ctx.stage_frames_range_host_ptr(0, 0, fr.data_ptr(), lb.data_ptr(), wl.N, evf.data_ptr(),
                                        evl.data_ptr())

    def stage_rings(w):
        if args.e2e_full_rings or not retr.local:
            ctx.stage_frames_range_host_ptr(0, wl.N, fr.data_ptr(), lb.data_ptr(), 0, 0, 0)
        else:
            ctx.stage_sampled_host_ptr(prep, GPU_S, DEPTH, w, fr.data_ptr(), lb.data_ptr(), 0, 0, 0)

    def window(w, timed):
        """Window w: its rings and eval sets were staged during window w-1 and
        become current at its start; window w+1's are staged on the copy
        stream as soon as window w's regroup matrix is enqueued (beside its
        greedy's chains); the assignments are read back at the end."""
        t0 = time.perf_counter()
        nxt = w + 1

        def stage_next():
            stage_eval()
            stage_rings(nxt)

        swap = lambda: ctx.swap_frame_parts(ecco.FRAMES_RINGS | ecco.FRAMES_EVAL)
        if MATRIX:
            retr.window(w, mid=swap, reserve_sms=RESERVE_SMS, after_launch=stage_next)
            with torch.cuda.stream(retr.stream):
                best_host.copy_(retr.best, non_blocking=True)  # group assignments to the host
            retr.stream.synchronize()
        else:  # (no regroup matrix) window w+1's staging overlaps the greedy's chains
            retr.retrain(w, mid=swap, after_initial=stage_next)
        return time.perf_counter() - t0, retr.stats["committed_samples"]

    # pipeline fill + one untimed warm-up window through the same ingest path
    # (first-touch costs of the pinned table and the staging buffers)
    stage_eval()
    stage_rings(9_999)
    window(9_999, False)
    ctx.synchronize()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    h0, d0 = ctx.transfer_bytes()
    wall, committed = 0.0, 0
    for k in range(steps):
        a, c = window(10_000 + k, True)
        wall, committed = wall + a, committed + c
    ctx.synchronize()
    h1, d1 = ctx.transfer_bytes()
    d1 += steps * best_host.numel() * 4
    el_s = reduce_max(dist, [wall])[0]
    return {"value": committed / el_s, "unit": "samples/s",
            "h2d_bytes_per_step": (h1 - h0) // steps, "d2h_bytes_per_step": (d1 - d0) // steps,
            "ms_per_step": el_s * 1e3 / steps, "steps": steps,
            "how": ("every window's frames from pinned host buffers on a copy stream, "
                    + ("ecco_stage_frames_range: every camera's full ring"
                       if args.e2e_full_rings else
                       "ecco_stage_sampled_frames: the ring rows this rank's SGD steps draw, marked "
                       "on the device and read zero-copy over PCIe (rows never drawn are not "
                       "transferred; extended chains top up with ecco_fetch_sampled_frames)")
                    + ", all labels and every camera's eval set; double-buffered: window k+1's "
                    "rings and eval sets stream in during window k (from its regroup-matrix "
                    "launch on) and become current at window k+1's start; the assignments read "
                    "back at the end of every window, trajectories read back for the host "
                    "replay; host wall clock per window (max over ranks), the pipeline fill in "
                    "the warm-up"),
            "pcie_gbs": (h1 - h0) / el_s / 1e9}


class _EmulatedMixin:
    """Rank 0 of an N-rank job on ONE GPU: its placed groups, every camera,
    the evaluation of its column block, the route over N blocks (the other
    ranks' blocks zero, as if gathered) and its chains; the other ranks'
    trajectories are stand-ins.  The all-gathers are not executed (one GPU):
    their NVLink time is modelled separately (scaling_emulation)."""

    def gather_blocks(self, M):
        out = self.torch.zeros((self.world, *M.shape), dtype=M.dtype, device=M.device)
        out[0].copy_(M)
        return out

    def gather_trajectories(self, acc):
        full = np.empty((self.G, acc.shape[1]))
        rows = acc if len(acc) else np.full((1, acc.shape[1]), 0.1)
        for g in range(self.G):
            full[g] = rows[self.slot_of[g]] if g in self.slot_of else rows[g % len(rows)]
        return full

    def broadcast(self, values, src):
        return values


def _emulated():
    from paper_2512_11727_b200.window import GroupRetrainer

    class E(_EmulatedMixin, GroupRetrainer):
        pass
    return E


EmulatedRank0 = None


def scaling_emulation(args, n1_ms, worlds=(2, 4, 8)):
    """One GPU standing in for rank 0 of an N-GPU run (its cost-balanced
    share of the groups, the full camera set, its column block, the route
    over N blocks, its chains, the replay over every group).  The NCCL
    all-gathers are modelled, not measured (one GPU): the matrix blocks
    (N x cameras x block x 8 B) and the trajectories at an assumed 600 GB/s
    all-gather bus bandwidth over NVLink 5 plus 25 us per collective."""
    import torch
    global EmulatedRank0
    EmulatedRank0 = _emulated()
    out = {}
    wl = Workload(args.config)
    for world in worlds:
        retr = make_retrainer(args, wl, 0, world, None, torch.cuda.current_device(), emulate=True)
        run = (lambda w: retr.window(w, reserve_sms=RESERVE_SMS)) if MATRIX else retr.retrain
        for w in range(2):
            run(w + 1)
        retr.ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 3
        committed = 0
        with torch.cuda.stream(retr.stream):
            e0.record(retr.stream)
        for k in range(n):
            run(10 + k)
            committed += retr.stats["committed_samples"]
        with torch.cuda.stream(retr.stream):
            e1.record(retr.stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        gb = retr.gb
        ag_bytes = (world * wl.N * gb * 8 if MATRIX else 0) + world * gb * (DEPTH + 1) * 8
        ag_ms = ag_bytes / 600e9 * 1e3 + 2 * 0.025
        local = len(retr.local)
        retr.close()
        torch.cuda.empty_cache()
        out[str(world)] = {"groups_on_rank0": local, "rank0_ms_per_step": ms,
                           "allgather_model_ms": ag_ms,
                           "projected_value": committed / n / ((ms + ag_ms) / 1e3),
                           "projected_efficiency": n1_ms / (world * (ms + ag_ms))}
    return out


# ------------------------------------------------------------ CPU baselines --

def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _window_units(N, G):
    """Work of one window the CPU must do for the same committed samples:
    the reference's sequential allocation (WindowAllocation::run_micro,
    gpu_allocator.cpp:125-135) runs W = W_PER_GROUP x G micro-windows, each one
    train(job) of STEPS SGD steps and two evaluate(job) over the job's
    members (orchestrator.cpp:43-62); the regroup adds the N x G matrix."""
    per = N // G
    W = W_PER_GROUP * G
    return {"micro_windows": W, "sgd_steps": W * int(GPU_S * STEPS), "train_eval_pairs": 2 * W * per,
            "matrix_pairs": N * G if MATRIX else 0,
            "committed_samples": W * int(GPU_S * STEPS) * DIMS["minibatch"]}


def cpu_sample(N, G, budget_s=12.0):
    """The oracle's restatement of the same window (oracle/ecco_oracle.c: the
    FFMA-order fp32 C that the device FFMA path matches bit for bit, built
    -O3 -march=x86-64-v3 so its fmaf chains vectorize) on every host core
    (one group per thread), timed on a bounded sample and scaled to the
    window: eval pairs (S frames each) and SGD steps measured separately."""
    import ctypes as C
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    from oracle import OrcLcfg

    if not os.path.exists(oracle.ORACLE_SO):
        oracle.build(ref=False)
    L = oracle.oracle()
    F, H, Cc, B, R, S = (DIMS["feat_dim"], DIMS["hidden_dim"], DIMS["num_classes"],
                         DIMS["minibatch"], DIMS["ring_frames"], DIMS["eval_samples"])
    lc = OrcLcfg(F=F, H=H, C=Cc, D=2, B=B, R=R, S=S, lr=0.05, noise=1.0,
                 steps_per_gpu_s=float(STEPS), seed=0x5eed0001)
    P = np.zeros(Cc * F, np.float32)
    Q = np.zeros(Cc * 2 * F, np.float32)
    L.orc_prototypes(C.byref(lc), P, Q)
    x = np.zeros(S * F, np.uint16)
    y = np.zeros(S, np.int32)
    L.orc_gen_frames(C.byref(lc), P, Q, 0, 0, 1, S, np.array([0.1, 0.2]), x, y)
    xb = np.ascontiguousarray(np.resize(x, B * F))
    yb = np.ascontiguousarray(np.resize(y, B))
    cores = os.cpu_count() or 1

    def weights():
        w = [np.zeros(F * H, np.float32), np.zeros(H, np.float32), np.zeros(H * Cc, np.float32),
             np.zeros(Cc, np.float32)]
        L.orc_init_weights(C.byref(lc), *w)
        return w

    def eval_work(n):
        w = weights()
        for _ in range(n):
            L.orc_count_correct(C.byref(lc), x, y, S, *w)
        return n

    def train_work(n):
        w = weights()
        for _ in range(n):
            L.orc_sgd_step(C.byref(lc), xb, yb, *w)
        return n

    # calibrate one unit each, then size the parallel sample to ~budget_s
    t = time.perf_counter()
    eval_work(4)
    t_pair = (time.perf_counter() - t) / 4
    t = time.perf_counter()
    train_work(2)
    t_step = (time.perf_counter() - t) / 2
    per_thread = budget_s / 2.0
    n_pairs = max(1, int(per_thread / max(t_pair, 1e-6)))
    n_steps = max(1, int(per_thread / max(t_step, 1e-6)))
    with ThreadPoolExecutor(cores) as ex:  # ctypes releases the GIL in the C calls
        t = time.perf_counter()
        list(ex.map(eval_work, [n_pairs] * cores))
        pair_rate = n_pairs * cores / (time.perf_counter() - t)
        t = time.perf_counter()
        list(ex.map(train_work, [n_steps] * cores))
        step_rate = n_steps * cores / (time.perf_counter() - t)
    u = _window_units(N, G)
    retrain_s = u["train_eval_pairs"] / pair_rate + u["sgd_steps"] / step_rate
    regroup_s = u["matrix_pairs"] / pair_rate
    window_s = retrain_s + regroup_s
    return {"value": u["committed_samples"] / window_s, "unit": "samples/s", "cores": cores,
            "kind": "port",
            "retrain_samples_per_s": u["committed_samples"] / retrain_s,
            "regroup_ms_per_window": regroup_s * 1e3,
            "cpu": cpu_model(),
            "sample": f"{n_pairs * cores} eval pairs (S={S} frames each) and {n_steps * cores} "
                      f"SGD steps (B={B}) of the oracle (oracle/ecco_oracle.c, FFMA-order fp32, "
                      f"AVX2/FMA-vectorized) on {cores} threads; window = {u['matrix_pairs']} "
                      f"matrix pairs + {u['train_eval_pairs']} allocator evaluation pairs + "
                      f"{u['sgd_steps']} SGD steps, scaled from the measured rates",
            "window_s": window_s}


def cpu_blas(N, G, budget_s=8.0):
    """A BLAS-batched CPU implementation of the same window beside the port:
    torch CPU fp32 (oneDNN / MKL GEMMs) on every core, SGD steps of many
    groups batched as bmm (speculatively, as the device does) and member
    evaluations as batched GEMMs; timed on a bounded sample, scaled to the
    window's units (_window_units)."""
    import torch
    cores = os.cpu_count() or 1
    torch.set_num_threads(cores)
    F, H, Cc, B, S = (DIMS["feat_dim"], DIMS["hidden_dim"], DIMS["num_classes"],
                      DIMS["minibatch"], DIMS["eval_samples"])
    g = 32  # groups per batched call
    gen = torch.Generator().manual_seed(0)
    X = torch.randn(g, B, F, generator=gen).bfloat16().float()
    Y = torch.randint(0, Cc, (g, B), generator=gen)
    W1 = torch.randn(g, F, H, generator=gen) * 0.05
    b1 = torch.zeros(g, 1, H)
    W2 = torch.randn(g, H, Cc, generator=gen) * 0.1
    b2 = torch.zeros(g, 1, Cc)
    E = torch.randn(g, 20 * S, F, generator=gen).bfloat16().float()
    lr = 0.05

    def sgd():
        Z = torch.baddbmm(b1, X, W1)
        Rl = Z.clamp_min(0)
        Lg = torch.baddbmm(b2, Rl, W2)
        P = torch.softmax(Lg, -1)
        P[torch.arange(g)[:, None], torch.arange(B)[None], Y] -= 1
        dL = P / B
        dH = torch.bmm(dL, W2.transpose(1, 2)) * (Z > 0)
        W2.sub_(lr * torch.bmm(Rl.transpose(1, 2), dL))
        b2.sub_(lr * dL.sum(1, keepdim=True))
        W1.sub_(lr * torch.bmm(X.transpose(1, 2), dH))
        b1.sub_(lr * dH.sum(1, keepdim=True))

    def evaluate():
        Lg = torch.baddbmm(b2, torch.baddbmm(b1, E, W1).clamp_min(0), W2)
        return Lg.argmax(-1)

    with torch.no_grad():
        sgd()
        evaluate()
        t = time.perf_counter()
        n = 0
        while time.perf_counter() - t < budget_s / 2:
            sgd()
            n += 1
        step_rate = n * g / (time.perf_counter() - t)  # group-steps / s
        t = time.perf_counter()
        m = 0
        while time.perf_counter() - t < budget_s / 2:
            evaluate()
            m += 1
        pair_rate = m * g * 20 / (time.perf_counter() - t)  # (camera, group) pairs / s
    u = _window_units(N, G)
    retrain_s = u["train_eval_pairs"] / pair_rate + u["sgd_steps"] / step_rate
    regroup_s = u["matrix_pairs"] / pair_rate
    window_s = retrain_s + regroup_s
    return {"value": u["committed_samples"] / window_s, "unit": "samples/s", "cores": cores,
            "kind": "blas",
            "retrain_samples_per_s": u["committed_samples"] / retrain_s,
            "regroup_ms_per_window": regroup_s * 1e3, "cpu": cpu_model(),
            "sample": f"{n * g} group SGD steps (B={B}, batched {g} groups per bmm) and "
                      f"{m * g * 20} eval pairs (S={S}) in torch CPU fp32 on {cores} threads "
                      f"(torch {torch.__version__}), scaled to the window",
            "window_s": window_s}


def parametric_leg(args):
    """The reference-pinned backend against the UNMODIFIED reference library
    (oracle/_ref, compiled from /root/reference; shipped prebuilt to the GPU
    box): (a) the camera x group eval matrix (K1, `eval` per pair,
    accuracy_model.cpp:60-67) at C4 size on the GPU vs the reference's own loop
    on a bounded sample, bit-exact check included; (b) Simulation::step_window
    (orchestrator.cpp:211-413) at C3 on the GPU window driver vs the reference,
    per-window wall time and byte-identical trace."""
    import ctypes as C

    import torch

    import oracle
    import paper_2512_11727_b200 as ecco
    from paper_2512_11727_b200 import scenarios

    if not oracle.have_ref():
        return {"unavailable": "oracle/_ref/libecco_ref.so not built"}
    R = oracle.ref()
    out = {}
    # (a) eval matrix, C4: 10,000 scenes x 500 models of K=3 clusters, D=2
    rng = np.random.default_rng(7)
    N, G, K, D = 10000, 500, 3, 2
    params = oracle.params_array(oracle.default_params())
    scenes = np.round(rng.random((N, D)), 2)
    ks = np.full(G, K, np.int32)
    cl = np.round(rng.random((G, K, D)), 2)
    pr = rng.random((G, K))
    ce = cl.mean(1)
    clen = np.full(G, D, np.int32)
    ctx = ecco.Context(backend=ecco.PARAMETRIC, max_jobs=G, max_cameras=N, max_clusters=K)
    ids = list(range(G))
    ctx.put_models(ids, ks, cl, pr, ce, clen)
    dM = torch.empty((N, G), dtype=torch.float64, device="cuda")
    stream = torch.cuda.ExternalStream(ctx.stream)
    for _ in range(3):
        ctx.eval_matrix_dev(ids, dM.data_ptr(), scenes=scenes)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    with torch.cuda.stream(stream):
        ev0.record(stream)
    for _ in range(reps):
        ctx.eval_matrix_dev(ids, dM.data_ptr(), scenes=scenes)
    with torch.cuda.stream(stream):
        ev1.record(stream)
    ev1.synchronize()
    gpu_s = ev0.elapsed_time(ev1) / 1e3 / reps
    ns = 1000  # bounded CPU sample: 1,000 scenes x 500 models
    want = np.zeros((ns, G))
    cpu_s = R.ref_eval_matrix(ns, np.ascontiguousarray(scenes[:ns]), G, ks,
                              np.ascontiguousarray(cl.reshape(-1)), np.ascontiguousarray(pr.reshape(-1)),
                              clen, np.ascontiguousarray(ce.reshape(-1)), K, D, params, want)
    got = dM[:ns].cpu().numpy()
    # K1's rooflines: HBM on the algorithmic bytes (the fp64
    # matrix written + scenes + models read), FP64 on (K+1)(3D+2) flops per
    # pair plus K+1 exp (glibc's algorithm, ~25 fp64 ops each) -- B200 FP64
    # is ~37 TFLOP/s (spec, not measured)
    k1_bytes = 8.0 * N * G + 8.0 * N * D + 8.0 * G * (K * D + K + D)
    k1_flops = N * G * ((K + 1) * (3 * D + 2) + (K + 1) * 25.0)
    out["eval_matrix"] = {
        "workload": f"{N} scenes x {G} models (K={K}, D={D}), fp64",
        "gpu_pairs_per_s": N * G / gpu_s, "gpu_ms": gpu_s * 1e3,
        "hbm_gbs": k1_bytes / gpu_s / 1e9,
        "hbm_frac": k1_bytes / gpu_s / 1e9 / peaks()[0]["hbm_gbs"],
        "fp64_tflops": k1_flops / gpu_s / 1e12, "fp64_frac_of_spec_37": k1_flops / gpu_s / 37e12,
        "reference_pairs_per_s": ns * G / cpu_s, "reference_cores": 1,
        "reference_sample": f"{ns} x {G} pairs through the reference's eval()",
        "bit_exact_vs_reference": bool(got.tobytes() == want.tobytes()),
        "speedup": (N * G / gpu_s) / (ns * G / cpu_s)}
    ctx.close()
    # (b) window driver, C3 (1,000 cameras / 50 clusters, W = 100 micro-windows)
    sc = json.dumps(scenarios.config("c3", windows=4, seed=1))  # (seed 3 makes the reference itself
    # raise set_aimd_params for a zero-gain job, and the GPU driver raises the same)
    sim = ecco.Simulation(sc, backend=ecco.PARAMETRIC)
    wins, regroup = [], []
    while True:
        t = time.perf_counter()
        if not sim.step_window():
            break
        wins.append(time.perf_counter() - t)
        regroup.append(sim.last_timings()["regroup_ms"])
    ref_s = np.zeros(8)
    n_run = C.c_int()
    R.ref_time_windows(sc.encode(), 8, ref_s, C.byref(n_run))
    ref_s = ref_s[:n_run.value]
    tcap = 1 << 26
    tb, sb = C.create_string_buffer(tcap), C.create_string_buffer(1 << 20)
    tl, sl = C.c_size_t(), C.c_size_t()
    R.ref_run_scenario(sc.encode(), -1, tb, tcap, C.byref(tl), sb, 1 << 20, C.byref(sl))
    # (c) the window driver at C4 (10,000 cameras / 500 jobs, W = 1000) on the
    # GPU and the UNMODIFIED reference's Simulation::step_window on one host
    # core, same scenario, measured here (window 0 builds every camera's
    # profile table: ~40 s for the reference), traces compared
    sc4 = json.dumps(scenarios.config("c4", windows=2, seed=1))
    sim4 = ecco.Simulation(sc4, backend=ecco.PARAMETRIC)
    w4 = []
    while sim4.step_window():
        w4.append({k: round(v, 3) for k, v in sim4.last_timings().items()})
    ref4 = None
    if not args.no_ref_c4:
        r4 = np.zeros(4)
        n4 = C.c_int()
        tb4 = C.create_string_buffer(1 << 27)
        tl4 = C.c_size_t()
        R.ref_time_windows_trace(sc4.encode(), 4, r4, C.byref(n4), tb4, 1 << 27, C.byref(tl4))
        ref4 = [float(v) * 1e3 for v in r4[:n4.value]]
        same4 = sim4.trace_csv() == tb4.raw[:tl4.value].decode()
    sim4.close()
    out["window_c4"] = {"workload": "c4 scenario (scenarios.config('c4', windows=2, seed=1)), "
                                    "parametric backend; window 0 builds 10,000 profile tables",
                        "gpu_windows": w4, "reference_window_ms": ref4, "reference_cores": 1,
                        "reference_cpu": cpu_model(),
                        "trace_identical_to_reference": same4 if ref4 is not None else None}
    # (d) the same window driver with the LEARNED backend at C4: routing and
    # regroup on the device evaluation matrix, every micro-window's SGD chain,
    # the netsim and allocator replay on the host (no reference counterpart:
    # the reference has no learned trainer)
    scl = json.dumps(scenarios.config("c4", windows=2, seed=1, local_acc=0.0))
    siml = ecco.Simulation(scl, backend=ecco.LEARNED, math=ecco.TC_BF16, full_matrix=1,
                           steps_per_gpu_s=5000.0)
    wl_ = []
    while siml.step_window():
        d = {k: round(v, 3) for k, v in siml.last_timings().items()}
        d["samples"] = siml.last_samples()
        d["samples_per_s"] = d["samples"] / (d["window_ms"] / 1e3)
        wl_.append(d)
    siml.close()
    out["learned_window_c4"] = {
        "workload": "c4 scenario, local_model_acc 0 (fresh group models accept joins), learned "
                    "F512-H256-C16 classifier, tf32/bf16 tensor-core math, steps_per_gpu_s 5000",
        "gpu_windows": wl_}
    out["window"] = {
        "workload": "c3 scenario (scenarios.config('c3', seed=1), 4 windows), parametric backend",
        "gpu_window_ms": [w * 1e3 for w in wins], "gpu_regroup_ms": regroup,
        "reference_window_ms": [w * 1e3 for w in ref_s], "reference_cores": 1,
        "trace_identical_to_reference": sim.trace_csv() == tb.raw[:tl.value].decode()}
    sim.close()
    return out


def run_reference(args, rank):
    """The reference arm: the CPU restatement of the same window (oracle
    port, every host core), each step a bounded sample scaled to the window
    (cpu_sample).  Rank 0 only; the other ranks exit without work."""
    if rank != 0:
        return
    wl = Workload(args.config)
    vals = []
    for _ in range(args.warmup):
        cpu_sample(wl.N, wl.G, budget_s=2.0)
    t0 = time.perf_counter()
    last = None
    for _ in range(args.steps):
        last = cpu_sample(wl.N, wl.G, budget_s=args.ref_budget)
        vals.append(last)
    wall = time.perf_counter() - t0
    value = statistics.median(v["value"] for v in vals)
    line = {
        "impl": "reference",
        "metric": "group-retrain samples/s (per-window regroup + retrain)",
        "value": value, "unit": "samples/s",
        "retrain_samples_per_s": statistics.median(v["retrain_samples_per_s"] for v in vals),
        "regroup_ms_per_window": statistics.median(v["regroup_ms_per_window"] for v in vals),
        "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup,
        # each step is a bounded sample (ref_budget s of CPU work) scaled to the window by
        # its measured rates: ms_per_step is the sample's wall time, the projected time of
        # the whole window on this CPU is window_ms_projected
        "ms_per_step": wall * 1e3 / max(1, args.steps),
        "window_ms_projected": last["window_s"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (counter-RNG camera streams, random-init group MLPs)",
        "config": {"workload": f"{args.config}: {wl.N} cameras / {wl.G} groups (same as the B200 arm)",
                   "cameras": wl.N, "groups": wl.G},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": last["cores"],
                         "kind": "port", "sample": last["sample"], "cpu": last["cpu"]},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": wall,
        "note": "the reference (a C++ simulator) has no learned trainer: its path is the "
                "parametric accuracy model (SURVEY.md 0); the learned path's CPU form is the "
                "oracle restatement (vectorized, bit-identical to the scalar restatement), run "
                "here on every host core",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--math", default="bf16", choices=["bf16", "tf32", "ffma"],
                    help="bf16: tensor-core math (tf32 is its round-1 name); ffma: fp32 exact")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e leg (profiling runs)")
    ap.add_argument("--e2e-full-rings", action="store_true",
                    help="e2e ingest copies every ring of the rank's cameras, not only the drawn rows")
    ap.add_argument("--no-scaling", action="store_true",
                    help="skip the single-GPU emulation of rank 0 at N = 2, 4, 8")
    ap.add_argument("--no-parametric", action="store_true",
                    help="skip the parametric-backend vs reference-library leg")
    ap.add_argument("--no-ref-c4", action="store_true",
                    help="skip timing the reference's C4 parametric windows (~40 s of CPU)")
    ap.add_argument("--no-probes", action="store_true",
                    help="skip the batched marginal-gain probe leg")
    ap.add_argument("--no-regroup", action="store_true",
                    help="c5: skip the separately timed regroup-matrix leg")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the production-grid parity spot check against the FFMA path")
    ap.add_argument("--decisions", action="store_true",
                    help="add the decision-agreement leg (learned window driver, FFMA vs TC)")
    args = ap.parse_args()
    global MATRIX, MAX_DEPTH
    if args.config == "c5":
        DIMS.update(DET_DIMS)
        MATRIX = False
        # 4.4 MB of parameters per snapshot: 500 groups x 32 snapshots = 70 GB
        # of HBM (of 180), so the least accurate group's ~500 serial
        # micro-windows take ~16 extension calls (each one launch)
        MAX_DEPTH = 32
    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
