"""Benchmark of the B200 group-retraining path (BASELINE.json `metric`).

One step = one retraining window of the hot path over the workload's
synthetic camera streams ("Measurement"):

  regroup   the camera x group evaluation matrix -- every camera's S labelled
            eval frames scored under every group model (ecco_eval_matrix_dev,
            the ModelEvalFn batch of grouping.cpp:33) -- all-gathered across
            ranks, then the warp-reduced argmax/threshold per camera
            (ecco_route_matrix_dev, group_request's join rule);
  retrain   every group's speculative micro-window chain: evaluate, then
            DEPTH x (STEPS SGD steps of B sampled frames, evaluate)
            (ecco_train_trajectories, the allocator's TrainingBackend probes of
            gpu_allocator.cpp:125-135); the chains' accuracy trajectories
            all-gathered across ranks, the reference's greedy allocation
            (WindowAllocation, ecco_allocate_trajectories) replayed over every
            group on the host with W = DEPTH x G micro-windows, and
            ecco_commit of each group's granted prefix.

value = retrain samples of all ranks / max-over-ranks device time of the
whole step (regroup included), in samples/s.  Groups are sharded across ranks
(contiguous blocks); cameras are replicated (their frames are generated per
rank from the counter RNG).  The only collective is the all-gather of the
evaluation-matrix column blocks.  `e2e` is the same step through the public
API with the window's frames uploaded from pinned host memory and the
assignments / accuracies read back, every step.

`--impl reference` times the CPU restatement of the same path (oracle/, the
reference itself has no learned trainer: SURVEY.md 0) on this box's cores.
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
DEPTH = 2             # micro-windows granted per group per window (initial pass + 1 greedy)
STEPS = 16            # SGD steps per micro-window
# configs[4]: the detection-head variant (larger per-group model and frame
# features).  Its window is the allocator's marginal-gain probing (every
# group's speculative chain + member evaluations); the full camera x group
# matrix at this shape has no fused kernel yet and is left out of the step.
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
    """Cameras, groups and the rank's shard (groups in contiguous blocks)."""

    def __init__(self, config, rank, world):
        self.config = config
        self.N, self.G = CONFIGS[config]
        self.per = self.N // self.G
        self.rank, self.world = rank, world
        from paper_2512_11727_b200 import shard
        self.gb = shard.block_size(self.G, world)  # column block per rank (last may be ragged)
        self.local = shard.rank_groups(self.G, world, rank)
        side = 10
        self.scenes = np.array([[0.1 * ((c // self.per) % side), 0.1 * ((c // self.per // side) % side)]
                                for c in range(self.N)], np.float64)
        self.tp = np.full(self.N, THROUGHPUT)

    def members(self, g):
        return list(range(g * self.per, (g + 1) * self.per))

    def samples_per_step_local(self):
        return len(self.local) * DEPTH * int(GPU_S * STEPS) * DIMS["minibatch"]


# ----------------------------------------------------------------- B200 arm --

def run_b200(args, rank, world, local_rank):
    import torch
    import paper_2512_11727_b200 as ecco
    from paper_2512_11727_b200 import shard

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
    wl = Workload(args.config, rank, world)
    math = ecco.TC_BF16 if args.math == "tf32" else ecco.FFMA_EXACT
    ctx = ecco.Context(backend=ecco.LEARNED, device=local_rank, math=math,
                       max_cameras=wl.N, max_jobs=max(1, len(wl.local)), max_depth=DEPTH,
                       steps_per_gpu_s=float(STEPS), **DIMS)
    ctx.set_cameras(wl.scenes, wl.tp)
    ctx.generate_frames(0)
    ctx.seed_models(wl.local)
    prep = ctx.prepare_trajectories(
        wl.local, [BATCH] * len(wl.local), [wl.members(g) for g in wl.local],
        [[1.0 / wl.per] * wl.per for _ in wl.local], [wl.members(g) for g in wl.local])
    cams = np.arange(wl.N, dtype=np.int32)
    stream = torch.cuda.ExternalStream(ctx.stream)
    dev = torch.device("cuda", local_rank)
    M_local = torch.full((wl.N if MATRIX else 1, wl.gb), float("nan"), dtype=torch.float64,
                         device=dev)
    M_part = None if len(wl.local) == wl.gb or not MATRIX else torch.empty((wl.N, max(1, len(wl.local))),
                                                             dtype=torch.float64, device=dev)
    best = torch.empty(wl.N, dtype=torch.int32, device=dev)
    best_acc = torch.empty(wl.N, dtype=torch.float64, device=dev)
    acc_host = np.zeros((len(wl.local), DEPTH + 1))
    ev = {k: torch.cuda.Event(enable_timing=True) for k in ("a", "b", "c")}
    phase = {"regroup": 0.0, "retrain": 0.0}

    def gather_trajectories(acc):
        """[gb, DEPTH+1] per rank -> [world*gb, DEPTH+1] (group-major)."""
        blk = np.zeros((wl.gb, DEPTH + 1))
        blk[:len(wl.local)] = acc
        if dist is None:
            return blk
        t = torch.from_numpy(blk).to(_red_device())
        out = torch.empty((world, wl.gb, DEPTH + 1), dtype=t.dtype, device=t.device)
        if t.is_cuda:
            dist.all_gather_into_tensor(out, t)
        else:
            dist.all_gather(list(out.unbind(0)), t)
        return out.reshape(world * wl.gb, DEPTH + 1).cpu().numpy()

    def step(w, timed=False, mid=None):
        with torch.cuda.stream(stream):
            if timed:
                ev["a"].record(stream)
            if not MATRIX:
                pass
            elif wl.local:
                if M_part is None:
                    ctx.eval_matrix_dev(wl.local, M_local.data_ptr(), cams=cams)
                else:  # ragged last block: columns beyond the rank's groups stay NaN
                    ctx.eval_matrix_dev(wl.local, M_part.data_ptr(), cams=cams)
                    M_local[:, :len(wl.local)].copy_(M_part)
            if MATRIX:
                if backend == "nccl":
                    M = shard.gather_blocks(M_local, world, dist)  # NCCL all-gather of column blocks
                else:
                    M = shard.gather_blocks(M_local.cpu(), world, dist).to(dev)
                ctx.route_matrix_dev(wl.N, wl.gb, M.data_ptr(), best.data_ptr(),
                                     best_acc.data_ptr(), n_blocks=world)
            if timed:
                ev["b"].record(stream)
            if mid is not None:
                mid()  # (e2e: this window's rings become current here)
            if wl.local:
                ctx.train_prepared(prep, GPU_S, DEPTH, window=w, out=acc_host)
            # the allocator's decisions over EVERY group: trajectories
            # all-gathered (G x (DEPTH+1) fp64), the reference's greedy
            # (WindowAllocation, gpu_allocator.cpp:100-181) replayed on the
            # host with W = DEPTH x G micro-windows, each rank commits the
            # granted prefixes of its own groups
            traj = gather_trajectories(acc_host)
            jobs, _, _, _ = ecco.allocate_trajectories(
                np.arange(wl.G, dtype=np.int32), np.full(wl.G, wl.per, np.int32), traj[:wl.G],
                1.0, 1.0, DEPTH * wl.G, GPU_S, 1, True, 0)
            counts = np.bincount(jobs, minlength=wl.G)
            if wl.local:
                ctx.commit(wl.local, np.minimum(counts[wl.local], DEPTH).astype(np.int32))
            if timed:
                ev["c"].record(stream)
                ev["c"].synchronize()
                phase["regroup"] += ev["a"].elapsed_time(ev["b"])
                phase["retrain"] += ev["b"].elapsed_time(ev["c"])

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
    # <= 512, H = 256 / 512), else the unfused forward; DW1 / HEAD are the
    # unfused tensor-core / FFMA kernels (other shapes, --math ffma)
    F, H = DIMS["feat_dim"], DIMS["hidden_dim"]
    chain = (args.math == "tf32" and DIMS["minibatch"] == 128 and DIMS["num_classes"] == 16
             and F <= 512 and F % 128 == 0 and F & (F - 1) == 0 and H in (256, 512))
    kst = {name: ctx.kernel_stat(getattr(ecco, "KSTAT_" + stat)) for name, stat in
           (("EVAL_MATRIX", "EVAL_MATRIX"), ("EVAL_PAIRS", "EVAL_PAIRS"),
            ("TRAIN_CHAIN" if chain else "TRAIN_FWD", "TRAIN_STEP"), ("TRAIN_DW1", "TRAIN_DW1"),
            ("TRAIN_HEAD", "TRAIN_HEAD"))}
    ctx.profile(False)
    ms, regroup_ms, retrain_ms = reduce_max(dist, [ms, phase["regroup"], phase["retrain"]])
    samples = reduce_sum(dist, wl.samples_per_step_local() * args.steps)

    # ---- e2e: same step through the public API, frames from pinned host memory
    e2e = None if args.no_e2e else run_e2e(args, ctx, wl, step, torch, dist, stream, best, prep)

    if rank == 0:
        pk, pk_kind = peaks()
        roof = roofline(kst, pk, pk_kind, args, fused=chain)
        line = {
            "metric": "group-retrain samples/s (per-window regroup + retrain)",
            "value": samples / (ms / 1e3),
            "unit": "samples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            # operand type of the tensor-core contractions (fp32 accumulation
            # and fp32 masters throughout): the fused chain and the evaluation
            # kernels run kind::f16 bf16; shapes outside the chain train with
            # a bf16 forward and a tf32 dW1; --math ffma is fp32 on CUDA cores
            "dtype": ("f32" if args.math != "tf32" else "bf16" if chain
                      else "bf16+tf32" if DIMS["minibatch"] % 128 == 0 and H % 256 == 0 else "tf32"),
            "data": "synthetic (counter-RNG camera streams, random-init group MLPs)",
            "config": {
                "workload": f"{args.config}: {wl.N} cameras / {wl.G} groups, learned classifier "
                            f"F{DIMS['feat_dim']}-H{DIMS['hidden_dim']}-C{DIMS['num_classes']}, "
                            f"B={DIMS['minibatch']}, S={DIMS['eval_samples']} eval frames/camera, "
                            f"R={DIMS['ring_frames']} ring frames/camera, depth {DEPTH} x "
                            f"{STEPS} SGD steps per group per window, "
                            + ("full camera x group matrix" if MATRIX else
                               "marginal-gain probes only (no regroup matrix)"),
                "cameras": wl.N, "groups": wl.G, "groups_per_rank": wl.gb,
                "parallelism": f"groups sharded over {world} rank(s); eval matrix all-gather",
                "l2": "inputs larger than L2 (frames "
                      f"{wl.N * (DIMS['ring_frames'] + DIMS['eval_samples']) * DIMS['feat_dim'] * 2 / 2**30:.1f} GiB)",
            },
            "regroup_ms_per_window": regroup_ms / args.steps,
            "retrain_ms_per_window": retrain_ms / args.steps,
            "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": e2e,
            "roofline": roof[0],
            "rooflines": roof[1],
            "kernels": {k: {"launches": v[0], "ms": v[1], "tflops": (v[2] / v[1] / 1e9) if v[1] else None}
                        for k, v in kst.items()},
        }
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_sample(wl.N, wl.G)
        if world == 1 and not args.no_scaling:
            try:
                line["scaling_emulation"] = scaling_emulation(args, ms / args.steps)
            except Exception as e:  # reported, never fatal for the headline line
                line["scaling_emulation"] = {"error": repr(e)}
        if world == 1 and not args.no_parametric:
            try:
                line["parametric"] = parametric_leg(args)
            except Exception as e:  # reported, never fatal for the headline line
                line["parametric"] = {"error": repr(e)}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def scaling_emulation(args, n1_ms, worlds=(2, 4, 8)):
    """One GPU standing in for rank 0 of an N-GPU run: its shard of the
    groups (the largest block), the full camera set, the evaluation of its
    column block, the route over N blocks (the other ranks' blocks as they
    would arrive from the all-gather) and its chains.  The per-rank device
    time projects the N-GPU step; the NCCL all-gather of the blocks
    (N x cameras x block x 8 B) is not included -- at C4 and N = 8 it moves
    40 MB per rank over NVLink."""
    import torch
    import paper_2512_11727_b200 as ecco
    out = {}
    for world in worlds:
        wl = Workload(args.config, 0, world)
        ctx = ecco.Context(backend=ecco.LEARNED, device=torch.cuda.current_device(),
                           math=ecco.TC_BF16 if args.math == "tf32" else ecco.FFMA_EXACT,
                           max_cameras=wl.N, max_jobs=max(1, len(wl.local)), max_depth=DEPTH,
                           steps_per_gpu_s=float(STEPS), **DIMS)
        ctx.set_cameras(wl.scenes, wl.tp)
        ctx.generate_frames(0)
        ctx.seed_models(wl.local)
        prep = ctx.prepare_trajectories(
            wl.local, [BATCH] * len(wl.local), [wl.members(g) for g in wl.local],
            [[1.0 / wl.per] * wl.per for _ in wl.local], [wl.members(g) for g in wl.local])
        cams = np.arange(wl.N, dtype=np.int32)
        stream = torch.cuda.ExternalStream(ctx.stream)
        blocks = torch.zeros((world, wl.N if MATRIX else 1, wl.gb), dtype=torch.float64,
                             device="cuda")
        best = torch.empty(wl.N, dtype=torch.int32, device="cuda")
        best_acc = torch.empty(wl.N, dtype=torch.float64, device="cuda")
        acc_host = np.zeros((len(wl.local), DEPTH + 1))

        def step(w):
            with torch.cuda.stream(stream):
                if MATRIX:
                    ctx.eval_matrix_dev(wl.local, blocks[0].data_ptr(), cams=cams)
                    ctx.route_matrix_dev(wl.N, wl.gb, blocks.data_ptr(), best.data_ptr(),
                                         best_acc.data_ptr(), n_blocks=world)
                ctx.train_prepared(prep, GPU_S, DEPTH, window=w, out=acc_host)
                # the allocator replay over all groups (other ranks' rows as
                # the all-gather would deliver them; here zeros)
                traj = np.zeros((world * wl.gb, DEPTH + 1))
                traj[:len(wl.local)] = acc_host
                jobs, _, _, _ = ecco.allocate_trajectories(
                    np.arange(wl.G, dtype=np.int32), np.full(wl.G, wl.per, np.int32),
                    traj[:wl.G], 1.0, 1.0, DEPTH * wl.G, GPU_S, 1, True, 0)
                counts = np.bincount(jobs, minlength=wl.G)
                ctx.commit(wl.local, np.minimum(counts[wl.local], DEPTH).astype(np.int32))

        for w in range(2):
            step(w + 1)
        ctx.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 3
        with torch.cuda.stream(stream):
            e0.record(stream)
        for k in range(n):
            step(10 + k)
        with torch.cuda.stream(stream):
            e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        ctx.close()
        del blocks
        torch.cuda.empty_cache()
        samples = wl.samples_per_step_local() * world
        out[str(world)] = {"groups_on_rank0": len(wl.local), "rank0_ms_per_step": ms,
                           "projected_value": samples / (ms / 1e3),
                           "projected_efficiency": n1_ms / (world * ms)}
    return out


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
    if args.math != "tf32" or name == "TRAIN_HEAD" or (name == "EVAL_PAIRS" and not fused):
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
    return {"kernel": name, "bound": bound, "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s", "frac": achieved / peak, "frac_burst": achieved / burst,
            "peak_source": how, "avg_launch_ms": ms / n, "launches": n, "traffic": traffic,
            "algorithmic_gbs": gbs, "hbm_frac": gbs / pk["hbm_gbs"]}


def roofline(kst, pk, pk_kind, args, fused=True):
    """The dominant kernel's roofline (the headline `roofline` key) and every
    kernel family's."""
    name = max(kst.items(), key=lambda kv: kv[1][1])[0]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "dram_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(args.config, {}).get(name)
        except (OSError, ValueError, AttributeError):
            traffic = None
    head = kernel_roofline(name, kst[name], pk, pk_kind, args, traffic, fused)
    every = {k: kernel_roofline(k, v, pk, pk_kind, args, fused=fused) for k, v in kst.items() if v[0]}
    return head, every


def run_e2e(args, ctx, wl, step, torch, dist, stream, best_dev, prep):
    """Frames uploaded from pinned host memory and results read back every step."""
    import paper_2512_11727_b200 as ecco
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
    # this rank's groups train on their members' rings only.  Default: the
    # ring rows the window's SGD steps draw (marked on the device from the
    # same counter-RNG draws, read zero-copy from the pinned table); with
    # --e2e-full-rings every ring of the rank's camera range is copied.  Both
    # add every camera's eval set and all labels.
    c0, c1 = (wl.local[0] * wl.per, (wl.local[-1] + 1) * wl.per) if wl.local else (0, 0)
    ptrs = (fr[c0].data_ptr() if c1 > c0 else fr.data_ptr(), lb[c0].data_ptr() if c1 > c0 else lb.data_ptr(),
            wl.N, evf.data_ptr(), evl.data_ptr())

    def stage_eval():
        ctx.stage_frames_range_host_ptr(0, 0, fr.data_ptr(), lb.data_ptr(), wl.N, evf.data_ptr(),
                                        evl.data_ptr())

    def stage_rings(w):
        if args.e2e_full_rings or not wl.local:
            ctx.stage_frames_range_host_ptr(c0, c1 - c0, ptrs[0], ptrs[1], 0, 0, 0)
        else:
            ctx.stage_sampled_host_ptr(prep, GPU_S, DEPTH, w, fr.data_ptr(), lb.data_ptr(), 0, 0, 0)

    # double-buffered ingest in two parts on the copy stream: window k+1's
    # eval sets stream in during window k and become current at window k+1's
    # start (its regroup reads them); its rings (the drawn rows) stream in
    # during window k+1's own regroup and become current between that regroup
    # and its SGD chains (configs without a regroup matrix stage them a whole
    # window ahead instead).  Window 0's eval sets are the only unoverlapped
    # copy.
    # one untimed warm-up window through the same ingest path (first-touch
    # costs of the pinned table and the staging buffers), like the W warm-up
    # steps of the device-only leg
    stage_eval()
    ctx.swap_frame_parts(ecco.FRAMES_EVAL)
    stage_rings(9_999)
    step(9_999, mid=lambda: ctx.swap_frame_parts(ecco.FRAMES_RINGS))
    ctx.synchronize()
    h0, d0 = ctx.transfer_bytes()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    stage_eval()
    ctx.swap_frame_parts(ecco.FRAMES_EVAL)
    stage_rings(10_000)
    for k in range(steps):
        if k + 1 < steps:
            stage_eval()

        def mid(k=k):  # window k's rings become current
            ctx.swap_frame_parts(ecco.FRAMES_RINGS)
            if k + 1 < steps and not MATRIX:
                stage_rings(10_000 + k + 1)  # no regroup to hide them behind: a window ahead

        step(10_000 + k, mid=mid)
        if k + 1 < steps and MATRIX:
            stage_rings(10_000 + k + 1)  # streams during window k+1's regroup
        if os.environ.get("ECCO_E2E_TRACE"):
            print(f"e2e window {k}: host {1e3 * (time.perf_counter() - t0):.1f} ms", file=sys.stderr)
        with torch.cuda.stream(stream):
            best_host.copy_(best_dev, non_blocking=True)  # group assignments back to the host
        if k + 1 < steps:
            ctx.swap_frame_parts(ecco.FRAMES_EVAL)
    ctx.synchronize()
    el_s = time.perf_counter() - t0
    h1, d1 = ctx.transfer_bytes()
    d1 += steps * best_host.numel() * 4
    el_s = reduce_max(dist, [el_s])[0]
    samples = reduce_sum(dist, wl.samples_per_step_local() * steps)
    return {"value": samples / el_s, "unit": "samples/s",
            "h2d_bytes_per_step": (h1 - h0) // steps, "d2h_bytes_per_step": (d1 - d0) // steps,
            "ms_per_step": el_s * 1e3 / steps, "steps": steps,
            "how": ("every window's frames from pinned host buffers on a copy stream, "
                    + ("ecco_stage_frames_range: the full rings of this rank's group members"
                       if args.e2e_full_rings else
                       "ecco_stage_sampled_frames: the ring rows this rank's SGD steps draw, marked "
                       "on the device and read zero-copy over PCIe (rows never drawn are not "
                       "transferred)")
                    + ", all labels and every camera's eval set; double-buffered in two parts "
                    "(ecco_swap_frame_parts): window k+1's eval sets upload during window k and "
                    "its rings from window k's mid-point, current at window k+1's start / before "
                    "its SGD chains + the step + assignments/accuracies read back; wall clock with "
                    "a device synchronize at the end, window 0's unoverlapped eval-set upload "
                    "included"),
            "pcie_gbs": (h1 - h0) / steps / (el_s / steps) / 1e9}


# ------------------------------------------------------------ CPU baselines --

def cpu_sample(N, G, budget_s=12.0):
    """The oracle's restatement of the same step (FFMA-order fp32 C, one
    thread per group) timed on a bounded sample and scaled to the window:
    pairs of the eval matrix and SGD steps measured separately."""
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
    eval_work(1)
    t_pair = time.perf_counter() - t
    t = time.perf_counter()
    train_work(1)
    t_step = time.perf_counter() - t
    per_thread = budget_s / 2.0
    n_pairs = max(1, int(per_thread / max(t_pair, 1e-6)))
    n_steps = max(1, int(per_thread / max(t_step, 1e-6)))
    with ThreadPoolExecutor(cores) as ex:
        t = time.perf_counter()
        list(ex.map(eval_work, [n_pairs] * cores))
        pair_rate = n_pairs * cores / (time.perf_counter() - t)
        t = time.perf_counter()
        list(ex.map(train_work, [n_steps] * cores))
        step_rate = n_steps * cores / (time.perf_counter() - t)
    per = N // G
    steps_window = G * DEPTH * int(GPU_S * STEPS)
    pairs_window = (N * G if MATRIX else 0) + G * (DEPTH + 1) * per  # regroup matrix + chain evaluations
    window_s = pairs_window / pair_rate + steps_window / step_rate
    samples = steps_window * B
    return {"value": samples / window_s, "unit": "samples/s", "cores": cores, "kind": "port",
            "sample": f"{n_pairs * cores} eval pairs (S={S} frames each) and {n_steps * cores} "
                      f"SGD steps (B={B}) of the oracle (oracle/ecco_oracle.c, FFMA-order fp32) on "
                      f"{cores} threads; window = {pairs_window} pairs + {steps_window} steps, "
                      f"scaled from the measured rates",
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
    # (c) the window driver at C4 (10,000 cameras / 500 jobs, W = 1000): GPU
    # only -- the reference needs ~40 s for window 0 there; its numbers, from
    # the same scenario on the same kind of box, are in
    # profiles/r01c_param_window_c4.json (tools/param_window_probe.py)
    sc4 = json.dumps(scenarios.config("c4", windows=2, seed=1))
    sim4 = ecco.Simulation(sc4, backend=ecco.PARAMETRIC)
    w4 = []
    while sim4.step_window():
        w4.append({k: round(v, 3) for k, v in sim4.last_timings().items()})
    sim4.close()
    ref4 = None
    try:
        ref4 = json.load(open(os.path.join(ROOT, "profiles", "r01c_param_window_c4.json")))
        ref4 = ref4.get("reference_window_ms")
    except (OSError, ValueError):
        pass
    out["window_c4"] = {"workload": "c4 scenario (scenarios.config('c4', windows=2, seed=1)), "
                                    "parametric backend; window 0 builds 10,000 profile tables",
                        "gpu_windows": w4, "reference_window_ms_recorded": ref4}
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
    if rank != 0:
        return
    wl = Workload(args.config, 0, 1)
    vals = []
    for _ in range(args.warmup):
        cpu_sample(wl.N, wl.G, budget_s=2.0)
    t0 = time.perf_counter()
    last = None
    for _ in range(args.steps):
        last = cpu_sample(wl.N, wl.G, budget_s=args.ref_budget)
        vals.append(last["value"])
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {
        "impl": "reference",
        "metric": "group-retrain samples/s (per-window regroup + retrain)",
        "value": value, "unit": "samples/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": last["window_s"] * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (counter-RNG camera streams, random-init group MLPs)",
        "config": {"workload": f"{args.config}: {wl.N} cameras / {wl.G} groups (same as the B200 arm)",
                   "cameras": wl.N, "groups": wl.G},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": last["cores"],
                         "kind": "port", "sample": last["sample"]},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": wall,
        "note": "the reference (a C++ simulator) has no learned trainer: its path is the "
                "parametric accuracy model (SURVEY.md 0); the learned path's CPU form is the "
                "oracle restatement, run here on every host core",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--math", default="tf32", choices=["tf32", "ffma"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--ref-budget", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e leg (profiling runs)")
    ap.add_argument("--e2e-full-rings", action="store_true",
                    help="e2e ingest copies every ring of the rank's cameras, not only the drawn rows")
    ap.add_argument("--no-scaling", action="store_true",
                    help="skip the single-GPU emulation of rank 0 at N = 2, 4, 8")
    ap.add_argument("--no-parametric", action="store_true",
                    help="skip the parametric-backend vs reference-library leg")
    args = ap.parse_args()
    global MATRIX
    if args.config == "c5":
        DIMS.update(DET_DIMS)
        MATRIX = False
    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_b200(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
