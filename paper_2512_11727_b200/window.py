"""Group-sharded retraining window: one process per GPU.

One window of the north-star path over groups placed on ranks by cost
(``shard.Placement``), every rank driving its own GPU through the C-ABI:

  regroup   the camera x group evaluation matrix of the rank's groups
            (ecco_eval_matrix_dev, a ModelEvalFn batch of grouping.cpp:33),
            all-gathered across ranks (NCCL over NVLink), then group_request's
            join rule per camera (ecco_route_matrix_ids_dev: highest
            accuracy >= the camera's, ties to the lowest GROUP id whatever
            rank holds it, grouping.cpp:30-39);
  retrain   every local group's speculative chain of `depth` micro-windows
            (ecco_train_trajectories: evaluate, then depth x (train, evaluate),
            the TrainingBackend probes of gpu_allocator.cpp:125-135), the
            trajectories all-gathered, WindowAllocation's greedy
            (gpu_allocator.cpp:100-181) replayed on every rank over ALL groups
            (ecco_allocate_trajectories), and each group's granted prefix
            committed (ecco_commit).

Exactness of the replay: a group whose speculative chain the greedy
exhausts (it is granted more micro-windows than the chain covers) is not
frozen.  The first exhausted group -- found by re-running the replay, whose
prefix up to that pick is exact -- has its chain committed and extended by
its owner (depth doubling, as the window driver csrc/sim.cpp does), the
extension broadcast to every rank, and the replay re-run, until the
schedule touches no accuracy the device did not compute.  So the committed
schedule is WindowAllocation's on the real trajectories, at any world size.

Nothing here depends on the world size but the placement: a group's
trajectory depends on its id, its members' frames (regenerated per rank from
the counter RNG) and its own model; its eval-matrix column on its model and
the cameras' eval sets; the replay on the gathered trajectories.  So the
results are bit-identical at 1, 2, ... ranks (tests/test_gpu_multirank.py).
"""
import math
import os

import numpy as np

from . import FFMA_EXACT, TC_BF16, LEARNED, Context, allocate_trajectories
from .shard import Placement


def learned_steps(batch, gpu_s, throughputs, steps_per_gpu_s):
    """SGD steps one micro-window buys (the learned backend's effort,
    accuracy_model.cpp:80-86: gpu_s x min(1, fps*pix(res)/mean throughput)
    x quality, times steps_per_gpu_s, floored)."""
    fps, res, quality = batch
    if not len(throughputs):
        return 0
    supplied = fps * (res * (16.0 * res / 9.0))
    required = float(np.sum(throughputs)) / len(throughputs)
    suff = min(1.0, supplied / required) if required > 0.0 else 1.0
    effort = gpu_s * suff * quality
    return int(math.floor(effort * steps_per_gpu_s)) if effort > 0.0 else 0


def first_exhausted(jobs, chain_len):
    """Index of the first pick that grants a group a micro-window beyond its
    chain (occurrence count > chain_len[group]), or -1."""
    W = len(jobs)
    if W == 0:
        return -1
    order = np.argsort(jobs, kind="stable")
    sj = jobs[order]
    start = np.r_[0, np.flatnonzero(np.diff(sj)) + 1]
    run = np.diff(np.r_[start, W])
    occ = np.empty(W, np.int64)
    occ[order] = np.arange(W) - np.repeat(start, run) + 1
    over = occ > chain_len[jobs]
    return int(np.argmax(over)) if over.any() else -1


class GroupRetrainer:
    """This rank's share of the group-retraining window.

    scenes / throughput: every camera (replicated on all ranks); groups: the
    member cameras of group g at index g (source mix = members, uniform
    fractions); batch: the (fps, resolution, quality) every group's
    micro-windows deliver; gpu_s: GPU-seconds per micro-window; depth: the
    speculative chain each group trains up front; micro_windows: the
    allocator's budget W (default depth x groups)."""

    def __init__(self, scenes, throughput, groups, *, rank=0, world=1, dist=None, device=0,
                 math=TC_BF16, depth=2, gpu_s=1.0, batch=(30.0, 1080.0, 1.0),
                 steps_per_gpu_s=16.0, micro_windows=None, max_depth=8, alpha=1.0, beta=1.0,
                 bonus=True, policy=0, frames_window=0, dims=None, placement=None):
        import torch
        self.torch = torch
        self.rank, self.world, self.dist = rank, world, dist
        self.groups = [list(m) for m in groups]
        self.G = len(self.groups)
        self.N = len(scenes)
        self.depth, self.gpu_s, self.batch = depth, gpu_s, tuple(batch)
        self.max_depth = max(depth, max_depth)
        self.W = micro_windows if micro_windows is not None else depth * self.G
        self.alpha, self.beta, self.bonus, self.policy = alpha, beta, bonus, policy
        tp = np.asarray(throughput, np.float64)
        self.steps = np.array([learned_steps(self.batch, gpu_s, tp[m], steps_per_gpu_s)
                               for m in self.groups], np.int64)
        dims = dict(dims or {})
        self.B = dims.get("minibatch", 128)
        self.sizes = np.array([len(m) for m in self.groups], np.int32)
        if placement is None:
            placement = Placement(world).place(
                {g: float(self.sizes[g]) * float(max(1, self.steps[g]) * self.B)
                 for g in range(self.G)})
        self.placement = placement
        self.local = placement.groups(rank)
        self.gb = placement.block_size()
        self.dev = torch.device("cuda", device)
        self.ctx = Context(backend=LEARNED, device=device, math=math, max_cameras=self.N,
                           max_jobs=max(1, len(self.local)), max_depth=self.max_depth,
                           steps_per_gpu_s=float(steps_per_gpu_s), **dims)
        self.ctx.set_cameras(np.asarray(scenes, np.float64), tp)
        self.ctx.generate_frames(frames_window)
        self.ctx.seed_models(self.local)
        mem = [self.groups[g] for g in self.local]
        fr = [[1.0 / len(m)] * len(m) for m in mem]
        self.prep = self.ctx.prepare_trajectories(self.local, [self.batch] * len(self.local), mem,
                                                  fr, mem)
        self.cams = np.arange(self.N, dtype=np.int32)
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=self.dev)
        self.M_local = torch.full((self.N, self.gb), float("nan"), dtype=torch.float64,
                                  device=self.dev)
        self.M_part = None if len(self.local) in (0, self.gb) else torch.empty(
            (self.N, len(self.local)), dtype=torch.float64, device=self.dev)
        self.col_ids = torch.from_numpy(placement.column_ids()).to(self.dev)
        self.best = torch.empty(self.N, dtype=torch.int32, device=self.dev)
        self.best_acc = torch.empty(self.N, dtype=torch.float64, device=self.dev)
        self.acc_local = np.zeros((len(self.local), depth + 1))
        self.slot_of = {g: k for k, g in enumerate(self.local)}
        self.stats = {}
        self.host_frames_ptr = 0  # pinned [N][R][F] table of a sampled ingest (set_host_frames)
        self.prev_counts = np.zeros(self.G, np.int64)  # last window's grants (extension depths)

    # ---------------------------------------------------------- collectives --
    def _coll_device(self):
        if self.dist is None:
            return None
        return self.dev if self.dist.get_backend() == "nccl" else self.torch.device("cpu")

    def gather_blocks(self, M):
        """[N, gb] -> [world, N, gb] (all-gather of column blocks)."""
        torch = self.torch
        if self.dist is None or self.world == 1:
            return M.reshape(1, *M.shape)
        cd = self._coll_device()
        src = M if cd.type == "cuda" else M.cpu()
        out = torch.empty((self.world, *M.shape), dtype=M.dtype, device=cd)
        if cd.type == "cuda":
            self.dist.all_gather_into_tensor(out, src.contiguous())
            return out
        self.dist.all_gather(list(out.unbind(0)), src.contiguous())
        return out.to(self.dev)

    def gather_trajectories(self, acc):
        """Local [n_local, depth+1] rows -> [G, depth+1] in group-id order."""
        L = acc.shape[1]
        if self.dist is None or self.world == 1:
            full = np.empty((self.G, L))
            full[self.local] = acc
            return full
        torch = self.torch
        blk = np.zeros((self.gb, L))
        blk[:len(self.local)] = acc
        t = torch.from_numpy(blk).to(self._coll_device())
        out = torch.empty((self.world, self.gb, L), dtype=t.dtype, device=t.device)
        if t.is_cuda:
            self.dist.all_gather_into_tensor(out, t)
        else:
            self.dist.all_gather(list(out.unbind(0)), t)
        rows = out.reshape(self.world * self.gb, L).cpu().numpy()
        ids = self.placement.column_ids()
        full = np.empty((self.G, L))
        full[ids[ids >= 0]] = rows[ids >= 0]
        return full

    def broadcast(self, values, src):
        if self.dist is None or self.world == 1:
            return values
        t = self.torch.from_numpy(np.ascontiguousarray(values, np.float64)).to(self._coll_device())
        self.dist.broadcast(t, src=src)
        return t.cpu().numpy()

    # --------------------------------------------------------------- phases --
    def regroup(self):
        """Enqueues the evaluation matrix, its all-gather and the join rule on
        the context stream; returns (best group id, its accuracy) per camera
        (device tensors, -1 = no group qualifies)."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            if self.local:
                if self.M_part is None:
                    self.ctx.eval_matrix_dev(self.local, self.M_local.data_ptr(), cams=self.cams)
                else:  # fewer groups than the block: columns beyond them stay NaN
                    self.ctx.eval_matrix_dev(self.local, self.M_part.data_ptr(), cams=self.cams)
                    self.M_local[:, :len(self.local)].copy_(self.M_part)
            M = self.gather_blocks(self.M_local)
            self.ctx.route_matrix_ids_dev(self.N, self.gb, M.data_ptr(), self.col_ids.data_ptr(),
                                          self.best.data_ptr(), self.best_acc.data_ptr(),
                                          n_blocks=self.world)
        return self.best, self.best_acc

    def retrain(self, window, mid=None, after_initial=None):
        """Speculative chains, replay over every group, exact extension of
        exhausted chains, commit.  Returns the committed micro-windows per
        group (G,).  With `after_initial`, every local group's first
        micro-window (the initial pass, which always grants each group
        exactly one, gpu_allocator.cpp:160-166) is committed as soon as the
        initial chains have run, and after_initial() is called before the
        greedy remainder (the window step overlaps the regroup matrix with
        it)."""
        if mid is not None:
            mid()
        if self.local:
            self.ctx.train_prepared(self.prep, self.gpu_s, self.depth, window=window,
                                    out=self.acc_local)
        traj = self.gather_trajectories(self.acc_local)
        chain = np.full(self.G, self.depth, np.int64)   # micro-windows each chain covers
        last_d = np.full(self.G, self.depth, np.int64)
        # micro-windows committed before the group's LAST chain started (ecco_commit
        # counts from there); local groups only
        start = np.zeros(self.G, np.int64)
        if after_initial is not None:
            if self.local:
                self.ctx.commit(self.local, [1] * len(self.local))
            after_initial()
        # trajectories as the replay reads them: row g holds the chain's
        # accuracies, padded with its last one (beyond the chain: never read by
        # the final replay); grown in place as chains are extended
        T = np.array(traj, dtype=np.float64, copy=True)
        ids = np.arange(self.G, dtype=np.int32)
        extensions, ext_samples = 0, 0
        fetched = set()  # groups whose remaining rows were topped up this window
        first_ext = set()
        while True:
            jobs, _, _, _ = allocate_trajectories(ids, self.sizes, T, self.alpha, self.beta,
                                                  self.W, self.gpu_s, 1, self.bonus, self.policy)
            p = first_exhausted(jobs, chain)
            if p < 0:
                break
            k = int(jobs[p])
            d = max(1, 2 * int(last_d[k]))
            if k not in first_ext:
                # a group extended last window too is likely to take as many
                # micro-windows again (the greedy's fairness bonus keeps
                # feeding the least accurate group): start its doubling there
                # -- fewer round trips, no effect on the schedule (a chain the
                # greedy does not use up is simply not committed)
                first_ext.add(k)
                d = max(d, int(self.prev_counts[k]) - int(chain[k]))
            d = int(min(self.max_depth, d, self.W - p))
            owner = self.placement.owner[k]
            ext = np.zeros(d + 1)
            if owner == self.rank:
                self.ctx.commit([k], [int(chain[k] - start[k])])
                start[k] = chain[k]
                mem = self.groups[k]
                p1 = self.ctx.prepare_trajectories([k], [self.batch], [mem],
                                                   [[1.0 / len(mem)] * len(mem)], [mem])
                mb = [int(chain[k])]
                if self.host_frames_ptr and k not in fetched:
                    # sampled ingest: the extension's rows were not staged.  The
                    # group's rows for every micro-window the budget could still
                    # give it are fetched at once (one top-up per group and
                    # window, at most its members' rings), not per extension
                    self.ctx.fetch_sampled_host_ptr(p1, self.gpu_s, int(min(self.W - p, 65535)),
                                                    window, self.host_frames_ptr, micro_base=mb)
                    fetched.add(k)
                ext = self.ctx.train_prepared(p1, self.gpu_s, d, window=window, micro_base=mb)[0]
            ext = self.broadcast(ext, owner)
            need = int(chain[k]) + d + 1
            if need > T.shape[1]:
                T = np.concatenate([T, np.repeat(T[:, -1:], need - T.shape[1], axis=1)], axis=1)
            T[k, int(chain[k]) + 1:need] = ext[1:]
            T[k, need:] = ext[-1]
            chain[k] += d
            last_d[k] = d
            extensions += 1
            ext_samples += d * int(self.steps[k]) * self.B
        counts = np.bincount(jobs, minlength=self.G)
        self.prev_counts = counts
        self.traj = T  # the trajectories the final replay read (extensions included)
        self.schedule = jobs
        if self.local:
            self.ctx.commit(self.local, (counts[self.local] - start[self.local]).astype(np.int32))
        self.stats = {"extensions": extensions, "extension_samples": ext_samples,
                      "committed_samples": int((counts * self.steps).sum()) * self.B,
                      "speculative_samples": int(self.depth * self.steps.sum()) * self.B + ext_samples,
                      "max_micro_windows": int(counts.max()) if self.G else 0}
        self.counts = counts
        return counts

    def window(self, window, mid=None, reserve_sms=8, after_launch=None, mark=None):
        """One window in the reference's order -- retrain (initial pass, greedy
        remainder) then the window-end regroup matrix over the trained models
        and the join rule -- with the two overlapped where the data allows:
        once the initial pass is committed, every group's model is final
        unless the greedy trains it again, so the matrix of all groups runs on
        the context's matrix stream (ecco_eval_matrix_dev_async, leaving
        `reserve_sms` SMs) while the greedy's extension chains run on the
        context stream; afterwards the columns of the groups the greedy
        trained beyond their first micro-window are re-evaluated on their
        final models.  The result equals retrain() followed by regroup()
        (tests/test_gpu_multirank.py checks it bit for bit).  after_launch()
        runs right after the matrix is enqueued (e.g. the next window's
        ingest), mark() once the retrain is committed (phase timing).
        Returns (counts, best group per camera, its accuracy)."""
        torch = self.torch
        # the overlap needs a matrix that can run beside the chains: the
        # fused tensor-core evaluation, or FFMA_EXACT's persistent GEMM (on a
        # copy of the committed masters), which leaves whole SMs to the
        # exact chain's cluster of H/16 CTAs
        # (on one or two ranks the exact matrix share -- seconds -- dwarfs the
        # exact chains: keeping SMs from it costs more than the overlap saves;
        # C4 measured: 1 rank 2.54 s without / 3.01 s with, emulated 2 ranks
        # 1.38 / 1.46 s, 4 ranks 0.80 / 0.73 s, 8 ranks 0.51 / 0.37 s)
        math = self.ctx.cfg.math
        exact_overlap = self.world >= 4 or os.environ.get("ECCO_EXACT_OVERLAP") == "1"
        fused = bool(self.local) and (math == TC_BF16 or (math == FFMA_EXACT and exact_overlap))
        if math == FFMA_EXACT:
            reserve_sms = max(reserve_sms, self.ctx.cfg.hidden_dim // 16)

        def launch_matrix():
            if self.local and fused:
                self.ctx.eval_matrix_dev_async(self.local, self._m_target(), self.cams,
                                               reserve_sms=reserve_sms)
            if after_launch is not None:
                after_launch()

        counts = self.retrain(window, mid=mid, after_initial=launch_matrix)
        if mark is not None:
            mark()
        with torch.cuda.stream(self.stream):
            if self.local:
                if fused:
                    self.ctx.matrix_join()
                    redo = [g for g in self.local if counts[g] > 1]
                    if redo:
                        M2 = torch.empty((self.N, len(redo)), dtype=torch.float64, device=self.dev)
                        self.ctx.eval_matrix_dev(redo, M2.data_ptr(), cams=self.cams)
                        cols = torch.tensor([self.slot_of[g] for g in redo], device=self.dev)
                        self._m_view().index_copy_(1, cols, M2)
                    if self.M_part is not None:
                        self.M_local[:, :len(self.local)].copy_(self.M_part)
                else:  # (exact math: no side stream) the matrix after the retrain
                    self.ctx.eval_matrix_dev(self.local, self._m_target(), cams=self.cams)
                    if self.M_part is not None:
                        self.M_local[:, :len(self.local)].copy_(self.M_part)
            M = self.gather_blocks(self.M_local)
            self.ctx.route_matrix_ids_dev(self.N, self.gb, M.data_ptr(), self.col_ids.data_ptr(),
                                          self.best.data_ptr(), self.best_acc.data_ptr(),
                                          n_blocks=self.world)
        return counts, self.best, self.best_acc

    def _m_target(self):
        """Device pointer the local eval matrix is written to ([N, local] contiguous)."""
        return (self.M_local if self.M_part is None else self.M_part).data_ptr()

    def _m_view(self):
        return self.M_local if self.M_part is None else self.M_part

    def set_host_frames(self, frames_ptr):
        """Registers the pinned frame table the window's rings are staged
        from by ecco_stage_sampled_frames (the e2e ingest): extension chains
        top their rows up from it (ecco_fetch_sampled_frames)."""
        self.host_frames_ptr = int(frames_ptr)

    def step(self, window, mid=None):
        """One window (retrain, then the overlapped window-end regroup);
        returns the committed micro-windows per group."""
        return self.window(window, mid=mid)[0]

    def local_samples(self, counts=None):
        """Committed samples of this rank's groups."""
        c = self.counts if counts is None else counts
        return int((c[self.local] * self.steps[self.local]).sum()) * self.B if self.local else 0

    def close(self):
        self.ctx.close()
