"""Multi-rank group retraining on the device.

Two ranks (gloo process group, both on the one GPU of the test box -- the
collectives go through host memory, the kernels are the product's) run the
group-sharded window of paper_2512_11727_b200/window.py over a cost-balanced
placement; a single rank runs the same windows.  Everything a window decides
or trains must be bit-identical: the routed group of every camera and its
accuracy, the trajectories the allocator replay read (extension chains
included), the schedule, and every group's committed weights.  The budget
W = 3 x groups with depth-2 chains forces chain extensions (the exact
replay of window.py), so the owner-trains / broadcast path runs too.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = dict(feat_dim=512, hidden_dim=256, num_classes=16, minibatch=128, ring_frames=128,
            eval_samples=64)
SIZES = [12, 4, 8, 6, 10, 8, 5, 7]  # unequal groups: the placement balances members x samples
WINDOWS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _layout():
    groups, c = [], 0
    for n in SIZES:
        groups.append(list(range(c, c + n)))
        c += n
    scenes = np.array([[0.1 * (g % 5), 0.2 * (g // 5)] for g, m in enumerate(groups) for _ in m])
    return groups, scenes, np.full(c, 8.192e6)


def _worker(rank, world, port, q, mode="split", exact=False):
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2512_11727_b200 import FFMA_EXACT, TC_BF16
        from paper_2512_11727_b200.window import GroupRetrainer
        groups, scenes, tp = _layout()
        r = GroupRetrainer(scenes, tp, groups, rank=rank, world=world, dist=dist, device=0,
                           math=FFMA_EXACT if exact else TC_BF16, depth=2,
                           micro_windows=3 * len(groups),
                           steps_per_gpu_s=4.0, dims=DIMS)
        out = []
        for w in range(WINDOWS):
            if mode == "split":  # retrain, then the window-end regroup, in sequence
                counts = r.retrain(w + 1)
                best, acc = r.regroup()
            else:  # the overlapped window (matrix beside the greedy's extension chains)
                counts, best, acc = r.window(w + 1)
            torch.cuda.synchronize()
            out.append({"best": best.cpu().numpy(), "acc": acc.cpu().numpy(), "counts": counts,
                        "traj": r.traj.copy(), "schedule": r.schedule.copy(),
                        "extensions": r.stats["extensions"]})
        weights = {g: [a.tobytes() for a in r.ctx.get_weights(g)] for g in r.local}
        q.put((rank, r.local, out, weights))
        r.close()
    finally:
        if dist is not None:
            dist.destroy_process_group()


def _spawn(world, mode="split", exact=False):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, mode, exact))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("mode", ["split", "window"])
def test_two_ranks_bit_identical_to_one(mode):
    """split: retrain() then regroup() per window, 1 rank vs 2 ranks;
    window: the overlapped GroupRetrainer.window() on 2 ranks vs the split
    sequence on 1 rank (the overlap must not change a bit)."""
    one = _spawn(1)[0]
    two = _spawn(2, mode)
    if mode == "window":
        two = two + _spawn(1, mode)  # and the overlapped window on a single rank
    owned = sorted(g for _, local, _, _ in two[:2] for g in local)
    assert owned == list(range(len(SIZES)))  # every group on exactly one rank
    assert all(local for _, local, _, _ in two[:2])  # both ranks hold groups
    ext = 0
    for w in range(WINDOWS):
        a = one[2][w]
        for _, _, out, _ in two:
            b = out[w]
            assert a["best"].tobytes() == b["best"].tobytes(), w
            assert a["acc"].tobytes() == b["acc"].tobytes(), w
            assert a["traj"].tobytes() == b["traj"].tobytes(), w
            assert (a["schedule"] == b["schedule"]).all() and (a["counts"] == b["counts"]).all()
        ext += a["extensions"]
    assert ext > 0  # the exact replay extended chains (W > depth x groups)
    for _, local, _, weights in two:
        for g in local:
            assert weights[g] == one[3][g], g



def test_exact_window_overlap_bit_identical(monkeypatch):
    """FFMA_EXACT (the oracle-exact math): the overlapped window -- the
    persistent FFMA GEMM (forced on) evaluating a copy of the committed
    masters on the matrix stream beside the exact chains, extended groups
    re-evaluated -- equals retrain() then regroup(), on 1 and 2 ranks."""
    monkeypatch.setenv("ECCO_FFMA_HIDDEN8", "1")
    monkeypatch.setenv("ECCO_EXACT_OVERLAP", "1")  # (the product overlaps from 4 ranks on)
    one = _spawn(1, "split", exact=True)[0]
    runs = _spawn(2, "window", exact=True) + _spawn(1, "window", exact=True)
    ext = 0
    for w in range(WINDOWS):
        a = one[2][w]
        for _, _, out, _ in runs:
            b = out[w]
            assert a["best"].tobytes() == b["best"].tobytes(), w
            assert a["acc"].tobytes() == b["acc"].tobytes(), w
            assert a["traj"].tobytes() == b["traj"].tobytes(), w
            assert (a["schedule"] == b["schedule"]).all() and (a["counts"] == b["counts"]).all()
        ext += a["extensions"]
    assert ext > 0
    for _, local, _, weights in runs:
        for g in local:
            assert weights[g] == one[3][g], g
