"""N>1 host path on CPU: world_size-2 gloo process group (one process per
"GPU" as bench.py runs under torchrun).  Covers the group sharding, the
all-gather of evaluation-matrix column blocks in the blocked layout the
device argmax reads, the routing decision on the gathered matrix, and the
max-over-ranks timing / summed-samples reductions of bench.py."""
import os
import socket

import numpy as np
import pytest

from paper_2512_11727_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _full_matrix(n, g, seed=0):
    rng = np.random.default_rng(seed)
    M = np.round(rng.random((n, g)) * 8) / 8  # many ties
    M[1, :] = np.nan                          # a camera no group may take
    return M


def _worker(rank, world, port, n, g, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = _full_matrix(n, g)
        gb = shard.block_size(g, world)
        mine = shard.rank_groups(g, world, rank)
        local = torch.full((n, gb), float("nan"), dtype=torch.float64)
        if mine:
            local[:, :len(mine)] = torch.from_numpy(full[:, mine])
        blocks = shard.gather_blocks(local, world, dist)
        got_full = shard.blocked_to_full(blocks.numpy(), g)
        best, acc = shard.route_reference(got_full, req=np.full(n, 0.25))
        # bench.py's reductions: max of per-rank device time, sum of samples
        t = torch.tensor([10.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        s = torch.tensor([float(len(mine) * 100)], dtype=torch.float64)
        dist.all_reduce(s)
        q.put((rank, mine, got_full, best, acc, t.item(), s.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,g", [(2, 7), (2, 8), (3, 5)])
def test_sharded_gather_and_route_match_single_rank(world, g):
    import torch.multiprocessing as mp
    n = 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, g, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _full_matrix(n, g)
    want_best, want_acc = shard.route_reference(full, req=np.full(n, 0.25))
    owned = sorted(j for r in res for j in r[1])
    assert owned == list(range(g))  # every group on exactly one rank
    for rank, mine, got_full, best, acc, tmax, samples in res:
        assert all(shard.owner(j, g, world) == rank for j in mine)
        np.testing.assert_array_equal(got_full, full)  # NaN-equal
        np.testing.assert_array_equal(best, want_best)
        np.testing.assert_array_equal(acc, want_acc)
        assert tmax == 10.0 + world - 1
        assert samples == g * 100


def test_block_layout_column_mapping():
    g, world = 500, 8
    gb = shard.block_size(g, world)
    assert gb == 63
    cols = [j for r in range(world) for j in shard.rank_groups(g, world, r)]
    assert cols == list(range(g))
    # gathered column b*gb + jb is group b*gb + jb: the device argmax index is
    # the global group id directly
    for r in range(world):
        for jb, j in enumerate(shard.rank_groups(g, world, r)):
            assert r * gb + jb == j


def test_cost_balanced_placement():
    """shard.Placement: LPT by members x samples, ties to the
    lowest rank / lowest group id; new groups by the same rule; drops give
    the load back; the gathered column map lists every group once."""
    from paper_2512_11727_b200.shard import Placement
    sizes = [12, 4, 8, 6, 10, 8, 5, 7]
    costs = {g: float(n * 64) for g, n in enumerate(sizes)}
    pl = Placement(2).place(costs)
    assert pl.owner[0] == 0 and pl.owner[4] == 1  # the two largest first, lowest rank first
    loads = [sum(costs[g] for g in pl.groups(r)) for r in range(2)]
    assert loads == pl.load
    assert abs(loads[0] - loads[1]) <= max(costs.values())
    assert Placement(2).place(costs).owner == pl.owner  # deterministic
    least = int(np.argmin(pl.load)) if pl.load[0] != pl.load[1] else 0
    assert pl.add(99, 1.0) == least
    pl.drop(99)
    assert pl.load == loads
    ids = pl.column_ids()
    gb = pl.block_size()
    assert len(ids) == 2 * gb and sorted(ids[ids >= 0].tolist()) == list(range(len(sizes)))
    for r in range(2):
        assert ids[r * gb:r * gb + len(pl.groups(r))].tolist() == pl.groups(r)
    # equal costs: round robin in id order
    eq = Placement(3).place({g: 1.0 for g in range(7)})
    assert [eq.owner[g] for g in range(7)] == [0, 1, 2, 0, 1, 2, 0]
    with pytest.raises(ValueError):
        eq.add(3, 1.0)


def test_first_exhausted_pick():
    from paper_2512_11727_b200.window import first_exhausted
    chain = np.array([2, 2, 2])
    assert first_exhausted(np.array([0, 1, 2, 0, 1, 2]), chain) == -1
    assert first_exhausted(np.array([0, 1, 0, 2, 0, 1, 1]), chain) == 4  # job 0's third pick
    assert first_exhausted(np.array([], np.int64), chain) == -1
    assert first_exhausted(np.array([1, 1, 1]), np.array([2, 5, 2])) == -1
