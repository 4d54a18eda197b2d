"""Group sharding across ranks (one process per GPU).

Groups (jobs) are independent: a job's model depends only on its own batches
(proj/core/src/orchestrator.cpp:52-62; the reference's ScriptedBackend,
proj/tests/support/scripted_backend.hpp:17-42, shows the allocator needs
nothing but per-job trajectories).  So every rank owns a contiguous block of
groups, trains and evaluates only those, and the only exchange is the
all-gather of the camera x group evaluation matrix column blocks (NCCL over
NVLink on the GPU path; gloo in the CPU tests).  Cameras are replicated: each
rank regenerates their frames from the counter RNG, so no frame moves.
``Placement`` is the product's cost-balanced placement (window.py uses it);
the contiguous blocks below are the equal-cost special case.

The gathered matrix keeps the blocked layout [rank][camera][column of the
rank's block]; ecco_route_matrix_dev reads it directly (column j = b*gb + jb),
so no transpose kernel runs between the collective and the argmax.
"""
import numpy as np


class Placement:
    """Deterministic cost-balanced group -> rank placement.

    A group's cost is its share of the window's device work, members x
    samples (its eval-matrix column and member evaluations scale with the
    members, its SGD chain with the samples it trains).  Groups are placed
    longest-processing-time first -- descending cost, ties by ascending group
    id -- each on the least-loaded rank, ties to the lowest rank; a group
    created later (new_job, grouping.cpp:56-60) is placed by the same rule
    against the current loads, and a terminated group (orchestrator.cpp:375)
    gives its load back.  Placed groups never move, so no model weights
    cross ranks.  Every rank computes the same placement from the same
    inputs, so nothing about it is communicated."""

    def __init__(self, world):
        if world < 1:
            raise ValueError("placement: world size must be >= 1")
        self.world = world
        self.load = [0.0] * world
        self.owner = {}
        self.cost = {}

    def add(self, group, cost):
        if group in self.owner:
            raise ValueError(f"placement: group {group} already placed")
        r = min(range(self.world), key=lambda k: (self.load[k], k))
        self.owner[group] = r
        self.cost[group] = float(cost)
        self.load[r] += float(cost)
        return r

    def place(self, costs):
        """Places every group of {group: cost} (LPT order)."""
        for g in sorted(costs, key=lambda g: (-float(costs[g]), g)):
            self.add(g, costs[g])
        return self

    def drop(self, group):
        r = self.owner.pop(group)
        self.load[r] -= self.cost.pop(group)

    def groups(self, rank):
        """The rank's groups in ascending id (its column order)."""
        return sorted(g for g, r in self.owner.items() if r == rank)

    def block_size(self):
        return max(1, max(len(self.groups(r)) for r in range(self.world)))

    def column_ids(self):
        """Group id of every column of the gathered [world][block] layout
        (-1 = padding), the map ecco_route_matrix_ids_dev reads."""
        gb = self.block_size()
        ids = np.full(self.world * gb, -1, np.int32)
        for r in range(self.world):
            g = self.groups(r)
            ids[r * gb:r * gb + len(g)] = g
        return ids


def block_size(n_groups, world):
    """Columns per rank: ceil(G / world); the last block may be ragged and is
    padded with NaN (masked) columns."""
    return -(-n_groups // world)


def rank_groups(n_groups, world, rank):
    """Contiguous block of group indices owned by `rank`."""
    gb = block_size(n_groups, world)
    lo, hi = rank * gb, min(n_groups, (rank + 1) * gb)
    return list(range(lo, max(lo, hi)))


def owner(group, n_groups, world):
    """Rank that owns `group`."""
    return group // block_size(n_groups, world)


def gather_blocks(local, world, dist=None):
    """All-gather one [n, gb] column block per rank into [world, n, gb]
    (torch tensors; NCCL on CUDA tensors, gloo on CPU tensors)."""
    import torch
    if world == 1 or dist is None:
        return local.reshape(1, *local.shape)
    out = torch.empty((world, *local.shape), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local.contiguous())
    else:
        parts = list(out.unbind(0))
        dist.all_gather(parts, local.contiguous())
    return out


def blocked_to_full(blocks, n_groups):
    """[world, n, gb] -> [n, G] (host-side view for checks and the CPU path)."""
    w, n, gb = blocks.shape
    return np.concatenate([np.asarray(blocks[b]) for b in range(w)], axis=1)[:, :n_groups]


def route_reference(full, req=None):
    """group_request's join rule (grouping.cpp:30-39) on a full matrix: per
    row the lowest column maximising the accuracy among non-NaN entries >=
    req (strict > between candidates); -1 when none qualifies.  The device
    kernel (ecco_route_matrix_dev) is checked against this in the GPU tests."""
    n, g = full.shape
    best = np.full(n, -1, np.int32)
    acc = np.zeros(n)
    for i in range(n):
        r = 0.0 if req is None else req[i]
        for j in range(g):
            a = full[i, j]
            if a != a or a < r:
                continue
            if best[i] < 0 or a > acc[i]:
                best[i], acc[i] = j, a
    return best, acc
