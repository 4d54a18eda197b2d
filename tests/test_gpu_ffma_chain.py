"""The fused FP32 SGD chain (ffma_chain.cu): the oracle-exact math
(FFMA_EXACT) in one launch per micro-window on a cluster of H/16 CTAs.

Bar: bit-exact.  Trajectories, committed weights and losses equal the CPU
oracle's (orc_sgd_step, oracle/ecco_oracle.c) and the general per-step FFMA
kernels' (ECCO_FFMA_CHAIN=0) bit for bit -- with jobs of unequal step
budgets (including idle jobs), in serial mode (one job, several
micro-windows in one launch) and at other shapes (H = 128, F = 128)."""
import numpy as np
import pytest

import paper_2512_11727_b200 as ecco

from test_gpu_learned import BENCH, setup

pytestmark = pytest.mark.gpu


def _jobs(n, members_per=2, fps=None):
    ids = list(range(3, 3 + n))
    members = [[(2 * k + i) % 6 for i in range(members_per)] for k in range(n)]
    fracs = [[1.0 / members_per] * members_per] * n
    fps = fps or [30.0] * n
    batches = [(f, 1080.0, 1.0) for f in fps]
    return ids, members, fracs, batches


def _run(ctx, ids, members, fracs, batches, depth, window=3):
    ctx.seed_models(ids)
    got = ctx.train_trajectories(ids, batches, members, fracs, members, 1.0, depth, window=window)
    losses = ctx.last_losses(ids, depth)
    ctx.commit(ids, [depth] * len(ids))
    return got, losses, [ctx.get_weights(j) for j in ids]


# fps 30: sufficiency 1 (16 steps); 0.1: 0 steps (idle job); 2.0: 8 steps
@pytest.mark.parametrize("fps", [[30.0, 30.0, 30.0], [30.0, 0.1, 2.0]], ids=["equal", "unequal"])
def test_ffma_chain_equals_oracle_and_per_step_kernels(fps, monkeypatch):
    ids, members, fracs, batches = _jobs(3, fps=fps)
    ctx, orc, _ = setup(seed=41, **BENCH)
    got, losses, weights = _run(ctx, ids, members, fracs, batches, 2)
    # the oracle
    for j in ids:
        orc.seed(j)
    want = orc.trajectories(ids, batches, members, fracs, members, 1.0, 2)
    assert got.tobytes() == want.tobytes()
    orc.commit(ids, [2] * len(ids))
    for j, w in zip(ids, weights):
        for a, b in zip(w, orc.models[j]):
            assert a.reshape(-1).tobytes() == b.tobytes(), j
    # the per-step FFMA kernels (incl. the losses the oracle does not keep)
    monkeypatch.setenv("ECCO_FFMA_CHAIN", "0")
    ctx2, _, _ = setup(seed=41, **BENCH)
    got2, losses2, weights2 = _run(ctx2, ids, members, fracs, batches, 2)
    assert got.tobytes() == got2.tobytes()
    assert np.array_equal(losses, losses2, equal_nan=True)
    for w, w2 in zip(weights, weights2):
        for a, b in zip(w, w2):
            assert a.tobytes() == b.tobytes()


def test_ffma_serial_chain_equals_per_micro_window_launches(monkeypatch):
    """One job, depth 4: serial mode (one launch, snapshots written at the
    micro-window ends, one batched evaluation) vs one launch per
    micro-window."""
    ids, members, fracs, batches = _jobs(1, members_per=3)
    ctx, _, _ = setup(seed=42, **BENCH)
    got, losses, weights = _run(ctx, ids, members, fracs, batches, 4)
    monkeypatch.setenv("ECCO_NO_SERIAL_CHAIN", "1")
    ctx2, _, _ = setup(seed=42, **BENCH)
    got2, losses2, weights2 = _run(ctx2, ids, members, fracs, batches, 4)
    assert got.tobytes() == got2.tobytes()
    assert np.array_equal(losses, losses2, equal_nan=True)
    for a, b in zip(weights[0], weights2[0]):
        assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("hidden,feat", [(128, 256), (256, 128)])
def test_ffma_chain_other_cluster_sizes(hidden, feat, monkeypatch):
    """H = 128 (8-CTA clusters, 16 owned rows per CTA) and F = 128 against
    the per-step FFMA kernels bit for bit."""
    dims = dict(BENCH, hidden_dim=hidden, feat_dim=feat)
    ids, members, fracs, batches = _jobs(2)
    ctx, _, _ = setup(seed=43, **dims)
    got, losses, weights = _run(ctx, ids, members, fracs, batches, 2)
    monkeypatch.setenv("ECCO_FFMA_CHAIN", "0")
    ctx2, _, _ = setup(seed=43, **dims)
    got2, losses2, weights2 = _run(ctx2, ids, members, fracs, batches, 2)
    assert got.tobytes() == got2.tobytes()
    assert np.array_equal(losses, losses2, equal_nan=True)
    for w, w2 in zip(weights, weights2):
        for a, b in zip(w, w2):
            assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("fused,wide,t16", [("1", "1", "1"), ("0", "1", "1"), ("0", "1", "0"),
                                            ("0", "0", "1")])
@pytest.mark.parametrize("feat", [512, 128])
def test_ffma_eval_matrix_hidden_tiles_bit_exact(fused, wide, t16, feat, monkeypatch):
    """The FFMA evaluation matrix through the fused per-pair kernel
    (k_l_eval_ffma_fused: hidden layer, head, argmax, count in one block) and,
    with it disabled, through the chunked kernels with the wide-grid hidden
    tiles forced on (8 x 16 per thread, k_l_hidden_ffma16, or 8 x 8,
    k_l_hidden_ffma8) and with the 4 x 8 one: all equal the oracle's counts
    bit for bit."""
    monkeypatch.setenv("ECCO_FFMA_FUSED_EVAL", fused)
    monkeypatch.setenv("ECCO_FFMA_HIDDEN8", wide)
    monkeypatch.setenv("ECCO_FFMA_HIDDEN16", t16)
    ctx, orc, _ = setup(seed=44, **dict(BENCH, feat_dim=feat))
    ids = [2, 5, 6]
    ctx.seed_models(ids)
    for j in ids:
        orc.seed(j)
    members, fracs = [[0, 1], [2, 3], [4, 5]], [[0.5, 0.5]] * 3
    batches = [(30.0, 1080.0, 1.0)] * 3
    ctx.train_trajectories(ids, batches, members, fracs, members, 1.0, 1, window=3)
    orc.trajectories(ids, batches, members, fracs, members, 1.0, 1)
    ctx.commit(ids, [1, 1, 1])
    orc.commit(ids, [1, 1, 1])
    M = ctx.eval_matrix(ids, cams=np.arange(6))
    W = np.array([[orc.count(orc.models[j], c) / 64 for j in ids] for c in range(6)])
    assert M.tobytes() == W.tobytes()


@pytest.mark.parametrize("tile", ["2", "3", "64"])
def test_ffma_eval_matrix_group_tiles_and_mask(tile, monkeypatch):
    """The evaluation matrix's pairs are ordered in group tiles (ECCO_PAIR_TILE
    groups, cameras outer): with several tiles, a ragged last tile and a
    mask, every unmasked entry equals the oracle's count bit for bit and
    every masked one is NaN (through k_l_eval_ffma_fused at the bench shape,
    and through the chunked kernels with it disabled)."""
    monkeypatch.setenv("ECCO_PAIR_TILE", tile)
    ctx, orc, rng = setup(seed=45, **BENCH)
    ids = [1, 3, 4, 6, 9]
    ctx.seed_models(ids)
    for j in ids:
        orc.seed(j)
    members = [[0, 1], [2, 3], [4, 5], [1, 2], [3, 4]]
    fracs = [[0.5, 0.5]] * 5
    batches = [(30.0, 1080.0, 1.0), (2.0, 1080.0, 1.0), (30.0, 1080.0, 1.0), (0.1, 1080.0, 1.0),
               (30.0, 1080.0, 1.0)]
    ctx.train_trajectories(ids, batches, members, fracs, members, 1.0, 1, window=3)
    orc.trajectories(ids, batches, members, fracs, members, 1.0, 1)
    ctx.commit(ids, [1] * 5)
    orc.commit(ids, [1] * 5)
    want = np.array([[orc.count(orc.models[j], c) / 64 for j in ids] for c in range(6)])
    mask = (rng.random((6, 5)) < 0.7).astype(np.uint8)
    mask[0, :] = 0
    for fused in ("1", "0"):
        monkeypatch.setenv("ECCO_FFMA_FUSED_EVAL", fused)
        M = ctx.eval_matrix(ids, cams=np.arange(6))
        assert M.tobytes() == want.tobytes(), fused
        Mm = ctx.eval_matrix(ids, cams=np.arange(6), mask=mask)
        assert np.isnan(Mm[mask == 0]).all()
        assert Mm[mask == 1].tobytes() == want[mask == 1].tobytes(), fused
