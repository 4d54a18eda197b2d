"""The wide fused evaluation kernel (k_eval_wide, eval_kernels.cu): the
camera x group counts of models whose 128-row X tile does not fit in shared
memory -- the detection head of BASELINE configs[4] (F1024-H1024-C96) and
any F % 64 == 0 -- with X streamed beside the model.

Numerics are those of the resident kernel (tests/test_gpu_fused_eval.py):
X exact in bf16, W1 / W2 / relu(Z + b1) rounded to bf16, fp32 accumulation
in TMEM.  `_emulate` restates that in float64; logits must agree to
accumulation-order noise (|diff| <= 4e-2 absolute here: K = 1024 and 1024
hidden terms, twice the resident kernel's sums), counts within 2 of the
emulated argmax with mean <= 0.2.  Pairs-mode tiles reproduce the dense
entries bit for bit, and a capped grid (many tiles per CTA: the pipeline's
stage / W2 / bias / TMEM phases across tiles) equals the full grid bitwise.
"""
import numpy as np
import pytest

import paper_2512_11727_b200 as ecco

pytestmark = pytest.mark.gpu

DET = dict(feat_dim=1024, hidden_dim=1024, num_classes=96, minibatch=128, ring_frames=64,
           eval_samples=64)
# odd shape: 9 K chunks, 3 hidden halves (odd), C = 48 (two logits buffers)
ODD = dict(feat_dim=576, hidden_dim=384, num_classes=48, minibatch=128, ring_frames=64,
           eval_samples=64)


def _bf16(a):
    a = np.asarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16 << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def _emulate(dims, x, w):
    F, H, C = dims["feat_dim"], dims["hidden_dim"], dims["num_classes"]
    w1, b1, w2, b2 = w
    Z = x.astype(np.float64) @ _bf16(w1.reshape(F, H)) + b1.astype(np.float64)
    R = _bf16(np.maximum(Z, 0.0).astype(np.float32))
    return R @ _bf16(w2.reshape(H, C)) + b2.astype(np.float64)


def _ctx(dims, n_cams, seed, max_jobs=16):
    ctx = ecco.Context(backend=ecco.LEARNED, math=ecco.TC_BF16, max_cameras=64,
                       max_jobs=max_jobs, max_depth=2, **dims)
    rng = np.random.default_rng(seed)
    scenes = np.round(rng.random((n_cams, 2)), 1)
    ctx.set_cameras(scenes, np.full(n_cams, 8.192e6))
    ctx.generate_frames(1)
    return ctx, rng


def _random_models(ctx, rng, ids):
    ctx.seed_models(ids)
    models = {}
    for j in ids:
        w1, b1, w2, b2 = ctx.get_weights(j)
        w1 = (w1 + rng.normal(0, 0.02, w1.shape)).astype(np.float32)
        b1 = rng.normal(0, 0.1, b1.shape).astype(np.float32)
        w2 = (w2 + rng.normal(0, 0.05, w2.shape)).astype(np.float32)
        b2 = rng.normal(0, 0.1, b2.shape).astype(np.float32)
        ctx.set_weights(j, w1, b1, w2, b2)
        models[j] = (w1.reshape(-1), b1, w2.reshape(-1), b2)  # API layout W1[F][H]
    return models


def _frames(ctx, n):
    _, _, ev, el = ctx.read_frames(n)
    x = (ev.astype(np.uint32) << 16).view(np.float32)
    return x, el


@pytest.mark.parametrize("dims", [DET, ODD], ids=["det", "odd"])
def test_wide_logits_match_bf16_emulation(dims):
    n_cams, ids = 5, [3, 1, 4]  # odd camera count: the last tile half padded
    ctx, rng = _ctx(dims, n_cams, 0)
    models = _random_models(ctx, rng, ids)
    cams = np.arange(n_cams)[::-1].copy()
    got = ctx.debug_eval_logits(ids, cams)
    x, _ = _frames(ctx, n_cams)
    for jj, j in enumerate(ids):
        for ii, c in enumerate(cams):
            want = _emulate(dims, x[c], models[j])
            err = np.abs(got[ii, :, jj, :] - want).max()
            assert err <= 4e-2, (j, c, err)


@pytest.mark.parametrize("dims", [DET, ODD], ids=["det", "odd"])
def test_wide_counts_match_emulated_argmax(dims):
    n_cams, ids = 7, [0, 1, 2, 3, 4]
    ctx, rng = _ctx(dims, n_cams, 1)
    models = _random_models(ctx, rng, ids)
    M = ctx.eval_matrix(ids, cams=np.arange(n_cams))
    x, el = _frames(ctx, n_cams)
    S = dims["eval_samples"]
    want = np.zeros((n_cams, len(ids)))
    for jj, j in enumerate(ids):
        for c in range(n_cams):
            want[c, jj] = (np.argmax(_emulate(dims, x[c], models[j]), 1) == el[c]).sum()
    diff = np.abs(M * S - want)
    assert diff.max() <= 2 and diff.mean() <= 0.2, (diff.max(), diff.mean())
    assert (M * S == np.round(M * S)).all()


def test_wide_pairs_equal_dense_matrix():
    n_cams, ids = 10, [2, 9, 4]
    ctx, rng = _ctx(DET, n_cams, 2)
    _random_models(ctx, rng, ids)
    M = ctx.eval_matrix(ids, cams=np.arange(n_cams))
    members = [[0, 3, 5], [1, 2, 4, 6, 7], [8, 9]]
    got = ctx.eval_jobs(ids, members)
    for jj, m in enumerate(members):
        want = 0.0
        for c in m:
            want += M[c, jj]
        assert got[jj] == want / len(m)
    pj = [ids[k % 3] for k in range(7)]
    pc = list(range(7))
    got = ctx.eval_pairs(pj, cams=pc)
    for k in range(7):
        assert got[k] == M[pc[k], ids.index(pj[k])]


@pytest.mark.parametrize("cap", [1, 2, 5])
def test_wide_multi_tile_regime_equals_full_grid(cap, monkeypatch):
    """Many tiles per persistent CTA (ECCO_EVAL_MAX_CTAS): the stage ring,
    W2^T / bias buffers and TMEM Z / R / logits phases carried across tiles
    and entries give the same counts as one tile per CTA."""
    n_cams, ids = 19, [0, 1, 2, 3, 4, 5]  # 10 tiles x 6 entries
    ctx, rng = _ctx(DET, n_cams, 4)
    _random_models(ctx, rng, ids)
    full = ctx.eval_matrix(ids, cams=np.arange(n_cams))
    monkeypatch.setenv("ECCO_EVAL_MAX_CTAS", str(cap))
    capped = ctx.eval_matrix(ids, cams=np.arange(n_cams))
    assert capped.tobytes() == full.tobytes()


def test_wide_fused_counts_close_to_general_path(monkeypatch):
    """The fused kernel against the general (unfused) path it replaces (bf16
    forward, fp32 CUDA-core head on unrounded R): decisions differ only where
    bf16 rounding of R flips an argmax."""
    n_cams, ids = 6, [0, 1, 2]
    ctx, rng = _ctx(DET, n_cams, 5)
    models = _random_models(ctx, rng, ids)
    a = ctx.eval_matrix(ids, cams=np.arange(n_cams)) * 64
    monkeypatch.setenv("ECCO_EVAL_WIDE", "0")
    ctx2, _ = _ctx(DET, n_cams, 5)
    ctx2.seed_models(ids)
    for j in ids:
        w1, b1, w2, b2 = models[j]
        ctx2.set_weights(j, w1, b1, w2, b2)
    b = ctx2.eval_matrix(ids, cams=np.arange(n_cams)) * 64
    diff = np.abs(a - b)
    assert diff.max() <= 3 and diff.mean() <= 0.5, (diff.max(), diff.mean())


# edges: S = 128 (a tile is one camera's frames), C = 128 (the logits take
# the last TMEM columns), F = 64 (one K chunk), H = 128 (one hidden half)
EDGE = [dict(feat_dim=1024, hidden_dim=256, num_classes=128, minibatch=128, ring_frames=64,
             eval_samples=128),
        dict(feat_dim=64, hidden_dim=128, num_classes=80, minibatch=128, ring_frames=64,
             eval_samples=64)]


@pytest.mark.parametrize("dims", EDGE, ids=["s128_c128", "f64_h128"])
def test_wide_edges_match_bf16_emulation(dims):
    n_cams, ids = 3, [0, 2]
    ctx, rng = _ctx(dims, n_cams, 6)
    models = _random_models(ctx, rng, ids)
    got = ctx.debug_eval_logits(ids, np.arange(n_cams))
    x, el = _frames(ctx, n_cams)
    M = ctx.eval_matrix(ids, cams=np.arange(n_cams))
    S = dims["eval_samples"]
    for jj, j in enumerate(ids):
        for c in range(n_cams):
            want = _emulate(dims, x[c], models[j])
            assert np.abs(got[c, :, jj, :] - want).max() <= 4e-2, (j, c)
            cnt = (np.argmax(want, 1) == el[c]).sum()
            assert abs(M[c, jj] * S - cnt) <= 2, (j, c)
