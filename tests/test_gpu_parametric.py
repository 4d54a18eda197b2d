"""Parity of the parametric backend's CUDA kernels with the oracle (bit-exact).

K1 eval matrix / sparse pairs / fused route proposal, K2 trajectories +
commit, K3 profile tables, the exp port on 1e7 device samples, and the error
mapping of the C-ABI.  All comparisons are on the raw fp64 bits.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2512_11727_b200 as ecco

pytestmark = pytest.mark.gpu
P = oracle.default_params()


def make_ctx(**kw):
    return ecco.Context(backend=ecco.PARAMETRIC, max_clusters=8, max_jobs=1024, max_cameras=4096,
                        max_depth=16, **kw)


def random_models(rng, g, kmax=8, D=2):
    ks = rng.integers(0, 5, g).astype(np.int32)
    cl = rng.random((g, kmax, D))
    pr = rng.random((g, kmax))
    ce = rng.random((g, D))
    clen = np.where(rng.random(g) < 0.9, D, 0).astype(np.int32)
    return ks, cl, pr, ce, clen


def oracle_matrix(orc, scenes, models, kmax=8, D=2):
    ks, cl, pr, ce, clen = models
    n, g = len(scenes), len(ks)
    out = np.zeros(n * g)
    orc.orc_eval_matrix(n, np.ascontiguousarray(scenes).reshape(-1), g, ks, cl.reshape(-1),
                        pr.reshape(-1), clen, ce.reshape(-1), kmax, D, oracle.orc_params(P), out)
    return out.reshape(n, g)


def test_eval_matrix_golden_vectors():
    import os
    from conftest import GOLD
    z = np.load(os.path.join(GOLD, "kat_param.npz"))
    ctx = make_ctx()
    n = len(z["ev"])
    K = 8
    cl = np.zeros((n, K, 2))
    cl[:, :4] = z["cl"]
    pr = np.zeros((n, K))
    pr[:, :4] = z["pr"]
    ids = np.arange(n, dtype=np.int32)
    ctx.put_models(ids, z["ks"], cl, pr, z["ce"], z["clen"])
    got = ctx.eval_pairs(ids, scenes=z["sc"])
    assert got.tobytes() == z["ev"].tobytes()


def test_eval_matrix_bit_exact(orc):
    rng = np.random.default_rng(1)
    ctx = make_ctx()
    g, n = 37, 300
    models = random_models(rng, g)
    ids = np.arange(100, 100 + g, dtype=np.int32)
    ctx.put_models(ids, *models)
    scenes = rng.random((n, 2))
    # half of the scenes near a model's cluster so the 0.9 threshold matters
    for i in range(0, n, 2):
        j = rng.integers(0, g)
        if models[0][j]:
            scenes[i] = models[1][j, rng.integers(0, models[0][j])] + rng.normal(0, 0.02, 2)
    got = ctx.eval_matrix(ids, scenes=scenes)
    want = oracle_matrix(orc, scenes, models)
    assert got.tobytes() == want.tobytes()
    mask = (rng.random((n, g)) < 0.5).astype(np.uint8)
    gm = ctx.eval_matrix(ids, scenes=scenes, mask=mask)
    assert np.all(np.isnan(gm[mask == 0]))
    assert gm[mask == 1].tobytes() == want[mask == 1].tobytes()


@pytest.mark.parametrize("lam", [0.3, 0.25, 1.0])
def test_eval_matrix_bit_exact_any_lambda(orc, lam):
    """similarity's -sqrt(d)/lambda: a power-of-two lambda runs as an exact
    multiply by 1/lambda (param_model.cuh), any other as the division; both
    equal the oracle (and so the reference) bit for bit, over a matrix large
    enough that every block walks several probe rows."""
    rng = np.random.default_rng(11)
    ctx = make_ctx(params=dict(similarity_lambda=lam))
    g, n = 45, 1500
    models = random_models(rng, g)
    ids = np.arange(g, dtype=np.int32)
    ctx.put_models(ids, *models)
    scenes = rng.random((n, 2))
    for i in range(0, n, 3):
        j = rng.integers(0, g)
        if models[0][j]:
            scenes[i] = models[1][j, rng.integers(0, models[0][j])] + rng.normal(0, 0.01, 2)
    got = ctx.eval_matrix(ids, scenes=scenes)
    ks, cl, pr, ce, clen = models
    want = np.zeros(n * g)
    orc.orc_eval_matrix(n, np.ascontiguousarray(scenes).reshape(-1), g, ks, cl.reshape(-1),
                        pr.reshape(-1), clen, ce.reshape(-1), 8, 2,
                        oracle.orc_params(dict(P, similarity_lambda=lam)), want)
    assert got.tobytes() == want.tobytes()


def test_route_propose_matches_sequential_scan(orc):
    rng = np.random.default_rng(2)
    ctx = make_ctx()
    g, n = 64, 200
    models = random_models(rng, g)
    ids = np.arange(g, dtype=np.int32)
    ctx.put_models(ids, *models)
    scenes = rng.random((n, 2))
    want = oracle_matrix(orc, scenes, models)
    req = rng.uniform(0.1, 0.4, n)
    mask = (rng.random((n, g)) < 0.7).astype(np.uint8)
    # duplicate a column so exact ties must go to the lowest column
    best, acc = ctx.route_propose(ids, req, scenes=scenes, mask=mask)
    for i in range(n):
        b, ba = -1, 0.0
        for j in range(g):  # grouping.cpp:30-39
            if not mask[i, j] or want[i, j] < req[i]:
                continue
            if b < 0 or want[i, j] > ba:
                b, ba = j, want[i, j]
        assert best[i] == b and (b < 0 or acc[i] == ba)


def _traj_inputs(rng, n_jobs, n_cams):
    members, sources, fracs, batches = [], [], [], []
    for j in range(n_jobs):
        m = sorted(rng.choice(n_cams, rng.integers(1, 6), replace=False).tolist())
        members.append(m)
        s = sorted(set(m) | set(rng.choice(n_cams, rng.integers(0, 2), replace=False).tolist()))
        f = rng.random(len(s)) + 0.1
        fracs.append((f / f.sum()).tolist())
        sources.append(s)
        batches.append((float(rng.choice([1, 2, 5, 10, 15])), float(rng.choice([360, 480, 720, 960])),
                        float(rng.random())))
    return members, sources, fracs, batches


def test_trajectories_and_commit_bit_exact(orc):
    rng = np.random.default_rng(3)
    ctx = make_ctx()
    n_cams, n_jobs, depth, K, D = 64, 40, 6, 8, 2
    scenes = rng.random((n_cams, D))
    tp = rng.uniform(2e6, 2e7, n_cams)
    ctx.set_cameras(scenes, tp)
    ks, cl, pr, ce, clen = random_models(rng, n_jobs)
    ks[:] = np.minimum(ks, 2)
    ids = np.arange(n_jobs, dtype=np.int32) * 3 + 1
    ctx.put_models(ids, ks, cl, pr, ce, clen)
    members, sources, fracs, batches = _traj_inputs(rng, n_jobs, n_cams)
    got = ctx.train_trajectories(ids, batches, sources, fracs, members, 6.0, depth)
    # oracle: same chains on host copies
    so = np.zeros(n_jobs + 1, np.int32)
    so[1:] = np.cumsum([len(s) for s in sources])
    mo = np.zeros(n_jobs + 1, np.int32)
    mo[1:] = np.cumsum([len(m) for m in members])
    k2, c2, p2, e2, l2 = ks.copy(), cl.copy(), pr.copy(), ce.copy(), clen.copy()
    want = np.zeros((n_jobs, depth + 1))
    rc = orc.orc_param_trajectories(
        n_jobs, k2, c2.reshape(-1), p2.reshape(-1), l2, e2.reshape(-1), K, D, scenes.reshape(-1), tp,
        np.array(batches, float).reshape(-1), so, np.array(sum(sources, []), np.int32),
        np.array(sum(fracs, []), float), mo, np.array(sum(members, []), np.int32), 6.0, depth,
        oracle.orc_params(P), want.reshape(-1))
    assert rc == 0
    assert got.tobytes() == want.tobytes()
    # commit a different prefix per job; the committed state must equal the
    # oracle after that many steps
    granted = rng.integers(0, depth + 1, n_jobs).astype(np.int32)
    ctx.commit(ids, granted)
    gk, gc, gp, ge, gl = ctx.get_models(ids)
    for j in range(n_jobs):
        kk, cc = C.c_int(int(ks[j])), C.c_int(int(clen[j]))
        c3, p3, e3 = cl[j].copy(), pr[j].copy(), ce[j].copy()
        for _ in range(granted[j]):
            src = sources[j]
            orc.orc_train_step(C.byref(kk), c3.reshape(-1), p3, C.byref(cc), e3, K, D, *batches[j], 6.0,
                               len(src), np.ascontiguousarray(scenes[src]).reshape(-1), tp[src],
                               np.array(fracs[j]), oracle.orc_params(P))
        assert gk[j] == kk.value and gl[j] == cc.value
        assert gp[j, :kk.value].tobytes() == p3[:kk.value].tobytes()
        assert ge[j].tobytes() == e3.tobytes()
        assert gc[j, :kk.value].tobytes() == c3[:kk.value].tobytes()


def test_eval_jobs_is_trajectory_column_zero():
    rng = np.random.default_rng(4)
    ctx = make_ctx()
    n_cams = 32
    ctx.set_cameras(rng.random((n_cams, 2)), rng.uniform(2e6, 2e7, n_cams))
    ks, cl, pr, ce, clen = random_models(rng, 10)
    ks[:] = np.minimum(ks, 2)
    ids = np.arange(10, dtype=np.int32)
    ctx.put_models(ids, ks, cl, pr, ce, clen)
    members, sources, fracs, batches = _traj_inputs(rng, 10, n_cams)
    ev = ctx.eval_jobs(ids, members)
    tr = ctx.train_trajectories(ids, batches, sources, fracs, members, 6.0, 1)
    assert ev.tobytes() == np.ascontiguousarray(tr[:, 0]).tobytes()


def test_profile_tables_bit_exact(orc):
    rng = np.random.default_rng(5)
    ctx = make_ctx()
    n_cams, W = 300, 25
    scenes = rng.random((n_cams, 2))
    tp = rng.uniform(2e6, 2e7, n_cams)
    ctx.set_cameras(scenes, tp)
    fps, res = [1, 2, 5, 10, 15], [360, 480, 720, 960]
    gf = np.array([f for f in fps for _ in res], float)
    gq = np.array([q for _ in fps for q in res], float)
    levels = np.array([k * 2.4 for k in range(W, 0, -1)])  # unsorted on purpose
    bias = rng.integers(0, 2, n_cams).astype(np.int32)
    cams = np.arange(n_cams, dtype=np.int32)
    ob, of, oq, fe = ctx.profile_tables(cams, levels, gf, gq, 60.0, bias=bias)
    for c in range(n_cams):
        b, f, q, e = np.zeros(W), np.zeros(W), np.zeros(W), np.zeros(W, np.uint8)
        assert orc.orc_profile_table(scenes[c].copy(), 2, tp[c], int(bias[c]), W, levels, 20, gf, gq,
                                     60.0, 1e-9, 1e6, 0.1, oracle.orc_params(P), b, f, q, e) == 0
        assert (ob[c].tobytes(), of[c].tobytes(), oq[c].tobytes(), fe[c].tobytes()) == \
               (b.tobytes(), f.tobytes(), q.tobytes(), e.tobytes()), c


def test_seed_and_rename():
    ctx = make_ctx()
    ctx.seed_models([7, 8], scenes=[[0.2, 0.2], [0.5, 0.1]], device_acc=[0.3, 0.05])
    k, cl, pr, ce, clen = ctx.get_models([7, 8])
    assert list(k) == [1, 1] and pr[0, 0] == (0.3 - 0.1) / 0.5 and pr[1, 0] == 0.0
    ctx.rename_models([7], [70])
    assert ctx.get_models([70])[2][0, 0] == pr[0, 0]
    with pytest.raises(ecco.InvalidArgument):
        ctx.get_models([7])


def test_error_mapping():
    ctx = make_ctx()
    ctx.set_cameras(np.zeros((2, 2)), np.full(2, 8.192e6))
    ctx.seed_models([1], scenes=[[0.0, 0.0]], device_acc=[0.2])
    with pytest.raises(ecco.InvalidArgument, match="negative gpu_time"):
        ctx.train_trajectories([1], [(5, 360, 1)], [[0]], [[1.0]], [[0]], -1.0, 1)
    with pytest.raises(ecco.InvalidArgument, match="sum to 1"):
        ctx.train_trajectories([1], [(5, 360, 1)], [[0]], [[0.4]], [[0]], 6.0, 1)
    with pytest.raises(ecco.InvalidArgument, match="missing"):
        ctx.train_trajectories([1], [(5, 360, 1)], [[9]], [[1.0]], [[0]], 6.0, 1)
    with pytest.raises(ecco.InvalidArgument):
        ctx.profile_tables([0], [], [1.0], [360.0], 60.0)
    with pytest.raises(ecco.InvalidArgument):
        ctx.profile_tables([0], [6.0, -1.0], [1.0], [360.0], 60.0)


def test_exp_port_on_device_matches_libm():
    """The device exp is exercised through similarity: eval on a 1-cluster
    model at prof 1 is floor + span * exp(-d/l) * exp(-d/l); instead compare
    p_similarity-driven evals on 1e6 random scenes with the oracle (libm)."""
    rng = np.random.default_rng(6)
    ctx = make_ctx()
    import oracle as O
    orc = O.oracle()
    n = 1_000_000
    scenes = rng.random((n, 2)) * 6.0 - 3.0
    ctx.put_models([0], [1], np.zeros((1, 8, 2)), np.ones((1, 8)), np.zeros((1, 2)), [2])
    got = ctx.eval_pairs(np.zeros(n, np.int32), scenes=scenes)
    want = np.zeros(n)
    orc.orc_eval_matrix(n, scenes.reshape(-1), 1, np.array([1], np.int32), np.zeros(16), np.ones(8),
                        np.array([2], np.int32), np.zeros(2), 8, 2, O.orc_params(P), want)
    assert got.tobytes() == want.tobytes()
