"""Pins the CPU oracle (oracle/ecco_oracle.c) before it is trusted as the checker.

1. Known-answer tests copied from the reference's own doctest suite
   (proj/tests/test_accuracy_model.cpp, test_transmission.cpp) -- same inputs,
   same expected values, same 1e-12 tolerance.
2. Bit-exact agreement with the unmodified reference library
   (oracle/_ref/libecco_ref.so) on randomised inputs, and with the committed
   golden vectors tests/golden/kat_param.npz generated from it.
"""
import ctypes as C
import math
import os

import numpy as np
import pytest

import oracle
from conftest import GOLD

P = oracle.default_params()


def approx(a, b, eps=1e-12):
    # doctest::Approx(b).epsilon(eps): |a-b| <= eps * (1 + max(|a|,|b|))
    return abs(a - b) <= eps * (1.0 + max(abs(a), abs(b)))


def d(*v):
    return np.array(v, dtype=np.float64)


def train(orc, k, clusters, prof, centroid, fps, res, q, gpu_s, src_scenes, src_tp, src_frac,
          kmax=8):
    D = len(centroid) if centroid is not None else 2
    kk = C.c_int(k)
    cl = np.zeros((kmax, D))
    cl[:k] = np.array(clusters).reshape(k, D) if k else 0
    pr = np.zeros(kmax)
    pr[:k] = prof
    clen = C.c_int(len(centroid) if centroid is not None else 0)
    ce = np.zeros(D)
    if centroid is not None:
        ce[:] = centroid
    rc = orc.orc_train_step(C.byref(kk), cl.reshape(-1), pr, C.byref(clen), ce, kmax, D, fps, res,
                            q, gpu_s, len(src_frac), np.array(src_scenes, float).reshape(-1),
                            np.array(src_tp, float), np.array(src_frac, float),
                            oracle.orc_params(P))
    return rc, kk.value, cl[:kk.value], pr[:kk.value], clen.value, ce


# ---- 1. reference KATs (proj/tests/test_accuracy_model.cpp) ----

def test_similarity_kat(orc):
    # test_accuracy_model.cpp:40-44
    assert approx(orc.orc_similarity(d(0, 0), d(0.3, 0.4), 2, 0.5), 0.36787944117144233)


def test_eval_kats(orc):
    # test_accuracy_model.cpp:66-92
    pp = oracle.orc_params(P)
    cl, pr, ce = d(0, 0), d(0.4), d(0, 0)
    assert approx(orc.orc_eval(1, cl, pr, 2, ce, 2, d(0, 0), pp), 0.30)
    assert approx(orc.orc_eval(1, cl, pr, 2, ce, 2, d(0.02, 0), pp), 0.29215788783046465)
    assert orc.orc_eval(1, cl, pr, 2, ce, 2, d(0.9, 0.9), pp) == P["acc_floor"]
    assert orc.orc_eval(0, cl, pr, 0, ce, 2, d(0, 0), pp) == P["acc_floor"]


def test_cluster_threshold_and_ties(orc):
    # test_accuracy_model.cpp:114-143
    pp = oracle.orc_params(P)
    d_in, d_out = -0.5 * math.log(0.95), -0.5 * math.log(0.85)
    assert orc.orc_find_cluster(1, d(0, 0), 2, d(d_in, 0), pp) == 0
    assert orc.orc_find_cluster(1, d(0, 0), 2, d(d_out, 0), pp) == -1
    assert orc.orc_find_cluster(2, d(0.2, 0, 0.2, 0), 2, d(0.2, 0), pp) == 0
    rc, k, cl, pr, _, _ = train(orc, 1, [0, 0], [0.5], [0, 0], 5, 360, 1, 60, [[d_out, 0]],
                                [8.192e6], [1.0])
    assert rc == 0 and k == 2 and pr[1] > 0 and list(cl[1]) == [d_out, 0]


def test_train_single_source_kat(orc):
    # test_accuracy_model.cpp:145-168
    rc, k, cl, pr, clen, ce = train(orc, 1, [0, 0], [0.4], [0, 0], 5.0, 360.0, 1.0, 60.0,
                                    [[0, 0]], [8.192e6], [1.0])
    assert rc == 0 and approx(pr[0], 0.606510393237099)
    assert list(ce) == [0.0, 0.0]
    acc = orc.orc_eval(k, cl.reshape(-1).copy(), pr.copy(), clen, ce, 2, d(0, 0), oracle.orc_params(P))
    assert approx(acc, 0.40325519661854947)


def test_train_two_source_kat(orc):
    # test_accuracy_model.cpp:170-199
    rc, k, cl, pr, clen, ce = train(orc, 1, [0, 0], [0.2], [0, 0], 10.0, 480.0, 0.5, 30.0,
                                    [[0, 0], [1, 0]], [8.192e6, 8.192e6], [0.75, 0.25])
    assert rc == 0 and k == 2
    assert approx(pr[0], 0.39612831840879403) and approx(pr[1], 0.08948963861996584)
    assert list(cl[1]) == [1.0, 0.0]
    assert approx(ce[0], 0.25) and approx(ce[1], 0.0)


def test_train_zero_effort_and_validation(orc):
    # test_accuracy_model.cpp:201-222, 295-317
    for q, g, src in ((0.0, 60.0, [1.0]), (1.0, 0.0, [1.0])):
        rc, k, cl, pr, _, ce = train(orc, 1, [0, 0], [0.3], [0, 0], 5, 360, q, g, [[0, 0]], [8.192e6], src)
        assert rc == 0 and k == 1 and pr[0] == 0.3
    rc, *_ = train(orc, 1, [0, 0], [0.3], [0, 0], 5, 360, 1, 60, np.zeros((0, 2)), [], [])
    assert rc == 0
    assert train(orc, 0, [], [], None, 5, 360, 1, -1.0, [[0, 0]], [8.192e6], [1.0])[0] == 1
    assert train(orc, 0, [], [], None, 5, 360, 1, 10.0, [[0, 0]], [8.192e6], [0.4])[0] == 1


def test_seed_reproduces_device_accuracy(orc):
    # test_accuracy_model.cpp:319-337
    rng = np.random.default_rng(3)
    pp = oracle.orc_params(P)
    for _ in range(50):
        sc = rng.random(2)
        acc = rng.uniform(0.1, 0.6)
        cl, pr = np.zeros(2), np.zeros(1)
        orc.orc_seed_model(sc, 2, acc, pp, cl, pr)
        assert approx(orc.orc_eval(1, cl, pr, 2, sc.copy(), 2, sc, pp), acc)
    cl, pr = np.zeros(2), np.zeros(1)
    orc.orc_seed_model(d(0.5, 0.5), 2, 0.01, pp, cl, pr)
    assert pr[0] == 0.0
    orc.orc_seed_model(d(0.5, 0.5), 2, 0.99, pp, cl, pr)
    assert pr[0] == 1.0


# ---- 2. bit-exact against the reference library ----

def test_eval_matches_golden_vectors(orc):
    z = np.load(os.path.join(GOLD, "kat_param.npz"))
    pp = oracle.orc_params(P)
    for i in range(len(z["ev"])):
        v = orc.orc_eval(int(z["ks"][i]), np.ascontiguousarray(z["cl"][i]).reshape(-1),
                         np.ascontiguousarray(z["pr"][i]), int(z["clen"][i]),
                         np.ascontiguousarray(z["ce"][i]), 2, np.ascontiguousarray(z["sc"][i]), pp)
        assert v == z["ev"][i], i


def test_train_step_matches_reference(orc, ref):
    rng = np.random.default_rng(7)
    pa = oracle.params_array(P)
    for trial in range(300):
        K0 = int(rng.integers(0, 4))
        kmax = 12
        D = 2
        cl = np.zeros((kmax, D))
        cl[:K0] = rng.random((K0, D))
        pr = np.zeros(kmax)
        pr[:K0] = rng.random(K0)
        ce = rng.random(D)
        clen = D if rng.random() < 0.9 else 0
        ns = int(rng.integers(1, 6))
        sc = rng.random((ns, D))
        for s in range(ns):
            if K0 and rng.random() < 0.5:
                sc[s] = cl[rng.integers(0, K0)] + rng.normal(0, 0.02, D)
        tp = rng.uniform(1e6, 1e7, ns)
        fr = rng.random(ns) + 0.05
        fr = fr / fr.sum()
        fps, res, q, g = rng.choice([1, 2, 5, 10, 15]), rng.choice([360, 480, 720, 960]), rng.random(), rng.uniform(0, 60)
        outs = []
        for lib, is_ref in ((ref, True), (orc, False)):
            kk, cc = C.c_int(K0), C.c_int(clen)
            c2, p2, e2 = cl.copy(), pr.copy(), ce.copy()
            if is_ref:
                rc = lib.ref_train_step(C.byref(kk), c2.reshape(-1), p2, C.byref(cc), e2, kmax, D,
                                        fps, res, q, g, ns, sc.reshape(-1).copy(), tp, fr, pa)
            else:
                rc = lib.orc_train_step(C.byref(kk), c2.reshape(-1), p2, C.byref(cc), e2, kmax, D,
                                        fps, res, q, g, ns, sc.reshape(-1).copy(), tp, fr,
                                        oracle.orc_params(P))
            outs.append((rc, kk.value, c2.tobytes(), p2.tobytes(), cc.value, e2.tobytes()))
        assert outs[0] == outs[1], trial


def test_profile_tables_match_reference(orc, ref):
    rng = np.random.default_rng(11)
    pa = oracle.params_array(P)
    fps = [1, 2, 5, 10, 15]
    res = [360, 480, 720, 960]
    gf = np.array([f for f in fps for _ in res], float)
    gq = np.array([q for _ in fps for q in res], float)
    W = 10
    levels = np.array([k * 6.0 for k in range(1, W + 1)])
    for trial in range(40):
        sc = rng.random(2)
        tp = rng.uniform(2e6, 2e7)
        bias = int(rng.integers(0, 2))
        rr = rng.choice([2e5, 1e6, 5e6])
        outs = []
        for lib, is_ref in ((ref, True), (orc, False)):
            ob, of, oq = np.zeros(W), np.zeros(W), np.zeros(W)
            fe = np.zeros(W, np.uint8)
            if is_ref:
                rc = lib.ref_profile_table(sc, 2, tp, bias, W, levels, 20, gf, gq, 60.0, 1e-9, rr,
                                           0.1, pa, ob, of, oq, fe)
            else:
                rc = lib.orc_profile_table(sc, 2, tp, bias, W, levels, 20, gf, gq, 60.0, 1e-9, rr,
                                           0.1, oracle.orc_params(P), ob, of, oq, fe)
            outs.append((rc, ob.tobytes(), of.tobytes(), oq.tobytes(), fe.tobytes()))
        assert outs[0] == outs[1], trial


def test_eval_matrix_matches_reference(orc, ref):
    rng = np.random.default_rng(5)
    pa = oracle.params_array(P)
    n, g, kmax, D = 60, 9, 4, 2
    ks = rng.integers(0, kmax + 1, g).astype(np.int32)
    cl = rng.random((g, kmax, D))
    pr = rng.random((g, kmax))
    ce = rng.random((g, D))
    clen = np.full(g, D, np.int32)
    sc = rng.random((n, D))
    a, b = np.zeros(n * g), np.zeros(n * g)
    ref.ref_eval_matrix(n, sc.reshape(-1), g, ks, cl.reshape(-1), pr.reshape(-1), clen,
                        ce.reshape(-1), kmax, D, pa, a)
    orc.orc_eval_matrix(n, sc.reshape(-1), g, ks, cl.reshape(-1), pr.reshape(-1), clen,
                        ce.reshape(-1), kmax, D, oracle.orc_params(P), b)
    assert a.tobytes() == b.tobytes()
