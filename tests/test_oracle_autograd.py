"""Pins the learned backend's oracle (oracle/ecco_oracle.c) against an
independent implementation: float64 torch autograd of the same model.

The learned backend has no reference numerics (the reference's
"trainer" is a closed-form proficiency formula), so the FFMA device path is
pinned to the builder's C restatement bit for bit -- and here that
restatement is checked against autograd, so a gradient bug in the oracle
cannot hide behind bit-exact agreement with the device:

* orc_sgd_step (one SGD step of softmax cross-entropy, mean over the
  minibatch) equals W - lr * dL/dW from torch.autograd in float64 to 2e-6 of
  the update (measured 1-4e-7), per tensor (W1, b1, W2, b2), at the bench shape
  F512-H256-C16-B128 and a small shape;
* its returned loss equals autograd's forward loss to 1e-5 relative;
* orc_count_correct equals the count of float64 argmax(logits) == label,
  exactly wherever the top two logits are further apart than fp32 noise.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import OrcLcfg

SHAPES = [dict(F=512, H=256, C=16, B=128), dict(F=128, H=128, C=16, B=64)]


def _setup(orc, shape, lr, seed):
    lc = OrcLcfg(F=shape["F"], H=shape["H"], C=shape["C"], D=2, B=shape["B"], R=256, S=64, lr=lr,
                 noise=1.0, steps_per_gpu_s=16.0, seed=0x5eed0001 + seed)
    F, H, Cc, B = shape["F"], shape["H"], shape["C"], shape["B"]
    P = np.zeros(Cc * F, np.float32)
    Q = np.zeros(Cc * 2 * F, np.float32)
    orc.orc_prototypes(C.byref(lc), P, Q)
    x = np.zeros(B * F, np.uint16)
    y = np.zeros(B, np.int32)
    orc.orc_gen_frames(C.byref(lc), P, Q, seed, 1, 0, B, np.array([0.3, 0.6]), x, y)
    w = [np.zeros(F * H, np.float32), np.zeros(H, np.float32), np.zeros(H * Cc, np.float32),
         np.zeros(Cc, np.float32)]
    orc.orc_init_weights(C.byref(lc), *w)
    rng = np.random.default_rng(seed)  # non-zero biases: every term of the gradient is live
    w[1] = rng.normal(0, 0.1, H).astype(np.float32)
    w[3] = rng.normal(0, 0.1, Cc).astype(np.float32)
    return lc, x, y, w


def _x64(x, B, F):
    return torch.from_numpy((x.astype(np.uint32) << 16).view(np.float32).reshape(B, F)).double()


def _autograd_step(x, y, w, lr, shape):
    F, H, Cc, B = shape["F"], shape["H"], shape["C"], shape["B"]
    X = _x64(x, B, F)
    W1 = torch.tensor(w[0].reshape(F, H), dtype=torch.float64, requires_grad=True)
    b1 = torch.tensor(w[1], dtype=torch.float64, requires_grad=True)
    W2 = torch.tensor(w[2].reshape(H, Cc), dtype=torch.float64, requires_grad=True)
    b2 = torch.tensor(w[3], dtype=torch.float64, requires_grad=True)
    logits = torch.relu(X @ W1 + b1) @ W2 + b2
    loss = torch.nn.functional.cross_entropy(logits, torch.from_numpy(y).long())
    loss.backward()
    with torch.no_grad():
        new = [(p - lr * p.grad).numpy().reshape(-1) for p in (W1, b1, W2, b2)]
    return new, loss.item()


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "F%(F)d-H%(H)d-C%(C)d-B%(B)d" % s)
@pytest.mark.parametrize("seed", [0, 1])
def test_sgd_step_equals_float64_autograd(orc, shape, seed):
    lr = 4.0  # a large step: the update dominates the fp32 rounding of the stored weights
    lc, x, y, w = _setup(orc, shape, lr, seed)
    old = [t.astype(np.float64) for t in w]
    want, want_loss = _autograd_step(x, y, w, lr, shape)
    got = [t.copy() for t in w]
    loss = orc.orc_sgd_step(C.byref(lc), x, y, *got)
    assert abs(loss - want_loss) <= 1e-5 * abs(want_loss)
    for name, g, t, o in zip(("W1", "b1", "W2", "b2"), got, want, old):
        upd = np.abs(t - o).max()
        assert upd > 0, name
        err = np.abs(g.astype(np.float64) - t).max() / upd
        assert err <= 2e-6, (name, err)  # measured 1-4e-7


def test_sgd_step_at_the_bench_learning_rate(orc):
    """At the production learning rate the fp32 weight rounding is added:
    |oracle - autograd| <= 1e-5 of the update + one fp32 ulp of the weight."""
    shape = SHAPES[0]
    import paper_2512_11727_b200 as ecco
    lr = ecco.default_config().sgd_lr
    lc, x, y, w = _setup(orc, shape, lr, 3)
    want, _ = _autograd_step(x, y, w, lr, shape)
    old = [t.copy() for t in w]
    orc.orc_sgd_step(C.byref(lc), x, y, *w)
    for g, t, o in zip(w, want, old):
        upd = np.abs(t - o.astype(np.float64)).max()
        ulp = np.spacing(np.abs(t).astype(np.float32)).astype(np.float64)
        assert (np.abs(g - t) <= 1e-5 * upd + ulp).all()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_count_correct_equals_float64_argmax(orc, seed):
    shape = SHAPES[0]
    F, H, Cc = shape["F"], shape["H"], shape["C"]
    lc, _, _, w = _setup(orc, shape, 0.05, seed)
    S = 64
    P = np.zeros(Cc * F, np.float32)
    Q = np.zeros(Cc * 2 * F, np.float32)
    orc.orc_prototypes(C.byref(lc), P, Q)
    x = np.zeros(S * F, np.uint16)
    y = np.zeros(S, np.int32)
    orc.orc_gen_frames(C.byref(lc), P, Q, 7 + seed, 2, 1, S, np.array([0.2, 0.1]), x, y)
    rng = np.random.default_rng(seed)
    w[0] = (w[0] + rng.normal(0, 0.05, w[0].shape)).astype(np.float32)  # a partly trained model
    w[2] = (w[2] + rng.normal(0, 0.2, w[2].shape)).astype(np.float32)
    got = orc.orc_count_correct(C.byref(lc), x, y, S, *w)
    X = _x64(x, S, F)
    t = [torch.from_numpy(a.astype(np.float64)) for a in w]
    logits = (torch.relu(X @ t[0].reshape(F, H) + t[1]) @ t[2].reshape(H, Cc) + t[3]).numpy()
    top2 = np.sort(logits, 1)[:, -2:]
    clear = (top2[:, 1] - top2[:, 0]) > 1e-4 * np.abs(logits).max()
    correct = logits.argmax(1) == y
    lo, hi = int(correct[clear].sum()), int(correct[clear].sum() + (~clear).sum())
    assert lo <= got <= hi
    assert clear.mean() > 0.9  # the check is not vacuous
