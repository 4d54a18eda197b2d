"""Allocator decisions (WindowAllocation, core/src/gpu_allocator.cpp:100-181)
of the window driver vs the UNMODIFIED reference (oracle/_ref) on the same
accuracy trajectories: every micro-window record (job, accuracy before,
after) and the initial scores must be bit-identical, under all three
policies, including the ties that counts/64 accuracies produce.  Host code
only: runs without a GPU.  (the device proposes
trajectories, the host replays the reference's decision code.)"""
import numpy as np
import pytest

import oracle
import paper_2512_11727_b200 as ecco

pytestmark = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


def _ref(ids, members, traj, alpha, beta, W, mu, gpus, bonus, policy):
    n, L = traj.shape
    job = np.zeros(W, np.int32)
    b, a, init = np.zeros(W), np.zeros(W), np.zeros(n)
    st = oracle.ref().ref_allocate_trajectories(
        n, np.ascontiguousarray(ids, np.int32), np.ascontiguousarray(members, np.int32),
        np.ascontiguousarray(traj), L, alpha, beta, W, mu, gpus, int(bonus), policy, job, b, a,
        init)
    return st, job, b, a, init


def _case(rng, n, L, quantized):
    ids = rng.choice(10 * n + 10, n, replace=False).astype(np.int32)
    members = rng.integers(1, 25, n).astype(np.int32)
    if quantized:  # learned accuracies: member-mean of counts/64 -> many exact ties
        steps = rng.integers(0, 3, (n, L)) / 64.0
        traj = np.minimum(0.1 + np.cumsum(steps, 1), 1.0)
    else:
        traj = np.cumsum(rng.random((n, L)) * 0.05, 1)
    return ids, members, traj


@pytest.mark.parametrize("policy", [0, 1, 2])
@pytest.mark.parametrize("quantized", [False, True])
def test_decisions_bit_identical(policy, quantized):
    rng = np.random.default_rng(17 + policy + 10 * quantized)
    for trial in range(30):
        n = int(rng.integers(1, 40))
        L = int(rng.integers(1, 12))
        W = int(rng.integers(n, 3 * n + 5))
        ids, members, traj = _case(rng, n, L, quantized)
        alpha, beta = float(rng.choice([0.0, 0.5, 1.0, 2.0])), float(rng.choice([0.5, 1.0, -0.5]))
        bonus = bool(rng.integers(0, 2))
        st, rj, rb, ra, ri = _ref(ids, members, traj, alpha, beta, W, 0.6, 2, bonus, policy)
        assert st == 0
        gj, gb, ga, gi = ecco.allocate_trajectories(ids, members, traj, alpha, beta, W, 0.6, 2,
                                                    bonus, policy)
        assert (gj == rj).all() and gb.tobytes() == rb.tobytes() and ga.tobytes() == ra.tobytes()
        if policy != 1:
            assert gi.tobytes() == ri.tobytes()


# The driver's picks come from tournament trees (O(log J) per micro-window);
# at the bench's scale (J = 500, W = 1000) and with NaN trajectories (which
# fall back to the scans) they must still be the reference's.
@pytest.mark.parametrize("policy", [0, 2])
@pytest.mark.parametrize("quantized", [False, True])
def test_decisions_bit_identical_at_scale(policy, quantized):
    rng = np.random.default_rng(91 + policy + quantized)
    for trial in range(3):
        n, L = 500, 3
        ids, members, traj = _case(rng, n, L, quantized)
        if trial == 2:
            traj[rng.integers(0, n, 3), rng.integers(0, L, 3)] = np.nan
        for bonus in (True, False):
            st, rj, rb, ra, ri = _ref(ids, members, traj, 1.0, 0.5, 2 * n, 1.0, 1, bonus, policy)
            assert st == 0
            gj, gb, ga, gi = ecco.allocate_trajectories(ids, members, traj, 1.0, 0.5, 2 * n, 1.0,
                                                        1, bonus, policy)
            assert (gj == rj).all() and gb.tobytes() == rb.tobytes() and ga.tobytes() == ra.tobytes()


def test_reference_kat_sequences():
    # test_gpu_allocator.cpp:155-176: three equal jobs, one better trajectory
    ids = np.array([1, 2, 3], np.int32)
    traj = np.array([[0.1, 0.2, 0.25, 0.27, 0.28], [0.1, 0.3, 0.45, 0.55, 0.6],
                     [0.1, 0.15, 0.17, 0.18, 0.19]])
    for policy in (0, 1, 2):
        st, rj, rb, ra, _ = _ref(ids, [2, 2, 2], traj, 1.0, 1.0, 8, 6.0, 1, True, policy)
        gj, gb, ga, _ = ecco.allocate_trajectories(ids, [2, 2, 2], traj, 1.0, 1.0, 8, 6.0, 1, True,
                                                   policy)
        assert (gj == rj).all() and gb.tobytes() == rb.tobytes()


def test_errors_like_the_reference():
    t = np.zeros((2, 3))
    with pytest.raises(ecco.InfeasibleScheduleError):
        ecco.allocate_trajectories([1, 2], [1, 1], t, micro_windows=1)
    with pytest.raises(ecco.InvalidArgument):
        ecco.allocate_trajectories([1, 1], [1, 1], t)
    with pytest.raises(ecco.InvalidArgument):
        ecco.allocate_trajectories([1, 2], [0, 1], t)
    with pytest.raises(ecco.InvalidArgument):
        ecco.allocate_trajectories([1, 2], [1, 1], t, beta=1.5)
