"""Network model of the window driver vs the UNMODIFIED reference
(core/src/netsim.cpp:64-94 through oracle/_ref): per-flow mean rates must be
bit-identical, including congestion-test ties (sum(rates) == capacity), for
which the guarded parallel sum falls back to the reference's sequential sum.
Host code only: runs without a GPU."""
import numpy as np
import pytest

import oracle
import paper_2512_11727_b200 as ecco

pytestmark = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


def _ref(alpha, beta, caps, capacity, rtt, dur):
    out = np.zeros(len(alpha))
    st = oracle.ref().ref_simulate_window(len(alpha), np.ascontiguousarray(alpha),
                                          np.ascontiguousarray(beta), np.ascontiguousarray(caps),
                                          capacity, rtt, dur, out)
    assert st == 0
    return out


@pytest.mark.parametrize("n", [1, 3, 8, 37, 1000, 10000])
def test_random_flows_bit_identical(n):
    rng = np.random.default_rng(n)
    alpha = rng.uniform(1e3, 5e5, n)
    beta = np.full(n, 0.5) if n % 2 else rng.uniform(0.1, 0.9, n)
    caps = np.where(rng.random(n) < 0.3, 0.0, rng.uniform(1e5, 5e6, n))
    capacity = float(rng.uniform(0.2, 0.8) * n * 2e6)
    got, _ = ecco.netsim_mean_rates(alpha, beta, caps, capacity, 0.05, 60.0)
    want = _ref(alpha, beta, caps, capacity, 0.05, 60.0)
    assert got.tobytes() == want.tobytes()


def test_exact_ties_take_the_sequential_sum():
    # every flow pinned at a cap of 1e6 and the capacity equal to their sum:
    # total == capacity exactly, which the reference counts as congestion (>=)
    for n in (8, 100, 4096):
        alpha = np.full(n, 2.5e5)
        beta = np.full(n, 0.5)
        caps = np.full(n, 1e6)
        got, exact = ecco.netsim_mean_rates(alpha, beta, caps, n * 1e6, 0.05, 30.0)
        want = _ref(alpha, beta, caps, n * 1e6, 0.05, 30.0)
        assert got.tobytes() == want.tobytes()
        assert exact > 0


def test_invalid_arguments_raise_like_the_reference():
    with pytest.raises(ecco.InvalidArgument):
        ecco.netsim_mean_rates([0.0], [0.5], [0.0], 1e6, 0.05, 1.0)
    with pytest.raises(ecco.InvalidArgument):
        ecco.netsim_mean_rates([1.0], [1.0], [0.0], 1e6, 0.05, 1.0)
    with pytest.raises(ecco.InvalidArgument):
        ecco.netsim_mean_rates([1.0], [0.5], [0.0], 0.0, 0.05, 1.0)
