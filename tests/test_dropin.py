"""The reference-side C++ binding (include/ecco_b200_dropin.hpp) inside the
UNMODIFIED reference library: the reference's own WindowAllocation and
group_request, driven once by its JobTrainingBackend / eval_job_on_scene
semantics and once by ecco_b200::CudaTrainingBackend / make_eval_fn on the
GPU, must produce identical schedules, trained models and assignments
(oracle/dropin_test.cpp, built by oracle/Makefile where /root/reference
exists and shipped prebuilt)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/dropin_test not built")
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_reference_allocator_and_router_over_the_dropin(seed):
    r = subprocess.run([BIN, str(seed), "9"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [x for x in r.stdout.splitlines() if x.startswith("trial")]
    assert len(lines) == 9 and all(x.endswith("identical") for x in lines)
    assert all("profile rows" in x for x in lines)


LEARNED_BIN = os.path.join(os.path.dirname(BIN), "dropin_learned_test")


@pytest.mark.skipif(not os.path.exists(LEARNED_BIN), reason="oracle/_ref/dropin_learned_test not built")
@pytest.mark.parametrize("seed", [1, 2])
def test_reference_allocator_and_router_over_the_learned_dropin(seed):
    """The learned backend behind the same seams: the reference's
    WindowAllocation over ecco_b200::CudaTrainingBackend (FFMA math) equals it
    over the CPU oracle's trainer, schedule and weights bit for bit; its
    group_request over ecco_b200::BatchedRouter equals the oracle eval_fn's
    assignments (oracle/dropin_learned_test.cpp)."""
    r = subprocess.run([LEARNED_BIN, str(seed), "6"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    lines = [x for x in r.stdout.splitlines() if x.startswith("trial")]
    assert len(lines) == 6 and all(x.endswith("identical") for x in lines)
