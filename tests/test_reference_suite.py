"""The reference's OWN unit tests (proj/tests/*.cpp: accuracy model,
allocator, grouping, netsim, transmission, scenario, metrics, orchestrator;
96 test cases) compiled with a doctest stand-in (oracle/doctest/doctest.h):
  * against the reference library itself (oracle/_ref/unit_tests_ref): the
    checker build is the reference;
  * with eval / train_step / seed_model running on the B200 build
    (oracle/_ref/unit_tests_b200, oracle/accuracy_model_b200.cpp): the
    reference's known-answer and property tests hold for the device
    arithmetic, and the allocator / grouping / orchestrator suites that call
    it pass unchanged.
Both binaries are built by oracle/Makefile where /root/reference exists and
shipped prebuilt."""
import os
import subprocess

import pytest

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _run(name):
    path = os.path.join(REF, name)
    if not os.path.exists(path):
        pytest.skip(f"oracle/_ref/{name} not built")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "| 0 failed" in r.stdout


def test_reference_unit_suite_on_the_reference():
    _run("unit_tests_ref")


@pytest.mark.gpu
def test_reference_unit_suite_on_the_b200_build():
    _run("unit_tests_b200")


@pytest.mark.gpu
def test_reference_acceptance_suite_on_the_b200_build():
    """acceptance_main.cpp's ten criteria (equivalence to the reference
    allocator on 120 instances, Fig. 7 regroup, determinism, ..., #10 runs
    unit_tests_b200) with the device arithmetic."""
    path = os.path.join(REF, "acceptance_b200")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref/acceptance_b200 not built")
    r = subprocess.run([path], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "FAIL" not in r.stdout
