"""Shared fixtures.  `-m gpu` tests need a B200 (run through gpurun); the
rest run on CPU.  Oracle libraries are built on demand (they are test
infrastructure, see oracle/__init__.py)."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLD = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    if not os.path.exists(oracle.ORACLE_SO):
        oracle.build(ref=False)
    return oracle.oracle()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.have_ref():
        if os.path.isdir(oracle.REFERENCE_ROOT):
            oracle.build()
        else:
            pytest.skip("reference library not built and /root/reference absent")
    return oracle.ref()


def scenario_names():
    d = os.path.join(GOLD, "scenarios")
    return sorted(f[:-5] for f in os.listdir(d) if f.endswith(".json"))


def scenario_text(name):
    with open(os.path.join(GOLD, "scenarios", name + ".json")) as f:
        return f.read()


def golden(name, policy):
    d = os.path.join(GOLD, "traces", name, policy)
    with open(os.path.join(d, "trace.csv")) as f:
        t = f.read()
    with open(os.path.join(d, "summary.json")) as f:
        s = f.read()
    return t, s


def with_policy(text, policy):
    d = json.loads(text)
    d["policy"] = policy
    return json.dumps(d)
