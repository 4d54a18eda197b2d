"""End-to-end parity: the B200 window driver (parametric backend) reproduces
the unmodified reference's trace.csv and summary.json byte for byte, for
every committed scenario (the reference's bundled fixtures, the C1 fixture
and synthetic drift scenarios) under all three policies.  The golden files
were produced by the reference itself (tools/make_golden.py)."""
import pytest

import paper_2512_11727_b200 as ecco
from conftest import golden, scenario_names, scenario_text, with_policy

pytestmark = pytest.mark.gpu
POLICIES = ["ecco", "naive", "total_acc_greedy"]


@pytest.mark.parametrize("policy", POLICIES)
@pytest.mark.parametrize("name", scenario_names())
def test_trace_and_summary_identical(name, policy):
    sim = ecco.Simulation(with_policy(scenario_text(name), policy), backend=ecco.PARAMETRIC)
    sim.run()
    trace, summary = golden(name, policy)
    got = sim.trace_csv()
    if got != trace:
        a, b = got.splitlines(), trace.splitlines()
        for i, (x, y) in enumerate(zip(a, b)):
            assert x == y, f"first divergence at line {i + 1}"
        assert len(a) == len(b)
    assert sim.summary_json() == summary
    assert sim.launches > 0


def test_schema_errors_map_to_schema_error():
    with pytest.raises(ecco.SchemaError, match="unknown field"):
        ecco.Simulation('{"cameras": [], "bogus": 1}')
    with pytest.raises(ecco.SchemaError, match="cameras"):
        ecco.Simulation('{"cameras": []}')


def test_infeasible_window_raises():
    import json
    sc = json.loads(scenario_text("shared_bottleneck"))
    sc["allocator"] = {"micro_windows": 1}
    for c in sc["cameras"]:
        c["location"] = [c["location"][0] * 100, c["location"][1] * 100]
    sim = ecco.Simulation(json.dumps(sc))
    with pytest.raises(ecco.InfeasibleScheduleError):
        sim.step_window()
