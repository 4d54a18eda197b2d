"""decision_agreement (paper_2512_11727_b200/agreement.py) on the reference's
golden traces: identical traces agree everywhere; two policies of the same
scenario diverge at their first different allocator pick."""
import os

from paper_2512_11727_b200.agreement import decision_agreement

GOLD = os.path.join(os.path.dirname(__file__), "golden", "traces")


def _trace(name, policy):
    with open(os.path.join(GOLD, name, policy, "trace.csv")) as f:
        return f.read()


def test_identical_traces_agree():
    t = _trace("c1_ten_cameras", "ecco")
    r = decision_agreement(t, t)
    assert r["identical_decisions"] and r["first_divergence"] is None
    assert r["routing_agreement"] == r["schedule_agreement"] == r["assignment_agreement"] == 1.0
    assert r["mean_abs_acc_diff"] == 0.0


def test_policies_diverge_at_the_first_different_pick():
    a, b = _trace("c1_ten_cameras", "ecco"), _trace("c1_ten_cameras", "naive")
    r = decision_agreement(a, b)
    assert not r["identical_decisions"]
    fd = r["first_divergence"]
    assert fd["window"] == 0 and fd["a"].startswith("micro") and fd["b"].startswith("micro")
    # ecco: 0,1,2,1,1,...; naive round robin: 0,1,2,0,1,2,...
    assert fd["a"].split(",")[3] == "1" and fd["b"].split(",")[3] == "0"
    assert r["routing_agreement"] == 1.0  # same grouping before the allocator runs
    assert r["schedule_agreement"] < 1.0
