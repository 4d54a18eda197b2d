"""Decision agreement of the tensor-core path.

The learned window driver (ecco_sim, csrc/sim.cpp) runs the same scenario
with FFMA_EXACT math (bit-exact to the fp32 oracle op by op, so its
decisions are the oracle's) and with tensor-core math (bf16 operands, fp32
accumulation).  The agreement of routing, allocator schedule and window-end
assignment, and the first divergence, are reported (pytest -s) and bounded.
"""
import json

import pytest

import paper_2512_11727_b200 as ecco
from paper_2512_11727_b200 import scenarios
from paper_2512_11727_b200.agreement import decision_agreement

pytestmark = pytest.mark.gpu

OPTS = dict(feat_dim=512, hidden_dim=256, num_classes=16, minibatch=128, ring_frames=512,
            eval_samples=64, steps_per_gpu_s=4.0, full_matrix=1)


def _run(sc, math):
    sim = ecco.Simulation(sc, backend=ecco.LEARNED, math=math, **OPTS)
    sim.run()
    t = sim.trace_csv()
    sim.close()
    return t


def test_ffma_decisions_are_deterministic_and_tc_agreement_reported():
    # C2's cameras and clusters (100 / 10) with enough micro-windows for the
    # jobs that drifted cameras create (W = 60 x 2 s)
    sc = json.dumps(scenarios.synthetic(100, 10, windows=3, micro_windows=60, micro_s=2.0,
                                        seed=1, local_acc=0.0, drift_frac=0.1))
    ffma = _run(sc, ecco.FFMA_EXACT)
    assert _run(sc, ecco.FFMA_EXACT) == ffma  # the oracle-exact path is deterministic
    tc = _run(sc, ecco.TC_BF16)
    assert _run(sc, ecco.TC_BF16) == tc  # so is the tensor-core path
    r = decision_agreement(ffma, tc)
    print("c2 decision agreement (ffma vs tc):",
          json.dumps({k: v for k, v in r.items() if k != "per_window"}))
    for w in r["per_window"]:
        print("  window", json.dumps(w))
    assert r["decision_rows"][0] > 0
    # grouping is spatial first (correlation_filter, 500 m): the window-0
    # routing of fresh cameras cannot diverge; accuracies are counts / 64
    assert r["per_window"][0]["routing_agreement"] == 1.0
    assert r["assignment_agreement"] >= 0.9
    assert r["mean_abs_acc_diff"] <= 4.0 / 64
