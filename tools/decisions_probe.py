"""Decision agreement of the tensor-core path at a BASELINE config (SURVEY.md
H8(iii)): the learned window driver (ecco_sim) on the same scenario with
FFMA_EXACT math (op-by-op bit-exact to the fp32 oracle, so its decisions are
the oracle's) and with tensor-core math; per-window routing / schedule /
assignment agreement, the first divergence and each run's window times.

  python tools/decisions_probe.py [c3] [windows] > profiles/r02_decisions_c3.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2512_11727_b200 as ecco  # noqa: E402
from paper_2512_11727_b200 import scenarios  # noqa: E402
from paper_2512_11727_b200.agreement import decision_agreement  # noqa: E402


def run(sc, math, opts):
    sim = ecco.Simulation(sc, backend=ecco.LEARNED, math=math, **opts)
    wins = []
    while True:
        t = time.perf_counter()
        if not sim.step_window():
            break
        d = {k: round(v, 3) for k, v in sim.last_timings().items()}
        d["wall_ms"] = round((time.perf_counter() - t) * 1e3, 3)
        d["samples"] = sim.last_samples()
        wins.append(d)
    tr = sim.trace_csv()
    sim.close()
    return tr, wins


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
    windows = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    sc = json.dumps(scenarios.config(cfg, windows=windows, seed=1, local_acc=0.0))
    opts = dict(feat_dim=512, hidden_dim=256, num_classes=16, minibatch=128, ring_frames=512,
                eval_samples=64, steps_per_gpu_s=16.0 / 0.6)
    ffma, wf = run(sc, ecco.FFMA_EXACT, opts)
    tc, wt = run(sc, ecco.TC_BF16, opts)
    r = decision_agreement(ffma, tc)
    print(json.dumps({"config": cfg, "windows": windows,
                      "workload": f"scenarios.config('{cfg}', windows={windows}, seed=1, "
                                  "local_acc=0.0), learned F512-H256-C16, B=128, 16 SGD steps "
                                  "per micro-window",
                      "agreement": r, "ffma_windows": wf, "tc_windows": wt}, indent=1))


if __name__ == "__main__":
    main()
