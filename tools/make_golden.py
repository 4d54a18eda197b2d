"""Generates tests/golden/ from the reference itself (oracle/_ref/libecco_ref.so).

Run here, where /root/reference exists:  python tools/make_golden.py
Outputs (committed):
  tests/golden/scenarios/*.json          the reference's bundled scenario
                                         fixtures + the C1 / synthetic ones
  tests/golden/traces/<name>/<policy>/{trace.csv,summary.json}
                                         Simulation::run output of the
                                         unmodified reference
  tests/golden/kat_param.npz             random eval / train_step / profile
                                         cases answered by the reference
"""
import json
import os
import shutil
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2512_11727_b200 import scenarios  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
POLICIES = ["ecco", "naive", "total_acc_greedy"]


def run_ref(text, policy):
    import ctypes as C
    R = oracle.ref()
    cap = 1 << 26
    tb, sb = C.create_string_buffer(cap), C.create_string_buffer(1 << 22)
    tl, sl = C.c_size_t(), C.c_size_t()
    rc = R.ref_run_scenario(text.encode(), POLICIES.index(policy), tb, cap, C.byref(tl), sb,
                            1 << 22, C.byref(sl))
    if rc:
        raise RuntimeError(R.ref_last_error().decode())
    return tb.raw[:tl.value].decode(), sb.raw[:sl.value].decode()


def first_runnable(n, g, windows, W, mu, frac):
    for seed in range(1, 100):
        sc = scenarios.synthetic(n, g, windows=windows, micro_windows=W, micro_s=mu,
                                 drift_frac=frac, seed=seed)
        try:
            trace, _ = run_ref(json.dumps(sc), "ecco")
        except RuntimeError:
            continue
        if "remove," in trace:
            return sc
    raise RuntimeError("no runnable seed")


def main():
    oracle.build()
    sdir = os.path.join(GOLD, "scenarios")
    os.makedirs(sdir, exist_ok=True)
    names = []
    for f in sorted(os.listdir(os.path.join(oracle.REFERENCE_ROOT, "scenarios"))):
        shutil.copy(os.path.join(oracle.REFERENCE_ROOT, "scenarios", f), os.path.join(sdir, f))
        names.append(f[:-5])
    # Synthetic fixtures with drift-driven evictions.  The reference aborts a
    # window when a job's measured gain is <= 0 while others are positive
    # (set_aimd_params rejects p_share 0, transmission.cpp:142-143), so the
    # seeds are the first ones the reference runs to completion.
    extra = {"c1_ten_cameras": scenarios.c1_fixture(),
             "synthetic_40x4": first_runnable(40, 4, 4, 12, 6.0, 0.05),
             "synthetic_100x10": first_runnable(100, 10, 4, 20, 6.0, 0.05)}
    for n, sc in extra.items():
        with open(os.path.join(sdir, n + ".json"), "w") as f:
            json.dump(sc, f, indent=1)
        names.append(n)
    for n in names:
        text = open(os.path.join(sdir, n + ".json")).read()
        for pol in POLICIES:
            d = os.path.join(GOLD, "traces", n, pol)
            os.makedirs(d, exist_ok=True)
            trace, summary = run_ref(text, pol)
            open(os.path.join(d, "trace.csv"), "w").write(trace)
            open(os.path.join(d, "summary.json"), "w").write(summary)
    make_kats()


def make_kats():
    R = oracle.ref()
    rng = np.random.default_rng(20251211)
    p = oracle.params_array(oracle.default_params())
    K, D = 4, 2
    n = 400
    ks = rng.integers(0, K + 1, n).astype(np.int32)
    cl = rng.random((n, K, D))
    pr = rng.random((n, K))
    ce = rng.random((n, D))
    clen = np.where(rng.random(n) < 0.9, D, 0).astype(np.int32)
    sc = rng.random((n, D))
    # a third of the scenes sit right next to a cluster so the threshold matters
    near = rng.random(n) < 0.33
    for i in np.nonzero(near)[0]:
        if ks[i] > 0:
            sc[i] = cl[i, rng.integers(0, ks[i])] + rng.normal(0, 0.03, D)
    ev = np.array([R.ref_eval(int(ks[i]), np.ascontiguousarray(cl[i]), np.ascontiguousarray(pr[i]),
                              int(clen[i]), np.ascontiguousarray(ce[i]), D,
                              np.ascontiguousarray(sc[i]), p) for i in range(n)])
    np.savez_compressed(os.path.join(GOLD, "kat_param.npz"), ks=ks, cl=cl, pr=pr, ce=ce,
                        clen=clen, sc=sc, ev=ev)


if __name__ == "__main__":
    main()
