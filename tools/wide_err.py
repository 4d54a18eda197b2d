"""Where the wide fused chain's single SGD step differs from the bf16
emulation (tests/test_gpu_learned.py::_step_emulated): per-tensor error as a
fraction of the update, and for W1 whether the worst columns are hidden units
whose pre-activation sits next to 0 in some row (a ReLU-mask flip between the
fp32 MMA accumulation and the float64 emulation).

  python tools/wide_err.py [hidden]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2512_11727_b200 as ecco  # noqa: E402
from test_gpu_learned import WIDE, _bf16, _jobs, _step_emulated, setup  # noqa: E402


def main():
    hidden = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    cfg = dict(WIDE, hidden_dim=hidden)
    ctx, orc, rng = setup(seed=5, math=ecco.TC_BF16, **cfg)
    ids = [1, 2, 3, 4, 5]
    ctx.seed_models(ids)
    for j in ids:
        orc.seed(j)
    members, sources, fracs, _ = _jobs(rng, len(ids), 6)
    batches = [(5.0, 720.0, 1.0)] * len(ids)
    ctx.train_trajectories(ids, batches, sources, fracs, members, 4.0, 1, window=3)
    ctx.commit(ids, [1] * len(ids))
    base = orc.base_weights()
    B, F, H = orc.c.B, orc.c.F, hidden
    for j, jid in enumerate(ids):
        got = [g.reshape(-1) for g in ctx.get_weights(jid)]
        cams, frames = np.zeros(B, np.int32), np.zeros(B, np.int32)
        orc.L.orc_sample(orc.cp, jid, len(sources[j]), np.array(sources[j], np.int32),
                         np.array(fracs[j]), 3, 0, 0, cams, frames)
        x = (orc.frames[cams, frames].astype(np.uint32) << 16).view(np.float32)
        y = orc.labels[cams, frames]
        emul = _step_emulated(x, y, base, orc.c.lr)
        Z = x.astype(np.float64) @ _bf16(base[0].reshape(F, H)) + base[1]
        row = []
        for k, name in enumerate(["W1", "b1", "W2", "b2"]):
            upd = np.abs(emul[k].reshape(-1) - base[k].astype(np.float64)).max()
            err = np.abs(got[k] - emul[k].reshape(-1))
            row.append(f"{name} {err.max() / upd:.2e}")
            if name == "W1":
                e2 = err.reshape(F, H)
                colmax = e2.max(0)
                worst = np.argsort(colmax)[::-1][:4]
                near = [float(np.abs(Z[:, h]).min()) for h in worst]
                med = float(np.median(np.abs(Z).min(0)))
                row.append(f"worst cols {worst.tolist()} err/upd {(colmax[worst] / upd).round(4).tolist()}"
                           f" min|Z| {np.round(near, 6).tolist()} (median over cols {med:.4f})")
                # error with the worst 8 columns excluded
                keep = np.ones(H, bool)
                keep[np.argsort(colmax)[::-1][:8]] = False
                row.append(f"W1 w/o 8 worst cols {e2[:, keep].max() / upd:.2e}")
        print(f"job {jid}: " + "; ".join(row))


if __name__ == "__main__":
    main()
