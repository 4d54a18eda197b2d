"""Synthetic scenario builders for the BASELINE.json configurations.

The JSON schema is the reference's (proj/README.md:107-169, parsed by
scenario.cpp:291-357).  Camera layout follows the correlated-scenario pattern
of the reference acceptance suite (proj/tests/acceptance_main.cpp:454-473):
cameras of one spatial cluster sit within a few hundred metres, clusters are
5 km apart, so the grouping filter (delta 500 m) can only join cameras of the
same cluster.  Drift is a counter-RNG-chosen subset of cameras moving to
another cluster's scene each window.
"""
import hashlib


def _u01(*key):
    h = hashlib.blake2b(repr(key).encode(), digest_size=8).digest()
    return int.from_bytes(h, "little") / 2.0**64


def cluster_layout(n_clusters, per_cluster, spacing_m=5000.0, pitch_m=40.0):
    cams = []
    cols = 4
    side = max(1, int(round(n_clusters ** 0.5)))
    for c in range(n_clusters):
        cx, cy = (c % side) * spacing_m, (c // side) * spacing_m
        for k in range(per_cluster):
            cams.append((c, cx + (k % cols) * pitch_m, cy + (k // cols) * pitch_m))
    return cams


def cluster_scene(c):
    # scenes on a 0.1 grid, distinct per cluster
    return [round(0.1 * (c % 10), 10), round(0.1 * ((c // 10) % 10), 10)]


def synthetic(n_cameras, n_clusters, windows=2, micro_windows=None, micro_s=6.0, gpus=1,
              drift_frac=0.05, local_acc=0.1, seed=1, name=None, policy="ecco"):
    """A C2/C3/C4-style scenario: n_cameras in n_clusters correlated clusters."""
    per = max(1, n_cameras // n_clusters)
    layout = cluster_layout(n_clusters, per)[:n_cameras]
    width = len(str(n_cameras - 1))
    cameras = []
    for i, (c, x, y) in enumerate(layout):
        cameras.append({"id": f"cam{i:0{width}d}", "location": [x, y], "scene": cluster_scene(c),
                        "local_model_acc": local_acc})
    if micro_windows is None:
        micro_windows = max(2 * n_clusters, 10)
    T = micro_windows * micro_s
    events = []
    for w in range(1, windows):
        for i, (c, _, _) in enumerate(layout):
            if _u01(seed, "drift", w, i) < drift_frac:
                other = (c + 1 + int(_u01(seed, "to", w, i) * (n_clusters - 1))) % n_clusters
                events.append({"camera": cameras[i]["id"], "time_s": w * T,
                               "new_scene": cluster_scene(other), "acc_drop": 0.3})
    return {
        "name": name or f"synthetic_{n_cameras}x{n_clusters}",
        "seed": seed,
        "num_windows": windows,
        "policy": policy,
        "drift_threshold": 0.25,
        "shared_capacity_bps": 6e6 * max(1, n_cameras // 10),
        "allocator": {"micro_windows": micro_windows, "micro_window_duration_s": micro_s,
                      "gpu_count": gpus},
        "cameras": cameras,
        "drift_events": events,
    }


def c1_fixture():
    """10 cameras, 3 correlated drift clusters, one window."""
    groups = [(4, (0.0, 0.0), [0.2, 0.2], [0.25, 0.2]),
              (3, (5000.0, 0.0), [0.6, 0.2], [0.65, 0.2]),
              (3, (0.0, 5000.0), [0.2, 0.7], [0.2, 0.75])]
    offs = [(0.0, 0.0), (30.0, 0.0), (0.0, 40.0), (30.0, 40.0)]
    cams, events, i = [], [], 0
    for n, (bx, by), scene, drifted in groups:
        for k in range(n):
            cid = f"c{i:02d}"
            cams.append({"id": cid, "location": [bx + offs[k][0], by + offs[k][1]],
                         "scene": scene, "local_model_acc": 0.5})
            events.append({"camera": cid, "time_s": 0, "new_scene": drifted, "acc_drop": 0.4})
            i += 1
    return {"name": "c1_ten_cameras", "seed": 11, "num_windows": 1, "policy": "ecco",
            "drift_threshold": 0.25, "cameras": cams, "drift_events": events}


# BASELINE.json configs -> (n_cameras, n_clusters, micro_windows, micro_s)
CONFIGS = {
    "c1": None,
    "c2": (100, 10, 20, 6.0),
    "c3": (1000, 50, 100, 0.6),
    "c4": (10000, 500, 1000, 0.06),
}


def config(name, windows=2, **kw):
    if name == "c1":
        return c1_fixture()
    n, g, W, mu = CONFIGS[name]
    return synthetic(n, g, windows=windows, micro_windows=W, micro_s=mu, **kw)
