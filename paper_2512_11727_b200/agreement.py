"""Decision agreement between two window-driver traces (SURVEY.md hazard H8).

The learned backend's tensor-core math (bf16 operands, fp32 accumulation) is
not bit-exact against the fp32 oracle, so its decisions can differ from the
FFMA path's.  H8(iii) asks for the agreement rate and the first divergence:
this compares two ``trace.csv`` texts of the same scenario (metrics.cpp:49-59
layout: record,window,time_s,camera,job,v1..v5) decision by decision:

* routing   -- the ``new_job`` / ``join`` rows (group_request's commit,
               grouping.cpp:18-62) of each window, as (camera, job) pairs;
* schedule  -- the ``micro`` rows (WindowAllocation's picks,
               gpu_allocator.cpp:125-181), the job of every micro-window;
* assignment -- the window-end ``accuracy`` rows (orchestrator.cpp:328-352):
               the job every camera belongs to after regrouping, and the
               accuracy it reports;
* regroup   -- ``remove`` / ``terminate`` rows (update_grouping,
               grouping.cpp:64-121).

The first divergence is the first decision row (in trace order, numeric
values ignored) where the two traces differ.  Host logic only; no device.
"""
import csv
import io

DECISIONS = ("new_job", "join", "micro", "remove", "terminate")


def _rows(text):
    return list(csv.DictReader(io.StringIO(text)))


def _key(r):
    return (r["record"], r["window"], r["camera"], r["job"])


def _frac(a, b):
    n = max(len(a), len(b))
    if n == 0:
        return 1.0
    return sum(1 for x, y in zip(a, b) if x == y) / n


def decision_agreement(trace_a, trace_b):
    ra, rb = _rows(trace_a), _rows(trace_b)
    wins = sorted({int(r["window"]) for r in ra} | {int(r["window"]) for r in rb})
    per_window = []
    for w in wins:
        sw = str(w)
        a = [r for r in ra if r["window"] == sw]
        b = [r for r in rb if r["window"] == sw]
        route_a = [(r["camera"], r["job"]) for r in a if r["record"] in ("new_job", "join")]
        route_b = [(r["camera"], r["job"]) for r in b if r["record"] in ("new_job", "join")]
        micro_a = [r["job"] for r in a if r["record"] == "micro"]
        micro_b = [r["job"] for r in b if r["record"] == "micro"]
        acc_a = {r["camera"]: r for r in a if r["record"] == "accuracy"}
        acc_b = {r["camera"]: r for r in b if r["record"] == "accuracy"}
        cams = sorted(set(acc_a) | set(acc_b))
        same = sum(1 for c in cams if c in acc_a and c in acc_b and acc_a[c]["job"] == acc_b[c]["job"])
        dacc = [abs(float(acc_a[c]["v1"]) - float(acc_b[c]["v1"])) for c in cams
                if c in acc_a and c in acc_b]
        rg_a = [_key(r) for r in a if r["record"] in ("remove", "terminate")]
        rg_b = [_key(r) for r in b if r["record"] in ("remove", "terminate")]
        per_window.append({
            "window": w,
            "routing_agreement": _frac(route_a, route_b),
            "schedule_agreement": _frac(micro_a, micro_b),
            "assignment_agreement": same / len(cams) if cams else 1.0,
            "regroup_agreement": _frac(rg_a, rg_b),
            "mean_abs_acc_diff": sum(dacc) / len(dacc) if dacc else 0.0,
            "max_abs_acc_diff": max(dacc) if dacc else 0.0,
            "micro_windows": max(len(micro_a), len(micro_b)),
        })
    da = [(i, r) for i, r in enumerate(ra) if r["record"] in DECISIONS]
    db = [(i, r) for i, r in enumerate(rb) if r["record"] in DECISIONS]
    first = None
    for (ia, x), (ib, y) in zip(da, db):
        if _key(x) != _key(y):
            first = {"window": int(x["window"]), "decision_index": len([1 for i, _ in da if i < ia]),
                     "a": ",".join(_key(x)), "b": ",".join(_key(y))}
            break
    if first is None and len(da) != len(db):
        k = min(len(da), len(db))
        longer = da if len(da) > len(db) else db
        first = {"window": int(longer[k][1]["window"]), "decision_index": k,
                 "a": ",".join(_key(da[k][1])) if len(da) > k else None,
                 "b": ",".join(_key(db[k][1])) if len(db) > k else None}
    n = len(per_window)
    mean = lambda k: sum(p[k] for p in per_window) / n if n else 1.0
    return {
        "identical_decisions": first is None,
        "first_divergence": first,
        "decision_rows": [len(da), len(db)],
        "routing_agreement": mean("routing_agreement"),
        "schedule_agreement": mean("schedule_agreement"),
        "assignment_agreement": mean("assignment_agreement"),
        "mean_abs_acc_diff": mean("mean_abs_acc_diff"),
        "per_window": per_window,
    }
