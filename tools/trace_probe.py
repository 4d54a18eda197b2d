import json, sys, time
sys.path.insert(0, '/root/repo')
import paper_2512_11727_b200 as ecco
from paper_2512_11727_b200 import scenarios
sc = json.dumps(scenarios.config("c4", windows=2, seed=1))
t = time.perf_counter(); sim = ecco.Simulation(sc, backend=ecco.PARAMETRIC); t_create = time.perf_counter() - t
while sim.step_window(): pass
t = time.perf_counter(); tr = sim.trace_csv(); t_trace = time.perf_counter() - t
t = time.perf_counter(); tr2 = sim.trace_csv(); t_trace2 = time.perf_counter() - t
t = time.perf_counter(); sm = sim.summary_json(); t_sum = time.perf_counter() - t
print(json.dumps({"scenario_bytes": len(sc), "create_s": t_create, "trace_bytes": len(tr), "trace_rows": tr.count("\n"), "trace_s": t_trace, "trace_again_s": t_trace2, "same": tr == tr2, "summary_s": t_sum}))
