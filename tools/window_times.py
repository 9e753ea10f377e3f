"""Per-window node-updates and wall time of a BASELINE config (JSON lines).
    python tools/window_times.py C3 8 [stable|default] [dtau]"""
import json
import sys
import time
sys.path.insert(0, ".")
import paper_2006_14602_b200 as P
from paper_2006_14602_b200.plan import Plan
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 6
prof = sys.argv[3] if len(sys.argv) > 3 else "default"
kw = dict(tol=1e-300, max_windows=W, transmission="parallel")
if prof == "stable":
    kw.update(rtol=1e-6, atol=1e-9)
if len(sys.argv) > 4:
    kw["dtau"] = float(sys.argv[4])
g, d, m = bench.case(name, P)
plan = Plan.for_grid(g, d.subdomains, m, P.SolverConfig(**kw))
plan.set_state(None)
prev = plan.counters()
for w in range(W):
    t0 = time.perf_counter()
    _, _, fres, hres, hstats = plan.run(1, 1e-300)
    dt = time.perf_counter() - t0
    c = plan.counters()
    ev = plan.sub_evals()
    print(json.dumps({"window": w, "ms": round(dt * 1e3, 2), "node_updates": c["node_updates"] - prev["node_updates"],
                      "residual": float(fres), "jac_min": float(hstats[0, 1]), "max_sub_evals": int(ev.max())}), flush=True)
    prev = c
