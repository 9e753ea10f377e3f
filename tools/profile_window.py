"""Run W warm-up windows of a BASELINE config, then one more window (the one
ncu captures with -k k_windowP -s W).  Prints the node-updates and algorithmic
bytes of every window (exact controller tallies) as JSON lines."""
import json
import sys
sys.path.insert(0, ".")
import paper_2006_14602_b200 as P
from paper_2006_14602_b200.plan import Plan
import bench
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
W = int(sys.argv[2]) if len(sys.argv) > 2 else 2
DTAU = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
g, d, m = bench.case(name, P)
plan = Plan.for_grid(g, d.subdomains, m, P.SolverConfig(tol=1e-300, max_windows=W + 1, transmission="parallel", dtau=DTAU))
plan.set_state(None)
prev = plan.counters()
for w in range(W + 1):
    plan.run(1, 1e-300)
    c = plan.counters()
    print(json.dumps({"window": w, "node_updates": c["node_updates"] - prev["node_updates"],
                      "algo_bytes": c["algo_bytes"] - prev["algo_bytes"]}), flush=True)
    prev = c
