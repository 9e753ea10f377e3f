"""Debug: per-window max|psi_gpu - psi_oracle| for C1 (first divergence)."""
import sys
import numpy as np
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import ddpma_oracle as O
import paper_2006_14602_b200 as P
from paper_2006_14602_b200.plan import Plan

W = int(sys.argv[1]); tr = sys.argv[2] if len(sys.argv) > 2 else "parallel"
g, lay, ov, mon, dom, _ = O.baseline_case("C1")
d = O.make_decomposition(g, lay, ov)
snaps = []
O.solve(g, d, mon, dom, O.Config(tol=1e-300, max_windows=W, transmission=tr),
        callback=lambda w, boxes: snaps.append([b.psi.copy() for b in boxes]))
pg = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65)); pd = P.build_decomposition(pg, (2, 2), 4)
pm = P.density_monitor(P.RingDensity(), pg.extents)
plan = Plan.for_grid(pg, pd.subdomains, pm, P.SolverConfig(tol=1e-300, max_windows=W, transmission=tr))
plan.set_state(None)
for w in range(W):
    plan.run(1, 1e-300)
    diffs = [float(np.abs(plan.sub_psi(i) - snaps[w][i]).max()) for i in range(4)]
    print(w, " ".join(f"{x:.2e}" for x in diffs))
