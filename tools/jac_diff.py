import sys
import numpy as np
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import ddpma_oracle as O
import paper_2006_14602_b200 as P
W = int(sys.argv[1]); tr = sys.argv[2]
g, lay, ov, mon, dom, _ = O.baseline_case("C1")
d = O.make_decomposition(g, lay, ov)
r = O.solve(g, d, mon, dom, O.Config(tol=1e-300, max_windows=W, transmission=tr))
pg = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65)); pd = P.build_decomposition(pg, (2, 2), 4)
pm = P.density_monitor(P.RingDensity(), pg.extents)
a = P.solve(pg, pd, pm, P.SolverConfig(tol=1e-300, max_windows=W, transmission=tr))
b = P.solve(pg, pd, pm, P.SolverConfig(tol=1e-300, max_windows=W, transmission=tr, rtol=np.nextafter(1e-3, 1)))
print("gpu-vs-gpu(rtol+1ulp): coords %.3g nodes %d %d" % (np.abs(a.mesh.coords-b.mesh.coords).max(), a.stats["node_updates"], b.stats["node_updates"]))
print("gpu-vs-oracle: coords %.3g nodes %d %d" % (np.abs(a.mesh.coords-r.coords).max(), a.stats["node_updates"], r.counter.node_updates))
for w in range(0, W, max(1, W // 25)):
    print(w, "oracle minJ %.4g maxJ %.4g res %s" % (r.jac_min[w], r.jac_max[w], " ".join("%.2e" % x for x in r.residuals[w])))
    h = a.history[w]
    print(w, "gpu    minJ %.4g maxJ %.4g res %s" % (h.jac_min, h.jac_max, " ".join("%.2e" % x for x in h.residuals)))
