"""Small solves through every window kernel, for compute-sanitizer runs
(tools/gcall_r2_san_*.sh): C1 (65^2, 2x2, overlap 4) parallel + alternating
through k_windowD (and k_windowP with DDPMA_KERNEL=P), T3 (33^3, 2x2x2) through
k_windowP<3> with 3D TMA tiles.  Prints a digest of every result so a sanitizer
run can be compared with a plain run."""
import hashlib
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2006_14602_b200 as P

W2 = int(sys.argv[1]) if len(sys.argv) > 1 else 3
W3 = int(sys.argv[2]) if len(sys.argv) > 2 else 2


def digest(res):
    return hashlib.sha256(np.ascontiguousarray(res.mesh.coords).tobytes()).hexdigest()[:16]


g = P.build_grid(2, ((0.0, 1.0),) * 2, (65, 65))
d = P.build_decomposition(g, (2, 2), 4)
m = P.density_monitor(P.RingDensity(), g.extents)
for tr in ("parallel", "alternating"):
    r = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=W2, transmission=tr))
    print("C1", tr, r.windows, r.stats["node_updates"], digest(r), flush=True)
g = P.build_grid(3, ((0.0, 1.0),) * 3, (33, 33, 33))
d = P.build_decomposition(g, (2, 2, 2), 4)
m = P.density_monitor(P.ShellDensity(), g.extents)
r = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=W3, transmission="parallel"))
print("T3 parallel", r.windows, r.stats["node_updates"], digest(r), flush=True)
print("sanitize_case ok")
