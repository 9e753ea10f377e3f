"""Debug: device integrator protocol vs the oracle Rkc2, step traces."""
import os, sys
sys.path[:0] = [".", "oracle", "tests/golden", "tests"]
import numpy as np
import ddpma_oracle as O
import recipes as R
import paper_2006_14602_b200 as P
from test_api import _c1_box
geom, ogeom, y, rho, rmax = _c1_box(3)
fn = lambda v: O.rhs_frozen(v, rho, ogeom, O.DET_FLOOR, ogeom.mask(), rmax)
tr = []
oi = O.Rkc2(1e-3, trace=tr)
integ = P.make_integrator(P.IntegrationWindow(dtau=1e-3))
rhs = P.frozen_rhs(rho, geom, max_rho=rmax)
a = b = y
for w in range(3):
    print("=== window", w, flush=True)
    n0 = len(tr)
    a = integ.advance(a, rhs)
    sys.stderr.flush()
    b = oi.advance(b, fn)
    for t in tr[n0:]:
        print("ORACLE", t, flush=True)
    print("diff", float(np.max(np.abs(a - b))), flush=True)
