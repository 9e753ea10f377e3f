"""Golden fixtures for monitor smoothing and relaxation (SolverConfig
``monitor_smooth_passes`` / ``monitor_relax``, ddmesh/schwarz.py:162-192,
monitor._smooth ddmesh/monitor.py:395-409) from the REAL reference.
Build container only (needs /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_smooth_golden.py

Writes tests/golden/smooth.npz: short solves (coordinates, residual
history, node-update counts) and one quality_measure(sample_on_mesh,
smooth_passes).  Bytecode writing is disabled.
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import ddmesh  # noqa: E402
from ddmesh import metrics as rmet  # noqa: E402
from ddmesh import monitor as rmon  # noqa: E402
from ddmesh import pma as rpma  # noqa: E402


def ring(p, center=(0.5, 0.5, 0.5)):
    """BASELINE ring / shell density (same formula as the device RingDensity)."""
    acc = (p[..., 0] - center[0]) ** 2
    for k in range(1, p.shape[-1]):
        acc = acc + (p[..., k] - center[k]) ** 2
    return 1.0 + 10.0 * np.exp(-50.0 * np.abs(acc - 0.0625))


UNIT2 = ((0.0, 1.0), (0.0, 1.0))
UNIT3 = ((0.0, 1.0),) * 3

# (tag, monitor, dim, counts, layout|None, overlap, transmission, windows, passes, relax)
CASES = [
    ("ring_par_s2_r3", "ring", 2, (33, 33), (2, 2), 4, "parallel", 5, 2, 0.3),
    ("ring_alt_s1", "ring", 2, (33, 33), (2, 2), 4, "alternating", 5, 1, 0.0),
    ("ring_single_r5", "ring", 2, (33, 33), None, 0, "parallel", 5, 0, 0.5),
    ("shell_par_s1_r2", "ring", 3, (17, 17, 17), (2, 2, 2), 2, "parallel", 3, 1, 0.2),
    ("burgers_par_s2_r25", "burgers2d", 2, (33, 33), (2, 2), 4, "parallel", 4, 2, 0.25),
]


def monitor(name, dim):
    if name == "ring":
        return ddmesh.density_monitor(ring, UNIT2 if dim == 2 else UNIT3)
    return rmon.arc_length_monitor(rmon.test_function_registry(name, eps=0.05))


def main():
    out = {}
    for tag, mname, dim, counts, layout, ov, tr, nwin, passes, relax in CASES:
        mon = monitor(mname, dim)
        g = ddmesh.build_grid(dim, mon.domain, counts)
        cfg = ddmesh.SolverConfig(tol=1e-300, max_windows=nwin, transmission=tr, workers=1,
                                  rtol=1e-6, atol=1e-9, monitor_smooth_passes=passes,
                                  monitor_relax=relax)
        calls = [0]
        orig = rpma.pma_rhs_frozen

        def wrapped(psi, *a, **k):
            calls[0] += psi.size
            return orig(psi, *a, **k)

        rpma.pma_rhs_frozen = wrapped
        try:
            if layout is None:
                res = ddmesh.solve_single_domain(g, mon, cfg)
            else:
                res = ddmesh.solve(g, ddmesh.build_decomposition(g, layout, ov), mon, cfg)
        finally:
            rpma.pma_rhs_frozen = orig
        out[f"{tag}_psi"] = res.psi
        out[f"{tag}_coords"] = res.mesh.coords
        out[f"{tag}_residuals"] = np.array([h.residuals for h in res.history])
        out[f"{tag}_node_updates"] = np.array(calls[0])
        print(tag, res.windows, calls[0], res.final_residual)
    # quality_measure with the smoothed, u pulled-back density
    mon = monitor("burgers2d", 2)
    g = ddmesh.build_grid(2, mon.domain, (33, 33))
    q = rmet.quality_measure(out["burgers_par_s2_r25_psi"], mon, g, sample_on_mesh=True,
                             smooth_passes=2)
    out["quality_e"] = q.e_adp
    out["quality_e2"] = np.array(q.e2)
    np.savez_compressed(os.path.join(HERE, "smooth.npz"), **out)


if __name__ == "__main__":
    main()
