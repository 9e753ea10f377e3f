"""Golden fixtures for the arc-length (u-backed) monitors, from the REAL
reference (``ddmesh``).  Build container only (needs /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_arc_golden.py

Writes tests/golden/arc.npz:
* ``op_<name>_*``: the analytic raw (arc_length_monitor's raw,
  monitor.py:88-97) and the solver's nodal density (mesh_density's u
  pull-back, monitor.py:151-216) of every registered test function
  (monitor.py:223-345) on the box mesh of a perturbed potential;
* ``run_<tag>_*``: short ``solve`` / ``solve_single_domain`` runs with
  arc-length monitors (coordinates, residual history, node-update counts).
Bytecode writing is disabled; nothing is written under /root/reference.
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
from ddmesh import grid as rgrid  # noqa: E402
from ddmesh import monitor as rmon  # noqa: E402
from ddmesh import pma as rpma  # noqa: E402

# (name, params, dim, counts, layout, overlap)
OP_CASES = [
    ("burgers2d", {"eps": 0.05}, 2, (33, 33), (2, 2), 4),
    ("spiral2d", {}, 2, (33, 33), (2, 2), 4),
    ("quasi1d_linear", {}, 2, (33, 33), (1, 2), 4),
    ("sphere3d", {}, 3, (17, 17, 17), (2, 2, 2), 2),
    ("nine_spheres3d", {}, 3, (17, 17, 17), (2, 2, 2), 2),
]

# (tag, name, params, dim, counts, layout or None (single domain), overlap,
#  transmission, windows, rtol, atol)
RUN_CASES = [
    ("burgers_par", "burgers2d", {"eps": 0.05}, 2, (33, 33), (2, 2), 4, "parallel", 4, 1e-6, 1e-9),
    ("spiral_alt", "spiral2d", {}, 2, (33, 33), (2, 2), 4, "alternating", 4, 1e-6, 1e-9),
    ("quasi1d_single", "quasi1d_linear", {}, 2, (33, 33), None, 0, "parallel", 4, 1e-6, 1e-9),
    ("sphere_par", "sphere3d", {}, 3, (17, 17, 17), (2, 2, 2), 2, "parallel", 3, 1e-6, 1e-9),
    ("nine_single", "nine_spheres3d", {}, 3, (17, 17, 17), None, 0, "parallel", 3, 1e-6, 1e-9),
    # normalize() drops u_fn (monitor.py:147-148): the analytic-density path the
    # reference's own drivers take (experiments.run_mesh, :142-158)
    ("burgers_norm_par", "burgers2d:norm", {"eps": 0.05}, 2, (33, 33), (2, 2), 4, "parallel", 4,
     1e-6, 1e-9),
]

# normalize() probe quadrature: (name, params, counts)
NORM_CASES = [
    ("burgers2d", {"eps": 0.05}, (33, 33)),
    ("spiral2d", {}, (65, 65)),
    ("quasi1d_linear", {}, (17, 17)),
    ("sphere3d", {}, (17, 17, 17)),
    ("nine_spheres3d", {}, (33, 33, 33)),
]


def perturbed_psi(geom, seed):
    psi = rpma.initial_potential(geom)
    rng = np.random.default_rng(seed)
    h = min(geom.spacing)
    return psi + 0.02 * h * h * rng.standard_normal(psi.shape)


def main():
    out = {}
    for i, (name, params, dim, counts, layout, ov) in enumerate(OP_CASES):
        tf = rmon.test_function_registry(name, **params)
        mon = rmon.arc_length_monitor(tf)
        g = ddmesh.build_grid(dim, tf.domain, counts)
        d = ddmesh.build_decomposition(g, layout, ov)
        sub = d.subdomains[-1]
        geom = rgrid.subdomain_geometry(g, sub)
        psi = perturbed_psi(geom, 100 + i)
        mesh = rpma.physical_mesh(psi, geom)
        out[f"op_{name}_psi"] = psi
        out[f"op_{name}_sub"] = np.array(sub.id)
        out[f"op_{name}_analytic"] = mon.raw(mon.clamp(mesh.coords))
        out[f"op_{name}_u"] = mon.u_fn(mon.clamp(mesh.coords))
        out[f"op_{name}_pull"] = rmon.mesh_density(mon, mesh.coords, geom.spacing)
        # moving-point pma_rhs (pma.py:152-183) with the normalised monitor
        nmon = rmon.normalize(mon, g)
        ev = rpma.pma_rhs(psi, nmon, geom)
        out[f"op_{name}_pmarhs"] = ev.values
        out[f"op_{name}_pmarhs_flag"] = np.array(ev.det_clamped)
        out[f"op_{name}_norm"] = np.array([nmon.normalizer, nmon.max_value])
        print("op", name, psi.shape)
    for name, params, counts in NORM_CASES:
        tf = rmon.test_function_registry(name, **params)
        g = ddmesh.build_grid(len(counts), tf.domain, counts)
        nm = rmon.normalize(rmon.arc_length_monitor(tf), g)
        out[f"norm_{name}"] = np.array([nm.normalizer, nm.max_value])
        print("norm", name, nm.normalizer, nm.max_value)
    for (tag, name, params, dim, counts, layout, ov, tr, nwin, rtol, atol) in RUN_CASES:
        norm = name.endswith(":norm")
        name = name.split(":")[0]
        tf = rmon.test_function_registry(name, **params)
        mon = rmon.arc_length_monitor(tf)
        g = ddmesh.build_grid(dim, tf.domain, counts)
        if norm:
            mon = rmon.normalize(mon, g)
        cfg = ddmesh.SolverConfig(tol=1e-300, max_windows=nwin, transmission=tr, workers=1,
                                  rtol=rtol, atol=atol)
        calls = [0, 0]
        orig = rpma.pma_rhs_frozen

        def wrapped(psi, *a, **k):
            calls[0] += 1
            calls[1] += psi.size
            return orig(psi, *a, **k)

        rpma.pma_rhs_frozen = wrapped
        try:
            if layout is None:
                res = ddmesh.solve_single_domain(g, mon, cfg)
            else:
                res = ddmesh.solve(g, ddmesh.build_decomposition(g, layout, ov), mon, cfg)
        finally:
            rpma.pma_rhs_frozen = orig
        out[f"run_{tag}_psi"] = res.psi
        out[f"run_{tag}_coords"] = res.mesh.coords
        out[f"run_{tag}_jac"] = res.mesh.jac
        out[f"run_{tag}_residuals"] = np.array([h.residuals for h in res.history])
        out[f"run_{tag}_node_updates"] = np.array(calls[1])
        print("run", tag, res.windows, calls, res.final_residual)
    np.savez_compressed(os.path.join(HERE, "arc.npz"), **out)


if __name__ == "__main__":
    main()
