"""Golden fixtures for SampledField arc-length monitors (ddmesh/monitor.py:
361-444) from the REAL reference.  Build container only:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_sampled_golden.py

Writes tests/golden/sampled.npz (+ sampled2d.csv, a CSV lattice for
sampled_field_from_csv): lattice inputs, the pull-back density on a box,
normalize()'s quadrature, and short solves.
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


def lattices():
    """Seeded synthetic scalar fields on uniform lattices."""
    ax2 = (np.linspace(0.0, 1.0, 41), np.linspace(0.0, 1.0, 37))
    X, Y = np.meshgrid(*ax2, indexing="ij")
    u2 = np.tanh(12.0 * (X + 0.7 * Y - 0.9)) + 0.3 * np.sin(5.0 * X * Y)
    ax3 = (np.linspace(0.0, 1.0, 19), np.linspace(0.0, 1.0, 17), np.linspace(0.0, 1.0, 21))
    X, Y, Z = np.meshgrid(*ax3, indexing="ij")
    u3 = np.exp(-12.0 * ((X - 0.4) ** 2 + (Y - 0.55) ** 2 + (Z - 0.5) ** 2))
    return ax2, u2, ax3, u3


# (tag, dim, smooth, counts, layout|None, overlap, transmission, windows)
RUNS = [
    ("s2_par", 2, 1, (33, 33), (2, 2), 4, "parallel", 4),
    ("s2_single", 2, 0, (33, 33), None, 0, "parallel", 3),
    ("s3_par", 3, 0, (17, 17, 17), (2, 2, 2), 2, "parallel", 3),
]


def main():
    ax2, u2, ax3, u3 = lattices()
    out = {"ax2_0": ax2[0], "ax2_1": ax2[1], "u2": u2,
           "ax3_0": ax3[0], "ax3_1": ax3[1], "ax3_2": ax3[2], "u3": u3}
    fields = {}
    for dim, smooth in ((2, 0), (2, 1), (3, 0)):
        ax, u = (ax2, u2) if dim == 2 else (ax3, u3)
        fields[(dim, smooth)] = rmon.SampledField(ax, u, smooth_passes=smooth)
    # operator: pull-back density and analytic raw on a perturbed box mesh
    for dim, smooth in ((2, 1), (3, 0)):
        sf = fields[(dim, smooth)]
        mon = rmon.arc_length_monitor(sf)
        counts = (33, 33) if dim == 2 else (17, 17, 17)
        g = ddmesh.build_grid(dim, sf.domain, counts)
        d = ddmesh.build_decomposition(g, (2,) * dim, 4 if dim == 2 else 2)
        geom = rgrid.subdomain_geometry(g, d.subdomains[-1])
        psi = rpma.initial_potential(geom)
        h = min(geom.spacing)
        psi = psi + 0.02 * h * h * np.random.default_rng(5 + dim).standard_normal(psi.shape)
        mesh = rpma.physical_mesh(psi, geom)
        out[f"op{dim}_psi"] = psi
        out[f"op{dim}_analytic"] = mon.raw(mon.clamp(mesh.coords))
        out[f"op{dim}_pull"] = rmon.mesh_density(mon, mesh.coords, geom.spacing)
        nm = rmon.normalize(mon, g)
        out[f"norm{dim}"] = np.array([nm.normalizer, nm.max_value])
        print("op", dim, nm.normalizer)
    for tag, dim, smooth, counts, layout, ov, tr, nwin in RUNS:
        sf = fields[(dim, smooth)]
        mon = rmon.arc_length_monitor(sf)
        g = ddmesh.build_grid(dim, sf.domain, counts)
        cfg = ddmesh.SolverConfig(tol=1e-300, max_windows=nwin, transmission=tr, workers=1,
                                  rtol=1e-6, atol=1e-9)
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
        out[f"{tag}_coords"] = res.mesh.coords
        out[f"{tag}_residuals"] = np.array([h.residuals for h in res.history])
        out[f"{tag}_node_updates"] = np.array(calls[0])
        print(tag, res.windows, calls[0], res.final_residual)
    # CSV ingestion: a shuffled lattice file and the reference reader's values
    X, Y = np.meshgrid(*ax2, indexing="ij")
    rows = np.column_stack([X.ravel(), Y.ravel(), u2.ravel()])
    rows = rows[np.random.default_rng(3).permutation(len(rows))]
    path = os.path.join(HERE, "sampled2d.csv")
    with open(path, "w") as fp:
        fp.write("# x,y,u\n")
        for r in rows:
            fp.write(f"{r[0]:.17g},{r[1]:.17g},{r[2]:.17g}\n")
    sf = rmon.sampled_field_from_csv(path, smooth_passes=1)
    out["csv_values"] = sf.values
    np.savez_compressed(os.path.join(HERE, "sampled.npz"), **out)


if __name__ == "__main__":
    main()
