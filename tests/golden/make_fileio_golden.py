"""Reference outputs of the mesh/report writers (ddmesh/fileio.py:45-80,
:215-223), for byte-identity tests of the native writers.  Build container
only (needs /root/reference):

    python tests/golden/make_fileio_golden.py
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from ddmesh import fileio as RF  # noqa: E402
from ddmesh import pma as RP  # noqa: E402


def inputs():
    """Seeded meshes with the awkward values a writer must spell like Python."""
    rng = np.random.default_rng(7)
    out = {}
    for tag, shp in (("2d", (6, 5, 2)), ("3d", (4, 3, 5, 3))):
        c = rng.standard_normal(shp)
        flat = c.reshape(-1)
        flat[3], flat[4], flat[5], flat[6], flat[7] = np.nan, -0.0, np.inf, 1e-300, -np.inf
        out[tag] = (c, rng.standard_normal(shp[:-1]), rng.standard_normal(shp[:-1]))
    return out


def main():
    np.savez(os.path.join(HERE, "fileio_inputs.npz"),
             **{f"{t}_{k}": a for t, v in inputs().items() for k, a in zip("cje", v)})
    for tag, (c, j, e) in inputs().items():
        RF.write_mesh_vtk(RP.PhysicalMesh(coords=c, jac=j), os.path.join(HERE, f"ref_mesh{tag}.vtk"),
                          e_adp=e)
    axes = (np.linspace(0.0, 1.0, 5), np.linspace(-1.0, 2.0, 4))
    vals = np.arange(20.0).reshape(5, 4) / 7.0
    RF.write_scalar_field_vtk(axes, vals, os.path.join(HERE, "ref_field.vtk"), name="rho")
    RF.write_field_csv(os.path.join(HERE, "ref_report.csv"), ["n", "e2", "name"],
                       [(33, 0.1, "a"), (65, 1.0 / 3.0, "b"), (129, float("nan"), "c")])


if __name__ == "__main__":
    main()
