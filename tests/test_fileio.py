"""Mesh output formats: the native VTK writer and the
CSV writer are byte-identical to the reference writers (fixtures from
tests/golden/make_fileio_golden.py); the readers invert them exactly and
raise MeshFileError like the reference (fileio.py:83-212).  Host-only: the
writers run in libddpma.so without a GPU."""

from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import GOLDEN

import paper_2006_14602_b200 as P
from paper_2006_14602_b200 import fileio as F
from paper_2006_14602_b200.schwarz import PhysicalMesh


def _read(path):
    with open(path, "rb") as fp:
        return fp.read()


@pytest.mark.parametrize("tag", ["2d", "3d"])
def test_mesh_vtk_bytes_and_roundtrip(tag, tmp_path):
    z = np.load(os.path.join(GOLDEN, "fileio_inputs.npz"))
    c, j, e = z[f"{tag}_c"], z[f"{tag}_j"], z[f"{tag}_e"]
    out = tmp_path / "m.vtk"
    F.write_mesh_vtk(PhysicalMesh(coords=c, jac=j), str(out), e_adp=e)
    assert _read(out) == _read(os.path.join(GOLDEN, f"ref_mesh{tag}.vtk"))
    m = F.read_mesh_vtk(str(out))
    assert np.array_equal(m.coords, c, equal_nan=True)
    assert np.array_equal(m.jac, j)
    dims, pts, data = F.read_structured_vtk(str(out))
    assert np.array_equal(data["e_adp"], e.ravel(order="F"))


def test_scalar_field_and_csv(tmp_path):
    axes = (np.linspace(0.0, 1.0, 5), np.linspace(-1.0, 2.0, 4))
    vals = np.arange(20.0).reshape(5, 4) / 7.0
    out = tmp_path / "f.vtk"
    F.write_scalar_field_vtk(axes, vals, str(out), name="rho")
    assert _read(out) == _read(os.path.join(GOLDEN, "ref_field.vtk"))
    ax, v = F.read_scalar_field_vtk(str(out))
    assert np.array_equal(v, vals) and all(np.array_equal(a, b) for a, b in zip(ax, axes))
    csv = tmp_path / "r.csv"
    F.write_field_csv(str(csv), ["n", "e2", "name"],
                      [(33, 0.1, "a"), (65, 1.0 / 3.0, "b"), (129, float("nan"), "c")])
    assert _read(csv) == _read(os.path.join(GOLDEN, "ref_report.csv"))


def test_reader_errors(tmp_path):
    bad = tmp_path / "bad.vtk"
    bad.write_text("# vtk DataFile Version 3.0\nother title v1\nASCII\n")
    with pytest.raises(P.MeshFileError, match="line 2: not a ddmesh VTK file"):
        F.read_mesh_vtk(str(bad))
    src = _read(os.path.join(GOLDEN, "ref_mesh2d.vtk")).decode()
    trunc = tmp_path / "trunc.vtk"
    trunc.write_text(src[: len(src) // 3].rsplit("\n", 1)[0] + "\n")
    with pytest.raises(P.MeshFileError, match="unexpected end of file"):
        F.read_mesh_vtk(str(trunc))
    wrong = tmp_path / "wrong.vtk"
    wrong.write_text(src.replace("POINTS 30", "POINTS 31", 1))
    with pytest.raises(P.MeshFileError, match="POINTS count 31"):
        F.read_mesh_vtk(str(wrong))
    with pytest.raises(OSError):
        F.write_mesh_vtk(PhysicalMesh(coords=np.zeros((3, 3, 2)), jac=np.zeros((3, 3))),
                         str(tmp_path / "no" / "dir" / "x.vtk"))
