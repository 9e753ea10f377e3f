"""Mesh output formats (ddmesh/fileio.py:1-230).

Legacy-VTK structured grids and CSV reports, ASCII with 17 significant
digits so write/read round-trips are exact.  The VTK writer is native
(``ddpma_write_mesh_vtk`` in libddpma.so: rows formatted on every host
thread) and byte-identical to the reference writer; the readers restate the
reference's token reader with its ``MeshFileError`` messages and line numbers.
"""

from __future__ import annotations

import ctypes as C
from typing import Iterable

import numpy as np

from . import _lib
from .errors import MeshFileError
from .schwarz import PhysicalMesh

VTK_TITLE = "ddmesh structured-grid v1"      # fileio.py:20
CSV_HEADER_COMMENT = "# ddmesh report v1"    # fileio.py:21


def _write_vtk(coords: np.ndarray, first: np.ndarray, name: str, path: str,
               e_adp: np.ndarray | None) -> None:
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    dim = coords.shape[-1]
    counts = coords.shape[:-1]
    if dim not in (2, 3) or len(counts) != dim:
        raise ValueError("coords must have shape counts + (dim,) with dim 2 or 3")
    jac = np.ascontiguousarray(first, dtype=np.float64).reshape(counts)
    e = None if e_adp is None else np.ascontiguousarray(e_adp, dtype=np.float64).reshape(counts)
    cnt = (C.c_int * 3)(*(list(counts) + [1] * (3 - dim)))
    L = _lib.lib()
    st = L.ddpma_write_mesh_vtk(str(path).encode(), dim, cnt, _lib.dptr(coords), _lib.dptr(jac),
                                None if e is None else _lib.dptr(e), VTK_TITLE.encode(),
                                name.encode())
    if st != _lib.OK:
        _lib.raise_status(st, L.ddpma_io_error().decode())


def write_mesh_vtk(mesh: PhysicalMesh, path: str, e_adp: np.ndarray | None = None) -> None:
    """Structured mesh with its Jacobian (and optional quality field) as point
    data (fileio.py:45-68)."""
    _write_vtk(mesh.coords, mesh.jac, "jacobian", path, e_adp)


def write_scalar_field_vtk(axes: tuple[np.ndarray, ...], values: np.ndarray, path: str,
                           name: str = "u") -> None:
    """Scalar sampled on a uniform lattice (monitor ingestion format, fileio.py:71-80)."""
    mesh = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1)
    _write_vtk(mesh, values, name, path, None)


def _cell(v) -> str:
    return "%.17g" % v if isinstance(v, float) else str(v)


def write_field_csv(path: str, header: list[str], rows: Iterable[Iterable]) -> None:
    """One report row per sweep point; floats keep 17 significant digits
    (fileio.py:215-223)."""
    with open(path, "w", newline="\n") as fp:
        fp.write(CSV_HEADER_COMMENT + "\n")
        fp.write(",".join(header) + "\n")
        for row in rows:
            fp.write(",".join(_cell(v) for v in row) + "\n")


# ------------------------------------------------------------- readers --

class _Tokens:
    """Whitespace tokens with line numbers (fileio.py:83-132)."""

    def __init__(self, path: str):
        with open(path) as fp:
            self.lines = fp.read().splitlines()
        self.q: list[tuple[str, int]] = []
        self.pos = 0
        self.ln = 0

    def _fill(self) -> None:
        while self.pos >= len(self.q):
            if self.ln >= len(self.lines):
                raise MeshFileError("unexpected end of file", self.ln)
            self.q = [(t, self.ln + 1) for t in self.lines[self.ln].split()]
            self.pos = 0
            self.ln += 1

    def next(self) -> tuple[str, int]:
        self._fill()
        t = self.q[self.pos]
        self.pos += 1
        return t

    def expect(self, *words: str) -> None:
        for w in words:
            tok, line = self.next()
            if tok != w:
                raise MeshFileError(f"expected {w!r}, found {tok!r}", line)

    def number(self, kind=float):
        tok, line = self.next()
        try:
            return kind(tok)
        except ValueError:
            what = "a number" if kind is float else "an integer"
            raise MeshFileError(f"expected {what}, found {tok!r}", line) from None

    def at_eof(self) -> bool:
        try:
            self._fill()
        except MeshFileError:
            return True
        return False


def read_structured_vtk(path: str):
    """Dimensions, (n, 3) points and named point scalars (fileio.py:135-175)."""
    t = _Tokens(path)
    t.expect("#", "vtk", "DataFile", "Version")
    t.next()
    title, line = t.next()
    if title != "ddmesh":
        raise MeshFileError(f"not a ddmesh VTK file (title {title!r})", line)
    t.next()
    t.next()
    t.expect("ASCII", "DATASET")
    tok, line = t.next()
    if tok != "STRUCTURED_GRID":
        raise MeshFileError(f"unsupported dataset {tok!r}", line)
    t.expect("DIMENSIONS")
    dims = (t.number(int), t.number(int), t.number(int))
    t.expect("POINTS")
    n = t.number(int)
    if n != dims[0] * dims[1] * dims[2]:
        raise MeshFileError(f"POINTS count {n} != product of DIMENSIONS {dims}")
    t.next()
    points = np.array([t.number() for _ in range(3 * n)], dtype=np.float64).reshape(n, 3)
    data: dict[str, np.ndarray] = {}
    if not t.at_eof():
        t.expect("POINT_DATA")
        m = t.number(int)
        if m != n:
            raise MeshFileError(f"POINT_DATA count {m} != POINTS count {n}")
        while not t.at_eof():
            t.expect("SCALARS")
            name, _ = t.next()
            t.next()
            t.expect("LOOKUP_TABLE")
            t.next()
            data[name] = np.array([t.number() for _ in range(n)])
    return dims, points, data


def _grid(dims, flat):
    nx, ny, nz = dims
    arr = flat.reshape((nz, ny, nx)).transpose(2, 1, 0)
    return arr[:, :, 0] if nz == 1 else arr


def read_mesh_vtk(path: str) -> PhysicalMesh:
    """Inverse of write_mesh_vtk (fileio.py:185-195)."""
    dims, points, data = read_structured_vtk(path)
    dim = 2 if dims[2] == 1 else 3
    coords = np.stack([_grid(dims, points[:, k]) for k in range(dim)], axis=-1)
    jac = _grid(dims, data["jacobian"]) if "jacobian" in data else np.full(coords.shape[:-1],
                                                                               np.nan)
    return PhysicalMesh(coords=coords, jac=jac)


def read_scalar_field_vtk(path: str):
    """Scalar lattice field of write_scalar_field_vtk (fileio.py:198-212)."""
    dims, points, data = read_structured_vtk(path)
    dim = 2 if dims[2] == 1 else 3
    if len(data) != 1:
        raise MeshFileError(f"expected exactly one scalar field, found {sorted(data)}")
    values = _grid(dims, next(iter(data.values())))
    coords = [_grid(dims, points[:, k]) for k in range(dim)]
    axes = []
    for k in range(dim):
        take = [0] * dim
        take[k] = slice(None)
        axes.append(np.asarray(coords[k][tuple(take)]))
    return tuple(axes), values
