"""Grids, overlapping decompositions and box geometry — the reference's
``ddmesh.grid`` interface (grid.py:24-307) with the decomposition computed by
the native host layer (``ddpma_build_decomposition``, csrc/decomp.cpp).

The returned objects have the reference's fields, so code written against
``ddmesh`` (``sub.box``, ``sub.owned``, ``sub.neighbors``, ``slices()``…)
runs unchanged.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigurationError

PHYSICAL = "physical"      # grid.py:20
INTERFACE = "interface"    # grid.py:21


@dataclass(frozen=True)
class CompGrid:
    """Uniform node-centred grid (grid.py:24-55)."""

    dim: int
    extents: tuple[tuple[float, float], ...]
    counts: tuple[int, ...]

    @property
    def spacing(self) -> tuple[float, ...]:
        return tuple((b - a) / (n - 1) for (a, b), n in zip(self.extents, self.counts))

    @property
    def measure(self) -> float:
        out = 1.0
        for a, b in self.extents:
            out *= b - a
        return out

    def axes(self) -> tuple[np.ndarray, ...]:
        return tuple(a + np.arange(n) * h
                     for (a, _), n, h in zip(self.extents, self.counts, self.spacing))

    def shape(self) -> tuple[int, ...]:
        return self.counts


def build_grid(dim: int, extents, counts) -> CompGrid:
    """Validate and build a CompGrid (grid.py:58-75; same messages)."""
    if dim not in (2, 3):
        raise ConfigurationError(f"dim must be 2 or 3, got {dim}")
    extents = tuple((float(a), float(b)) for a, b in extents)
    counts = tuple(int(n) for n in counts)
    if len(extents) != dim or len(counts) != dim:
        raise ConfigurationError(
            f"need {dim} extents and counts, got {len(extents)} and {len(counts)}")
    for (a, b) in extents:
        if not np.isfinite([a, b]).all() or b <= a:
            raise ConfigurationError(f"degenerate extent [{a}, {b}]")
    for n in counts:
        if n < 3:
            raise ConfigurationError(f"need at least 3 nodes per axis, got {n}")
    return CompGrid(dim=dim, extents=extents, counts=counts)


@dataclass(frozen=True)
class Subdomain:
    """One overlapping index box (grid.py:78-110)."""

    id: int
    pos: tuple[int, ...]
    box: tuple[tuple[int, int], ...]
    faces: tuple[tuple[str, str], ...]
    neighbors: dict
    owned: tuple[tuple[int, int], ...]

    def shape(self) -> tuple[int, ...]:
        return tuple(hi - lo + 1 for lo, hi in self.box)

    def slices(self) -> tuple[slice, ...]:
        return tuple(slice(lo, hi + 1) for lo, hi in self.box)

    def owned_global_slices(self) -> tuple[slice, ...]:
        return tuple(slice(lo, hi + 1) for lo, hi in self.owned)

    def owned_local_slices(self) -> tuple[slice, ...]:
        return tuple(slice(olo - blo, ohi - blo + 1)
                     for (olo, ohi), (blo, _) in zip(self.owned, self.box))


@dataclass(frozen=True)
class Decomposition:
    grid: CompGrid
    layout: tuple[int, ...]
    overlap: int
    subdomains: tuple[Subdomain, ...]

    @property
    def nsub(self) -> int:
        return len(self.subdomains)


def _from_c(s: _lib.Subdomain, dim: int) -> Subdomain:
    kinds = {_lib.FACE_PHYSICAL: PHYSICAL, _lib.FACE_INTERFACE: INTERFACE}
    neighbors = {}
    for k in range(dim):
        for side in (0, 1):
            if s.donor[k][side] >= 0:
                neighbors[(k, side)] = int(s.donor[k][side])
    return Subdomain(
        id=int(s.id), pos=tuple(int(s.pos[k]) for k in range(dim)),
        box=tuple((int(s.box[k][0]), int(s.box[k][1])) for k in range(dim)),
        faces=tuple((kinds[s.face[k][0]], kinds[s.face[k][1]]) for k in range(dim)),
        neighbors=neighbors,
        owned=tuple((int(s.owned[k][0]), int(s.owned[k][1])) for k in range(dim)))


def to_c(sub: Subdomain, dim: int) -> _lib.Subdomain:
    out = _lib.Subdomain()
    out.id = sub.id
    for k in range(3):
        out.donor[k][0] = out.donor[k][1] = -1
    for k in range(dim):
        out.pos[k] = sub.pos[k]
        out.box[k][0], out.box[k][1] = sub.box[k]
        out.owned[k][0], out.owned[k][1] = sub.owned[k]
        for side in (0, 1):
            out.face[k][side] = (_lib.FACE_PHYSICAL if sub.faces[k][side] == PHYSICAL
                                 else _lib.FACE_INTERFACE)
            out.donor[k][side] = sub.neighbors.get((k, side), -1)
    return out


def alternating_levels(dec: "Decomposition") -> list[int]:
    """Wavefront level of every subdomain under alternating transmission
    (native host code, ``ddpma_alternating_levels``): the id-ordered sweep of
    ``ddmesh/schwarz.py:216-233`` only orders a subdomain after its face
    neighbours of lower id, so equal-level subdomains are independent and the
    device advances them in one launch."""
    dim = len(dec.subdomains[0].pos)
    arr = (_lib.Subdomain * dec.nsub)(*[to_c(s, dim) for s in dec.subdomains])
    lev = (C.c_int * dec.nsub)()
    _lib.lib().ddpma_alternating_levels(dim, arr, dec.nsub, lev)
    return list(lev)


def build_decomposition(grid: CompGrid, layout, overlap: int = 3) -> Decomposition:
    """Overlapping slab/block decomposition (grid.py:176-237), computed by the
    native host layer; bit-exact boxes, ownership, faces and donor ids."""
    layout = tuple(int(m) for m in layout)
    if len(layout) != grid.dim:
        raise ConfigurationError(f"layout {layout} does not match dim {grid.dim}")
    dim = grid.dim
    counts = (C.c_int * 3)(*grid.counts, *([1] * (3 - dim)))
    lay = (C.c_int * 3)(*layout, *([1] * (3 - dim)))
    nsub = C.c_int(0)
    L = _lib.lib()
    _lib.check_global(L.ddpma_build_decomposition(dim, counts, lay, int(overlap), None, 0,
                                                  C.byref(nsub)))
    arr = (_lib.Subdomain * nsub.value)()
    _lib.check_global(L.ddpma_build_decomposition(dim, counts, lay, int(overlap), arr,
                                                  nsub.value, C.byref(nsub)))
    subs = tuple(_from_c(arr[i], dim) for i in range(nsub.value))
    return Decomposition(grid=grid, layout=layout, overlap=overlap, subdomains=subs)


@dataclass(frozen=True)
class BoxGeometry:
    """Geometry of one index box (grid.py:261-288)."""

    axes: tuple[np.ndarray, ...]
    spacing: tuple[float, ...]
    faces: tuple[tuple[str, str], ...]
    domain_measure: float

    @property
    def dim(self) -> int:
        return len(self.axes)

    def shape(self) -> tuple[int, ...]:
        return tuple(len(ax) for ax in self.axes)

    def dirichlet_mask(self) -> np.ndarray:
        mask = np.zeros(self.shape(), dtype=bool)
        for k, (lo_kind, hi_kind) in enumerate(self.faces):
            sl = [slice(None)] * self.dim
            if lo_kind == INTERFACE:
                sl[k] = 0
                mask[tuple(sl)] = True
            if hi_kind == INTERFACE:
                sl[k] = -1
                mask[tuple(sl)] = True
        return mask


def grid_geometry(grid: CompGrid) -> BoxGeometry:
    """Geometry of the whole grid (grid.py:297-301)."""
    return BoxGeometry(axes=grid.axes(), spacing=grid.spacing,
                       faces=tuple((PHYSICAL, PHYSICAL) for _ in range(grid.dim)),
                       domain_measure=grid.measure)


def subdomain_geometry(grid: CompGrid, sub: Subdomain) -> BoxGeometry:
    """grid.py:304-307."""
    axes = tuple(ax[lo:hi + 1] for ax, (lo, hi) in zip(grid.axes(), sub.box))
    return BoxGeometry(axes=axes, spacing=grid.spacing, faces=sub.faces,
                       domain_measure=grid.measure)
