"""Operator-level PMA API (ddmesh/pma.py) evaluated by the CUDA kernels.

Each call stages the box into a single-box device plan built from the given
``BoxGeometry`` and runs the same kernels the solver uses; these are the
parity seams of the operator tests.  Plans are cached per (geometry,
det_floor, monitor), so a caller looping over ``pma_rhs_frozen`` /
``hessian_det_fd`` on one box pays the plan setup (arena, tensor maps,
coefficient tables) once.
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from contextlib import contextmanager
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from .grid import BoxGeometry
from .monitor import MonitorField
from .plan import Plan
from .schwarz import DET_FLOOR, PhysicalMesh, SolverConfig


class RhsEval(NamedTuple):
    values: np.ndarray
    det_clamped: bool


@dataclass
class PotentialField:
    """Nodal values of the mesh potential on one index box (pma.py:27-33)."""

    values: np.ndarray
    geom: BoxGeometry
    tau: float = 0.0


def initial_potential(geom: BoxGeometry) -> np.ndarray:
    """psi0 = |xi|^2 / 2 on the box's own node coordinates (pma.py:61-64).

    A setup helper evaluated from the geometry's axes exactly as the
    reference writes it; the solver's own psi0 is formed on the device
    (k_psi0) from the global grid and is bitwise identical to this on every
    subdomain box (both are ``0.5 * (x0*x0 + x1*x1 [+ x2*x2])`` of the same
    axis values)."""
    squares = np.meshgrid(*[ax * ax for ax in geom.axes], indexing="ij")
    return 0.5 * np.sum(squares, axis=0)


def _geom_key(geom: BoxGeometry):
    return (tuple((float(ax[0]), float(ax[-1]), len(ax)) for ax in geom.axes),
            tuple(float(h) for h in geom.spacing), tuple(tuple(f) for f in geom.faces),
            float(geom.domain_measure))


_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_MAX = 8
_LOCK = threading.RLock()


@contextmanager
def _plan(geom: BoxGeometry, det_floor: float = DET_FLOOR, mon: MonitorField | None = None):
    """A cached single-box plan (one caller at a time: plans are not
    re-entrant, ddpma.h).  The monitor is part of the key by identity and the
    cache entry keeps it alive, so an id is never reused while cached."""
    key = (_geom_key(geom), float(det_floor), None if mon is None else id(mon))
    with _LOCK:
        ent = _CACHE.pop(key, None)
        if ent is None:
            ent = (Plan.for_geometry(geom, SolverConfig(det_floor=det_floor), mon), mon)
        _CACHE[key] = ent
        while len(_CACHE) > _CACHE_MAX:
            _, (old, _m) = _CACHE.popitem(last=False)
            old.close()
        yield ent[0]


def clear_plan_cache() -> None:
    with _LOCK:
        while _CACHE:
            _, (p, _m) = _CACHE.popitem()
            p.close()


def pma_rhs_frozen(psi: np.ndarray, rho_values: np.ndarray, geom: BoxGeometry,
                   det_floor: float = DET_FLOOR, dirichlet_mask: np.ndarray | None = None,
                   max_rho: float | None = None) -> RhsEval:
    """Frozen-density right-hand side and positivity flag (pma.py:195-219).
    The Dirichlet mask is derived from ``geom.faces`` (as the reference's
    default does); a custom mask is not supported on the device path."""
    if dirichlet_mask is not None and not np.array_equal(dirichlet_mask, geom.dirichlet_mask()):
        from .errors import ConfigurationError
        raise ConfigurationError("custom dirichlet masks are not supported on the device path")
    with _plan(geom, det_floor) as p:
        f, flag = p.rhs_frozen(0, psi, rho_values, max_rho)
    return RhsEval(f, flag)


def hessian_det_fd(psi: np.ndarray, geom: BoxGeometry) -> np.ndarray:
    """Discrete Hessian determinant (pma.py:133-149)."""
    with _plan(geom) as p:
        return p.mesh(0, psi)[1]


def gradient_fd(psi: np.ndarray, geom: BoxGeometry) -> list[np.ndarray]:
    """Per-axis mesh coordinates (pma.py:67-84)."""
    with _plan(geom) as p:
        coords = p.mesh(0, psi)[0]
    return [coords[..., k] for k in range(geom.dim)]


def physical_mesh(psi: np.ndarray, geom: BoxGeometry) -> PhysicalMesh:
    """Coordinates and Jacobian (pma.py:222-225)."""
    with _plan(geom) as p:
        coords, jac = p.mesh(0, psi)
    return PhysicalMesh(coords=coords, jac=jac)


def mesh_density(mon: MonitorField, psi: np.ndarray, geom: BoxGeometry) -> np.ndarray:
    """Unnormalised nodal density on the mesh of ``psi`` (monitor.py:151-180,
    density-only monitors), evaluated on the device."""
    with _plan(geom, mon=mon) as p:
        return p.raw_density(0, psi)


def pma_rhs(psi: np.ndarray, monitor: MonitorField, geom: BoxGeometry,
            det_floor: float = DET_FLOOR,
            dirichlet_mask: np.ndarray | None = None) -> RhsEval:
    """Moving-point right-hand side (pma.py:152-183): the monitor evaluated at
    the clamped mesh points of ``psi`` (``eval_clamped``: analytic raw over the
    normaliser, never the u pull-back) with the guard from ``max_value``.
    Exported by the reference but unused by its ``solve``;
    here a composition of the device mesh-density and frozen-RHS kernels."""
    if dirichlet_mask is not None and not np.array_equal(dirichlet_mask, geom.dirichlet_mask()):
        from .errors import ConfigurationError
        raise ConfigurationError("custom dirichlet masks are not supported on the device path")
    analytic = MonitorField(raw=monitor.raw, domain=monitor.domain)
    with _plan(geom, det_floor, analytic) as p:
        rho = p.raw_density(0, psi) / monitor.normalizer
        f, flag = p.rhs_frozen(0, psi, rho, getattr(monitor, "max_value", None))
    return RhsEval(f, flag)
