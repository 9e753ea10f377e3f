"""Operator-level PMA API (ddmesh/pma.py) evaluated by the CUDA kernels.

Each call stages the box into a single-box device plan built from the given
``BoxGeometry`` and runs the same kernels the solver uses; these are the
parity seams of the operator tests.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

from .grid import BoxGeometry
from .monitor import MonitorField
from .plan import Plan
from .schwarz import DET_FLOOR, PhysicalMesh, SolverConfig


class RhsEval(NamedTuple):
    values: np.ndarray
    det_clamped: bool


def _plan(geom: BoxGeometry, det_floor: float = DET_FLOOR, mon: MonitorField | None = None):
    return Plan.for_geometry(geom, SolverConfig(det_floor=det_floor), mon)


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
