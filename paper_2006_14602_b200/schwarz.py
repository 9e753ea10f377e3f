"""Non-iterative overlapping Schwarz solve — the reference's public entry points
(ddmesh/schwarz.py:35-406) on the B200 path.

``solve`` and ``solve_single_domain`` take the reference's arguments and
return the reference's ``SolveResult`` (assembled ``psi``, ``mesh.coords``,
``mesh.jac``, ``sub_psi``, per-window ``history`` …).  The window loop, the
RKC2/Euler integrators, densities, traces, residuals and the owned-block
assembly all run inside libddpma.so on the GPU; this module
only validates arguments and marshals results.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError
from .grid import BoxGeometry, CompGrid, Decomposition, build_decomposition
from .integrate import IntegrationWindow
from .monitor import MonitorField
from .plan import Plan

DET_FLOOR = 1e-12   # pma.py:23


@dataclass(frozen=True)
class SolverConfig:
    """Pseudo-time window, stopping rule, transmission mode, integrator
    (schwarz.py:35-67; same fields, defaults and validation)."""

    dtau: float = 1e-3
    tol: float = 1e-6
    transmission: str = "alternating"
    stop_rule: str = "min"
    max_windows: int = 5000
    workers: int | None = None
    scheme: str = "adaptive"
    substeps: int = 1
    rtol: float = 1e-3
    atol: float = 1e-6
    max_stages: int = 512
    det_floor: float = DET_FLOOR
    monitor_smooth_passes: int = 0
    monitor_relax: float = 0.0

    def __post_init__(self):
        if self.tol <= 0.0:
            raise ConfigurationError(f"tol must be > 0, got {self.tol}")
        if self.max_windows < 1:
            raise ConfigurationError("max_windows must be >= 1")
        if self.transmission not in ("alternating", "parallel"):
            raise ConfigurationError(f"unknown transmission {self.transmission!r}")
        if self.stop_rule not in ("min", "max"):
            raise ConfigurationError(f"unknown stop rule {self.stop_rule!r}")

    def window(self) -> IntegrationWindow:
        return IntegrationWindow(dtau=self.dtau, scheme=self.scheme,
                                 substeps=self.substeps, rtol=self.rtol,
                                 atol=self.atol, max_stages=self.max_stages)


@dataclass(frozen=True)
class WindowRecord:
    residuals: tuple[float, ...]
    stop_residual: float
    jac_min: float
    jac_max: float
    seconds: float


@dataclass(frozen=True)
class PhysicalMesh:
    """Mesh map x = grad(psi) and its Jacobian determinant (pma.py:35-47)."""

    coords: np.ndarray
    jac: np.ndarray

    @property
    def dim(self) -> int:
        return self.coords.shape[-1]

    def min_jac(self) -> float:
        return float(self.jac.min())


@dataclass
class SolveResult:
    """schwarz.py:93-108."""

    psi: np.ndarray
    mesh: PhysicalMesh
    sub_psi: list[np.ndarray]
    history: list[WindowRecord] = field(default_factory=list)
    converged: bool = False
    windows: int = 0
    final_residual: float = np.inf
    overlap_gap: float = 0.0
    stats: dict = field(default_factory=dict)   # device counters (node-updates, …)

    @property
    def min_jac(self) -> float:
        return float(self.mesh.jac.min())


def _validate(config: SolverConfig):
    config.window()   # IntegrationWindow validation (integrate.py:52-60)


def _history(hist_res, hist_stats):
    return [WindowRecord(residuals=tuple(float(x) for x in hist_res[w]),
                         stop_residual=float(hist_stats[w, 0]),
                         jac_min=float(hist_stats[w, 1]), jac_max=float(hist_stats[w, 2]),
                         seconds=float(hist_stats[w, 3]))
            for w in range(hist_res.shape[0])]


def _solve_plan(grid: CompGrid, dec: Decomposition, mon: MonitorField, config: SolverConfig,
                initial, single: bool) -> SolveResult:
    _validate(config)
    if initial is not None:
        initial = np.asarray(initial)
        if initial.shape != grid.counts:
            raise ConfigurationError(
                f"warm-start field shape {initial.shape} != grid {grid.counts}")
    with Plan.for_grid(grid, dec.subdomains, mon, config) as plan:
        plan.set_state(initial)
        w, conv, fres, hres, hstats = plan.run(config.max_windows, config.tol)
        psi, coords, jac = plan.assemble(grid.counts)
        sub_psi = [psi] if single else [plan.sub_psi(i) for i in range(dec.nsub)]
        gap = 0.0 if single else plan.overlap_gap()
        stats = plan.counters()
    return SolveResult(psi=psi, mesh=PhysicalMesh(coords=coords, jac=jac), sub_psi=sub_psi,
                       history=_history(hres, hstats), converged=conv, windows=w,
                       final_residual=fres, overlap_gap=gap, stats=stats)


def solve(grid: CompGrid, dec: Decomposition, mon: MonitorField,
          config: SolverConfig, initial: np.ndarray | None = None) -> SolveResult:
    """Run windows until the stop rule over subdomain residuals meets tol
    (schwarz.py:307-350).  Non-convergence is reported, not raised."""
    return _solve_plan(grid, dec, mon, config, initial, single=False)


def solve_single_domain(grid: CompGrid, mon: MonitorField, config: SolverConfig,
                        initial: np.ndarray | None = None) -> SolveResult:
    """Whole-domain relaxation (schwarz.py:353-406) — a 1x1 decomposition,
    which the reference itself makes bitwise identical."""
    dec = build_decomposition(grid, (1,) * grid.dim, 3)
    return _solve_plan(grid, dec, mon, config, initial, single=True)


def residual(psi_new: np.ndarray, psi_old: np.ndarray, geom: BoxGeometry) -> float:
    """Trapezoid-weighted L2 norm of the window update (schwarz.py:111-115)."""
    if psi_new.shape != psi_old.shape:
        raise ValueError(f"field shapes differ: {psi_new.shape} vs {psi_old.shape}")
    with Plan.for_geometry(geom, SolverConfig()) as plan:
        return plan.residual(0, psi_new, psi_old)
