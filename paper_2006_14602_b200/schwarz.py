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
        stats["sub_rhs_evals"] = plan.sub_evals()
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


# ------------------------------------------------------------ sweeps ----
# The reference's window-level API (schwarz.py:70-81,118-134,216-268): a list
# of per-subdomain states advanced one window at a time by
# ``alternating_sweep`` / ``parallel_sweep``.  Here the states are views of
# one device plan; a sweep is one window of the device window loop (density
# pass, traces, every subdomain's integrator, mesh/residual pass).

class SubdomainState:
    """Per-subdomain view of a device sweep state (schwarz.py:70-81):
    ``psi``, ``mesh`` and ``res`` read the device state of the last sweep."""

    def __init__(self, states: "SweepStates", sub):
        self._states = states
        self.sub = sub
        from .grid import subdomain_geometry
        self.geom = subdomain_geometry(states.grid, sub)
        self.mask = self.geom.dirichlet_mask()
        self.integrator = None   # lives in the device controller
        self._cache = {}

    @property
    def psi(self) -> np.ndarray:
        if "psi" not in self._cache:
            self._cache["psi"] = self._states._sub_psi(self.sub.id)
        return self._cache["psi"]

    @property
    def mesh(self) -> PhysicalMesh:
        if "mesh" not in self._cache:
            from .pma import physical_mesh
            self._cache["mesh"] = physical_mesh(self.psi, self.geom)
        return self._cache["mesh"]

    @property
    def res(self) -> float:
        return self._states._res.get(self.sub.id, np.inf)


class SweepStates(list):
    """``init_states`` result: the SubdomainState list plus the device plan
    (created by the first sweep, which knows the monitor and transmission)."""

    def __init__(self, grid: CompGrid, dec: Decomposition, config: SolverConfig, initial):
        self.grid, self.dec, self.config, self.initial = grid, dec, config, initial
        self.plan = None
        self.transmission = None
        self.mon = None
        self._res = {}
        super().__init__(SubdomainState(self, sub) for sub in dec.subdomains)

    def _sub_psi(self, sid):
        if self.plan is None:
            from .pma import initial_potential
            if self.initial is None:
                return initial_potential(self[sid].geom)
            return np.array(self.initial[self.dec.subdomains[sid].slices()], copy=True)
        return self.plan.sub_psi(sid)

    def _sweep(self, mon, config, dec, transmission):
        import dataclasses
        if dec is not self.dec and dec.subdomains != self.dec.subdomains:
            raise ConfigurationError("sweep decomposition differs from init_states'")
        if self.plan is None:
            cfg = dataclasses.replace(config, transmission=transmission, tol=1e-300)
            self.plan = Plan.for_grid(self.grid, self.dec.subdomains, mon, cfg)
            self.plan.set_state(self.initial)
            self.transmission, self.mon, self.config = transmission, mon, config
        elif transmission != self.transmission or mon is not self.mon:
            raise ConfigurationError("one state set runs one transmission mode and monitor "
                                     "on the device path")
        _w, _c, _f, hres, _hs = self.plan.run(1, 1e-300)
        self._res = {i: float(hres[0][i]) for i in range(self.dec.nsub)}
        for st in self:
            st._cache.clear()

    def close(self):
        if self.plan is not None:
            self.plan.close()
            self.plan = None


def init_states(grid: CompGrid, dec: Decomposition, config: SolverConfig,
                initial: np.ndarray | None = None) -> SweepStates:
    """schwarz.py:118-134: fresh integrators, psi from ``initial`` or psi0."""
    _validate(config)
    if initial is not None:
        initial = np.asarray(initial)
        if initial.shape != grid.counts:
            raise ConfigurationError(
                f"warm-start field shape {initial.shape} != grid {grid.counts}")
    return SweepStates(grid, dec, config, initial)


def _check_states(states):
    if not isinstance(states, SweepStates):
        raise ConfigurationError("sweeps run on device states: create them with init_states")


def alternating_sweep(states, mon: MonitorField, config: SolverConfig, dec: Decomposition,
                      weights: np.ndarray | None = None) -> None:
    """One serial sweep in id order, each subdomain reading the freshest
    neighbour traces (schwarz.py:216-233); the device runs the serial chain.
    ``weights`` (the global trapezoid weights) are formed on the device."""
    _check_states(states)
    states._sweep(mon, config, dec, "alternating")


def parallel_sweep(states, mon: MonitorField, config: SolverConfig, dec: Decomposition,
                   pool=None, weights: np.ndarray | None = None) -> None:
    """One parallel sweep from the level-n snapshot (schwarz.py:236-268).
    ``pool`` is accepted for signature compatibility: every subdomain's
    integrator already runs concurrently inside the device window kernel,
    and failures are reported for the lowest subdomain id as in the
    reference."""
    _check_states(states)
    states._sweep(mon, config, dec, "parallel")


def residual(psi_new: np.ndarray, psi_old: np.ndarray, geom: BoxGeometry) -> float:
    """Trapezoid-weighted L2 norm of the window update (schwarz.py:111-115)."""
    if psi_new.shape != psi_old.shape:
        raise ValueError(f"field shapes differ: {psi_new.shape} vs {psi_old.shape}")
    from .pma import _plan
    with _plan(geom) as plan:
        return plan.residual(0, psi_new, psi_old)
