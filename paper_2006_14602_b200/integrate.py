"""Integration windows, RKC2 coefficients and the integrator protocol
(ddmesh/integrate.py:33-262) on the device.

``make_integrator(window)`` returns an integrator whose ``advance(y,
rhs_fn)`` runs the reference's Rkc2Integrator / EulerIntegrator controller
(integrate.py:63-250) inside the persistent CUDA window kernel.  A Python
``rhs_fn`` cannot be called per node on the GPU, so ``advance`` accepts the
one right-hand side the reference's solver builds (schwarz.py:201-205): the
frozen-density PMA operator ``pma_rhs_frozen`` bound to a nodal density and a
box geometry — a :class:`FrozenPmaRhs` (``frozen_rhs(...)``) or a
``functools.partial`` of ``pma_rhs_frozen``.  Anything else raises
``ConfigurationError``; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import functools
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigurationError, StiffnessError

DET_FLOOR = 1e-12   # pma.py:23


@dataclass(frozen=True)
class IntegrationWindow:
    """One pseudo-time window (integrate.py:41-60)."""

    dtau: float
    scheme: str = "adaptive"
    substeps: int = 1
    rtol: float = 1e-3
    atol: float = 1e-6
    max_stages: int = 512

    def __post_init__(self):
        if self.dtau <= 0.0:
            raise ConfigurationError(f"window length must be > 0, got {self.dtau}")
        if self.scheme not in ("adaptive", "euler"):
            raise ConfigurationError(f"unknown scheme {self.scheme!r}")
        if self.scheme == "euler" and self.substeps < 1:
            raise ConfigurationError("euler mode needs at least 1 substep")
        if self.rtol <= 0.0 or self.atol <= 0.0:
            raise ConfigurationError("rtol and atol must be positive")


def rkc_coeffs(s: int):
    """(w0, w1, mu1_t, mu, nu, mu_t, gamma_t) of the s-stage damped RKC2
    scheme, computed by the native controller (integrate.py:77-106)."""
    arrs = [np.zeros(s + 1) for _ in range(4)]
    w0, w1, m1 = C.c_double(), C.c_double(), C.c_double()
    _lib.check_global(_lib.lib().ddpma_rkc_coeffs(int(s), C.byref(w0), C.byref(w1),
                                                  C.byref(m1), *[_lib.dptr(a) for a in arrs]))
    return (w0.value, w1.value, m1.value, *arrs)


class FrozenPmaRhs:
    """``y -> pma_rhs_frozen(y, rho_values, geom, det_floor, mask, max_rho)``:
    the right-hand side closure of schwarz._advance_state (schwarz.py:201-205).
    Calling it evaluates the operator on the device (returns (F, flag)); the
    device integrators consume its parameters directly."""

    def __init__(self, rho_values, geom, det_floor: float = DET_FLOOR,
                 dirichlet_mask=None, max_rho=None):
        self.rho_values = np.asarray(rho_values, dtype=np.float64)
        self.geom = geom
        self.det_floor = float(det_floor)
        self.dirichlet_mask = dirichlet_mask
        self.max_rho = max_rho

    def __call__(self, y):
        from .pma import pma_rhs_frozen
        return pma_rhs_frozen(y, self.rho_values, self.geom, self.det_floor,
                              self.dirichlet_mask, self.max_rho)


def frozen_rhs(rho_values, geom, det_floor: float = DET_FLOOR, dirichlet_mask=None,
               max_rho=None) -> FrozenPmaRhs:
    return FrozenPmaRhs(rho_values, geom, det_floor, dirichlet_mask, max_rho)


def _as_frozen(rhs_fn) -> FrozenPmaRhs:
    if isinstance(rhs_fn, FrozenPmaRhs):
        return rhs_fn
    if isinstance(rhs_fn, functools.partial):
        from .pma import pma_rhs_frozen
        if rhs_fn.func is pma_rhs_frozen:
            names = ("rho_values", "geom", "det_floor", "dirichlet_mask", "max_rho")
            kw = dict(zip(names, rhs_fn.args))
            kw.update(rhs_fn.keywords)
            if "rho_values" in kw and "geom" in kw and set(kw) <= set(names):
                return FrozenPmaRhs(**kw)
    raise ConfigurationError(
        "the device integrators run the frozen-density PMA right-hand side only: pass "
        "frozen_rhs(rho, geom, ...) or functools.partial(pma_rhs_frozen, rho, geom, ...); "
        "an arbitrary Python rhs_fn cannot run on the GPU")


class DeviceIntegrator:
    """Stateful Rkc2Integrator / EulerIntegrator (integrate.py:63-250): one
    instance per subdomain, its sigma / step-size caches persist across
    ``advance`` calls (schwarz.py:133) in the device controller state."""

    def __init__(self, window: IntegrationWindow):
        self.window = window
        self._plan = None
        self._key = None

    def _plan_for(self, rhs: FrozenPmaRhs):
        from .pma import _geom_key
        from .plan import Plan
        from .schwarz import SolverConfig
        geom = rhs.geom
        if rhs.dirichlet_mask is not None and not np.array_equal(rhs.dirichlet_mask,
                                                                 geom.dirichlet_mask()):
            raise ConfigurationError("custom dirichlet masks are not supported on the device path")
        key = (_geom_key(geom), rhs.det_floor)
        if self._plan is None:
            w = self.window
            cfg = SolverConfig(dtau=w.dtau, scheme=w.scheme, substeps=w.substeps, rtol=w.rtol,
                               atol=w.atol, max_stages=w.max_stages, det_floor=rhs.det_floor)
            self._plan = Plan.for_geometry(geom, cfg)
            self._key = key
        elif key != self._key:
            raise ConfigurationError("an integrator instance advances one subdomain box "
                                     "(schwarz.py:133); make a new one for another geometry")
        return self._plan

    def advance(self, y: np.ndarray, rhs_fn) -> np.ndarray:
        rhs = _as_frozen(rhs_fn)
        y = np.asarray(y, dtype=np.float64)
        if y.shape != rhs.geom.shape():
            raise ValueError(f"field shape {y.shape} != box {rhs.geom.shape()}")
        plan = self._plan_for(rhs)
        try:
            return plan.integrate_window(0, y, rhs.rho_values, rhs.max_rho)
        except StiffnessError as err:
            err.subdomain = None   # the integrator does not know its subdomain (schwarz.py:209-211)
            raise

    def close(self):
        if self._plan is not None:
            self._plan.close()
            self._plan = None


def make_integrator(window: IntegrationWindow) -> DeviceIntegrator:
    """integrate.py:253-256 (both schemes run in the device controller)."""
    return DeviceIntegrator(window)


def advance_window(psi: np.ndarray, rhs_fn, window: IntegrationWindow) -> np.ndarray:
    """One-shot window advance, fresh integrator (integrate.py:259-262)."""
    integ = make_integrator(window)
    try:
        return integ.advance(psi, rhs_fn)
    finally:
        integ.close()
