"""Integration-window description and RKC2 coefficients
(ddmesh/integrate.py:41-106).

The integrators themselves (Rkc2Integrator.advance, EulerIntegrator) run in
the native controller + CUDA kernels (csrc/plan.cu, csrc/kernels.cu); they
cannot accept an arbitrary Python ``rhs_fn`` because the right-hand side is
the fused device kernel.  ``rkc_coeffs`` exposes the host-side coefficient
table the controller uses, for parity checks.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigurationError


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
