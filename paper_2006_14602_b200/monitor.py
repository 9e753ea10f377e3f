"""Mesh-density monitors (ddmesh/monitor.py:31-104) with device-evaluable
native densities.

A GPU path cannot call an arbitrary Python ``raw`` callable per node, so the
solver accepts monitors whose ``raw`` is one of the native density objects
below.  They are still ordinary numpy callables — a
``MonitorField`` built from them works with the reference package and the CPU
oracle unchanged — and they carry their parameters to the CUDA kernels.  Any
other ``raw`` makes the solver raise :class:`ConfigurationError`; there is no
CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from .errors import ConfigurationError

Extents = tuple[tuple[float, float], ...]


@dataclass(frozen=True)
class MonitorField:
    """Positive density on a physical box (monitor.py:31-74)."""

    raw: Callable[[np.ndarray], np.ndarray]
    domain: Extents
    normalizer: float = 1.0
    max_value: float | None = None
    u_fn: Callable[[np.ndarray], np.ndarray] | None = None

    @property
    def dim(self) -> int:
        return len(self.domain)

    def __call__(self, points: np.ndarray) -> np.ndarray:
        from .errors import DomainError
        points = np.asarray(points, dtype=float)
        for k, (a, b) in enumerate(self.domain):
            pk = points[..., k]
            slack = 1e-12 * (b - a)
            if (pk < a - slack).any() or (pk > b + slack).any():
                raise DomainError(
                    f"monitor evaluated outside axis-{k} extent [{a}, {b}]")
        return self.raw(points) / self.normalizer

    def eval_clamped(self, points: np.ndarray) -> np.ndarray:
        return self.raw(self.clamp(points)) / self.normalizer

    def clamp(self, points: np.ndarray) -> np.ndarray:
        points = np.asarray(points, dtype=float)
        lo = np.array([a for a, _ in self.domain])
        hi = np.array([b for _, b in self.domain])
        return np.clip(points, lo, hi)


def density_monitor(fn: Callable[[np.ndarray], np.ndarray], domain: Extents) -> MonitorField:
    """Unnormalized monitor from an explicit density callback (monitor.py:100-104)."""
    return MonitorField(raw=fn, domain=tuple((float(a), float(b)) for a, b in domain))


# ------------------------------------------------------- native densities --
# The numpy bodies fix the evaluation order the CUDA kernel (kernels.cu
# mon_raw) restates, so both sides round identically up to exp().

@dataclass(frozen=True)
class UniformDensity:
    """raw = constant (the uniform-monitor exactness case)."""
    constant: float = 1.0

    def __call__(self, p):
        return np.full(np.shape(p)[:-1], float(self.constant))


@dataclass(frozen=True)
class RingDensity:
    """raw = 1 + amp * exp(-sharp * |sum_k (x_k - c_k)^2 - r2|).

    2D: the BASELINE ring monitor (config 1); 3D: the spherical shell
    (config 4) with r measured from ``center``."""
    center: tuple = (0.5, 0.5)
    amp: float = 10.0
    sharp: float = 50.0
    r2: float = 0.0625

    def __call__(self, p):
        acc = (p[..., 0] - self.center[0]) ** 2
        for k in range(1, p.shape[-1]):
            acc = acc + (p[..., k] - self.center[k]) ** 2
        return 1.0 + self.amp * np.exp(-self.sharp * np.abs(acc - self.r2))


def ShellDensity(center=(0.5, 0.5, 0.5), amp=10.0, sharp=50.0, r2=0.0625):
    """Spherical-shell monitor of BASELINE config 4."""
    return RingDensity(tuple(center), amp, sharp, r2)


@dataclass(frozen=True)
class MixtureDensity:
    """raw = 1 + sum_k a_k exp(-|x - c_k|^2 / (2 s_k^2))  (configs 2, 3, 5)."""
    c: tuple
    s: tuple
    a: tuple

    def __call__(self, p):
        tot = 0.0
        for ck, sk, ak in zip(self.c, self.s, self.a):
            d2 = (p[..., 0] - ck[0]) ** 2
            for k in range(1, p.shape[-1]):
                d2 = d2 + (p[..., k] - ck[k]) ** 2
            tot = tot + ak * np.exp(-d2 / (2.0 * sk * sk))
        return 1.0 + tot


def seeded_mixture(nbumps: int, dim: int, seed: int = 0) -> MixtureDensity:
    """BASELINE Gaussian mixture: ``default_rng(seed)``, draws in the order
    c ~ U[0.1,0.9]^d, s ~ U[0.02,0.08], a ~ U[2,20] (recorded in DESIGN.md)."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.1, 0.9, (nbumps, dim))
    s = rng.uniform(0.02, 0.08, nbumps)
    a = rng.uniform(2.0, 20.0, nbumps)
    return MixtureDensity(tuple(tuple(float(x) for x in row) for row in c),
                          tuple(float(x) for x in s), tuple(float(x) for x in a))


@dataclass
class NativeMonitor:
    """A MonitorField lowered to the C descriptor (keeps buffers alive)."""
    desc: _lib.Monitor
    keep: list = field(default_factory=list)


def lower_monitor(mon: MonitorField, dim: int) -> NativeMonitor:
    """MonitorField -> ddpma_monitor, or ConfigurationError (no CPU fallback)."""
    if not isinstance(mon, MonitorField):
        raise ConfigurationError("monitor must be a MonitorField")
    if mon.u_fn is not None:
        raise ConfigurationError(
            "monitors backed by a physical scalar u (arc-length / sampled fields) "
            "are not supported on the device path yet")
    if mon.dim != dim:
        raise ConfigurationError("grid dimension does not match monitor domain")
    d = _lib.Monitor()
    d.dim = dim
    for k, (a, b) in enumerate(mon.domain):
        d.domain[k][0], d.domain[k][1] = float(a), float(b)
    keep = []
    raw = mon.raw
    if isinstance(raw, UniformDensity):
        d.kind = _lib.MON_UNIFORM
        d.constant = float(raw.constant)
    elif isinstance(raw, RingDensity):
        if len(raw.center) != dim:
            raise ConfigurationError("ring/shell centre does not match the dimension")
        d.kind = _lib.MON_RING
        for k in range(dim):
            d.center[k] = float(raw.center[k])
        d.amp, d.sharp, d.r2 = float(raw.amp), float(raw.sharp), float(raw.r2)
    elif isinstance(raw, MixtureDensity):
        c = np.ascontiguousarray(np.array(raw.c, dtype=np.float64).reshape(-1, dim))
        s = np.ascontiguousarray(np.array(raw.s, dtype=np.float64))
        a = np.ascontiguousarray(np.array(raw.a, dtype=np.float64))
        if not (len(c) == len(s) == len(a)):
            raise ConfigurationError("mixture parameter lengths differ")
        if len(s) > 64:
            raise ConfigurationError("mixture monitor supports at most 64 bumps")
        d.kind = _lib.MON_MIXTURE
        d.nbumps = len(s)
        d.c, d.s, d.a = _lib.dptr(c), _lib.dptr(s), _lib.dptr(a)
        keep = [c, s, a]
    else:
        raise ConfigurationError(
            "the device solver needs a native density (UniformDensity, RingDensity, "
            "ShellDensity, MixtureDensity); arbitrary Python callables cannot run "
            "on the GPU and there is no CPU fallback")
    return NativeMonitor(d, keep)
