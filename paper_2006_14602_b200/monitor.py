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


# ------------------------------------------- arc-length test functions --
# monitor.py:76-97 (TestFunction, arc_length_monitor) and :223-345 (the
# analytic test functions and their registry).  The numpy bodies are the
# reference formulas; the device restates them in stencil.cuh (tf_u/tf_grad).

_UNIT_SQUARE: Extents = ((0.0, 1.0), (0.0, 1.0))
_DOMAINS = {"burgers2d": _UNIT_SQUARE, "spiral2d": _UNIT_SQUARE,
            "sphere3d": ((-1.0, 1.0),) * 3, "nine_spheres3d": ((-2.0, 2.0),) * 3,
            "quasi1d_linear": _UNIT_SQUARE}
_KIND = {"burgers2d": 3, "spiral2d": 4, "sphere3d": 5, "nine_spheres3d": 6,
         "quasi1d_linear": 7}
_NINE_CENTERS = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.5], [0.5, -0.5, 0.5],
                          [-0.5, 0.5, 0.5], [-0.5, -0.5, 0.5], [0.5, 0.5, -0.5],
                          [0.5, -0.5, -0.5], [-0.5, 0.5, -0.5], [-0.5, -0.5, -0.5]])


def _tf_u(name: str, eps: float, p: np.ndarray) -> np.ndarray:
    if name == "burgers2d":
        a = (p[..., 0] + p[..., 1] - 1.0) / (2.0 * eps)
        return 0.5 * (1.0 - np.tanh(0.5 * a))
    if name == "spiral2d":
        dx, dy = p[..., 0] - 0.7, p[..., 1] - 0.5
        r2 = dx * dx + dy * dy
        g = np.arctan2(dy, dx) - 20.0 * r2
        return 1.0 + 9.0 / (1.0 + 100.0 * r2 * np.cos(g) ** 2)
    if name == "sphere3d":
        return np.tanh(100.0 * (np.sum(p * p, axis=-1) - 0.125))
    if name == "nine_spheres3d":
        out = np.zeros(p.shape[:-1])
        for c in _NINE_CENTERS:
            d = p - c
            out += np.tanh(50.0 * (np.sum(d * d, axis=-1) - 0.1875))
        return out
    w = p[..., 0] + 1.0
    s = np.sqrt(np.maximum(w * w - 1.0, 0.0))
    return 0.5 * (w * s - np.arccosh(np.maximum(w, 1.0)))


def _tf_grad(name: str, eps: float, p: np.ndarray) -> np.ndarray:
    if name == "burgers2d":
        a = (p[..., 0] + p[..., 1] - 1.0) / (2.0 * eps)
        uu = 0.5 * (1.0 - np.tanh(0.5 * a))
        d = -uu * (1.0 - uu) / (2.0 * eps)
        return np.stack([d, d], axis=-1)
    if name == "spiral2d":
        dx, dy = p[..., 0] - 0.7, p[..., 1] - 0.5
        r2 = dx * dx + dy * dy
        g = np.arctan2(dy, dx) - 20.0 * r2
        c2 = np.cos(g) ** 2
        s2g = np.sin(2.0 * g)
        den = 1.0 + 100.0 * r2 * c2
        ddx = 100.0 * (2.0 * dx * c2 + dy * s2g + 40.0 * dx * r2 * s2g)
        ddy = 100.0 * (2.0 * dy * c2 - dx * s2g + 40.0 * dy * r2 * s2g)
        scale = -9.0 / (den * den)
        return np.stack([np.where(r2 > 0.0, scale * ddx, 0.0),
                         np.where(r2 > 0.0, scale * ddy, 0.0)], axis=-1)
    if name == "sphere3d":
        t = np.tanh(100.0 * (np.sum(p * p, axis=-1) - 0.125))
        return (200.0 * (1.0 - t * t))[..., None] * p
    if name == "nine_spheres3d":
        out = np.zeros_like(p)
        for c in _NINE_CENTERS:
            d = p - c
            t = np.tanh(50.0 * (np.sum(d * d, axis=-1) - 0.1875))
            out += (100.0 * (1.0 - t * t))[..., None] * d
        return out
    x = p[..., 0]
    gx = np.sqrt(np.maximum(x * x + 2.0 * x, 0.0))
    return np.stack([gx, np.zeros_like(gx)], axis=-1)


@dataclass(frozen=True)
class _TfU:
    name: str
    eps: float

    def __call__(self, p):
        return _tf_u(self.name, self.eps, np.asarray(p, dtype=float))


@dataclass(frozen=True)
class _TfGrad:
    name: str
    eps: float

    def __call__(self, p):
        return _tf_grad(self.name, self.eps, np.asarray(p, dtype=float))


@dataclass(frozen=True)
class TestFunction:
    """Closed-form physical solution u with its analytic gradient (monitor.py:76-84)."""
    __test__ = False   # not a pytest class

    name: str
    domain: Extents
    u: Callable[[np.ndarray], np.ndarray]
    gradient: Callable[[np.ndarray], np.ndarray]
    params: dict = field(default_factory=dict)


@dataclass(frozen=True)
class ArcLengthDensity:
    """raw = sqrt(1 + |grad u|^2) of a registered test function
    (arc_length_monitor's raw, monitor.py:92-95); device kinds 3..7."""
    name: str
    eps: float = 0.01

    def __call__(self, p):
        g = _tf_grad(self.name, self.eps, np.asarray(p, dtype=float))
        return np.sqrt(1.0 + np.sum(g * g, axis=-1))


def test_function_registry(name: str, **params) -> TestFunction:
    """Named analytic test functions with gradients and domains (monitor.py:341-357)."""
    if name not in _KIND:
        raise ConfigurationError(
            f"unknown test function {name!r}; known: {sorted(_KIND)}")
    eps = 0.0
    extra = {}
    if name == "burgers2d":
        eps = float(params.pop("eps", 0.01))
        if eps <= 0.0:
            raise ConfigurationError(f"burgers2d needs eps > 0, got {eps}")
        if params:
            raise ConfigurationError(f"unknown parameters {sorted(params)}")
        extra = {"eps": eps}
    elif params:
        raise ConfigurationError(f"{name} takes no parameters, got {sorted(params)}")
    return TestFunction(name, _DOMAINS[name], _TfU(name, eps), _TfGrad(name, eps), extra)


test_function_registry.__test__ = False   # not a pytest function


# ------------------------------------------------------ sampled fields --

def _smooth(values: np.ndarray, passes: int) -> np.ndarray:
    """Per-axis [1, 2, 1]/4 averaging with reflected edges (monitor.py:395-409)."""
    out = values
    for _ in range(passes):
        for axis in range(out.ndim):
            n = out.shape[axis]
            left = np.take(out, [1] + list(range(0, n - 1)), axis=axis)
            right = np.take(out, list(range(1, n)) + [n - 2], axis=axis)
            out = 0.25 * left + 0.5 * out + 0.25 * right
    return out


class SampledField:
    """Scalar u sampled on a lattice over a physical box (monitor.py:361-392).

    Construction (smoothing, central-difference gradient lattices) is the
    reference's one-time numpy preprocessing; the solver's per-window
    interpolation of u and grad u at the mesh nodes runs on the device
    (``DDPMA_MON_SAMPLED``).  ``u`` / ``gradient`` here are the host-side
    API evaluations the reference class offers (scipy linear interpolation),
    never called by ``solve``."""

    def __init__(self, axes, values, smooth_passes: int = 0):
        self.axes = tuple(np.ascontiguousarray(ax, dtype=np.float64) for ax in axes)
        values = np.asarray(values, dtype=float)
        if values.shape != tuple(len(ax) for ax in self.axes):
            raise ConfigurationError("sample array shape does not match axes")
        if smooth_passes:
            values = _smooth(values, smooth_passes)
        self.values = np.ascontiguousarray(values)
        self.domain: Extents = tuple((float(ax[0]), float(ax[-1])) for ax in self.axes)
        spacing = [float(ax[1] - ax[0]) for ax in self.axes]
        self.grads = tuple(np.ascontiguousarray(np.gradient(self.values, h, axis=k, edge_order=2))
                           for k, h in enumerate(spacing))

    def _interp(self, field_values, points):
        from scipy.interpolate import RegularGridInterpolator
        points = np.asarray(points, dtype=float)
        it = RegularGridInterpolator(self.axes, field_values, method="linear")
        return it(points.reshape(-1, len(self.axes))).reshape(points.shape[:-1])

    def u(self, points):
        return self._interp(self.values, points)

    def gradient(self, points):
        return np.stack([self._interp(g, points) for g in self.grads], axis=-1)


@dataclass(frozen=True, eq=False)
class SampledArcLength:
    """raw = sqrt(1 + |grad u|^2) of a SampledField (device kind 8)."""
    field: SampledField

    def __call__(self, p):
        g = self.field.gradient(p)
        return np.sqrt(1.0 + np.sum(g * g, axis=-1))


def sampled_field_from_csv(path: str, smooth_passes: int = 0) -> SampledField:
    """``x,y[,z],u`` rows covering a full uniform lattice (monitor.py:412-437)."""
    rows = np.loadtxt(path, delimiter=",", comments="#", ndmin=2)
    if rows.shape[1] not in (3, 4):
        raise ConfigurationError(
            f"{path}: expected 3 or 4 columns (x,y[,z],u), got {rows.shape[1]}")
    dim = rows.shape[1] - 1
    coords, u = rows[:, :dim], rows[:, dim]
    axes = []
    for k in range(dim):
        ax = np.unique(coords[:, k])
        if len(ax) < 3:
            raise ConfigurationError(f"{path}: axis {k} has fewer than 3 levels")
        steps = np.diff(ax)
        if not np.allclose(steps, steps[0], rtol=1e-9, atol=1e-12):
            raise ConfigurationError(f"{path}: axis {k} is not uniformly spaced")
        axes.append(ax)
    shape = tuple(len(ax) for ax in axes)
    if rows.shape[0] != int(np.prod(shape)):
        raise ConfigurationError(f"{path}: {rows.shape[0]} rows do not fill a {shape} lattice")
    order = np.lexsort([coords[:, k] for k in reversed(range(dim))])
    return SampledField(tuple(axes), u[order].reshape(shape), smooth_passes=smooth_passes)


def sampled_field_from_vtk(path: str, smooth_passes: int = 0) -> SampledField:
    """Scalar field in the package's structured-grid VTK format (monitor.py:440-444)."""
    from . import fileio
    axes, values = fileio.read_scalar_field_vtk(path)
    return SampledField(axes, values, smooth_passes=smooth_passes)


def arc_length_monitor(source) -> MonitorField:
    """Unnormalised arc-length density of ``source`` (monitor.py:88-97): a
    registered analytic TestFunction or a SampledField; u-backed, so the
    solver's nodal density is the mesh pull-back of u (mesh_density)."""
    if isinstance(source, SampledField):
        return MonitorField(raw=SampledArcLength(source), domain=source.domain, u_fn=source.u)
    if not isinstance(source, TestFunction) or not isinstance(source.u, _TfU):
        raise ConfigurationError(
            "the device path supports arc-length monitors of the registered analytic "
            "test functions (test_function_registry) and of SampledField")
    return MonitorField(raw=ArcLengthDensity(source.u.name, source.u.eps),
                        domain=source.domain, u_fn=source.u)


@dataclass
class NativeMonitor:
    """A MonitorField lowered to the C descriptor (keeps buffers alive)."""
    desc: _lib.Monitor
    keep: list = field(default_factory=list)


def lower_monitor(mon: MonitorField, dim: int) -> NativeMonitor:
    """MonitorField -> ddpma_monitor, or ConfigurationError (no CPU fallback)."""
    if not isinstance(mon, MonitorField):
        raise ConfigurationError("monitor must be a MonitorField")
    if mon.u_fn is not None and not (
            (isinstance(mon.raw, ArcLengthDensity) and mon.u_fn == _TfU(mon.raw.name, mon.raw.eps))
            or (isinstance(mon.raw, SampledArcLength) and mon.u_fn == mon.raw.field.u)):
        raise ConfigurationError(
            "monitors backed by a physical scalar u are supported for the registered "
            "analytic test functions (arc_length_monitor); sampled fields are not")
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
    elif isinstance(raw, ArcLengthDensity):
        # u_fn set: the solver's density is the pull-back of u (mesh_density
        # monitor.py:170-180); absent (normalize() drops it, :147-148): the
        # analytic arc length at the clamped mesh points (:166-168)
        d.kind = _KIND[raw.name]
        d.eps = float(raw.eps)
        d.u_backed = 1 if mon.u_fn is not None else 0
        if len(_DOMAINS[raw.name]) != dim:
            raise ConfigurationError("grid dimension does not match monitor domain")
    elif isinstance(raw, SampledArcLength):
        fld = raw.field
        if len(fld.axes) != dim:
            raise ConfigurationError("grid dimension does not match monitor domain")
        d.kind = _lib.MON_SAMPLED
        d.u_backed = 1 if mon.u_fn is not None else 0
        for k, ax in enumerate(fld.axes):
            d.lat[k] = len(ax)
            d.axes[k] = _lib.dptr(ax)
            d.grads[k] = _lib.dptr(fld.grads[k])
        d.values = _lib.dptr(fld.values)
        keep = [fld]
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


def _device_mass(mon: MonitorField, counts: tuple[int, ...]) -> tuple[float, float]:
    """_trapezoid_mass (monitor.py:112-120) on the device."""
    nm = lower_monitor(MonitorField(raw=mon.raw, domain=mon.domain), mon.dim)
    cnt = (C.c_int * 3)(*(list(counts) + [1] * (3 - len(counts))))
    z, peak, bad = C.c_double(), C.c_double(), C.c_int()
    import torch
    st = _lib.lib().ddpma_monitor_mass(C.byref(nm.desc), cnt, int(torch.cuda.current_device()),
                                       C.byref(z), C.byref(peak), C.byref(bad))
    _lib.check_global(st)
    if bad.value:
        from .errors import InvalidMonitorError
        raise InvalidMonitorError("density is nonpositive or non-finite on Omega")
    return z.value, peak.value


def normalize(fld: MonitorField, grid, z_rtol: float = 1e-5) -> MonitorField:
    """Normalise by converged composite-trapezoid quadrature on refined probe
    grids (monitor.py:123-148); the probe sums run on the device.  Like the
    reference, the result carries no ``u_fn``."""
    from .errors import InvalidMonitorError
    if len(grid.counts) != fld.dim:
        raise ConfigurationError("grid dimension does not match monitor domain")
    _lib.require_cuda()
    cap = 4097 if fld.dim == 2 else 257
    counts = tuple(grid.counts)
    z, peak = _device_mass(fld, counts)
    while max(counts) < cap:
        counts = tuple(min(cap, 2 * n - 1) for n in counts)
        z_new, peak = _device_mass(fld, counts)
        done = abs(z_new - z) <= z_rtol * abs(z_new)
        z = z_new
        if done:
            break
    if not np.isfinite(z) or z <= 0.0:
        raise InvalidMonitorError(f"quadrature of the density is {z}")
    return MonitorField(raw=fld.raw, domain=fld.domain, normalizer=z, max_value=peak / z)
