"""CPU oracle for the DDPMA hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package's explicit PMA
stepping path (``ddmesh`` = /root/reference/pkg/src/ddmesh).  It exists so the
CUDA product path can be checked against something on the GPU box, where the
reference itself is absent.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / ``--impl reference`` legs may import it; the
product package never does (and must fail loudly without its CUDA library).

Parity pin: ``tests/golden/make_golden.py`` runs the real reference in the
build container and stores its outputs as fixtures; ``tests/test_oracle.py``
asserts this restatement reproduces them BITWISE (same numpy operations in the
same order).  Each function cites the reference line it restates.

Notation: a "box" is one subdomain's index box; arrays are C-order fp64 with
the last axis fastest, exactly as in the reference.
"""

from __future__ import annotations

import itertools
import math
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

PHYSICAL = "physical"      # ddmesh/grid.py:20
INTERFACE = "interface"    # ddmesh/grid.py:21
DET_FLOOR = 1e-12          # ddmesh/pma.py:23

# ddmesh/integrate.py:35-38
DAMPING = 2.0 / 13.0
STAB_PER_S2 = 0.653
MIN_STEP_FRACTION = 1e-14
SIGMA_REFRESH = 25


class OracleError(Exception):
    pass


class OracleConfigError(OracleError):
    pass


class OracleStiffness(OracleError):
    def __init__(self, msg, nodes=None, subdomain=None):
        super().__init__(msg)
        self.nodes = nodes
        self.subdomain = subdomain


class OracleInvalidMonitor(OracleError):
    pass


# ---------------------------------------------------------------- grid ----

@dataclass(frozen=True)
class Grid:
    """ddmesh/grid.py:24-55 (CompGrid)."""
    dim: int
    extents: tuple
    counts: tuple

    @property
    def spacing(self):
        return tuple((b - a) / (n - 1) for (a, b), n in zip(self.extents, self.counts))

    @property
    def measure(self):
        m = 1.0
        for a, b in self.extents:
            m *= b - a
        return m

    def axes(self):
        return tuple(a + np.arange(n) * h
                     for (a, _), n, h in zip(self.extents, self.counts, self.spacing))


def make_grid(dim, extents, counts):
    """ddmesh/grid.py:58-75."""
    if dim not in (2, 3):
        raise OracleConfigError("dim")
    extents = tuple((float(a), float(b)) for a, b in extents)
    counts = tuple(int(n) for n in counts)
    if len(extents) != dim or len(counts) != dim:
        raise OracleConfigError("arity")
    for a, b in extents:
        if not (math.isfinite(a) and math.isfinite(b)) or b <= a:
            raise OracleConfigError("extent")
    if any(n < 3 for n in counts):
        raise OracleConfigError("count")
    return Grid(dim, extents, counts)


@dataclass(frozen=True)
class Sub:
    """ddmesh/grid.py:78-110 (Subdomain)."""
    id: int
    pos: tuple
    box: tuple
    faces: tuple
    neighbors: dict
    owned: tuple

    def shape(self):
        return tuple(hi - lo + 1 for lo, hi in self.box)

    def gslices(self):
        return tuple(slice(lo, hi + 1) for lo, hi in self.box)

    def owned_g(self):
        return tuple(slice(lo, hi + 1) for lo, hi in self.owned)

    def owned_l(self):
        return tuple(slice(o0 - b0, o1 - b0 + 1)
                     for (o0, o1), (b0, _) in zip(self.owned, self.box))


@dataclass(frozen=True)
class Decomp:
    grid: Grid
    layout: tuple
    overlap: int
    subs: tuple


def axis_segments(n, parts):
    """ddmesh/grid.py:125-135: remainder to the low segments."""
    q, r = divmod(n, parts)
    segs, start = [], 0
    for p in range(parts):
        ln = q + (1 if p < r else 0)
        segs.append((start, start + ln - 1))
        start += ln
    return segs


def axis_boxes(segs, overlap, n, axis):
    """ddmesh/grid.py:138-173: extend and cut at the overlap midline."""
    up = overlap // 2
    down = overlap - up
    last = len(segs) - 1
    boxes = [((s - down) if p else s, (e + up) if p < last else e)
             for p, (s, e) in enumerate(segs)]
    cuts = [(boxes[p + 1][0] + boxes[p][1]) // 2 for p in range(last)]
    for p in range(last):
        if not (boxes[p][0] < boxes[p + 1][0] < boxes[p][1] < boxes[p + 1][1]):
            raise OracleConfigError(f"overlap too large axis {axis}")
    for p in range(len(boxes) - 2):
        if boxes[p + 2][0] <= boxes[p][1]:
            raise OracleConfigError(f"non-adjacent touch axis {axis}")
    if any(hi - lo + 1 < 3 for lo, hi in boxes):
        raise OracleConfigError(f"thin box axis {axis}")
    return boxes, cuts


def make_decomposition(grid, layout, overlap=3):
    """ddmesh/grid.py:176-237 (+ the per-axis form of _check_decomposition :240-258)."""
    layout = tuple(int(m) for m in layout)
    if len(layout) != grid.dim or any(m < 1 for m in layout):
        raise OracleConfigError("layout")
    if any(m > 1 for m in layout) and overlap < 2:
        raise OracleConfigError("overlap")
    per_axis = []
    for k, m in enumerate(layout):
        n = grid.counts[k]
        if m == 1:
            boxes, cuts = [(0, n - 1)], []
        else:
            boxes, cuts = axis_boxes(axis_segments(n, m), overlap, n, k)
        bounds = [-1] + cuts + [n - 1]
        owned = [(bounds[p] + 1, bounds[p + 1]) for p in range(m)]
        per_axis.append((boxes, owned))
    positions = list(itertools.product(*[range(m) for m in layout]))
    index = {p: i for i, p in enumerate(positions)}
    subs = []
    for i, pos in enumerate(positions):
        faces, nbrs = [], {}
        for k in range(grid.dim):
            lo_i = pos[k] > 0
            hi_i = pos[k] < layout[k] - 1
            faces.append((INTERFACE if lo_i else PHYSICAL, INTERFACE if hi_i else PHYSICAL))
            if lo_i:
                nbrs[(k, 0)] = index[pos[:k] + (pos[k] - 1,) + pos[k + 1:]]
            if hi_i:
                nbrs[(k, 1)] = index[pos[:k] + (pos[k] + 1,) + pos[k + 1:]]
        subs.append(Sub(i, pos,
                        tuple(per_axis[k][0][pos[k]] for k in range(grid.dim)),
                        tuple(faces), nbrs,
                        tuple(per_axis[k][1][pos[k]] for k in range(grid.dim))))
    for s in subs:
        for (ax, side), d in s.neighbors.items():
            line = s.box[ax][side]
            lo, hi = subs[d].box[ax]
            if not lo < line < hi:
                raise OracleConfigError("trace line not interior")
    return Decomp(grid, layout, overlap, tuple(subs))


@dataclass(frozen=True)
class Geom:
    """ddmesh/grid.py:261-307 (BoxGeometry / subdomain_geometry)."""
    axes: tuple
    spacing: tuple
    faces: tuple
    measure: float

    def shape(self):
        return tuple(len(a) for a in self.axes)

    def mask(self):
        m = np.zeros(self.shape(), dtype=bool)
        for k, (lo, hi) in enumerate(self.faces):
            if lo == INTERFACE:
                m[_at(len(self.axes), k, 0)] = True
            if hi == INTERFACE:
                m[_at(len(self.axes), k, -1)] = True
        return m


def whole_geom(grid):
    return Geom(grid.axes(), grid.spacing,
                tuple((PHYSICAL, PHYSICAL) for _ in range(grid.dim)), grid.measure)


def box_geom(grid, sub):
    ax = tuple(a[lo:hi + 1] for a, (lo, hi) in zip(grid.axes(), sub.box))
    return Geom(ax, grid.spacing, sub.faces, grid.measure)


def _at(nd, axis, idx):
    s = [slice(None)] * nd
    s[axis] = idx
    return tuple(s)


# --------------------------------------------------------- quadrature ----

def trap_weights(counts, spacing):
    """ddmesh/quadrature.py:8-23 (tensor trapezoid weights)."""
    def w1(n, h):
        w = np.full(n, h)
        w[0] = 0.5 * h
        w[-1] = 0.5 * h
        return w
    w = w1(counts[0], spacing[0])
    for n, h in zip(counts[1:], spacing[1:]):
        w = np.multiply.outer(w, w1(n, h))
    return w


def l2_norm(v, spacing):
    """ddmesh/quadrature.py:29-31."""
    return float(np.sqrt(np.sum(v * v * trap_weights(v.shape, spacing))))


# ----------------------------------------------------------- operator ----

def psi0(geom):
    """ddmesh/pma.py:61-64: 0.5 * sum_k xi_k^2."""
    sq = np.meshgrid(*[a * a for a in geom.axes], indexing="ij")
    return 0.5 * np.sum(sq, axis=0)


def coords_fd(psi, geom):
    """ddmesh/pma.py:67-84: np.gradient(edge_order=2); exact face coordinate
    on the normal component at physical faces."""
    nd = psi.ndim
    out = []
    for k in range(nd):
        g = np.gradient(psi, geom.spacing[k], axis=k, edge_order=2)
        lo, hi = geom.faces[k]
        if lo == PHYSICAL:
            g[_at(nd, k, 0)] = geom.axes[k][0]
        if hi == PHYSICAL:
            g[_at(nd, k, -1)] = geom.axes[k][-1]
        out.append(g)
    return out


def d2_axis(psi, k, geom):
    """ddmesh/pma.py:87-115: second difference, Neumann reflection on
    physical faces, 4-point one-sided formula on interface faces."""
    nd = psi.ndim
    h = geom.spacing[k]
    n = psi.shape[k]
    hh = h * h
    out = np.empty_like(psi)
    out[_at(nd, k, slice(1, -1))] = (psi[_at(nd, k, slice(2, None))]
                                     - 2.0 * psi[_at(nd, k, slice(1, -1))]
                                     + psi[_at(nd, k, slice(None, -2))]) / hh
    lo, hi = geom.faces[k]
    p0, p1 = psi[_at(nd, k, 0)], psi[_at(nd, k, 1)]
    q0, q1 = psi[_at(nd, k, -1)], psi[_at(nd, k, -2)]
    if lo == PHYSICAL:
        out[_at(nd, k, 0)] = 2.0 * (p1 - p0 - h * geom.axes[k][0]) / hh
    elif n >= 4:
        out[_at(nd, k, 0)] = (2.0 * p0 - 5.0 * p1 + 4.0 * psi[_at(nd, k, 2)]
                              - psi[_at(nd, k, 3)]) / hh
    else:
        out[_at(nd, k, 0)] = out[_at(nd, k, 1)]
    if hi == PHYSICAL:
        out[_at(nd, k, -1)] = 2.0 * (q1 - q0 + h * geom.axes[k][-1]) / hh
    elif n >= 4:
        out[_at(nd, k, -1)] = (2.0 * q0 - 5.0 * q1 + 4.0 * psi[_at(nd, k, -3)]
                               - psi[_at(nd, k, -4)]) / hh
    else:
        out[_at(nd, k, -1)] = out[_at(nd, k, -2)]
    return out


def dkl(psi, k, l, geom):
    """ddmesh/pma.py:118-130: nested np.gradient, zero on physical faces."""
    nd = psi.ndim
    g = np.gradient(np.gradient(psi, geom.spacing[l], axis=l, edge_order=2),
                    geom.spacing[k], axis=k, edge_order=2)
    for a in (k, l):
        lo, hi = geom.faces[a]
        if lo == PHYSICAL:
            g[_at(nd, a, 0)] = 0.0
        if hi == PHYSICAL:
            g[_at(nd, a, -1)] = 0.0
    return g


def hess_det(psi, geom):
    """ddmesh/pma.py:133-149."""
    if psi.ndim == 2:
        a, b, c = d2_axis(psi, 0, geom), d2_axis(psi, 1, geom), dkl(psi, 0, 1, geom)
        return a * b - c * c
    a, b, c = d2_axis(psi, 0, geom), d2_axis(psi, 1, geom), d2_axis(psi, 2, geom)
    x01, x02, x12 = dkl(psi, 0, 1, geom), dkl(psi, 0, 2, geom), dkl(psi, 1, 2, geom)
    return (a * (b * c - x12 * x12)
            - x01 * (x01 * c - x12 * x02)
            + x02 * (x01 * x12 - b * x02))


def log_equi(rho, det, measure, floor, rho_max):
    """ddmesh/pma.py:186-192: C1 rational saturation below the guard."""
    guard = floor
    if rho_max:
        guard = max(floor, 0.1 / (measure * rho_max))
    eff = np.where(det >= guard, det, guard / (2.0 - det / guard))
    return np.log(measure * rho * np.maximum(eff, floor))


def rhs_frozen(psi, rho, geom, floor=DET_FLOOR, mask=None, rho_max=None):
    """ddmesh/pma.py:195-219 -> (F, positivity flag)."""
    det = hess_det(psi, geom)
    if mask is None:
        mask = geom.mask()
    bad = det <= floor
    anymask = mask.any()
    if anymask:
        bad &= ~mask
    f = log_equi(rho, det, geom.measure, floor, rho_max)
    if anymask:
        f[mask] = 0.0
    return f, bool(bad.any())


def mesh_of(psi, geom):
    """ddmesh/pma.py:222-225 -> (coords[..., dim], jac)."""
    return np.stack(coords_fd(psi, geom), axis=-1), hess_det(psi, geom)


# --------------------------------------------------------- integrator ----

_COEFF_CACHE: dict = {}


def rkc_coeffs(s):
    """ddmesh/integrate.py:77-106 (damped RKC2 Chebyshev recurrences)."""
    if s in _COEFF_CACHE:
        return _COEFF_CACHE[s]
    w0 = 1.0 + DAMPING / (s * s)
    T = np.empty(s + 1)
    T1 = np.empty(s + 1)
    T2 = np.empty(s + 1)
    T[0], T[1] = 1.0, w0
    T1[0], T1[1] = 0.0, 1.0
    T2[0], T2[1] = 0.0, 0.0
    for j in range(2, s + 1):
        T[j] = 2.0 * w0 * T[j - 1] - T[j - 2]
        T1[j] = 2.0 * w0 * T1[j - 1] - T1[j - 2] + 2.0 * T[j - 1]
        T2[j] = 2.0 * w0 * T2[j - 1] - T2[j - 2] + 4.0 * T1[j - 1]
    w1 = T1[s] / T2[s]
    b = np.empty(s + 1)
    b[2:] = T2[2:] / T1[2:] ** 2
    b[0] = b[1] = b[2]
    a = 1.0 - b * T
    mu1t = b[1] * w1
    mu, nu, mut, gt = (np.zeros(s + 1) for _ in range(4))
    for j in range(2, s + 1):
        mu[j] = 2.0 * b[j] * w0 / b[j - 1]
        nu[j] = -b[j] / b[j - 2]
        mut[j] = mu[j] * w1 / w0
        gt[j] = -a[j - 1] * mut[j]
    out = (w0, w1, mu1t, mu, nu, mut, gt)
    _COEFF_CACHE[s] = out
    return out


def stage_count(hs):
    """ddmesh/integrate.py:157-161."""
    if hs <= 0.0:
        return 2
    return max(2, int(np.ceil(np.sqrt(1.05 * hs / STAB_PER_S2))))


@dataclass
class Counter:
    """Node-update counter: box nodes per RHS evaluation."""
    rhs_calls: int = 0
    node_updates: int = 0


class Rkc2:
    """ddmesh/integrate.py:109-250: adaptive RKC2, caches persist across
    windows.  ``trace`` (optional list) receives one tuple per step attempt:
    (h, s, emax, flagged, accepted) and ('sigma', value) per estimate."""

    def __init__(self, dtau, rtol=1e-3, atol=1e-6, max_stages=512, trace=None):
        self.dtau, self.rtol, self.atol, self.max_stages = dtau, rtol, atol, max_stages
        self.sigma = None
        self.since = 0
        self.interval = SIGMA_REFRESH
        self.h_last = None
        self.trace = trace

    def _sigma(self, y, f0, fn):
        """ddmesh/integrate.py:127-153 (checkerboard-seeded power iteration)."""
        v = np.where(np.indices(y.shape).sum(axis=0) % 2 == 0, 1.0, -1.0)
        delta = np.sqrt(np.finfo(float).eps) * (1.0 + float(np.linalg.norm(y.ravel())))
        sig = 0.0
        for _ in range(20):
            vn = float(np.linalg.norm(v.ravel()))
            if vn == 0.0:
                break
            fv, _ = fn(y + (delta / vn) * v)
            diff = fv - f0
            new = float(np.linalg.norm(diff.ravel())) / delta
            v = diff
            if sig > 0.0 and abs(new - sig) <= 0.01 * new:
                sig = new
                break
            sig = new
        self.since = 0
        if self.sigma is not None and sig <= 1.05 * self.sigma / 1.2:
            self.interval = min(500, 2 * self.interval)
        else:
            self.interval = SIGMA_REFRESH
        if self.trace is not None:
            self.trace.append(("sigma", 1.2 * sig))
        return 1.2 * sig

    def _step(self, y, f0, h, s, fn):
        """ddmesh/integrate.py:163-178."""
        _, _, mu1t, mu, nu, mut, gt = rkc_coeffs(s)
        flagged = False
        dm2 = np.zeros_like(y)
        dm1 = (h * mu1t) * f0
        for j in range(2, s + 1):
            fj, fl = fn(y + dm1)
            flagged |= fl
            dn = mu[j] * dm1 + nu[j] * dm2 + (h * mut[j]) * fj + (h * gt[j]) * f0
            dm2, dm1 = dm1, dn
        fnew, endf = fn(y + dm1)
        return dm1, fnew, flagged | endf, endf

    def advance(self, y, fn):
        """ddmesh/integrate.py:180-250 (statement for statement)."""
        total = self.dtau
        t = 0.0
        f0, start_flag = fn(y)
        if self.sigma is None or self.since >= self.interval:
            self.sigma = self._sigma(y, f0, fn)
        sigma = self.sigma
        if sigma <= 0.0:
            h = total
        else:
            h = min(total, max(10.0 * MIN_STEP_FRACTION * total, 0.25 / sigma))
        if self.h_last is not None:
            h = min(total, self.h_last)
        state_flag = start_flag
        rej_row = 0
        flag_rej = 0
        while t < total * (1.0 - 1e-13):
            h = min(h, total - t)
            cap = STAB_PER_S2 * self.max_stages ** 2
            if sigma > 0.0 and h * sigma > cap:
                h = cap / sigma
            s = min(self.max_stages, stage_count(h * sigma))
            d, fnew, flagged, endf = self._step(y, f0, h, s, fn)
            ynew = y + d
            err = -0.8 * d + (0.4 * h) * (f0 + fnew)
            scale = self.atol + self.rtol * np.maximum(np.abs(y), np.abs(ynew))
            ratio = np.abs(err) / scale
            emax = float(ratio.max())
            flag_fail = flagged and not state_flag and flag_rej < 8
            bad = flag_fail or not np.isfinite(emax)
            ok = (not bad) and emax <= 1.0
            if self.trace is not None:
                self.trace.append((h, s, emax, bool(flagged), ok))
            if ok:
                t += h
                y = ynew
                f0 = fnew
                state_flag = endf
                self.since += 1
                rej_row = 0
                if self.since >= self.interval and t < total:
                    self.sigma = sigma = self._sigma(y, f0, fn)
                grow = 5.0 if emax == 0.0 else min(5.0, 0.8 * emax ** (-1.0 / 3.0))
                h = h * max(0.1, grow)
                self.h_last = h
            else:
                if flag_fail:
                    flag_rej += 1
                    h *= 0.5
                elif not np.isfinite(emax):
                    h *= 0.5
                    rej_row += 1
                else:
                    h *= max(0.1, 0.8 * emax ** (-1.0 / 3.0))
                    rej_row += 1
                if rej_row >= 2:
                    self.sigma = sigma = self._sigma(y, f0, fn)
                    rej_row = 0
                if h < MIN_STEP_FRACTION * total or flag_rej + rej_row > 60:
                    nodes = np.argwhere(ratio > 1.0) if np.isfinite(emax) else None
                    raise OracleStiffness(f"underflow at {t:.3e} h={h:.3e}", nodes=nodes)
        return y


class Euler:
    """ddmesh/integrate.py:63-74."""

    def __init__(self, dtau, substeps=1):
        self.dtau, self.m = dtau, substeps

    def advance(self, y, fn):
        h = self.dtau / self.m
        for _ in range(self.m):
            f, _ = fn(y)
            y = y + h * f
        return y


def make_stepper(cfg, trace=None):
    if cfg.scheme == "euler":
        return Euler(cfg.dtau, cfg.substeps)
    return Rkc2(cfg.dtau, cfg.rtol, cfg.atol, cfg.max_stages, trace)


# ----------------------------------------------------------- monitors ----

@dataclass(frozen=True)
class Ring:
    """BASELINE C1: 1 + amp*exp(-sharp*|(x-cx)^2 + (y-cy)^2 - r2|)."""
    center: tuple = (0.5, 0.5)
    amp: float = 10.0
    sharp: float = 50.0
    r2: float = 0.0625

    def __call__(self, p):
        acc = (p[..., 0] - self.center[0]) ** 2
        for k in range(1, p.shape[-1]):
            acc = acc + (p[..., k] - self.center[k]) ** 2
        return 1.0 + self.amp * np.exp(-self.sharp * np.abs(acc - self.r2))


def Shell(center=(0.5, 0.5, 0.5), amp=10.0, sharp=50.0, r2=0.0625):
    """BASELINE C4: the ring formula with r measured from the cube centre."""
    return Ring(tuple(center), amp, sharp, r2)


@dataclass(frozen=True)
class Mixture:
    """BASELINE C2/C3/C5: 1 + sum_k a_k exp(-|x-c_k|^2 / (2 s_k^2))."""
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


def seeded_mixture(nbumps, dim, seed=0):
    """Seeded Gaussian-mixture parameters: default_rng(seed), order c, s, a."""
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.1, 0.9, (nbumps, dim))
    s = rng.uniform(0.02, 0.08, nbumps)
    a = rng.uniform(2.0, 20.0, nbumps)
    return Mixture(tuple(tuple(float(x) for x in row) for row in c),
                   tuple(float(x) for x in s), tuple(float(x) for x in a))


# Arc-length monitors of the analytic test functions (ddmesh/monitor.py:
# 88-97 arc_length_monitor, 223-345 the registry).  ``__call__`` is the
# analytic raw sqrt(1 + |grad u|^2); ``u`` marks the monitor as u-backed, so
# the solver's nodal density is the mesh pull-back (mesh_density below).

_NINE = np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.5], [0.5, -0.5, 0.5],
                  [-0.5, 0.5, 0.5], [-0.5, -0.5, 0.5], [0.5, 0.5, -0.5],
                  [0.5, -0.5, -0.5], [-0.5, 0.5, -0.5], [-0.5, -0.5, -0.5]])


@dataclass(frozen=True)
class ArcLength:
    """name in {burgers2d, spiral2d, sphere3d, nine_spheres3d, quasi1d_linear}."""
    name: str
    eps: float = 0.01

    @property
    def domain(self):
        if self.name == "sphere3d":
            return ((-1.0, 1.0),) * 3
        if self.name == "nine_spheres3d":
            return ((-2.0, 2.0),) * 3
        return ((0.0, 1.0), (0.0, 1.0))

    def u(self, p):
        n = self.name
        if n == "burgers2d":                                  # monitor.py:240-243
            a = (p[..., 0] + p[..., 1] - 1.0) / (2.0 * self.eps)
            return 0.5 * (1.0 - np.tanh(0.5 * a))
        if n == "spiral2d":                                   # :255-264
            dx, dy = p[..., 0] - 0.7, p[..., 1] - 0.5
            r2 = dx * dx + dy * dy
            g = np.arctan2(dy, dx) - 20.0 * r2
            return 1.0 + 9.0 / (1.0 + 100.0 * r2 * np.cos(g) ** 2)
        if n == "sphere3d":                                   # :282-284
            return np.tanh(100.0 * (np.sum(p * p, axis=-1) - 0.125))
        if n == "nine_spheres3d":                             # :308-313
            out = np.zeros(p.shape[:-1])
            for c in _NINE:
                d = p - c
                out += np.tanh(50.0 * (np.sum(d * d, axis=-1) - 0.1875))
            return out
        x = p[..., 0]                                         # :329-333
        w = x + 1.0
        s = np.sqrt(np.maximum(w * w - 1.0, 0.0))
        return 0.5 * (w * s - np.arccosh(np.maximum(w, 1.0)))

    def gradient(self, p):
        n = self.name
        if n == "burgers2d":                                  # :245-249
            a = (p[..., 0] + p[..., 1] - 1.0) / (2.0 * self.eps)
            uu = 0.5 * (1.0 - np.tanh(0.5 * a))
            d = -uu * (1.0 - uu) / (2.0 * self.eps)
            return np.stack([d, d], axis=-1)
        if n == "spiral2d":                                   # :266-276
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
        if n == "sphere3d":                                   # :286-289
            t = np.tanh(100.0 * (np.sum(p * p, axis=-1) - 0.125))
            return (200.0 * (1.0 - t * t))[..., None] * p
        if n == "nine_spheres3d":                             # :315-321
            out = np.zeros_like(p)
            for c in _NINE:
                d = p - c
                t = np.tanh(50.0 * (np.sum(d * d, axis=-1) - 0.1875))
                out += (100.0 * (1.0 - t * t))[..., None] * d
            return out
        x = p[..., 0]                                         # :335-338
        gx = np.sqrt(np.maximum(x * x + 2.0 * x, 0.0))
        return np.stack([gx, np.zeros_like(gx)], axis=-1)

    def __call__(self, p):                                    # monitor.py:93-95
        g = self.gradient(p)
        return np.sqrt(1.0 + np.sum(g * g, axis=-1))


class Sampled:
    """ddmesh/monitor.py:361-392 (SampledField) as an arc-length monitor:
    u / grad u by scipy's RegularGridInterpolator(linear) of the (smoothed)
    lattice and its np.gradient lattices; ``__call__`` is the arc length."""

    def __init__(self, axes, values, smooth_passes=0):
        from scipy.interpolate import RegularGridInterpolator as RGI
        self.axes = tuple(np.asarray(a, dtype=float) for a in axes)
        values = np.asarray(values, dtype=float)
        if smooth_passes:
            values = smooth(values, smooth_passes)
        self.values = values
        self.domain = tuple((float(a[0]), float(a[-1])) for a in self.axes)
        hs = [float(a[1] - a[0]) for a in self.axes]
        grads = [np.gradient(values, h, axis=k, edge_order=2) for k, h in enumerate(hs)]
        self._iu = RGI(self.axes, values, method="linear")
        self._ig = [RGI(self.axes, g, method="linear") for g in grads]

    def u(self, p):
        p = np.asarray(p, dtype=float)
        return self._iu(p.reshape(-1, len(self.axes))).reshape(p.shape[:-1])

    def gradient(self, p):
        p = np.asarray(p, dtype=float)
        flat = p.reshape(-1, len(self.axes))
        return np.stack([g(flat) for g in self._ig], axis=-1).reshape(p.shape)

    def __call__(self, p):
        g = self.gradient(p)
        return np.sqrt(1.0 + np.sum(g * g, axis=-1))


def _pullback_gradient_sq(gxi, jac):
    """ddmesh/monitor.py:183-216."""
    dim = len(gxi)
    if dim == 2:
        a, b = jac[0][0], jac[0][1]
        c, d = jac[1][0], jac[1][1]
        det = a * d - b * c
        comps = [d * gxi[0] - c * gxi[1], -b * gxi[0] + a * gxi[1]]
    else:
        m = jac
        det = (m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1])
               - m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0])
               + m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]))
        comps = []
        for i in range(3):
            i1, i2 = [r for r in range(3) if r != i]
            acc = 0
            for j in range(3):
                j1, j2 = [q for q in range(3) if q != j]
                minor = m[i1][j1] * m[i2][j2] - m[i1][j2] * m[i2][j1]
                acc = acc + (minor if (i + j) % 2 == 0 else -minor) * gxi[j]
            comps.append(acc)
    g2 = sum(c * c for c in comps)
    safe = np.abs(det) > 1e-12
    return np.where(safe, g2 / np.where(safe, det * det, 1.0), 0.0)


def smooth(values, passes):
    """ddmesh/monitor.py:395-409: per-axis [1,2,1]/4 with reflected edges."""
    out = values
    for _ in range(passes):
        for axis in range(out.ndim):
            n = out.shape[axis]
            left = np.take(out, [1] + list(range(0, n - 1)), axis=axis)
            right = np.take(out, list(range(1, n)) + [n - 2], axis=axis)
            out = 0.25 * left + 0.5 * out + 0.25 * right
    return out


def mesh_density(mon, coords, spacing, domain, smooth_passes=0):
    """ddmesh/monitor.py:151-180: raw at the clamped mesh nodes, or for a
    u-backed monitor the pull-back of u sampled there; then smoothing."""
    rho = _mesh_density(mon, coords, spacing, domain)
    return smooth(rho, smooth_passes) if smooth_passes else rho


def _mesh_density(mon, coords, spacing, domain):
    pts = clamp(coords, domain)
    if not hasattr(mon, "u"):
        return mon(pts)
    dim = coords.shape[-1]
    u = mon.u(pts)
    gxi = [np.gradient(u, spacing[l], axis=l, edge_order=2) for l in range(dim)]
    jac = [[np.gradient(coords[..., k], spacing[l], axis=l, edge_order=2)
            for l in range(dim)] for k in range(dim)]
    return np.sqrt(1.0 + _pullback_gradient_sq(gxi, jac))


def clamp(points, domain):
    """ddmesh/monitor.py:70-74."""
    lo = np.array([a for a, _ in domain])
    hi = np.array([b for _, b in domain])
    return np.clip(np.asarray(points, dtype=float), lo, hi)


# ------------------------------------------------------------- solver ----

@dataclass(frozen=True)
class Config:
    """ddmesh/schwarz.py:35-67 (SolverConfig)."""
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


@dataclass
class Box:
    sub: Sub
    geom: Geom
    psi: np.ndarray
    coords: np.ndarray
    jac: np.ndarray
    mask: np.ndarray
    stepper: object
    res: float = np.inf
    rho_raw: object = None


@dataclass
class Result:
    psi: np.ndarray
    coords: np.ndarray
    jac: np.ndarray
    sub_psi: list
    residuals: list = field(default_factory=list)      # per window tuple
    jac_min: list = field(default_factory=list)
    jac_max: list = field(default_factory=list)
    converged: bool = False
    windows: int = 0
    final_residual: float = np.inf
    overlap_gap: float = 0.0
    counter: Counter = field(default_factory=Counter)


def _counted(fn, counter, lock=None):
    def wrapped(y):
        if lock is None:
            counter.rhs_calls += 1
            counter.node_updates += y.size
        else:
            with lock:
                counter.rhs_calls += 1
                counter.node_updates += y.size
        return fn(y)
    return wrapped


def init_boxes(grid, dec, cfg, initial=None, traces=None):
    """ddmesh/schwarz.py:118-134."""
    if initial is None:
        initial = psi0(whole_geom(grid))
    elif initial.shape != grid.counts:
        raise OracleConfigError("warm-start shape")
    out = []
    for sub in dec.subs:
        g = box_geom(grid, sub)
        p = initial[sub.gslices()].copy()
        c, j = mesh_of(p, g)
        tr = None if traces is None else traces.setdefault(sub.id, [])
        out.append(Box(sub, g, p, c, j, g.mask(), make_stepper(cfg, tr)))
    return out


def apply_traces(box, sources, dec):
    """ddmesh/schwarz.py:137-159: descending donor id, lowest donor wins."""
    sub = box.sub
    nd = len(sub.box)
    for (axis, side), donor in sorted(sub.neighbors.items(), key=lambda kv: -kv[1]):
        dbox = dec.subs[donor].box
        line = sub.box[axis][side]
        dst = [slice(None)] * nd
        dst[axis] = -side
        src = [line - dbox[a][0] if a == axis else
               slice(sub.box[a][0] - dbox[a][0], sub.box[a][1] - dbox[a][0] + 1)
               for a in range(nd)]
        box.psi[tuple(dst)] = sources[donor][tuple(src)]


def densities(boxes, mon, domain, weights, smooth_passes=0, relax=0.0):
    """ddmesh/schwarz.py:162-192.  Returns (rho per box, rho_max, z)."""
    raws = [mesh_density(mon, b.coords, b.geom.spacing, domain, smooth_passes)
            for b in boxes]
    if relax > 0.0:
        raws = [raw if b.rho_raw is None else (1.0 - relax) * raw + relax * b.rho_raw
                for b, raw in zip(boxes, raws)]
    for b, raw in zip(boxes, raws):
        b.rho_raw = raw
    z = 0.0
    for b, raw in zip(boxes, raws):
        z += float(np.sum(weights[b.sub.owned_g()] * raw[b.sub.owned_l()]
                          * b.jac[b.sub.owned_l()]))
    if not np.isfinite(z) or z <= 0.0:
        raise OracleInvalidMonitor(f"transport quadrature {z}")
    rho = [raw / z for raw in raws]
    return rho, max(float(r.max()) for r in rho), z


def advance_box(box, rho, rho_max, cfg, psi_n, counter, lock=None):
    """ddmesh/schwarz.py:195-213."""
    def fn(y):
        return rhs_frozen(y, rho, box.geom, cfg.det_floor, box.mask, rho_max)
    try:
        box.psi = box.stepper.advance(box.psi, _counted(fn, counter, lock))
    except OracleStiffness as e:
        e.subdomain = box.sub.id
        raise
    box.coords, box.jac = mesh_of(box.psi, box.geom)
    box.res = l2_norm(box.psi - psi_n, box.geom.spacing)


def sweep(boxes, mon, domain, cfg, dec, weights, counter, pool=None, lock=None):
    """ddmesh/schwarz.py:216-268 (alternating or parallel)."""
    rho, rmax, _ = densities(boxes, mon, domain, weights, cfg.monitor_smooth_passes,
                             cfg.monitor_relax)
    if cfg.transmission == "alternating":
        src = [b.psi for b in boxes]
        for b in boxes:
            old = b.psi.copy()
            apply_traces(b, src, dec)
            advance_box(b, rho[b.sub.id], rmax, cfg, old, counter)
            src[b.sub.id] = b.psi
        return
    snap = [b.psi.copy() for b in boxes]
    for b in boxes:
        apply_traces(b, snap, dec)
    if pool is None:
        for b in boxes:
            advance_box(b, rho[b.sub.id], rmax, cfg, snap[b.sub.id], counter)
        return
    futs = [pool.submit(advance_box, b, rho[b.sub.id], rmax, cfg, snap[b.sub.id],
                        counter, lock) for b in boxes]
    first = None
    for f in futs:
        e = f.exception()
        if e is not None and first is None:
            first = e
    if first is not None:
        raise first


def assemble(grid, boxes):
    """ddmesh/schwarz.py:271-282."""
    psi = np.empty(grid.counts)
    coords = np.empty(grid.counts + (grid.dim,))
    jac = np.empty(grid.counts)
    for b in boxes:
        g, l = b.sub.owned_g(), b.sub.owned_l()
        psi[g] = b.psi[l]
        coords[g] = b.coords[l]
        jac[g] = b.jac[l]
    return psi, coords, jac


def overlap_gap(boxes):
    """ddmesh/schwarz.py:285-304."""
    gap = 0.0
    for i, bi in enumerate(boxes):
        for bj in boxes[i + 1:]:
            com = []
            for (a0, a1), (b0, b1) in zip(bi.sub.box, bj.sub.box):
                lo, hi = max(a0, b0), min(a1, b1)
                if lo > hi:
                    com = None
                    break
                com.append((lo, hi))
            if com is None:
                continue
            si = tuple(slice(lo - b[0], hi - b[0] + 1) for (lo, hi), b in zip(com, bi.sub.box))
            sj = tuple(slice(lo - b[0], hi - b[0] + 1) for (lo, hi), b in zip(com, bj.sub.box))
            gap = max(gap, float(np.abs(bi.psi[si] - bj.psi[sj]).max()))
    return gap


def solve(grid, dec, mon, domain, cfg, initial=None, traces=None, callback=None):
    """ddmesh/schwarz.py:307-350 (solve).  ``mon`` is the raw density
    callable, ``domain`` its clamp box."""
    boxes = init_boxes(grid, dec, cfg, initial, traces)
    reduce_res = min if cfg.stop_rule == "min" else max
    weights = trap_weights(grid.counts, grid.spacing)
    pool = lock = None
    if cfg.transmission == "parallel" and len(boxes) > 1 and (cfg.workers or 0) > 1:
        import threading
        pool = ThreadPoolExecutor(max_workers=cfg.workers)
        lock = threading.Lock()
    res = Result(None, None, None, None)
    stop = np.inf
    try:
        for w in range(cfg.max_windows):
            sweep(boxes, mon, domain, cfg, dec, weights, res.counter, pool, lock)
            stop = reduce_res(b.res for b in boxes)
            res.residuals.append(tuple(b.res for b in boxes))
            res.jac_min.append(min(float(b.jac.min()) for b in boxes))
            res.jac_max.append(max(float(b.jac.max()) for b in boxes))
            if callback is not None:
                callback(w, boxes)
            if stop <= cfg.tol:
                res.converged = True
                break
    finally:
        if pool is not None:
            pool.shutdown(wait=False)
    res.psi, res.coords, res.jac = assemble(grid, boxes)
    res.sub_psi = [b.psi for b in boxes]
    res.windows = len(res.residuals)
    res.final_residual = stop
    res.overlap_gap = overlap_gap(boxes)
    return res


def solve_single(grid, mon, domain, cfg, initial=None, trace=None):
    """ddmesh/schwarz.py:353-406 (solve_single_domain)."""
    geom = whole_geom(grid)
    psi = psi0(geom) if initial is None else initial.copy()
    if psi.shape != grid.counts:
        raise OracleConfigError("warm-start shape")
    mask = geom.mask()
    stepper = make_stepper(cfg, trace)
    weights = trap_weights(grid.counts, grid.spacing)
    out = Result(None, None, None, None)
    res = np.inf
    coords, jac = mesh_of(psi, geom)
    full = tuple(slice(0, n) for n in grid.counts)
    rho_prev = None
    for _ in range(cfg.max_windows):
        raw = mesh_density(mon, coords, geom.spacing, domain, cfg.monitor_smooth_passes)
        if cfg.monitor_relax > 0.0 and rho_prev is not None:
            raw = (1.0 - cfg.monitor_relax) * raw + cfg.monitor_relax * rho_prev
        rho_prev = raw
        z = float(np.sum(weights[full] * raw[full] * jac[full]))
        if not np.isfinite(z) or z <= 0.0:
            raise OracleInvalidMonitor(f"transport quadrature {z}")
        rho = raw / z
        rmax = float(rho.max())

        def fn(y, rho=rho, mx=rmax):
            return rhs_frozen(y, rho, geom, cfg.det_floor, mask, mx)

        old = psi
        psi = stepper.advance(psi, _counted(fn, out.counter))
        coords, jac = mesh_of(psi, geom)
        res = l2_norm(psi - old, geom.spacing)
        out.residuals.append((res,))
        out.jac_min.append(float(jac.min()))
        out.jac_max.append(float(jac.max()))
        if res <= cfg.tol:
            out.converged = True
            break
    out.psi, out.coords, out.jac = psi, coords, jac
    out.sub_psi = [psi]
    out.windows = len(out.residuals)
    out.final_residual = res
    return out


# -------------------------------------------------------- BASELINE cfgs ----

# ------------------------------------------------------------ metrics ----

def quality_measure(psi, raw_fn, domain, normalizer, geom, sample_on_mesh=False,
                    smooth_passes=0):
    """ddmesh/metrics.py:57-85 (no smoothing): -> (e_adp, e2, emax, node_mean,
    tangled).  rho = raw(clamp(x)) / normalizer (monitor.py:66-68), or with
    sample_on_mesh raw / sum(w raw J) (metrics.py:75-77, mesh_density
    monitor.py:151-180 without smoothing)."""
    coords, jac = mesh_of(psi, geom)
    w = trap_weights(jac.shape, geom.spacing)
    raw = (mesh_density(raw_fn, coords, geom.spacing, domain, smooth_passes) if sample_on_mesh
           else raw_fn(clamp(coords, domain)))
    if sample_on_mesh:
        rho = raw / float(np.sum(w * raw * jac))
    else:
        rho = raw / normalizer
    e = geom.measure * rho * jac
    e2 = float(np.sqrt(np.sum(w * e * e) / np.sum(w)))
    return e, e2, float(np.abs(e).max()), float(e.mean()), bool((jac <= 0.0).any())


def relative_errors(psi_dd, psi_sd, geom):
    """ddmesh/metrics.py:100-118 -> (e1, e2, einf)."""
    diff = np.abs(psi_sd - psi_dd)
    ref = np.abs(psi_sd)
    w = trap_weights(diff.shape, geom.spacing)
    e1 = float(np.sum(w * diff) / np.sum(w * ref))
    e2 = float(np.sqrt(np.sum(w * diff * diff) / np.sum(w * ref * ref)))
    return e1, e2, float(diff.max() / ref.max())


def baseline_case(name):
    """The five BASELINE.json configs as (grid, layout, overlap, monitor,
    domain, windows, transmission) — SURVEY §8(d) restatement."""
    if name == "C1":
        g = make_grid(2, ((0, 1), (0, 1)), (65, 65))
        return g, (2, 2), 4, Ring(), g.extents, 2000
    if name == "C2":
        g = make_grid(2, ((0, 1), (0, 1)), (513, 513))
        return g, (4, 4), 8, seeded_mixture(8, 2), g.extents, None
    if name == "C3":
        g = make_grid(2, ((0, 1), (0, 1)), (4097, 4097))
        return g, (8, 8), 16, seeded_mixture(32, 2), g.extents, 5000
    if name == "C4":
        g = make_grid(3, ((0, 1),) * 3, (129,) * 3)
        return g, (2, 2, 2), 4, Shell(), g.extents, 2000
    if name == "C5":
        g = make_grid(3, ((0, 1),) * 3, (513,) * 3)
        return g, (4, 4, 4), 8, seeded_mixture(16, 3), g.extents, 3000
    raise KeyError(name)


if __name__ == "__main__":  # quick self-timing
    g, lay, ov, mon, dom, _ = baseline_case("C1")
    d = make_decomposition(g, lay, ov)
    t0 = time.perf_counter()
    r = solve(g, d, mon, dom, Config(tol=1e-300, max_windows=50, transmission="parallel"))
    print(r.windows, r.final_residual, r.counter, time.perf_counter() - t0)
