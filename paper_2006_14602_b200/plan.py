"""Thin owner of a native ``ddpma_plan`` (device arena + controller state).

Everything numeric happens inside libddpma.so; this class only marshals
arguments, maps status codes onto the reference's exceptions and copies
results into numpy arrays.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import StiffnessError
from .grid import INTERFACE, PHYSICAL, BoxGeometry, CompGrid, Subdomain, to_c
from .monitor import MonitorField, NativeMonitor, UniformDensity, lower_monitor


def _cfg_to_c(config) -> _lib.SolverCfg:
    c = _lib.SolverCfg()
    c.dtau = float(config.dtau)
    c.tol = float(config.tol)
    c.transmission = _lib.PARALLEL if config.transmission == "parallel" else _lib.ALTERNATING
    c.stop_rule = _lib.STOP_MAX if config.stop_rule == "max" else _lib.STOP_MIN
    c.max_windows = int(config.max_windows)
    c.scheme = _lib.SCHEME_EULER if config.scheme == "euler" else _lib.SCHEME_ADAPTIVE
    c.substeps = int(config.substeps)
    c.rtol = float(config.rtol)
    c.atol = float(config.atol)
    c.max_stages = int(config.max_stages)
    c.det_floor = float(config.det_floor)
    c.monitor_smooth_passes = max(0, int(config.monitor_smooth_passes))
    c.monitor_relax = float(config.monitor_relax)
    return c


def _grid_to_c(grid: CompGrid) -> _lib.Grid:
    g = _lib.Grid()
    g.dim = grid.dim
    for k in range(3):
        g.counts[k] = grid.counts[k] if k < grid.dim else 1
    for k in range(grid.dim):
        g.extents[k][0], g.extents[k][1] = grid.extents[k]
    g.explicit_geom = 0
    return g


def _geom_to_c(geom: BoxGeometry):
    """One BoxGeometry as an explicit single-box 'grid' + its subdomain."""
    dim = geom.dim
    g = _lib.Grid()
    g.dim = dim
    shape = geom.shape()
    for k in range(3):
        g.counts[k] = shape[k] if k < dim else 1
    g.explicit_geom = 1
    g.measure = float(geom.domain_measure)
    for k in range(dim):
        g.extents[k][0] = float(geom.axes[k][0])
        g.extents[k][1] = float(geom.axes[k][-1])
        g.face_coord[k][0] = float(geom.axes[k][0])
        g.face_coord[k][1] = float(geom.axes[k][-1])
        g.spacing[k] = float(geom.spacing[k])
    sub = Subdomain(id=0, pos=(0,) * dim,
                    box=tuple((0, n - 1) for n in shape),
                    faces=tuple(geom.faces), neighbors={},
                    owned=tuple((0, n - 1) for n in shape))
    return g, sub


class Plan:
    """A native plan over ``subs`` (all subdomains; ``local`` = ids this
    process integrates, default all)."""

    def __init__(self, grid_c: _lib.Grid, subs, dim: int, native: NativeMonitor, config,
                 local=None, device: int | None = None):
        _lib.require_cuda()
        L = _lib.lib()
        self.L = L
        self.dim = dim
        self.nsub = len(subs)
        self.subs = list(subs)
        arr = (_lib.Subdomain * self.nsub)(*[to_c(s, dim) for s in subs])
        self._native = native
        self.cfg = _cfg_to_c(config)
        if device is None:
            import torch
            device = torch.cuda.current_device()
        self.device = device
        if local is None:
            loc, nloc = None, 0
        else:
            loc = (C.c_int * len(local))(*local)
            nloc = len(local)
        self.local = list(range(self.nsub)) if local is None else sorted(local)
        h = C.c_void_p()
        st = L.ddpma_plan_create(C.byref(grid_c), arr, self.nsub, loc, nloc,
                                 C.byref(native.desc), C.byref(self.cfg), int(device),
                                 C.byref(h))
        _lib.check_global(st)
        self.h = h
        self.grid_c = grid_c

    @classmethod
    def for_grid(cls, grid: CompGrid, subs, mon: MonitorField, config, local=None,
                 device=None):
        return cls(_grid_to_c(grid), subs, grid.dim, lower_monitor(mon, grid.dim), config,
                   local, device)

    @classmethod
    def for_geometry(cls, geom: BoxGeometry, config, mon: MonitorField | None = None):
        g, sub = _geom_to_c(geom)
        if mon is None:
            mon = MonitorField(raw=UniformDensity(1.0),
                               domain=tuple((float(ax[0]), float(ax[-1])) for ax in geom.axes))
        return cls(g, [sub], geom.dim, lower_monitor(mon, geom.dim), config)

    # ---------------------------------------------------------------------
    def close(self):
        if getattr(self, "h", None):
            self.L.ddpma_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def check(self, st: int):
        if st == _lib.OK:
            return
        msg = self.L.ddpma_last_error(self.h).decode()
        if st == _lib.ERR_STIFFNESS:
            raise self.stiffness_error()
        _lib.raise_status(st, msg)

    def stiffness_error(self) -> StiffnessError:
        """Rebuild StiffnessError(message, nodes, subdomain) exactly as the
        reference raises it (integrate.py:245-249, schwarz.py:209-211)."""
        sub = C.c_int(-1)
        t = C.c_double(0.0)
        h = C.c_double(0.0)
        nn = C.c_int64(0)
        self.L.ddpma_error_info(self.h, C.byref(sub), C.byref(t), C.byref(h), C.byref(nn))
        total = self.cfg.dtau
        msg = (f"internal step underflow at tau offset {t.value:.3e} "
               f"(h = {h.value:.3e}, window = {total:.3e})")
        nodes = None
        if nn.value != -1:
            cnt = self._error_node_count()
            out = np.empty(max(cnt, 1), dtype=np.int64)
            self.L.ddpma_error_nodes(self.h, out.ctypes.data_as(C.POINTER(C.c_int64)), cnt)
            shape = self.subs[sub.value].shape() if sub.value >= 0 else None
            nodes = np.stack(np.unravel_index(out[:cnt], shape), axis=-1) if shape else None
        return StiffnessError(msg, nodes=nodes, subdomain=sub.value)

    def _error_node_count(self) -> int:
        self.L.ddpma_error_nodes(self.h, None, 0)
        nn = C.c_int64(0)
        self.L.ddpma_error_info(self.h, None, None, None, C.byref(nn))
        return int(nn.value)

    def set_state(self, psi_global: np.ndarray | None):
        if psi_global is None:
            self.check(self.L.ddpma_set_state(self.h, None))
        else:
            a = np.ascontiguousarray(psi_global, dtype=np.float64)
            self.check(self.L.ddpma_set_state(self.h, _lib.dptr(a)))

    def run(self, max_windows: int, tol: float):
        hist_res = np.zeros((max_windows, self.nsub))
        hist_stats = np.zeros((max_windows, 4))
        w = C.c_int(0)
        conv = C.c_int(0)
        fres = C.c_double(0.0)
        self.check(self.L.ddpma_run(self.h, int(max_windows), float(tol), _lib.dptr(hist_res),
                                    _lib.dptr(hist_stats), C.byref(w), C.byref(conv),
                                    C.byref(fres)))
        return w.value, bool(conv.value), fres.value, hist_res[:w.value], hist_stats[:w.value]

    def assemble(self, counts):
        psi = np.empty(counts)
        coords = np.empty(tuple(counts) + (self.dim,))
        jac = np.empty(counts)
        self.check(self.L.ddpma_assemble_host(self.h, _lib.dptr(psi), _lib.dptr(coords),
                                              _lib.dptr(jac)))
        return psi, coords, jac

    def sub_psi(self, sub_id: int) -> np.ndarray:
        out = np.empty(self.subs[sub_id].shape())
        self.check(self.L.ddpma_get_sub_psi(self.h, int(sub_id), _lib.dptr(out)))
        return out

    def overlap_gap(self) -> float:
        g = C.c_double(0.0)
        self.check(self.L.ddpma_overlap_gap(self.h, C.byref(g)))
        return g.value

    def counters(self):
        nu, ev, la = C.c_int64(), C.c_int64(), C.c_int64()
        by = C.c_double()
        self.L.ddpma_counters(self.h, C.byref(nu), C.byref(ev), C.byref(la), C.byref(by))
        return {"node_updates": nu.value, "rhs_evals": ev.value, "launches": la.value,
                "algo_bytes": by.value}

    def sub_evals(self) -> np.ndarray:
        """RHS evaluations of every local subdomain since set_state (local
        order = ascending global id): the controller's per-subdomain tally."""
        out = np.zeros(len(self.local), dtype=np.int64)
        self.check(self.L.ddpma_sub_evals(self.h, out.ctypes.data_as(C.POINTER(C.c_int64)),
                                          len(self.local)))
        return out

    def set_profiling(self, on: bool):
        self.L.ddpma_set_profiling(self.h, 1 if on else 0)

    def profile(self):
        ms = np.zeros(_lib.NCLASS)
        by = np.zeros(_lib.NCLASS)
        la = np.zeros(_lib.NCLASS, dtype=np.int64)
        nu = np.zeros(_lib.NCLASS, dtype=np.int64)
        self.L.ddpma_profile(self.h, _lib.dptr(ms), _lib.dptr(by),
                             la.ctypes.data_as(C.POINTER(C.c_int64)),
                             nu.ctypes.data_as(C.POINTER(C.c_int64)), _lib.NCLASS)
        return {"ms": ms, "bytes": by, "launches": la, "node_updates": nu}

    # ----------------------------------------------- sharded window phases --
    def density(self):
        n = self.nsub
        z, rm, res, jmn, jmx = (np.zeros(n) for _ in range(5))
        self.check(self.L.ddpma_density(self.h, _lib.dptr(z), _lib.dptr(rm), _lib.dptr(res),
                                        _lib.dptr(jmn), _lib.dptr(jmx)))
        return z, rm, res, jmn, jmx

    def begin_window(self, z: float, rho_max: float):
        self.check(self.L.ddpma_begin_window(self.h, float(z), float(rho_max)))

    def trace_counts(self, rank_of, nranks: int, my_rank: int):
        ro = (C.c_int * self.nsub)(*rank_of)
        sc = np.zeros(nranks, dtype=np.int64)
        rc = np.zeros(nranks, dtype=np.int64)
        self.check(self.L.ddpma_trace_counts(self.h, ro, nranks, my_rank,
                                             sc.ctypes.data_as(C.POINTER(C.c_int64)),
                                             rc.ctypes.data_as(C.POINTER(C.c_int64))))
        return sc, rc

    def pack_traces(self, send_ptr: int):
        self.check(self.L.ddpma_pack_traces(self.h, C.c_void_p(send_ptr)))

    def apply_traces(self, recv_ptr: int | None):
        self.check(self.L.ddpma_apply_traces(self.h, C.c_void_p(recv_ptr) if recv_ptr else None))

    def advance(self):
        self.check(self.L.ddpma_advance(self.h))

    def assemble_dev(self, psi_ptr, coords_ptr, jac_ptr):
        self.check(self.L.ddpma_assemble_dev(self.h, C.c_void_p(psi_ptr), C.c_void_p(coords_ptr),
                                             C.c_void_p(jac_ptr)))

    # ------------------------------------------------ operator-level calls --
    def rhs_frozen(self, sub_id, psi, rho, rho_max):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        rho = np.ascontiguousarray(np.broadcast_to(rho, psi.shape), dtype=np.float64)
        out = np.empty_like(psi)
        flag = C.c_int(0)
        self.check(self.L.ddpma_rhs_frozen(self.h, int(sub_id), _lib.dptr(psi), _lib.dptr(rho),
                                           float(rho_max or 0.0), _lib.dptr(out), C.byref(flag)))
        return out, bool(flag.value)

    def mesh(self, sub_id, psi):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        coords = np.empty(psi.shape + (self.dim,))
        jac = np.empty_like(psi)
        self.check(self.L.ddpma_mesh(self.h, int(sub_id), _lib.dptr(psi), _lib.dptr(coords),
                                     _lib.dptr(jac)))
        return coords, jac

    def raw_density(self, sub_id, psi):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        raw = np.empty_like(psi)
        self.check(self.L.ddpma_raw_density(self.h, int(sub_id), _lib.dptr(psi), _lib.dptr(raw)))
        return raw

    def residual(self, sub_id, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        out = C.c_double(0.0)
        self.check(self.L.ddpma_residual(self.h, int(sub_id), _lib.dptr(a), _lib.dptr(b),
                                         C.byref(out)))
        return out.value

    def quality(self, sub_id, psi, normalizer, sample_on_mesh):
        psi = np.ascontiguousarray(psi, dtype=np.float64)
        e = np.empty_like(psi)
        rep = (C.c_double * 5)()
        self.check(self.L.ddpma_quality(self.h, int(sub_id), _lib.dptr(psi), float(normalizer),
                                        int(bool(sample_on_mesh)), _lib.dptr(e),
                                        C.cast(rep, C.POINTER(C.c_double))))
        return e, list(rep)

    def relative_errors(self, sub_id, dd, sd):
        dd = np.ascontiguousarray(dd, dtype=np.float64)
        sd = np.ascontiguousarray(sd, dtype=np.float64)
        out = (C.c_double * 3)()
        self.check(self.L.ddpma_relative_errors(self.h, int(sub_id), _lib.dptr(dd), _lib.dptr(sd),
                                                C.cast(out, C.POINTER(C.c_double))))
        return list(out)

    def rkc_step(self, sub_id, y, rho, rho_max, h, s):
        y = np.ascontiguousarray(y, dtype=np.float64)
        rho = np.ascontiguousarray(np.broadcast_to(rho, y.shape), dtype=np.float64)
        d = np.empty_like(y)
        fnew = np.empty_like(y)
        fl = C.c_int(0)
        ef = C.c_int(0)
        self.check(self.L.ddpma_rkc_step(self.h, int(sub_id), _lib.dptr(y), _lib.dptr(rho),
                                         float(rho_max or 0.0), float(h), int(s), _lib.dptr(d),
                                         _lib.dptr(fnew), C.byref(fl), C.byref(ef)))
        return d, fnew, bool(fl.value), bool(ef.value)

    def pack_owned(self, out_ptr) -> int:
        """ddpma_pack_owned: owned blocks of the local subdomains into the
        device buffer at out_ptr (None: just the element count)."""
        n = C.c_int64(0)
        self.check(self.L.ddpma_pack_owned(self.h, C.c_void_p(out_ptr) if out_ptr else None,
                                           C.byref(n)))
        return int(n.value)

    def integrate_window(self, sub_id, y, rho, rho_max):
        """One window of the plan's integrator on box field ``y`` (returned
        as a new array) with a frozen nodal density (ddpma_integrate_window)."""
        out = np.array(y, dtype=np.float64, order="C", copy=True)
        rho = np.ascontiguousarray(np.broadcast_to(rho, out.shape), dtype=np.float64)
        self.check(self.L.ddpma_integrate_window(self.h, int(sub_id), _lib.dptr(out),
                                                 _lib.dptr(rho), float(rho_max or 0.0)))
        return out


__all__ = ["Plan", "PHYSICAL", "INTERFACE"]
