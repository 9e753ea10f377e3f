"""Multi-GPU DDPMA: whole subdomains sharded over ranks (one process per GPU).

Parallel transmission makes every window embarrassingly parallel across
subdomains (schwarz.py:236-268); the only per-window exchange is

  1. one all-reduce of per-subdomain scalars [z partial, raw max, residual,
     J min, J max] — each entry has exactly one non-zero contributor, so the
     SUM is exact and the id-ordered z sum below is bitwise independent of
     the rank count;
  2. the face traces whose donor lives on another rank: packed on the device
     by the donor rank, moved with one all_to_all_single (NCCL over NVLink),
     applied by the receiver with the same corner precedence as a local
     trace (lowest donor id wins, schwarz.py:141-147).

The local compute is an *engine*: in production the native CUDA plan
(:class:`paper_2006_14602_b200.plan.Plan`); the CPU test-suite injects an
oracle-backed engine to exercise exactly this orchestration under gloo.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .errors import DdmeshError, InvalidMonitorError
from .grid import CompGrid, Decomposition


def partition(dec: Decomposition, world: int) -> list[int]:
    """rank_of[sub id]: recursive bisection of the subdomain lattice along
    its longest axis, balancing box-node counts — contiguous blocks keep
    most faces rank-local."""
    subs = list(dec.subdomains)
    rank_of = [0] * len(subs)

    def split(items, r0, nr):
        if nr == 1 or len(items) <= 1:
            for s in items:
                rank_of[s.id] = r0
            return
        dim = len(items[0].pos)
        spans = [max(s.pos[k] for s in items) - min(s.pos[k] for s in items) for k in range(dim)]
        ax = int(np.argmax(spans))
        items = sorted(items, key=lambda s: (s.pos[ax], s.id))
        left_r = nr // 2
        w = np.array([np.prod(s.shape()) for s in items], dtype=np.float64)
        target = w.sum() * left_r / nr
        # cut between lattice lines of `ax` closest to the target weight
        cands = []
        acc = 0.0
        for i in range(1, len(items)):
            acc += w[i - 1]
            if items[i].pos[ax] != items[i - 1].pos[ax]:
                cands.append((abs(acc - target), i))
        cut = min(cands)[1] if cands else len(items) // 2
        split(items[:cut], r0, left_r)
        split(items[cut:], r0 + left_r, nr - left_r)

    split(subs, 0, world)
    return rank_of


def partition_lpt(dec: Decomposition, world: int, weights) -> list[int]:
    """rank_of[sub id] by greedy longest-processing-time: subdomains in order
    of decreasing measured work (e.g. RHS evaluations x box nodes of the
    previous window, Plan.sub_evals) go to the least-loaded rank (ties: the
    lowest rank).  The reference's parallel_sweep balances nothing: its
    thread pool takes subdomains in id order (schwarz.py:259-268)."""
    w = np.asarray(weights, dtype=np.float64)
    order = sorted(range(dec.nsub), key=lambda i: (-w[i], i))
    load = np.zeros(world)
    rank_of = [0] * dec.nsub
    for i in order:
        r = int(np.argmin(load))
        rank_of[i] = r
        load[r] += w[i]
    return rank_of


def makespan(weights, rank_of, world: int) -> tuple[float, float]:
    """(max rank load, parallel efficiency sum/(world * max)) of a partition
    under per-subdomain costs `weights` (a projection: no exchange cost, no
    intra-window dynamics)."""
    w = np.asarray(weights, dtype=np.float64)
    load = np.zeros(world)
    for i, r in enumerate(rank_of):
        load[r] += w[i]
    mx = float(load.max())
    return mx, float(w.sum() / (world * mx)) if mx > 0 else 1.0


def owned_sizes(dec: Decomposition, ids) -> list[int]:
    """Packed length (ddpma_pack_owned layout) of each subdomain in `ids`."""
    dim = dec.grid.dim
    return [int(np.prod([hi - lo + 1 for lo, hi in dec.subdomains[i].owned])) * (2 + dim)
            for i in ids]


def unpack_owned(dec: Decomposition, ids, buf: torch.Tensor, psi: torch.Tensor,
                 coords: torch.Tensor, jac: torch.Tensor) -> None:
    """Scatter a ddpma_pack_owned buffer of subdomains `ids` (ascending) into
    the global arrays (schwarz.py:271-282 assembly, on the device)."""
    dim = dec.grid.dim
    off = 0
    for i in sorted(ids):
        sub = dec.subdomains[i]
        shape = tuple(hi - lo + 1 for lo, hi in sub.owned)
        n = int(np.prod(shape))
        gs = sub.owned_global_slices()
        psi[gs] = buf[off:off + n].view(shape)
        coords[gs] = buf[off + n:off + n * (1 + dim)].view(shape + (dim,))
        jac[gs] = buf[off + n * (1 + dim):off + n * (2 + dim)].view(shape)
        off += n * (2 + dim)


class PlanEngine:
    """Adapter of the native plan to the engine interface."""

    def __init__(self, grid, dec, mon, config, local, device):
        from .plan import Plan
        self.plan = Plan.for_grid(grid, dec.subdomains, mon, config, local=local, device=device)
        self.device = torch.device("cuda", device)

    def set_state(self, initial):
        self.plan.set_state(initial)

    def density(self):
        return self.plan.density()

    def begin_window(self, z, rho_max):
        self.plan.begin_window(z, rho_max)

    def trace_counts(self, rank_of, world, rank):
        return self.plan.trace_counts(rank_of, world, rank)

    def pack_traces(self, send: torch.Tensor):
        self.plan.pack_traces(send.data_ptr() if send.numel() else 0)

    def apply_traces(self, recv: torch.Tensor | None):
        self.plan.apply_traces(recv.data_ptr() if recv is not None and recv.numel() else None)

    def advance(self):
        self.plan.advance()

    def assemble_into(self, psi: torch.Tensor, coords: torch.Tensor, jac: torch.Tensor):
        self.plan.assemble_dev(psi.data_ptr(), coords.data_ptr(), jac.data_ptr())

    def pack_owned(self, out: torch.Tensor | None) -> int:
        return self.plan.pack_owned(out.data_ptr() if out is not None and out.numel() else None)

    def sub_psi(self, sid):
        return self.plan.sub_psi(sid)

    def sub_evals(self):
        return self.plan.sub_evals()

    def counters(self):
        return self.plan.counters()


class ShardedSolver:
    """Parallel-transmission solve() with subdomains sharded over ranks."""

    def __init__(self, grid: CompGrid, dec: Decomposition, mon, config, rank: int, world: int,
                 device: int | None = None, engine=None, rank_of=None, group=None):
        if config.transmission != "parallel" and world > 1:
            raise DdmeshError("alternating transmission is a sequential sweep; it runs on one "
                              "GPU only (SURVEY §8(e))")
        self.grid, self.dec, self.config = grid, dec, config
        self.rank, self.world, self.group = rank, world, group
        self.rank_of = list(rank_of) if rank_of is not None else partition(dec, world)
        self.local = [i for i in range(dec.nsub) if self.rank_of[i] == rank]
        self.engine = engine if engine is not None else PlanEngine(
            grid, dec, mon, config, self.local, device if device is not None else 0)
        self.device = self.engine.device
        sc, rc = self.engine.trace_counts(self.rank_of, world, rank)
        self.send_splits = [int(x) for x in sc]
        self.recv_splits = [int(x) for x in rc]
        self.send = torch.zeros(sum(self.send_splits), dtype=torch.float64, device=self.device)
        self.recv = torch.zeros(sum(self.recv_splits), dtype=torch.float64, device=self.device)
        self.stats = None
        self.history = []

    # exposed for bench.py
    @property
    def plan(self):
        return self.engine.plan

    @property
    def stream(self):
        from . import _lib
        return torch.cuda.ExternalStream(_lib.lib().ddpma_stream(self.engine.plan.h))

    def counters(self):
        return self.engine.counters()

    def _allreduce_stats(self, z, rm, res, jmn, jmx):
        t = torch.tensor(np.stack([z, rm, res, jmn, jmx]), dtype=torch.float64,
                         device=self.device)
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def set_state(self, initial):
        self.engine.set_state(initial)
        self.stats = self._allreduce_stats(*self.engine.density())
        self.history = []

    def _exchange(self):
        self.engine.pack_traces(self.send)
        if self.world > 1 and (sum(self.send_splits) or sum(self.recv_splits)):
            if self.device.type == "cuda":
                torch.cuda.synchronize(self.device)
            dist.all_to_all_single(self.recv, self.send, self.recv_splits, self.send_splits,
                                   group=self.group)
            if self.device.type == "cuda":
                torch.cuda.synchronize(self.device)
        self.engine.apply_traces(self.recv)

    def _check_errors(self, err):
        """Propagate the failure of the lowest subdomain id (schwarz.py:262-268)."""
        gid = float(err.subdomain) if err is not None and getattr(err, "subdomain", None) \
            is not None else (1e9 if err is not None else 2e9)
        t = torch.tensor([gid], dtype=torch.float64, device=self.device)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        first = float(t.item())
        if first >= 2e9:
            return
        if err is not None and gid == first:
            raise err
        raise DdmeshError(f"subdomain {int(first) if first < 1e9 else '?'} failed on another rank")

    def window(self):
        """One window (schwarz.py:327-339); returns the stop residual."""
        z_part, raw_max = self.stats[0], self.stats[1]
        z = 0.0
        for v in z_part:                 # id order, as schwarz.py:182-186
            z += float(v)
        if not np.isfinite(z) or z <= 0.0:
            raise InvalidMonitorError(f"transport quadrature of the mesh density is {z}")
        rho_max = max(float(r) / z for r in raw_max)
        self.engine.begin_window(z, rho_max)
        self._exchange()
        err = None
        try:
            self.engine.advance()
        except (DdmeshError, ValueError, OverflowError) as e:
            err = e
        self._check_errors(err)
        self.stats = self._allreduce_stats(*self.engine.density())
        res = self.stats[2]
        stop = float(res.min() if self.config.stop_rule == "min" else res.max())
        self.history.append((tuple(float(x) for x in res), stop, float(self.stats[3].min()),
                             float(self.stats[4].max())))
        return stop

    def run(self, max_windows=None, tol=None):
        max_windows = max_windows or self.config.max_windows
        tol = self.config.tol if tol is None else tol
        converged = False
        stop = np.inf
        for _ in range(max_windows):
            stop = self.window()
            if stop <= tol:
                converged = True
                break
        return converged, stop

    def assemble(self):
        """Owned blocks of every rank packed on the device (ddpma_pack_owned)
        and gathered onto rank 0 with one all-gather over NCCL (SURVEY
        §8(e)); rank 0 scatters them into the global psi / coords / jac.
        Other ranks return None."""
        n = self.engine.pack_owned(None)
        buf = torch.empty(n, dtype=torch.float64, device=self.device)
        self.engine.pack_owned(buf)
        sizes = [sum(owned_sizes(self.dec, [i for i in range(self.dec.nsub)
                                            if self.rank_of[i] == r])) for r in range(self.world)]
        if self.world > 1:
            mx = max(sizes)
            send = torch.zeros(mx, dtype=torch.float64, device=self.device)
            send[:n] = buf
            if self.device.type == "cuda":
                allb = torch.empty(self.world * mx, dtype=torch.float64, device=self.device)
                dist.all_gather_into_tensor(allb, send, group=self.group)
                parts = [allb[r * mx:r * mx + sizes[r]] for r in range(self.world)]
            else:   # gloo (CPU test engines)
                lst = [torch.empty(mx, dtype=torch.float64) for _ in range(self.world)]
                dist.all_gather(lst, send, group=self.group)
                parts = [lst[r][:sizes[r]] for r in range(self.world)]
        else:
            parts = [buf]
        if self.rank != 0:
            return None
        counts = tuple(self.grid.counts)
        psi = torch.zeros(counts, dtype=torch.float64, device=self.device)
        coords = torch.zeros(counts + (self.grid.dim,), dtype=torch.float64, device=self.device)
        jac = torch.zeros(counts, dtype=torch.float64, device=self.device)
        for r in range(self.world):
            ids = [i for i in range(self.dec.nsub) if self.rank_of[i] == r]
            unpack_owned(self.dec, ids, parts[r], psi, coords, jac)
        return psi, coords, jac


class InProcessShards:
    """`world` native plans on ONE device, each owning the subdomains with
    rank_of[i] == r, stepped in lockstep with the per-window exchange done in
    process (the all-reduce as a sum over plans, the all_to_all as a re-split
    of the packed trace buffers, the owned blocks gathered as in
    ShardedSolver.assemble).  It runs the exact native sharded code path of
    a multi-GPU job (ddpma_density / _begin_window / _trace_counts /
    _pack_traces / _apply_traces / _advance / _pack_owned) without needing
    more than one GPU, and must be bitwise identical to a single-plan
    solve.  The plans' kernels never wait on one another."""

    def __init__(self, grid, dec, mon, config, rank_of, device=0, engines=None):
        self.grid, self.dec, self.config = grid, dec, config
        self.rank_of = list(rank_of)
        self.world = max(self.rank_of) + 1
        self.device = torch.device("cuda", device) if engines is None else engines[0].device
        self.locals = [[i for i in range(dec.nsub) if self.rank_of[i] == r]
                       for r in range(self.world)]
        self.engines = engines if engines is not None else [
            PlanEngine(grid, dec, mon, config, loc, device) for loc in self.locals]
        self.splits = []
        for r, e in enumerate(self.engines):
            sc, rc = e.trace_counts(self.rank_of, self.world, r)
            self.splits.append(([int(x) for x in sc], [int(x) for x in rc]))
        self.send = [torch.zeros(sum(sc), dtype=torch.float64, device=self.device)
                     for sc, _ in self.splits]
        self.recv = [torch.zeros(sum(rc), dtype=torch.float64, device=self.device)
                     for _, rc in self.splits]
        self.history = []

    def _stats(self):
        tot = None
        for e in self.engines:
            t = np.stack(e.density())
            tot = t if tot is None else tot + t   # one non-zero contributor per entry: exact
        return tot

    def set_state(self, initial=None):
        for e in self.engines:
            e.set_state(initial)
        self.stats = self._stats()
        self.history = []

    def window(self):
        z_part, raw_max = self.stats[0], self.stats[1]
        z = 0.0
        for v in z_part:                 # id order, as schwarz.py:182-186
            z += float(v)
        if not np.isfinite(z) or z <= 0.0:
            raise InvalidMonitorError(f"transport quadrature of the mesh density is {z}")
        rho_max = max(float(r) / z for r in raw_max)
        for r, e in enumerate(self.engines):
            e.begin_window(z, rho_max)
            e.pack_traces(self.send[r])
        # all_to_all_single: recv[r] gathers, in source-rank order, the
        # segment of send[s] addressed to r
        pieces = [list(torch.split(self.send[s], self.splits[s][0])) for s in range(self.world)]
        for r in range(self.world):
            if self.recv[r].numel():
                torch.cat([pieces[s][r] for s in range(self.world)], out=self.recv[r])
        for r, e in enumerate(self.engines):
            e.apply_traces(self.recv[r])
        errs = []
        for e in self.engines:
            try:
                e.advance()
            except (DdmeshError, ValueError, OverflowError) as err:
                errs.append(err)
        if errs:   # the lowest failing subdomain id wins (schwarz.py:262-268)
            raise min(errs, key=lambda x: getattr(x, "subdomain", None) or 10 ** 9)
        self.stats = self._stats()
        res = self.stats[2]
        stop = float(res.min() if self.config.stop_rule == "min" else res.max())
        self.history.append((tuple(float(x) for x in res), stop, float(self.stats[3].min()),
                             float(self.stats[4].max())))
        return stop

    def assemble(self):
        counts = tuple(self.grid.counts)
        psi = torch.zeros(counts, dtype=torch.float64, device=self.device)
        coords = torch.zeros(counts + (self.grid.dim,), dtype=torch.float64, device=self.device)
        jac = torch.zeros(counts, dtype=torch.float64, device=self.device)
        for r, e in enumerate(self.engines):
            n = e.pack_owned(None)
            buf = torch.empty(n, dtype=torch.float64, device=self.device)
            e.pack_owned(buf)
            unpack_owned(self.dec, self.locals[r], buf, psi, coords, jac)
        return psi, coords, jac

    def sub_evals(self):
        out = np.zeros(self.dec.nsub, dtype=np.int64)
        for r, e in enumerate(self.engines):
            out[self.locals[r]] = e.sub_evals()
        return out

    def node_updates(self):
        return sum(e.counters()["node_updates"] for e in self.engines)
