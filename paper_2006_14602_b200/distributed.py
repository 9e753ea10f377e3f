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

    def sub_psi(self, sid):
        return self.plan.sub_psi(sid)

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
        """Owned blocks of every rank, reduced onto rank 0 (exact: disjoint)."""
        counts = tuple(self.grid.counts)
        psi = torch.zeros(counts, dtype=torch.float64, device=self.device)
        coords = torch.zeros(counts + (self.grid.dim,), dtype=torch.float64, device=self.device)
        jac = torch.zeros(counts, dtype=torch.float64, device=self.device)
        self.engine.assemble_into(psi, coords, jac)
        if self.world > 1:
            for t in (psi, coords, jac):
                dist.reduce(t, dst=0, group=self.group)
        return psi, coords, jac
