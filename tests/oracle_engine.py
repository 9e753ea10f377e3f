"""Test-only local engine for paper_2006_14602_b200.distributed.ShardedSolver.

It integrates the rank's subdomains with the CPU oracle (oracle/ddpma_oracle.py)
and implements the same engine interface as the CUDA PlanEngine, including
the canonical trace-segment order of ddpma_trace_counts (receiver id, axis,
side; peers in rank order).  This lets the CPU suite run the sharded
orchestration (z / rho_max / residual all-reduce, all_to_all face exchange,
corner precedence, owned-block reduction) under gloo with world_size 2 and
compare it bitwise with the single-process reference restatement.
"""

from __future__ import annotations

import numpy as np
import torch

import ddpma_oracle as O


class OracleEngine:
    def __init__(self, grid, dec, mon, domain, cfg, local):
        self.g, self.d, self.mon, self.dom, self.cfg = grid, dec, mon, domain, cfg
        self.local = sorted(local)
        self.device = torch.device("cpu")
        self.weights = O.trap_weights(grid.counts, grid.spacing)
        self.boxes = {}
        self.evals = 0

    # ------------------------------------------------------------ engine --
    def set_state(self, initial):
        allb = O.init_boxes(self.g, self.d, self.cfg, initial)
        self.boxes = {b.sub.id: b for b in allb if b.sub.id in self.local}
        self.snap = {}
        self.raw = {}

    def density(self):
        n = len(self.d.subs)
        z, rm, res, jmn, jmx = (np.zeros(n) for _ in range(5))
        for sid, b in self.boxes.items():
            raw = self.mon(O.clamp(b.coords, self.dom))
            self.raw[sid] = raw
            z[sid] = float(np.sum(self.weights[b.sub.owned_g()] * raw[b.sub.owned_l()]
                                  * b.jac[b.sub.owned_l()]))
            rm[sid] = float(raw.max())
            res[sid] = b.res if np.isfinite(b.res) else 0.0
            jmn[sid] = float(b.jac.min())
            jmx[sid] = float(b.jac.max())
        return z, rm, res, jmn, jmx

    def begin_window(self, z, rho_max):
        self.rho = {sid: raw / z for sid, raw in self.raw.items()}
        self.rho_max = rho_max
        self.snap = {sid: b.psi.copy() for sid, b in self.boxes.items()}

    def _segments(self):
        segs = []
        for R in self.d.subs:
            for (axis, side), donor in sorted(R.neighbors.items()):
                segs.append((R.id, axis, side, donor))
        return segs

    def _face_ext(self, R, axis):
        return [R.box[a][1] - R.box[a][0] + 1 for a in range(len(R.box)) if a != axis]

    def _donor_slab(self, R, axis, side, donor_psi, D):
        idx = []
        for a in range(len(R.box)):
            if a == axis:
                idx.append(R.box[axis][side] - D.box[a][0])
            else:
                idx.append(slice(R.box[a][0] - D.box[a][0], R.box[a][1] - D.box[a][0] + 1))
        return donor_psi[tuple(idx)]

    def trace_counts(self, rank_of, world, rank):
        self.rank_of, self.world, self.rank = list(rank_of), world, rank
        send, recv = [[] for _ in range(world)], [[] for _ in range(world)]
        for seg in self._segments():
            R, axis, side, donor = seg
            rr, rd = rank_of[R], rank_of[donor]
            if rr == rd:
                continue
            if rd == rank:
                send[rr].append(seg)
            if rr == rank:
                recv[rd].append(seg)
        self.send_segs, self.recv_segs = [], []
        off = 0
        sc = np.zeros(world, dtype=np.int64)
        for r in range(world):
            for seg in send[r]:
                n = int(np.prod(self._face_ext(self.d.subs[seg[0]], seg[1])))
                self.send_segs.append((seg, off, n))
                off += n
                sc[r] += n
        off = 0
        rc = np.zeros(world, dtype=np.int64)
        for r in range(world):
            for seg in recv[r]:
                n = int(np.prod(self._face_ext(self.d.subs[seg[0]], seg[1])))
                self.recv_segs.append((seg, off, n))
                off += n
                rc[r] += n
        return sc, rc

    def pack_traces(self, send):
        buf = send.numpy()
        for (R, axis, side, donor), off, n in self.send_segs:
            slab = self._donor_slab(self.d.subs[R], axis, side, self.snap[donor],
                                    self.d.subs[donor])
            buf[off:off + n] = np.ascontiguousarray(slab).reshape(-1)

    def apply_traces(self, recv):
        rbuf = recv.numpy() if recv is not None else None
        remote = {(seg[0], seg[1], seg[2]): (off, n) for seg, off, n in self.recv_segs}
        for sid, b in self.boxes.items():
            R = b.sub
            nd = len(R.box)
            # descending donor id: the lowest donor wins at corners (schwarz.py:141-147)
            for (axis, side), donor in sorted(R.neighbors.items(), key=lambda kv: -kv[1]):
                dst = [slice(None)] * nd
                dst[axis] = -side
                ext = self._face_ext(R, axis)
                if donor in self.snap:
                    vals = self._donor_slab(R, axis, side, self.snap[donor], self.d.subs[donor])
                else:
                    off, n = remote[(sid, axis, side)]
                    vals = rbuf[off:off + n].reshape(ext)
                b.psi[tuple(dst)] = vals

    def advance(self):
        counter = O.Counter()
        for sid in sorted(self.boxes):
            b = self.boxes[sid]
            O.advance_box(b, self.rho[sid], self.rho_max, self.cfg, self.snap[sid], counter)
        self.evals += counter.node_updates

    def assemble_into(self, psi, coords, jac):
        p, c, j = psi.numpy(), coords.numpy(), jac.numpy()
        for b in self.boxes.values():
            gs, ls = b.sub.owned_g(), b.sub.owned_l()
            p[gs] = b.psi[ls]
            c[gs] = b.coords[ls]
            j[gs] = b.jac[ls]

    def pack_owned(self, out):
        """ddpma_pack_owned layout: per local subdomain (ascending id) its
        owned block as [psi | coords (interleaved) | jac], C order."""
        parts = []
        for sid in sorted(self.boxes):
            b = self.boxes[sid]
            ls = b.sub.owned_l()
            parts += [b.psi[ls].reshape(-1), b.coords[ls].reshape(-1), b.jac[ls].reshape(-1)]
        flat = np.concatenate(parts) if parts else np.zeros(0)
        if out is not None and out.numel():
            out.copy_(torch.from_numpy(flat))
        return flat.size

    def sub_evals(self):
        return np.zeros(len(self.local), dtype=np.int64)

    def counters(self):
        return {"node_updates": self.evals}
