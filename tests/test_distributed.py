"""Multi-rank orchestration (paper_2006_14602_b200/distributed.py) on CPU:
world_size 2 over gloo with the oracle-backed test engine.  The sharded run
must be BITWISE identical to the single-process parallel-transmission solve
(the reference restatement), for any rank layout — the per-window exchange
(exact z / rho_max / residual all-reduce, face traces, owned-block gather) may
not change a single bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import ddpma_oracle as O

import paper_2006_14602_b200 as P
from paper_2006_14602_b200.distributed import ShardedSolver, partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(name):
    if name == "C1":
        og = O.make_grid(2, ((0, 1), (0, 1)), (65, 65))
        lay, ov, mon = (2, 2), 4, O.Ring()
    elif name == "slab":
        og = O.make_grid(2, ((0, 1), (0, 1)), (41, 33))
        lay, ov, mon = (3, 2), 3, O.Ring(amp=4.0, sharp=20.0)
    else:  # 3D
        og = O.make_grid(3, ((0, 1),) * 3, (17, 17, 17))
        lay, ov, mon = (2, 2, 2), 4, O.Shell()
    return og, lay, ov, mon


def _worker(rank, world, port, name, windows, rank_of, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_engine import OracleEngine
        og, lay, ov, mon = _case(name)
        od = O.make_decomposition(og, lay, ov)
        g = P.build_grid(og.dim, og.extents, og.counts)
        d = P.build_decomposition(g, lay, ov)
        cfg = P.SolverConfig(tol=1e-300, max_windows=windows, transmission="parallel")
        ocfg = O.Config(tol=1e-300, max_windows=windows, transmission="parallel")
        rank_of = rank_of or partition(d, world)
        local = [i for i in range(d.nsub) if rank_of[i] == rank]
        eng = OracleEngine(og, od, mon, og.extents, ocfg, local)
        solver = ShardedSolver(g, d, None, cfg, rank=rank, world=world, engine=eng,
                               rank_of=rank_of)
        solver.set_state(None)
        solver.run()
        out_ = solver.assemble()
        if rank == 0:
            psi, coords, jac = out_
            np.savez(out, psi=psi.numpy(), coords=coords.numpy(), jac=jac.numpy(),
                     res=np.array([h[0] for h in solver.history]),
                     jmin=np.array([h[2] for h in solver.history]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,windows,rank_of", [
    ("C1", 6, None),
    ("C1", 4, [1, 0, 0, 1]),          # interleaved: every face crosses ranks
    ("slab", 5, None),
    ("3d", 3, None),
])
def test_sharded_equals_single_process(tmp_path, name, windows, rank_of):
    out = str(tmp_path / "r.npz")
    mp.spawn(_worker, args=(2, _free_port(), name, windows, rank_of, out), nprocs=2)
    got = np.load(out)
    og, lay, ov, mon = _case(name)
    od = O.make_decomposition(og, lay, ov)
    ref = O.solve(og, od, mon, og.extents,
                  O.Config(tol=1e-300, max_windows=windows, transmission="parallel"))
    assert np.array_equal(got["psi"], ref.psi)
    assert np.array_equal(got["coords"], ref.coords)
    assert np.array_equal(got["jac"], ref.jac)
    assert np.array_equal(got["res"], np.array(ref.residuals))
    assert np.array_equal(got["jmin"], np.array(ref.jac_min))


def test_partition_is_contiguous_and_balanced():
    g = P.build_grid(2, ((0.0, 1.0),) * 2, (4097, 4097))
    d = P.build_decomposition(g, (8, 8), 16)
    for world in (1, 2, 4, 8):
        ro = partition(d, world)
        assert sorted(set(ro)) == list(range(world))
        loads = np.zeros(world)
        for s in d.subdomains:
            loads[ro[s.id]] += np.prod(s.shape())
        assert loads.max() / loads.min() < 1.05
        # each rank's block is a contiguous rectangle of the lattice
        for r in range(world):
            pos = np.array([s.pos for s in d.subdomains if ro[s.id] == r])
            span = np.prod(pos.max(0) - pos.min(0) + 1)
            assert span == len(pos)
    g3 = P.build_grid(3, ((0.0, 1.0),) * 3, (513, 513, 513))
    d3 = P.build_decomposition(g3, (4, 4, 4), 8)
    for world in (2, 4, 8):
        ro = partition(d3, world)
        counts = np.bincount(ro, minlength=world)
        assert counts.min() == counts.max() == 64 // world


def test_alternating_refuses_sharding():
    g = P.build_grid(2, ((0.0, 1.0),) * 2, (65, 65))
    d = P.build_decomposition(g, (2, 2), 4)
    with pytest.raises(P.DdmeshError):
        ShardedSolver(g, d, None, P.SolverConfig(transmission="alternating"), rank=0, world=2,
                      engine=object())


def test_lpt_partition_and_makespan():
    g = P.build_grid(2, ((0.0, 1.0),) * 2, (65, 65))
    d = P.build_decomposition(g, (4, 4), 4)
    from paper_2006_14602_b200.distributed import makespan, partition_lpt
    rng = np.random.default_rng(1)
    w = rng.uniform(1.0, 50.0, d.nsub)
    for world in (2, 4, 8):
        ro = partition_lpt(d, world, w)
        mx, eff = makespan(w, ro, world)
        # LPT bound: makespan <= (4/3 - 1/(3m)) * OPT, OPT >= max(mean load, max item)
        opt_lb = max(w.sum() / world, w.max())
        assert mx <= (4.0 / 3.0 - 1.0 / (3 * world)) * opt_lb + 1e-9
        assert 0.0 < eff <= 1.0
        assert sorted(set(ro)) == list(range(world))


# ------------------------------------------------------------------- GPU ---

@pytest.mark.gpu
@pytest.mark.parametrize("name,rank_of", [
    ("C1", [0, 0, 1, 1]),
    ("C1", [1, 0, 0, 1]),                      # interleaved: every face crosses ranks
    ("C1", [0, 1, 2, 3]),
    ("T3", [0, 1, 1, 0, 1, 0, 0, 1]),          # 3D, interleaved
    ("T3", [0, 0, 1, 1, 2, 2, 3, 3]),
])
def test_native_sharded_plans_bitwise(name, rank_of):
    """The native multi-GPU code path (PlanEngine: per-rank plans owning a
    subset, ddpma_density / _begin_window / _trace_counts / _pack_traces /
    _apply_traces / _advance / _pack_owned) with 2-4 plans on cuda:0 and the
    exchange done in process: bitwise equal to the single-plan solve."""
    from paper_2006_14602_b200.distributed import InProcessShards
    if name == "C1":
        g = P.build_grid(2, ((0.0, 1.0),) * 2, (65, 65))
        d = P.build_decomposition(g, (2, 2), 4)
        m = P.density_monitor(P.RingDensity(), g.extents)
        windows = 12
    else:
        g = P.build_grid(3, ((0.0, 1.0),) * 3, (33, 33, 33))
        d = P.build_decomposition(g, (2, 2, 2), 4)
        m = P.density_monitor(P.ShellDensity(), g.extents)
        windows = 6
    cfg = P.SolverConfig(tol=1e-300, max_windows=windows, transmission="parallel")
    ref = P.solve(g, d, m, cfg)
    sh = InProcessShards(g, d, m, cfg, rank_of)
    sh.set_state(None)
    for _ in range(windows):
        sh.window()
    psi, coords, jac = (t.cpu().numpy() for t in sh.assemble())
    assert np.array_equal(psi, ref.psi)
    assert np.array_equal(coords, ref.mesh.coords)
    assert np.array_equal(jac, ref.mesh.jac)
    assert np.array_equal(np.array([h[0] for h in sh.history]),
                          np.array([h.residuals for h in ref.history]))
    assert np.array_equal(sh.sub_evals(), ref.stats["sub_rhs_evals"])
    assert sh.node_updates() == ref.stats["node_updates"]
