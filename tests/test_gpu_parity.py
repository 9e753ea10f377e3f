"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference's golden fixtures.  Run on a B200 with ``pytest -m gpu``.

Tolerances (north_star): node coordinates within max-abs 1e-10 relative to
the domain size at a fixed window count; index ranges and node ordering
bit-exact.  Pure-arithmetic operator outputs (Hessian determinant, mesh
coordinates) must be bitwise identical; values through log/exp agree to a
few ulp (CUDA's fp64 log/exp vs numpy's differ by <= 1 ulp).
"""

import numpy as np
import pytest

import ddpma_oracle as O
import recipes as R
from conftest import golden

import paper_2006_14602_b200 as P
from paper_2006_14602_b200 import pma as G
from paper_2006_14602_b200.plan import Plan

pytestmark = pytest.mark.gpu

COORD_TOL = 1e-10          # max-abs, domain size 1 (north_star)


def rel_close(a, b, rtol):
    a, b = np.asarray(a), np.asarray(b)
    scale = np.maximum(np.abs(b), 1.0)
    return float(np.max(np.where(a == b, 0.0, np.abs(a - b) / scale))) <= rtol


def ring_case():
    g = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65))
    d = P.build_decomposition(g, (2, 2), 4)
    m = P.density_monitor(P.RingDensity(), g.extents)
    return g, d, m


def baseline(name):
    og, lay, ov, omon, dom, win = O.baseline_case(name)
    g = P.build_grid(og.dim, og.extents, og.counts)
    d = P.build_decomposition(g, lay, ov)
    if isinstance(omon, O.Mixture):
        raw = P.MixtureDensity(omon.c, omon.s, omon.a)
    else:
        raw = P.RingDensity(omon.center, omon.amp, omon.sharp, omon.r2)
    return og, g, d, P.density_monitor(raw, g.extents), lay, raw


# ------------------------------------------------------------ operators ----

@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_rhs_operator_parity(name):
    og, g, d, mon, lay, raw = baseline(name)
    for sid in R.rhs_case_subs(lay):
        sub = d.subdomains[sid]
        geom = P.subdomain_geometry(g, sub)
        ogeom = O.box_geom(og, O.make_decomposition(og, lay, d.overlap).subs[sid])
        psi = R.perturbed_global(geom.axes)
        # oracle
        ocoords = np.stack(O.coords_fd(psi, ogeom), axis=-1)
        oraw = raw(np.clip(ocoords, 0.0, 1.0))
        rho = oraw / R.RHS_Z
        rmax = float(rho.max())
        oF, oflag = O.rhs_frozen(psi, rho, ogeom, O.DET_FLOOR, ogeom.mask(), rmax)
        odet = O.hess_det(psi, ogeom)
        # device
        mesh = G.physical_mesh(psi, geom)
        assert np.array_equal(mesh.jac, odet), (name, sid, "det bitwise")
        assert np.array_equal(mesh.coords, ocoords), (name, sid, "coords bitwise")
        draw = G.mesh_density(mon, psi, geom)
        assert rel_close(draw, oraw, 4e-16 * 8), (name, sid, "raw")
        F, flag = G.pma_rhs_frozen(psi, rho, geom, max_rho=rmax)
        assert flag == oflag
        assert rel_close(F, oF, 1e-14), (name, sid, "F")
        # golden pin of the same case
        gold = golden(f"rhs_{name}.npz")
        assert R.digest(mesh.jac) == str(gold[f"s{sid}_det_sha"])


def test_rkc_step_parity():
    g, d, mon = ring_case()
    og = O.make_grid(2, ((0, 1), (0, 1)), (65, 65))
    od = O.make_decomposition(og, (2, 2), 4)
    for sid in (0, 3):
        geom = P.subdomain_geometry(g, d.subdomains[sid])
        ogeom = O.box_geom(og, od.subs[sid])
        y = R.perturbed_global(geom.axes)
        coords = np.stack(O.coords_fd(y, ogeom), axis=-1)
        rho = O.Ring()(np.clip(coords, 0, 1)) / 1.3
        rmax = float(rho.max())
        fn = lambda v: O.rhs_frozen(v, rho, ogeom, O.DET_FLOOR, ogeom.mask(), rmax)
        f0, _ = fn(y)
        integ = O.Rkc2(1e-3)
        for h, s in ((1e-5, 2), (3e-5, 3), (2e-4, 9), (5e-4, 17)):
            od_, ofn, ofl, oend = integ._step(y, f0, h, s, fn)
            with Plan.for_geometry(geom, P.SolverConfig()) as p:
                dd, fnew, fl, end = p.rkc_step(0, y, rho, rmax, h, s)
            assert (fl, end) == (ofl, oend)
            assert rel_close(dd, od_, 1e-12), (sid, h, s)
            assert rel_close(fnew, ofn, 1e-12), (sid, h, s)


def test_rkc_coeffs_bitwise():
    for s in (2, 3, 7, 23, 100, 512):
        got = P.rkc_coeffs(s)
        ref = O.rkc_coeffs(s)
        for a, b in zip(got, ref):
            assert np.array_equal(np.asarray(a), np.asarray(b)), s


def test_residual_operator():
    g, d, _ = ring_case()
    geom = P.subdomain_geometry(g, d.subdomains[1])
    a = R.perturbed_global(geom.axes)
    b = R.perturbed_global(geom.axes, eps=0.3)
    assert rel_close(P.residual(a, b, geom), O.l2_norm(a - b, geom.spacing), 1e-13)


# ---------------------------------------------------------- trajectories ---

def envelope(tag):
    """Spread of the reference itself under 1-ulp log noise (tests/golden/env_*,
    make_golden.py gen_envelopes) — None for converged runs."""
    import os
    from conftest import GOLDEN
    path = os.path.join(GOLDEN, f"env_{tag}.npz")
    return golden(f"env_{tag}.npz") if os.path.exists(path) else None


def check_run(res, gold, tag=None, coord_tol=COORD_TOL):
    """Trajectory parity at a fixed window count.

    Converged runs (no envelope): coordinates within 1e-10 of the reference
    (north_star), psi within 1e-10 up to its free additive constant.
    Transient runs: the reference is chaotically sensitive to 1-ulp changes
    of np.log (positivity-flag decisions flip), so the
    device must stay within a small multiple of the reference's own spread
    under such perturbations — and within 1e-10 wherever that spread is
    below it (3D shell, Euler)."""
    env = envelope(tag) if tag else None
    assert res.windows == int(gold["windows"])
    assert res.converged == bool(gold["converged"])
    hr = np.array([h.residuals for h in res.history])
    if env is not None and float(env["coords"]) > 1e-6:
        # chaotic at the reference's own 1-ulp level (it tangles irrecoverably in
        # some perturbed realizations).  Accept the run if its deterministic
        # prefix matches, or if the whole trajectory lies within the reference's
        # own spread under one-ulp perturbations (runs tangled from window 0).
        k = min(3, len(hr))
        # prefix tolerance: 1e-9, or 4x the reference's own 1-ulp spread over
        # that prefix where it is larger (warm start: flagged from window 0)
        penv = golden("env_prefix3_C1.npz")
        pkey = tag[:-4] if tag.endswith("_100") else tag
        p_rtol = max(1e-9, 4.0 * float(penv[pkey + "_res_rel"])) if pkey + "_res_rel" in penv else 1e-9
        prefix_ok = rel_close(hr[:k], gold["residuals"][:k], p_rtol)
        if "coords" in gold:
            dc = np.max(np.abs(res.mesh.coords - gold["coords"]))
        else:
            flat = res.mesh.coords.reshape(res.psi.size, -1)[gold["coords_idx"]]
            dc = np.max(np.abs(flat - gold["coords_smp"]))
        spread_ok = dc <= 20.0 * float(env["coords"])
        print(f"[parity] {tag}: chaotic reference; prefix({k}) match={prefix_ok}, "
              f"max|dcoords|={dc:.3g} vs reference spread {float(env['coords']):.3g}")
        # the final mesh must lie within the reference's own one-ulp spread;
        # C1 runs also have a deterministic prefix (coordinates of that
        # prefix are pinned at 1e-10 by test_c1_prefix_coords)
        assert spread_ok, (dc, float(env["coords"]))
        if tag.startswith("C1"):
            assert prefix_ok
        return
    n_ref = int(gold["node_updates"])
    n_rel = abs(res.stats["node_updates"] - n_ref) / n_ref
    # node-update count = the adaptive decision sequence: exact where the
    # reference is not chaotic (its 1-ulp envelope is 0), else within a
    # multiple of that envelope; chaotic (tangling) runs only report it
    if env is None:
        n_tol = 0.05
    elif float(env["nodes_rel"]) == 0.0:
        n_tol = 0.0
    elif float(env["coords"]) > 1e-6:
        n_tol = np.inf
    else:
        n_tol = 10.0 * float(env["nodes_rel"])
    assert n_rel <= n_tol + 1e-12, (res.stats["node_updates"], n_ref, n_tol)
    c_tol = coord_tol if env is None else max(coord_tol, 20.0 * float(env["coords"]))
    p_tol = coord_tol if env is None else max(coord_tol, 20.0 * float(env["psi_centered"]))
    if "coords" in gold:
        dc = np.max(np.abs(res.mesh.coords - gold["coords"]))
        dp = res.psi - gold["psi"]
        dpc = np.max(np.abs(dp - dp.mean()))
    else:
        idx = gold["coords_idx"]
        flat = res.mesh.coords.reshape(res.psi.size, -1)[idx]
        dc = np.max(np.abs(flat - gold["coords_smp"]))
        dp = res.psi.reshape(-1)[gold["psi_idx"]] - gold["psi_smp"]
        dpc = np.max(np.abs(dp - dp.mean()))
    print(f"[parity] {tag}: max|dcoords|={dc:.3g} (tol {c_tol:.3g}) "
          f"max|dpsi-const|={dpc:.3g} nodes_rel={n_rel:.3g}")
    assert dc <= c_tol, (dc, c_tol)
    assert dpc <= p_tol, (dpc, p_tol)
    hr = np.array([h.residuals for h in res.history])
    assert hr.shape == gold["residuals"].shape
    r_tol = 1e-6 if env is None else max(1e-6, 20.0 * float(env["res_rel"]))
    # the last window's residual is the stop quantity
    assert rel_close(hr[-1], gold["residuals"][-1], r_tol)


@pytest.mark.parametrize("tr", ["parallel", "alternating"])
def test_c1_default_prefix(tr):
    """C1 parallel transmission at the reference defaults is chaotic: one-ulp
    perturbations of np.log send the reference itself into an irrecoverable
    tangle in 3 of 6 trials by window ~12 (Parity).  Before the first
    positivity-flag event the trajectory is deterministic to ulps: the first
    windows must agree with the reference to 1e-10."""
    g, d, m = ring_case()
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=3, transmission=tr))
    gold = golden(f"run_C1_{tr}_100.npz")
    hr = np.array([h.residuals for h in res.history])
    assert rel_close(hr, gold["residuals"][:3], 1e-9)
    assert np.allclose([h.jac_min for h in res.history], gold["jac_min"][:3], rtol=1e-9)


@pytest.mark.parametrize("tr,nwin,prof", [("alternating", 2000, "stable"),
                                          ("parallel", 2000, "stable")])
def test_c1_trajectory(tr, nwin, prof):
    g, d, m = ring_case()
    kw = dict(rtol=1e-6, atol=1e-9) if prof == "stable" else {}
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=nwin, transmission=tr, **kw))
    tag = f"C1_{tr}_{nwin}" if prof == "default" else f"C1_{tr}_stable_{nwin}"
    gold = golden(f"run_{tag}.npz")
    check_run(res, gold, tag)
    env = envelope(tag)
    tol = COORD_TOL if env is None else 20.0 * float(env["psi"])
    for i, sp in enumerate(res.sub_psi):
        d = sp - gold[f"sub_psi{i}"]
        assert np.max(np.abs(d - d.mean())) <= tol
    if env is None:
        assert abs(res.overlap_gap - float(gold["overlap_gap"])) <= 1e-9


@pytest.mark.parametrize("nwin,prof", [(100, "default"), (2000, "stable")])
def test_c1_single_domain(nwin, prof):
    g, _, m = ring_case()
    kw = dict(rtol=1e-6, atol=1e-9) if prof == "stable" else {}
    res = P.solve_single_domain(g, m, P.SolverConfig(tol=1e-300, max_windows=nwin, **kw))
    tag = f"C1_single_{nwin}" if prof == "default" else f"C1_single_stable_{nwin}"
    check_run(res, golden(f"run_{tag}.npz"), tag)


def test_one_by_one_equals_single_domain_bitwise():
    g, _, m = ring_case()
    cfg = P.SolverConfig(tol=1e-300, max_windows=50)
    a = P.solve_single_domain(g, m, cfg)
    b = P.solve(g, P.build_decomposition(g, (1, 1), 3), m, cfg)
    assert np.array_equal(a.psi, b.psi) and np.array_equal(a.mesh.coords, b.mesh.coords)


def test_deterministic_rerun_bitwise():
    g, d, m = ring_case()
    cfg = P.SolverConfig(tol=1e-300, max_windows=30, transmission="parallel")
    a = P.solve(g, d, m, cfg)
    b = P.solve(g, d, m, cfg)
    assert np.array_equal(a.psi, b.psi) and np.array_equal(a.mesh.jac, b.mesh.jac)


@pytest.mark.parametrize("tag,kw,init", [
    ("C1_euler", dict(max_windows=20, transmission="parallel", scheme="euler", substeps=3,
                      dtau=1e-5), False),
    ("C1_stable", dict(max_windows=40, transmission="parallel", rtol=1e-6, atol=1e-9), False),
    ("C1_cap8", dict(max_windows=40, transmission="alternating", max_stages=8), False),
    ("C1_warm", dict(max_windows=30, transmission="parallel"), True),
])
def test_c1_variants(tag, kw, init):
    g, d, m = ring_case()
    initial = R.perturbed_global(g.axes()) if init else None
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, **kw), initial=initial)
    check_run(res, golden(f"run_{tag}.npz"), tag)


def test_c1_slab4():
    g, _, m = ring_case()
    d = P.build_decomposition(g, (4, 1), 3)
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=60, transmission="parallel"))
    check_run(res, golden("run_C1_slab4.npz"), "C1_slab4")


@pytest.mark.parametrize("rule", ["min", "max"])
def test_c1_stop_rule(rule):
    g, d, m = ring_case()
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-7, transmission="parallel", stop_rule=rule,
                                          rtol=1e-6, atol=1e-9))
    gold = golden(f"run_C1_stabletol_{rule}.npz")
    assert res.converged
    # the crossing window of tol=1e-7 moves under ulp noise (chaotic transient)
    assert abs(res.windows - int(gold["windows"])) <= max(2, 0.05 * int(gold["windows"]))
    assert res.final_residual <= 1e-7


@pytest.mark.parametrize("tr", ["parallel", "alternating"])
def test_uniform_monitor_exact(tr):
    g, d, _ = ring_case()
    m = P.density_monitor(P.UniformDensity(1.0), g.extents)
    res = P.solve(g, d, m, P.SolverConfig(transmission=tr))
    gold = golden(f"run_U2_{tr}.npz")
    assert res.windows == 1 and res.final_residual == 0.0 and res.converged
    assert np.array_equal(res.psi, gold["psi"])
    assert np.array_equal(res.mesh.coords, gold["coords"])


def test_uniform_monitor_exact_3d():
    g = P.build_grid(3, ((0.0, 1.0),) * 3, (33, 33, 33))
    d = P.build_decomposition(g, (2, 2, 2), 4)
    m = P.density_monitor(P.UniformDensity(1.0), g.extents)
    res = P.solve(g, d, m, P.SolverConfig(transmission="parallel"))
    gold = golden("run_U3_parallel.npz")
    assert res.windows == 1 and res.final_residual == 0.0
    assert np.array_equal(res.mesh.coords, gold["coords"])


@pytest.mark.parametrize("tr", ["parallel", "alternating"])
def test_t3_3d_trajectory(tr):
    g = P.build_grid(3, ((0.0, 1.0),) * 3, (33, 33, 33))
    d = P.build_decomposition(g, (2, 2, 2), 4)
    m = P.density_monitor(P.ShellDensity(), g.extents)
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=40, transmission=tr))
    check_run(res, golden(f"run_T3_{tr}.npz"), f"T3_{tr}")


def test_t3_single():
    g = P.build_grid(3, ((0.0, 1.0),) * 3, (33, 33, 33))
    m = P.density_monitor(P.ShellDensity(), g.extents)
    res = P.solve_single_domain(g, m, P.SolverConfig(tol=1e-300, max_windows=40))
    check_run(res, golden("run_T3_single.npz"), "T3_single")


def test_error_paths():
    g, d, _ = ring_case()
    neg = P.density_monitor(P.RingDensity(amp=-20.0), g.extents)
    with pytest.raises(P.InvalidMonitorError):
        P.solve(g, d, neg, P.SolverConfig(tol=1e-300, max_windows=3, transmission="parallel"))
    half = P.density_monitor(P.RingDensity(amp=-1.5), g.extents)
    with pytest.raises(ValueError) as ei:
        P.solve(g, d, half, P.SolverConfig(tol=1e-300, max_windows=3, transmission="parallel"))
    assert str(ei.value) == str(golden("run_E_stiff.npz")["message"])


def test_non_native_monitor_rejected():
    g, d, _ = ring_case()
    m = P.density_monitor(lambda p: np.ones(p.shape[:-1]), g.extents)
    with pytest.raises(P.ConfigurationError):
        P.solve(g, d, m, P.SolverConfig(max_windows=1))


@pytest.mark.slow
def test_c2_two_windows():
    og, g, d, m, lay, raw = baseline("C2")
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=2, transmission="parallel"))
    check_run(res, golden("run_C2_parallel_2.npz"), "C2_parallel_2")


@pytest.mark.slow
def test_c4_one_window():
    og, g, d, m, lay, raw = baseline("C4")
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=1, transmission="parallel"))
    check_run(res, golden("run_C4_parallel_1.npz"), "C4_parallel_1")


# ------------------------------------------- BASELINE configs as benched ---

@pytest.mark.parametrize("tr", ["parallel", "alternating"])
def test_c1_reference_defaults_2000(tr):
    """BASELINE config 1 literally: 65^2, 2x2, overlap 4, ring monitor, the
    reference defaults, 2000 windows.  The reference converges there (final
    residuals ~5e-17); the converged mesh is the steady state of the DD
    iteration, so coordinates must agree to 1e-10 even though the transient
    is chaotic at the ulp level (the node-update count is reported, not
    pinned)."""
    g, d, m = ring_case()
    res = P.solve(g, d, m, P.SolverConfig(tol=1e-300, max_windows=2000, transmission=tr))
    gold = golden(f"run_C1_{tr}_2000.npz")
    assert res.windows == 2000
    dc = float(np.max(np.abs(res.mesh.coords - gold["coords"])))
    dp = res.psi - gold["psi"]
    dpc = float(np.max(np.abs(dp - dp.mean())))
    nrel = res.stats["node_updates"] / int(gold["node_updates"]) - 1.0
    print(f"[parity] C1 defaults {tr} x2000: max|dcoords|={dc:.3g} max|dpsi-const|={dpc:.3g} "
          f"final residual {res.final_residual:.3g} (ref {float(gold['final_residual']):.3g}) "
          f"node-updates {res.stats['node_updates']} vs ref {int(gold['node_updates'])} ({nrel:+.3%})")
    assert float(np.max(res.history[-1].residuals)) < 1e-12
    assert dc <= COORD_TOL, dc
    assert dpc <= COORD_TOL, dpc
    assert np.max(np.abs(res.mesh.jac - gold["jac"])) <= 1e-8
    for i, sp in enumerate(res.sub_psi):
        ds = sp - gold[f"sub_psi{i}"] if f"sub_psi{i}" in gold else None
        if ds is not None:
            assert np.max(np.abs(ds - ds.mean())) <= COORD_TOL
    assert abs(res.overlap_gap - float(gold["overlap_gap"])) <= 1e-10


@pytest.mark.parametrize("tag", ["C1_parallel", "C1_alternating", "C1_single", "C1_warm",
                                 "C1_cap8", "C1_slab4"])
def test_c1_prefix_coords(tag):
    """The default-profile C1 variants whose long runs are chaotic: their
    first 3 windows are deterministic, so full coordinates and psi after 3
    windows are pinned at 1e-10 against the reference (make_golden.py
    gen_prefix), and so is the adaptive decision sequence (node-updates)."""
    gold = golden("prefix3_C1.npz")
    g, d, m = ring_case()
    cfg = dict(tol=1e-300, max_windows=3)
    initial = None
    if tag == "C1_single":
        res = P.solve_single_domain(g, m, P.SolverConfig(**cfg))
    else:
        if tag == "C1_slab4":
            d = P.build_decomposition(g, (4, 1), 3)
        if tag == "C1_warm":
            initial = R.perturbed_global(g.axes())
        cfg["transmission"] = "alternating" if tag in ("C1_alternating", "C1_cap8") else "parallel"
        if tag == "C1_cap8":
            cfg["max_stages"] = 8
        res = P.solve(g, d, m, P.SolverConfig(**cfg), initial=initial)
    dc = float(np.max(np.abs(res.mesh.coords - gold[tag + "_coords"])))
    dp = res.psi - gold[tag + "_psi"]
    dpc = float(np.max(np.abs(dp - dp.mean())))
    # The reference's own spread over this prefix when np.log is perturbed by
    # one ulp (make_golden.py gen_prefix_envelopes): ~1e-11 for the cold
    # starts, 6e-10 with max_stages=8, 1e-2 for the warm start (flagged from
    # window 0).  Tolerance: 1e-10, or 4x that spread where it is larger.
    env = golden("env_prefix3_C1.npz")
    c_tol = max(COORD_TOL, 4.0 * float(env[tag + "_coords"]))
    p_tol = max(COORD_TOL, 4.0 * float(env[tag + "_psi_centered"]))
    r_tol = max(1e-9, 4.0 * float(env[tag + "_res_rel"]))
    n_ref = int(gold[tag + "_node_updates"])
    n_rel = abs(res.stats["node_updates"] - n_ref) / n_ref
    hr = np.array([h.residuals for h in res.history])
    gr = gold[tag + "_residuals"]
    rr = float(np.max(np.abs(hr - gr) / np.abs(gr)))
    print(f"[parity] {tag} prefix 3: max|dcoords|={dc:.3g} (tol {c_tol:.3g}) "
          f"max|dpsi-const|={dpc:.3g} (tol {p_tol:.3g}) residual rel {rr:.3g} (tol {r_tol:.3g}) "
          f"node-updates rel {n_rel:.3g}")
    assert n_rel <= 4.0 * float(env[tag + "_nodes_rel"])   # exact where the reference's spread is 0
    assert rr <= r_tol
    assert dc <= c_tol and dpc <= p_tol


def _window_case(name):
    gold = golden(f"win_{name}.npz")
    og, g, d, mon, lay, raw = baseline(name)
    cfg = P.SolverConfig(tol=1e-300, max_windows=1, transmission="parallel",
                         dtau=float(gold["dtau"]))
    return gold, g, d, mon, cfg


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_baseline_window_parity(name):
    """One full window of the benched BASELINE configs (all 64 subdomains,
    reference defaults, reduced window length so the reference finishes on a
    CPU; make_golden.py gen_windows).  Pins every subdomain's adaptive
    decision sequence (RHS-evaluation count), the per-subdomain residuals,
    and sampled coordinates / psi / sub_psi at 1e-10."""
    gold, g, d, mon, cfg = _window_case(name)
    res = P.solve(g, d, mon, cfg)
    evals = np.asarray(res.stats["sub_rhs_evals"])
    assert np.array_equal(evals, gold["sub_rhs_calls"]), (evals, gold["sub_rhs_calls"])
    assert res.stats["node_updates"] == int(gold["node_updates"])
    hr = np.array([h.residuals for h in res.history])
    assert rel_close(hr, gold["residuals"], 1e-9)
    flat = res.mesh.coords.reshape(res.psi.size, -1)[gold["coords_idx"]]
    dc = float(np.max(np.abs(flat - gold["coords_smp"])))
    dp = res.psi.reshape(-1)[gold["psi_idx"]] - gold["psi_smp"]
    dpc = float(np.max(np.abs(dp - dp.mean())))
    dsub = 0.0
    for i, sp in enumerate(res.sub_psi):
        ds = sp.reshape(-1)[gold[f"sub{i}_idx"]] - gold[f"sub{i}_smp"]
        dsub = max(dsub, float(np.max(np.abs(ds))))
    dj = float(np.max(np.abs(res.mesh.jac.reshape(-1)[gold["jac_idx"]] - gold["jac_smp"])
                      / np.maximum(1.0, np.abs(gold["jac_smp"]))))
    print(f"[parity] {name} window dtau={float(gold['dtau'])}: max|dcoords|={dc:.3g} "
          f"max|dpsi-const|={dpc:.3g} max|dsub_psi|={dsub:.3g} jac rel {dj:.3g} "
          f"jac_min {res.history[0].jac_min:.6g} (ref {float(gold['jac_min'][0]):.6g})")
    assert dc <= COORD_TOL and dpc <= COORD_TOL and dsub <= COORD_TOL
    assert rel_close([res.history[0].jac_min, res.history[0].jac_max],
                     [float(gold["jac_min"][0]), float(gold["jac_max"][0])], 1e-6)


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_baseline_rerun_bitwise(name):
    """Two windows of C3 / C5 run twice: psi, Jacobian and every subdomain's
    RHS-evaluation count bitwise identical (deterministic fixed-order
    reductions, scheduling-independent results)."""
    gold, g, d, mon, cfg = _window_case(name)
    import dataclasses
    cfg = dataclasses.replace(cfg, max_windows=2)
    a = P.solve(g, d, mon, cfg)
    b = P.solve(g, d, mon, cfg)
    assert np.array_equal(a.stats["sub_rhs_evals"], b.stats["sub_rhs_evals"])
    assert np.array_equal(a.psi, b.psi)
    assert np.array_equal(a.mesh.jac, b.mesh.jac)
    assert all(np.array_equal(x, y) for x, y in zip(a.sub_psi, b.sub_psi))


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_rkc_step_baseline_boxes(name):
    """One RKC2 step (ddpma_rkc_step) on real C3 / C5 subdomain boxes (first,
    interior, last) against the oracle's _rkc_step (integrate.py:163-178)."""
    og, g, d, mon, lay, raw = baseline(name)
    od = O.make_decomposition(og, lay, d.overlap)
    steps = ((2e-9, 3), (1e-8, 9)) if name == "C3" else ((1e-7, 3), (5e-7, 5))
    for sid in R.rhs_case_subs(lay):
        geom = P.subdomain_geometry(g, d.subdomains[sid])
        ogeom = O.box_geom(og, od.subs[sid])
        y = R.perturbed_global(geom.axes)
        coords = np.stack(O.coords_fd(y, ogeom), axis=-1)
        rho = raw(np.clip(coords, 0.0, 1.0)) / R.RHS_Z
        rmax = float(rho.max())
        mask = ogeom.mask()
        fn = lambda v: O.rhs_frozen(v, rho, ogeom, O.DET_FLOOR, mask, rmax)
        f0, _ = fn(y)
        integ = O.Rkc2(1e-3)
        with Plan.for_geometry(geom, P.SolverConfig()) as p:
            for h, s in steps:
                od_, ofn, ofl, oend = integ._step(y, f0, h, s, fn)
                dd, fnew, fl, end = p.rkc_step(0, y, rho, rmax, h, s)
                assert (fl, end) == (ofl, oend), (name, sid, h, s)
                # relative to the field's scale (d_s ~ h*F is small)
                ed = float(np.max(np.abs(dd - od_))) / float(np.max(np.abs(od_)))
                ef = float(np.max(np.abs(fnew - ofn))) / float(np.max(np.abs(ofn)))
                print(f"[parity] rkc_step {name} box {sid} h={h} s={s}: d rel {ed:.3g}, f rel {ef:.3g}")
                assert ed <= 1e-12 and ef <= 1e-12, (name, sid, h, s, ed, ef)


@pytest.mark.parametrize("name,nwin", [("C2", 2), ("T3x3", 3)])
def test_alternating_wavefront_equals_serial(name, nwin, monkeypatch):
    """alternating_sweep (schwarz.py:216-233) visits subdomains in id order.
    The device runs the independent subdomains of one wavefront level in one
    window-kernel launch; DDPMA_ALT_SERIAL=1 is the literal one-by-one loop.
    Both must give bitwise identical states and RHS-evaluation counts."""
    if name == "C2":
        og, g, d, mon, lay, raw = baseline("C2")
    else:
        g = P.build_grid(3, ((0.0, 1.0),) * 3, (49, 49, 49))
        d = P.build_decomposition(g, (3, 3, 3), 3)
        mon = P.density_monitor(P.ShellDensity(), g.extents)
    cfg = P.SolverConfig(tol=1e-300, max_windows=nwin, transmission="alternating")
    monkeypatch.delenv("DDPMA_ALT_SERIAL", raising=False)
    a = P.solve(g, d, mon, cfg)
    monkeypatch.setenv("DDPMA_ALT_SERIAL", "1")
    b = P.solve(g, d, mon, cfg)
    assert np.array_equal(a.stats["sub_rhs_evals"], b.stats["sub_rhs_evals"])
    assert np.array_equal(a.psi, b.psi)
    assert np.array_equal(a.mesh.coords, b.mesh.coords)
    assert all(np.array_equal(x, y) for x, y in zip(a.sub_psi, b.sub_psi))


@pytest.mark.parametrize("case", ["huge_det", "tiny_det", "deep_saturation", "nan_node"])
def test_rkc_step_extreme_values(case):
    """The window kernel's two-node log-equidistribution (logequi_pair) takes
    a straight-line path when every operand is in range and logequi() itself
    otherwise: determinants beyond the 1e+-290 range of the reciprocal-multiply
    quotient, a saturation denominator beyond 2^100, a NaN.  One RKC2 step on a
    C1 box with such nodes planted, against the oracle (integrate.py:163-178,
    pma.py:186-192): same flags, same values (NaN where the oracle has NaN)."""
    g, d, mon = ring_case()
    og = O.make_grid(2, ((0, 1), (0, 1)), (65, 65))
    od = O.make_decomposition(og, (2, 2), 4)
    geom = P.subdomain_geometry(g, d.subdomains[0])
    ogeom = O.box_geom(og, od.subs[0])
    y = R.perturbed_global(geom.axes).copy()
    if case == "huge_det":          # |det| ~ 1e300: outside the Markstein range, true division
        y[12, 12] += 3e146
        y[20, 21] -= 2e147
    elif case == "tiny_det":        # det ~ 1e-300-scale products are not reachable; tiny positive det
        y[:] = 0.5 * (geom.axes[0][:, None] ** 2 + geom.axes[1][None, :] ** 2) * 1e-160
    elif case == "deep_saturation":  # det / guard ~ -1e40: saturation denominator > 2^100
        y[15, 15] += 1e18
        y[15, 16] -= 1e18
    else:
        y[9, 11] = np.nan
    coords = np.stack(O.coords_fd(np.nan_to_num(R.perturbed_global(geom.axes)), ogeom), axis=-1)
    rho = O.Ring()(np.clip(coords, 0, 1)) / 1.3
    rmax = float(rho.max())
    with np.errstate(all="ignore"):
        fn = lambda v: O.rhs_frozen(v, rho, ogeom, O.DET_FLOOR, ogeom.mask(), rmax)
        f0, _ = fn(y)
        od_, ofn, ofl, oend = O.Rkc2(1e-3)._step(y, f0, 1e-7, 3, fn)
    with Plan.for_geometry(geom, P.SolverConfig()) as p:
        dd, fnew, fl, end = p.rkc_step(0, y, rho, rmax, 1e-7, 3)
    assert (fl, end) == (ofl, oend), case
    for got, ref, name in ((dd, od_, "d"), (fnew, ofn, "f")):
        assert np.array_equal(np.isnan(got), np.isnan(ref)), (case, name)
        assert np.array_equal(np.isinf(got), np.isinf(ref)), (case, name)
        fin = np.isfinite(ref)
        assert np.array_equal(np.sign(got[~fin & ~np.isnan(ref)]), np.sign(ref[~fin & ~np.isnan(ref)]))
        scale = max(float(np.max(np.abs(ref[fin]))), 1e-300)
        err = float(np.max(np.abs(got[fin] - ref[fin]))) / scale
        print(f"[parity] rkc_step extreme {case} {name}: rel err {err:.3g}")
        assert err <= 1e-12, (case, name, err)
