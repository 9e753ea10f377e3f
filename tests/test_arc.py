"""Arc-length (u-backed) monitors: SURVEY §8(f) rank 1.

Golden fixtures: tests/golden/arc.npz from the real reference
(tests/golden/make_arc_golden.py).  CPU tests pin the oracle restatement
(bitwise) and the package's numpy API; GPU tests check the device pull-back
density (monitor.py:151-216) and short solves through the public API.
"""

from __future__ import annotations

import numpy as np
import pytest

import ddpma_oracle as O
from conftest import golden

import paper_2006_14602_b200 as P
from paper_2006_14602_b200 import pma as G

OP_CASES = [
    ("burgers2d", {"eps": 0.05}, 2, (33, 33), (2, 2), 4),
    ("spiral2d", {}, 2, (33, 33), (2, 2), 4),
    ("quasi1d_linear", {}, 2, (33, 33), (1, 2), 4),
    ("sphere3d", {}, 3, (17, 17, 17), (2, 2, 2), 2),
    ("nine_spheres3d", {}, 3, (17, 17, 17), (2, 2, 2), 2),
]

RUN_CASES = [
    ("burgers_par", "burgers2d", {"eps": 0.05}, 2, (33, 33), (2, 2), 4, "parallel", 4),
    ("spiral_alt", "spiral2d", {}, 2, (33, 33), (2, 2), 4, "alternating", 4),
    ("quasi1d_single", "quasi1d_linear", {}, 2, (33, 33), None, 0, "parallel", 4),
    ("sphere_par", "sphere3d", {}, 3, (17, 17, 17), (2, 2, 2), 2, "parallel", 3),
    ("nine_single", "nine_spheres3d", {}, 3, (17, 17, 17), None, 0, "parallel", 3),
    ("burgers_norm_par", "burgers2d:norm", {"eps": 0.05}, 2, (33, 33), (2, 2), 4, "parallel", 4),
]

NORM_CASES = [
    ("burgers2d", {"eps": 0.05}, (33, 33)),
    ("spiral2d", {}, (65, 65)),
    ("quasi1d_linear", {}, (17, 17)),
    ("sphere3d", {}, (17, 17, 17)),
    ("nine_spheres3d", {}, (33, 33, 33)),
]


@pytest.fixture(scope="module")
def gold():
    return golden("arc.npz")


def _oracle_box(name, params, dim, counts, layout, ov, sub_id):
    mon = O.ArcLength(name, **params)
    g = O.make_grid(dim, mon.domain, counts)
    d = O.make_decomposition(g, layout, ov)
    return mon, O.box_geom(g, d.subs[sub_id])


@pytest.mark.parametrize("case", OP_CASES, ids=[c[0] for c in OP_CASES])
def test_oracle_pullback_bitwise(case, gold):
    name, params, dim, counts, layout, ov = case
    sub = int(gold[f"op_{name}_sub"])
    mon, geom = _oracle_box(name, params, dim, counts, layout, ov, sub)
    psi = gold[f"op_{name}_psi"]
    coords, _ = O.mesh_of(psi, geom)
    pts = O.clamp(coords, mon.domain)
    assert np.array_equal(mon(pts), gold[f"op_{name}_analytic"])
    assert np.array_equal(mon.u(pts), gold[f"op_{name}_u"])
    assert np.array_equal(O.mesh_density(mon, coords, geom.spacing, mon.domain),
                          gold[f"op_{name}_pull"])


@pytest.mark.parametrize("case", RUN_CASES, ids=[c[0] for c in RUN_CASES])
def test_oracle_runs_bitwise(case, gold):
    tag, name, params, dim, counts, layout, ov, tr, nwin = case
    norm = name.endswith(":norm")
    arc = O.ArcLength(name.split(":")[0], **params)
    # normalize() drops u_fn: the solver then samples the analytic raw
    mon = (lambda p: arc(p)) if norm else arc
    g = O.make_grid(dim, arc.domain, counts)
    cfg = O.Config(tol=1e-300, max_windows=nwin, transmission=tr, rtol=1e-6, atol=1e-9)
    if layout is None:
        r = O.solve_single(g, mon, arc.domain, cfg)
    else:
        r = O.solve(g, O.make_decomposition(g, layout, ov), mon, arc.domain, cfg)
    assert np.array_equal(r.coords, gold[f"run_{tag}_coords"])
    assert np.array_equal(np.array(r.residuals), gold[f"run_{tag}_residuals"])
    assert r.counter.node_updates == int(gold[f"run_{tag}_node_updates"])


def test_package_test_functions_match_reference(gold):
    """The package's numpy API (TestFunction.u, the arc-length raw) is the
    reference's formula: bitwise on the golden points."""
    for name, params, dim, counts, layout, ov in OP_CASES:
        sub = int(gold[f"op_{name}_sub"])
        omon, geom = _oracle_box(name, params, dim, counts, layout, ov, sub)
        coords, _ = O.mesh_of(gold[f"op_{name}_psi"], geom)
        pts = O.clamp(coords, omon.domain)
        tf = P.test_function_registry(name, **params)
        mon = P.arc_length_monitor(tf)
        assert mon.u_fn is tf.u and tf.domain == omon.domain
        assert np.array_equal(tf.u(pts), gold[f"op_{name}_u"])
        assert np.array_equal(mon.raw(pts), gold[f"op_{name}_analytic"])


def test_registry_errors():
    with pytest.raises(P.ConfigurationError):
        P.test_function_registry("nope")
    with pytest.raises(P.ConfigurationError):
        P.test_function_registry("burgers2d", eps=-1.0)
    with pytest.raises(P.ConfigurationError):
        P.test_function_registry("burgers2d", eps=0.1, zeta=2)
    with pytest.raises(P.ConfigurationError):
        P.test_function_registry("spiral2d", eps=0.1)
    assert P.test_function_registry("burgers2d").params == {"eps": 0.01}


def test_lowering_kinds():
    from paper_2006_14602_b200 import _lib
    from paper_2006_14602_b200.monitor import lower_monitor
    kinds = {"burgers2d": _lib.MON_BURGERS2D, "spiral2d": _lib.MON_SPIRAL2D,
             "sphere3d": _lib.MON_SPHERE3D, "nine_spheres3d": _lib.MON_NINE_SPHERES3D,
             "quasi1d_linear": _lib.MON_QUASI1D_LINEAR}
    for name, kind in kinds.items():
        tf = P.test_function_registry(name)
        nm = lower_monitor(P.arc_length_monitor(tf), len(tf.domain))
        assert nm.desc.kind == kind
    nm = lower_monitor(P.arc_length_monitor(P.test_function_registry("burgers2d", eps=0.25)), 2)
    assert nm.desc.eps == 0.25
    with pytest.raises(P.ConfigurationError):   # dimension mismatch
        lower_monitor(P.arc_length_monitor(P.test_function_registry("sphere3d")), 2)
    # a foreign u_fn (e.g. a sampled field) has no device form: loud error
    bad = P.MonitorField(raw=P.ArcLengthDensity("burgers2d"), domain=((0, 1), (0, 1)),
                         u_fn=lambda p: p[..., 0])
    with pytest.raises(P.ConfigurationError):
        lower_monitor(bad, 2)


# ------------------------------------------------------------------ GPU --

@pytest.mark.gpu
@pytest.mark.parametrize("case", OP_CASES, ids=[c[0] for c in OP_CASES])
def test_device_pullback_density(case, gold):
    name, params, dim, counts, layout, ov = case
    tf = P.test_function_registry(name, **params)
    mon = P.arc_length_monitor(tf)
    g = P.build_grid(dim, tf.domain, counts)
    d = P.build_decomposition(g, layout, ov)
    sub = d.subdomains[int(gold[f"op_{name}_sub"])]
    geom = P.subdomain_geometry(g, sub)
    raw = G.mesh_density(mon, gold[f"op_{name}_psi"], geom)
    ref = gold[f"op_{name}_pull"]
    err = float(np.max(np.abs(raw - ref) / np.abs(ref)))
    print(f"[arc] {name}: pull-back density max rel err {err:.3g}")
    assert err <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("case", RUN_CASES, ids=[c[0] for c in RUN_CASES])
def test_device_arc_solve(case, gold):
    tag, name, params, dim, counts, layout, ov, tr, nwin = case
    norm = name.endswith(":norm")
    tf = P.test_function_registry(name.split(":")[0], **params)
    mon = P.arc_length_monitor(tf)
    g = P.build_grid(dim, tf.domain, counts)
    if norm:
        mon = P.normalize(mon, g)
        assert mon.u_fn is None
    cfg = P.SolverConfig(tol=1e-300, max_windows=nwin, transmission=tr, rtol=1e-6, atol=1e-9)
    if layout is None:
        res = P.solve_single_domain(g, mon, cfg)
    else:
        res = P.solve(g, P.build_decomposition(g, layout, ov), mon, cfg)
    dc = float(np.max(np.abs(res.mesh.coords - gold[f"run_{tag}_coords"])))
    hr = np.array([h.residuals for h in res.history])
    rr = float(np.max(np.abs(hr - gold[f"run_{tag}_residuals"]) / gold[f"run_{tag}_residuals"]))
    n_ref = int(gold[f"run_{tag}_node_updates"])
    print(f"[arc] {tag}: max|dcoords|={dc:.3g} residual rel={rr:.3g} "
          f"node-updates {res.stats['node_updates']} vs {n_ref}")
    assert res.windows == nwin
    assert res.stats["node_updates"] == n_ref
    assert dc <= 1e-10
    assert rr <= 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("case", NORM_CASES, ids=[c[0] for c in NORM_CASES])
def test_device_normalize(case, gold):
    """normalize (monitor.py:123-148): converged probe quadrature on the device."""
    name, params, counts = case
    tf = P.test_function_registry(name, **params)
    g = P.build_grid(len(counts), tf.domain, counts)
    nm = P.normalize(P.arc_length_monitor(tf), g)
    z_ref, mx_ref = gold[f"norm_{name}"]
    print(f"[arc] normalize {name}: z {nm.normalizer!r} vs {z_ref!r}")
    assert abs(nm.normalizer - z_ref) <= 1e-12 * abs(z_ref)
    assert abs(nm.max_value - mx_ref) <= 1e-12 * abs(mx_ref)


@pytest.mark.gpu
def test_device_normalize_invalid():
    """A nonpositive density raises InvalidMonitorError (monitor.py:116-117)."""
    g = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (9, 9))
    m = P.density_monitor(P.UniformDensity(-1.0), g.extents)
    with pytest.raises(P.InvalidMonitorError):
        P.normalize(m, g)


@pytest.mark.gpu
@pytest.mark.parametrize("sample", [False, True])
def test_device_quality_arc(sample, gold):
    """quality_measure (metrics.py:57-85) with an arc-length monitor: the
    analytic raw / normaliser, or with sample_on_mesh the u pull-back
    (mesh_density) transport-normalised; against the oracle."""
    name, params = "burgers2d", {"eps": 0.05}
    tf = P.test_function_registry(name, **params)
    g = P.build_grid(2, tf.domain, (33, 33))
    psi = gold["run_burgers_par_psi"]
    mon = P.arc_length_monitor(tf)
    norm = float(gold[f"norm_{name}"][0])
    if not sample:
        mon = P.MonitorField(raw=mon.raw, domain=mon.domain, normalizer=norm)
    rep = P.quality_measure(psi, mon, g, sample_on_mesh=sample)
    arc = O.ArcLength(name, **params)
    og = O.make_grid(2, arc.domain, (33, 33))
    e, e2, emax, mean, tangled = O.quality_measure(psi, arc, arc.domain, norm, O.whole_geom(og),
                                                   sample_on_mesh=sample)
    err = float(np.max(np.abs(rep.e_adp - e)) / np.max(np.abs(e)))
    print(f"[arc] quality sample_on_mesh={sample}: e_adp rel {err:.3g}")
    assert err <= 1e-12
    assert abs(rep.e2 - e2) <= 1e-12 * abs(e2)
    assert rep.tangled == tangled


@pytest.mark.parametrize("case", OP_CASES, ids=[c[0] for c in OP_CASES])
def test_oracle_pma_rhs_bitwise(case, gold):
    """Moving-point pma_rhs (pma.py:152-183) = the frozen RHS with
    rho = raw(clamp(grad psi)) / normaliser and the max_value guard."""
    name, params, dim, counts, layout, ov = case
    mon, geom = _oracle_box(name, params, dim, counts, layout, ov, int(gold[f"op_{name}_sub"]))
    psi = gold[f"op_{name}_psi"]
    z, mx = gold[f"op_{name}_norm"]
    coords, _ = O.mesh_of(psi, geom)
    rho = mon(O.clamp(coords, mon.domain)) / z
    f, flag = O.rhs_frozen(psi, rho, geom, O.DET_FLOOR, geom.mask(), mx)
    assert np.array_equal(f, gold[f"op_{name}_pmarhs"])
    assert flag == bool(gold[f"op_{name}_pmarhs_flag"])


@pytest.mark.gpu
@pytest.mark.parametrize("case", OP_CASES, ids=[c[0] for c in OP_CASES])
def test_device_pma_rhs(case, gold):
    name, params, dim, counts, layout, ov = case
    tf = P.test_function_registry(name, **params)
    z, mx = gold[f"op_{name}_norm"]
    mon = P.MonitorField(raw=P.arc_length_monitor(tf).raw, domain=tf.domain, normalizer=float(z),
                         max_value=float(mx))
    g = P.build_grid(dim, tf.domain, counts)
    d = P.build_decomposition(g, layout, ov)
    geom = P.subdomain_geometry(g, d.subdomains[int(gold[f"op_{name}_sub"])])
    ev = P.pma_rhs(gold[f"op_{name}_psi"], mon, geom)
    ref = gold[f"op_{name}_pmarhs"]
    err = float(np.max(np.abs(ev.values - ref)))
    print(f"[arc] pma_rhs {name}: max abs err {err:.3g}")
    assert err <= 1e-12 * max(1.0, float(np.max(np.abs(ref))))
    assert ev.det_clamped == bool(gold[f"op_{name}_pmarhs_flag"])
