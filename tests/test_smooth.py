"""Monitor smoothing and relaxation: SolverConfig
``monitor_smooth_passes`` / ``monitor_relax`` (ddmesh/schwarz.py:162-192,
:370-374; monitor._smooth ddmesh/monitor.py:395-409).

Golden fixtures: tests/golden/smooth.npz from the real reference
(tests/golden/make_smooth_golden.py).  CPU: the oracle restatement is
bitwise; GPU: the device path (k_rawfill / k_smooth / k_mesh blend) through
the public solve API.
"""

from __future__ import annotations

import numpy as np
import pytest

import ddpma_oracle as O
from conftest import golden

import paper_2006_14602_b200 as P

CASES = [
    ("ring_par_s2_r3", "ring", 2, (33, 33), (2, 2), 4, "parallel", 5, 2, 0.3),
    ("ring_alt_s1", "ring", 2, (33, 33), (2, 2), 4, "alternating", 5, 1, 0.0),
    ("ring_single_r5", "ring", 2, (33, 33), None, 0, "parallel", 5, 0, 0.5),
    ("shell_par_s1_r2", "ring", 3, (17, 17, 17), (2, 2, 2), 2, "parallel", 3, 1, 0.2),
    ("burgers_par_s2_r25", "burgers2d", 2, (33, 33), (2, 2), 4, "parallel", 4, 2, 0.25),
]
IDS = [c[0] for c in CASES]


@pytest.fixture(scope="module")
def gold():
    return golden("smooth.npz")


def _oracle_mon(name, dim):
    if name == "ring":
        m = O.Ring() if dim == 2 else O.Shell()
        return m, ((0.0, 1.0),) * dim
    a = O.ArcLength(name, eps=0.05)
    return a, a.domain


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_oracle_smooth_relax_bitwise(case, gold):
    tag, mname, dim, counts, layout, ov, tr, nwin, passes, relax = case
    mon, dom = _oracle_mon(mname, dim)
    g = O.make_grid(dim, dom, counts)
    cfg = O.Config(tol=1e-300, max_windows=nwin, transmission=tr, rtol=1e-6, atol=1e-9,
                   monitor_smooth_passes=passes, monitor_relax=relax)
    if layout is None:
        r = O.solve_single(g, mon, dom, cfg)
    else:
        r = O.solve(g, O.make_decomposition(g, layout, ov), mon, dom, cfg)
    assert np.array_equal(r.coords, gold[f"{tag}_coords"])
    assert np.array_equal(np.array(r.residuals), gold[f"{tag}_residuals"])
    assert r.counter.node_updates == int(gold[f"{tag}_node_updates"])


def test_oracle_quality_smoothed(gold):
    a = O.ArcLength("burgers2d", eps=0.05)
    g = O.make_grid(2, a.domain, (33, 33))
    e, e2, *_ = O.quality_measure(gold["burgers_par_s2_r25_psi"], a, a.domain, 1.0,
                                  O.whole_geom(g), sample_on_mesh=True, smooth_passes=2)
    assert np.array_equal(e, gold["quality_e"])
    assert e2 == float(gold["quality_e2"])


def _device_mon(name, dim):
    if name == "ring":
        raw = P.RingDensity() if dim == 2 else P.ShellDensity()
        return P.density_monitor(raw, ((0.0, 1.0),) * dim)
    return P.arc_length_monitor(P.test_function_registry(name, eps=0.05))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_device_smooth_relax(case, gold):
    tag, mname, dim, counts, layout, ov, tr, nwin, passes, relax = case
    mon = _device_mon(mname, dim)
    g = P.build_grid(dim, mon.domain, counts)
    cfg = P.SolverConfig(tol=1e-300, max_windows=nwin, transmission=tr, rtol=1e-6, atol=1e-9,
                         monitor_smooth_passes=passes, monitor_relax=relax)
    if layout is None:
        res = P.solve_single_domain(g, mon, cfg)
    else:
        res = P.solve(g, P.build_decomposition(g, layout, ov), mon, cfg)
    dc = float(np.max(np.abs(res.mesh.coords - gold[f"{tag}_coords"])))
    hr = np.array([h.residuals for h in res.history])
    ref = gold[f"{tag}_residuals"]
    rr = float(np.max(np.abs(hr - ref) / ref))
    n_ref = int(gold[f"{tag}_node_updates"])
    print(f"[smooth] {tag}: max|dcoords|={dc:.3g} residual rel={rr:.3g} "
          f"node-updates {res.stats['node_updates']} vs {n_ref}")
    assert res.stats["node_updates"] == n_ref
    assert dc <= 1e-10
    assert rr <= 1e-6


@pytest.mark.gpu
def test_device_quality_smoothed(gold):
    mon = _device_mon("burgers2d", 2)
    g = P.build_grid(2, mon.domain, (33, 33))
    q = P.quality_measure(gold["burgers_par_s2_r25_psi"], mon, g, sample_on_mesh=True,
                          smooth_passes=2)
    ref = gold["quality_e"]
    err = float(np.max(np.abs(q.e_adp - ref)) / np.max(np.abs(ref)))
    print(f"[smooth] quality(sample_on_mesh, smooth 2): e_adp rel {err:.3g}")
    assert err <= 1e-12
    assert abs(q.e2 - float(gold["quality_e2"])) <= 1e-12 * float(gold["quality_e2"])
