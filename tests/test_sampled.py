"""SampledField arc-length monitors (ddmesh/monitor.py:
361-444): lattice ingestion, the per-window pull-back of u interpolated at
the mesh nodes on the device, normalize, and short solves.

Golden fixtures: tests/golden/sampled.npz + sampled2d.csv from the real
reference (tests/golden/make_sampled_golden.py)."""

from __future__ import annotations

import os

import numpy as np
import pytest

import ddpma_oracle as O
from conftest import GOLDEN, golden

import paper_2006_14602_b200 as P
from paper_2006_14602_b200 import pma as G

RUNS = [
    ("s2_par", 2, 1, (33, 33), (2, 2), 4, "parallel", 4),
    ("s2_single", 2, 0, (33, 33), None, 0, "parallel", 3),
    ("s3_par", 3, 0, (17, 17, 17), (2, 2, 2), 2, "parallel", 3),
]


@pytest.fixture(scope="module")
def gold():
    return golden("sampled.npz")


def _lattice(gold, dim):
    if dim == 2:
        return (gold["ax2_0"], gold["ax2_1"]), gold["u2"]
    return (gold["ax3_0"], gold["ax3_1"], gold["ax3_2"]), gold["u3"]


def _op_setup(gold, dim, mod):
    ax, u = _lattice(gold, dim)
    smooth = 1 if dim == 2 else 0
    counts = (33, 33) if dim == 2 else (17, 17, 17)
    return ax, u, smooth, counts, (2,) * dim, 4 if dim == 2 else 2


@pytest.mark.parametrize("dim", [2, 3])
def test_oracle_sampled_bitwise(dim, gold):
    ax, u, smooth, counts, layout, ov = _op_setup(gold, dim, O)
    s = O.Sampled(ax, u, smooth)
    g = O.make_grid(dim, s.domain, counts)
    d = O.make_decomposition(g, layout, ov)
    geom = O.box_geom(g, d.subs[-1])
    coords, _ = O.mesh_of(gold[f"op{dim}_psi"], geom)
    assert np.array_equal(s(O.clamp(coords, s.domain)), gold[f"op{dim}_analytic"])
    assert np.array_equal(O.mesh_density(s, coords, geom.spacing, s.domain), gold[f"op{dim}_pull"])


@pytest.mark.parametrize("case", RUNS, ids=[r[0] for r in RUNS])
def test_oracle_sampled_runs_bitwise(case, gold):
    tag, dim, smooth, counts, layout, ov, tr, nwin = case
    ax, u = _lattice(gold, dim)
    s = O.Sampled(ax, u, smooth)
    g = O.make_grid(dim, s.domain, counts)
    cfg = O.Config(tol=1e-300, max_windows=nwin, transmission=tr, rtol=1e-6, atol=1e-9)
    if layout is None:
        r = O.solve_single(g, s, s.domain, cfg)
    else:
        r = O.solve(g, O.make_decomposition(g, layout, ov), s, s.domain, cfg)
    assert np.array_equal(r.coords, gold[f"{tag}_coords"])
    assert r.counter.node_updates == int(gold[f"{tag}_node_updates"])


def test_sampled_field_api(gold):
    ax, u = _lattice(gold, 2)
    sf = P.SampledField(ax, u, smooth_passes=1)
    ref = O.Sampled(ax, u, 1)
    pts = np.random.default_rng(0).uniform(0.0, 1.0, (50, 2))
    assert np.array_equal(sf.u(pts), ref.u(pts))
    assert np.array_equal(sf.gradient(pts), ref.gradient(pts))
    mon = P.arc_length_monitor(sf)
    assert mon.u_fn == sf.u and mon.domain == ref.domain
    assert np.array_equal(mon.raw(pts), ref(pts))
    with pytest.raises(P.ConfigurationError):
        P.SampledField(ax, u[:-1])
    csv = P.sampled_field_from_csv(os.path.join(GOLDEN, "sampled2d.csv"), smooth_passes=1)
    assert np.array_equal(csv.values, gold["csv_values"])


def test_sampled_vtk_roundtrip(gold, tmp_path):
    ax, u = _lattice(gold, 3)
    P.write_scalar_field_vtk(ax, u, str(tmp_path / "u.vtk"))
    sf = P.sampled_field_from_vtk(str(tmp_path / "u.vtk"))
    assert np.array_equal(sf.values, u)
    assert all(np.array_equal(a, b) for a, b in zip(sf.axes, ax))


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
def test_device_sampled_density_and_normalize(dim, gold):
    ax, u, smooth, counts, layout, ov = _op_setup(gold, dim, P)
    sf = P.SampledField(ax, u, smooth_passes=smooth)
    mon = P.arc_length_monitor(sf)
    g = P.build_grid(dim, sf.domain, counts)
    d = P.build_decomposition(g, layout, ov)
    geom = P.subdomain_geometry(g, d.subdomains[-1])
    raw = G.mesh_density(mon, gold[f"op{dim}_psi"], geom)
    ref = gold[f"op{dim}_pull"]
    err = float(np.max(np.abs(raw - ref) / ref))
    nm = P.normalize(mon, g)
    z_ref, mx_ref = gold[f"norm{dim}"]
    print(f"[sampled] {dim}D pull-back rel {err:.3g}; normalize z {nm.normalizer!r} vs {z_ref!r}")
    assert err <= 1e-12
    assert abs(nm.normalizer - z_ref) <= 1e-12 * z_ref
    assert abs(nm.max_value - mx_ref) <= 1e-12 * mx_ref


@pytest.mark.gpu
@pytest.mark.parametrize("case", RUNS, ids=[r[0] for r in RUNS])
def test_device_sampled_solve(case, gold):
    tag, dim, smooth, counts, layout, ov, tr, nwin = case
    ax, u = _lattice(gold, dim)
    sf = P.SampledField(ax, u, smooth_passes=smooth)
    mon = P.arc_length_monitor(sf)
    g = P.build_grid(dim, sf.domain, counts)
    cfg = P.SolverConfig(tol=1e-300, max_windows=nwin, transmission=tr, rtol=1e-6, atol=1e-9)
    if layout is None:
        res = P.solve_single_domain(g, mon, cfg)
    else:
        res = P.solve(g, P.build_decomposition(g, layout, ov), mon, cfg)
    dc = float(np.max(np.abs(res.mesh.coords - gold[f"{tag}_coords"])))
    hr = np.array([h.residuals for h in res.history])
    rr = float(np.max(np.abs(hr - gold[f"{tag}_residuals"]) / gold[f"{tag}_residuals"]))
    n_ref = int(gold[f"{tag}_node_updates"])
    print(f"[sampled] {tag}: max|dcoords|={dc:.3g} residual rel={rr:.3g} "
          f"node-updates {res.stats['node_updates']} vs {n_ref}")
    assert res.stats["node_updates"] == n_ref
    assert dc <= 1e-10
    assert rr <= 1e-6
