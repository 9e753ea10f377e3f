"""Host-side logic and the C ABI, without a GPU: libddpma.so loads and exports
every symbol include/ddpma.h declares; the native decomposition is bit-exact
with the reference's (golden) including its error messages; RKC2 tables are
bitwise the reference's; the Python mirror validates like the reference and
the compute path refuses to run without CUDA (no CPU fallback)."""

import json
import os
import re

import numpy as np
import pytest
import torch

import ddpma_oracle as O
from conftest import GOLDEN, REPO

import paper_2006_14602_b200 as P
from paper_2006_14602_b200 import _lib


def header_symbols():
    src = open(os.path.join(REPO, "include", "ddpma.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ddpma_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(L, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"


def test_library_is_in_tree_sm100a():
    assert os.path.dirname(_lib.LIB_PATH) == os.path.join(REPO, "paper_2006_14602_b200")
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob or b"sm_100" in blob


def _subs_json(d):
    return [{"id": s.id, "pos": list(s.pos), "box": [list(b) for b in s.box],
             "faces": [list(f) for f in s.faces],
             "neighbors": sorted([[k[0], k[1], v] for k, v in s.neighbors.items()]),
             "owned": [list(o) for o in s.owned]} for s in d.subdomains]


def test_native_decomposition_matches_reference_golden():
    cases = json.load(open(os.path.join(GOLDEN, "decomp.json")))
    for c in cases:
        if len(c["counts"]) != c["dim"]:
            with pytest.raises(P.ConfigurationError):
                P.build_grid(c["dim"], [(0.0, 1.0)] * len(c["counts"]), c["counts"])
            continue
        g = P.build_grid(c["dim"], [(0.0, 1.0)] * c["dim"], c["counts"])
        if "error" in c:
            with pytest.raises(P.ConfigurationError) as ei:
                P.build_decomposition(g, c["layout"], c["overlap"])
            assert str(ei.value) == c["message"]
        else:
            assert _subs_json(P.build_decomposition(g, c["layout"], c["overlap"])) == c["subs"]


@pytest.mark.parametrize("dim", [2, 3])
def test_native_decomposition_property_sweep(dim):
    """Bit-exact boxes/owned/faces/donors against the oracle restatement over
    a sweep of (n, parts, overlap), including rejections."""
    rng = np.random.default_rng(dim)
    for _ in range(150):
        counts = tuple(int(x) for x in rng.integers(3, 60, dim))
        layout = tuple(int(x) for x in rng.integers(1, 6, dim))
        ov = int(rng.integers(1, 12))
        og = O.make_grid(dim, [(0, 1)] * dim, counts)
        g = P.build_grid(dim, [(0.0, 1.0)] * dim, counts)
        try:
            od = O.make_decomposition(og, layout, ov)
        except O.OracleConfigError:
            with pytest.raises(P.ConfigurationError):
                P.build_decomposition(g, layout, ov)
            continue
        d = P.build_decomposition(g, layout, ov)
        for a, b in zip(d.subdomains, od.subs):
            assert (a.id, a.pos, a.box, a.faces, a.neighbors, a.owned) == \
                   (b.id, b.pos, b.box, b.faces, b.neighbors, b.owned)


@pytest.mark.parametrize("counts,layout,ov", [((65, 65), (2, 2), 4), ((513, 513), (4, 4), 8),
                                              ((257, 257), (8, 8), 4), ((65, 65), (4, 1), 3),
                                              ((65, 65, 65), (4, 4, 4), 3), ((33, 33, 33), (2, 3, 2), 2)])
def test_alternating_wavefront_levels(counts, layout, ov):
    """ddpma_alternating_levels: the id-ordered alternating sweep
    (schwarz.py:216-233) as wavefront levels.  Level = 1 + max over face
    neighbours of lower id; neighbours never share a level; on a lattice the
    levels are the anti-diagonals (sum of lattice positions)."""
    from paper_2006_14602_b200.grid import alternating_levels
    dim = len(counts)
    g = P.build_grid(dim, [(0.0, 1.0)] * dim, counts)
    d = P.build_decomposition(g, layout, ov)
    lev = alternating_levels(d)
    assert len(lev) == d.nsub
    for s in d.subdomains:
        nbs = [n for n in s.neighbors.values() if n is not None and n >= 0]
        lower = [lev[n] for n in nbs if n < s.id]
        assert lev[s.id] == (1 + max(lower) if lower else 0)
        assert all(lev[n] != lev[s.id] for n in nbs)
        assert lev[s.id] == sum(s.pos)
    assert max(lev) + 1 == sum(n - 1 for n in layout) + 1


def test_rkc_coefficients_bitwise():
    for s in (2, 3, 4, 9, 23, 64, 257, 512):
        got = P.rkc_coeffs(s)
        ref = O.rkc_coeffs(s)
        for x, y in zip(got, ref):
            assert np.array_equal(np.asarray(x), np.asarray(y)), s


def test_solver_config_validation_mirrors_reference():
    with pytest.raises(P.ConfigurationError):
        P.SolverConfig(tol=0.0)
    with pytest.raises(P.ConfigurationError):
        P.SolverConfig(max_windows=0)
    with pytest.raises(P.ConfigurationError):
        P.SolverConfig(transmission="both")
    with pytest.raises(P.ConfigurationError):
        P.SolverConfig(stop_rule="mean")
    with pytest.raises(P.ConfigurationError):
        P.SolverConfig(rtol=0.0).window()
    with pytest.raises(P.ConfigurationError):
        P.SolverConfig(dtau=-1.0).window()
    with pytest.raises(P.ConfigurationError):
        P.build_grid(2, ((0, 1), (1, 1)), (9, 9))
    with pytest.raises(P.ConfigurationError):
        P.build_grid(2, ((0, 1), (0, 1)), (9, 2))


def test_native_monitors_match_baseline_formulas():
    """Each native density is the BASELINE formula (same numpy expression as the
    oracle's, hence bitwise)."""
    pts = np.random.default_rng(0).uniform(0, 1, (1000, 2))
    assert np.array_equal(P.RingDensity()(pts), O.Ring()(pts))
    mix = P.seeded_mixture(32, 2)
    omix = O.seeded_mixture(32, 2)
    assert np.array_equal(mix(pts), omix(pts))
    p3 = np.random.default_rng(1).uniform(0, 1, (500, 3))
    assert np.array_equal(P.ShellDensity()(p3), O.Shell()(p3))
    assert np.array_equal(P.seeded_mixture(16, 3)(p3), O.seeded_mixture(16, 3)(p3))


def test_monitor_lowering():
    from paper_2006_14602_b200.monitor import lower_monitor
    g = P.build_grid(2, ((0.0, 1.0),) * 2, (9, 9))
    nm = lower_monitor(P.density_monitor(P.seeded_mixture(8, 2), g.extents), 2)
    assert nm.desc.kind == _lib.MON_MIXTURE and nm.desc.nbumps == 8
    with pytest.raises(P.ConfigurationError):
        lower_monitor(P.density_monitor(lambda p: np.ones(p.shape[:-1]), g.extents), 2)
    with pytest.raises(P.ConfigurationError):
        lower_monitor(P.density_monitor(P.RingDensity(), ((0, 1),) * 3), 2)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    g = P.build_grid(2, ((0.0, 1.0),) * 2, (9, 9))
    d = P.build_decomposition(g, (1, 1), 3)
    m = P.density_monitor(P.RingDensity(), g.extents)
    with pytest.raises(P.DdmeshError, match="no CPU fallback"):
        P.solve(g, d, m, P.SolverConfig(max_windows=1))
