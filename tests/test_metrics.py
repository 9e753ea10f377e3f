"""Metrics row: quality_measure / relative_errors.

Golden values come from the real reference (tests/golden/make_metrics_golden.py).
The CPU tests pin the oracle restatement to them; the GPU tests run the
device implementation (ddpma_quality / ddpma_relative_errors through the C ABI).

Tolerances: e_adp goes through the monitor's exp and one division (CUDA vs
numpy differ by <= 1 ulp each), so per-node values agree to 1e-14 relative;
the reductions sum in a different (fixed) order than numpy's pairwise sum,
so the norms agree to 1e-12 relative; `tangled` is exact.
"""

import numpy as np
import pytest

import ddpma_oracle as O
from conftest import golden

CASES = [("Q2ring", 2, (65, 65), "ring"), ("Q2tangled", 2, (65, 65), "ring"),
         ("Q2mix", 2, (129, 129), "mix"), ("Q3shell", 3, (33, 33, 33), "shell")]


def rclose(a, b, rtol):
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    scale = np.maximum(np.abs(b), 1e-300)
    return float(np.max(np.where(a == b, 0.0, np.abs(a - b) / scale)))


def oracle_monitor(kind, dim):
    if kind == "ring":
        return O.Ring()
    if kind == "shell":
        return O.Shell()
    return O.seeded_mixture(8, dim)


@pytest.mark.parametrize("name,dim,counts,kind", CASES)
def test_oracle_metrics_pinned(name, dim, counts, kind):
    G = golden("metrics.npz")
    grid = O.make_grid(dim, tuple((0.0, 1.0) for _ in range(dim)), counts)
    geom = O.whole_geom(grid)
    mon = oracle_monitor(kind, dim)
    psi = G[f"{name}_psi"]
    for sample, ek, rk in ((False, "_e", "_rep"), (True, "_es", "_reps")):
        e, e2, emax, mean, tang = O.quality_measure(psi, mon, grid.extents,
                                                    float(G[f"{name}_norm"]), geom, sample)
        assert np.array_equal(e, G[name + ek])
        assert [e2, emax, mean, float(tang)] == list(G[name + rk])
    assert list(O.relative_errors(psi, G[f"{name}_other"], geom)) == list(G[f"{name}_rel"])


@pytest.mark.gpu
@pytest.mark.parametrize("name,dim,counts,kind", CASES)
def test_device_quality_measure(name, dim, counts, kind):
    import paper_2006_14602_b200 as P
    G = golden("metrics.npz")
    grid = P.build_grid(dim, tuple((0.0, 1.0) for _ in range(dim)), counts)
    raw = {"ring": P.RingDensity(), "shell": P.ShellDensity(),
           "mix": P.seeded_mixture(8, dim)}[kind]
    mon = P.MonitorField(raw=raw, domain=grid.extents, normalizer=float(G[f"{name}_norm"]))
    psi = G[f"{name}_psi"]
    for sample, ek, rk in ((False, "_e", "_rep"), (True, "_es", "_reps")):
        q = P.quality_measure(psi, mon, grid, sample_on_mesh=sample)
        ref = G[name + rk]
        assert q.e_adp.shape == psi.shape
        assert rclose(q.e_adp, G[name + ek], 0) <= 1e-13
        assert rclose([q.e2, q.emax, q.node_mean], ref[:3], 0) <= 1e-12
        assert q.tangled == bool(ref[3])
    r = P.relative_errors(psi, G[f"{name}_other"], grid, meta={"case": name})
    assert rclose([r.e1, r.e2, r.einf], G[f"{name}_rel"], 0) <= 1e-12
    assert r.meta == {"case": name}


@pytest.mark.gpu
def test_device_metrics_errors_and_restrict():
    import paper_2006_14602_b200 as P
    grid = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65))
    with pytest.raises(P.ConfigurationError):
        P.relative_errors(np.zeros((65, 65)), np.zeros((33, 33)), grid)
    with pytest.raises(P.ConfigurationError):
        P.restrict_to_grid(np.zeros((65, 65)), (40, 40))
    fine = np.arange(129 * 129, dtype=float).reshape(129, 129)
    assert np.array_equal(P.restrict_to_grid(fine, (65, 65)), fine[::2, ::2])
    # a perfect identity mesh with a uniform density: e_adp == 1 everywhere
    ax = grid.axes()
    x = np.meshgrid(*ax, indexing="ij")
    psi = 0.5 * (x[0] ** 2 + x[1] ** 2)
    q = P.quality_measure(psi, P.density_monitor(P.UniformDensity(1.0), grid.extents), grid)
    assert np.allclose(q.e_adp, 1.0, rtol=0, atol=1e-12) and not q.tangled
    assert abs(q.e2 - 1.0) < 1e-12
