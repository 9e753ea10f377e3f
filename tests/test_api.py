"""Drop-in surface: every public name of the reference package, the host
helpers pinned to reference outputs (CPU), and the integrator protocol and
window-level sweeps on the device (GPU)."""

import functools

import numpy as np
import pytest

import ddpma_oracle as O
import recipes as R
from conftest import golden

import paper_2006_14602_b200 as P


def test_every_reference_name_is_exported():
    """`import paper_2006_14602_b200 as ddmesh` works for any caller of the
    reference API (ddmesh/__init__.py:28-44; names pinned in api.npz)."""
    names = [str(n) for n in golden("api.npz")["names"]]
    missing = [n for n in names if not hasattr(P, n)]
    assert not missing, missing
    assert set(names) <= set(P.__all__)


def test_initial_potential_bitwise():
    gold = golden("api.npz")
    g = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65))
    d = P.build_decomposition(g, (2, 2), 4)
    for sid in (0, 3):
        geom = P.subdomain_geometry(g, d.subdomains[sid])
        assert np.array_equal(P.initial_potential(geom), gold[f"psi0_s{sid}"])
    pf = P.PotentialField(values=P.initial_potential(geom), geom=geom)
    assert pf.tau == 0.0


def test_host_helpers_match_reference():
    gold = golden("api.npz")
    fit = P.convergence_slope([(1 / 16, 3.1e-3), (1 / 32, 8.2e-4), (1 / 64, 2.05e-4),
                               (1 / 128, 5.3e-5)])
    assert np.array_equal([fit.slope, fit.intercept, fit.residual], gold["slope"])
    a = 0.7
    x = P.quasi1d_oracle(lambda x: 1.0 + a * (2.0 * x - 1.0), lambda x: x + a * (x * x - x), 33)
    assert np.array_equal(x, gold["quasi1d"])
    with pytest.raises(P.ConfigurationError):
        P.convergence_slope([(1, 1), (2, 2)])
    with pytest.raises(P.InvalidMonitorError):
        P.quasi1d_oracle(lambda x: x, lambda x: 1.0 - x, 9)


def test_integrator_rejects_python_callables():
    win = P.IntegrationWindow(dtau=1e-3)
    integ = P.make_integrator(win)
    with pytest.raises(P.ConfigurationError):
        integ.advance(np.zeros((4, 4)), lambda y: (y, False))


def test_sweeps_need_device_states():
    g = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65))
    d = P.build_decomposition(g, (2, 2), 4)
    m = P.density_monitor(P.RingDensity(), g.extents)
    with pytest.raises(P.ConfigurationError):
        P.parallel_sweep([], m, P.SolverConfig(), d)


# ------------------------------------------------------------------- GPU ---

def _c1_box(sid):
    g = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65))
    d = P.build_decomposition(g, (2, 2), 4)
    og = O.make_grid(2, ((0, 1), (0, 1)), (65, 65))
    od = O.make_decomposition(og, (2, 2), 4)
    geom = P.subdomain_geometry(g, d.subdomains[sid])
    ogeom = O.box_geom(og, od.subs[sid])
    y = R.perturbed_global(geom.axes, eps=0.1)
    coords = np.stack(O.coords_fd(y, ogeom), axis=-1)
    rho = O.Ring()(np.clip(coords, 0, 1)) / 1.3
    return geom, ogeom, y, rho, float(rho.max())


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", ["adaptive", "euler"])
def test_make_integrator_matches_oracle(scheme):
    """make_integrator(window).advance(y, frozen rhs) over 4 consecutive
    windows (caches carried, integrate.py:118-123) against the oracle's
    Rkc2Integrator / EulerIntegrator restatement."""
    geom, ogeom, y, rho, rmax = _c1_box(3)
    dtau = 1e-3 if scheme == "adaptive" else 2e-5
    win = P.IntegrationWindow(dtau=dtau, scheme=scheme, substeps=3)
    integ = P.make_integrator(win)
    fn = lambda v: O.rhs_frozen(v, rho, ogeom, O.DET_FLOOR, ogeom.mask(), rmax)
    ointeg = O.Rkc2(dtau) if scheme == "adaptive" else O.Euler(dtau, 3)
    rhs = P.frozen_rhs(rho, geom, max_rho=rmax)
    a, b = y, y
    for w in range(4):
        a = integ.advance(a, rhs)
        b = ointeg.advance(b, fn)
        err = float(np.max(np.abs(a - b)))
        print(f"[parity] integrator {scheme} window {w}: max|dpsi|={err:.3g}")
        assert err <= 1e-12
    # the reference's functools.partial form of the same closure
    part = functools.partial(P.pma_rhs_frozen, rho, geom, max_rho=rmax)
    c = P.advance_window(y, part, win)
    d = O.Rkc2(dtau).advance(y, fn) if scheme == "adaptive" else O.Euler(dtau, 3).advance(y, fn)
    assert float(np.max(np.abs(c - d))) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("tr", ["parallel", "alternating"])
def test_sweeps_equal_solve(tr):
    """init_states + N sweeps == solve(max_windows=N), bitwise."""
    g = P.build_grid(2, ((0.0, 1.0), (0.0, 1.0)), (65, 65))
    d = P.build_decomposition(g, (2, 2), 4)
    m = P.density_monitor(P.RingDensity(), g.extents)
    cfg = P.SolverConfig(tol=1e-300, max_windows=5, transmission=tr)
    ref = P.solve(g, d, m, cfg)
    states = P.init_states(g, d, cfg)
    assert np.array_equal(states[0].psi, P.initial_potential(states[0].geom))
    sweep = P.parallel_sweep if tr == "parallel" else P.alternating_sweep
    for _ in range(5):
        sweep(states, m, cfg, d)
    for i, st in enumerate(states):
        assert np.array_equal(st.psi, ref.sub_psi[i])
        assert st.res == ref.history[-1].residuals[i]
    assert np.array_equal(states[1].mesh.coords, P.physical_mesh(ref.sub_psi[1], states[1].geom).coords)
    states.close()
