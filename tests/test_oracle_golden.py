"""Pin the oracle (oracle/) against the reference's own numbers.

CPU-only.  Fixtures in tests/golden/ were produced by running the real
reference (tests/golden/make_golden.py); the frozen mpmath values below are
the reference's own goldens (reference pkg/tests/test_materials.py:17-35).
"""

import numpy as np
import pytest

import oracle
from conftest import golden, rel_l2

# reference pkg/tests/test_materials.py:17-35 (50-digit mpmath, frozen)
F2_REF = np.array([[1.1, 0.2], [-0.05, 0.95]])
W2_REF = 0.0504162529935612362
S2_REF = np.array([[0.925048886255924171, 0.233423625592417062],
                   [0.0413054976303317536, 0.650319763033175355]])
F3_REF = np.array([[1.05, 0.10, -0.02], [0.03, 0.95, 0.08], [-0.07, 0.01, 1.02]])
W3_REF = 0.015866975881478478
S3_REF = np.array([
    [0.0887625404635236158, 0.0941621524842185965, -0.0585865134239171891],
    [0.0892146956874900707, -0.0489181850033207401, 0.0676805985766250121],
    [-0.0670214949467928758, 0.0634673508332843443, 0.0502082694597957404],
])


def test_mr_frozen_energy_stress():
    m2 = oracle.MR(mu=1.3, kappa=12.74, dim=2)
    np.testing.assert_allclose(m2.energy(F2_REF[None])[0], W2_REF, rtol=1e-14)
    np.testing.assert_allclose(m2.stress(F2_REF[None])[0], S2_REF, rtol=1e-13)
    m3 = oracle.MR(mu=0.7, kappa=2.1, dim=3)
    np.testing.assert_allclose(m3.energy(F3_REF[None])[0], W3_REF, rtol=1e-14)
    np.testing.assert_allclose(m3.stress(F3_REF[None])[0], S3_REF, rtol=1e-13)


@pytest.mark.parametrize("name,dim", [("local_mr2d", 2), ("local_mr2d_long", 2),
                                      ("local_mr3d", 3), ("local_mr3d_long", 3),
                                      ("local_mr3d_loose", 3)])
def test_local_mr_matches_reference(name, dim):
    g = golden(name)
    m = oracle.MR(g["mu"], g["kappa"], dim=dim, mu_rep=float(g["mu_rep"]))
    F = g["F0"].copy()
    res, sweeps, frac, _ = m.local_sweeps(F, {}, g["G"], g["lam"], float(g["rho"]), 0.0, None,
                                          None, {}, int(g["max_sweeps"]), float(g["point_tol"]))
    assert sweeps == int(g["sweeps"])
    assert frac == float(g["frac"])
    assert rel_l2(F, g["F"]) < 1e-12
    # residuals at the stationarity noise floor (~1e-10) are roundoff noise
    np.testing.assert_allclose(res, g["res"], rtol=1e-6, atol=2e-11 * float(g["mu_rep"]))


@pytest.mark.parametrize("name,dim", [("local_quad", 2), ("local_quad3d", 3)])
def test_local_quadratic_matches_reference(name, dim):
    g = golden(name)
    q = oracle.Quadratic(g["c"], dim=dim)
    F = g["F0"].copy()
    res, sweeps, frac, _ = q.local_sweeps(F, {}, g["G"], g["lam"], float(g["rho"]), 0.0, None,
                                          None, {}, int(g["max_sweeps"]), float(g["point_tol"]))
    assert sweeps == int(g["sweeps"])
    assert frac == float(g["frac"])
    assert rel_l2(F, g["F"]) < 1e-12


def _lce_from_golden(g, dim):
    m = oracle.LCE(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=g["n0"], dim=dim,
                   nu_F=float(g["nu_F"]), nu_n=float(g["nu_n"]))
    internal = {"angles": g["angles0"].copy(), "p_inc": g["p_inc0"].copy()}
    if dim == 3:
        internal["chart"] = g["chart0"].copy()
    prev_F = prev_int = None
    if float(g["dt"]) > 0:
        prev_F = g["prev_F"]
        prev_int = {"angles": g["prev_angles"], "p_inc": g["prev_p_inc"]}
        if dim == 3:
            prev_int["chart"] = g["prev_chart"]
    return m, internal, prev_F, prev_int


@pytest.mark.parametrize("name,dim", [("local_lce2d", 2), ("local_lce2d_visc", 2),
                                      ("local_lce3d", 3), ("local_lce3d_visc", 3)])
def test_local_lce_matches_reference(name, dim):
    g = golden(name)
    m, internal, prev_F, prev_int = _lce_from_golden(g, dim)
    F = g["F0"].copy()
    res, sweeps, frac, (nsw, ok) = m.local_sweeps(
        F, internal, g["G"], g["lam"], float(g["rho"]), float(g["dt"]), prev_F, prev_int,
        {"frank_force": g["ff"]}, int(g["max_sweeps"]), float(g["point_tol"]))
    assert np.array_equal(nsw, g["nsw"])
    assert np.array_equal(ok.astype(bool), g["ok"])
    assert sweeps == int(g["sweeps"])
    assert rel_l2(F, g["F"]) < 1e-10
    assert rel_l2(internal["angles"], g["angles"]) < 1e-10
    if dim == 3:
        assert rel_l2(internal["chart"], g["chart"]) < 1e-10


@pytest.mark.parametrize("name", ["project_2d", "project_2d_odd", "project_3d", "project_3d_n12"])
def test_projection_matches_reference(name):
    g = golden(name)
    dim, n, L = int(g["dim"]), int(g["n"]), float(g["L"])
    u_mean, u_tilde, grad_u = oracle.project(dim, n, L, g["F"], g["lam"], float(g["rho"]),
                                             g["mask"], g["value"])
    assert rel_l2(u_mean, g["u_mean"]) < 1e-14
    assert rel_l2(u_tilde, g["u_tilde"]) < 1e-13
    assert rel_l2(grad_u, g["grad_u"]) < 1e-13


@pytest.mark.parametrize("name", ["frank_2d", "frank_3d"])
def test_frank_force_matches_reference(name):
    g = golden(name)
    dim, n, L = int(g["dim"]), int(g["n"]), float(g["L"])
    m = oracle.LCE(mu=1.0, r=2.0, alpha=0.1, frank_kappa=float(g["kappa"]), n0=g["n_field"],
                   dim=dim)
    ff = m.frank_force(dim, n, L, g["n_field"].reshape((n,) * dim + (dim,)))
    assert rel_l2(ff, g["ff"]) < 1e-13


def _mr_traj(g, dim):
    n, L = int(g["n"]), float(g["L"])
    m = oracle.MR(g["mu"], g["kappa"], dim=dim, mu_rep=float(g["mu_rep"]))
    params = oracle.Params(max_outer=int(g["K"]))
    st = oracle.init_state(dim, n, m, g["mask"], g["value"], params)
    if "F0" in g:
        st.F = g["F0"].copy()
    st, _ = oracle.solve(dim, n, L, m, g["mask"], g["value"], params,
                         policy=oracle.RatioToDual(0.3), state=st, raise_on_max=False)
    return st


@pytest.mark.parametrize("name,dim", [("traj_mr2d", 2), ("traj_mr3d", 3)])
def test_mr_trajectory_matches_reference(name, dim):
    g = golden(name)
    st = _mr_traj(g, dim)
    hist = np.array(st.history)
    assert np.array_equal(hist[:, 0], g["hist"][:, 0])
    np.testing.assert_allclose(hist[:, 1:], g["hist"][:, 1:], rtol=1e-9)
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(getattr(st, k), g[k]) < 1e-10, k
    assert st.total_sweeps == int(g["total_sweeps"])


@pytest.mark.parametrize("name,conv", [("lce_uniform_solve", True), ("lce_stripe_iters", False)])
def test_lce_convergent_solve_matches_reference(name, conv):
    """Local-convergent LCE (strain control, ExactAll): full-trajectory parity."""
    g = golden(name)
    n, L = int(g["n"]), float(g["L"])
    m = oracle.LCE(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=g["n0"], dim=2)
    if conv:
        params = oracle.Params(r_p_tol=1e-8, r_d_tol=1e-8, point_tol=1e-12, max_outer=4000)
    else:
        params = oracle.Params(point_tol=1e-12, max_outer=int(g["K"]))
    st, ok = oracle.solve(2, n, L, m, g["mask"], g["value"], params, raise_on_max=False)
    assert ok == conv
    hist = np.array(st.history)
    assert hist.shape == g["hist"].shape
    assert st.total_sweeps == int(g["total_sweeps"])
    for k in ("F", "lam", "grad_u"):
        assert rel_l2(getattr(st, k), g[k]) < 1e-10, k
    assert rel_l2(st.internal["angles"], g["angles"]) < 1e-10


@pytest.mark.parametrize("name", ["lce_poly_2d", "lce_poly_3d"])
def test_lce_polydomain_one_iteration(name):
    g = golden(name)
    dim, n, L = int(g["dim"]), int(g["n"]), float(g["L"])
    m = oracle.LCE(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=g["n0"], dim=dim)
    mask = np.zeros((dim, dim), bool)
    val = np.zeros((dim, dim))
    params = oracle.Params(max_outer=1, max_local=int(g["max_local"]))
    st = oracle.init_state(dim, n, m, mask, val, params)
    st.F = g["F0"].copy()
    st, _ = oracle.solve(dim, n, L, m, mask, val, params, policy=oracle.RatioToDual(0.3),
                         state=st, raise_on_max=False)
    assert st.total_sweeps == int(g["total_sweeps"])
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(getattr(st, k), g[k]) < 1e-9, k


@pytest.mark.slow
def test_config1_load_step_history():
    """SURVEY §8(d) config 1 through the oracle: same cumulative outer
    iteration counts per load step as the reference."""
    g = golden("config1_protocol")
    n, L = int(g["n"]), float(g["L"])
    m = oracle.MR(g["mu"], g["kappa"], dim=2, mu_rep=1.0)
    params = oracle.Params()
    pol = oracle.RatioToDual(0.3)
    # relax_zero_stress (scenarios.py:712-756): one stress-free solve
    mask0 = np.zeros((2, 2), bool)
    st = oracle.init_state(2, n, m, mask0, np.zeros((2, 2)), params)
    st, ok = oracle.solve(2, n, L, m, mask0, np.zeros((2, 2)), params, policy=pol, state=st,
                          raise_on_max=False)
    assert ok
    ref = st.u_mean.copy()
    mask = np.zeros((2, 2), bool)
    for ij in ((0, 0), (0, 1), (1, 0)):
        mask[ij] = True
    iters = []
    for step, lam in enumerate(g["lams"]):
        P = np.eye(2)
        P[0, 0] = lam
        target = P @ ref
        value = np.where(mask, target, 0.0)
        rng = np.random.default_rng(np.random.SeedSequence((0, step)))
        st.F = st.F + 1e-4 * rng.standard_normal(st.F.shape)
        st, ok = oracle.solve(2, n, L, m, mask, value, params, policy=pol, state=st,
                              raise_on_max=False)
        assert ok
        iters.append(st.outer_iter)
    assert iters == list(g["outer_iters"])
    assert rel_l2(st.F, g["F"]) < 1e-9
