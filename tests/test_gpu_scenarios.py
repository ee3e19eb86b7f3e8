"""§8(f) rows 1-2 on the device: the load-stepping drivers keep the state
resident across steps (run_lce_protocol / relax_zero_stress) and
equilibrium_residual runs as one stress + stencil-divergence + FFT pass;
both against fixtures from the reference (tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_2010_06697_b200")


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_config1_through_run_lce_protocol():
    """SURVEY §8(d) config 1 through the driver itself (relaxation, mixed
    control relative to the relaxed reference, seeded perturbations)."""
    g = golden("config1_protocol")
    grid = mm.Grid(2, int(g["n"]), 0.5)
    m = mm.MooneyRivlin(g["mu"], g["kappa"], dim=2, mu_rep=1.0)
    study = mm.run_lce_protocol(grid, m, mm.ProtocolSpec("monodomain", 1.0, 0.8, -0.02),
                                relax=True, seed=0, perturb=1e-4)
    assert study.completed
    assert [r.outer_iters for r in study.records] == list(g["outer_iters"])
    np.testing.assert_allclose(study.lams, g["lams"], rtol=0, atol=0)
    np.testing.assert_allclose(study.nominal, g["nominal"], rtol=1e-8, atol=1e-12)
    np.testing.assert_allclose(np.array([r.Fbar for r in study.records]), g["Fbar"],
                               rtol=1e-10, atol=1e-13)
    assert rel_l2(study.state.F, g["F"]) < 1e-10
    assert rel_l2(study.state.lam, g["lam"]) < 1e-10


def test_viscous_lce_protocol():
    """Viscous relaxation (implicit time steps until the mean stress is
    below tolerance) followed by rate-controlled loading of a stripe LCE."""
    g = golden("lce_protocol_visc")
    grid = mm.Grid(2, int(g["n"]), 0.5)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=g["n0"],
                                  dim=2, nu_F=0.5, nu_n=0.2)
    study = mm.run_lce_protocol(grid, m, mm.ProtocolSpec("monodomain", 1.0, 1.04, 0.02,
                                                         rate=0.2),
                                relax=True, seed=3, perturb=1e-4)
    assert [r.outer_iters for r in study.records] == list(g["outer_iters"])
    assert study.state.total_sweeps == int(g["total_sweeps"])
    np.testing.assert_allclose(study.reference, g["reference"], rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(study.nominal, g["nominal"], rtol=1e-8, atol=1e-11)
    np.testing.assert_allclose(study.S, g["S"], rtol=1e-9, atol=1e-12)
    assert rel_l2(study.state.F, g["F"]) < 1e-10
    assert rel_l2(study.state.lam, g["lam"]) < 1e-10
    assert rel_l2(study.state.internal["angles"], g["angles"]) < 1e-10


def test_perturb_F_on_device_is_numpy_addition():
    grid = mm.Grid(3, 8, 0.5)
    m = mm.MooneyRivlin(np.ones(grid.npoints), 9.8 * np.ones(grid.npoints), dim=3)
    bc = mm.MacroBC.strain(np.diag([0.97, 1.0, 1.0]))
    st, _ = mm.solve(grid, m, bc, mm.SolverParams(max_outer=3), raise_on_max=False)
    F0 = np.array(st.F)
    dF = 1e-4 * np.random.default_rng(5).standard_normal(F0.shape)
    mm.scenarios.perturb_F(st, dF)
    assert "F" in st._dev and "F" not in st._dirty
    assert np.array_equal(st.F, F0 + dF)


def _eq_state(grid, F, internal=None, prev_F=None, prev_internal=None):
    d = grid.dim
    z = np.zeros(grid.shape + (d, d))
    return mm.ADMMState(u_mean=np.eye(d), u_tilde=np.zeros(grid.shape + (d,)), grad_u=z.copy(),
                        F=F, lam=z.copy(), internal=internal or {}, rho=1.0, prev_F=prev_F,
                        prev_internal=prev_internal)


def test_equilibrium_residual_matches_reference():
    g = golden("eq_residual_cases")
    tol = 1e-10
    grid = mm.Grid(2, 16, 0.5)
    m = mm.MooneyRivlin(g["mr2d_mu"], g["mr2d_kappa"], dim=2, mu_rep=1.0)
    v = mm.equilibrium_residual(grid, m, _eq_state(grid, g["mr2d_F"]))
    assert abs(v - g["mr2d_val"]) <= tol * g["mr2d_val"]
    grid = mm.Grid(3, 8, 0.5)
    m = mm.MooneyRivlin(g["mr3d_mu"], g["mr3d_kappa"], dim=3, mu_rep=1.0)
    v = mm.equilibrium_residual(grid, m, _eq_state(grid, g["mr3d_F"]))
    assert abs(v - g["mr3d_val"]) <= tol * g["mr3d_val"]
    grid = mm.Grid(2, 9, 0.5)
    m = mm.QuadraticMaterial(g["quad_c"], dim=2)
    v = mm.equilibrium_residual(grid, m, _eq_state(grid, g["quad_F"]))
    assert abs(v - g["quad_val"]) <= tol * g["quad_val"]
    grid = mm.Grid(2, 16, 0.5)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=g["lce2d_n0"],
                                  dim=2, nu_F=0.5, nu_n=0.2)
    internal = {"angles": g["lce2d_angles"], "p_inc": g["lce2d_p_inc"]}
    st = _eq_state(grid, g["lce2d_F"], internal, prev_F=g["lce2d_Fk"],
                   prev_internal=m.init_internal(grid.npoints))
    v = mm.equilibrium_residual(grid, m, st, dt=0.1)
    assert abs(v - g["lce2d_val"]) <= tol * g["lce2d_val"]
    grid = mm.Grid(3, 8, 0.5)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=g["lce3d_n0"],
                                  dim=3)
    internal = {"angles": g["lce3d_angles"], "chart": g["lce3d_chart"],
                "p_inc": g["lce3d_p_inc"]}
    v = mm.equilibrium_residual(grid, m, _eq_state(grid, g["lce3d_F"], internal))
    assert abs(v - g["lce3d_val"]) <= tol * g["lce3d_val"]


def test_equilibrium_residual_bounds_after_solve():
    """reference test_solver.py:117-136: converged iterates have a small
    equilibrium residual; homogeneous strain is an exact equilibrium."""
    grid = mm.Grid(3, 16, 0.5)
    x = grid.coords()[..., 0]
    mu = np.where((x + 0.5) < 0.5, 0.05, 1.0).ravel()
    m = mm.MooneyRivlin(mu, 9.8 * mu, dim=3, mu_rep=1.0)
    bc = mm.MacroBC.strain(np.diag([0.97, 1.0, 1.0]))
    st, conv = mm.solve(grid, m, bc, mm.SolverParams(r_p_tol=1e-6, r_d_tol=1e-6))
    assert conv
    last = st.history[-1]
    r_eq = mm.equilibrium_residual(grid, m, st)
    assert r_eq <= 10.0 * m.mu_rep * (last.r_d + last.r_l)
    g2 = mm.Grid(2, 8, 0.5)
    m2 = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    Fbar = np.array([[0.95, 0.1], [0.0, 1.02]])
    st2, conv = mm.solve(g2, m2, mm.MacroBC.strain(Fbar), mm.SolverParams())
    assert conv and mm.equilibrium_residual(g2, m2, st2) < 1e-10


def test_equilibrium_residual_inadmissible():
    grid = mm.Grid(2, 8, 0.5)
    m = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    F = np.broadcast_to(np.eye(2), grid.shape + (2, 2)).copy()
    F[3, 4] = [[-1.0, 0.0], [0.0, 1.0]]
    with pytest.raises(mm.InadmissibleStateError):
        mm.equilibrium_residual(grid, m, _eq_state(grid, F))
