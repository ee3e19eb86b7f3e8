"""LCE on the device: per-call parity of the Newton kernels with the
reference's goldens, Frank force, local-convergent trajectories and one
polydomain outer iteration (SURVEY §8(c) parity plan for the chaotic LCE).
"""

import numpy as np
import pytest

import oracle
from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_2010_06697_b200")


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _model(g, dim):
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=g["n0"], dim=dim,
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
def test_local_lce_per_call(name, dim):
    """One local_sweeps call (<= 50 sweeps) against the reference's numba
    kernels: identical per-point sweep counts and convergence flags, fields
    within 1e-10 on the points that converge (a point still iterating at the
    cap is in its chaotic regime)."""
    g = golden(name)
    m, internal, prev_F, prev_int = _model(g, dim)
    F = g["F0"].copy()
    st = m.local_sweeps(F, internal, g["G"], g["lam"], float(g["rho"]), float(g["dt"]), prev_F,
                        prev_int, {"frank_force": g["ff"]}, int(g["max_sweeps"]),
                        float(g["point_tol"]))
    ok = g["ok"]
    assert st.sweeps == int(g["sweeps"])
    assert st.converged_frac == pytest.approx(float(g["frac"]))
    assert rel_l2(F[ok], g["F"][ok]) < 1e-10
    assert rel_l2(internal["angles"][ok], g["angles"][ok]) < 1e-10
    assert rel_l2(internal["p_inc"][ok], g["p_inc"][ok]) < 1e-9
    if dim == 3:
        assert rel_l2(internal["chart"][ok], g["chart"][ok]) < 1e-10


@pytest.mark.parametrize("dim,ms", [(2, 10), (3, 5)])
def test_local_lce_matches_oracle_short_calls(dim, ms):
    """Polydomain-like inputs, short metered calls (the policy chunk regime):
    every point within 1e-10 of the oracle."""
    rng = np.random.default_rng(11 + dim)
    npts = 2000
    n0 = rng.standard_normal((npts, dim))
    n0 /= np.linalg.norm(n0, axis=1, keepdims=True)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=dim)
    om = oracle.LCE(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=dim)
    F0 = np.tile(np.eye(dim), (npts, 1, 1)) + 1e-3 * rng.standard_normal((npts, dim, dim))
    G = np.tile(np.eye(dim), (npts, 1, 1))
    lam = np.zeros((npts, dim, dim))
    ff = 1e-3 * rng.standard_normal((npts, dim))
    i1 = m.init_internal(npts)
    i2 = om.init_internal(npts)
    F1, F2 = F0.copy(), F0.copy()
    s1 = m.local_sweeps(F1, i1, G, lam, 1.0, 0.0, None, None, {"frank_force": ff}, ms, 1.0)
    r2 = om.local_sweeps(F2, i2, G, lam, 1.0, 0.0, None, None, {"frank_force": ff}, ms, 1.0)
    assert s1.sweeps == r2[1]
    assert rel_l2(F1, F2) < 1e-10
    assert rel_l2(i1["angles"], i2["angles"]) < 1e-10


@pytest.mark.parametrize("name", ["frank_2d", "frank_3d"])
def test_frank_force(name):
    g = golden(name)
    dim, n, L = int(g["dim"]), int(g["n"]), float(g["L"])
    grid = mm.Grid(dim, n, L)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=float(g["kappa"]),
                                  n0=g["n_field"], dim=dim)
    ff = m.frank_force(grid, g["n_field"].reshape(grid.shape + (dim,)))
    assert rel_l2(ff, g["ff"]) < 1e-12


@pytest.mark.parametrize("name,conv", [("lce_uniform_solve", True), ("lce_stripe_iters", False)])
def test_lce_convergent_trajectories(name, conv):
    g = golden(name)
    n, L = int(g["n"]), float(g["L"])
    grid = mm.Grid(2, n, L)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=g["n0"], dim=2)
    bc = mm.MacroBC(g["mask"], g["value"])
    if conv:
        params = mm.SolverParams(r_p_tol=1e-8, r_d_tol=1e-8, point_tol=1e-12, max_outer=4000)
    else:
        params = mm.SolverParams(point_tol=1e-12, max_outer=int(g["K"]))
    st, ok = mm.solve(grid, m, bc, params, raise_on_max=False)
    assert ok == conv
    assert len(st.history) == g["hist"].shape[0]
    assert st.total_sweeps == int(g["total_sweeps"])
    for k in ("F", "lam", "grad_u"):
        assert rel_l2(getattr(st, k), g[k]) < 1e-10, k
    assert rel_l2(st.internal["angles"], g["angles"]) < 1e-10


@pytest.mark.parametrize("name", ["lce_poly_2d", "lce_poly_3d"])
def test_lce_polydomain_one_iteration(name):
    """SURVEY §8(d) config 3 material on a polydomain director field, one
    outer iteration with a short local budget (max_local 10 in 2D, 5 in 3D,
    below the horizon where sweeps amplify roundoff past 1e-10)."""
    g = golden(name)
    dim, n, L = int(g["dim"]), int(g["n"]), float(g["L"])
    grid = mm.Grid(dim, n, L)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=g["n0"], dim=dim)
    bc = mm.MacroBC.stress(np.zeros((dim, dim)))
    params = mm.SolverParams(max_outer=1, max_local=int(g["max_local"]))
    st = mm.solver.init_state(grid, m, bc, params)
    st.F = g["F0"].copy()
    st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                     raise_on_max=False)
    assert st.total_sweeps == int(g["total_sweeps"])
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(getattr(st, k), g[k]) < 1e-9, k


def test_lce_viscous_needs_previous_step():
    grid = mm.Grid(2, 8)
    n0 = np.tile([1.0, 0.0], (grid.npoints, 1))
    m = mm.LiquidCrystalElastomer(mu=1.0, r=1.5, alpha=0.2, frank_kappa=0.0, n0=n0, dim=2,
                                  nu_F=0.5, nu_n=0.2)
    with pytest.raises(mm.ParameterError):
        mm.solve(grid, m, mm.MacroBC.stress(np.zeros((2, 2))), mm.SolverParams(max_outer=1),
                 dt=0.1, raise_on_max=False)


def test_lce_viscous_time_step_matches_oracle():
    """begin_time_step + a viscous outer iteration (device copies of F and
    the internals) against the oracle on a stripe microstructure."""
    n = 12
    grid = mm.Grid(2, n, 0.5)
    y = grid.coords()[..., 1]
    band = ((y + 0.5) / 1.0 * 4).astype(int) % 2
    n0 = np.where(band.reshape(-1, 1) == 0, [1.0, 0.2], [0.2, 1.0])
    n0 = n0 / np.linalg.norm(n0, axis=1, keepdims=True)
    kw = dict(mu=1.0, r=1.5, alpha=0.2, frank_kappa=1e-4, n0=n0, dim=2, nu_F=0.3, nu_n=0.1)
    m = mm.LiquidCrystalElastomer(**kw)
    om = oracle.LCE(**kw)
    bc = mm.MacroBC.strain(np.diag([1.02, 1 / 1.02]))
    p = mm.SolverParams(point_tol=1e-12, max_outer=3)
    st = mm.solver.init_state(grid, m, bc, p)
    st, _ = mm.solve(grid, m, bc, p, raise_on_max=False)
    mm.solver.begin_time_step(st)
    st, _ = mm.solve(grid, m, bc, p, state=st, dt=0.05, raise_on_max=False)
    op = oracle.Params(point_tol=1e-12, max_outer=3)
    ost = oracle.init_state(2, n, om, bc.strain_mask, bc.value, op)
    ost, _ = oracle.solve(2, n, 0.5, om, bc.strain_mask, bc.value, op, raise_on_max=False)
    oracle.begin_time_step(ost)
    ost, _ = oracle.solve(2, n, 0.5, om, bc.strain_mask, bc.value, op, state=ost, dt=0.05,
                          raise_on_max=False)
    for k in ("F", "lam", "grad_u"):
        assert rel_l2(getattr(st, k), getattr(ost, k)) < 1e-10, k
    assert st.total_sweeps == ost.total_sweeps


@pytest.mark.parametrize("chunk,kind", [(5, "3"), (25, "3"), (25, "2")])
def test_lce3d_newton_compacted_schedule_is_the_plain_loop(chunk, kind, monkeypatch):
    """The Newton-compacted rounds (MM_LCE_SPLIT_MIN=0 forces them) perform
    every point's sweeps exactly as the single-launch loop: fields, angles,
    chart, p_inc, per-point residuals, sweep counts and flags bit for bit;
    the batch sums (reduced afterwards in another order) to roundoff."""
    rng = np.random.default_rng(21)
    npts = 3000
    n0 = rng.standard_normal((npts, 3))
    n0 /= np.linalg.norm(n0, axis=1, keepdims=True)
    F0 = np.tile(np.eye(3), (npts, 1, 1)) + 1e-2 * rng.standard_normal((npts, 3, 3))
    G = np.tile(np.eye(3), (npts, 1, 1)) + 1e-2 * rng.standard_normal((npts, 3, 3))
    lam = 1e-2 * rng.standard_normal((npts, 3, 3))
    ff = 1e-3 * rng.standard_normal((npts, 3))
    out = {}
    monkeypatch.setenv("MM_LCE_SPLIT_KIND", kind)
    for split in ("0", "1000000000"):
        monkeypatch.setenv("MM_LCE_SPLIT_MIN", split)
        m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=3)
        internal = m.init_internal(npts)
        F = F0.copy()
        st = m.local_sweeps(F, internal, G, lam, 1.0, 0.0, None, None, {"frank_force": ff},
                            chunk, 1e-6)
        res, nsw, ok = m._pts_ctx.download_points()
        out[split] = (F, internal, st, res, nsw, ok)
    a, b = out["0"], out["1000000000"]
    assert np.array_equal(a[0], b[0])
    for k in a[1]:
        assert np.array_equal(a[1][k], b[1][k]), k
    assert np.array_equal(a[3], b[3]) and np.array_equal(a[4], b[4]) and np.array_equal(a[5], b[5])
    assert a[2].sweeps == b[2].sweeps and a[2].converged_frac == b[2].converged_frac
