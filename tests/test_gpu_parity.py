"""Parity of the CUDA path against the reference's golden fixtures and the
oracle.  All tests here need a B200 and the built extension (marker gpu).

Tolerances: fp64 fields within 1e-10 relative L2 (north star), integer
sweep counts / histories exact.
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


# ---------------------------------------------------------------------------
# local step, one call through MaterialModel.local_sweeps
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name,dim", [("local_mr2d", 2), ("local_mr2d_long", 2),
                                      ("local_mr3d", 3), ("local_mr3d_long", 3),
                                      ("local_mr3d_loose", 3)])
def test_local_mr(name, dim):
    g = golden(name)
    m = mm.MooneyRivlin(g["mu"], g["kappa"], dim=dim, mu_rep=float(g["mu_rep"]))
    F = g["F0"].copy()
    st = m.local_sweeps(F, {}, g["G"], g["lam"], float(g["rho"]), 0.0, None, None, {},
                        int(g["max_sweeps"]), float(g["point_tol"]))
    assert st.sweeps == int(g["sweeps"])
    assert st.converged_frac == float(g["frac"])
    assert rel_l2(F, g["F"]) < 1e-10
    np.testing.assert_allclose(st.res_pts, g["res"], rtol=1e-6, atol=2e-11 * float(g["mu_rep"]))


def test_local_mr2d_numpy_path_matches_kernel():
    """reference test_materials.py:255-265 through the device: the 2D kernel
    and the vectorised-descent path reach the same minimiser."""
    rng = np.random.default_rng(34)
    m = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    G = np.empty((32, 2, 2))
    n = 0
    while n < 32:
        A = np.eye(2) + 0.2 * rng.standard_normal((2, 2))
        if np.linalg.det(A) > 0.2:
            G[n] = A
            n += 1
    lam = 0.4 * rng.standard_normal((32, 2, 2))
    Fk = G.copy()
    m.local_sweeps(Fk, {}, G, lam, 5.0, 0.0, None, None, {}, 8000, 1e-11)
    Fn = G.copy()
    mu, kap = m._flat_moduli(32)
    m._sweeps_numpy(Fn, G, lam, mu, kap, 5.0, 1e-11 * m.mu_rep, 8000)
    np.testing.assert_allclose(Fk, Fn, atol=1e-8)
    # and the descent path equals the oracle's restatement of it
    Fo = G.copy()
    om = oracle.MR(1.0, 9.8, dim=2)
    om.descent(Fo, np.ascontiguousarray(G), np.ascontiguousarray(lam), *om.flat_moduli(32), 5.0,
               1e-11, 8000, np.empty(32))
    assert rel_l2(Fn, Fo) < 1e-12


@pytest.mark.parametrize("name,dim", [("local_quad", 2), ("local_quad3d", 3)])
def test_local_quadratic(name, dim):
    g = golden(name)
    q = mm.QuadraticMaterial(g["c"], dim=dim)
    F = g["F0"].copy()
    st = q.local_sweeps(F, {}, g["G"], g["lam"], float(g["rho"]), 0.0, None, None, {},
                        int(g["max_sweeps"]), float(g["point_tol"]))
    assert st.sweeps == int(g["sweeps"])
    assert st.converged_frac == float(g["frac"])
    assert rel_l2(F, g["F"]) < 1e-10


def test_inadmissible_raises_and_leaves_F():
    m = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=3)
    F = np.tile(np.eye(3), (8, 1, 1))
    F[3] = -np.eye(3)
    F0 = F.copy()
    with pytest.raises(mm.InadmissibleStateError):
        m.local_sweeps(F, {}, np.tile(np.eye(3), (8, 1, 1)), np.zeros((8, 3, 3)), 1.0, 0.0, None,
                       None, {}, 10, 1e-11)
    assert np.array_equal(F, F0)


# ---------------------------------------------------------------------------
# projection
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["project_2d", "project_2d_odd", "project_3d", "project_3d_n12"])
def test_projection(name):
    g = golden(name)
    dim, n, L = int(g["dim"]), int(g["n"]), float(g["L"])
    grid = mm.Grid(dim, n, L)
    bc = mm.MacroBC(g["mask"], g["value"])
    pr = mm.helmholtz_project(grid, g["F"], g["lam"], float(g["rho"]), bc)
    assert rel_l2(pr.u_mean, g["u_mean"]) < 1e-13
    assert rel_l2(pr.u_tilde, g["u_tilde"]) < 1e-12
    assert rel_l2(pr.grad_u, g["grad_u"]) < 1e-12


@pytest.mark.parametrize("dim,n", [(2, 5), (2, 7), (2, 16), (2, 64), (2, 128), (3, 6), (3, 9),
                                   (3, 16), (3, 32), (3, 64),
                                   # mixed-radix lines (tile_fft_mixed): 2^a 3^b 5^c and primes
                                   (2, 22), (2, 26), (2, 96), (2, 160), (2, 250), (3, 14),
                                   (3, 24), (3, 40), (3, 60), (3, 96)])
def test_projection_matches_oracle(dim, n):
    rng = np.random.default_rng(100 + n)
    L = 0.5
    F = np.eye(dim) + 0.1 * rng.standard_normal((n,) * dim + (dim, dim))
    lam = 0.3 * rng.standard_normal((n,) * dim + (dim, dim))
    mask = rng.random((dim, dim)) < 0.5
    value = 0.1 * rng.standard_normal((dim, dim)) + np.eye(dim)
    ou, ot, og = oracle.project(dim, n, L, F, lam, 2.5, mask, value)
    pr = mm.helmholtz_project(mm.Grid(dim, n, L), F, lam, 2.5, mm.MacroBC(mask, value))
    assert rel_l2(pr.u_tilde, ot) < 1e-12
    assert rel_l2(pr.grad_u, og) < 1e-12
    assert rel_l2(pr.u_mean, ou) < 1e-13  # device-order mean over up to 0.9M points


def test_discrete_grad_div_match_oracle_stencils():
    rng = np.random.default_rng(7)
    grid = mm.Grid(3, 12, 0.4)
    u = rng.standard_normal(grid.shape + (3,))
    G = mm.discrete_grad(grid, u)
    np.testing.assert_allclose(G, oracle.core.stencil_grad(3, 12, 0.4, u), atol=1e-12)
    T = rng.standard_normal(grid.shape + (3, 3))
    dv = mm.discrete_div(grid, T)
    ref = sum(oracle.core.stencil_grad(3, 12, 0.4, T[..., j])[..., j] for j in range(3))
    np.testing.assert_allclose(dv, ref, atol=1e-12)


# ---------------------------------------------------------------------------
# full outer iterations
# ---------------------------------------------------------------------------

def _traj(g, dim):
    n, L = int(g["n"]), float(g["L"])
    grid = mm.Grid(dim, n, L)
    m = mm.MooneyRivlin(g["mu"], g["kappa"], dim=dim, mu_rep=float(g["mu_rep"]))
    bc = mm.MacroBC(g["mask"], g["value"])
    params = mm.SolverParams(max_outer=int(g["K"]))
    st = mm.solver.init_state(grid, m, bc, params)
    if "F0" in g:
        st.F = g["F0"].copy()
    st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                     raise_on_max=False)
    return st


@pytest.mark.parametrize("name,dim", [("traj_mr2d", 2), ("traj_mr3d", 3)])
def test_trajectory_matches_reference(name, dim):
    g = golden(name)
    st = _traj(g, dim)
    hist = np.array([r[:5] for r in st.history])
    assert np.array_equal(hist[:, 0], g["hist"][:, 0])
    # r_l at the stationarity noise floor (~1e-11) is roundoff: absolute floor
    np.testing.assert_allclose(hist[:, 1:], g["hist"][:, 1:], rtol=1e-9, atol=1e-11)
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(getattr(st, k), g[k]) < 1e-10, k
    assert st.total_sweeps == int(g["total_sweeps"])


def _laminate(dim, n, axis):
    grid = mm.Grid(dim, n, 0.5)
    x = grid.coords()[..., axis]
    phase = ((x + grid.length) / (2 * grid.length) < 0.5)
    chi = phase.ravel().astype(float)
    mu = 1.0 + (1.0 / 20.0 - 1.0) * chi
    return grid, mu, 9.8 * mu


@pytest.mark.parametrize("n,K", [(16, 15), (32, 10)])
def test_3d_laminate_matches_oracle(n, K):
    """SURVEY §8(d) config 2 inputs at oracle-feasible sizes: K iterations."""
    grid, mu, kap = _laminate(3, n, 0)
    Fbar = np.diag([0.95, 1.0, 1.0])
    bc = mm.MacroBC.strain(Fbar)
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    params = mm.SolverParams(max_outer=K)
    st = mm.solver.init_state(grid, m, bc, params)
    F0 = st.F + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape)
    st.F = F0.copy()  # solve() writes F back into the array it was given
    st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                     raise_on_max=False)
    om = oracle.MR(mu, kap, dim=3, mu_rep=1.0)
    op = oracle.Params(max_outer=K)
    ost = oracle.init_state(3, n, om, bc.strain_mask, bc.value, op)
    ost.F = F0.copy()
    ost, _ = oracle.solve(3, n, 0.5, om, bc.strain_mask, bc.value, op,
                          policy=oracle.RatioToDual(0.3), state=ost, raise_on_max=False)
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(getattr(st, k), getattr(ost, k)) < 1e-10, k
    assert st.total_sweeps == ost.total_sweeps
    hist = np.array([r[:5] for r in st.history])
    np.testing.assert_allclose(hist, np.array(ost.history), rtol=1e-9)


def test_config1_load_step_history():
    """same cumulative outer-iteration history as the
    reference (2D 64^2 laminate, monodomain mask, lam 1.0 -> 0.8)."""
    g = golden("config1_protocol")
    n = int(g["n"])
    grid = mm.Grid(2, n, 0.5)
    m = mm.MooneyRivlin(g["mu"], g["kappa"], dim=2, mu_rep=1.0)
    params = mm.SolverParams()
    pol = mm.RatioToDual(0.3)
    bc0 = mm.MacroBC.stress(np.zeros((2, 2)))
    st, ok = mm.solve(grid, m, bc0, params, policy=pol, raise_on_max=False)
    assert ok
    ref = st.u_mean.copy()
    mask = np.zeros((2, 2), bool)
    for ij in ((0, 0), (0, 1), (1, 0)):
        mask[ij] = True
    iters, nominal = [], []
    for step, lam in enumerate(g["lams"]):
        P = np.eye(2)
        P[0, 0] = lam
        bc = mm.MacroBC(mask, np.where(mask, P @ ref, 0.0))
        rng = np.random.default_rng(np.random.SeedSequence((0, step)))
        st.F = st.F + 1e-4 * rng.standard_normal(st.F.shape)
        st, ok = mm.solve(grid, m, bc, params, policy=pol, state=st, raise_on_max=False)
        assert ok
        iters.append(st.outer_iter)
        nominal.append(mm.macro_stress(grid, st))
    assert iters == list(g["outer_iters"])
    np.testing.assert_allclose(np.array(nominal), g["nominal"], rtol=1e-8, atol=1e-12)
    assert rel_l2(st.F, g["F"]) < 1e-10
    assert rel_l2(st.lam, g["lam"]) < 1e-10


def test_split_run_bitwise_continuation():
    """reference test_solver.py:245-264: a run split in two equals one run."""
    rng = np.random.default_rng(41)
    grid = mm.Grid(2, 8)
    mu = np.where(rng.random(grid.npoints) < 0.3, 1.0, 20.0)
    m = mm.MooneyRivlin(mu=mu, kappa=9.8 * mu, dim=2, mu_rep=20.0)
    bc = mm.MacroBC.strain(np.array([[0.95, 0.02], [0.0, 1.01]]))
    st_a, _ = mm.solve(grid, m, bc, mm.SolverParams(max_outer=7), raise_on_max=False)
    st_a, conv_a = mm.solve(grid, m, bc, mm.SolverParams(max_outer=600), state=st_a)
    st_b, conv_b = mm.solve(grid, m, bc, mm.SolverParams(max_outer=600))
    assert conv_a and conv_b
    assert st_a.outer_iter == st_b.outer_iter
    assert np.array_equal(st_a.grad_u, st_b.grad_u)
    assert np.array_equal(st_a.lam, st_b.lam)
    assert st_a.history[-1][:5] == st_b.history[-1][:5]


def test_quadratic_dense_least_squares():
    """reference test_solver.py:80-90: the splitting reproduces the dense
    weighted least-squares equilibrium for a quadratic energy."""
    rng = np.random.default_rng(5)
    grid = mm.Grid(dim=2, n=6)
    c = rng.uniform(0.5, 3.0, grid.npoints)
    m = mm.QuadraticMaterial(c=c, dim=2)
    Fbar = np.array([[1.0, 0.08], [0.02, 0.97]])
    params = mm.SolverParams(r_p_tol=1e-10, r_d_tol=1e-10, max_outer=60000)
    state, conv = mm.solve(grid, m, mm.MacroBC.strain(Fbar), params)
    assert conv
    d, npts, h = 2, grid.npoints, grid.h
    idx = np.arange(npts).reshape(grid.shape)
    Ds = []
    for axis in range(d):
        D = np.zeros((npts, npts))
        D[np.arange(npts), np.roll(idx, -1, axis=axis).ravel()] += 1.0 / (2 * h)
        D[np.arange(npts), np.roll(idx, 1, axis=axis).ravel()] -= 1.0 / (2 * h)
        Ds.append(D)
    A = np.zeros((npts * d * d, npts * d))
    for i in range(d):
        for j in range(d):
            A[np.ix_((np.arange(npts) * d + i) * d + j, np.arange(npts) * d + i)] = Ds[j]
    b = np.tile(Fbar.ravel(), npts)
    w = np.repeat(np.sqrt(c), d * d)
    u, *_ = np.linalg.lstsq(w[:, None] * A, -w * b, rcond=None)
    Fexact = (b + A @ u).reshape(npts, d, d)
    assert np.abs(state.grad_u.reshape(-1, 2, 2) - Fexact).max() < 5e-9


def test_divergence_guard():
    grid = mm.Grid(2, 8)
    m = mm.MooneyRivlin(mu=1.0, kappa=9.8, dim=2)
    bc = mm.MacroBC.strain(np.array([[0.9, 0.0], [0.0, 1.0]]))
    with pytest.raises(mm.DivergenceError):
        mm.solve(grid, m, bc, mm.SolverParams(divergence_limit=1e-12))


def test_stress_control_pins_mean_multiplier():
    rng = np.random.default_rng(21)
    grid = mm.Grid(2, 8)
    mu = np.where(rng.random(grid.npoints) < 0.3, 1.0, 20.0)
    m = mm.MooneyRivlin(mu=mu, kappa=9.8 * mu, dim=2, mu_rep=20.0)
    Sbar = np.array([[0.5, 0.1], [0.1, -0.2]])
    state, conv = mm.solve(grid, m, mm.MacroBC.stress(Sbar), mm.SolverParams(max_outer=2000))
    assert conv
    np.testing.assert_allclose(mm.macro_stress(grid, state), Sbar, atol=1e-12)
    np.testing.assert_allclose(mm.mean_field(grid, state.lam), Sbar, atol=1e-12)


# ---------------------------------------------------------------------------
# size-independent properties at BASELINE sizes
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n", [128, 256])
def test_large_grid_invariants(n):
    """After one outer iteration at config-2/3 sizes: the ascended multiplier
    is discretely solenoidal, <grad u> equals the pinned mean, and the
    fluctuation is mean-free (properties the reference asserts on small grids,
    test_solver.py:92-99, test_projection.py:87-104)."""
    grid, mu, kap = _laminate(3, n, 0)
    Fbar = np.diag([0.95, 1.0, 1.0])
    bc = mm.MacroBC.strain(Fbar)
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    params = mm.SolverParams(max_outer=2)
    st = mm.solver.init_state(grid, m, bc, params)
    st.F = st.F + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape)
    st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                     raise_on_max=False)
    lam = st.lam
    div = mm.discrete_div(grid, lam)
    assert np.sqrt(np.mean(div ** 2)) < 1e-9 * max(1.0, np.abs(lam).max())
    np.testing.assert_allclose(mm.mean_field(grid, st.grad_u), Fbar, atol=1e-12)
    assert np.abs(mm.mean_field(grid, st.u_tilde)).max() < 1e-13


def test_device_log_accuracy():
    """The table-driven log of the MR objective (csrc/mm_local.cu log_pos)
    against an 80-bit reference: absolute error far below one ulp of the
    objective near J = 1, <= 1 ulp relative elsewhere, libm fallback for
    non-normal arguments."""
    rng = np.random.default_rng(3)
    near = 1.0 + np.concatenate([rng.uniform(-0.3, 0.3, 20000),
                                 rng.standard_normal(20000) * 1e-3,
                                 rng.standard_normal(5000) * 1e-8, [0.0, 1e-16, -1e-16]])
    wide = np.exp(rng.uniform(-700, 700, 20000))
    edge = np.array([np.finfo(float).tiny, 5e-324, 1e-310, np.finfo(float).max, 0.6875,
                     1.375, np.nextafter(0.6875, 0), np.nextafter(1.375, 2), 0.5, 2.0])
    x = np.concatenate([near, wide, edge])
    ctx = mm._lib.Context(3, npts=8)
    y = ctx.selftest_log(x)
    ref = np.log(x.astype(np.longdouble))
    err = np.abs(y.astype(np.longdouble) - ref)
    ulp = np.spacing(np.abs(ref.astype(float)))
    # the objective needs log J to absolute accuracy (it enters as I1 - 2 log J
    # - d with I1 ~ d, and decisions are only taken on decreases above
    # 64 eps (|phi| + phi_scale), base.py:168-171)
    m = np.abs(x - 1.0) < 0.05
    assert float(np.max(err[m])) < 4e-18
    far = np.abs(x - 1.0) >= 0.3
    assert float(np.max(err[far] / ulp[far])) <= 1.0
    assert np.isneginf(ctx.selftest_log(np.array([0.0])))[0]


@pytest.mark.parametrize("n", [16, 32, 64, 128, 256])
def test_plane_fft_matches_row_layout(n, monkeypatch):
    """The single-launch cluster pass over (component, k2) planes (k_plane)
    performs the column sequence's per-line arithmetic; the compiler may
    contract a complex product's two roundings differently in the two
    kernels, so whole outer iterations agree with MM_PLANE_FFT=0 (three
    launches) to roundoff (1e-13 relative L2), the history to 1e-11."""
    grid, mu, kap = _laminate(3, n, 0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    params = mm.SolverParams(max_outer=3)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("MM_PLANE_FFT", flag)
        st = mm.solver.init_state(grid, m, bc, params)
        st.F = st.F + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape)
        st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        out[flag] = (st.F.copy(), st.lam.copy(), st.u_tilde.copy(), st.history[-1][:5])
    for a, b in zip(out["1"][:3], out["0"][:3]):
        assert rel_l2(a, b) < 1e-13
    assert out["1"][3][0] == out["0"][3][0]
    np.testing.assert_allclose(out["1"][3][1:], out["0"][3][1:], rtol=1e-11)


def test_row_fwd_warp_kernel_matches_tiled():
    """n = 256: the warp-per-task R2C rows (k_row_fwd_w, MM_OPT_ROWFWD_WARP)
    perform tile_fft<16, 8>'s four-step and k_row_fwd's stencil and split in
    the same order, with the step-1 twiddles formed from four table loads and
    products (MM_RFW_TWP; with table twiddles the two kernels agree bit for
    bit); whole outer iterations agree with the block-tiled kernel to
    roundoff, sweep counts exactly."""
    import os
    grid, mu, kap = _laminate(3, 256, 0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    params = mm.SolverParams(max_outer=3)
    out = {}
    for flag in ("1", "0"):
        os.environ["MM_ROWFWD_WARP"] = flag
        try:
            st = mm.solver.init_state(grid, m, bc, params)
            st.F = st.F + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape)
            st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                             raise_on_max=False)
        finally:
            del os.environ["MM_ROWFWD_WARP"]
        out[flag] = ([np.array(getattr(st, k)) for k in ("F", "lam", "grad_u", "u_tilde")],
                     st.history[-1][:5], st.total_sweeps)
        del st
    bitwise = all(np.array_equal(a, b) for a, b in zip(out["1"][0], out["0"][0]))
    print("row_fwd warp vs tiled bitwise:", bitwise)
    for a, b in zip(out["1"][0], out["0"][0]):
        assert rel_l2(a, b) < 1e-13
    assert out["1"][2] == out["0"][2]
    np.testing.assert_allclose(out["1"][1][1:], out["0"][1][1:], rtol=1e-11)


def test_solve_updates_caller_F_and_lam_in_place():
    """The reference's local step writes F in place (base.py:109-111) and the
    ascent does lam += ... (solver.py:279): arrays the caller handed in as F
    and lam hold the final values after solve(), and are the state's
    (read-only) F and lam; a read-only caller array is left untouched."""
    grid, mu, kap = _laminate(3, 8, 0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    params = mm.SolverParams(max_outer=5)
    runs = []
    for writeable in (True, False):
        st = mm.solver.init_state(grid, m, bc, params)
        F0 = np.ascontiguousarray(st.F + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape))
        lam0 = np.zeros_like(F0)
        keep = (F0.copy(), lam0.copy())
        F0.flags.writeable = writeable
        lam0.flags.writeable = writeable
        st.F, st.lam = F0, lam0
        st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        if writeable:
            assert st.F is F0 and st.lam is lam0
            assert not F0.flags.writeable
            # the arrays stay the state's F / lam through later solves, and
            # receive every solve's result (reference: state.F keeps identity)
            st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                             raise_on_max=False)
            assert st.F is F0 and st.lam is lam0
            eng = st._engine
            assert np.array_equal(F0, eng.ctx.download(mm._lib.FIELD_F, F0.shape))
            assert np.array_equal(lam0, eng.ctx.download(mm._lib.FIELD_LAM, lam0.shape))
        else:
            assert np.array_equal(F0, keep[0]) and np.array_equal(lam0, keep[1])
            st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                             raise_on_max=False)
        runs.append((np.array(st.F), np.array(st.lam)))
    assert np.array_equal(runs[0][0], runs[1][0]) and np.array_equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("n,K", [(16, 12), (64, 6)])
def test_speculative_projection_front_is_exact(n, K, monkeypatch):
    """mm_update_and_sweep queues the next projection's rows / column passes /
    C2R behind the fused pass (MM_OPT_SPECULATE); whether they are used or
    recomputed (an extra local chunk, a host access in between), every field
    and the history equal the non-speculative run bit for bit."""
    grid, mu, kap = _laminate(3, n, 0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    out = {}
    for flag in ("1", "0"):
        monkeypatch.setenv("MM_SPECULATE", flag)
        params = mm.SolverParams(max_outer=K // 2)
        st = mm.solver.init_state(grid, m, bc, params)
        st.F = st.F + 1e-3 * np.random.default_rng(0).standard_normal(st.F.shape)
        st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        _ = st.grad_u  # host access between two solves
        st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        out[flag] = ([np.array(getattr(st, k)) for k in ("F", "lam", "grad_u", "u_tilde")],
                     [r[:5] for r in st.history], st.total_sweeps)
    for a, b in zip(out["1"][0], out["0"][0]):
        assert np.array_equal(a, b)
    assert out["1"][1] == out["0"][1] and out["1"][2] == out["0"][2]


@pytest.mark.parametrize("dim,n,pol", [(2, 32, "ratio"), (3, 16, "ratio"), (3, 16, "exact"),
                                       (2, 16, "fraction"), (3, 16, "mixed")])
def test_library_decision_step_matches_host_loop(dim, n, pol, monkeypatch):
    """mm_residuals_and_step takes the loop's decisions (r_d, r_p, guard,
    penalty update, convergence, policy tolerance) in the library -- on the
    device, ahead of the host, when pipelined; fields, history and sweeps
    equal the host-decided loop (MM_HOST_DECIDE=1) bit for bit, through
    convergence."""
    grid, mu, kap = _laminate(dim, n, 0)
    Fbar = np.eye(dim)
    Fbar[0, 0] = 0.95
    bc = mm.MacroBC.strain(Fbar)
    if pol == "mixed":  # F_00 prescribed, the other entries stress-free (u_mean from sum F)
        bc = mm.MacroBC.mixed({(0, 0): 0.95},
                              {(i, j): 0.0 for i in range(dim) for j in range(dim)
                               if (i, j) != (0, 0)}, dim)
    m = mm.MooneyRivlin(mu, kap, dim=dim, mu_rep=1.0)
    policy = {"ratio": mm.RatioToDual(0.3), "exact": mm.ExactAll(),
              "fraction": mm.FractionConverged(0.9, 2), "mixed": mm.RatioToDual(0.3)}[pol]
    params = mm.SolverParams(max_outer=400)
    out = {}
    # "0": the library loop (mm_solve_fused; K1, the device-side decision and
    # the next fused pass queued back to back, MM_OPT_PIPELINE); "nopipe": the
    # same with the host deciding between K1 and the fused pass; "py": the
    # Python loop over mm_residuals_and_step; "1": the host-decided loop
    for flag in ("0", "nopipe", "py", "1"):
        monkeypatch.setenv("MM_HOST_DECIDE", "1" if flag == "1" else "0")
        monkeypatch.setenv("MM_C_LOOP", "0" if flag == "py" else "1")
        monkeypatch.setenv("MM_PIPELINE", "0" if flag == "nopipe" else "1")
        st = mm.solver.init_state(grid, m, bc, params)
        st.F = st.F + 1e-3 * np.random.default_rng(1).standard_normal(st.F.shape)
        st, conv = mm.solve(grid, m, bc, params, policy=policy, state=st, raise_on_max=False)
        out[flag] = (conv, [np.array(getattr(st, k)) for k in ("F", "lam", "grad_u", "u_tilde")],
                     [r[:5] for r in st.history], st.total_sweeps, st.rho)
    for other in ("nopipe", "py", "1"):
        a, b = out["0"], out[other]
        assert a[0] == b[0] and a[2] == b[2] and a[3] == b[3] and a[4] == b[4]
        for x, y in zip(a[1], b[1]):
            assert np.array_equal(x, y)


def test_reassigned_moduli_reach_the_device():
    """Assigning new moduli to a model between solves on the same state is
    seen by the device (upload + energy scale), as the reference re-reads
    them on every local_sweeps call (mooney_rivlin.py:111-116): the result
    equals a solve with a fresh model holding the new moduli."""
    grid, mu, kap = _laminate(3, 8, 0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    params = mm.SolverParams(max_outer=3)
    out = []
    for reassign in (True, False):
        m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
        st = mm.solver.init_state(grid, m, bc, params)
        st.F = st.F + 1e-3 * np.random.default_rng(0).standard_normal(st.F.shape)
        st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        if reassign:
            m.mu = 3.0 * mu
            m.kappa = 2.0 * kap
        else:
            m = mm.MooneyRivlin(3.0 * mu, 2.0 * kap, dim=3, mu_rep=1.0)
        st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        out.append((np.array(st.F), np.array(st.lam), [r[:5] for r in st.history]))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert out[0][2] == out[1][2]


@pytest.mark.parametrize("n,K", [(24, 8), (40, 6)])
def test_mixed_radix_grid_trajectory_matches_oracle(n, K):
    """Non-power-of-two 3D grids run the row layout with mixed-radix line
    FFTs (radices 4, 2, 3, 5): whole outer iterations against the oracle."""
    grid, mu, kap = _laminate(3, n, 0)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    params = mm.SolverParams(max_outer=K)
    st = mm.solver.init_state(grid, m, bc, params)
    F0 = np.array(st.F) + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape)
    st.F = F0.copy()
    st, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=st,
                     raise_on_max=False)
    om = oracle.MR(mu, kap, dim=3, mu_rep=1.0)
    op = oracle.Params(max_outer=K)
    ost = oracle.init_state(3, n, om, bc.strain_mask, bc.value, op)
    ost.F = F0.copy()
    ost, _ = oracle.solve(3, n, 0.5, om, bc.strain_mask, bc.value, op,
                          policy=oracle.RatioToDual(0.3), state=ost, raise_on_max=False)
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(getattr(st, k), getattr(ost, k)) < 1e-10, k
    assert st.total_sweeps == ost.total_sweeps
