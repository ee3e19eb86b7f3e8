"""Device slab decomposition on one GPU: P virtual ranks (threads, one
context each, exchanges through ThreadComm; every kernel runs to completion
on its own) must reproduce the single-context solver (1-vs-P
field equality)."""

import threading

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_2010_06697_b200")


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _problem(n):
    grid = mm.Grid(3, n, 0.5)
    x = grid.coords()[..., 0]
    chi = ((x + 0.5) < 0.5).ravel().astype(float)
    mu = 1.0 + (0.05 - 1.0) * chi
    kap = 9.8 * mu
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    F = np.broadcast_to(bc.value, grid.shape + (3, 3)).copy()
    F = F + 1e-3 * np.random.default_rng(0).standard_normal(F.shape)
    G = np.broadcast_to(bc.value, grid.shape + (3, 3)).copy()
    lam = np.zeros_like(F)
    return grid, mu, kap, bc, F, G, lam


@pytest.mark.parametrize("n,P,K", [(16, 2, 6), (32, 4, 6), (32, 1, 4)])
def test_slab_solver_matches_single_gpu(n, P, K):
    from paper_2010_06697_b200.slab import SlabLayout, SlabSolver, ThreadComm
    grid, mu, kap, bc, F, G, lam = _problem(n)
    params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
    pol = mm.RatioToDual(0.3)
    # single context
    model = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    st = mm.ADMMState(u_mean=bc.value.copy(), u_tilde=np.zeros(grid.shape + (3,)), grad_u=G,
                      F=F, lam=lam, internal={}, rho=1.0)
    st, _ = mm.solve(grid, model, bc, params, policy=pol, state=st, raise_on_max=False)
    # P virtual ranks
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": {}}
    out = [None] * P
    err = []

    def rank_main(r):
        try:
            lay = SlabLayout(n, P, r, 0.5)
            sl = lay.plane_slice()
            pts = slice(r * lay.npts_local, (r + 1) * lay.npts_local)
            mloc = mm.MooneyRivlin(mu[pts], kap[pts], dim=3, mu_rep=1.0)
            mloc._phi_cache = ((id(mloc.mu), id(mloc.kappa)), float(mu.max() + kap.max()))
            sv = SlabSolver(lay, mloc, bc, params, pol, ThreadComm(shared, r), F[sl], G[sl],
                            lam[sl])
            sv.solve()
            out[r] = (sv.fields(), sv.history, sv.total_sweeps)
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            shared["barrier"].abort()

    ths = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]
    fields = {k: np.concatenate([o[0][k] for o in out], axis=0) for k in out[0][0]}
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(fields[k], getattr(st, k)) < 1e-12, k
    h_slab = np.array([r[:5] for r in out[0][1]])
    h_one = np.array([r[:5] for r in st.history])
    np.testing.assert_allclose(h_slab, h_one, rtol=1e-10, atol=1e-14)
    assert out[0][2] == st.total_sweeps
