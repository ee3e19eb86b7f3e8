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


@pytest.mark.parametrize("n,P,K,exchange", [(16, 2, 6, "collective"), (32, 4, 6, "collective"),
                                            (32, 1, 4, "collective"), (16, 2, 6, "push"),
                                            (32, 4, 6, "push"), (64, 2, 5, "push"),
                                            (64, 4, 5, "collective"), (64, 4, 5, "push")])
def test_slab_solver_matches_single_gpu(n, P, K, exchange):
    from paper_2010_06697_b200.slab import SlabLayout, SlabSolver, ThreadComm
    grid, mu, kap, bc, F, G, lam = _problem(n)
    params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
    pol = mm.RatioToDual(0.3)
    # single context
    model = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    # copies: solve() writes F and lam back into the arrays it was given
    st = mm.ADMMState(u_mean=bc.value.copy(), u_tilde=np.zeros(grid.shape + (3,)), grad_u=G,
                      F=F.copy(), lam=lam.copy(), internal={}, rho=1.0)
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
            mloc._override_max("phi", mu.max() + kap.max())
            sv = SlabSolver(lay, mloc, bc, params, pol, ThreadComm(shared, r), F[sl], G[sl],
                            lam[sl], exchange=exchange)
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


def _ipc_rank(rank, P, n, K, port, out_dir):
    """One process of the multi-process push test (same GPU, CUDA IPC)."""
    import os
    import torch
    import torch.distributed as dist
    import paper_2010_06697_b200 as mm_
    from paper_2010_06697_b200.slab import SlabLayout, SlabSolver, TorchComm
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=P)
    try:
        torch.cuda.set_device(0)
        grid, mu, kap, bc, F, G, lam = _problem(n)
        lay = SlabLayout(n, P, rank, 0.5)
        sl = lay.plane_slice()
        pts = slice(rank * lay.npts_local, (rank + 1) * lay.npts_local)
        mloc = mm_.MooneyRivlin(mu[pts], kap[pts], dim=3, mu_rep=1.0)
        params = mm_.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
        sv = SlabSolver(lay, mloc, bc, params, mm_.RatioToDual(0.3), TorchComm(dist, "cuda:0"),
                        F[sl], G[sl], lam[sl], exchange="push")
        sv.solve()
        f = sv.fields()
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), hist=np.array(
            [r[:5] for r in sv.history]), sweeps=sv.total_sweeps, **f)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_push_exchange_across_processes_with_ipc(tmp_path):
    """Two processes on one GPU map each other's exchange buffers with CUDA
    IPC handles and run the fused (peer-store) transposes; the result equals
    the single-context solver.  Synchronisation is host-side (gloo barrier),
    so no kernel waits on the other process."""
    import socket
    import torch.multiprocessing as tmp
    n, P, K = 16, 2, 5
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    procs = [ctx.Process(target=_ipc_rank, args=(r, P, n, K, port, str(tmp_path)))
             for r in range(P)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    grid, mu, kap, bc, F, G, lam = _problem(n)
    params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
    model = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    st = mm.ADMMState(u_mean=bc.value.copy(), u_tilde=np.zeros(grid.shape + (3,)), grad_u=G,
                      F=F, lam=lam, internal={}, rho=1.0)
    st, _ = mm.solve(grid, model, bc, params, policy=mm.RatioToDual(0.3), state=st,
                     raise_on_max=False)
    outs = [dict(np.load(tmp_path / f"rank{r}.npz")) for r in range(P)]
    for k in ("F", "lam", "grad_u", "u_tilde"):
        full = np.concatenate([o[k] for o in outs], axis=0)
        assert rel_l2(full, getattr(st, k)) < 1e-12, k
    np.testing.assert_allclose(outs[0]["hist"], np.array([r[:5] for r in st.history]),
                               rtol=1e-10, atol=1e-14)

