"""Device slab decomposition on one GPU: P virtual ranks (threads, one
context each, exchanges through ThreadComm after a stream synchronise; no
kernel ever waits on another rank) run solve(..., comm=...) -- the same
fused loop as one GPU -- and must reproduce the single-context solver
(1-vs-P field equality)."""

import threading

import numpy as np
import pytest

import oracle
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


def _run_ranks(P, body):
    """body(rank, shared) on P threads; returns the per-rank results."""
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": {}}
    out = [None] * P
    err = []

    def main(r):
        try:
            out[r] = body(r, shared)
        except Exception as e:  # pragma: no cover - surfaced below
            err.append(e)
            shared["barrier"].abort()

    ths = [threading.Thread(target=main, args=(r,)) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]
    return out


def _fields(st):
    return {k: np.array(getattr(st, k)) for k in ("F", "lam", "grad_u", "u_tilde")}


@pytest.mark.parametrize("n,P,K,exchange", [(16, 2, 6, "collective"), (32, 4, 6, "collective"),
                                            (32, 1, 4, "collective"), (16, 2, 6, "push"),
                                            (32, 4, 6, "push"), (64, 2, 5, "push"),
                                            (64, 4, 5, "collective"), (64, 4, 5, "push"),
                                            (64, 2, 8, "push")])
def test_slab_solve_matches_single_gpu(n, P, K, exchange):
    from paper_2010_06697_b200.slab import ThreadComm, local_planes, local_points
    grid, mu, kap, bc, F, G, lam = _problem(n)
    params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
    params2 = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=2)
    pol = mm.RatioToDual(0.3)
    model = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    # copies: solve() writes F and lam back into the arrays it was given
    st = mm.ADMMState(u_mean=bc.value.copy(), u_tilde=np.zeros(grid.shape + (3,)), grad_u=G,
                      F=F.copy(), lam=lam.copy(), internal={}, rho=1.0)
    st, _ = mm.solve(grid, model, bc, params, policy=pol, state=st, raise_on_max=False)
    # a second call continues the same device state (warm start)
    st, _ = mm.solve(grid, model, bc, params2, policy=pol, state=st, raise_on_max=False)

    def body(r, shared):
        comm = ThreadComm(shared, r, exchange=exchange)
        sl, pts = local_planes(grid, comm), local_points(grid, comm)
        m = mm.MooneyRivlin(mu[pts], kap[pts], dim=3, mu_rep=1.0)
        s = mm.ADMMState(u_mean=bc.value.copy(), u_tilde=np.zeros((n // P, n, n, 3)),
                         grad_u=G[sl].copy(), F=F[sl].copy(), lam=lam[sl].copy(), internal={},
                         rho=1.0)
        s, _ = mm.solve(grid, m, bc, params, policy=pol, state=s, raise_on_max=False, comm=comm)
        s, _ = mm.solve(grid, m, bc, params2, policy=pol, state=s, raise_on_max=False, comm=comm)
        return _fields(s), [h[:5] for h in s.history], s.total_sweeps, mm.macro_stress(grid, s)

    out = _run_ranks(P, body)
    fields = {k: np.concatenate([o[0][k] for o in out], axis=0) for k in out[0][0]}
    for k in ("F", "lam", "grad_u", "u_tilde"):
        assert rel_l2(fields[k], getattr(st, k)) < 1e-12, k
    h_slab = np.array(out[0][1])
    h_one = np.array([r[:5] for r in st.history])
    np.testing.assert_allclose(h_slab, h_one, rtol=1e-10, atol=1e-14)
    assert out[0][2] == st.total_sweeps
    for o in out[1:]:
        assert o[1] == out[0][1] and o[2] == out[0][2]    # identical decisions on every rank
    lam_mean = fields["lam"].reshape(-1, 3, 3).mean(axis=0)
    print("macro_stress slab", out[0][3].ravel(), "single", mm.macro_stress(grid, st).ravel(),
          "host mean", lam_mean.ravel())
    np.testing.assert_allclose(out[0][3], lam_mean, rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(mm.macro_stress(grid, st), lam_mean, rtol=1e-10, atol=1e-14)


@pytest.mark.parametrize("n,P,K", [(16, 2, 2), (32, 4, 2)])
def test_slab_lce_matches_single_gpu(n, P, K):
    """Config-3 material on a polydomain director, split over P ranks: the
    Frank force from the two-plane director ghosts, LCE internals resident
    per slab, the unfused schedule (outer_iteration: frozen data, local
    chunks, projection + ascent).  Short local budget (max_local 5): the
    non-converging Newton points amplify the slab FFT's different roundoff,
    as they do between any two implementations, so the bar is
    1e-10 or 3x the single-GPU run's own drift under a one-ulp change of F."""
    from paper_2010_06697_b200.slab import ThreadComm, local_planes, local_points
    grid = mm.Grid(3, n, 0.5)
    n0 = oracle.polydomain_n0(3, n, 0.5, 0.25, seed=1)
    kw = dict(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, dim=3)
    bc = mm.MacroBC.stress(np.zeros((3, 3)))
    params = mm.SolverParams(max_outer=K, max_local=5)
    m1 = mm.LiquidCrystalElastomer(n0=n0, **kw)
    st = mm.solver.init_state(grid, m1, bc, params)
    F0 = np.array(st.F) + 1e-3 * np.random.default_rng(3).standard_normal(st.F.shape)
    runs = []
    for Fs in (F0, np.nextafter(F0, np.inf)):   # the second: F moved by one ulp
        st = mm.solver.init_state(grid, m1, bc, params)
        st.F = Fs.copy()
        st, _ = mm.solve(grid, m1, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        f = _fields(st)
        f["angles"] = np.array(st.internal["angles"])
        runs.append((f, np.array([h[:5] for h in st.history]), st.total_sweeps))
    (ref, h_ref, sw_ref), (env, h_env, _) = runs

    def body(r, shared):
        comm = ThreadComm(shared, r)
        sl, pts = local_planes(grid, comm), local_points(grid, comm)
        m = mm.LiquidCrystalElastomer(n0=n0[pts], **kw)
        s = mm.solver.init_state(grid, m, bc, params, comm=comm)
        s.F = F0[sl].copy()
        s, _ = mm.solve(grid, m, bc, params, policy=mm.RatioToDual(0.3), state=s,
                        raise_on_max=False, comm=comm)
        f = _fields(s)
        f["angles"] = np.array(s.internal["angles"])
        return f, [h[:5] for h in s.history], s.total_sweeps

    out = _run_ranks(P, body)
    for k in ref:
        full = np.concatenate([o[0][k] for o in out], axis=0)
        e, en = rel_l2(full, ref[k]), rel_l2(env[k], ref[k])
        print(f"LCE slab {n}^3 P={P} {k}: {e:.3e} (single GPU, F moved by one ulp: {en:.3e})")
        assert e < max(1e-10, 3.0 * en), k
    assert out[0][2] == sw_ref
    h = np.array(out[0][1])
    assert np.array_equal(h[:, 0], h_ref[:, 0])
    dev = np.abs(h[:, 1:] - h_ref[:, 1:]) / np.abs(h_ref[:, 1:])
    dev_env = np.abs(h_env[:, 1:] - h_ref[:, 1:]) / np.abs(h_ref[:, 1:])
    assert np.all(dev.max(axis=0) <= np.maximum(1e-9, 3.0 * dev_env.max(axis=0)))


def test_slab_frank_force_matches_single_gpu():
    """The two-plane ghost exchange of the director reproduces the radius-2
    Frank stencil of the whole grid (lce.py:213-229) bit for bit."""
    from paper_2010_06697_b200 import _lib
    from paper_2010_06697_b200.slab import ThreadComm, local_points
    n, P = 16, 4
    grid = mm.Grid(3, n, 0.5)
    n0 = oracle.polydomain_n0(3, n, 0.5, 0.25, seed=2)
    kw = dict(mu=1.0, r=2.0, alpha=0.1, frank_kappa=3e-3, dim=3)
    m1 = mm.LiquidCrystalElastomer(n0=n0, **kw)
    st = mm.solver.init_state(grid, m1, mm.MacroBC.stress(np.zeros((3, 3))), mm.SolverParams())
    eng = st._attach(grid, m1)
    m1._device_prepare_frozen(eng.ctx)
    ff = eng.ctx.download(_lib.FIELD_FF, (grid.npoints, 3))

    def body(r, shared):
        comm = ThreadComm(shared, r)
        pts = local_points(grid, comm)
        m = mm.LiquidCrystalElastomer(n0=n0[pts], **kw)
        s = mm.solver.init_state(grid, m, mm.MacroBC.stress(np.zeros((3, 3))),
                                 mm.SolverParams(), comm=comm)
        e = s._attach(grid, m)
        m._device_prepare_frozen(e.ctx)
        return e.ctx.download(_lib.FIELD_FF, (e.npts, 3))

    out = _run_ranks(P, body)
    assert np.array_equal(np.concatenate(out, axis=0), ff)


def _ipc_rank(rank, P, n, K, port, out_dir):
    """One process of the multi-process push test (same GPU, CUDA IPC)."""
    import os
    import torch
    import torch.distributed as dist
    import paper_2010_06697_b200 as mm_
    from paper_2010_06697_b200.slab import TorchComm, local_planes, local_points
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=P)
    try:
        torch.cuda.set_device(0)
        grid, mu, kap, bc, F, G, lam = _problem(n)
        comm = TorchComm(dist, 0, exchange="push")
        sl, pts = local_planes(grid, comm), local_points(grid, comm)
        mloc = mm_.MooneyRivlin(mu[pts], kap[pts], dim=3, mu_rep=1.0)
        params = mm_.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
        s = mm_.ADMMState(u_mean=bc.value.copy(), u_tilde=np.zeros((n // P, n, n, 3)),
                          grad_u=G[sl].copy(), F=F[sl].copy(), lam=lam[sl].copy(), internal={},
                          rho=1.0)
        s, _ = mm_.solve(grid, mloc, bc, params, policy=mm_.RatioToDual(0.3), state=s,
                         raise_on_max=False, comm=comm)
        f = _fields(s)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), hist=np.array(
            [r[:5] for r in s.history]), sweeps=s.total_sweeps, **f)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_push_exchange_across_processes_with_ipc(tmp_path):
    """Two processes on one GPU map each other's exchange buffers with CUDA
    IPC handles and run the fused (peer-store) transposes through solve();
    the result equals the single-context solver.  Synchronisation is
    host-side (gloo barrier after a stream synchronise), so no kernel waits on
    the other process."""
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
