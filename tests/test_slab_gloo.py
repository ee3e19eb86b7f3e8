"""Multi-rank slab decomposition tested on CPU with gloo.

solve(..., comm=...) -- the real solver loop, SlabContext and TorchComm of
paper_2010_06697_b200 -- runs with world_size 2 and 4 over gloo; the
per-rank compute is the host restatement of the device steps
(tests/slab_numpy_backend.py, same buffer layouts, oracle local kernels).
The orchestration under test: slab partition, T halos, the two all-to-all
transposes, global frequency indexing in the axis-0 pass, u ghost planes
for the residual / ascent stencils, two-plane director ghosts for the LCE
Frank stencil, rank-ordered reductions, identical decisions on every rank.
Reference: the single-process oracle (reference algorithm) on the whole grid.
"""

import os
import socket
import tempfile

import numpy as np
import pytest

import oracle
import paper_2010_06697_b200 as mm
from paper_2010_06697_b200.slab import SlabLayout, TorchComm, local_planes, local_points


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class HostComm(TorchComm):
    """gloo communicator whose slab backend is the host restatement."""

    def __init__(self, dist):
        super().__init__(dist, None, exchange="collective")

    def make_backend(self, lay):
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from slab_numpy_backend import NumpySlabBackend
        return NumpySlabBackend(lay)


def _mr_problem(n):
    x = -0.5 + np.arange(n) / n
    chi = np.broadcast_to(((x + 0.5) < 0.5).astype(float).reshape(n, 1, 1), (n, n, n)).ravel()
    mu = 1.0 + (1.0 / 20.0 - 1.0) * chi
    F0 = np.broadcast_to(np.diag([0.95, 1.0, 1.0]), (n, n, n, 3, 3)) + \
        1e-3 * np.random.default_rng(n).standard_normal((n, n, n, 3, 3))
    return mu, 9.8 * mu, F0


def _lce_problem(n):
    n0 = oracle.polydomain_n0(3, n, 0.5, 0.25, seed=1)
    F0 = np.broadcast_to(np.eye(3), (n, n, n, 3, 3)) + \
        1e-3 * np.random.default_rng(3).standard_normal((n, n, n, 3, 3))
    return n0, F0


LCE_KW = dict(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, dim=3)


def _rank_main(rank, world, port, case, n, K, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = HostComm(dist)
        grid = mm.Grid(3, n, 0.5)
        sl, pts = local_planes(grid, comm), local_points(grid, comm)
        if case == "mr":
            mu, kap, F0 = _mr_problem(n)
            model = mm.MooneyRivlin(mu[pts], kap[pts], dim=3, mu_rep=1.0)
            bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
            params = mm.SolverParams(max_outer=K)
        else:
            n0, F0 = _lce_problem(n)
            model = mm.LiquidCrystalElastomer(n0=n0[pts], **LCE_KW)
            bc = mm.MacroBC.stress(np.zeros((3, 3)))
            params = mm.SolverParams(max_outer=K, max_local=5)
        st = mm.solver.init_state(grid, model, bc, params, comm=comm)
        st.F = np.array(F0[sl])
        st, _ = mm.solve(grid, model, bc, params, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False, comm=comm)
        out = {k: np.array(getattr(st, k)) for k in ("F", "lam", "grad_u", "u_tilde")}
        if case == "lce":
            out["angles"] = np.array(st.internal["angles"])
            out["chart"] = np.array(st.internal["chart"])
        np.savez(os.path.join(outdir, f"r{rank}.npz"),
                 hist=np.array([h[:5] for h in st.history]), sweeps=st.total_sweeps,
                 stress=mm.macro_stress(grid, st), **out)
    finally:
        dist.destroy_process_group()


def _gather(td, world):
    parts = [dict(np.load(os.path.join(td, f"r{r}.npz"))) for r in range(world)]
    for p in parts[1:]:   # identical decisions and reductions on every rank
        assert np.array_equal(p["hist"], parts[0]["hist"])
        assert p["sweeps"] == parts[0]["sweeps"]
        assert np.array_equal(p["stress"], parts[0]["stress"])
    return parts


@pytest.mark.parametrize("n,world,K", [(8, 2, 6), (16, 2, 5), (8, 4, 6)])
def test_slab_solve_mr_matches_oracle(n, world, K):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_rank_main, args=(world, _free_port(), "mr", n, K, td), nprocs=world, join=True)
        parts = _gather(td, world)
    mu, kap, F0 = _mr_problem(n)
    om = oracle.MR(mu, kap, dim=3, mu_rep=1.0)
    mask, val = np.ones((3, 3), bool), np.diag([0.95, 1.0, 1.0])
    op = oracle.Params(max_outer=K)
    ost = oracle.init_state(3, n, om, mask, val, op)
    ost.F = np.array(F0)
    ost, _ = oracle.solve(3, n, 0.5, om, mask, val, op, policy=oracle.RatioToDual(0.3),
                          state=ost, raise_on_max=False)
    for k in ("F", "lam", "grad_u", "u_tilde"):
        full = np.concatenate([p[k] for p in parts], axis=0)
        ref = getattr(ost, k)
        assert np.linalg.norm(full - ref) / np.linalg.norm(ref) < 1e-10, k
    assert int(parts[0]["sweeps"]) == ost.total_sweeps
    np.testing.assert_allclose(parts[0]["hist"], np.array(ost.history), rtol=1e-9)
    np.testing.assert_allclose(parts[0]["stress"], oracle.macro_stress(ost, 3), rtol=1e-10,
                               atol=1e-15)


@pytest.mark.parametrize("n,world", [(8, 2), (8, 4)])
def test_slab_solve_lce_matches_oracle(n, world):
    """Config-3 material (polydomain director) over 2 and 4 ranks: the Frank
    force from two-plane director ghosts (nl = 2 at world 4: the stencil
    reaches across a whole neighbour slab), LCE internals per slab."""
    import torch.multiprocessing as mp
    K = 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_rank_main, args=(world, _free_port(), "lce", n, K, td), nprocs=world, join=True)
        parts = _gather(td, world)
    n0, F0 = _lce_problem(n)
    om = oracle.LCE(n0=n0, **LCE_KW)
    mask, val = np.zeros((3, 3), bool), np.zeros((3, 3))
    op = oracle.Params(max_outer=K, max_local=5)
    ost = oracle.init_state(3, n, om, mask, val, op)
    ost.F = np.array(F0)
    ost, _ = oracle.solve(3, n, 0.5, om, mask, val, op, policy=oracle.RatioToDual(0.3),
                          state=ost, raise_on_max=False)
    for k in ("F", "lam", "grad_u", "u_tilde"):
        full = np.concatenate([p[k] for p in parts], axis=0)
        ref = getattr(ost, k)
        assert np.linalg.norm(full - ref) / np.linalg.norm(ref) < 1e-9, k
    ang = np.concatenate([p["angles"] for p in parts], axis=0)
    assert np.linalg.norm(ang - ost.internal["angles"]) / np.linalg.norm(ang) < 1e-9
    assert int(parts[0]["sweeps"]) == ost.total_sweeps


def test_layout_validation():
    with pytest.raises(mm.ConfigurationError):
        SlabLayout(10, 3, 0)
    with pytest.raises(mm.ConfigurationError):
        SlabLayout(9, 3, 0)
    lay = SlabLayout(16, 4, 2)
    assert lay.nl == 4 and lay.i0 == 8 and lay.neighbours() == (1, 3)
    assert lay.point_slice() == slice(8 * 256, 12 * 256)
