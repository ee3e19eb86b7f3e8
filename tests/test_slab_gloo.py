"""Multi-rank slab decomposition tested on CPU with gloo.

The orchestration in paper_2010_06697_b200/slab.py (slab partition, T and u
halo exchanges, the two all-to-all transposes, global frequency indexing in
the fused axis-0 pass, rank-ordered reductions) runs with world_size 2 and 4
over gloo, with the host restatement of the per-rank steps
(NumpySlabBackend, same buffer layouts as the device kernels), and must
reproduce the single-process oracle projection + multiplier ascent.
"""

import os
import socket
import tempfile

import numpy as np
import pytest

import oracle
from paper_2010_06697_b200.grid import Grid, axis_symbol_tables
from paper_2010_06697_b200.slab import NumpySlabBackend, SlabLayout, SlabProjector, TorchComm


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(n, seed):
    rng = np.random.default_rng(seed)
    F = np.eye(3) + 0.1 * rng.standard_normal((n, n, n, 3, 3))
    lam = 0.3 * rng.standard_normal((n, n, n, 3, 3))
    G = np.eye(3) + 0.05 * rng.standard_normal((n, n, n, 3, 3))
    rho = 2.7
    mask = np.array([[1, 0, 1], [0, 1, 0], [1, 1, 1]], bool)
    value = np.eye(3) + 0.02 * rng.standard_normal((3, 3))
    return F, lam, G, rho, mask, value


def _rank_main(rank, world, port, n, seed, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        F, lam, G, rho, mask, value = _problem(n, seed)
        lay = SlabLayout(n, world, rank, 0.5)
        sl = lay.plane_slice()
        tab, thr = axis_symbol_tables(Grid(3, n, 0.5))
        be = NumpySlabBackend(lay, F[sl], lam[sl], G[sl], tab, thr)
        comm = TorchComm(dist)
        # macro control from the global means (ordered sums)
        Fm = comm.ordered_sum(F[sl].reshape(-1, 9).sum(axis=0)) / n ** 3
        Lm = comm.ordered_sum(lam[sl].reshape(-1, 9).sum(axis=0)) / n ** 3
        u_mean = np.where(mask, value, Fm.reshape(3, 3) - (Lm.reshape(3, 3) - value) / rho)
        sums = SlabProjector(lay, be, comm).project_update(rho, u_mean)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), u=be.u, G=be.G, lam=be.lam, sums=sums,
                 u_mean=u_mean)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(8, 2), (12, 2), (8, 4)])
def test_slab_projection_matches_single_process(n, world):
    import torch.multiprocessing as mp
    seed = 7 + n + world
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_rank_main, args=(world, _free_port(), n, seed, td), nprocs=world, join=True)
        parts = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(world)]
        u = np.concatenate([p["u"] for p in parts], axis=0)
        G = np.concatenate([p["G"] for p in parts], axis=0)
        lam_new = np.concatenate([p["lam"] for p in parts], axis=0)
        sums = parts[0]["sums"]
        for p in parts[1:]:
            assert np.array_equal(p["sums"], sums)  # every rank holds the same totals
    F, lam, G0, rho, mask, value = _problem(n, seed)
    u_mean, u_tilde, grad_u = oracle.project(3, n, 0.5, F, lam, rho, mask, value)
    np.testing.assert_allclose(parts[0]["u_mean"], u_mean, rtol=0, atol=1e-14)
    scale = np.abs(u_tilde).max()
    np.testing.assert_allclose(u, u_tilde, rtol=0, atol=1e-12 * scale)
    np.testing.assert_allclose(G, grad_u, rtol=0, atol=1e-12)
    lam_ref = lam + rho * (grad_u - F)
    np.testing.assert_allclose(lam_new, lam_ref, rtol=0, atol=1e-12)
    dG = grad_u - G0
    mis = grad_u - F
    np.testing.assert_allclose(sums[0], np.sum(dG * dG), rtol=1e-12)
    np.testing.assert_allclose(sums[1], np.sum(mis * mis), rtol=1e-12)
    np.testing.assert_allclose(sums[2:], lam_ref.reshape(-1, 9).sum(axis=0), rtol=1e-10, atol=1e-10)


def test_layout_validation():
    with pytest.raises(ValueError):
        SlabLayout(10, 3, 0)
    lay = SlabLayout(16, 4, 2)
    assert lay.nl == 4 and lay.i0 == 8 and lay.neighbours() == (1, 3)
