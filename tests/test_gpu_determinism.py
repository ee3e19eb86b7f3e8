"""Race evidence without compute-sanitizer (closed on this GPU pool): the
kernels whose correctness depends on intra-kernel synchronisation --
cluster barriers and DSMEM of the plane pass (k_plane), the cp.async double
buffers of the persistent column / C2R kernels (k_colp, k_row_inv_p), the
last-block grid_finalize reductions of every reducing kernel, the shared-
memory accumulators of the fused pass, the slab path's ghost planes and
peer-store transposes -- are run repeatedly on identical inputs, interleaved
with unrelated work that perturbs the scheduling, and every repetition must
reproduce the first bit for bit.  A read-before-write race, a missing
barrier or an unordered reduction shows up as run-to-run variation long
before it shows up as a wrong answer."""

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

mm = pytest.importorskip("paper_2010_06697_b200")


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _laminate(n):
    grid = mm.Grid(3, n, 0.5)
    x = grid.coords()[..., 0]
    chi = ((x + 0.5) < 0.5).ravel().astype(float)
    mu = 1.0 + (0.05 - 1.0) * chi
    return grid, mu, 9.8 * mu


def _run(n, K, seed=0):
    grid, mu, kap = _laminate(n)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    st = mm.solver.init_state(grid, m, bc, mm.SolverParams())
    st.F = st.F + 1e-3 * np.random.default_rng(seed).standard_normal(st.F.shape)
    st, _ = mm.solve(grid, m, bc, mm.SolverParams(max_outer=K), policy=mm.RatioToDual(0.3),
                     state=st, raise_on_max=False)
    return ([np.array(getattr(st, k)) for k in ("F", "lam", "grad_u", "u_tilde")],
            [h[:5] for h in st.history])


def _noise():
    """Unrelated device work between repetitions (changes which SMs and
    which L2 lines the next run starts on)."""
    import torch
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(3):
        a = a @ a.T
        a = a / a.norm()
    torch.cuda.synchronize()


@pytest.mark.parametrize("n,plane", [(64, "1"), (128, "1"), (64, "0")])
def test_repeated_solves_are_bitwise_identical(n, plane, monkeypatch):
    monkeypatch.setenv("MM_PLANE_FFT", plane)
    ref = _run(n, 6)
    for rep in range(4):
        _noise()
        got = _run(n, 6)
        for a, b in zip(got[0], ref[0]):
            assert np.array_equal(a, b), rep
        assert got[1] == ref[1]


def test_repeated_slab_push_runs_are_bitwise_identical():
    from paper_2010_06697_b200.slab import ThreadComm, local_planes, local_points
    n, P, K = 32, 4, 4
    grid, mu, kap = _laminate(n)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    F = np.broadcast_to(bc.value, grid.shape + (3, 3)) + \
        1e-3 * np.random.default_rng(0).standard_normal(grid.shape + (3, 3))

    def once():
        shared = {"P": P, "barrier": threading.Barrier(P), "slots": {}}
        out = [None] * P

        def body(r):
            comm = ThreadComm(shared, r, exchange="push")
            sl, pts = local_planes(grid, comm), local_points(grid, comm)
            m = mm.MooneyRivlin(mu[pts], kap[pts], dim=3, mu_rep=1.0)
            s = mm.solver.init_state(grid, m, bc, mm.SolverParams(), comm=comm)
            s.F = np.array(F[sl])
            s, _ = mm.solve(grid, m, bc, mm.SolverParams(max_outer=K),
                            policy=mm.RatioToDual(0.3), state=s, raise_on_max=False, comm=comm)
            out[r] = np.array(s.lam), np.array(s.u_tilde)

        ths = [threading.Thread(target=body, args=(r,)) for r in range(P)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return [np.concatenate([o[i] for o in out]) for i in range(2)]

    ref = once()
    for rep in range(3):
        _noise()
        got = once()
        assert all(np.array_equal(a, b) for a, b in zip(got, ref)), rep
