"""Small solves that reach every kernel family under compute-sanitizer
(memcheck / racecheck / synccheck): the single-GPU fused schedule with the
cluster plane pass (k_plane) and the persistent C2R rows (k_row_inv_p), the
row layout with the persistent column kernel (k_colp) and the one-tile
solve pass, 2D, LCE 2D/3D (Newton kernels, Frank stencil), the slab path
(ghost planes, peer-store transposes between two contexts of this process),
equilibrium residual, Bloch iteration, and the last-block grid_finalize
reductions inside all of them.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""

import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2010_06697_b200 as mm  # noqa: E402
from paper_2010_06697_b200.slab import ThreadComm, local_planes, local_points  # noqa: E402


def laminate(dim, n):
    grid = mm.Grid(dim, n, 0.5)
    x = grid.coords()[..., 0]
    chi = ((x + 0.5) < 0.5).ravel().astype(float)
    mu = 1.0 + (0.05 - 1.0) * chi
    return grid, mu, 9.8 * mu


def mr(dim, n, K, env=None):
    if env:
        os.environ.update(env)
    grid, mu, kap = laminate(dim, n)
    Fbar = np.eye(dim)
    Fbar[0, 0] = 0.95
    bc = mm.MacroBC.strain(Fbar)
    m = mm.MooneyRivlin(mu, kap, dim=dim, mu_rep=1.0)
    st = mm.solver.init_state(grid, m, bc, mm.SolverParams())
    st.F = st.F + 1e-3 * np.random.default_rng(0).standard_normal(st.F.shape)
    st, _ = mm.solve(grid, m, bc, mm.SolverParams(max_outer=K), policy=mm.RatioToDual(0.3),
                     state=st, raise_on_max=False)
    mm.solver.equilibrium_residual(grid, m, st)
    if env:
        for k in env:
            os.environ.pop(k)
    return st


def lce(dim, n, K):
    import oracle
    grid = mm.Grid(dim, n, 0.5)
    n0 = oracle.polydomain_n0(dim, n, 0.5, 0.25, seed=1)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=dim)
    bc = mm.MacroBC.stress(np.zeros((dim, dim)))
    mm.solve(grid, m, bc, mm.SolverParams(max_outer=K, max_local=30), raise_on_max=False)


def slab(n, P, K, exchange):
    grid, mu, kap = laminate(3, n)
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    F = np.broadcast_to(bc.value, grid.shape + (3, 3)) + \
        1e-3 * np.random.default_rng(0).standard_normal(grid.shape + (3, 3))
    shared = {"P": P, "barrier": threading.Barrier(P), "slots": {}}
    err = []

    def body(r):
        try:
            comm = ThreadComm(shared, r, exchange=exchange)
            sl, pts = local_planes(grid, comm), local_points(grid, comm)
            m = mm.MooneyRivlin(mu[pts], kap[pts], dim=3, mu_rep=1.0)
            s = mm.solver.init_state(grid, m, bc, mm.SolverParams(), comm=comm)
            s.F = np.array(F[sl])
            mm.solve(grid, m, bc, mm.SolverParams(max_outer=K), policy=mm.RatioToDual(0.3),
                     state=s, raise_on_max=False, comm=comm)
        except Exception as e:  # pragma: no cover
            err.append(e)
            shared["barrier"].abort()

    ths = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if err:
        raise err[0]


def bloch():
    grid, mu, kap = laminate(2, 16)
    m = mm.MooneyRivlin(mu, kap, dim=2, mu_rep=1.0)
    st = mr(2, 16, 3)
    mm.stability_sweep(grid, m, st, k_max=2)


def main():
    which = sys.argv[1:] or ["mr3", "row", "mr2", "lce", "slab", "bloch"]
    if "mr3" in which:
        mr(3, 16, 4)                                  # k_plane, k_row_inv_p, K1 march, fused K2
        mr(3, 32, 3)
    if "row" in which:
        mr(3, 32, 3, {"MM_PLANE_FFT": "0"})           # row layout: k_colp, k_col, k_row_inv_p
    if "mr2" in which:
        mr(2, 32, 4)
    if "lce" in which:
        lce(2, 16, 2)
        lce(3, 8, 2)
    if "slab" in which:
        slab(32, 2, 3, "push")                        # peer-store transposes, ghost planes
        slab(32, 4, 2, "collective")
    if "bloch" in which:
        bloch()
    print("sanitize_run: done", which)


if __name__ == "__main__":
    main()
