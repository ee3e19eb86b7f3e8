"""Per-iteration divergence trace of the device solver against the oracle
(config-2 laminate): relative L2 / max abs error of F, lam, grad_u, u_tilde
and the per-iteration sweep counts, one outer iteration at a time (split
runs are bitwise identical to one run on both sides).

  python tools/parity_trace.py [--n 128] [--K 20]
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2010_06697_b200 as mm  # noqa: E402


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--K", type=int, default=20)
    ap.add_argument("--fuse", default="1")
    args = ap.parse_args()
    os.environ["MM_FUSE"] = args.fuse
    oracle.set_threads(len(os.sched_getaffinity(0)))
    n, K = args.n, args.K
    grid = mm.Grid(3, n, 0.5)
    x = -0.5 + np.arange(n) / n
    chi = np.broadcast_to(((x + 0.5) < 0.5).astype(float).reshape(n, 1, 1), (n, n, n)).ravel()
    mu = 1.0 + (1.0 / 20.0 - 1.0) * chi
    kap = 9.8 * mu
    bc = mm.MacroBC.strain(np.diag([0.95, 1.0, 1.0]))
    m = mm.MooneyRivlin(mu, kap, dim=3, mu_rep=1.0)
    p1 = mm.SolverParams(max_outer=1)
    st = mm.solver.init_state(grid, m, bc, p1)
    F0 = st.F + 1e-4 * np.random.default_rng(0).standard_normal(st.F.shape)
    st.F = F0.copy()
    om = oracle.MR(mu, kap, dim=3, mu_rep=1.0)
    op = oracle.Params(max_outer=1)
    ost = oracle.init_state(3, n, om, bc.strain_mask, bc.value, op)
    ost.F = F0.copy()
    sym = oracle.symbols(3, n, 0.5)
    for k in range(K):
        s0 = st.total_sweeps
        st, _ = mm.solve(grid, m, bc, p1, policy=mm.RatioToDual(0.3), state=st,
                         raise_on_max=False)
        o0 = ost.total_sweeps
        oracle.outer_iteration(3, n, 0.5, om, ost, op, bc.strain_mask, bc.value,
                               oracle.RatioToDual(0.3), sym=sym)
        errs = []
        for nm in ("F", "lam", "grad_u", "u_tilde"):
            a, b = np.asarray(getattr(st, nm)), getattr(ost, nm)
            errs.append(f"{nm} {rel(a, b):.2e}/{np.abs(a - b).max():.1e}")
        h, oh = st.history[-1], ost.history[-1]
        print(f"it {k + 1:2d} sweeps {st.total_sweeps - s0:3d}/{ost.total_sweeps - o0:3d} "
              f"r_p {h.r_p:.6e}/{oh[1]:.6e} r_d {h.r_d:.3e} r_l {h.r_l:.3e} rho {h.rho:.3f} | "
              + "  ".join(errs), flush=True)
        # pin the next iteration on the same inputs: copy the oracle's state
        # into ours?  No: both evolve on their own (the test's setting).


if __name__ == "__main__":
    main()
