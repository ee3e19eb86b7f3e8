"""LCE local-step timing on a polydomain director field.

python tools/lce_perf.py [n] [max_local] [dim]
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2010_06697_b200 as mm  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    max_local = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    dim = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    grid = mm.Grid(dim, n, 0.5)
    t0 = time.perf_counter()
    n0 = mm.generate_polydomain_n0(grid, 0.25, seed=1)
    m = mm.LiquidCrystalElastomer(mu=1.0, r=2.0, alpha=0.1, frank_kappa=1e-4, n0=n0, dim=dim)
    bc = mm.MacroBC.stress(np.zeros((dim, dim)))
    params = mm.SolverParams(max_outer=2, max_local=max_local)
    st = mm.solver.init_state(grid, m, bc, params)
    st.F = st.F + 1e-3 * np.random.default_rng(1).standard_normal(st.F.shape)
    print(f"setup {time.perf_counter() - t0:.1f} s", flush=True)
    pol = mm.RatioToDual(0.3)
    r = mm.solver.outer_iteration(grid, m, st, params, bc, pol)
    ctx = st._engine.ctx
    ctx.synchronize()
    ctx.profile_read(reset=True)
    ctx.profile_enable(True)
    import ctypes
    from paper_2010_06697_b200 import _lib
    cnt = (ctypes.c_double * 8)()
    lib = _lib.load_library()
    lib.mm_debug_lce_counters(cnt, 1)
    eng = st._engine
    ps0 = eng.point_sweeps
    t0 = time.perf_counter()
    r = mm.solver.outer_iteration(grid, m, st, params, bc, pol)
    ctx.synchronize()
    wall = time.perf_counter() - t0
    ms, nl = ctx.profile_read(reset=True)
    sw = st.total_sweeps
    psw = eng.point_sweeps - ps0
    print(f"{dim}D LCE n={n}: outer iteration {wall * 1e3:.1f} ms, residuals {r}, "
          f"total sweeps {sw}", flush=True)
    print({k: round(v, 3) for k, v in ms.items() if v}, nl)
    print(f"voxel-iter/s {grid.npoints / wall:.3e}; point sweeps/voxel {psw / grid.npoints:.1f}; "
          f"voxel-sweeps/s {psw / (ms['local'] / 1e3):.3e} (local stage {ms['local']:.1f} ms)")
    lib.mm_debug_lce_counters(cnt, 1)
    names = ["multiplier-only sweeps", "Newton steps", "eliminations", "Armijo evaluations",
             "det-guard trials", "fallback passes", "fallback evaluations",
             "warp Newton iterations x32"]
    if any(cnt):
        for nm, v in zip(names, cnt):
            print(f"  {nm:28s} {v / grid.npoints:10.2f} per voxel")


if __name__ == "__main__":
    main()
