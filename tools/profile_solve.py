"""Stage profile of solve() outer iterations (fused schedule).  python tools/profile_solve.py [n] [K]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa
import paper_2010_06697_b200 as mm  # noqa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
grid, model, bc, _, st = bench.setup_problem(mm, n)
pol = mm.RatioToDual(0.3)
mm.solve(grid, model, bc, mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=5), policy=pol,
         state=st, raise_on_max=False)
ctx = st._engine.ctx
ctx.synchronize(); ctx.profile_read(reset=True); ctx.profile_enable(True)
t0 = time.perf_counter()
mm.solve(grid, model, bc, mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K), policy=pol,
         state=st, raise_on_max=False)
ctx.synchronize()
wall = (time.perf_counter() - t0) * 1e3 / K
ms, nl = ctx.profile_read(reset=True)
print(f"n={n} fuse={os.environ.get('MM_FUSE', '1')} ms/iter {wall:.3f}  sweeps {st.total_sweeps}")
print({k: round(v / K, 4) for k, v in ms.items() if v}, {k: v for k, v in nl.items() if v})
