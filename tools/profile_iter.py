"""Host/device timing breakdown of outer iterations (diagnostic tool).

python tools/profile_iter.py [n] [iters]
"""

import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2010_06697_b200 as mm  # noqa: E402
from paper_2010_06697_b200 import _lib, solver  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    grid, model, bc, params, st = bench.setup_problem(mm, n)
    pol = mm.RatioToDual(0.3)
    for _ in range(3):
        solver.outer_iteration(grid, model, st, params, bc, pol)
    eng = st._engine
    ctx = eng.ctx
    ctx.synchronize()
    ctx.profile_read(reset=True)
    ctx.profile_enable(True)
    npts = grid.npoints
    for it in range(iters):
        t0 = time.perf_counter()
        eng = st._attach(grid, model)
        t1 = time.perf_counter()
        stats = model._device_local(ctx, npts, st.rho, 0.0, 25, pol.target_tol(params, st.r_d_prev))
        t2 = time.perf_counter()
        d = 3
        F_mean = (stats.sum_F[: d * d] / npts).reshape(d, d)
        u_mean = mm.projection.macro_gradient(bc, F_mean, eng.lam_mean(), st.rho)
        t3 = time.perf_counter()
        up = ctx.project_update(st.rho, u_mean)
        t4 = time.perf_counter()
        eng.lam_sum = np.array(up.sum_lam[:9])
        st._mark_device("F", "grad_u", "lam", "u_tilde")
        st.r_d_prev = st.rho * float(np.sqrt(up.sum_dG2 / npts))
        t5 = time.perf_counter()
        print(f"it {it}: attach {1e3*(t1-t0):.3f} local {1e3*(t2-t1):.3f} (sweeps {stats.sweeps}) "
              f"macro {1e3*(t3-t2):.3f} project {1e3*(t4-t3):.3f} tail {1e3*(t5-t4):.3f} ms",
              flush=True)
    ms, nl = ctx.profile_read(reset=True)
    print({k: round(v / iters, 4) for k, v in ms.items()})
    print(nl)


if __name__ == "__main__":
    main()
