"""Per-iteration breakdown of the bench workload (256^3 laminate): point
sweeps per voxel and device time per stage for every outer iteration."""
import sys
import numpy as np
import torch

sys.path.insert(0, ".")
import bench
import paper_2010_06697_b200 as mm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 55
torch.cuda.set_device(0)
grid, model, bc, _, st = bench.setup_problem(mm, n)
pol = mm.RatioToDual(0.3)
params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=1)
mm.solve(grid, model, bc, params, policy=pol, state=st, raise_on_max=False)
eng = st._engine
ctx = eng.ctx
ctx.profile_read(reset=True)
ctx.profile_enable(True)
rows = []
last = [eng.point_sweeps]


def cb(state, resid):
    ms, nl = ctx.profile_read(reset=True)
    ps = eng.point_sweeps - last[0]
    last[0] = eng.point_sweeps
    rows.append((state.outer_iter, ps / n ** 3, ms))


params = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
mm.solve(grid, model, bc, params, policy=pol, state=st, raise_on_max=False, callback=cb)
tot = {}
for it, sw, ms in rows:
    print(f"it {it:3d} sweeps/voxel {sw:6.2f} " + " ".join(f"{k}={v:.3f}" for k, v in ms.items() if v > 0))
    for k, v in ms.items():
        tot[k] = tot.get(k, 0.0) + v
print("mean ms:", {k: round(v / len(rows), 3) for k, v in tot.items() if v > 0})
