"""Breakdown of the e2e path (host state -> solve -> host fields) at 256^3."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_2010_06697_b200 as mm

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
grid, model, bc, _, st = bench.setup_problem(mm, n)
pol = mm.RatioToDual(0.3)
p = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=3)
mm.solve(grid, model, bc, p, policy=pol, state=st, raise_on_max=False)
host = dict(F=np.array(st.F), grad_u=np.array(st.grad_u), lam=np.array(st.lam),
            u_tilde=np.array(st.u_tilde), u_mean=st.u_mean.copy())
pinned = {}
for k in ("F", "grad_u", "lam", "u_tilde"):
    t = torch.empty(host[k].shape, dtype=torch.float64, pin_memory=True)
    t.numpy()[...] = host[k]
    pinned[k] = t
rho, rdp, oi = st.rho, st.r_d_prev, st.outer_iter
del st
import gc; gc.collect(); torch.cuda.synchronize()

T = {}
def tic(): return time.perf_counter()
t0 = tic()
hs = mm.ADMMState(u_mean=host["u_mean"], u_tilde=pinned["u_tilde"].numpy(),
                  grad_u=pinned["grad_u"].numpy(), F=pinned["F"].numpy(),
                  lam=pinned["lam"].numpy(), internal={}, rho=rho, outer_iter=oi, r_d_prev=rdp)
t1 = tic(); T["state"] = t1 - t0
eng = hs._attach(grid, model); eng.ctx.synchronize()
t2 = tic(); T["attach(engine+uploads)"] = t2 - t1
eng.ctx.profile_read(reset=True); eng.ctx.profile_enable(True)
p = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=K)
hs, _ = mm.solve(grid, model, bc, p, policy=pol, state=hs, raise_on_max=False)
hs._engine.ctx.synchronize()
t3 = tic(); T[f"solve K={K}"] = t3 - t2
ms, nl = eng.ctx.profile_read(reset=True); eng.ctx.profile_enable(False)
print("solve stages", {k: round(v, 2) for k, v in ms.items() if v}, {k: v for k, v in nl.items() if v})
print("history wall_ms", [round(r.wall_ms, 2) for r in hs.history[-K:]] if hasattr(hs.history[-1], "wall_ms") else "")
for k in ("F", "grad_u", "lam", "u_tilde"):
    a = tic(); v = getattr(hs, k); b = tic(); T["D2H " + k] = b - a
print({k: round(v * 1e3, 1) for k, v in T.items()}, "total ms", round((tic() - t0) * 1e3, 1))
# engine creation alone, by piece
from paper_2010_06697_b200 import _lib
from paper_2010_06697_b200.grid import axis_symbol_tables
a = tic(); c2 = _lib.Context(3, n=n, length=0.5); c2.synchronize(); b = tic()
print("Context() ms", round((b - a) * 1e3, 1))
a = tic(); tab, th = axis_symbol_tables(grid); b = tic()
print("axis_symbol_tables ms", round((b - a) * 1e3, 1))
del c2
a = tic(); e2 = mm._engine.Engine(grid); e2.ctx.synchronize(); b = tic()
print("Engine() ms", round((b - a) * 1e3, 1))
a = tic(); e2.bind_model(model); e2.ctx.synchronize(); b = tic()
print("bind_model ms", round((b - a) * 1e3, 1))
x = pinned["F"].numpy()
a = tic(); e2.ctx.upload(0, x); e2.ctx.synchronize(); b = tic()
print("upload F pinned ms", round((b - a) * 1e3, 1), "GB/s", round(x.nbytes / (b - a) / 1e9, 1))
y = np.array(x)
a = tic(); e2.ctx.upload(0, y); e2.ctx.synchronize(); b = tic()
print("upload F pageable ms", round((b - a) * 1e3, 1), "GB/s", round(y.nbytes / (b - a) / 1e9, 1))
a = tic(); z = e2.ctx.download(0, x.shape); b = tic()
print("download F fresh pageable ms", round((b - a) * 1e3, 1), "GB/s", round(z.nbytes / (b - a) / 1e9, 1))
a = tic(); e2.ctx.download_into(0, z); b = tic()
print("download F into touched pageable ms", round((b - a) * 1e3, 1), "GB/s", round(z.nbytes / (b - a) / 1e9, 1))
a = tic(); e2.ctx.download_into(0, x); b = tic()
print("download F into pinned ms", round((b - a) * 1e3, 1), "GB/s", round(x.nbytes / (b - a) / 1e9, 1))
print("cores", len(os.sched_getaffinity(0)))
