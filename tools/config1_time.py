"""SURVEY 8(d) config 1 (2D 64^2 two-phase laminate, load steps 1.0 -> 0.8)
timed end to end on the device, plus the oracle port on the host."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_06697_b200 as mm  # noqa: E402


def run(mod, n=64):
    grid = mod.Grid(2, n, 0.5)
    y = grid.coords()[..., 1]
    phase = ((y + grid.length) / (2 * grid.length) < 0.5).ravel()
    mu = np.where(phase, 0.05, 1.0)
    kap = 9.8 * mu
    m = mod.MooneyRivlin(mu, kap, dim=2, mu_rep=1.0)
    spec = mod.ProtocolSpec("monodomain", 1.0, 0.8, -0.02)
    t0 = time.perf_counter()
    study = mod.run_lce_protocol(grid, m, spec, params=mod.SolverParams(),
                                 policy=mod.RatioToDual(0.3), relax=True, seed=0, perturb=1e-4)
    dt = time.perf_counter() - t0
    return study, dt


def breakdown():
    """Time inside the library loop (mm_solve_fused) vs the rest of the study."""
    import time as _t
    from paper_2010_06697_b200 import _lib
    acc = {"t": 0.0, "calls": 0, "iters": 0}
    orig = _lib.Context.solve_fused

    def timed(self, sp, max_outer):
        t0 = _t.perf_counter()
        out = orig(self, sp, max_outer)
        acc["t"] += _t.perf_counter() - t0
        acc["calls"] += 1
        acc["iters"] += out[0].iterations
        return out

    from paper_2010_06697_b200 import _engine
    eacc = {"t": 0.0}
    eorig = _engine.Engine.__init__

    def etimed(self, *a, **k):
        t0 = _t.perf_counter()
        eorig(self, *a, **k)
        eacc["t"] += _t.perf_counter() - t0

    _lib.Context.solve_fused = timed
    _engine.Engine.__init__ = etimed
    try:
        run(mm)
        for k in acc:
            acc[k] = 0
        eacc["t"] = 0.0
        study, dt = run(mm)
    finally:
        _lib.Context.solve_fused = orig
        _engine.Engine.__init__ = eorig
    print(f"study {dt*1e3:.1f} ms; engine creation {eacc['t']*1e3:.1f} ms; inside mm_solve_fused "
          f"{acc['t']*1e3:.1f} ms over {acc['calls']} calls, {acc['iters']} iterations = "
          f"{acc['t']/max(acc['iters'],1)*1e6:.1f} us per iteration")


if __name__ == "__main__":
    if "--breakdown" in sys.argv:
        breakdown()
        sys.exit(0)
    run(mm)  # warm-up (context, JIT-free)
    study, dt = run(mm)
    it = study.state.outer_iter
    print(f"device: {len(study.records)} load steps, {it} outer iterations in {dt * 1e3:.1f} ms "
          f"= {dt / it * 1e6:.1f} us per outer iteration ({64 * 64 * it / dt:.3e} voxel-iter/s)")

