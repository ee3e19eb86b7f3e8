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


if __name__ == "__main__":
    run(mm)  # warm-up (context, JIT-free)
    study, dt = run(mm)
    it = study.state.outer_iter
    print(f"device: {len(study.records)} load steps, {it} outer iterations in {dt * 1e3:.1f} ms "
          f"= {dt / it * 1e6:.1f} us per outer iteration ({64 * 64 * it / dt:.3e} voxel-iter/s)")
