"""Kernel timeline of solve() outer iterations (diagnostic tool).

Records every kernel of K outer iterations through the public solve() with
the CUPTI tracer of torch.profiler and prints, per kernel in launch order,
its duration and the idle gap before it, then the per-iteration totals:
busy time vs. the span from the first to the last kernel.

python tools/timeline.py [n] [iters]
"""

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2010_06697_b200 as mm  # noqa: E402


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    grid, model, bc, _, st = bench.setup_problem(mm, n)
    pol = mm.RatioToDual(0.3)
    p = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=5)
    mm.solve(grid, model, bc, p, policy=pol, state=st, raise_on_max=False)
    st._engine.ctx.synchronize()
    p = mm.SolverParams(r_p_tol=1e-300, r_d_tol=1e-300, max_outer=iters)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        mm.solve(grid, model, bc, p, policy=pol, state=st, raise_on_max=False)
        st._engine.ctx.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    t_first = ev[0].time_range.start
    last_end = None
    busy = 0.0
    gaps = {}
    for e in ev:
        s, t = e.time_range.start, e.time_range.end
        gap = (s - last_end) if last_end is not None else 0.0
        name = e.name.split("(")[0][-48:]
        busy += t - s
        if last_end is not None:
            gaps[name] = gaps.get(name, 0.0) + max(gap, 0.0)
        print(f"{(s - t_first) / 1e3:10.3f} ms  gap {gap:8.1f} us  dur {t - s:8.1f} us  {name}")
        last_end = max(t, last_end or t)
    span = last_end - t_first
    print(f"iterations {iters}: span {span / 1e3:.3f} ms = {span / 1e3 / iters:.3f} ms/iter, "
          f"busy {busy / 1e3 / iters:.3f} ms/iter, idle {(span - busy) / 1e3 / iters:.3f} ms/iter")
    print("idle before, per kernel name (us/iter):",
          {k: round(v / iters, 1) for k, v in sorted(gaps.items(), key=lambda kv: -kv[1])})


if __name__ == "__main__":
    main()
