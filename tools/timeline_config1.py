"""CUPTI kernel timeline of the config-1 study (2D 64^2): per-iteration GPU
busy time vs wall time, kernel durations by name."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import config1_time as c1  # noqa: E402


def main():
    from torch.profiler import ProfilerActivity, profile
    c1.run(c1.mm)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        study, dt = c1.run(c1.mm)
    it = study.state.outer_iter
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    print(f"{it} iterations, wall {dt*1e3:.1f} ms, GPU span {span/1e3:.1f} ms, busy {busy/1e3:.1f} ms "
          f"({busy/it:.1f} us/iter busy, {len(ev)/it:.1f} ops/iter)")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        nm = e.name[:70]
        agg[nm][0] += 1
        agg[nm][1] += e.time_range.end - e.time_range.start
    for nm, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
        print(f"{t/it:8.2f} us/iter  {c/it:5.2f}/iter  {t/c:7.2f} us each  {nm}")


if __name__ == "__main__":
    main()
