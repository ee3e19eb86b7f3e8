"""Host-side CUDA runtime calls of the config-1 study (2D 64^2): how many per
outer iteration and how long the host spends in them (torch profiler, CPU +
CUDA activities; the library's calls show as cuda* runtime events)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import config1_time as c1  # noqa: E402


def main():
    from torch.profiler import ProfilerActivity, profile
    c1.run(c1.mm)
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        study, dt = c1.run(c1.mm)
    it = study.state.outer_iter
    ev = [e for e in prof.events() if e.device_type.name == "CPU" and e.name.startswith("cu")]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        agg[e.name][0] += 1
        agg[e.name][1] += e.time_range.end - e.time_range.start
    tot = sum(v[1] for v in agg.values())
    print(f"{it} iterations, wall {dt*1e3:.1f} ms; runtime calls {len(ev)/it:.1f}/iter, "
          f"{tot/it:.1f} us/iter inside them")
    for nm, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
        print(f"{t/it:8.2f} us/iter  {c/it:6.2f}/iter  {t/c:7.2f} us each  {nm}")


if __name__ == "__main__":
    main()
