"""Context creation / destruction cost of a small 2D grid, with the runtime calls inside."""
import time, collections
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_06697_b200 as mm
from paper_2010_06697_b200 import _lib
c = _lib.Context(2, n=64, length=0.5, device=0); del c
ts = []
for i in range(5):
    t0 = time.perf_counter(); c = _lib.Context(2, n=64, length=0.5, device=0); t1 = time.perf_counter(); del c; t2 = time.perf_counter()
    ts.append((t1 - t0, t2 - t1))
print("create / destroy ms:", [(round(a*1e3, 2), round(b*1e3, 2)) for a, b in ts])
from torch.profiler import ProfilerActivity, profile
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    c = _lib.Context(2, n=64, length=0.5, device=0); del c
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name == "CPU" and e.name.startswith("cu"):
        agg[e.name][0] += 1; agg[e.name][1] += e.time_range.end - e.time_range.start
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]): print(f"{t:9.1f} us {n:4d} {k}")
