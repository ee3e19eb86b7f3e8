import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.zeros(1, device="cuda")
from paper_2010_06697_b200 import _lib
n = 256
t = time.perf_counter(); c = _lib.Context(3, n=n, length=0.5); c.synchronize(); a = time.perf_counter() - t
del c
t = time.perf_counter(); c = _lib.Context(3, n=n, length=0.5); c.synchronize(); b = time.perf_counter() - t
t = time.perf_counter(); c2 = _lib.Context(3, n=n, length=0.5); c2.synchronize(); d = time.perf_counter() - t
print(os.environ.get("MM_DEVICE_POOL", "1"), "first", round(a * 1e3, 1), "after destroy", round(b * 1e3, 1),
      "second live", round(d * 1e3, 1))
