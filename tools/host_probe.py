import mmap, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
print("thp", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
N = 1 << 27  # 1 GiB of doubles
src = np.ones(N)
def fill(dst):
    # 16-thread copy like the library's par_memcpy
    import threading
    nt = 16; per = N // nt
    th = [threading.Thread(target=lambda i=i: np.copyto(dst[i*per:(i+1)*per], src[i*per:(i+1)*per])) for i in range(nt)]
    [t.start() for t in th]; [t.join() for t in th]
for kind in ("numpy", "mmap_huge", "mmap_plain", "numpy_touched"):
    t = time.perf_counter()
    if kind == "numpy":
        a = np.empty(N)
    elif kind == "numpy_touched":
        a = np.empty(N); a[::512] = 0; 
    else:
        m = mmap.mmap(-1, N * 8, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
        if kind == "mmap_huge":
            m.madvise(mmap.MADV_HUGEPAGE)
        a = np.frombuffer(m, dtype=np.float64)
    t1 = time.perf_counter()
    fill(a)
    t2 = time.perf_counter()
    print(kind, "alloc ms", round((t1 - t) * 1e3, 1), "fill ms", round((t2 - t1) * 1e3, 1),
          "GB/s", round(N * 8 / (t2 - t1) / 1e9, 1))
