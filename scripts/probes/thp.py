"""Host page-fault cost of a fresh 8 GiB float64 array: plain numpy vs an
mmap with MADV_HUGEPAGE, touched by 16 threads (the probabilities drain)."""
import ctypes, json, mmap, os, time, threading
import numpy as np
out = {"thp": open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
       "defrag": open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip(), "cpus": os.cpu_count()}
N = 1 << 30
def touch(a, nt=16):
    step = len(a) // nt
    def w(i): a[i * step:(i + 1) * step] = 1.0
    ts = [threading.Thread(target=w, args=(i,)) for i in range(nt)]
    t0 = time.perf_counter(); [t.start() for t in ts]; [t.join() for t in ts]
    return time.perf_counter() - t0
a = np.empty(N, np.float64); out["numpy_touch_s"] = touch(a); del a
m = mmap.mmap(-1, 8 * N, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
m.madvise(mmap.MADV_HUGEPAGE)
b = np.frombuffer(m, np.float64); out["thp_touch_s"] = touch(b); del b; m.close()
a = np.empty(N, np.float64); out["numpy_touch_1thread_s"] = touch(a, 1); del a
print(json.dumps(out))
