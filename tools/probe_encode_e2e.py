import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_1908_10396_b200 import anisoq as aq, workload as wl
n = 10_000_000
w = wl.config3(n=n)
s = aq.Session.default(); L = aq._L
wt = aq.ThresholdWeights(0.2, "parallel_only")
keep = []; cw = aq._weights(wt, n, keep)
xs = np.ascontiguousarray(w.base)
codes_h = np.zeros((n, 64), np.uint32)
for it in range(4):
    if it == 2: codes_h[:] = 1
    t0 = time.perf_counter()
    aq._check(L.aq_pq_quantize(s.h, xs.ctypes.data, n, 128, w.codebook.ctypes.data, 64, 16, 2, C.byref(cw), 3, codes_h.ctypes.data))
    print(it, f"{time.perf_counter()-t0:.3f} s", flush=True)
# breakdown
t0 = time.perf_counter(); ds = s.upload_dataset(w.base); t1 = time.perf_counter()
print("upload_dataset", f"{t1-t0:.3f}")
