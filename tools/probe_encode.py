"""Quick timing probe for the encode kernel (config-3 shape)."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 2_000_000
t0 = time.time()
w = wl.config3(n=n)
print(f"gen {time.time()-t0:.1f}s", flush=True)
s = aq.Session.default()
ds = s.upload_dataset(w.base)
cb = s.upload_codebook(aq.ProductCodebook(64, 16, 2, w.codebook))
out = s.alloc_codes(n, 64, 16)
wt = aq.ThresholdWeights(0.2, "parallel_only")
import ctypes as C
L = aq._L
for passes in (0, 1, 3):
    L.aq_debug_exact_window_count(s.h, 1, None)
    aq.dev_pq_quantize(ds, cb, wt, passes, out)
    cnt = (C.c_uint64 * 9)(); L.aq_debug_exact_window_count(s.h, 0, cnt)
    print(f"passes={passes}: exact windows {cnt[0]} = {cnt[0]/(n*64*(passes+1)):.4%} of subspace decisions; sweeps hist {list(cnt)[1:6]}", flush=True)
    ts = []
    for _ in range(5):
        t = time.perf_counter(); aq.dev_pq_quantize(ds, cb, wt, passes, out); ts.append(time.perf_counter() - t)
    b = min(ts)
    print(f"passes={passes}: {b*1e3:.2f} ms  {n/b:.3e} pts/s", flush=True)
codes = out.download().codes
from oracle import Port
P = Port()
sub = 20000
from tests.helpers import threshold_hp_ho
hp, ho = threshold_hp_ho(w.base[:sub], 0.2, 1)
want = P.pq_quantize(w.base[:sub].astype(np.float64), w.codebook, 64, 16, 2, hp, ho, 3)
print("parity first", sub, np.array_equal(codes[:sub], want))
