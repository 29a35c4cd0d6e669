"""Probe: one config-5 training iteration split into its calls (assignment
pass, codebook update = buckets + weights + assembly + Cholesky + reseed
check), wall time after a device sync, at n points (default 1e7)."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
w = wl.config5(n=n)
s = aq.Session.default(); L = aq._L
ds = s.upload_dataset(w.base)
cb, codes = aq.dev_train_l2_pq(ds, 128, 16, aq.TrainConfig(max_iterations=1, seed=0))
wt = aq.ThresholdWeights(0.2)
out = s.upload_codebook(aq.ProductCodebook(128, 16, 2, np.zeros(128 * 16 * 2)))
keep = []
cw = aq._weights(wt, n, keep)
L.aq_session_timing(s.h, 1)
for rep in range(3):
    for slot in range(9): L.aq_session_timer_read(s.h, slot, None, None, 1)
    s.sync(); t = time.perf_counter()
    aq.dev_pq_assign_pass(ds, cb, wt, codes)
    s.sync(); ta = time.perf_counter() - t
    t = time.perf_counter()
    aq._check(L.aq_dev_pq_codebook_update(ds.h, codes.h, C.byref(cw), -1.0, out.h))
    s.sync(); tu = time.perf_counter() - t
    ph = {}
    for slot, nm in ((0, "encode"), (5, "assemble"), (6, "llt")):
        ms, cnt = C.c_double(0), C.c_uint64(0)
        L.aq_session_timer_read(s.h, slot, C.byref(ms), C.byref(cnt), 1)
        ph[nm] = round(ms.value, 1)
    print(f"rep {rep}: assign pass {ta*1e3:.1f} ms, codebook update {tu*1e3:.1f} ms, timers {ph}",
          flush=True)
