"""Timing probe for ADC search (config-4 shape, reduced n)."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 100
t0 = time.time()
w = wl.config4(n=n, nq=nq)
print(f"gen {time.time()-t0:.1f}s", flush=True)
s = aq.Session.default()
dc = s.upload_packed_codes(w.packed_codes, n, 48, 16)
dcb = s.upload_codebook(aq.ProductCodebook(48, 16, 2, w.codebook))
Q = w.queries.astype(np.float64)
ids, sc = aq.dev_adc_search(dc, dcb, Q, topn)
ts = []
for _ in range(3):
    t = time.perf_counter(); aq.dev_adc_search(dc, dcb, Q, topn); ts.append(time.perf_counter() - t)
b = min(ts)
import ctypes as C
L = aq._L
L.aq_session_timing(s.h, 1)
aq.dev_adc_search(dc, dcb, Q, topn)
for slot, nm in ((4, "lut"), (1, "score"), (2, "merge")):
    ms = C.c_double(); cnt = C.c_uint64()
    L.aq_session_timer_read(s.h, slot, C.byref(ms), C.byref(cnt), 1)
    print(f"  {nm}: {ms.value:.2f} ms", flush=True)
L.aq_session_timing(s.h, 0)
print(f"n={n} nq={nq} topn={topn}: {b*1e3:.2f} ms  {n*nq/b:.3e} scores/s", flush=True)
from oracle import Port
P = Port()
codes = wl.unpack_codes(w.packed_codes[:200000], 48)
wi, ws = P.adc_search_batch(Q[:4], codes, 16, w.codebook, 48, 16, 2, topn)
dc2 = s.upload_packed_codes(w.packed_codes[:200000], 200000, 48, 16)
gi, gs = aq.dev_adc_search(dc2, dcb, Q[:4], topn)
print("parity", np.array_equal(gi, wi), np.array_equal(gs, ws))
