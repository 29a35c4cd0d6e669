"""Single-query ADC search latency (the reference's per-query adc_search,
index.hpp:118-134, as timed by evaluate): config-2 index (random codes),
host -> device -> host per call, top-N = 100."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_183_514
M = 50
g = np.random.default_rng(0)
s = aq.Session.default()
codes = aq.CodeMatrix(n, M, 16, g.integers(0, 16, (n, M), dtype=np.uint32))
cb = aq.ProductCodebook(M, 16, 2, g.standard_normal(M * 32) / 10)
dc, dcb = s.upload_codes(codes), s.upload_codebook(cb)
Q = g.standard_normal((300, 2 * M))
for nq in (1, 8, 64):
    lat = []
    for i in range(0, 300 - nq + 1, nq):
        t = time.perf_counter()
        aq.dev_adc_search(dc, dcb, Q[i:i + nq], 100)
        lat.append((time.perf_counter() - t) * 1e6)
    lat = np.sort(lat[3:])
    print(f"batch {nq}: mean {lat.mean():.0f} us  p50 {lat[len(lat)//2]:.0f} us  p99 {lat[min(len(lat)-1, int(0.99*len(lat)))]:.0f} us per call", flush=True)
import ctypes as C
L = aq._L
L.aq_session_timing(s.h, 1)
for slot in range(9): L.aq_session_timer_read(s.h, slot, None, None, 1)
for i in range(20):
    aq.dev_adc_search(dc, dcb, Q[i:i + 1], 100)
for slot, nm in ((4, "lut"), (1, "score"), (2, "merge")):
    ms, cnt = C.c_double(0), C.c_uint64(0)
    L.aq_session_timer_read(s.h, slot, C.byref(ms), C.byref(cnt), 1)
    print(f"  nq=1 {nm}: {ms.value / max(cnt.value, 1) * 1e3:.0f} us per call", flush=True)
L.aq_session_timing(s.h, 0)
