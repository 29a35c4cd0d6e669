"""ADC scoring variant sweep (config-2 shape: n = 1,183,514, M = 50, 10,000
queries): kernel time from the session timers, parity against variant 1."""
import os, sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, _lib
import ctypes as C

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_183_514
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
M = int(sys.argv[3]) if len(sys.argv) > 3 else 50
variants = [int(v) for v in (sys.argv[4].split(",") if len(sys.argv) > 4 else "1,0,2".split(","))]
g = np.random.default_rng(0)
codes = g.integers(0, 16, (n, M), dtype=np.uint32)
cb = g.standard_normal(M * 16 * 2) * 0.3
Q = g.standard_normal((nq, 2 * M))
s = aq.Session.default()
dc = s.upload_codes(aq.CodeMatrix(n, M, 16, codes))
dcb = s.upload_codebook(aq.ProductCodebook(M, 16, 2, cb))
L = aq._L
L.aq_session_timing(s.h, 1)
ref = None
for v in variants:
    os.environ["AQ_ADC_VARIANT"] = str(v)
    ids, sc = aq.dev_adc_search(dc, dcb, Q, 100)
    ms = C.c_double(); cnt = C.c_uint64()
    L.aq_session_timer_read(s.h, 1, C.byref(ms), C.byref(cnt), 1)
    best = 1e9
    for _ in range(3):
        aq.dev_adc_search(dc, dcb, Q, 100)
        L.aq_session_timer_read(s.h, 1, C.byref(ms), C.byref(cnt), 1)
        best = min(best, ms.value / max(cnt.value, 1))
    ok = ""
    if ref is None:
        ref = (ids, sc)
    else:
        ok = "parity " + str(np.array_equal(ids, ref[0]) and np.array_equal(sc, ref[1]))
    print(f"variant {v}: k_adc_score {best:.2f} ms  {n*nq/best/1e-3:.3e} scores/s {ok}", flush=True)
