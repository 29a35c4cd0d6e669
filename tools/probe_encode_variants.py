"""Encode kernel A/B on the config-3 workload: kernel time from the library's
CUDA-event timers (slot 0), per AQ_ENC_VARIANT, plus the sweep histogram and a
parity check of the first rows against the oracle."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["11", "12"]
w = wl.config3(n=n)
s = aq.Session.default()
L = aq._L
ds = s.upload_dataset(w.base)
cb = s.upload_codebook(aq.ProductCodebook(64, 16, 2, w.codebook))
out = s.alloc_codes(n, 64, 16)
wt = aq.ThresholdWeights(0.2, "parallel_only")
from oracle import Port  # noqa: E402
from tests.helpers import threshold_hp_ho  # noqa: E402

sub = 20000
hp, ho = threshold_hp_ho(w.base[:sub], 0.2, 1)
want = Port().pq_quantize(w.base[:sub].astype(np.float64), w.codebook, 64, 16, 2, hp, ho, 3)
for v in variants:
    os.environ["AQ_ENC_VARIANT"] = v
    L.aq_debug_exact_window_count(s.h, 1, None)
    aq.dev_pq_quantize(ds, cb, wt, 3, out)
    cnt = (C.c_uint64 * 9)()
    L.aq_debug_exact_window_count(s.h, 0, cnt)
    hist = list(cnt)[1:6]
    ok = np.array_equal(out.download().codes[:sub], want)
    for _ in range(2):
        aq.dev_pq_quantize(ds, cb, wt, 3, out)
    L.aq_session_timing(s.h, 1)
    L.aq_session_timer_read(s.h, 0, None, None, 1)
    for _ in range(5):
        aq.dev_pq_quantize(ds, cb, wt, 3, out)
    ms, k = C.c_double(0), C.c_uint64(0)
    L.aq_session_timer_read(s.h, 0, C.byref(ms), C.byref(k), 1)
    L.aq_session_timing(s.h, 0)
    t = ms.value / k.value
    sweeps = sum(i * h for i, h in enumerate(hist)) / max(sum(hist), 1)
    print(f"variant {v}: {t:.3f} ms  {n / t * 1e3:.3e} pts/s  frac(27648 ops) "
          f"{n * 27648 / (t / 1e3) / 3.72e13:.3f}  exact windows {cnt[0]}  sweep hist {hist} "
          f"mean sweeps {sweeps:.3f}  parity {ok}", flush=True)
