"""Probe: train_apq phase breakdown at config-5 shape (d=256, M=128) for a given n."""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t = time.time(); w = wl.config5(n=n); print(f"gen {time.time()-t:.1f}s", flush=True)
s = aq.Session.default(); L = aq._L
ds = s.upload_dataset(w.base)
L.aq_session_timing(s.h, 1)
for slot in range(8): L.aq_session_timer_read(s.h, slot, None, None, 1)
cfg = aq.TrainConfig(max_iterations=iters, relative_tolerance=0.0, seed=0)
hist = []
t = time.perf_counter()
cb, codes = aq.dev_train_apq(ds, 128, 16, aq.ThresholdWeights(0.2), cfg, True, hist)
s.sync(); tt = time.perf_counter() - t
names = ["encode", "adc_score", "adc_merge", "rerank", "lut", "assemble", "llt", "kmeans"]
out = {}
for slot, nm in enumerate(names):
    ms, cnt = C.c_double(0), C.c_uint64(0)
    L.aq_session_timer_read(s.h, slot, C.byref(ms), C.byref(cnt), 1)
    if cnt.value: out[nm] = (round(ms.value, 1), cnt.value)
print(f"config5 n={n} train_apq warm + {iters} it: {tt:.2f} s; phases ms (total, launches): {out}", flush=True)
print("history", hist, flush=True)
