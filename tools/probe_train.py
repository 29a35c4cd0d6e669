"""Probe: train_apq timing at config-1 and config-2 scale, config-1 parity."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

s = aq.Session.default()
w = wl.config1()
ds = s.upload_dataset(w.base)
cfg = aq.TrainConfig(max_iterations=10, relative_tolerance=0.0, seed=0)
hist = []
t = time.perf_counter()
cb, codes = aq.dev_train_apq(ds, 16, 16, aq.ThresholdWeights(0.2), cfg, True, hist)
s.sync(); t1 = time.perf_counter() - t
print(f"config1 train_apq (warm + 10 it): {t1*1e3:.1f} ms, history {hist}", flush=True)
from oracle import Port
from tests.helpers import threshold_hp_ho
P = Port()
hp, ho = threshold_hp_ho(w.base, 0.2)
t = time.perf_counter()
wcb, wcodes, whist = P.train_apq(w.base.astype(np.float64), 16, 16, hp, ho, max_it=10, tol=0.0, seed=0)
print(f"oracle (1 thread) {time.perf_counter()-t:.2f} s; parity cb={np.array_equal(cb.download().dictionaries, wcb)} codes={np.array_equal(codes.download().codes, wcodes)} hist={np.array_equal(np.array(hist), whist)}", flush=True)
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1183514
w2 = wl.config2(n=n, nq=1000)
ds2 = s.upload_dataset(w2.base)
import ctypes as C
L = aq._L
for warm in (True, True):  # second run: warm caches and clocks
    L.aq_session_timing(s.h, 1)
    for slot in range(9): L.aq_session_timer_read(s.h, slot, None, None, 1)
    hist = []
    t = time.perf_counter()
    cb2, codes2 = aq.dev_train_apq(ds2, 50, 16, aq.ThresholdWeights(0.2), cfg, warm, hist)
    s.sync()
    tt = time.perf_counter() - t
    ph = {}
    for slot, nm in ((0, "encode"), (5, "assemble"), (6, "llt"), (7, "kmeans")):
        ms, cnt = C.c_double(0), C.c_uint64(0)
        L.aq_session_timer_read(s.h, slot, C.byref(ms), C.byref(cnt), 1)
        ph[nm] = round(ms.value, 1)
    L.aq_session_timing(s.h, 0)
    print(f"config2 n={n} train_apq: {tt:.2f} s phases ms {ph} hist {hist[:2]}..{hist[-1]}", flush=True)
t = time.perf_counter()
gt, _ = aq.dev_exact_search(ds2, w2.queries.astype(np.float64), 10)
print(f"exact ground truth 1000 q: {(time.perf_counter()-t)*1e3:.1f} ms", flush=True)
aid, asc, rid, rsc = aq.dev_search_rerank(ds2, codes2, cb2, w2.queries.astype(np.float64), 100, 10)
rec = np.mean([len(set(rid[q]) & set(gt[q])) / 10 for q in range(len(gt))])
rec1 = np.mean([gt[q][0] in aid[q][:10] for q in range(len(gt))])
print(f"recall10@10 (ADC100+rerank) {rec:.4f}  recall1@10 (ADC) {rec1:.4f}", flush=True)
