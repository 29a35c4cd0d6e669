"""Repro: evaluate on d = 6, M = 1, k = 1 (reference test_index.cpp:211-234)."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1908_10396_b200 import anisoq as aq

def step(name, f):
    try:
        r = f()
        aq.Session.default().sync()
        print("ok", name, flush=True)
        return r
    except Exception as e:
        print("FAIL", name, e, flush=True)
        sys.exit(1)

data = aq.generate_synthetic("uniform_sphere", 30, 6, 6)
q = aq.generate_synthetic("uniform_sphere", 10, 6, 7)
X = data.values if hasattr(data, "values") else data
Q = q.values if hasattr(q, "values") else q
cb = aq.ProductCodebook(1, 1, 6, np.array(X[0], dtype=np.float64))
codes = aq.CodeMatrix(30, 1, 1, np.zeros(30, dtype=np.uint32))
s = aq.Session.default()
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("exact", "all"):
    step("exact_search", lambda: aq.exact_search(Q[0], data, 10))
    ds = s.upload_dataset(np.asarray(X, np.float32))
    step("dev_exact", lambda: aq.dev_exact_search(ds, np.asarray(Q, np.float64), 30))
if which in ("adc", "all"):
    for topn in (1, 10, 30):
        step(f"adc_search topn={topn}", lambda: aq.adc_search(Q[0], codes, cb, topn))
    dc = s.upload_codes(codes)
    dcb = s.upload_codebook(cb)
    step("dev_adc", lambda: aq.dev_adc_search(dc, dcb, np.asarray(Q, np.float64), 30))
if which in ("rerank", "all"):
    ds = s.upload_dataset(np.asarray(X, np.float32))
    cand = np.tile(np.arange(30, dtype=np.uint32), (10, 1))
    step("dev_rerank", lambda: aq.dev_rerank(ds, np.asarray(Q, np.float64), cand, 30))
print("done")
