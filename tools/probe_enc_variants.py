"""Encode variant sweep (config-3 shape): pq_quantize passes=3 time per
AQ_ENC_VARIANT, parity of the first 20,000 codes against the oracle."""
import os, sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 4_000_000
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["11", "1"]
w = wl.config3(n=n)
s = aq.Session.default()
ds = s.upload_dataset(w.base)
cb = s.upload_codebook(aq.ProductCodebook(64, 16, 2, w.codebook))
out = s.alloc_codes(n, 64, 16)
wt = aq.ThresholdWeights(0.2, "parallel_only")
from oracle import Port
from tests.helpers import threshold_hp_ho
sub = 20000
hp, ho = threshold_hp_ho(w.base[:sub], 0.2, 1)
want = Port().pq_quantize(w.base[:sub].astype(np.float64), w.codebook, 64, 16, 2, hp, ho, 3)
for v in variants:
    os.environ["AQ_ENC_VARIANT"] = v
    aq.dev_pq_quantize(ds, cb, wt, 3, out)
    ts = []
    for _ in range(5):
        t = time.perf_counter(); aq.dev_pq_quantize(ds, cb, wt, 3, out); ts.append(time.perf_counter() - t)
    b = min(ts)
    ok = np.array_equal(out.download().codes[:sub], want)
    print(f"variant {v}: {b*1e3:.2f} ms  {n/b:.3e} pts/s parity {ok}", flush=True)
