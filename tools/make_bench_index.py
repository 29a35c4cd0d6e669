"""Builds bench_data/config2_codebook.npz: the config-2 codebook trained by the
REFERENCE ITSELF (oracle/_ref: train_apq, warm start + 10 iterations, T = 0.2,
seed 0) on workload.config2's rows. bench.py's reference arm searches the
index (this codebook, pq_quantize codes) without re-running the reference's
~5-minute serial training; the device arm retrains the codebook and checks it
equals this file bit for bit. Run in this container (needs /root/reference):

    python tools/make_bench_index.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import Reference  # noqa: E402
from paper_1908_10396_b200 import workload as wl  # noqa: E402

R = Reference()
w = wl.config2(nq=1)
x = w.base.astype(np.float64)
norms = R.row_norms(x)
hp = np.array([R.eta_limit(w.threshold, v, w.d) for v in norms])
ho = np.ones_like(hp)
t = time.time()
cb, codes, hist = R.train_apq(x, w.M, w.k, hp, ho, max_it=w.iterations, tol=0.0, seed=0,
                              threads=os.cpu_count() or 1)
print(f"reference train_apq: {time.time() - t:.0f} s, history {hist}")
out = os.path.join(ROOT, "bench_data", "config2_codebook.npz")
np.savez_compressed(out, dictionaries=cb, history=hist,
                    note="oracle/_ref train_apq(config2, M=50, k=16, T=0.2, warm start, "
                         "10 iterations, tol 0, seed 0)")
print("wrote", out)
