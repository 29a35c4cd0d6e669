"""Exact search timing at the config-2 shape (ground truth of 10,000 queries
over 1,183,514 points). The path is chosen once per process by
AQ_EXACT_FILTER (1: float32 filter + float64 window, 0: all float64); the
ids/scores are saved so two runs can be compared bit for bit."""
import sys, time
import numpy as np
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_183_514
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000
out = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != "-" else None
depth = int(sys.argv[4]) if len(sys.argv) > 4 else 10
w = wl.config2(n=n, nq=nq)
s = aq.Session.default()
ds = s.upload_dataset(w.base)
Q = np.ascontiguousarray(w.queries, np.float64)
ids, sc = aq.dev_exact_search(ds, Q, depth)
ts = []
for _ in range(3):
    t = time.perf_counter(); aq.dev_exact_search(ds, Q, depth); ts.append(time.perf_counter() - t)
b = min(ts)
print(f"exact top-{depth}: {b*1e3:.1f} ms  {n*nq/b:.3e} dots/s", flush=True)
if out:
    np.savez(out, ids=ids, sc=sc)
