"""Probe: train_l2_pq (k-means warm start) at the config-5 shape, n points."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_1908_10396_b200 import anisoq as aq, workload as wl

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
its = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = wl.config5(n=n)
s = aq.Session.default()
ds = s.upload_dataset(w.base)
for rep in range(2):
    s.sync(); t = time.perf_counter()
    cb, codes = aq.dev_train_l2_pq(ds, 128, 16, aq.TrainConfig(max_iterations=its, seed=0))
    s.sync()
    print(f"train_l2_pq n={n} its={its}: {(time.perf_counter()-t)*1e3:.1f} ms", flush=True)
