"""Probe: codebook-update assembly time per AQ_ASM_VARIANT at config 2 / 5
scale, and a digest of the updated codebook (every variant must agree bit for
bit). Each variant runs in a child process (the variable is read once).

    python tools/probe_assemble.py [config=2|5] [n] [variants=0,1,3] [train_apq iterations, 0 = k-means codes]
"""
import hashlib
import os
import subprocess
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]

CHILD = r"""
import sys, time, ctypes as C, hashlib
import numpy as np
sys.path.insert(0, %(root)r)
from paper_1908_10396_b200 import anisoq as aq, workload as wl
cfg, n = %(cfg)d, %(n)d
w = wl.config5(n=n) if cfg == 5 else wl.config2(n=n, nq=16)
M = 128 if cfg == 5 else 50
s = aq.Session.default(); L = aq._L
ds = s.upload_dataset(w.base)
wt = aq.ThresholdWeights(0.2)
if %(trained)d:  # balanced strips, as inside train_apq
    cb, codes = aq.dev_train_apq(ds, M, 16, wt, aq.TrainConfig(max_iterations=%(trained)d, seed=0), True, [])
else:
    cb, codes = aq.dev_train_l2_pq(ds, M, 16, aq.TrainConfig(max_iterations=1, seed=0))
    aq.dev_pq_assign_pass(ds, cb, wt, codes)
cnt = np.bincount((codes.download().codes[:, 0]).astype(np.int64), minlength=16)
print(f"  strip sizes of subspace 0: min {cnt.min()} max {cnt.max()} mean {cnt.mean():.0f}", flush=True)
out = s.upload_codebook(aq.ProductCodebook(M, 16, 2, np.zeros(M * 16 * 2)))
keep = []
cw = aq._weights(wt, n, keep)
L.aq_session_timing(s.h, 1)
best = 1e30
for rep in range(4):
    for slot in range(9): L.aq_session_timer_read(s.h, slot, None, None, 1)
    s.sync(); t = time.perf_counter()
    aq._check(L.aq_dev_pq_codebook_update(ds.h, codes.h, C.byref(cw), -1.0, out.h))
    s.sync(); tu = time.perf_counter() - t
    ms, cnt = C.c_double(0), C.c_uint64(0)
    L.aq_session_timer_read(s.h, 5, C.byref(ms), C.byref(cnt), 1)
    best = min(best, ms.value)
    print(f"  rep {rep}: update {tu*1e3:.1f} ms, assembly {ms.value:.2f} ms", flush=True)
dig = hashlib.sha1(out.download().dictionaries.tobytes()).hexdigest()[:16]
print(f"RESULT assembly_best_ms={best:.3f} codebook={dig}", flush=True)
"""


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    n = int(float(sys.argv[2])) if len(sys.argv) > 2 else (1183514 if cfg == 2 else 10_000_000)
    variants = (sys.argv[3] if len(sys.argv) > 3 else "0,1,3").split(",")
    trained = int(sys.argv[4]) if len(sys.argv) > 4 else 0
    for v in variants:
        env = dict(os.environ, AQ_ASM_VARIANT=v)
        r = subprocess.run([sys.executable, "-c", CHILD % {"root": ROOT, "cfg": cfg, "n": n, "trained": trained}],
                           env=env, capture_output=True, text=True, timeout=1200)
        print(f"config {cfg} n={n} AQ_ASM_VARIANT={v} rc={r.returncode}")
        print(r.stdout + (r.stderr[-2000:] if r.returncode else ""), flush=True)


if __name__ == "__main__":
    main()
