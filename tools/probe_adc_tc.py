"""Probe: ADC filter timing, tensor-core (AQ_ADC_TC=1) vs scalar (0), on
random codes / codebook / unit queries of a given shape.

    python tools/probe_adc_tc.py n nq M [topn] [variants=0,1]
"""
import os
import subprocess
import sys

ROOT = __file__.rsplit("/tools/", 1)[0]
CHILD = r"""
import sys, time, ctypes as C
import numpy as np
sys.path.insert(0, %(root)r)
from paper_1908_10396_b200 import anisoq as aq, workload as wl
n, nq, M, topn = %(n)d, %(nq)d, %(M)d, %(topn)d
g = np.random.default_rng(7)
cb = aq.ProductCodebook(M, 16, 2, g.standard_normal(M * 32) / np.sqrt(2 * M))
packed = g.integers(0, 256, (n, (M + 1) // 2), dtype=np.uint8)
Q = wl._normalize_rows(g.standard_normal((nq, 2 * M)))
s = aq.Session.default(); L = aq._L
dc = s.upload_packed_codes(packed, n, M, 16)
dcb = s.upload_codebook(cb)
aq.dev_adc_search(dc, dcb, Q, topn)
L.aq_session_timing(s.h, 1)
best = 1e30
for rep in range(3):
    L.aq_session_timer_read(s.h, 1, None, None, 1)
    aq.dev_adc_search(dc, dcb, Q, topn)
    ms, cnt = C.c_double(), C.c_uint64()
    L.aq_session_timer_read(s.h, 1, C.byref(ms), C.byref(cnt), 1)
    best = min(best, ms.value)
print(f"RESULT score {best:.2f} ms  {n * nq / best * 1e3:.3e} scores/s", flush=True)
"""


def main():
    n, nq, M = (int(float(v)) for v in sys.argv[1:4])
    topn = int(sys.argv[4]) if len(sys.argv) > 4 else 100
    for v in (sys.argv[5] if len(sys.argv) > 5 else "0,1").split(","):
        env = dict(os.environ, AQ_ADC_TC=v)
        r = subprocess.run([sys.executable, "-c", CHILD % dict(root=ROOT, n=n, nq=nq, M=M, topn=topn)],
                           env=env, capture_output=True, text=True, timeout=900)
        out = [l for l in r.stdout.splitlines() if l.startswith("RESULT") or "PROF" in l][-6:]
        print(f"n={n} nq={nq} M={M} topn={topn} AQ_ADC_TC={v}:", *out[-6:], r.stderr[-800:] if r.returncode else "",
              flush=True)


if __name__ == "__main__":
    main()
