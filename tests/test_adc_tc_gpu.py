"""GPU parity for the tensor-core ADC filter (csrc/adc_tc.cu, tcgen05.mma
kind::i8 over one-hot code images). The default picks it only for long
per-SM slices (config-4 scale), so it is forced here with AQ_ADC_TC=1 in a
child process (the variable is read once per process): ids and scores must
equal the oracle's (index.hpp:118-134) across both tile widths (TN = 64 for
M <= 48, 48 for M = 49, 50), odd code strides, partial tiles, query blocks
with padding queries, k < 16, deep top-N and massive ties (exact fallback)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
import numpy as np
from oracle import Port
from paper_1908_10396_b200 import anisoq as aq, workload as wl
P = Port()
cases = [(20000, 16, 100, 100, 16), (300000, 50, 100, 64, 16), (5000, 48, 7, 33, 16),
         (224, 50, 10, 1, 16), (70000, 49, 512, 20, 16), (200, 8, 100, 5, 16),
         (25000, 13, 50, 130, 16), (12000, 16, 100, 50, 9), (3000, 50, 10, 300, 16),
         (60000, 50, 2000, 20, 16), (20000, 16, 4096, 9, 16), (400000, 48, 100, 256, 16),
         (5000, 1, 10, 3, 16), (3000, 2, 20, 129, 7), (1, 50, 5, 2, 16), (63, 48, 100, 5, 16)]
for n, M, topn, nq, k in cases:
    g = np.random.default_rng(n + M + k)
    cb = aq.ProductCodebook(M, k, 2, g.standard_normal(M * k * 2) / np.sqrt(2 * M))
    codes = g.integers(0, k, (n, M)).astype(np.uint32)
    Q = wl._normalize_rows(g.standard_normal((nq, 2 * M)))
    s = aq.Session.default()
    dc = s.upload_codes(aq.CodeMatrix(n, M, k, codes))
    dcb = s.upload_codebook(cb)
    ids, sc = aq.dev_adc_search(dc, dcb, Q, topn)
    want_i, want_s = P.adc_search_batch(Q, codes, k, cb.dictionaries, M, k, 2, topn)
    assert np.array_equal(ids, want_i), (n, M, topn, nq, k)
    assert np.array_equal(sc, want_s), (n, M, topn, nq, k)
# massive ties: every point scores alike (windows overflow -> exact fallback)
n, M = 50000, 48
cb = aq.ProductCodebook(M, 16, 2, np.zeros(M * 16 * 2))
codes = np.random.default_rng(3).integers(0, 16, (n, M)).astype(np.uint32)
Q = wl._normalize_rows(np.random.default_rng(4).standard_normal((5, 2 * M)))
s = aq.Session.default()
ids, sc = aq.dev_adc_search(s.upload_codes(aq.CodeMatrix(n, M, 16, codes)), s.upload_codebook(cb), Q, 100)
want_i, want_s = P.adc_search_batch(Q, codes, 16, cb.dictionaries, M, 16, 2, 100)
assert np.array_equal(ids, want_i) and np.array_equal(sc, want_s)
print("ok")
"""


def test_tensor_core_filter_matches_oracle():
    env = dict(os.environ, AQ_ADC_TC="1", PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr[-4000:]
