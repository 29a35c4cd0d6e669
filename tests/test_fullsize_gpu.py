"""Config 2 at full size over all 10 training iterations (the reference
comparisons of configs 1-5, including full-n config 2 for two iterations,
all 1e7 config-3 codes and config-4 top-100 over all 1e8 codes, are in
tests/test_config_pins_gpu.py):

* config 2 (1,183,514 x 100, M = 50): train_apq's loss history is
  non-increasing; ADC top-100 and the exact rerank of a few queries over the
  whole database equal the oracle's; the trained codebook encodes a row
  sample exactly as the oracle does.
"""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200 import workload as wl
from tests.helpers import threshold_hp_ho

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
P = Port()


def _sample_rows(n, count, seed, extra=()):
    g = np.random.default_rng(seed)
    rows = set(g.choice(n, count, replace=False).tolist())
    rows |= set(range(64)) | set(range(n - 64, n)) | set(r for r in extra if 0 <= r < n)
    return np.array(sorted(rows))


def test_config2_train_search_full_size():
    w = wl.config2(nq=4)
    n = w.n
    cfg = aq.TrainConfig(max_iterations=10, relative_tolerance=0.0, seed=0)
    hist: list = []
    cb, codes = aq.train_apq(w.base, 50, 16, aq.ThresholdWeights(w.threshold), cfg, True, hist)
    assert len(hist) == 11
    assert all(b <= a for a, b in zip(hist, hist[1:]))
    Q = w.queries.astype(np.float64)
    s = aq.Session.default()
    ds = s.upload_dataset(w.base)
    dc = s.upload_codes(codes)
    dcb = s.upload_codebook(cb)
    aid, asc, rid, rsc = aq.dev_search_rerank(ds, dc, dcb, Q, 100, 10)
    wi, wsc = P.adc_search_batch(Q, codes.codes, 16, cb.dictionaries, 50, 16, 2, 100)
    assert np.array_equal(aid, wi) and np.array_equal(asc, wsc)
    x64 = w.base.astype(np.float64)
    ri, rs = P.rerank(Q, x64, wi, 10)
    assert np.array_equal(rid, ri) and np.array_equal(rsc, rs)
    # the trained codebook encodes a row sample exactly as the oracle does
    rows = _sample_rows(n, 2000, 32)
    got = aq.pq_quantize(w.base, cb, aq.ThresholdWeights(w.threshold), 1).codes
    hp, ho = threshold_hp_ho(w.base[rows], w.threshold)
    want = P.pq_quantize(x64[rows], cb.dictionaries, 50, 16, 2, hp, ho, 1)
    assert np.array_equal(got[rows], want)
