"""BASELINE.json configs 1-5 pinned against the REFERENCE ITSELF (oracle/_ref:
the unmodified reference headers compiled in place), run on the GPU box's
host cores with every thread. Each test runs the
device path and the reference on the same seeded inputs and requires
bit-identical results:

* C1 — the exact BASELINE workload (seed 0, n = 20,000, d = 32, M = 16,
  warm start + 10 iterations, ADC top-100 -> exact rerank -> top-10,
  recall@10 against exact_ground_truth): codebook, codes, loss history, ADC
  ids/scores, rerank ids/scores, ground truth and recall equal;
* C2 — full n = 1,183,514: train_apq warm start + 2 iterations
  (pq.hpp:513-575; the reference's serial pq_codebook_update takes ~25 s per
  iteration here), then ADC top-100 + rerank for 32 queries;
* C3 — all 1e7 codes of pq_quantize(passes = 3) (pq.hpp:581-612), the
  reference run in row chunks (points are independent);
* C4 — ADC top-100 of 8 queries over all 1e8 codes (index.hpp:118-134):
  the reference's per-chunk top-100 lists merged in (score desc, index asc)
  order — the reference's own global order;
* C5 — the config-5 shape (d = 256, M = 128, k = 16, T = 0.2) at n = 200,000:
  warm start + 2 iterations, i.e. two dim-4096 normal-equation assemblies
  (pq.hpp:290-343) and 64-panel Cholesky solves (pq.hpp:424-441).

The reference library is built in this container and travels with the
repository; its absence is a failure, not a skip.
"""
import os

import numpy as np
import pytest

from oracle import Reference
from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200 import workload as wl

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
THREADS = os.cpu_count() or 1


@pytest.fixture(scope="module")
def R():
    assert Reference.available(), "oracle/_ref/libanisoq_ref.so missing (make -C oracle)"
    return Reference()


def _weights(R, x, t, d):
    """resolve_weights (anisoq_main.cpp:108-142) with the reference's own
    eta_limit per point: h_par = eta, h_perp = 1."""
    norms = R.row_norms(x)
    hp = np.array([R.eta_limit(t, v, d) for v in norms])
    return hp, np.ones_like(hp)


def _recall(ids, gt, kk=10):
    return float(np.mean([len(set(a[:kk].tolist()) & set(b[:kk].tolist())) / kk
                          for a, b in zip(ids, gt)]))


def test_c1_baseline_workload(R):
    w = wl.config1()  # seed 0
    x = w.base.astype(np.float64)
    Q = w.queries.astype(np.float64)
    hp, ho = _weights(R, x, w.threshold, 32)
    cfg = aq.TrainConfig(max_iterations=10, relative_tolerance=0.0, seed=0)
    hist = []
    cb, codes = aq.train_apq(w.base, 16, 16, aq.ThresholdWeights(w.threshold), cfg, True, hist)
    rcb, rcodes, rhist = R.train_apq(x, 16, 16, hp, ho, max_it=10, tol=0.0, seed=0,
                                     threads=THREADS)
    assert np.array_equal(np.array(hist), rhist)
    assert np.array_equal(codes.codes, rcodes)
    assert np.array_equal(cb.dictionaries, rcb)
    s = aq.Session.default()
    ds, dc, dcb = s.upload_dataset(w.base), s.upload_codes(codes), s.upload_codebook(cb)
    aid, asc, rid, rsc = aq.dev_search_rerank(ds, dc, dcb, Q, 100, 10)
    wi, ws = R.adc_search_batch(Q, rcodes, 16, rcb, 16, 16, 2, 100, threads=THREADS)
    assert np.array_equal(aid, wi) and np.array_equal(asc, ws)
    ri, rs = R.rerank(Q, x, wi, 10, threads=THREADS)
    assert np.array_equal(rid, ri) and np.array_equal(rsc, rs)
    gi, gs = aq.dev_exact_search(ds, Q, 10)
    wgi, wgs = R.exact_search_batch(Q, x, 10, threads=THREADS)
    assert np.array_equal(gi, wgi) and np.array_equal(gs, wgs)
    # recall@10 (recall_k@k, kk = 10) and recall_1@10 identical
    assert _recall(rid, gi) == _recall(ri, wgi)
    r1 = np.mean([gi[q, 0] in rid[q, :10] for q in range(len(Q))])
    assert r1 == np.mean([wgi[q, 0] in ri[q, :10] for q in range(len(Q))])
    assert _recall(rid, gi) > 0.5


def test_c2_full_train_and_search(R):
    w = wl.config2(nq=32)
    x = w.base.astype(np.float64)
    Q = w.queries.astype(np.float64)
    hp, ho = _weights(R, x, w.threshold, 100)
    cfg = aq.TrainConfig(max_iterations=2, relative_tolerance=0.0, seed=0)
    hist = []
    cb, codes = aq.train_apq(w.base, 50, 16, aq.ThresholdWeights(w.threshold), cfg, True, hist)
    rcb, rcodes, rhist = R.train_apq(x, 50, 16, hp, ho, max_it=2, tol=0.0, seed=0,
                                     threads=THREADS)
    assert np.array_equal(np.array(hist), rhist)
    assert np.array_equal(codes.codes, rcodes)
    assert np.array_equal(cb.dictionaries, rcb)
    s = aq.Session.default()
    ds, dc, dcb = s.upload_dataset(w.base), s.upload_codes(codes), s.upload_codebook(cb)
    aid, asc, rid, rsc = aq.dev_search_rerank(ds, dc, dcb, Q, 100, 10)
    wi, ws = R.adc_search_batch(Q, rcodes, 16, rcb, 50, 16, 2, 100, threads=THREADS)
    assert np.array_equal(aid, wi) and np.array_equal(asc, ws)
    ri, rs = R.rerank(Q, x, wi, 10, threads=THREADS)
    assert np.array_equal(rid, ri) and np.array_equal(rsc, rs)


def test_c3_all_codes(R):
    w = wl.config3()  # n = 1e7, d = 128, lognormal norms
    cb = aq.ProductCodebook(64, 16, 2, w.codebook)
    # |x| <= T (0.06% of rows): the documented parallel-only policy (eta = inf)
    codes = aq.pq_quantize(w.base, cb, aq.ThresholdWeights(w.threshold, "parallel_only"), 3)
    from tests.helpers import threshold_hp_ho
    step = 1_000_000
    for b in range(0, w.n, step):
        e = min(w.n, b + step)
        x = w.base[b:e].astype(np.float64)
        hp, ho = threshold_hp_ho(w.base[b:e], w.threshold, 1)
        want = R.pq_quantize(x, w.codebook, 64, 16, 2, hp, ho, 3, threads=THREADS)
        assert np.array_equal(codes.codes[b:e], want), f"rows [{b}, {e})"


def test_c4_all_codes_top100(R):
    nq, topn, M = 8, 100, 48
    w = wl.config4(nq=nq)  # n = 1e8 uniform 4-bit codes
    s = aq.Session.default()
    dc = s.upload_packed_codes(w.packed_codes, w.n, M, 16)
    dcb = s.upload_codebook(aq.ProductCodebook(M, 16, 2, w.codebook))
    Q = w.queries.astype(np.float64)
    ids, sc = aq.dev_adc_search(dc, dcb, Q, topn)
    # 384 queries (3 blocks of 128, 2e6 points per SM slice) take the
    # tensor-core filter (csrc/adc_tc.cu); its first 8 rows are Q's
    extra = wl._normalize_rows(np.random.default_rng(44).standard_normal((376, 2 * M)))
    ids_tc, sc_tc = aq.dev_adc_search(dc, dcb, np.concatenate([Q, extra]), topn)
    dc.free()
    cand_i, cand_s = [], []
    step = 10_000_000
    for b in range(0, w.n, step):
        e = min(w.n, b + step)
        codes = wl.unpack_codes(w.packed_codes[b:e], M)
        ci, cs = R.adc_search_batch(Q, codes, 16, w.codebook, M, 16, 2, topn, threads=THREADS)
        cand_i.append(ci.astype(np.int64) + b)
        cand_s.append(cs)
    ci, cs = np.concatenate(cand_i, 1), np.concatenate(cand_s, 1)
    for q in range(nq):
        order = np.lexsort((ci[q], -cs[q]))[:topn]  # score desc, index asc
        assert np.array_equal(ids[q].astype(np.int64), ci[q][order]), q
        assert np.array_equal(sc[q], cs[q][order]), q
        assert np.array_equal(ids_tc[q].astype(np.int64), ci[q][order]), q
        assert np.array_equal(sc_tc[q], cs[q][order]), q


def test_c5_shape_train(R):
    w = wl.config5(n=200_000)
    x = w.base.astype(np.float64)
    hp, ho = _weights(R, x, w.threshold, 256)
    cfg = aq.TrainConfig(max_iterations=2, relative_tolerance=0.0, seed=0)
    hist = []
    cb, codes = aq.train_apq(w.base, 128, 16, aq.ThresholdWeights(w.threshold), cfg, True, hist)
    rcb, rcodes, rhist = R.train_apq(x, 128, 16, hp, ho, max_it=2, tol=0.0, seed=0,
                                     threads=THREADS)
    assert np.array_equal(np.array(hist), rhist)
    assert np.array_equal(codes.codes, rcodes)
    assert np.array_equal(cb.dictionaries, rcb)
