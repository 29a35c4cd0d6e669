"""GPU parity: LUT build, ADC top-N and exact rerank (index.hpp:56-147)
through the C ABI against the oracle. Ids and scores must be bit-identical
(the float32 filter only narrows the window; the float64 re-score and the
exact sort reproduce the reference's order)."""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200 import workload as wl
from tests.helpers import mixture_rows, random_codebook

pytestmark = pytest.mark.gpu
P = Port()


def test_lut_worked_example():
    # test_index.cpp:58-67
    cb = aq.ProductCodebook(2, 2, 2, [-1, -1, 1, 1, -2, -2, 2, 2])
    lut = aq.build_lut([1.0, 0.0, 1.0, 0.0], cb)
    assert lut.partials.tolist() == [-1.0, 1.0, -2.0, 2.0]
    assert aq.build_lut(np.zeros(4), cb).partials.tolist() == [0.0] * 4
    with pytest.raises(aq.DimensionMismatch):
        aq.build_lut(np.ones(3), cb)


def test_lut_matches_oracle():
    cb = aq.ProductCodebook(16, 16, 2, random_codebook(16, 16, 2, 41))
    q = np.random.default_rng(1).standard_normal(32)
    assert np.array_equal(aq.build_lut(q, cb).partials, P.build_lut(q, cb.dictionaries, 16, 16, 2))


def test_adc_full_ranking_reference_case():
    # test_index.cpp:114-142: M=4, k=16, sd=2, n=1000, full ranking + top 25
    g = np.random.default_rng(10)
    cb = aq.ProductCodebook(4, 16, 2, g.standard_normal(128))
    codes = g.integers(0, 16, (1000, 4)).astype(np.uint32)
    q = g.standard_normal(8)
    want_i, want_s = P.adc_search_batch(q, codes, 16, cb.dictionaries, 4, 16, 2, 1000)
    got = aq.adc_search(q, aq.CodeMatrix(1000, 4, 16, codes), cb, 1000)
    assert [h.index for h in got.hits] == want_i[0].tolist()
    assert [h.score for h in got.hits] == want_s[0].tolist()
    top = aq.adc_search(q, aq.CodeMatrix(1000, 4, 16, codes), cb, 25)
    assert [h.index for h in top.hits] == want_i[0, :25].tolist()


def test_adc_validation():
    cb = aq.ProductCodebook(2, 4, 2, random_codebook(2, 4, 2, 3))
    with pytest.raises(aq.EmptyIndex):
        aq.adc_search(np.ones(4), aq.CodeMatrix(0, 2, 4, np.zeros((0, 2))), cb, 5)
    codes = aq.CodeMatrix(10, 2, 4, np.zeros((10, 2)))
    with pytest.raises(aq.InvalidArgument):
        aq.adc_search(np.ones(4), codes, cb, 0)
    with pytest.raises(aq.DimensionMismatch):
        aq.adc_search(np.ones(4), aq.CodeMatrix(10, 3, 4, np.zeros((10, 3))), cb, 5)


# every compiled M specialisation (16, 32, 48, 50, 64, 128), the generic
# kernel with and without a tail chunk (8, 13), k < 16, large top-N on the fast
# path (1000, 2000, 4096) and beyond it (5000), and slices that cross query-block edges (small n, many queries)
@pytest.mark.parametrize("n,M,topn,nq,k", [(20000, 16, 100, 100, 16), (300000, 50, 100, 64, 16),
                                           (5000, 48, 7, 33, 16), (70000, 16, 512, 20, 16),
                                           (200, 8, 100, 5, 16), (50000, 64, 1000, 3, 16),
                                           (40000, 32, 100, 40, 16), (30000, 128, 100, 20, 16),
                                           (25000, 13, 50, 17, 16), (12000, 16, 100, 50, 9),
                                           (3000, 50, 10, 300, 16), (60000, 50, 2000, 20, 16),
                                           (20000, 16, 4096, 9, 16), (30000, 16, 5000, 3, 16)])
def test_adc_batch_matches_oracle(n, M, topn, nq, k):
    g = np.random.default_rng(n + M + k)
    cb = aq.ProductCodebook(M, k, 2, g.standard_normal(M * k * 2) / np.sqrt(2 * M))
    codes = g.integers(0, k, (n, M)).astype(np.uint32)
    Q = wl._normalize_rows(g.standard_normal((nq, 2 * M)))
    s = aq.Session.default()
    dc = s.upload_codes(aq.CodeMatrix(n, M, k, codes))
    dcb = s.upload_codebook(cb)
    ids, sc = aq.dev_adc_search(dc, dcb, Q, topn)
    want_i, want_s = P.adc_search_batch(Q, codes, k, cb.dictionaries, M, k, 2, topn)
    assert np.array_equal(ids, want_i)
    assert np.array_equal(sc, want_s)


def test_adc_massive_ties_take_exact_fallback():
    # one codeword per subspace: every point ties (test_index.cpp:206-231 shape);
    # order must be index ascending, as select_top's tie rule says
    n, M = 3000, 8
    cb = aq.ProductCodebook(M, 1, 2, np.random.default_rng(3).standard_normal(M * 2))
    codes = np.zeros((n, M), np.uint32)
    q = np.random.default_rng(4).standard_normal(2 * M)
    got = aq.adc_search(q, aq.CodeMatrix(n, M, 1, codes), cb, 100)
    assert [h.index for h in got.hits] == list(range(100))
    # duplicated codewords: many exact float64 ties at the boundary
    d = random_codebook(M, 16, 2, 5).reshape(M, 16, 2)
    d[:, 1:] = d[:, :1]
    cb2 = aq.ProductCodebook(M, 16, 2, d.ravel())
    codes2 = np.random.default_rng(6).integers(0, 16, (n, M)).astype(np.uint32)
    got2 = aq.adc_search(q, aq.CodeMatrix(n, M, 16, codes2), cb2, 100)
    wi, ws = P.adc_search_batch(q, codes2, 16, cb2.dictionaries, M, 16, 2, 100)
    assert [h.index for h in got2.hits] == wi[0].tolist()


def test_rerank_and_pipeline_config1_shape():
    w = wl.config1(n=20000, nq=100, seed=3)
    cb = aq.ProductCodebook(16, 16, 2, random_codebook(16, 16, 2, 7, 0.25))
    codes = aq.pq_quantize(w.base, cb, aq.ThresholdWeights(0.2), 1)
    s = aq.Session.default()
    ds = s.upload_dataset(w.base)
    dc = s.upload_codes(codes)
    dcb = s.upload_codebook(cb)
    Q = w.queries.astype(np.float64)
    aid, asc, ids, sc = aq.dev_search_rerank(ds, dc, dcb, Q, 100, 10)
    wi, ws = P.adc_search_batch(Q, codes.codes, 16, cb.dictionaries, 16, 16, 2, 100)
    assert np.array_equal(aid, wi) and np.array_equal(asc, ws)
    ri, rs = P.rerank(Q, w.base.astype(np.float64), wi, 10)
    assert np.array_equal(ids, ri) and np.array_equal(sc, rs)
    ri2, rs2 = aq.dev_rerank(ds, Q, wi, 10)
    assert np.array_equal(ri2, ri) and np.array_equal(rs2, rs)


def test_rerank_long_candidate_lists():
    """More than 4096 candidates per query (beyond the one-warp sort): the
    fused ADC + rerank with top-N = 5000 and a direct rerank of 6000 ids equal
    the oracle's (score desc, index asc) order."""
    g = np.random.default_rng(41)
    n, M, k, sd = 9000, 8, 16, 2
    x = g.standard_normal((n, M * sd)).astype(np.float32)
    cb = aq.ProductCodebook(M, k, sd, g.standard_normal(M * k * sd) * 0.5)
    codes = g.integers(0, k, (n, M)).astype(np.uint32)
    Q = g.standard_normal((3, M * sd))
    s = aq.Session.default()
    ds, dc, dcb = s.upload_dataset(x), s.upload_codes(aq.CodeMatrix(n, M, k, codes)), \
        s.upload_codebook(cb)
    aid, asc, rid, rsc = aq.dev_search_rerank(ds, dc, dcb, Q, 5000, 4500)
    wi, ws = P.adc_search_batch(Q, codes, k, cb.dictionaries, M, k, sd, 5000)
    assert np.array_equal(aid, wi) and np.array_equal(asc, ws)
    ri, rs = P.rerank(Q, x.astype(np.float64), wi, 4500)
    assert np.array_equal(rid, ri) and np.array_equal(rsc, rs)
    cand = np.stack([g.permutation(n)[:6000] for _ in range(3)]).astype(np.uint32)
    ids, sc = aq.dev_rerank(ds, Q, cand, 7)
    ri, rs = P.rerank(Q, x.astype(np.float64), cand, 7)
    assert np.array_equal(ids, ri) and np.array_equal(sc, rs)
