"""GPU parity for datasets whose values are NOT float32-exact (float64 rows on
the device): unit_normalize output (dataset.hpp:225-236) and random float64
points, as the reference's own tests use them (test_vq.cpp:106-142,
test_index.cpp:188-263). Every hot-path entry — encode, assignment pass,
normal equations, codebook update, trainers, exact search, ADC + rerank — is
bit-identical to the oracle, as on the float32 fast paths."""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows, random_codebook, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()


def _unit_rows(n, d, seed):
    x = mixture_rows(n, d, seed, centers=12, sigma=0.4, normalize=False).astype(np.float64)
    x = aq.unit_normalize(x)
    assert aq.Dataset(x).f64  # genuinely float64 data
    return x


@pytest.mark.parametrize("d,M,k", [(32, 16, 16), (30, 10, 8), (24, 8, 16)])
def test_pq_quantize_f64(d, M, k):
    x = _unit_rows(3000, d, 11)
    sd = d // M
    cb = aq.ProductCodebook(M, k, sd, random_codebook(M, k, sd, 3) * 0.3)
    hp, ho = threshold_hp_ho(x, 0.2)
    got = aq.pq_quantize(x, cb, aq.ThresholdWeights(0.2), 3)
    want = P.pq_quantize(x, cb.dictionaries, M, k, sd, hp, ho, 3)
    assert np.array_equal(got.codes, want)


def test_assign_pass_and_update_f64():
    x = _unit_rows(2500, 24, 12)
    M, k, sd = 12, 16, 2
    cb = aq.ProductCodebook(M, k, sd, random_codebook(M, k, sd, 4) * 0.3)
    hp, ho = threshold_hp_ho(x, 0.2)
    codes0 = aq.CodeMatrix(len(x), M, k, P.pq_quantize(x, cb.dictionaries, M, k, sd, hp, ho, 0))
    got, gl = aq.pq_assign_pass(x, cb, aq.ThresholdWeights(0.2), codes0)
    want, wl_ = P.pq_assign_pass(x, cb.dictionaries, M, k, sd, hp, ho, codes0.codes)
    assert np.array_equal(got.codes, want) and np.array_equal(gl, wl_)
    A, rhs = aq.assemble_selector_system(x, got, aq.ThresholdWeights(0.2), M, k)
    wA, wr = P.assemble_selector_system(x, want, hp, ho, M, k)
    assert np.array_equal(A, wA) and np.array_equal(rhs, wr)
    new = aq.pq_codebook_update(x, got, aq.ThresholdWeights(0.2), M, k)
    assert np.array_equal(new.dictionaries, P.pq_codebook_update(x, want, hp, ho, M, k))


def test_trainers_f64():
    x = _unit_rows(3000, 16, 13)
    cfg = aq.TrainConfig(max_iterations=3, relative_tolerance=0.0, seed=5)
    cb, codes = aq.train_l2_pq(x, 8, 16, cfg)
    wcb, wcodes = P.train_l2_pq(x, 8, 16, 3, 0.0, 5)
    assert np.array_equal(cb.dictionaries, wcb) and np.array_equal(codes.codes, wcodes)
    hp, ho = threshold_hp_ho(x, 0.2)
    hist = []
    cb, codes = aq.train_apq(x, 8, 16, aq.ThresholdWeights(0.2), cfg, True, hist)
    wcb, wcodes, whist = P.train_apq(x, 8, 16, hp, ho, max_it=3, tol=0.0, seed=5)
    assert np.array_equal(np.array(hist), whist)
    assert np.array_equal(codes.codes, wcodes) and np.array_equal(cb.dictionaries, wcb)


def test_vq_f64():
    # test_vq.cpp:106-142 style: random float64 points
    g = np.random.default_rng(21)
    pts = g.standard_normal((40, 5))
    w = aq.AnisotropicWeights.from_eta(3.0)
    got = aq.update_codeword(5, pts, w)
    want = P.update_codeword(5, pts, np.full(40, 3.0), np.ones(40))
    assert np.array_equal(got, want)
    x = _unit_rows(1500, 8, 14)
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=4, relative_tolerance=0.0, seed=2)
    cw, asg = aq.train_avq(x, 6, aq.ThresholdWeights(0.2), cfg)
    wcw, wasg, whist = P.train_avq(x, 6, hp, ho, max_it=4, tol=0.0, seed=2)
    assert np.array_equal(cw.codewords.ravel(), np.asarray(wcw).ravel())
    assert np.array_equal(asg.assignments, np.asarray(wasg).ravel())
    assert np.array_equal(np.array(asg.loss_history), whist)
    q = aq.vq_quantize(x, cw, aq.ThresholdWeights(0.2))
    assert np.array_equal(q, P.vq_quantize(x, np.asarray(wcw).ravel(), hp, ho))


def test_search_f64():
    x = _unit_rows(5000, 32, 15)
    Q = _unit_rows(24, 32, 16)
    ids, sc = aq.dev_exact_search(aq.Session.default().upload_dataset(x), Q, 20)
    wi, ws = P.exact_search_batch(Q, x, 20)
    assert np.array_equal(ids, wi) and np.array_equal(sc, ws)
    M, k, sd = 16, 16, 2
    cb = aq.ProductCodebook(M, k, sd, random_codebook(M, k, sd, 6) * 0.3)
    hp, ho = threshold_hp_ho(x, 0.2)
    codes = P.pq_quantize(x, cb.dictionaries, M, k, sd, hp, ho, 2)
    s = aq.Session.default()
    ds, dc, dcb = s.upload_dataset(x), s.upload_codes(aq.CodeMatrix(len(x), M, k, codes)), \
        s.upload_codebook(cb)
    aid, asc, rid, rsc = aq.dev_search_rerank(ds, dc, dcb, Q, 100, 10)
    wi, ws = P.adc_search_batch(Q, codes, k, cb.dictionaries, M, k, sd, 100)
    assert np.array_equal(aid, wi) and np.array_equal(asc, ws)
    ri, rs = P.rerank(Q, x, wi, 10)
    assert np.array_equal(rid, ri) and np.array_equal(rsc, rs)


def test_adc_single_codeword_odd_lut():
    # test_index.cpp:211-234 shape (M = 1, k = 1, d = 6): the filter table
    # follows nq M k doubles, which is an odd multiple of 8 bytes here
    g = np.random.default_rng(5)
    x = g.standard_normal((30, 6)).astype(np.float32)
    cb = aq.ProductCodebook(1, 1, 6, x[0].astype(np.float64))
    codes = aq.CodeMatrix(30, 1, 1, np.zeros((30, 1), np.uint32))
    for topn in (1, 10, 30):
        for q in g.standard_normal((3, 6)):
            res = aq.adc_search(q, codes, cb, topn)
            wi, ws = P.adc_search_batch(q[None, :], codes.codes, 1, cb.dictionaries, 1, 1, 6, topn)
            assert [h.index for h in res.hits] == list(wi[0])
