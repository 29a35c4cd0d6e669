"""GPU: the reference's property pins that are not plain
oracle comparisons, restated against the device path with the reference
tests' parameters:

  M = 1 assignment == VQ assignment bitwise          test_pq.cpp:79-95
  coordinate descent descends, reaches a fixed point,
    never beats brute force (M = 2, k = 2)           test_pq.cpp:125-162
  codebook update with fixed codes never raises loss test_pq.cpp:288-302
  score-aware codes lower the top-1 relative error   test_index.cpp:265-291
  retraining reproduces the codebook bytes           acceptance_main.cpp:731-750
  ADC scores == reconstructed dot products           acceptance check 9 (638-696)
"""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows

pytestmark = pytest.mark.gpu


def _residual_terms(x, c):  # geometry.hpp:182-192
    d2 = rd = 0.0
    for xt, ct in zip(x, c):
        diff = float(xt) - float(ct)
        d2 += diff * diff
        rd += diff * float(xt)
    return d2, rd


def _vq_assign(x, C, w):
    """assign_point / assign_scan (vq.hpp:83-126), restated in IEEE doubles."""
    iso = w.h_parallel == w.h_perpendicular
    inv = 0.0
    if not iso:
        n2 = 0.0
        for xt in x:
            n2 += float(xt) * float(xt)
        inv = 1.0 / n2
    best, bj = None, 0
    for j in range(C.shape[0]):
        d2, rd = _residual_terms(x, C[j])
        s = d2 if iso else (w.h_perpendicular * d2 +
                            (w.h_parallel - w.h_perpendicular) * (rd * rd) * inv)
        if best is None or s < best:
            best, bj = s, j
    return bj


def _aniso_loss(x, xq, w):  # anisotropic_loss (geometry.hpp:405-415)
    n2 = float(np.dot(x, x))
    d2, rd = _residual_terms(x, xq)
    return max(0.0, w.h_perpendicular * d2 +
               (w.h_parallel - w.h_perpendicular) * (rd * rd) * (1.0 / n2))


def _reconstruct(codes, cb):
    return np.concatenate([cb.codeword(m, int(c)) for m, c in enumerate(codes)])


def test_m1_assignment_equals_vq_bitwise():
    g = np.random.default_rng(301)
    C = g.standard_normal((6, 5))
    cb = aq.ProductCodebook(1, 6, 5, C.reshape(-1).copy())
    for rep in range(30):
        x = g.standard_normal(5)
        w = aq.AnisotropicWeights.from_eta(4.125) if rep % 2 == 0 else \
            aq.AnisotropicWeights.isotropic()
        start = np.array([g.integers(0, 6)], np.uint32)
        got = aq.pq_assign_point(x, start, cb, w)
        assert int(got[0]) == _vq_assign(x, C, w)


def test_descent_fixed_point_and_brute_force_bound():
    g = np.random.default_rng(303)
    w = aq.AnisotropicWeights.from_eta(4.125)
    for _ in range(20):
        cb = aq.ProductCodebook(2, 2, 2, g.standard_normal(8))
        x = g.standard_normal(4)
        x /= np.linalg.norm(x)
        brute = min(_aniso_loss(x, _reconstruct([a, b], cb), w)
                    for a in range(2) for b in range(2))
        for a in range(2):
            for b in range(2):
                start = np.array([a, b], np.uint32)
                l0 = _aniso_loss(x, _reconstruct(start, cb), w)
                end = aq.pq_assign_point(x, start, cb, w)
                l1 = _aniso_loss(x, _reconstruct(end, cb), w)
                assert l1 <= l0 * (1.0 + 1e-12) + 1e-15
                assert l1 >= brute - 1e-12
                for _ in range(8):
                    nxt = aq.pq_assign_point(x, end, cb, w)
                    if np.array_equal(nxt, end):
                        break
                    end = nxt
                assert np.array_equal(aq.pq_assign_point(x, end, cb, w), end)


def test_update_with_fixed_codes_never_increases_loss():
    x = mixture_rows(120, 8, 7, centers=6)
    M, k, sd = 4, 4, 2
    w = aq.AnisotropicWeights.from_eta(4.125)
    cb0, codes = aq.train_l2_pq(x, M, k, aq.TrainConfig())
    cb1 = aq.pq_codebook_update(x, codes, w, M, k)
    hp = np.full(len(x), 4.125)
    ho = np.ones(len(x))
    P = Port()
    xd = x.astype(np.float64)
    before = P.pq_point_losses(xd, cb0.dictionaries, M, k, sd, hp, ho, codes.codes).sum()
    after = P.pq_point_losses(xd, cb1.dictionaries, M, k, sd, hp, ho, codes.codes).sum()
    assert after <= before + 1e-9


def test_score_aware_codes_lower_top1_relative_error():
    data = mixture_rows(3000, 32, 91, centers=24, sigma=0.25)
    queries = mixture_rows(200, 32, 92, centers=24, sigma=0.25)
    cb, l2_codes = aq.train_l2_pq(data, 8, 16, aq.TrainConfig(seed=15))
    aniso_codes = aq.pq_quantize(data, cb, aq.ThresholdWeights(0.2), 2)
    opt = aq.EvalOptions(recall_ns=(1, 10))
    base = aq.evaluate(queries, data, l2_codes, cb, opt)
    aniso = aq.evaluate(queries, data, aniso_codes, cb, opt)
    assert aniso.relative_error_mean <= base.relative_error_mean


def test_retrain_reproduces_codebook_bytes():
    x = mixture_rows(5000, 32, 3)
    cfg = aq.TrainConfig(max_iterations=5, seed=9)
    w = aq.ThresholdWeights(0.2, "parallel_only")
    cb1, c1 = aq.train_apq(x, 16, 16, w, cfg)
    cb2, c2 = aq.train_apq(x, 16, 16, w, cfg)
    assert cb1.dictionaries.tobytes() == cb2.dictionaries.tobytes()
    assert np.array_equal(c1.codes, c2.codes)


def test_adc_scores_equal_reconstructed_dots():
    g = np.random.default_rng(9)
    M, k, sd, n = 16, 16, 2, 5000
    cb = aq.ProductCodebook(M, k, sd, g.standard_normal(M * k * sd))
    codes = aq.CodeMatrix(n, M, k, g.integers(0, k, (n, M), dtype=np.uint32))
    Q = g.standard_normal((20, M * sd))
    s = aq.Session.default()
    ids, sc = aq.dev_adc_search(s.upload_codes(codes), s.upload_codebook(cb), Q, n)
    rec = np.stack([_reconstruct(codes.codes[i], cb) for i in range(n)])
    want = Q @ rec.T  # 1e5 (query, point) pairs
    got = np.take_along_axis(want, ids.astype(np.int64), axis=1)
    assert np.max(np.abs(got - sc)) <= 1e-6
