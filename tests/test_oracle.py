"""Pins the oracle (C restatement) before it is trusted as the parity checker.

* against the reference itself, compiled in place (oracle/_ref), on seeded
  inputs covering every hot-path function;
* against the reference tests' worked examples and golden bytes
  (test_index.cpp:58-112, test_pq.cpp:29-37, rng contract test_pq.cpp:334-357);
* against the committed golden fixtures (tests/golden/, made by
  tests/golden/make_golden.py from oracle/_ref).
"""
import os

import numpy as np
import pytest

from oracle import Port, Reference
from tests.helpers import lognormal_rows, mixture_rows, random_codebook, threshold_hp_ho

P = Port()
# the reference is built by build() (make -C oracle) and travels with the
# repository: tests that need it fail, not skip, when it is missing
needs_ref = pytest.mark.usefixtures()
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz")


def _ref():
    assert Reference.available(), "oracle/_ref/libanisoq_ref.so missing (make -C oracle)"
    return Reference()


def test_lut_worked_example():
    # test_index.cpp:58-67 (Appendix A.5 dictionaries)
    cb = np.array([-1, -1, 1, 1, -2, -2, 2, 2], np.float64)
    lut = P.build_lut(np.array([1.0, 0.0, 1.0, 0.0]), cb, 2, 2, 2)
    assert lut.tolist() == [-1.0, 1.0, -2.0, 2.0]
    assert P.build_lut(np.zeros(4), cb, 2, 2, 2).tolist() == [0.0] * 4


def test_adc_score_worked_example():
    # test_index.cpp:85-90: codes {0, 1} under q = (1,0,1,0) score exactly 1
    cb = np.array([-1, -1, 1, 1, -2, -2, 2, 2], np.float64)
    codes = np.array([[0, 1], [1, 0], [1, 1], [0, 0]], np.uint32)
    ids, sc = P.adc_search_batch(np.array([[1.0, 0.0, 1.0, 0.0]]), codes, 2, cb, 2, 2, 2, 4)
    assert ids[0].tolist() == [2, 0, 1, 3]
    assert sc[0].tolist() == [3.0, 1.0, -1.0, -3.0]


def test_eta_limit_config_values():
    # eta = (d-1) T^2 / (1 - T^2) for unit norms (geometry.hpp:395-402)
    hp, ho = P.threshold_weights(np.ones(3), 32, 0.2)
    assert abs(hp[0] - 31 * 0.04 / 0.96) < 1e-15 and ho[0] == 1.0
    hp, _ = P.threshold_weights(np.ones(1), 100, 0.2)
    assert abs(hp[0] - 4.125) < 1e-12
    hp, _ = P.threshold_weights(np.ones(1), 256, 0.2)
    assert abs(hp[0] - 10.625) < 1e-12
    # |x| <= T: reference throws; policy 1 = parallel only
    hp, ho = P.threshold_weights(np.array([0.1]), 32, 0.2, policy=1)
    assert (hp[0], ho[0]) == (1.0, 0.0)
    with pytest.raises(Exception):
        P.threshold_weights(np.array([0.1]), 32, 0.2, policy=0)


@needs_ref
def test_sample_distinct_contract():
    R = _ref()
    for seed, n, k in [(0, 100, 16), (40, 300, 6), (7, 5, 9), (123, 20000, 16)]:
        assert P.sample_distinct(seed, n, k).tolist() == R.sample_distinct(seed, n, k).tolist()


@needs_ref
@pytest.mark.parametrize("passes", [0, 1, 3])
@pytest.mark.parametrize("shape", ["c1", "c3", "iso"])
def test_pq_quantize_port_equals_reference(passes, shape):
    R = _ref()
    if shape == "c3":
        x = lognormal_rows(1500, 32, 3).astype(np.float64)
        hp, ho = threshold_hp_ho(x, 0.2)
    else:
        x = mixture_rows(1500, 32, 4).astype(np.float64)
        hp, ho = threshold_hp_ho(x, 0.2)
        if shape == "iso":
            hp = ho = np.ones(len(x))
    cb = random_codebook(16, 16, 2, 5)
    a = P.pq_quantize(x, cb, 16, 16, 2, hp, ho, passes)
    b = R.pq_quantize(x, cb, 16, 16, 2, hp, ho, passes, threads=4)
    assert np.array_equal(a, b)


@needs_ref
@pytest.mark.parametrize("fixed", [False, True])
def test_assign_pass_port_equals_reference(fixed):
    R = _ref()
    x = mixture_rows(1200, 24, 6).astype(np.float64)
    hp, ho = threshold_hp_ho(x, 0.2)
    cb = random_codebook(8, 8, 3, 7)
    c0 = np.random.default_rng(1).integers(0, 8, (len(x), 8)).astype(np.uint32)
    a = P.pq_assign_pass(x, cb, 8, 8, 3, hp, ho, c0, fixed)
    b = R.pq_assign_pass(x, cb, 8, 8, 3, hp, ho, c0, fixed, threads=3)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@needs_ref
@pytest.mark.parametrize("case", ["aniso", "iso", "m1", "unused"])
def test_codebook_update_port_equals_reference(case):
    R = _ref()
    x = mixture_rows(600, 16, 8).astype(np.float64)
    hp, ho = threshold_hp_ho(x, 0.2)
    M, k = (8, 6) if case != "m1" else (1, 5)
    g = np.random.default_rng(2)
    codes = g.integers(0, k, (len(x), M)).astype(np.uint32)
    if case == "iso":
        hp = ho = np.full(len(x), 1.5)
    if case == "unused":
        codes[:, :] = g.integers(0, 2, codes.shape)
    A1, r1 = P.assemble_selector_system(x, codes, hp, ho, M, k)
    A2, r2 = R.assemble_selector_system(x, codes, hp, ho, M, k)
    assert np.array_equal(A1, A2) and np.array_equal(r1, r2)
    u1 = P.pq_codebook_update(x, codes, hp, ho, M, k)
    u2 = R.pq_codebook_update(x, codes, hp, ho, M, k)
    assert np.array_equal(u1, u2)


@needs_ref
@pytest.mark.parametrize("warm", [True, False])
def test_train_apq_port_equals_reference(warm):
    R = _ref()
    x = mixture_rows(1000, 16, 9).astype(np.float64)
    hp, ho = threshold_hp_ho(x, 0.2)
    a = P.train_apq(x, 8, 16, hp, ho, max_it=4, tol=0.0, seed=3, warm_start=warm)
    b = R.train_apq(x, 8, 16, hp, ho, max_it=4, tol=0.0, seed=3, warm_start=warm, threads=2)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)


@needs_ref
@pytest.mark.parametrize("keep", [False, True])
def test_train_avq_port_equals_reference(keep):
    # vq.hpp:243-329, including empty partitions (20 distinct rows, k = 30)
    R = _ref()
    g = np.random.default_rng(7)
    base = g.standard_normal((20, 5))
    dup = base[g.integers(0, 20, 400)].astype(np.float32).astype(np.float64)
    x = mixture_rows(900, 8, 10).astype(np.float64)
    for data, k in ((x, 16), (dup, 30)):
        hp, ho = threshold_hp_ho(data, 0.2)
        a = P.train_avq(data, k, hp, ho, max_it=5, tol=0.0, seed=3, keep_previous=keep)
        b = R.train_avq(data, k, hp, ho, max_it=5, tol=0.0, seed=3, keep_previous=keep,
                        threads=2)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)


@needs_ref
def test_vq_api_port_equals_reference():
    # vq_quantize / assign_point / update_codeword (vq.hpp:112-192, 332-343)
    R = _ref()
    g = np.random.default_rng(3)
    x = g.standard_normal((500, 6)).astype(np.float32).astype(np.float64)
    cw = g.standard_normal(12 * 6)
    hp, ho = 1 + 2 * g.random(500), np.ones(500)
    assert np.array_equal(P.vq_quantize(x, cw, hp, ho), R.vq_quantize(x, cw, hp, ho, threads=3))
    for i in range(40):
        assert P.assign_point(x[i], cw, hp[i], 1.0) == R.assign_point(x[i], cw, hp[i], 1.0)
    for h in (hp[:40], np.ones(40)):
        assert np.array_equal(P.update_codeword(6, x[:40], h, ho[:40], 1e-3),
                              R.update_codeword(6, x[:40], h, ho[:40], 1e-3))


@needs_ref
def test_search_port_equals_reference():
    R = _ref()
    x = mixture_rows(3000, 32, 10).astype(np.float64)
    q = mixture_rows(12, 32, 11).astype(np.float64)
    cb = random_codebook(16, 16, 2, 12)
    codes = np.random.default_rng(3).integers(0, 16, (len(x), 16)).astype(np.uint32)
    i1, s1 = P.adc_search_batch(q, codes, 16, cb, 16, 16, 2, 100)
    i2, s2 = R.adc_search_batch(q, codes, 16, cb, 16, 16, 2, 100, threads=4)
    assert np.array_equal(i1, i2) and np.array_equal(s1, s2)
    j1, t1 = P.rerank(q, x, i1, 10)
    j2, t2 = R.rerank(q, x, i1, 10)
    assert np.array_equal(j1, j2) and np.array_equal(t1, t2)
    e1 = P.exact_search_batch(q, x, 10)
    e2 = R.exact_search_batch(q, x, 10, threads=2)
    assert np.array_equal(e1[0], e2[0]) and np.array_equal(e1[1], e2[1])


def test_golden_fixtures():
    """Port reproduces the reference outputs frozen in tests/golden (no _ref needed)."""
    g = np.load(GOLDEN)
    x = g["x"].astype(np.float64)
    hp, ho = g["hp"], g["ho"]
    cb = g["cb"]
    assert np.array_equal(P.pq_quantize(x, cb, 16, 16, 2, hp, ho, 3), g["quantize3"])
    c, l = P.pq_assign_pass(x, cb, 16, 16, 2, hp, ho, g["codes0"])
    assert np.array_equal(c, g["assign_codes"]) and np.array_equal(l, g["assign_losses"])
    assert np.array_equal(P.pq_codebook_update(x, g["codes0"], hp, ho, 16, 16), g["update"])
    ids, sc = P.adc_search_batch(g["q"].astype(np.float64), g["codes0"], 16, cb, 16, 16, 2, 100)
    assert np.array_equal(ids, g["adc_ids"]) and np.array_equal(sc, g["adc_scores"])
    cbt, ct, h = P.train_apq(x[:800], 16, 16, hp[:800], ho[:800], max_it=3, tol=0.0, seed=0)
    assert np.array_equal(cbt, g["train_cb"]) and np.array_equal(ct, g["train_codes"])
    assert np.array_equal(h, g["train_hist"])
    cw, a, h = P.train_avq(x[:1000], 24, hp[:1000], ho[:1000], max_it=4, tol=0.0, seed=5)
    assert np.array_equal(cw, g["avq_cw"]) and np.array_equal(a, g["avq_assign"])
    assert np.array_equal(h, g["avq_hist"])
