"""GPU: the C ABI's host-pointer entry points (the reference's by-value
semantics) called through ctypes, bit-identical to the oracle."""
import ctypes as C

import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import _lib, anisoq as aq
from tests.helpers import mixture_rows, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()
L = aq._L


def _ptr(a):
    return a.ctypes.data


def _w_threshold(t=0.2):
    w = _lib.aq_weights()
    w.mode = 2
    w.threshold = t
    w.threshold_policy = 1
    return w


def test_host_search_rerank_exact():
    s = aq.Session.default()
    x = mixture_rows(5000, 16, 3)
    g = np.random.default_rng(5)
    M, k, sd, n = 8, 16, 2, len(x)
    cbd = g.standard_normal(M * k * sd) * 0.3
    codes = g.integers(0, k, (n, M)).astype(np.uint32)
    Q = g.standard_normal((7, 16))
    ids = np.zeros((7, 50), np.uint32)
    sc = np.zeros((7, 50))
    aq._check(L.aq_adc_search_batch(s.h, _ptr(Q), 7, 16, _ptr(codes), n, M, k, _ptr(cbd), M, k,
                                    sd, 50, _ptr(ids), _ptr(sc)))
    wi, ws = P.adc_search_batch(Q, codes, k, cbd, M, k, sd, 50)
    assert np.array_equal(ids, wi) and np.array_equal(sc, ws)
    rid = np.zeros((7, 10), np.uint32)
    rsc = np.zeros((7, 10))
    aq._check(L.aq_rerank(s.h, _ptr(Q), 7, _ptr(x), n, 16, _ptr(ids), 50, 10, _ptr(rid),
                          _ptr(rsc)))
    wi, ws = P.rerank(Q, x.astype(np.float64), wi, 10)
    assert np.array_equal(rid, wi) and np.array_equal(rsc, ws)
    eid = np.zeros((7, 10), np.uint32)
    esc = np.zeros((7, 10))
    aq._check(L.aq_exact_search_batch(s.h, _ptr(Q), 7, _ptr(x), n, 16, 10, _ptr(eid),
                                      _ptr(esc)))
    wi, ws = P.exact_search_batch(Q, x.astype(np.float64), 10)
    assert np.array_equal(eid, wi) and np.array_equal(esc, ws)
    with pytest.raises(aq.EmptyIndex):
        aq._check(L.aq_adc_search_batch(s.h, _ptr(Q), 7, 16, _ptr(codes), 0, M, k, _ptr(cbd), M,
                                        k, sd, 50, _ptr(ids), _ptr(sc)))


def test_host_assemble_and_trainers():
    s = aq.Session.default()
    x = mixture_rows(3000, 16, 9)
    n, d, M, k = len(x), 16, 4, 16
    hp, ho = threshold_hp_ho(x, 0.2)
    w = _w_threshold()
    codes = np.random.default_rng(1).integers(0, k, (n, M)).astype(np.uint32)
    A = np.zeros((k * d, k * d))
    rhs = np.zeros(k * d)
    aq._check(L.aq_assemble_selector_system(s.h, _ptr(x), n, d, _ptr(codes), M, k, C.byref(w),
                                            _ptr(A), _ptr(rhs)))
    wa, wr = P.assemble_selector_system(x.astype(np.float64), codes, hp, ho, M, k)
    assert np.array_equal(A, wa) and np.array_equal(rhs, wr)
    cfg = aq.TrainConfig(max_iterations=4, relative_tolerance=0.0, seed=3).c()
    dic = np.zeros(k * d)
    cod = np.zeros((n, M), np.uint32)
    aq._check(L.aq_train_l2_pq(s.h, _ptr(x), n, d, M, k, C.byref(cfg), _ptr(dic), _ptr(cod)))
    wd, wc = P.train_l2_pq(x.astype(np.float64), M, k, 4, 0.0, 3)
    assert np.array_equal(dic, wd) and np.array_equal(cod, wc)
    hist = np.zeros(5)
    hl = C.c_size_t(0)
    aq._check(L.aq_train_apq(s.h, _ptr(x), n, d, M, k, C.byref(w), C.byref(cfg), 1, _ptr(dic),
                             _ptr(cod), _ptr(hist), C.byref(hl)))
    wd, wc, wh = P.train_apq(x.astype(np.float64), M, k, hp, ho, max_it=4, tol=0.0, seed=3)
    assert np.array_equal(dic, wd) and np.array_equal(cod, wc)
    assert hist[: hl.value].tolist() == wh.tolist()
