"""GPU: float64 sequential sums (std::accumulate order; pq.hpp:553,562,
vq.hpp:270,316) through the chunk-parallel path (train.cu, seq_sums_on) are
bit-identical to a value-by-value chain, including the cases that force the
value-by-value fallback: ties at half an ulp, binade crossings, zero and tiny
starts, negative or non-finite rows."""
import ctypes as C

import numpy as np
import pytest

from paper_1908_10396_b200 import anisoq as aq

pytestmark = pytest.mark.gpu
L = aq._L


def _chain(v, init=0.0):
    return float(np.add.accumulate(np.concatenate([[init], v]))[-1])


def _dev(arr):
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr, np.float64)).cuda()


def _sum(v, init=0.0):
    s = aq.Session.default()
    t = _dev(v)
    out = C.c_double(0.0)
    aq._check(L.aq_dev_seq_sum(s.h, t.data_ptr(), t.numel(), init, C.byref(out)))
    return out.value


def _rows():
    g = np.random.default_rng(7)
    n = 300_000
    tiny = 2.0 ** -53
    cases = {
        "exponential": g.exponential(1.0, n),
        "lognormal": g.lognormal(0.0, 3.0, n),
        # half-ulp ties around s in [1, 2) and [2, 4): values 2^-53, 3 * 2^-53
        "ties": np.where(g.random(n) < 0.5, tiny, 3 * tiny) * g.integers(1, 3, n),
        "growing": np.geomspace(1e-30, 1e10, n),
        "zeros_then_values": np.concatenate([np.zeros(n // 2), g.random(n - n // 2)]),
        "mixed_scales": g.random(n) * np.where(g.random(n) < 0.001, 1e12, 1e-3),
        "integers": np.ones(n),
    }
    return cases


@pytest.mark.parametrize("name", list(_rows().keys()))
def test_seq_sum_matches_chain(name):
    v = _rows()[name]
    assert _sum(v) == _chain(v)
    assert _sum(v, 1.0) == _chain(v, 1.0)


def test_seq_sum_ties_at_start_value():
    # s = 1 + k ulp, every addend exactly half an ulp: round-half-even decides
    v = np.full(200_000, 2.0 ** -53)
    for init in (1.0, 1.0 + 2.0 ** -52, 3.0):
        assert _sum(v, init) == _chain(v, init)


def test_seq_sum_negative_and_nonfinite_rows_take_the_plain_chain():
    g = np.random.default_rng(9)
    v = g.random(200_000)
    w = v.copy()
    w[1234] = -0.5
    assert _sum(w) == _chain(w)
    w = v.copy()
    w[-1] = np.inf
    assert _sum(w) == _chain(w)
    w = v.copy()
    w[77] = -0.0
    assert _sum(w) == _chain(w)


def test_seq_sums_rows_and_active():
    s = aq.Session.default()
    g = np.random.default_rng(11)
    rows, n = 5, 150_000
    v = g.exponential(2.0, (rows, n))
    v[3, ::7] = 2.0 ** -60
    t = _dev(v)
    act = np.array([1, 1, 0, 1, 1], np.int32)
    out = np.zeros(rows)
    aq._check(L.aq_dev_seq_sums(s.h, t.data_ptr(), n, n, rows, act.ctypes.data, out.ctypes.data))
    for r in range(rows):
        assert out[r] == (_chain(v[r]) if act[r] else 0.0)
