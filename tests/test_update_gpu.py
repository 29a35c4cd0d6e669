"""GPU parity: normal-equation assembly and the joint codebook update
(pq.hpp:290-464) against the oracle. The device accumulates every entry in
the reference's point order and mirrors the pinned blocked Cholesky, so the
matrix, rhs and codebooks are bit-identical."""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()


def _codes(n, M, k, seed, low=0):
    return np.random.default_rng(seed).integers(low, k, (n, M)).astype(np.uint32)


@pytest.mark.parametrize("n,d,M,k", [(3000, 32, 16, 16), (2000, 24, 8, 5), (1500, 12, 4, 16),
                                     (800, 16, 8, 6)])
def test_assemble_matches_oracle(n, d, M, k):
    x = mixture_rows(n, d, 51)
    codes = _codes(n, M, k, 52)
    hp, ho = threshold_hp_ho(x, 0.2)
    A, r = aq.assemble_selector_system(x, aq.CodeMatrix(n, M, k, codes), (hp, ho), M, k)
    A2, r2 = P.assemble_selector_system(x.astype(np.float64), codes, hp, ho, M, k)
    assert np.array_equal(A, A2)
    assert np.array_equal(r, r2)


@pytest.mark.parametrize("case", ["aniso", "iso", "unused", "per_point", "c1", "ridge"])
def test_codebook_update_matches_oracle(case):
    n, d, M, k = (2000, 32, 16, 16) if case != "c1" else (20000, 32, 16, 16)
    x = mixture_rows(n, d, 53)
    codes = _codes(n, M, k, 54)
    hp, ho = threshold_hp_ho(x, 0.2)
    w = aq.ThresholdWeights(0.2)
    ridge = -1.0
    if case == "iso":
        hp = ho = np.full(n, 1.5)
        w = aq.AnisotropicWeights.isotropic(1.5)
    elif case == "unused":
        codes = _codes(n, M, 3, 55)  # codewords 3..15 never used -> reseeded
    elif case == "per_point":
        g = np.random.default_rng(9)
        hp, ho = g.uniform(0.5, 8.0, n), g.uniform(0.5, 2.0, n)
        w = (hp, ho)
    elif case == "ridge":
        ridge = 1e-8
    got = aq.pq_codebook_update(x, aq.CodeMatrix(n, M, k, codes), w, M, k, ridge)
    want = P.pq_codebook_update(x.astype(np.float64), codes, hp, ho, M, k, ridge)
    assert np.array_equal(got.dictionaries, want)


def test_codebook_update_sd3():
    n, d, M, k = 1800, 24, 8, 8
    x = mixture_rows(n, d, 56)
    codes = _codes(n, M, k, 57)
    hp, ho = threshold_hp_ho(x, 0.2)
    got = aq.pq_codebook_update(x, aq.CodeMatrix(n, M, k, codes), aq.ThresholdWeights(0.2), M, k)
    want = P.pq_codebook_update(x.astype(np.float64), codes, hp, ho, M, k)
    assert np.array_equal(got.dictionaries, want)


def test_codebook_update_errors():
    x = mixture_rows(100, 8, 58)
    with pytest.raises(aq.EmptyDataset):
        aq.pq_codebook_update(np.zeros((0, 8), np.float32), aq.CodeMatrix(0, 4, 4, np.zeros((0, 4))),
                              aq.AnisotropicWeights(), 4, 4)
    with pytest.raises(aq.DimensionNotDivisible):
        aq.pq_codebook_update(x, aq.CodeMatrix(100, 3, 4, np.zeros((100, 3))),
                              aq.AnisotropicWeights(), 3, 4)
    with pytest.raises(aq.CodeOutOfRange):
        aq.pq_codebook_update(x, aq.CodeMatrix(100, 4, 9, np.full((100, 4), 8)),
                              aq.AnisotropicWeights(), 4, 4)
    x2 = x.copy()
    x2[5] = 0
    with pytest.raises(aq.ZeroNormDatapoint):
        aq.pq_codebook_update(x2, aq.CodeMatrix(100, 4, 4, _codes(100, 4, 4, 1)),
                              aq.AnisotropicWeights.from_eta(2.0), 4, 4)


@pytest.mark.parametrize("w", ["aniso", "iso", "mixed"])
def test_codebook_update_m1_vq_closed_form(w):
    # pq.hpp:387-404 -> update_codeword (vq.hpp:139-192); test_pq.cpp:209-239
    n, d, k = 400, 5, 5
    x = mixture_rows(n, d, 59)
    codes = _codes(n, 1, k, 60)
    if w == "aniso":
        hp, ho = np.full(n, 4.125), np.ones(n)
    elif w == "iso":
        hp = ho = np.full(n, 2.0)
    else:
        hp, ho = np.full(n, 4.125), np.ones(n)
        hp[codes[:, 0] == 2] = 1.0  # codeword 2 gets only isotropic members
    for ridge in (-1.0, 1e-9):
        got = aq.pq_codebook_update(x, aq.CodeMatrix(n, 1, k, codes), (hp, ho), 1, k, ridge)
        want = P.pq_codebook_update(x.astype(np.float64), codes, hp, ho, 1, k, ridge)
        assert np.array_equal(got.dictionaries, want)
