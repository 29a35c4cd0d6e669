"""Multi-device session (csrc/multi.cu, aq_multi_*): the database in row
shards over several sessions of one process. This box has one B200, so the
shards share it (devices [0, 0, 0]); the code path — per-shard sessions and
streams, peer copies between the shards' buffers, the shard-ordered chain
sums, the merge — is the one an 8-GPU box runs, and the results depend only
on the shard count.

* pq_quantize and adc_search equal the oracle bit for bit for any shard count
  (unequal shards, top-N larger than a shard);
* train_apq with W shards: codebooks within 1e-12 relative of the oracle's,
  loss history within 1e-12, codes equal except near-ties (a differing code
  within eps_c = 2^-20 x max loss of the oracle's under the trained codebook,
  SURVEY.md §8(c) rule 1), deterministic run to run.
"""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows, random_codebook, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()


@pytest.mark.parametrize("W", [1, 2, 3, 5])
def test_multi_quantize_and_search(W):
    ms = aq.MultiSession([0] * W)
    assert ms.shards == W
    x = mixture_rows(4003, 32, 81)
    M, k, sd = 16, 16, 2
    cb = aq.ProductCodebook(M, k, sd, random_codebook(M, k, sd, 5) * 0.3)
    hp, ho = threshold_hp_ho(x, 0.2)
    codes = ms.pq_quantize(x, cb, aq.ThresholdWeights(0.2), 3)
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, M, k, sd, hp, ho, 3)
    assert np.array_equal(codes.codes, want)
    Q = mixture_rows(9, 32, 82).astype(np.float64)
    for topn in (1, 100, 1000):  # 1000 > every shard of 4003 / 5
        ids, sc = ms.adc_search(Q, codes, cb, topn)
        wi, ws = P.adc_search_batch(Q, want, k, cb.dictionaries, M, k, sd, topn)
        assert np.array_equal(ids, wi) and np.array_equal(sc, ws)


def test_multi_errors_carry_global_indices():
    ms = aq.MultiSession([0, 0])
    x = mixture_rows(100, 8, 83)
    x[77] = 0.0  # zero norm in shard 1
    cb = aq.ProductCodebook(4, 4, 2, random_codebook(4, 4, 2, 6))
    with pytest.raises(aq.InvalidArgument):  # eta_limit needs |x| > 0 (geometry.hpp:396)
        ms.pq_quantize(x, cb, aq.ThresholdWeights(0.2), 1)


@pytest.mark.parametrize("W,warm", [(1, True), (2, True), (3, False), (4, True)])
def test_multi_train_apq(W, warm):
    ms = aq.MultiSession([0] * W)
    x = mixture_rows(3000, 16, 84)
    M, k = 8, 16
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=4, relative_tolerance=0.0, seed=3)
    hist = []
    cb, codes = ms.train_apq(x, M, k, aq.ThresholdWeights(0.2), cfg, warm, hist)
    wcb, wcodes, whist = P.train_apq(x.astype(np.float64), M, k, hp, ho, max_it=4, tol=0.0,
                                     seed=3, warm_start=warm)
    if W == 1:  # one shard: the single-device trainer, bit for bit
        assert np.array_equal(cb.dictionaries, wcb) and np.array_equal(codes.codes, wcodes)
        assert np.array_equal(np.array(hist), whist)
        return
    assert np.allclose(cb.dictionaries, wcb, rtol=0, atol=1e-12 * np.abs(wcb).max())
    assert np.allclose(hist, whist, rtol=1e-12)
    loss = P.pq_point_losses(x.astype(np.float64), cb.dictionaries, M, k, 2, hp, ho,
                             codes.codes)
    eps = 2.0 ** -20 * loss.max()
    for i in np.nonzero((codes.codes != wcodes).any(axis=1))[0]:
        alt = P.pq_point_losses(x[i:i + 1].astype(np.float64), cb.dictionaries, M, k, 2,
                                hp[i:i + 1], ho[i:i + 1], wcodes[i:i + 1])
        assert abs(alt[0] - loss[i]) <= eps
    hist2 = []
    cb2, codes2 = ms.train_apq(x, M, k, aq.ThresholdWeights(0.2), cfg, warm, hist2)
    assert np.array_equal(cb2.dictionaries, cb.dictionaries) and hist2 == hist


def test_multi_train_isotropic_and_reseed():
    """Isotropic weights (mean path) and duplicated rows, so codewords go
    unused and are reseeded from the global loss ranking across shards."""
    ms = aq.MultiSession([0, 0, 0])
    base = mixture_rows(50, 8, 85)
    x = np.repeat(base, 8, axis=0)
    M, k = 4, 64
    cfg = aq.TrainConfig(max_iterations=3, relative_tolerance=0.0, seed=1)
    for wts, arrs in ((aq.AnisotropicWeights.isotropic(), None), (aq.ThresholdWeights(0.2),
                                                                  threshold_hp_ho(x, 0.2))):
        hp, ho = arrs if arrs else (np.ones(len(x)), np.ones(len(x)))
        hist = []
        cb, codes = ms.train_apq(x, M, k, wts, cfg, False, hist)
        wcb, wcodes, whist = P.train_apq(x.astype(np.float64), M, k, hp, ho, max_it=3,
                                         tol=0.0, seed=1, warm_start=False)
        assert np.allclose(cb.dictionaries, wcb, rtol=0, atol=1e-12 * np.abs(wcb).max())
        assert np.allclose(hist, whist, rtol=1e-12)
