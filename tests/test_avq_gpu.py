"""GPU parity: anisotropic vector quantization (train_avq, vq.hpp:243-329)
against the oracle port on seeded inputs — codewords, assignments and loss
history bit-identical, including both empty-partition policies (vq.hpp:
276-292) and anisotropic / isotropic / per-point weights."""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()


def _check(x, k, weights, hp, ho, cfg, keep=False):
    cb, a = aq.train_avq(x, k, weights, cfg)
    want_cw, want_a, want_hist = P.train_avq(
        x.astype(np.float64), k, hp, ho, max_it=cfg.max_iterations,
        tol=cfg.relative_tolerance, seed=cfg.seed, ridge=cfg.ridge, keep_previous=keep)
    assert np.array_equal(np.array(a.loss_history), want_hist)
    assert np.array_equal(a.assignments, want_a)
    assert np.array_equal(cb.codewords, want_cw)
    return cb, a


@pytest.mark.parametrize("d", [8, 32])
def test_train_avq_threshold_weights(d):
    x = mixture_rows(3000, d, 71, centers=12, sigma=0.3, normalize=True)
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=6, relative_tolerance=0.0, seed=9)
    _, a = _check(x, 16, aq.ThresholdWeights(0.2), hp, ho, cfg)
    h = a.loss_history
    assert all(b <= q + 1e-9 for q, b in zip(h, h[1:]))  # non-increasing (vq.hpp:239-241)


def test_train_avq_isotropic_is_kmeans_with_tolerance():
    x = mixture_rows(2500, 6, 72, centers=9, sigma=0.4, normalize=False)
    ones = np.ones(len(x))
    cfg = aq.TrainConfig(max_iterations=30, relative_tolerance=1e-6, seed=4)
    _check(x, 20, aq.AnisotropicWeights.isotropic(), ones, ones, cfg)


@pytest.mark.parametrize("keep", [False, True])
def test_train_avq_empty_partitions(keep):
    # 20 distinct rows, k = 30: duplicated codewords leave partitions empty
    g = np.random.default_rng(7)
    base = g.standard_normal((20, 5))
    x = base[g.integers(0, 20, 400)].astype(np.float32)
    for eta in (1.0, 2.5):
        hp, ho = np.full(400, eta), np.ones(400)
        policy = "keep_previous" if keep else "reseed_highest_loss"
        cfg = aq.TrainConfig(max_iterations=6, relative_tolerance=0.0, seed=1,
                             empty_partition_policy=policy)
        _, a = _check(x, 30, aq.AnisotropicWeights.from_eta(eta), hp, ho, cfg, keep)
        assert (np.bincount(a.assignments, minlength=30) == 0).any()


def test_train_avq_per_point_weights_and_errors():
    x = mixture_rows(800, 4, 73, centers=5, sigma=0.3, normalize=False)
    g = np.random.default_rng(11)
    hp, ho = 1.0 + 3.0 * g.random(800), 0.5 + g.random(800)
    ws = [aq.AnisotropicWeights(float(a), float(b)) for a, b in zip(hp, ho)]
    cfg = aq.TrainConfig(max_iterations=5, relative_tolerance=0.0, seed=2, ridge=1e-3)
    _check(x, 12, ws, hp, ho, cfg)
    with pytest.raises(aq.InvalidArgument):
        aq.train_avq(x, 0, aq.AnisotropicWeights.isotropic(), cfg)
    with pytest.raises(aq.InvalidArgument):
        aq.train_avq(x[:5], 6, aq.AnisotropicWeights.isotropic(), cfg)
    with pytest.raises(aq.EmptyDataset):
        aq.train_avq(np.zeros((0, 4), np.float32), 1, aq.AnisotropicWeights.isotropic(), cfg)


def test_vq_api_matches_oracle():
    # vq_quantize, assign_point, update_codeword (vq.hpp:112-192, 332-343)
    g = np.random.default_rng(21)
    x = mixture_rows(3000, 12, 74, centers=10, sigma=0.3, normalize=False)
    cw = g.standard_normal((20, 12))
    hp, ho = 1.0 + 3.0 * g.random(3000), np.ones(3000)
    ws = [aq.AnisotropicWeights(float(a), 1.0) for a in hp]
    cb = aq.Codebook(20, 12, cw)
    got = aq.vq_quantize(x, cb, ws)
    assert np.array_equal(got, P.vq_quantize(x.astype(np.float64), cw, hp, ho))
    for i in range(0, 3000, 150):
        w = aq.AnisotropicWeights(float(hp[i]), 1.0)
        assert aq.assign_point(x[i].astype(np.float64), cb, w) == P.assign_point(
            x[i].astype(np.float64), cw, hp[i], 1.0)
    pts = x[:300]
    for h in (hp[:300], np.ones(300)):
        w = [aq.AnisotropicWeights(float(a), 1.0) for a in h]
        assert np.array_equal(aq.update_codeword(12, pts, w),
                              P.update_codeword(12, pts.astype(np.float64), h, np.ones(300)))
    with pytest.raises(aq.InvalidArgument):
        aq.update_codeword(12, pts[:, :5], [aq.AnisotropicWeights()] * 300)
    with pytest.raises(aq.DimensionMismatch):
        aq.vq_quantize(x[:, :6], cb, ws)
    with pytest.raises(aq.InvalidArgument):
        aq.assign_point(x[0], aq.Codebook(0, 12, np.zeros((0, 12))), aq.AnisotropicWeights())
