"""GPU: the sharded trainer's device backend (DeviceShard over the aq_dev_*
building blocks of csrc/shard.cu). With one shard every partial is the full
sequential sum, so the sharded trainer must equal the oracle's single-process
train_apq bit for bit — codebook, codes and loss history. (A world of more
ranks needs more GPUs; its host logic is covered by test_sharded_train.py.)"""
import numpy as np
import pytest
import torch

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200.distributed import DeviceShard, ShardedTrainer
from tests.helpers import mixture_rows, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()


def _train(x, weights, M, k, cfg, warm):
    s = aq.Session.default()
    rows = torch.from_numpy(x).cuda()
    sh = DeviceShard(s, rows, weights)
    hist = []
    dict_ = ShardedTrainer(sh, len(x), 0).train_apq(M, k, cfg, warm, hist)
    return dict_.cpu().numpy(), sh.codes.download().codes, hist


@pytest.mark.parametrize("warm", [True, False])
def test_device_shard_equals_oracle_threshold(warm):
    x = mixture_rows(6000, 16, 21)
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=6, relative_tolerance=0.0, seed=8)
    d, codes, hist = _train(x, aq.ThresholdWeights(0.2, "parallel_only"), 8, 16, cfg, warm)
    cb, want, h = P.train_apq(x.astype(np.float64), 8, 16, hp, ho, max_it=6, tol=0.0, seed=8,
                              warm_start=warm)
    assert np.array_equal(d, cb)
    assert np.array_equal(codes, want)
    assert hist == h.tolist()


def test_device_shard_isotropic_reseed_per_point():
    base = mixture_rows(50, 8, 4)
    x = np.repeat(base, 6, axis=0)  # duplicated rows: partitions empty out
    one = np.ones(len(x))
    cfg = aq.TrainConfig(max_iterations=4, relative_tolerance=0.0, seed=2)
    for weights, (hp, ho), warm in [(aq.AnisotropicWeights.isotropic(), (one, one), False),
                                    ((np.full(len(x), 3.0), one), (np.full(len(x), 3.0), one),
                                     True)]:
        d, codes, hist = _train(x, weights, 4, 64, cfg, warm)
        cb, want, h = P.train_apq(x.astype(np.float64), 4, 64, hp, ho, max_it=4, tol=0.0,
                                  seed=2, warm_start=warm)
        assert np.array_equal(d, cb)
        assert np.array_equal(codes, want)
        assert hist == h.tolist()


def test_device_shard_default_tolerance_config1_shape():
    """config1's shape (d=100, M=50, k=16) with the default stopping rule."""
    g = np.random.default_rng(1)
    x = g.standard_normal((3000, 100)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=5, seed=0)
    d, codes, hist = _train(x, aq.ThresholdWeights(0.2, "parallel_only"), 50, 16, cfg, True)
    cb, want, h = P.train_apq(x.astype(np.float64), 50, 16, hp, ho, max_it=5, seed=0)
    assert np.array_equal(d, cb)
    assert np.array_equal(codes, want)
    assert hist == h.tolist()
