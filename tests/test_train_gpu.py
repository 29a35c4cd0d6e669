"""GPU parity: trainers (train_l2_pq pq.hpp:469-501, train_apq pq.hpp:513-575)
against the oracle on seeded inputs: codebooks, codes and the loss history
are bit-identical (every step mirrors the reference's operation order)."""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200 import workload as wl
from tests.helpers import mixture_rows, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()


@pytest.mark.parametrize("tol", [0.0, 1e-6])
def test_train_l2_pq(tol):
    x = mixture_rows(4000, 16, 61, centers=8, sigma=0.4, normalize=False)
    cfg = aq.TrainConfig(max_iterations=12, relative_tolerance=tol, seed=40)
    cb, codes = aq.train_l2_pq(x, 8, 6, cfg)
    want_cb, want_codes = P.train_l2_pq(x.astype(np.float64), 8, 6, 12, tol, 40)
    assert np.array_equal(cb.dictionaries, want_cb)
    assert np.array_equal(codes.codes, want_codes)


def test_train_l2_pq_empty_partitions_reseed():
    # few distinct subvectors: k-means hits empty partitions (vq.hpp:284-292)
    g = np.random.default_rng(3)
    proto = g.standard_normal((3, 8))
    x = proto[g.integers(0, 3, 500)].astype(np.float32)
    cfg = aq.TrainConfig(max_iterations=5, relative_tolerance=0.0, seed=2)
    cb, codes = aq.train_l2_pq(x, 4, 5, cfg)
    want_cb, want_codes = P.train_l2_pq(x.astype(np.float64), 4, 5, 5, 0.0, 2)
    assert np.array_equal(cb.dictionaries, want_cb)
    assert np.array_equal(codes.codes, want_codes)


@pytest.mark.parametrize("warm", [True, False])
def test_train_apq_config1_shape(warm):
    w = wl.config1(n=20000, nq=1, seed=5)
    hp, ho = threshold_hp_ho(w.base, 0.2)
    cfg = aq.TrainConfig(max_iterations=4, relative_tolerance=0.0, seed=0)
    hist = []
    cb, codes = aq.train_apq(w.base, 16, 16, aq.ThresholdWeights(0.2), cfg, warm, hist)
    want_cb, want_codes, want_hist = P.train_apq(w.base.astype(np.float64), 16, 16, hp, ho,
                                                 max_it=4, tol=0.0, seed=0, warm_start=warm)
    assert np.array_equal(np.array(hist), want_hist)
    assert np.array_equal(codes.codes, want_codes)
    assert np.array_equal(cb.dictionaries, want_cb)
    assert all(b <= a + 1e-9 for a, b in zip(hist, hist[1:]))  # monotone (check 6)


def test_train_apq_isotropic_cold_start_is_classical_pq():
    # test_pq.cpp:403-428: eta = 1 cold start reproduces classical PQ bitwise
    x = mixture_rows(3500, 8, 62, centers=10, sigma=0.35, normalize=False)
    for iters in (1, 3, 8):
        cfg = aq.TrainConfig(max_iterations=iters, relative_tolerance=0.0, seed=88)
        cb, codes = aq.train_apq(x, 2, 5, aq.AnisotropicWeights.isotropic(), cfg, False)
        ones = np.ones(len(x))
        want_cb, want_codes, _ = P.train_apq(x.astype(np.float64), 2, 5, ones, ones, max_it=iters,
                                             tol=0.0, seed=88, warm_start=False)
        assert np.array_equal(cb.dictionaries, want_cb)
        assert np.array_equal(codes.codes, want_codes)


def test_train_apq_default_tolerance_and_sd3():
    x = mixture_rows(3000, 24, 63)
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=6, seed=7)  # default relative_tolerance 1e-6
    hist = []
    cb, codes = aq.train_apq(x, 8, 8, aq.ThresholdWeights(0.2), cfg, True, hist)
    want_cb, want_codes, want_hist = P.train_apq(x.astype(np.float64), 8, 8, hp, ho, max_it=6,
                                                 tol=1e-6, seed=7, warm_start=True)
    assert np.array_equal(np.array(hist), want_hist)
    assert np.array_equal(codes.codes, want_codes)
    assert np.array_equal(cb.dictionaries, want_cb)


def test_train_validation():
    x = mixture_rows(10, 6, 64)
    with pytest.raises(aq.DimensionNotDivisible):
        aq.train_apq(x, 4, 2, aq.AnisotropicWeights(), aq.TrainConfig())
    with pytest.raises(aq.EmptyDataset):
        aq.train_apq(np.zeros((0, 6), np.float32), 2, 2, aq.AnisotropicWeights(), aq.TrainConfig())
    with pytest.raises(aq.InvalidArgument):
        aq.train_apq(x, 2, 11, aq.AnisotropicWeights(), aq.TrainConfig())


def test_k64_byte_codes_end_to_end():
    """k = 64 (8-bit codes): every stage on its non-specialised path —
    generic encoder, generic normal-equation assembly, k-means, ADC exact
    fallback — bit-identical to the oracle."""
    x = mixture_rows(3000, 16, 71, centers=24)
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=3, relative_tolerance=0.0, seed=5)
    cb, codes = aq.train_apq(x, 8, 64, aq.ThresholdWeights(0.2, "parallel_only"), cfg)
    want_cb, want_codes, _ = P.train_apq(x.astype(np.float64), 8, 64, hp, ho, max_it=3, tol=0.0,
                                         seed=5)
    assert np.array_equal(cb.dictionaries, want_cb)
    assert np.array_equal(codes.codes, want_codes)
    q = np.random.default_rng(2).standard_normal((5, 16))
    s = aq.Session.default()
    ids, sc = aq.dev_adc_search(s.upload_codes(codes), s.upload_codebook(cb), q, 20)
    wi, ws = P.adc_search_batch(q, want_codes, 64, want_cb, 8, 64, 2, 20)
    assert np.array_equal(ids, wi) and np.array_equal(sc, ws)


def test_train_long_rows_take_the_chunked_loss_sums():
    # n >= 65536: k-means totals (tol > 0) and the train_apq loss history run
    # through the chunk-parallel sums (train.cu seq_sums_on); still bit-exact
    x = mixture_rows(90000, 16, 67, centers=32, sigma=0.3)
    hp, ho = threshold_hp_ho(x, 0.2)
    cfg = aq.TrainConfig(max_iterations=3, relative_tolerance=1e-7, seed=4)
    hist = []
    cb, codes = aq.train_apq(x, 8, 16, aq.ThresholdWeights(0.2), cfg, True, hist)
    want_cb, want_codes, want_hist = P.train_apq(x.astype(np.float64), 8, 16, hp, ho, max_it=3,
                                                 tol=1e-7, seed=4, warm_start=True)
    assert np.array_equal(np.array(hist), want_hist)
    assert np.array_equal(codes.codes, want_codes)
    assert np.array_equal(cb.dictionaries, want_cb)
