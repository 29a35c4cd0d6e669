"""GPU parity: anisotropic encode (pq_quantize, pq.hpp:581-612) and the
training assignment pass (pq.hpp:202-221) through the C ABI, against the
oracle on the same seeded inputs. Codes and losses must be bit-identical."""
import numpy as np
import pytest

from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import lognormal_rows, mixture_rows, random_codebook, threshold_hp_ho

pytestmark = pytest.mark.gpu
P = Port()


def _cb(M, k, sd, seed, scale=0.25):
    return aq.ProductCodebook(M, k, sd, random_codebook(M, k, sd, seed, scale))


@pytest.mark.parametrize("passes", [0, 1, 3])
def test_quantize_config1_shape(passes):
    x = mixture_rows(20000, 32, 21, centers=64)
    cb = _cb(16, 16, 2, 22)
    got = aq.pq_quantize(x, cb, aq.ThresholdWeights(0.2), passes).codes
    hp, ho = threshold_hp_ho(x, 0.2)
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, 16, 16, 2, hp, ho, passes)
    assert np.array_equal(got, want)


def test_quantize_config3_shape_lognormal_norms():
    # norms below T take the documented eta = inf policy (h_par 1, h_perp 0)
    x = lognormal_rows(60000, 128, 23)
    cb = _cb(64, 16, 2, 24, scale=1 / np.sqrt(128))
    got = aq.pq_quantize(x, cb, aq.ThresholdWeights(0.2, "parallel_only"), 3).codes
    hp, ho = threshold_hp_ho(x, 0.2, policy=1)
    assert (ho == 0).sum() > 0  # the policy path is exercised
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, 64, 16, 2, hp, ho, 3)
    assert np.array_equal(got, want)


# fast-path shapes of the other configs: M = 50 (config 2, a tail code word),
# M = 128 (config 5), the other M-specialised instances (32, 48, 96), an odd M
# (runtime-M kernel)
@pytest.mark.parametrize("n,d,M", [(6000, 100, 50), (3000, 256, 128), (5000, 26, 13),
                                   (4001, 64, 32), (3999, 96, 48), (2500, 192, 96)])
def test_quantize_config_shapes(n, d, M):
    x = mixture_rows(n, d, M, centers=32)
    cb = _cb(M, 16, 2, M + 1, scale=1 / np.sqrt(d))
    got = aq.pq_quantize(x, cb, aq.ThresholdWeights(0.2), 3).codes
    hp, ho = threshold_hp_ho(x, 0.2)
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, M, 16, 2, hp, ho, 3)
    assert np.array_equal(got, want)
    codes, losses = aq.pq_assign_pass(x, cb, aq.ThresholdWeights(0.2), aq.CodeMatrix(n, M, 16, want))
    wc, wl_ = P.pq_assign_pass(x.astype(np.float64), cb.dictionaries, M, 16, 2, hp, ho, want)
    assert np.array_equal(codes.codes, wc) and np.array_equal(losses, wl_)


@pytest.mark.parametrize("w", ["iso", "eta", "iso2", "per_point", "eta_small"])
def test_quantize_weight_kinds(w):
    x = mixture_rows(8000, 32, 25)
    n = len(x)
    cb = _cb(16, 16, 2, 26)
    if w == "iso":
        wt, hp, ho = aq.AnisotropicWeights.isotropic(), np.ones(n), np.ones(n)
    elif w == "iso2":
        wt, hp, ho = aq.AnisotropicWeights.isotropic(2.0), np.full(n, 2.0), np.full(n, 2.0)
    elif w == "eta":
        wt, hp, ho = aq.AnisotropicWeights.from_eta(4.125), np.full(n, 4.125), np.ones(n)
    elif w == "eta_small":  # h_par < h_perp: negative coupling coefficient
        wt, hp, ho = aq.AnisotropicWeights.from_eta(0.3), np.full(n, 0.3), np.ones(n)
    else:
        g = np.random.default_rng(5)
        hp = g.uniform(0.5, 12.0, n)
        ho = g.uniform(0.2, 2.0, n)
        wt = (hp, ho)
    got = aq.pq_quantize(x, cb, wt, 3).codes
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, 16, 16, 2, hp, ho, 3)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("k", [1, 2, 5, 16])
def test_quantize_small_k(k):
    x = mixture_rows(4000, 16, 27)
    cb = _cb(8, k, 2, 28)
    got = aq.pq_quantize(x, cb, aq.AnisotropicWeights.from_eta(4.125), 3).codes
    n = len(x)
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, 8, k, 2, np.full(n, 4.125),
                         np.ones(n), 3)
    assert np.array_equal(got, want)


def test_quantize_exact_ties_duplicate_codewords():
    # duplicated codewords tie exactly in float64: the lowest index must win
    x = mixture_rows(4000, 16, 29)
    d = random_codebook(8, 16, 2, 30).reshape(8, 16, 2)
    d[:, 9] = d[:, 3]
    d[:, 15] = d[:, 0]
    cb = aq.ProductCodebook(8, 16, 2, d.ravel())
    n = len(x)
    for wt, hp, ho in [(aq.AnisotropicWeights.from_eta(4.125), np.full(n, 4.125), np.ones(n)),
                       (aq.AnisotropicWeights.isotropic(), np.ones(n), np.ones(n))]:
        got = aq.pq_quantize(x, cb, wt, 3).codes
        want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, 8, 16, 2, hp, ho, 3)
        assert np.array_equal(got, want)
        assert not np.isin(got, [9, 15]).any()


@pytest.mark.parametrize("shape", [(24, 8, 8, 3), (5, 1, 6, 5), (32, 8, 20, 4), (12, 12, 4, 1)])
def test_quantize_generic_path(shape):
    d, M, k, sd = shape
    x = mixture_rows(3000, d, 31)
    cb = _cb(M, k, sd, 32)
    n = len(x)
    got = aq.pq_quantize(x, cb, aq.AnisotropicWeights.from_eta(4.125), 2).codes
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, M, k, sd, np.full(n, 4.125),
                         np.ones(n), 2)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("fixed", [False, True])
@pytest.mark.parametrize("sd", [2, 3])
def test_assign_pass(fixed, sd):
    M = 16 if sd == 2 else 8
    x = mixture_rows(10000, M * sd, 33)
    cb = _cb(M, 16, sd, 34)
    codes0 = np.random.default_rng(6).integers(0, 16, (len(x), M)).astype(np.uint32)
    hp, ho = threshold_hp_ho(x, 0.2)
    got_c, got_l = aq.pq_assign_pass(x, cb, aq.ThresholdWeights(0.2),
                                     aq.CodeMatrix(len(x), M, 16, codes0), fixed)
    want_c, want_l = P.pq_assign_pass(x.astype(np.float64), cb.dictionaries, M, 16, sd, hp, ho,
                                      codes0, fixed)
    assert np.array_equal(got_c.codes, want_c)
    assert np.array_equal(got_l, want_l)


def test_zero_norm_datapoint():
    x = mixture_rows(100, 8, 35)
    x[37] = 0
    cb = _cb(4, 16, 2, 36)
    w = aq.AnisotropicWeights.from_eta(2.0)
    with pytest.raises(aq.ZeroNormDatapoint):
        aq.pq_quantize(x, cb, w, 1)
    aq.pq_quantize(x, cb, w, 0)  # passes = 0 never needs 1/|x|^2 (pq.hpp:596)
    aq.pq_quantize(x, cb, aq.AnisotropicWeights.isotropic(), 2)


def test_validation_errors():
    x = mixture_rows(50, 8, 37)
    with pytest.raises(aq.DimensionMismatch):
        aq.pq_quantize(x, _cb(3, 4, 2, 1), aq.AnisotropicWeights(), 1)
    with pytest.raises(aq.InvalidArgument):
        aq.pq_quantize(x, _cb(4, 4, 2, 1), aq.AnisotropicWeights(), -1)
    with pytest.raises(aq.InvalidThreshold):
        aq.pq_quantize(x * 0.01, _cb(4, 4, 2, 1), aq.ThresholdWeights(0.2), 1)


def test_empty_dataset_quantize():
    x = np.zeros((0, 8), np.float32)
    out = aq.pq_quantize(x, _cb(4, 4, 2, 1), aq.AnisotropicWeights(), 2)
    assert out.codes.shape == (0, 4)


@pytest.mark.parametrize("chunk", ["1000", "4096"])
def test_quantize_streamed_host_path(monkeypatch, chunk):
    # aq_pq_quantize streams large host datasets in chunks (copies overlapped
    # with the device work); AQ_STREAM_CHUNK shrinks the chunk so every row is
    # checked: codes equal the oracle's, across chunk edges and a ragged tail
    monkeypatch.setenv("AQ_STREAM_CHUNK", chunk)
    x = mixture_rows(17003, 32, 91, centers=20)
    cb = _cb(16, 16, 2, 92, scale=0.25)
    got = aq.pq_quantize(x, cb, aq.ThresholdWeights(0.2), 3).codes
    hp, ho = threshold_hp_ho(x, 0.2)
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, 16, 16, 2, hp, ho, 3)
    assert np.array_equal(got, want)
    # a failing point deep in a later chunk reports its global index
    bad = x.copy()
    bad[12345] = 0.0
    with pytest.raises(aq.InvalidArgument, match="point 12345"):
        aq.pq_quantize(bad, cb, aq.ThresholdWeights(0.2), 3)


@pytest.mark.parametrize("weights,passes", [("iso", 0), ("eta", 2)])
def test_quantize_streamed_uniform_weights(monkeypatch, weights, passes):
    # the streamed host path with uniform weights (isotropic / explicit eta)
    monkeypatch.setenv("AQ_STREAM_CHUNK", "2500")
    x = mixture_rows(12345, 16, 93, centers=12, normalize=False)
    cb = _cb(8, 16, 2, 94, scale=0.3)
    w = aq.AnisotropicWeights.isotropic() if weights == "iso" else aq.AnisotropicWeights.from_eta(3.5)
    got = aq.pq_quantize(x, cb, w, passes).codes
    hp = np.full(len(x), w.h_parallel)
    ho = np.full(len(x), w.h_perpendicular)
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, 8, 16, 2, hp, ho, passes)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("pin_in,pin_out", [(True, True), (True, False), (False, True)])
def test_quantize_streamed_page_locked(monkeypatch, pin_in, pin_out):
    # page-locked caller buffers: rows go H2D straight from the caller's memory
    # and the codes are widened on the device and copied straight into the
    # caller's output; codes and error reporting equal the staged path's
    import ctypes as C

    import torch

    monkeypatch.setenv("AQ_STREAM_CHUNK", "3000")
    n, d, M = 20011, 32, 16
    x = mixture_rows(n, d, 95, centers=20)
    cb = _cb(M, 16, 2, 96, scale=0.25)
    xt = torch.from_numpy(x).pin_memory() if pin_in else torch.from_numpy(x.copy())
    ot = torch.zeros((n, M), dtype=torch.int32)
    if pin_out:
        ot = ot.pin_memory()
    keep: list = []
    w = aq._weights(aq.ThresholdWeights(0.2), n, keep)
    s = aq.Session.default()

    def call(rows):
        return aq._L.aq_pq_quantize(s.h, rows.data_ptr(), n, d, cb.dictionaries.ctypes.data,
                                    M, 16, 2, C.byref(w), 3, ot.data_ptr())

    aq._check(call(xt))
    hp, ho = threshold_hp_ho(x, 0.2)
    want = P.pq_quantize(x.astype(np.float64), cb.dictionaries, M, 16, 2, hp, ho, 3)
    assert np.array_equal(ot.numpy().view(np.uint32), want)
    xt[17777] = 0.0
    with pytest.raises(aq.InvalidArgument, match="point 17777"):
        aq._check(call(xt))
