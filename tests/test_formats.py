"""On-disk formats (pq.hpp:614-730, dataset.hpp:122-219): golden bytes from the
reference tests and round trips; host-only (no GPU needed)."""
import numpy as np
import pytest

from paper_1908_10396_b200 import anisoq as aq


def test_codes_golden_bytes(tmp_path):
    # test_pq.cpp:560-571
    p = tmp_path / "codes_small.bin"
    aq.save_codes(aq.CodeMatrix(1, 2, 4, np.array([[3, 1]])), str(p))
    assert list(p.read_bytes()) == [1, 0, 0, 0, 2, 0, 0, 0, 4, 0, 0, 0, 3, 1]


def test_codebook_and_codes_round_trip(tmp_path):
    g = np.random.default_rng(404)
    cb = aq.ProductCodebook(2, 3, 4, g.standard_normal(24))
    p1, p2 = tmp_path / "a.bin", tmp_path / "b.bin"
    aq.save_codebook(cb, str(p1))
    loaded = aq.load_codebook(str(p1))
    assert (loaded.M, loaded.k, loaded.sub_dimension) == (2, 3, 4)
    assert np.array_equal(loaded.dictionaries, cb.dictionaries.astype(np.float32).astype(np.float64))
    aq.save_codebook(loaded, str(p2))
    assert p1.read_bytes() == p2.read_bytes()
    cm = aq.CodeMatrix(10, 3, 300, g.integers(0, 300, (10, 3)))
    aq.save_codes(cm, str(tmp_path / "c.bin"))
    cm2 = aq.load_codes(str(tmp_path / "c.bin"))
    assert (cm2.n, cm2.M, cm2.k) == (10, 3, 300) and np.array_equal(cm2.codes, cm.codes)


def test_malformed_files(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"NOPE")
    with pytest.raises(aq.MalformedFile):
        aq.load_codebook(str(bad))
    c = tmp_path / "badcodes.bin"
    c.write_bytes(np.array([1, 1, 2], "<u4").tobytes() + bytes([7]))
    with pytest.raises(aq.CodeOutOfRange):
        aq.load_codes(str(c))


def test_fvecs_ivecs_round_trip(tmp_path):
    x = np.random.default_rng(1).standard_normal((7, 5)).astype(np.float32)
    aq.write_fvecs(aq.Dataset(x), str(tmp_path / "x.fvecs"))
    assert np.array_equal(aq.read_fvecs(str(tmp_path / "x.fvecs")).values, x)
    rows = [np.arange(3), np.arange(10, 12)]
    aq.write_ivecs(rows, str(tmp_path / "g.ivecs"))
    back = aq.read_ivecs(str(tmp_path / "g.ivecs"))
    assert all(np.array_equal(a, b) for a, b in zip(rows, back))
    (tmp_path / "t.fvecs").write_bytes(np.array([5], "<i4").tobytes() + b"\0" * 7)
    with pytest.raises(aq.MalformedFile):
        aq.read_fvecs(str(tmp_path / "t.fvecs"))


def test_python_generator_and_rng_match_reference():
    from oracle import Port, Reference
    from paper_1908_10396_b200 import anisoq as aq

    assert Reference.available(), "oracle/_ref/libanisoq_ref.so missing (make -C oracle)"
    R = Reference()
    mix = aq.generate_synthetic("gaussian_mixture", 60, 6, 7, centers=5, spread=0.25,
                                normalize=True)
    assert np.array_equal(mix.values.astype(np.float64),
                          R.generate_synthetic(1, 60, 6, 7, centers=5, spread=0.25,
                                               normalize=True))
    sph = aq.generate_synthetic("uniform_sphere", 20, 4, 3)
    assert np.array_equal(sph.values.astype(np.float64), R.generate_synthetic(0, 20, 4, 3))
    assert aq.Rng(9).sample_distinct(100, 7) == Port().sample_distinct(9, 100, 7).tolist()
    u = aq.unit_normalize(mix)
    assert np.allclose(np.linalg.norm(u, axis=1), 1.0, rtol=0, atol=1e-15)
