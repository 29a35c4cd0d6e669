"""CPU-side checks of the boundary: the C-ABI library loads and exports
every symbol include/anisoq_b200.h declares (no compute calls without a GPU),
and the host-side mirror behaves like the reference where no device is needed."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "anisoq_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const char\*|int|void\*|uint64_t|size_t)\s+(aq_\w+)\(",
                                 src, re.M)))


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_1908_10396_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) > 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_table_covers_header():
    from paper_1908_10396_b200 import _lib

    missing = [s for s in declared_symbols() if s not in _lib._SIGS and not s.startswith(
        ("aq_error_class", "aq_last_error", "aq_status_name"))]
    assert not missing, missing


def test_error_classes_match_reference():
    # error.hpp:43-55: QuadratureFailure and SingularSystem are runtime
    from paper_1908_10396_b200 import anisoq as aq

    assert aq.SingularSystem("x").error_class == "runtime"
    assert aq.QuadratureFailure("x").error_class == "runtime"
    for c in (aq.InvalidArgument, aq.ZeroNormDatapoint, aq.CodeOutOfRange, aq.EmptyIndex):
        assert c("x").error_class == "validation"


def test_host_weight_helpers():
    from paper_1908_10396_b200 import anisoq as aq

    w = aq.AnisotropicWeights.from_eta(4.125)
    assert (w.h_parallel, w.h_perpendicular) == (4.125, 1.0) and not w.is_isotropic()
    assert aq.AnisotropicWeights.isotropic(2.0).is_isotropic()
    with pytest.raises(aq.InvalidArgument):
        aq.AnisotropicWeights.from_h(-1, 1)
    assert abs(aq.eta_limit(0.2, 1.0, 32) - 31 * 0.04 / 0.96) < 1e-15
    with pytest.raises(aq.InvalidThreshold):
        aq.eta_limit(0.2, 0.1, 32)


def test_dataset_storage_type():
    """float32-exact values are stored as float32 (fast kernels); anything
    else (e.g. unit_normalize output) keeps float64 rows."""
    from paper_1908_10396_b200 import anisoq as aq

    a = aq.Dataset(np.ones((3, 4), np.float64))
    assert a.values.dtype == np.float32 and not a.f64
    b = aq.Dataset(np.full((3, 4), 0.1, np.float64))
    assert b.values.dtype == np.float64 and b.f64
    assert np.array_equal(b.values, np.full((3, 4), 0.1))


def test_workload_pack_roundtrip():
    from paper_1908_10396_b200 import workload as wl

    c = np.random.default_rng(0).integers(0, 16, (100, 50)).astype(np.uint32)
    assert np.array_equal(wl.unpack_codes(wl.pack_codes(c), 50), c)
