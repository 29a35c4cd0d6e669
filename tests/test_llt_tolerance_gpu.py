"""Device codebook update (assembly + pinned blocked Cholesky, one-launch
solves) against LAPACK on the same normal equations at the config-2 and
config-5 dimensions (1,600 and 4,096): the pinned solver is bit-exact with
the reference (test_update_gpu.py, test_config_pins_gpu.py) and within
rounding of an independent solver (pq.hpp:424-441)."""
import numpy as np
import pytest

from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows, threshold_hp_ho

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,M", [(20000, 100, 50), (12000, 256, 128)])
def test_device_update_agrees_with_lapack(n, d, M):
    k = 16
    x = mixture_rows(n, d, 11)
    codes = np.random.default_rng(12).integers(0, k, (n, M)).astype(np.uint32)
    cm = aq.CodeMatrix(n, M, k, codes)
    w = threshold_hp_ho(x, 0.2)
    A, r = aq.assemble_selector_system(x, cm, w, M, k)
    dim = k * d
    A = A + np.eye(dim) * (1e-6 * np.trace(A) / dim)
    want = np.linalg.solve(A, r)
    got = aq.pq_codebook_update(x, cm, w, M, k).dictionaries
    rel = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert rel <= 1e-8, rel
