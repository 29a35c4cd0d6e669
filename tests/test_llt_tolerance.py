"""The pinned blocked Cholesky (oracle/eigen_subset, the stand-in the
reference is compiled against) is an ordinary Cholesky solve: against
LAPACK (numpy.linalg.solve) on well-conditioned systems its solutions agree
to a few float64 ulps, and the reference's pq_codebook_update (compiled with
the stand-in, oracle/_ref) agrees with a LAPACK solve of the same assembled,
ridged normal equations (pq.hpp:424-441). So the bit-exact device pins are
pinned to a correct solver, and swapping in Eigen's own LLT moves a codebook
by rounding only."""
import numpy as np
import pytest

from oracle import Port, Reference
from tests.helpers import mixture_rows, threshold_hp_ho


@pytest.mark.parametrize("dim", [1, 63, 64, 65, 200, 700])
def test_pinned_llt_agrees_with_lapack(dim):
    g = np.random.default_rng(dim)
    X = g.standard_normal((dim + 40, dim))
    A = X.T @ X / dim + 0.5 * np.eye(dim)
    b = g.standard_normal(dim)
    got = Port().llt_solve(A, b)
    want = np.linalg.solve(A, b)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))


def test_reference_codebook_update_agrees_with_lapack():
    n, d, M, k = 3000, 16, 8, 16
    x = mixture_rows(n, d, 5).astype(np.float64)
    codes = np.random.default_rng(6).integers(0, k, (n, M)).astype(np.uint32)
    hp, ho = threshold_hp_ho(x, 0.2)
    P = Port()
    A, r = P.assemble_selector_system(x, codes, hp, ho, M, k)
    dim = k * d
    A = A + np.eye(dim) * (1e-6 * np.trace(A) / dim)  # pq.hpp:431-435 ridge
    want = np.linalg.solve(A, r)
    got = Reference().pq_codebook_update(x, codes, hp, ho, M, k)
    rel = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert rel <= 1e-9, rel
