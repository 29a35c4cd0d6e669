"""GPU parity for both sd = 2 assembly kernels (the staged k_assemble_sd2 and
the register-ring k_assemble_sd2r). The default picks one by launch size, so
each is forced here through AQ_ASM_VARIANT in a child process (the variable
is read once per process), including a shape with several point blocks
(resumed accumulators) with a partial column chunk (d = 100, M = 50)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import numpy as np
from oracle import Port
from paper_1908_10396_b200 import anisoq as aq
from tests.helpers import mixture_rows, threshold_hp_ho
P = Port()
# (130000, 100, 50): two point blocks of 125,829 rows (48 MB of float32)
# (9000, 32, 16) with codes in {0, 1} (every other subspace constant): runs of
# one slot, where a pair of points shares its accumulator slot
for n, d, M, kk in ((6000, 32, 16, 16), (130000, 100, 50, 16), (9000, 32, 16, 2)):
    x = mixture_rows(n, d, 61)
    codes = np.random.default_rng(62).integers(0, kk, (n, M)).astype(np.uint32)
    if kk == 2:
        codes[:, ::2] = 7
    hp, ho = threshold_hp_ho(x, 0.2)
    A, r = aq.assemble_selector_system(x, aq.CodeMatrix(n, M, 16, codes), (hp, ho), M, 16)
    A2, r2 = P.assemble_selector_system(x.astype(np.float64), codes, hp, ho, M, 16)
    assert np.array_equal(A, A2), (n, d, M)
    assert np.array_equal(r, r2), (n, d, M)
print("ok")
"""


@pytest.mark.parametrize("variant", ["1", "3"])
def test_assembly_variant_matches_oracle(variant):
    env = dict(os.environ, AQ_ASM_VARIANT=variant, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
