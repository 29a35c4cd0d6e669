"""Generates tests/golden/golden_v1.npz from the reference itself (oracle/_ref).

Run in the build container (needs /root/reference): `python tests/golden/make_golden.py`.
Inputs are seeded config-1-shaped data; every output array is produced by the
unmodified reference headers compiled in place.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import Port, Reference  # noqa: E402
from paper_1908_10396_b200 import workload as wl  # noqa: E402


def main():
    R = Reference()
    w = wl.config1(n=2000, nq=8, seed=11)
    x = w.base.astype(np.float64)
    norms = R.row_norms(x)
    hp = np.array([R.eta_limit(0.2, v, 32) for v in norms])
    ho = np.ones_like(hp)
    cb = np.random.Generator(np.random.PCG64([11, 3])).standard_normal(16 * 16 * 2) * 0.25
    codes0 = np.random.Generator(np.random.PCG64([11, 4])).integers(0, 16, (2000, 16)).astype(np.uint32)
    out = dict(x=w.base, q=w.queries, hp=hp, ho=ho, cb=cb, codes0=codes0)
    out["quantize3"] = R.pq_quantize(x, cb, 16, 16, 2, hp, ho, 3, threads=4)
    out["assign_codes"], out["assign_losses"] = R.pq_assign_pass(x, cb, 16, 16, 2, hp, ho, codes0)
    out["update"] = R.pq_codebook_update(x, codes0, hp, ho, 16, 16)
    out["adc_ids"], out["adc_scores"] = R.adc_search_batch(
        w.queries.astype(np.float64), codes0, 16, cb, 16, 16, 2, 100, threads=4)
    out["train_cb"], out["train_codes"], out["train_hist"] = R.train_apq(
        x[:800], 16, 16, hp[:800], ho[:800], max_it=3, tol=0.0, seed=0)
    out["avq_cw"], out["avq_assign"], out["avq_hist"] = R.train_avq(
        x[:1000], 24, hp[:1000], ho[:1000], max_it=4, tol=0.0, seed=5)
    # sanity: the port agrees
    assert np.array_equal(Port().pq_quantize(x, cb, 16, 16, 2, hp, ho, 3), out["quantize3"])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")
    np.savez_compressed(path, **out)
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
