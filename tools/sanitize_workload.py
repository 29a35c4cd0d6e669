"""Small end-to-end workload for compute-sanitizer (run by hand where the tool is
open: it is closed on this GPU pool, so no test drives it).

Runs every kernel family of the library once at a small shape, with the
variant switches the parity tests pin, so that `compute-sanitizer --tool
memcheck` / `--tool racecheck` / `--tool synccheck` see each kernel:

  encode      k_encode_sd2w (M = 16, 50), k_encode_sd2 (M = 7), k_encode_generic (sd = 3)
  training    bucket lists, k_assemble_sd2 / k_assemble_sd2r / k_assemble, k_trace_ridge,
              k_llt_panel / k_llt_trail / k_llt_flow, k_slot_sums, sort, k-means warm start
  VQ          k_vq_coef / k_vq_systems (train_avq)
  search      k_build_lut, k_adc_score or k_adc_tc (AQ_ADC_TC), k_adc_merge, k_rerank
  exact       k_exact_tc / k_exact_filter / k_exact_fmerge

Usage: python tools/sanitize_workload.py [part ...]   (default: all parts).
The results are checked by the parity tests, not here; this script only has
to drive the kernels (small sizes keep the sanitizers' replay affordable).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1908_10396_b200 import anisoq as aq  # noqa: E402
from paper_1908_10396_b200 import workload as wl  # noqa: E402


def part_encode(s):
    g = np.random.default_rng(1)
    for n, d, M in ((700, 32, 16), (301, 100, 50), (129, 14, 7), (97, 24, 8)):
        sd = d // M
        x = wl._normalize_rows(g.standard_normal((n, d))).astype(np.float32)
        x[::7] *= 1.7
        cb = aq.ProductCodebook(M, 16, sd, g.standard_normal(M * 16 * sd) * 0.3)
        aq.pq_quantize(x, cb, aq.ThresholdWeights(0.2), 3, session=s)


def part_train(s):
    g = np.random.default_rng(2)
    x = wl._normalize_rows(g.standard_normal((1500, 32))).astype(np.float32)
    ds = s.upload_dataset(x)
    cfg = aq.TrainConfig(max_iterations=2, seed=3)
    aq.dev_train_apq(ds, 16, 16, aq.ThresholdWeights(0.2), cfg)
    aq.dev_train_l2_pq(ds, 8, 16, cfg)
    aq.dev_train_avq(ds, 12, aq.ThresholdWeights(0.2), cfg)
    # generic assembly (sd = 4, k = 8) and the one-launch solves at dim > 64
    x2 = wl._normalize_rows(g.standard_normal((600, 16))).astype(np.float32)
    ds2 = s.upload_dataset(x2)
    aq.dev_train_apq(ds2, 4, 8, aq.ThresholdWeights(0.2), cfg)


def part_search(s):
    g = np.random.default_rng(4)
    n, M = 3000, 16
    x = wl._normalize_rows(g.standard_normal((n, 2 * M))).astype(np.float32)
    cb = aq.ProductCodebook(M, 16, 2, g.standard_normal(M * 32) * 0.3)
    codes = aq.CodeMatrix(n, M, 16, g.integers(0, 16, (n, M)).astype(np.uint32))
    ds, dc, dcb = s.upload_dataset(x), s.upload_codes(codes), s.upload_codebook(cb)
    Q = wl._normalize_rows(g.standard_normal((33, 2 * M)))
    aq.dev_search_rerank(ds, dc, dcb, Q, 100, 10)
    aq.dev_exact_search(ds, Q, 10)


PARTS = {"encode": part_encode, "train": part_train, "search": part_search}

if __name__ == "__main__":
    names = sys.argv[1:] or list(PARTS)
    s = aq.Session(0)
    for nm in names:
        PARTS[nm](s)
        s.sync()
    print("sanitize workload done:", " ".join(names), f"launches={s.launches}")
