"""GPU parity: exact MIPS ground truth (index.hpp:137-162), the single-point
API (pq.hpp:256-282) and evaluate()'s recall bookkeeping (index.hpp:213-332)."""
import numpy as np
import pytest

from oracle import Port, Reference
from paper_1908_10396_b200 import anisoq as aq
from paper_1908_10396_b200 import workload as wl
from tests.helpers import mixture_rows, random_codebook

pytestmark = pytest.mark.gpu
P = Port()


@pytest.mark.parametrize("n,d,depth,nq", [(20000, 32, 10, 100), (5000, 100, 100, 17),
                                          (300, 8, 1000, 3), (70000, 96, 64, 40),
                                          (30000, 64, 1000, 20), (40000, 32, 4096, 5),
                                          (20000, 16, 5000, 3),
                                          # tensor-core filter shapes: d not a multiple
                                          # of 16, the largest K tile, one query past a
                                          # 128-query block, and d > 128 (float32 filter)
                                          (50000, 30, 10, 129), (60000, 128, 10, 300),
                                          (9000, 130, 10, 40)])
def test_exact_search_matches_oracle(n, d, depth, nq):
    x = mixture_rows(n, d, 71)
    q = mixture_rows(nq, d, 72).astype(np.float64)
    s = aq.Session.default()
    ids, sc = aq.dev_exact_search(s.upload_dataset(x), q, depth)
    wi, ws = P.exact_search_batch(q, x.astype(np.float64), depth)
    assert np.array_equal(ids, wi) and np.array_equal(sc, ws)


def test_exact_search_reference_invariances():
    # test_index.cpp:156-186
    x = mixture_rows(100, 8, 73)
    q = np.random.default_rng(12).standard_normal(8)
    res = aq.exact_search(q, x, 10)
    assert len(res.hits) == 10
    res2 = aq.exact_search(q * 3.7, x, 10)
    assert [h.index for h in res2.hits] == [h.index for h in res.hits]
    top1 = aq.exact_search(x[17].astype(np.float64), aq.Dataset(x), 1).hits[0]
    wi, ws = P.exact_search_batch(x[17:18].astype(np.float64), x.astype(np.float64), 1)
    assert (top1.index, top1.score) == (int(wi[0, 0]), float(ws[0, 0]))
    assert len(aq.exact_search(q, x[3:4], 4).hits) == 1
    with pytest.raises(aq.EmptyDataset):
        aq.exact_search(q, np.zeros((0, 8), np.float32), 1)


def test_exact_search_ties():
    x = np.ones((500, 4), np.float32)
    ids, _ = aq.dev_exact_search(aq.Session.default().upload_dataset(x), np.ones((1, 4)), 50)
    assert ids[0].tolist() == list(range(50))


def _ref():
    # built here, travels with the repository: missing is a failure, not a skip
    assert Reference.available(), "oracle/_ref/libanisoq_ref.so missing (make -C oracle)"
    return Reference()


@pytest.mark.parametrize("eta", [4.125, 1.0, 0.5])
def test_assign_point_matches_reference(eta):
    # test_pq.cpp:79-162 style: random float64 points (not float32-exact)
    g = np.random.default_rng(int(eta * 10))
    w = aq.AnisotropicWeights.from_eta(eta)
    for rep in range(20):
        cb = aq.ProductCodebook(3, 4, 2, g.standard_normal(24))
        x = g.standard_normal(6)
        cur = g.integers(0, 4, 3).astype(np.uint32)
        got = aq.pq_assign_point(x, cur, cb, w)
        want = _ref().pq_assign_point(x, cur, cb.dictionaries, 3, 4, 2, w.h_parallel,
                                      w.h_perpendicular)
        assert np.array_equal(got, want)
    with pytest.raises(aq.CodeOutOfRange):
        aq.pq_assign_point(np.ones(6), [0, 0, 9], cb, w)
    with pytest.raises(aq.ZeroNormDatapoint):
        aq.pq_assign_point(np.zeros(6), [0, 0, 0], cb, aq.AnisotropicWeights.from_eta(2.0))


def test_assign_point_sweep_order_matches_reference():
    # pq.hpp:256-282 with explicit sweep orders: permutations and repeats
    g = np.random.default_rng(77)
    w = aq.AnisotropicWeights.from_eta(4.125)
    R = _ref()
    for order in ([2, 0, 1], [1, 1, 0, 2, 2], [0], [2, 1, 0, 0, 1, 2]):
        for rep in range(10):
            cb = aq.ProductCodebook(3, 4, 2, g.standard_normal(24))
            x = g.standard_normal(6)
            cur = g.integers(0, 4, 3).astype(np.uint32)
            got = aq.pq_assign_point(x, cur, cb, w, sweep_order=order)
            want = R.pq_assign_point_order(x, cur, cb.dictionaries, 3, 4, 2, w.h_parallel,
                                           w.h_perpendicular, order)
            assert np.array_equal(got, want)
    assert np.array_equal(aq.pq_assign_point(x, cur, cb, w, sweep_order=list(range(3))),
                          aq.pq_assign_point(x, cur, cb, w))
    with pytest.raises(aq.InvalidArgument):
        aq.pq_assign_point(x, cur, cb, w, sweep_order=[0, 3])


def test_evaluate_perfect_codes_recall_one():
    # test_index.cpp:189-204: data equal to reconstructions -> recall 1, error 0
    g = np.random.default_rng(13)
    cb = aq.ProductCodebook(2, 4, 3, np.round(g.standard_normal(24) * 64) / 64)
    codes = g.integers(0, 4, (16, 2)).astype(np.uint32)
    data = np.stack([np.concatenate([cb.codeword(m, c) for m, c in enumerate(r)]) for r in codes])
    q = wl._normalize_rows(g.standard_normal((20, 6)))
    rep = aq.evaluate(q, data.astype(np.float32), aq.CodeMatrix(16, 2, 4, codes), cb,
                      aq.EvalOptions(recall_ns=(1, 5, 16), kk=5))
    assert rep.recall_1_at_n[1] == 1.0 and rep.recall_1_at_n[16] == 1.0
    assert rep.recall_k_at_k == 1.0 and rep.relative_error_max <= 1e-12
    # per-query timing (extension): identical bookkeeping, measured latencies,
    # and the reference's text report layout (index.hpp:183-197)
    prep = aq.evaluate(q, data.astype(np.float32), aq.CodeMatrix(16, 2, 4, codes), cb,
                       aq.EvalOptions(recall_ns=(1, 5, 16), kk=5, per_query_latency=True))
    assert prep.recall_1_at_n == rep.recall_1_at_n and prep.recall_k_at_k == rep.recall_k_at_k
    assert 0.0 < prep.latency.p50_us <= prep.latency.p99_us
    lines = prep.write_text().splitlines()
    assert lines[:5] == ["num_queries 20", "num_datapoints 16", "recall_1@1 1", "recall_1@5 1",
                         "recall_1@16 1"]
    assert lines[5] == "recall_5@5 1" and lines[-3].startswith("latency_mean_us ")


def test_exact_tensor_core_and_float32_filters_agree(tmp_path):
    """The filter tiers — three-term tcgen05 ($AQ_EXACT_TC=1, default),
    one-term then three-term (13), the float32 FFMA filter alone (0) — give
    the same ids and scores (all equal to the oracle's), including duplicated
    rows (exact ties) and a zero query."""
    import subprocess
    import sys
    import os
    script = tmp_path / "ex.py"
    script.write_text(
        "import sys, numpy as np\n"
        f"sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})\n"
        "from paper_1908_10396_b200 import anisoq as aq\n"
        "from tests.helpers import mixture_rows\n"
        "x = np.repeat(mixture_rows(20000, 100, 91), 3, axis=0)\n"
        "q = mixture_rows(200, 100, 92).astype(np.float64); q[7] = 0.0\n"
        "ids, sc = aq.dev_exact_search(aq.Session.default().upload_dataset(x), q, 25)\n"
        "np.savez(sys.argv[1], ids=ids, sc=sc)\n")
    out = {}
    for flag in ("1", "13", "0"):
        f = tmp_path / f"r{flag}.npz"
        r = subprocess.run([sys.executable, str(script), str(f)], capture_output=True, text=True,
                           env=dict(os.environ, AQ_EXACT_TC=flag), timeout=300)
        assert r.returncode == 0, r.stderr
        out[flag] = np.load(f)
    for flag in ("13", "0"):
        assert np.array_equal(out["1"]["ids"], out[flag]["ids"])
        assert np.array_equal(out["1"]["sc"], out[flag]["sc"])
    x = np.repeat(mixture_rows(20000, 100, 91), 3, axis=0).astype(np.float64)
    q = mixture_rows(200, 100, 92).astype(np.float64)
    q[7] = 0.0
    wi, ws = P.exact_search_batch(q, x, 25)
    assert np.array_equal(out["1"]["ids"], wi) and np.array_equal(out["1"]["sc"], ws)
