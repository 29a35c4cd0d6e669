"""Multi-rank (world_size 2, gloo, CPU) tests of the sharded query path's host
logic: shard bounds, the all-gather of per-shard candidates and the exact merge.
Per-shard results come from the oracle (test infrastructure standing in for
each rank's device computation); the merged result must equal the oracle on
the whole database."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1908_10396_b200.distributed import (merge_candidates, order_desc, pad_candidates,
                                                shard_bounds, all_gather_candidates)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_cover():
    for n, w in [(10, 3), (1183514, 8), (5, 8)]:
        spans = [shard_bounds(n, r, w) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_order_desc_is_select_top_order():
    s = torch.tensor([[1.0, 3.0, 3.0, -1.0, 3.0]], dtype=torch.float64)
    i = torch.tensor([[9, 7, 2, 1, 5]])
    o = order_desc(s, i)
    assert torch.gather(i, 1, o).tolist() == [[2, 5, 7, 9, 1]]


def _worker(rank, world, port, data, queries, codes, cb, M, out, topn=100):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Port

    P = Port()
    lo, hi = shard_bounds(len(data), rank, world)
    ids, adc = P.adc_search_batch(queries, codes[lo:hi], 16, cb, M, 16, 2, topn)
    ex = np.stack([[float(np.add.accumulate(queries[q] * data[lo + int(i)])[-1]) for i in row]
                   for q, row in enumerate(ids)])
    # shards smaller than topn return fewer candidates: pad to one width
    g = pad_candidates(torch.from_numpy(ids.astype(np.int64) + lo), torch.from_numpy(adc),
                       torch.from_numpy(ex), min(topn, len(data)))
    g = all_gather_candidates(*g)
    res = merge_candidates(*g, topn, 10)
    if rank == 0:
        out.update({k: v.numpy() for k, v in zip(("aid", "asc", "rid", "rsc"), res)})
    dist.destroy_process_group()


def test_two_rank_merge_equals_single_process():
    from oracle import Port

    P = Port()
    rng = np.random.default_rng(0)
    n, M = 6000, 8
    data = rng.standard_normal((n, 2 * M)).astype(np.float32).astype(np.float64)
    queries = rng.standard_normal((6, 2 * M))
    cb = rng.standard_normal(M * 32) * 0.5
    codes = rng.integers(0, 16, (n, M)).astype(np.uint32)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), data, queries, codes, cb, M, out), nprocs=2,
             join=True)
    wi, ws = P.adc_search_batch(queries, codes, 16, cb, M, 16, 2, 100)
    ri, rs = P.rerank(queries, data, wi, 10)
    assert np.array_equal(out["aid"], wi) and np.array_equal(out["asc"], ws)
    assert np.array_equal(out["rid"], ri) and np.array_equal(out["rsc"], rs)


def test_unequal_shards_smaller_than_topn():
    """ADC top-100 over shards of 67/67/66 rows (3 ranks) and 75/75 (2 ranks):
    per-shard lists are shorter than top-N and are padded before the gather."""
    from oracle import Port

    P = Port()
    rng = np.random.default_rng(1)
    M = 4
    for n, world in ((200, 3), (150, 2)):
        data = rng.standard_normal((n, 2 * M)).astype(np.float32).astype(np.float64)
        queries = rng.standard_normal((3, 2 * M))
        cb = rng.standard_normal(M * 32) * 0.5
        codes = rng.integers(0, 16, (n, M)).astype(np.uint32)
        mgr = mp.Manager()
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), data, queries, codes, cb, M, out, 100),
                 nprocs=world, join=True)
        wi, ws = P.adc_search_batch(queries, codes, 16, cb, M, 16, 2, 100)
        ri, rs = P.rerank(queries, data, wi, 10)
        assert np.array_equal(out["aid"], wi) and np.array_equal(out["asc"], ws)
        assert np.array_equal(out["rid"], ri) and np.array_equal(out["rsc"], rs)
