"""Row-sharded multi-GPU query path (one process per GPU, torch.distributed).

Each rank owns a contiguous row range of the database and answers for it:
exact local ADC top-N (k_adc_score/k_adc_merge), exact float64 dots of those
local candidates (k_exact_dots), then ONE all-gather of (global id, ADC score,
exact score) per candidate. Every rank merges the gathered lists exactly:

  global ADC top-N  = first N of the union ordered by (ADC score desc, id asc)
  rerank top-K      = those N ordered by (exact score desc, id asc)

which equals the single-GPU result: an item of the global top-N is in its own
shard's top-N, and both orders are total. The merge is plain tensor sorting,
so it runs on NCCL/CUDA tensors in bench.py and on gloo/CPU tensors in the
tests (tests/test_distributed.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous row range of `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def order_desc(scores: torch.Tensor, ids: torch.Tensor) -> torch.Tensor:
    """Permutation per row ordering by (score desc, id asc) — select_top's order
    (index.hpp:88-112). Exact: two stable sorts, no arithmetic on scores."""
    o1 = torch.sort(ids, dim=-1, stable=True).indices
    s1 = torch.gather(scores, -1, o1)
    o2 = torch.sort(s1, dim=-1, descending=True, stable=True).indices
    return torch.gather(o1, -1, o2)


def merge_candidates(ids: torch.Tensor, adc: torch.Tensor, exact: torch.Tensor,
                     topn: int, keep: int):
    """ids/adc/exact: [nq, C] gathered candidates (global ids).
    Returns (adc_ids, adc_scores, ids, exact_scores) like the single-GPU pipeline."""
    o = order_desc(adc, ids)[:, :topn]
    g_ids = torch.gather(ids, 1, o)
    g_adc = torch.gather(adc, 1, o)
    g_ex = torch.gather(exact, 1, o)
    o2 = order_desc(g_ex, g_ids)[:, :keep]
    return g_ids, g_adc, torch.gather(g_ids, 1, o2), torch.gather(g_ex, 1, o2)


def all_gather_candidates(local_ids: torch.Tensor, local_adc: torch.Tensor,
                          local_exact: torch.Tensor, group=None):
    """[nq, K] per rank -> [nq, world*K] on every rank (one collective per field)."""
    world = dist.get_world_size(group)
    outs = []
    for t in (local_ids, local_adc, local_exact):
        buf = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(buf, t.contiguous(), group=group)
        outs.append(torch.cat(buf, dim=1))
    return outs


def sharded_search_rerank(ds, codes, cb, queries: torch.Tensor, offset: int, topn: int = 100,
                          keep: int = 10, group=None):
    """Per-rank device search over the local shard + exact merge across ranks.

    ds/codes/cb: this rank's DeviceDataset/DeviceCodes/DeviceCodebook;
    queries: float64 [nq, d] on this rank's GPU; offset: global id of local row 0."""
    from . import anisoq as aq

    L = aq._L
    nq = queries.shape[0]
    te = min(topn, codes.n)
    dev = queries.device
    aid = torch.empty((nq, te), dtype=torch.int32, device=dev)
    asc = torch.empty((nq, te), dtype=torch.float64, device=dev)
    exd = torch.empty((nq, te), dtype=torch.float64, device=dev)
    aq._check(L.aq_dev_adc_search_d(codes.h, cb.h, queries.data_ptr(), nq, topn,
                                    aid.data_ptr(), asc.data_ptr()))
    aq._check(L.aq_dev_exact_dots_d(ds.h, queries.data_ptr(), nq, aid.data_ptr(), te,
                                    exd.data_ptr()))
    gids = aid.to(torch.int64) + offset
    ids, adc, ex = all_gather_candidates(gids, asc, exd, group)
    return merge_candidates(ids, adc, ex, topn, keep)
