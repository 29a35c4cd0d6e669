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

import math
from typing import Optional

import numpy as np
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


_PAD_ID = 1 << 62  # sorts after every real id at score -inf


def pad_candidates(ids: torch.Tensor, adc: torch.Tensor, exact: torch.Tensor, width: int):
    """Right-pad [nq, K] candidate lists to `width` columns with (id 2^62,
    score -inf): shards smaller than top-N return fewer candidates, and the
    all-gather needs one shape on every rank. order_desc puts padding last."""
    k = ids.shape[1]
    if k >= width:
        return ids, adc, exact
    nq = ids.shape[0]
    pid = torch.full((nq, width - k), _PAD_ID, dtype=ids.dtype, device=ids.device)
    pin = torch.full((nq, width - k), -math.inf, dtype=adc.dtype, device=adc.device)
    return (torch.cat([ids, pid], 1), torch.cat([adc, pin], 1),
            torch.cat([exact, pin.to(exact.dtype)], 1))


def all_gather_candidates(local_ids: torch.Tensor, local_adc: torch.Tensor,
                          local_exact: torch.Tensor, group=None):
    """[nq, K] per rank -> [nq, world*K] on every rank: ONE all-gather of the
    packed (id, ADC score, exact score) triples (float64 bit patterns)."""
    world = dist.get_world_size(group)
    nq, K = local_ids.shape
    packed = torch.stack([local_ids.to(torch.int64),
                          local_adc.to(torch.float64).view(torch.int64),
                          local_exact.to(torch.float64).view(torch.int64)], 0).contiguous()
    buf = [torch.empty_like(packed) for _ in range(world)]
    dist.all_gather(buf, packed, group=group)
    allp = torch.cat(buf, dim=2)  # [3, nq, world*K]
    return allp[0], allp[1].view(torch.float64), allp[2].view(torch.float64)


def sharded_search_rerank(ds, codes, cb, queries: torch.Tensor, offset: int, topn: int = 100,
                          keep: int = 10, group=None, n_total: Optional[int] = None):
    """Per-rank device search over the local shard + exact merge across ranks.

    ds/codes/cb: this rank's DeviceDataset/DeviceCodes/DeviceCodebook;
    queries: float64 [nq, d] on this rank's GPU; offset: global id of local row 0;
    n_total: rows over all shards (one all-reduce finds it when omitted)."""
    from . import anisoq as aq

    L = aq._L
    nq = queries.shape[0]
    te = min(topn, codes.n)
    dev = queries.device
    # the library runs on its session stream: it must see the queries that
    # torch's stream produced (e.g. an H2D copy), and torch's stream must see
    # the library's outputs before the collective (stream waits, no host sync)
    lib = torch.cuda.ExternalStream(codes.s.stream, device=dev)
    torch_stream = torch.cuda.current_stream(dev)
    with torch.cuda.stream(torch_stream):
        aid = torch.empty((nq, te), dtype=torch.int32, device=dev)
        asc = torch.empty((nq, te), dtype=torch.float64, device=dev)
        exd = torch.empty((nq, te), dtype=torch.float64, device=dev)
    lib.wait_stream(torch_stream)
    aq._check(L.aq_dev_adc_search_d(codes.h, cb.h, queries.data_ptr(), nq, topn,
                                    aid.data_ptr(), asc.data_ptr()))
    aq._check(L.aq_dev_exact_dots_d(ds.h, queries.data_ptr(), nq, aid.data_ptr(), te,
                                    exd.data_ptr()))
    torch_stream.wait_stream(lib)
    for t in (queries, aid, asc, exd):
        t.record_stream(lib)
    gids = aid.to(torch.int64) + offset
    # every rank gathers the same width: min(topn, n_total)
    if n_total is None:
        t = torch.tensor([codes.n], dtype=torch.int64, device=dev)
        if dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(t, group=group)
        n_total = int(t.item())
    width = min(topn, n_total)
    gids, asc, exd = pad_candidates(gids, asc, exd, width)
    ids, adc, ex = all_gather_candidates(gids, asc, exd, group)
    return merge_candidates(ids, adc, ex, topn, keep)


# =============================================================================
# Row-sharded training (train_l2_pq pq.hpp:469-501 / train_apq pq.hpp:513-575)
# =============================================================================
#
# Every rank owns a contiguous row range and keeps its codes; the codebook is
# replicated. Per iteration the ranks exchange only sums:
#
#   assignment  local (encode.cu / k_kmeans_assign), per-shard loss sums and
#               change counts -> all-gather -> combined in rank order;
#   update      per-shard partials (normal equations, isotropic or k-means
#               sums, usage counts) -> all-gather -> summed in rank order on
#               every rank -> identical solve on every rank;
#   reseed      per-shard loss ranking (top U) -> all-gather -> exact merge by
#               (loss desc, id asc) -> rows fetched from their owners.
#
# Combining in rank order (not an all-reduce whose association depends on the
# NCCL algorithm) makes the result a deterministic function of the world
# size. With one rank every partial IS the full sequential sum, so the
# trainer equals the single-GPU one (aq_dev_train_apq) bit for bit; with W
# ranks the float64 sums are re-associated at W-1 shard boundaries (relative
# effect ~1e-16 per sum), the only difference from the reference.

_MASK64 = (1 << 64) - 1


class HostRng:
    """anisoq::Rng (rng.hpp:28-89) on the host: splitmix64, next_below by
    rejection, sample_distinct as a partial Fisher-Yates on iota(n) with only
    the touched positions materialised (O(k))."""

    def __init__(self, seed: int):
        self.state = seed & _MASK64

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        return z ^ (z >> 31)

    def next_below(self, n: int) -> int:
        threshold = ((1 << 64) - n) % n
        while True:
            r = self.next_u64()
            if r >= threshold:
                return r % n

    def sample_distinct(self, n: int, k: int) -> list:
        moved: dict = {}
        out = []
        for i in range(min(k, n)):
            j = i + self.next_below(n - i)
            vi, vj = moved.get(i, i), moved.get(j, j)
            moved[i], moved[j] = vj, vi
            out.append(vj)
        return out


class _Comm:
    """Rank-ordered exchange over torch.distributed (NCCL on GPUs, gloo in the
    CPU tests); a world of one needs no process group."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def gather(self, t: torch.Tensor) -> list:
        t = t.contiguous()
        if self.world == 1:
            return [t]
        buf = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(buf, t, group=self.group)
        return buf

    def chain_sum(self, t: torch.Tensor, chunk: int = 1 << 22) -> Optional[torch.Tensor]:
        """Rank-ordered sum ((P0 + P1) + P2) + ... of every rank's `t`, complete
        on the LAST rank (None elsewhere): rank r receives the running sum from
        r - 1 chunk by chunk, adds its own partial and forwards it, so every
        link carries the data once and chunks pipeline along the chain
        (instead of all-gathering W full partials onto every rank)."""
        flat = t.contiguous().view(-1)
        if self.world == 1:
            return flat.clone().view(t.shape)
        acc = flat.clone() if self.rank == 0 else torch.empty_like(flat)
        sends = []
        for lo in range(0, flat.numel(), chunk):
            hi = min(flat.numel(), lo + chunk)
            if self.rank > 0:
                dist.recv(acc[lo:hi], src=self.rank - 1, group=self.group)
                acc[lo:hi] += flat[lo:hi]  # running sum of ranks < r, then this rank's
            if self.rank < self.world - 1:
                sends.append(dist.isend(acc[lo:hi], dst=self.rank + 1, group=self.group))
        for h in sends:
            h.wait()
        return acc.view(t.shape) if self.rank == self.world - 1 else None

    def bcast_from_last(self, t: Optional[torch.Tensor], like: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t
        buf = t if t is not None else torch.empty_like(like)
        dist.broadcast(buf, src=self.world - 1, group=self.group)
        return buf

    def ordered_sum(self, t: torch.Tensor) -> torch.Tensor:
        """Rank-ordered sum on every rank (chain + broadcast)."""
        return self.bcast_from_last(self.chain_sum(t), t)

    def ordered_scalar_sum(self, v: float, device) -> float:
        """Per-shard float64 sums combined left to right in rank order."""
        parts = self.gather(torch.tensor([v], dtype=torch.float64, device=device))
        acc = float(parts[0].item())
        for p in parts[1:]:
            acc = acc + float(p.item())
        return acc

    def int_sum(self, t: torch.Tensor) -> torch.Tensor:
        t = t.to(torch.int64).contiguous()
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t


class ShardedTrainer:
    """Sharded train_l2_pq / train_apq over a compute backend `shard`.

    `shard` computes on this rank's rows (DeviceShard below on a B200; the
    tests drive the same orchestration with a CPU backend). Errors are the
    reference's (anisoq.py classes) with global point indices."""

    def __init__(self, shard, n_total: int, offset: int, group=None):
        self.sh = shard
        self.n_total = n_total
        self.offset = offset
        self.comm = _Comm(group)
        self._verified: set = set()
        self._tril: dict = {}

    # ---- helpers ---------------------------------------------------------
    def _do(self, fn, *args):
        """One per-shard step on every rank. A failure on any rank raises the
        same reference error on all ranks (the first failing rank's), so no
        rank is left waiting in a collective. The status exchange runs only
        the first time a step kind is taken: the data-dependent failures
        (weights of a zero-norm or |x| <= T point, device limits) show on a
        step's first call, so the steady-state loop carries no status
        collectives."""
        from . import anisoq as aq
        res, err = None, None
        try:
            res = fn(*args)
        except Exception as e:  # noqa: BLE001 - re-raised on every rank below
            err = e
        key = getattr(fn, "__name__", repr(fn))
        if self.comm.world == 1 or key in self._verified:
            if err is not None:
                raise err
            return res
        st = int(getattr(err, "status", 999) or 999) if err is not None else 0
        codes = self.comm.gather(torch.tensor([st], dtype=torch.int64, device=self.sh.device))
        first = next((r for r, c in enumerate(codes) if int(c.item())), None)
        if first is None:
            self._verified.add(key)
            return res
        msg = [str(err) if err is not None else ""]
        dist.broadcast_object_list(msg, src=first, group=self.comm.group)
        raise aq._BY_STATUS.get(int(codes[first].item()), aq.Error)(msg[0])

    def _validate(self, M: int, k: int) -> None:
        from . import anisoq as aq
        if self.n_total == 0:
            raise aq.EmptyDataset("EmptyDataset: cannot train on an empty dataset")
        if M == 0 or self.sh.d % M != 0:
            raise aq.DimensionNotDivisible("DimensionNotDivisible: dimension not divisible by M")
        if k == 0 or k > self.n_total:
            raise aq.InvalidArgument("InvalidArgument: need 1 <= k <= n")

    def _fetch_rows(self, gids: list) -> torch.Tensor:
        """float64 rows [len(gids), d] of global ids, taken from their owners."""
        dev = self.sh.device
        n_local = self.sh.n
        lo = self.offset
        g = torch.tensor(gids, dtype=torch.int64, device=dev)
        mine = (g >= lo) & (g < lo + n_local)
        rows = torch.zeros((len(gids), self.sh.d), dtype=torch.float64, device=dev)
        if bool(mine.any()):
            rows[mine] = self.sh.rows(g[mine] - lo)
        owned = self.comm.gather(mine.to(torch.int32))
        parts = self.comm.gather(rows)
        out = torch.zeros_like(rows)
        for o, p in zip(owned, parts):
            sel = o.bool()
            out[sel] = p[sel]
        return out

    def _global_ranking(self, losses: torch.Tensor, count: int) -> list:
        """First min(count, n_total) global ids of loss_ranking (vq.hpp:221-229):
        (loss desc, id asc) over all shards."""
        take = min(count, self.n_total)
        vals, lidx = self._do(self.sh.ranking, losses, min(take, self.sh.n))
        dev = self.sh.device
        v = torch.full((take,), -math.inf, dtype=torch.float64, device=dev)
        i = torch.full((take,), 1 << 62, dtype=torch.int64, device=dev)
        v[: vals.numel()] = vals
        i[: lidx.numel()] = lidx.to(torch.int64) + self.offset
        allv = torch.cat(self.comm.gather(v))
        alli = torch.cat(self.comm.gather(i))
        o = order_desc(allv, alli)[:take]
        return alli[o].tolist()

    def _init_rows(self, hidx: list, M: int, k: int, sd: int) -> torch.Tensor:
        rows = self._fetch_rows(hidx)  # [M*k, d]
        m = torch.arange(M * k, device=rows.device) // k
        cols = m[:, None] * sd + torch.arange(sd, device=rows.device)[None, :]
        return torch.gather(rows, 1, cols).reshape(-1).contiguous()

    # ---- train_l2_pq -------------------------------------------------------
    def train_l2_pq(self, M: int, k: int, cfg) -> torch.Tensor:
        """pq.hpp:469-501: per-subspace k-means (seed + m), lockstep. Returns the
        replicated dictionaries (float64 [M*k*sd]); codes stay in the shard."""
        from . import anisoq as aq
        self._validate(M, k)
        sd = self.sh.d // M
        hidx = []
        for m in range(M):
            hidx += HostRng(cfg.seed + m).sample_distinct(self.n_total, k)
        dict_ = self._init_rows(hidx, M, k, sd)
        self._do(self.sh.set_codebook, dict_, M, k, sd)
        active = [1] * M

        def assign():
            losses, changes = self._do(self.sh.kmeans_assign, active)
            chg = self.comm.int_sum(torch.as_tensor(changes, dtype=torch.int64,
                                                    device=self.sh.device)).tolist()
            # totals only feed the relative-tolerance test (vq.hpp:316-321;
            # train_l2_pq discards the histories)
            if cfg.relative_tolerance > 0.0:
                loc = self._do(self.sh.seq_sums, losses, active)
                tot = self.comm.ordered_sum(torch.tensor(loc, dtype=torch.float64,
                                                         device=self.sh.device)).tolist()
            else:
                tot = [0.0] * M
            return losses, chg, tot

        losses, chg, tot = assign()
        for _ in range(cfg.max_iterations):
            if not any(active):
                break
            num, den, cnt = self._do(self.sh.kmeans_partials, active)
            num = self.comm.ordered_sum(num).reshape(M * k, sd)
            den = self.comm.ordered_sum(den).reshape(M * k)
            cnt = self.comm.int_sum(cnt).reshape(M * k)
            act = torch.tensor(active, dtype=torch.bool, device=dict_.device).repeat_interleave(k)
            upd = act & (cnt > 0)
            d2 = dict_.reshape(M * k, sd)
            d2[upd] = num[upd] / den[upd, None]
            if cfg.empty_partition_policy == "reseed_highest_loss":
                cnt_h = cnt.tolist()
                for m in range(M):
                    if not active[m]:
                        continue
                    empty = [j for j in range(k) if cnt_h[m * k + j] == 0]
                    if not empty:
                        continue
                    order = self._global_ranking(losses[m], len(empty))
                    rows = self._fetch_rows(order[: len(empty)])
                    for c, j in enumerate(empty):
                        d2[m * k + j] = rows[c, m * sd:(m + 1) * sd]
            dict_ = d2.reshape(-1).contiguous()
            self._do(self.sh.set_codebook, dict_, M, k, sd)
            prev = tot
            losses, chg, tot = assign()
            for m in range(M):
                if not active[m]:
                    continue
                if chg[m] == 0:
                    active[m] = 0
                    continue
                if cfg.relative_tolerance > 0.0 and (
                        prev[m] == 0.0 or prev[m] - tot[m] <= cfg.relative_tolerance * prev[m]):
                    active[m] = 0
        return dict_

    # ---- pq_codebook_update ---------------------------------------------------
    def codebook_update(self, M: int, k: int, ridge: float) -> torch.Tensor:
        """pq.hpp:356-464 with per-shard partials (M > 1)."""
        from . import anisoq as aq
        sd = self.sh.d // M
        if M == 1:
            raise aq.Unsupported("Unsupported: the sharded trainer needs M > 1 "
                                 "(M == 1 runs the single-GPU update_codeword path)")
        if sd > 16:
            raise aq.Unsupported("Unsupported: device update supports sub_dimension <= 16")
        any_aniso, zero_idx = self._do(self.sh.weight_flags)
        dev = self.sh.device
        flag = self.comm.int_sum(torch.tensor([int(any_aniso)], device=dev)).item() > 0
        big = 1 << 62
        z = torch.tensor([zero_idx + self.offset if zero_idx is not None else big], device=dev)
        zmin = min(int(p.item()) for p in self.comm.gather(z))
        dim = k * self.sh.d
        if not flag:
            num, den, usage = self._do(self.sh.iso_partials, k)
            num = self.comm.ordered_sum(num).reshape(M * k, sd)
            den = self.comm.ordered_sum(den).reshape(M * k)
            usage = self.comm.int_sum(usage).reshape(M * k)
            used = usage > 0
            if bool((den[used] <= 0.0).any()):
                raise aq.SingularSystem("SingularSystem: zero total weight in block")
            x = torch.zeros((M * k, sd), dtype=torch.float64, device=dev)
            x[used] = num[used] / den[used, None]
            x = x.reshape(-1)
        else:
            if dim > 16384:
                raise aq.InvalidArgument("InvalidArgument: stacked codebook system exceeds "
                                         "16384 unknowns (pq.hpp:426-429)")
            if zmin != big:
                raise aq.ZeroNormDatapoint(
                    f"ZeroNormDatapoint: anisotropic update undefined at |x| = 0 (point {zmin})")
            A, rhs, usage = self._do(self.sh.normal_equations, k)
            # the solve reads the lower triangle only: pack it with rhs, sum
            # along the rank chain, solve on the last rank, broadcast x
            mask = self._tril.get(dim)
            if mask is None:
                mask = torch.ones((dim, dim), dtype=torch.bool, device=dev).tril_()
                self._tril[dim] = mask
            tot = self.comm.chain_sum(torch.cat([A[mask], rhs]))
            usage = self.comm.int_sum(usage).reshape(M * k)
            res = torch.empty(dim + 1, dtype=torch.float64, device=dev)
            msg = [""]
            if tot is not None:
                A = torch.zeros((dim, dim), dtype=torch.float64, device=dev)
                A[mask] = tot[:-dim]
                try:
                    res[:dim] = self.sh.solve(A, tot[-dim:], ridge)
                    res[dim] = 0.0
                except aq.Error as e:  # replicated below: every rank raises it
                    res[dim] = float(getattr(e, "status", 999) or 999)
                    msg[0] = str(e)
            res = self.comm.bcast_from_last(res if tot is not None else None, res)
            st = int(res[dim].item())
            if st:
                if self.comm.world > 1:
                    dist.broadcast_object_list(msg, src=self.comm.world - 1,
                                               group=self.comm.group)
                raise aq._BY_STATUS.get(st, aq.Error)(msg[0])
            x = res[:dim].clone()
        unused = [t for t, c in enumerate(usage.tolist()) if c == 0]
        if unused:
            # reseed from the loss ranking under the new codebook (pq.hpp:446-462)
            self._do(self.sh.set_codebook, x, M, k, sd)
            losses = self._do(self.sh.point_losses)
            order = self._global_ranking(losses, len(unused))
            rows = self._fetch_rows(order)
            x2 = x.reshape(M * k, sd)
            for c, t in enumerate(unused):
                m = t // k
                x2[t] = rows[c % len(order), m * sd:(m + 1) * sd]
            x = x2.reshape(-1).contiguous()
        self._do(self.sh.set_codebook, x, M, k, sd)
        return x

    # ---- train_apq ------------------------------------------------------------
    def train_apq(self, M: int, k: int, cfg, warm_start: bool = True,
                  loss_history: Optional[list] = None) -> torch.Tensor:
        """pq.hpp:513-575 over the shards. Returns the replicated dictionaries;
        this rank's codes are in the shard (shard.codes)."""
        self._validate(M, k)
        sd = self.sh.d // M
        if warm_start:
            dict_ = self.train_l2_pq(M, k, cfg)
        else:
            r = HostRng(cfg.seed)  # one generator for all subspaces (pq.hpp:533-542)
            hidx = []
            for _ in range(M):
                hidx += r.sample_distinct(self.n_total, k)
            dict_ = self._init_rows(hidx, M, k, sd)
            self._do(self.sh.set_codebook, dict_, M, k, sd)
            self._do(self.sh.nearest)

        def apass():
            losses, changed = self._do(self.sh.assign_pass, cfg.sweep_to_fixed_point)
            tot = self.comm.ordered_scalar_sum(self._do(self.sh.seq_sum, losses), self.sh.device)
            ch = int(self.comm.int_sum(torch.tensor([changed], device=self.sh.device)).item())
            return tot, ch

        tot, changed = apass()
        hist = [tot]
        for _ in range(cfg.max_iterations):
            dict_ = self.codebook_update(M, k, cfg.ridge)
            prev = tot
            tot, changed = apass()
            hist.append(tot)
            if changed == 0:
                break
            if cfg.relative_tolerance > 0.0 and (
                    prev == 0.0 or prev - tot <= cfg.relative_tolerance * prev):
                break
        if loss_history is not None:
            loss_history.extend(hist)
        return dict_


class DeviceShard:
    """This rank's rows on its B200 behind the C ABI (aq_dev_* building blocks).

    rows: float32 [n_local, d] CUDA tensor; weights: AnisotropicWeights,
    ThresholdWeights or this shard's per-point (h_par, h_perp) arrays."""

    def __init__(self, session, rows: torch.Tensor, weights):
        from . import anisoq as aq
        import ctypes as C
        self._aq, self._C = aq, C
        self.s = session
        self.x = rows.contiguous()
        self.n, self.d = self.x.shape
        self.device = self.x.device
        self._lib = torch.cuda.ExternalStream(session.stream, device=self.device)
        torch.cuda.current_stream(self.device).synchronize()
        self.ds = session.wrap_device_rows(self.x.data_ptr(), self.n, self.d)
        self._keep: list = []
        self.w = aq._weights(weights, self.n, self._keep)
        self.cb = None
        self.codes = None

    def _call(self, name, *args):
        # the library works on the session stream: order it after torch's
        # pending work on its inputs, and torch's stream after the library's
        # outputs (stream waits, no host synchronisation)
        ts = torch.cuda.current_stream(self.device)
        self._lib.wait_stream(ts)
        self._aq._check(getattr(self._aq._L, name)(*args))
        ts.wait_stream(self._lib)

    def _ensure(self, M, k, sd):
        aq = self._aq
        if self.cb is None or (self.cb.M, self.cb.k, self.cb.sd) != (M, k, sd):
            self.cb = self.s.upload_codebook(aq.ProductCodebook(
                M, k, sd, np.zeros(M * k * sd, np.float64)))
        if self.codes is None or (self.codes.M, self.codes.k) != (M, k):
            self.codes = self.s.alloc_codes(self.n, M, k)

    # codebook / rows
    def set_codebook(self, dict_: torch.Tensor, M: int, k: int, sd: int) -> None:
        self._ensure(M, k, sd)
        d = dict_.to(device=self.device, dtype=torch.float64).contiguous()
        self._call("aq_codebook_set_device", self.cb.h, d.data_ptr())

    def rows(self, local_idx: torch.Tensor) -> torch.Tensor:
        return self.x[local_idx].to(torch.float64)

    # assignment
    def nearest(self) -> None:
        iso = self._aq._weights(self._aq.AnisotropicWeights.isotropic(), self.n, [])
        self._call("aq_dev_pq_quantize", self.ds.h, self.cb.h, self._C.byref(iso), 0,
                   self.codes.h)

    def assign_pass(self, sweep_fixed: bool):
        losses = torch.empty(self.n, dtype=torch.float64, device=self.device)
        ch = self._C.c_uint64(0)
        self._call("aq_dev_pq_assign_pass", self.ds.h, self.cb.h, self._C.byref(self.w),
                   int(sweep_fixed), self.codes.h, losses.data_ptr() if self.n else None,
                   self._C.byref(ch))
        return losses, ch.value

    def kmeans_assign(self, active: list):
        M = self.cb.M
        losses = torch.zeros((M, self.n), dtype=torch.float64, device=self.device)
        act = np.asarray(active, np.int32)
        ch = np.zeros(M, np.uint64)
        self._call("aq_dev_kmeans_assign", self.ds.h, self.cb.h, self.codes.h,
                   act.ctypes.data, losses.data_ptr(), ch.ctypes.data)
        return losses, ch.astype(np.int64)

    def point_losses(self) -> torch.Tensor:
        losses = torch.empty(max(self.n, 1), dtype=torch.float64, device=self.device)
        self._call("aq_dev_point_losses", self.ds.h, self.cb.h, self._C.byref(self.w),
                   self.codes.h, losses.data_ptr())
        return losses[: self.n]

    def seq_sum(self, v: torch.Tensor) -> float:
        out = self._C.c_double(0.0)
        v = v.contiguous()
        self._call("aq_dev_seq_sum", self.s.h, v.data_ptr(), v.numel(), 0.0,
                   self._C.byref(out))
        return out.value

    def seq_sums(self, losses: torch.Tensor, active: list) -> list:
        """Row-wise sequential sums of losses [rows, n] (0 for inactive rows)."""
        v = losses.contiguous()
        rows, cnt = v.shape
        act = np.asarray(active, np.int32)
        out = np.zeros(rows, np.float64)
        self._call("aq_dev_seq_sums", self.s.h, v.data_ptr(), cnt, cnt, rows, act.ctypes.data,
                   out.ctypes.data)
        return out.tolist()

    def ranking(self, losses: torch.Tensor, top: int):
        idx = torch.arange(self.n, dtype=torch.int32, device=self.device)
        v = losses.contiguous()
        if self.n:
            self._call("aq_dev_sort_desc", self.s.h, v.data_ptr(), idx.data_ptr(), self.n)
        sel = idx[:top].to(torch.int64)
        return v[sel], sel

    # partial sums
    def weight_flags(self):
        fl = np.zeros(2, np.uint64)
        self._call("aq_dev_weight_flags", self.ds.h, self._C.byref(self.w), fl.ctypes.data)
        return bool(fl[0]), (int(fl[1]) - 1 if fl[1] else None)

    def kmeans_partials(self, active: list):
        M, k, sd = self.cb.M, self.cb.k, self.cb.sd
        num = torch.empty(M * k * sd, dtype=torch.float64, device=self.device)
        den = torch.empty(M * k, dtype=torch.float64, device=self.device)
        cnt = torch.zeros(M * k, dtype=torch.int32, device=self.device)
        act = np.asarray(active, np.int32)
        self._call("aq_dev_kmeans_partials", self.ds.h, self.codes.h, k, act.ctypes.data,
                   num.data_ptr(), den.data_ptr(), cnt.data_ptr())
        return num, den, cnt

    def iso_partials(self, k: int):
        M, sd = self.codes.M, self.d // self.codes.M
        num = torch.empty(M * k * sd, dtype=torch.float64, device=self.device)
        den = torch.empty(M * k, dtype=torch.float64, device=self.device)
        usage = torch.zeros(M * k, dtype=torch.int32, device=self.device)
        self._call("aq_dev_iso_partials", self.ds.h, self.codes.h, self._C.byref(self.w), k,
                   num.data_ptr(), den.data_ptr(), usage.data_ptr())
        return num, den, usage

    def normal_equations(self, k: int):
        M, dim = self.codes.M, k * self.d
        A = torch.empty((dim, dim), dtype=torch.float64, device=self.device)
        rhs = torch.empty(dim, dtype=torch.float64, device=self.device)
        usage = torch.zeros(M * k, dtype=torch.int32, device=self.device)
        fl = np.zeros(2, np.uint64)
        self._call("aq_dev_normal_equations_partial", self.ds.h, self.codes.h,
                   self._C.byref(self.w), k, A.data_ptr(), rhs.data_ptr(), usage.data_ptr(),
                   fl.ctypes.data)
        return A, rhs, usage

    def solve(self, A: torch.Tensor, rhs: torch.Tensor, ridge: float) -> torch.Tensor:
        A = A.contiguous().clone()
        x = rhs.contiguous().clone()
        self._call("aq_dev_solve_normal_equations", self.s.h, A.data_ptr(), x.data_ptr(),
                   x.numel(), float(ridge))
        return x
