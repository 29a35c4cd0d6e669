"""CPU compute backend for the sharded trainer (test infrastructure only).

Implements the per-shard interface of paper_1908_10396_b200.distributed
(DeviceShard's methods) with numpy and the C oracle (oracle/anisoq_oracle.c),
so the host orchestration — exchange, rank-ordered combination, reseed
ranking, stopping rules — runs under gloo with world_size 2 on a CPU-only
machine. Sums follow the same member order as the device kernels
(np.add.at applies its updates in index order).
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import Port


class OracleShard:
    def __init__(self, rows: np.ndarray, hp: np.ndarray, ho: np.ndarray):
        self.x = np.ascontiguousarray(rows, np.float64)
        self.n, self.d = self.x.shape
        self.hp = np.ascontiguousarray(hp, np.float64)
        self.ho = np.ascontiguousarray(ho, np.float64)
        self.port = Port()
        self.norms = self.port.row_norms(self.x) if self.n else np.zeros(0)
        self.device = torch.device("cpu")
        self.cb = None
        self.M = self.k = self.sd = 0
        self.codes = None

    def set_codebook(self, dict_, M, k, sd):
        self.cb = dict_.detach().cpu().numpy().astype(np.float64).copy()
        if self.codes is None or self.codes.shape[1] != M or self.k != k:
            self.codes = np.zeros((self.n, M), np.uint32)
        self.M, self.k, self.sd = M, k, sd

    def rows(self, local_idx):
        return torch.from_numpy(self.x[local_idx.numpy()].copy())

    def nearest(self):
        one = np.ones(self.n)
        self.codes = self.port.pq_quantize(self.x, self.cb, self.M, self.k, self.sd, one, one, 0)

    def assign_pass(self, sweep_fixed):
        new, losses = self.port.pq_assign_pass(self.x, self.cb, self.M, self.k, self.sd,
                                               self.hp, self.ho, self.codes, sweep_fixed)
        changed = int((new != self.codes).any(axis=1).sum())
        self.codes = new
        return torch.from_numpy(losses), changed

    def kmeans_assign(self, active):
        M, k, sd = self.M, self.k, self.sd
        cb = self.cb.reshape(M, k, sd)
        losses = np.zeros((M, self.n))
        ch = np.zeros(M, np.int64)
        for m in range(M):
            if not active[m]:
                continue
            xs = self.x[:, m * sd:(m + 1) * sd]
            d2 = np.zeros((self.n, k))
            for c in range(sd):  # sequential over the coordinates, like the reference
                diff = xs[:, c:c + 1] - cb[m][None, :, c]
                d2 = d2 + diff * diff
            best = np.argmin(d2, axis=1).astype(np.uint32)  # first index wins
            ch[m] = int((best != self.codes[:, m]).sum())
            self.codes[:, m] = best
            losses[m] = 1.0 * d2[np.arange(self.n), best]
        return torch.from_numpy(losses), ch

    def point_losses(self):
        return torch.from_numpy(self.port.pq_point_losses(
            self.x, self.cb, self.M, self.k, self.sd, self.hp, self.ho, self.codes))

    def seq_sum(self, v):
        a = v.numpy()
        return float(np.add.accumulate(a)[-1]) if a.size else 0.0

    def seq_sums(self, losses, active):
        return [self.seq_sum(losses[m]) if active[m] else 0.0 for m in range(losses.shape[0])]

    def ranking(self, losses, top):
        v = losses.numpy()
        idx = np.arange(v.size)
        o = np.lexsort((idx, -v))[:top]
        return torch.from_numpy(v[o].copy()), torch.from_numpy(o.astype(np.int64))

    def weight_flags(self):
        an = self.hp != self.ho
        z = np.nonzero(an & (self.norms * self.norms == 0.0))[0]
        return bool(an.any()), (int(z[0]) if z.size else None)

    def _slot_sums(self, wnum, wden, k, active=None):
        M, sd = self.codes.shape[1], self.d // self.codes.shape[1]
        num = np.zeros((M, k, sd))
        den = np.zeros((M, k))
        cnt = np.zeros((M, k), np.int64)
        for m in range(M):
            if active is not None and not active[m]:
                continue
            j = self.codes[:, m].astype(np.int64)
            for c in range(sd):
                np.add.at(num[m, :, c], j, wnum * self.x[:, m * sd + c])
            np.add.at(den[m], j, wden)
            np.add.at(cnt[m], j, 1)
        return (torch.from_numpy(num.reshape(-1)), torch.from_numpy(den.reshape(-1)),
                torch.from_numpy(cnt.reshape(-1)))

    def kmeans_partials(self, active):
        one = np.ones(self.n)
        return self._slot_sums(one, one, self.k, active)

    def iso_partials(self, k):
        return self._slot_sums(self.hp, self.ho, k)

    def normal_equations(self, k):
        M = self.codes.shape[1]
        if self.n:
            A, rhs = self.port.assemble_selector_system(self.x, self.codes, self.hp, self.ho, M, k)
        else:
            A, rhs = np.zeros((k * self.d, k * self.d)), np.zeros(k * self.d)
        usage = np.zeros((M, k), np.int64)
        for m in range(M):
            np.add.at(usage[m], self.codes[:, m].astype(np.int64), 1)
        return torch.from_numpy(A), torch.from_numpy(rhs), torch.from_numpy(usage.reshape(-1))

    def solve(self, A, rhs, ridge):
        A = A.numpy().copy()
        dim = A.shape[0]
        if ridge < 0.0:
            tr = 0.0
            for i in range(dim):
                tr = tr + A[i, i]
            ridge = (1e-6 * tr) / dim
        for i in range(dim):
            A[i, i] = A[i, i] + ridge
        return torch.from_numpy(self.port.llt_solve(A, rhs.numpy()))
