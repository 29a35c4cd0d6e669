"""Seeded synthetic workloads for BASELINE.json configs 1-5.

GloVe-1.2M and the paper's datasets are not available here, so these
generators stand in for them with the shapes, sizes and distributions the
configs name. All values are rounded to float32 after generation, so the
device (float32 rows) and the float64 oracle consume identical numbers
(as the reference's own generator does, dataset.hpp:288). Streams come from
numpy's PCG64 with one documented sub-stream per array.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

T_DEFAULT = 0.2


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed, stream]))


def _normalize_rows(x: np.ndarray) -> np.ndarray:
    n = np.sqrt(np.einsum("ij,ij->i", x, x))
    n[n == 0] = 1.0
    return x / n[:, None]


def gaussian_mixture(n: int, d: int, centers: int, sigma: float, seed: int, stream: int,
                     weights: Optional[np.ndarray] = None, normalize: bool = True,
                     means: Optional[np.ndarray] = None, chunk: int = 1 << 20) -> np.ndarray:
    """Mixture of isotropic Gaussians: means ~ N(0, I_d), per-coordinate sigma."""
    if means is None:
        means = _rng(seed, 1000 + stream).standard_normal((centers, d))
    g = _rng(seed, stream)
    out = np.empty((n, d), np.float32)
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        if weights is None:
            comp = g.integers(0, centers, e - b)
        else:
            comp = g.choice(centers, size=e - b, p=weights)
        x = means[comp] + sigma * g.standard_normal((e - b, d))
        if normalize:
            x = _normalize_rows(x)
        out[b:e] = x.astype(np.float32)
    return out


def zipf_weights(centers: int, s: float) -> np.ndarray:
    p = np.arange(1, centers + 1, dtype=np.float64) ** (-s)
    return p / p.sum()


@dataclass
class Workload:
    name: str
    base: Optional[np.ndarray]
    queries: Optional[np.ndarray]
    M: int
    k: int
    threshold: float
    iterations: int = 0
    passes: int = 0
    codebook: Optional[np.ndarray] = None  # fixed codebooks (configs 3, 4)
    packed_codes: Optional[np.ndarray] = None  # config 4
    n: int = 0

    @property
    def d(self) -> int:
        if self.base is not None:
            return self.base.shape[1]
        return self.queries.shape[1]


def config1(n: int = 20_000, nq: int = 100, seed: int = 0) -> Workload:
    """64-component mixture, sigma 0.3, d 32, L2-normalised; M 16, T 0.2, 10 iters."""
    means = _rng(seed, 1000).standard_normal((64, 32))
    base = gaussian_mixture(n, 32, 64, 0.3, seed, 1, means=means)
    q = gaussian_mixture(nq, 32, 64, 0.3, seed, 2, means=means)
    return Workload("config1", base, q, 16, 16, T_DEFAULT, iterations=10, n=n)


def config2(n: int = 1_183_514, nq: int = 10_000, seed: int = 0, shard: int = 0) -> Workload:
    """1000-component mixture, sigma 0.5, Zipf(1.1) weights, d 100, normalised; M 50.

    `shard` > 0 draws other rows of the same distribution (row shards of one
    dataset on several GPUs); the queries are the same for every shard."""
    means = _rng(seed, 1000).standard_normal((1000, 100))
    w = zipf_weights(1000, 1.1)
    base = gaussian_mixture(n, 100, 1000, 0.5, seed, 1 if shard == 0 else 10_000 + shard,
                            weights=w, means=means)
    q = gaussian_mixture(nq, 100, 1000, 0.5, seed, 2, weights=w, means=means)
    return Workload("config2", base, q, 50, 16, T_DEFAULT, iterations=10, n=n)


def config3(n: int = 10_000_000, seed: int = 0, chunk: int = 1 << 20) -> Workload:
    """Directions uniform on S^127, norms lognormal(0, 0.5); fixed codebook
    64 x 16 x 2 ~ N(0, 1/128); 3 CD sweeps."""
    d = 128
    g = _rng(seed, 1)
    base = np.empty((n, d), np.float32)
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        x = _normalize_rows(g.standard_normal((e - b, d)))
        r = np.exp(0.5 * g.standard_normal(e - b))
        base[b:e] = (x * r[:, None]).astype(np.float32)
    cb = _rng(seed, 3).standard_normal(64 * 16 * 2) / np.sqrt(d)
    return Workload("config3", base, None, 64, 16, T_DEFAULT, passes=3, codebook=cb, n=n)


def config4(n: int = 100_000_000, nq: int = 4096, seed: int = 0,
            chunk: int = 1 << 22) -> Workload:
    """Uniform random 4-bit codes (M 48), codebook ~ N(0, 1/96), 4096 unit queries."""
    M, d = 48, 96
    g = _rng(seed, 4)
    packed = np.empty((n, M // 2), np.uint8)
    for b in range(0, n, chunk):
        e = min(n, b + chunk)
        packed[b:e] = g.integers(0, 256, (e - b, M // 2), dtype=np.uint8)
    cb = _rng(seed, 3).standard_normal(M * 16 * 2) / np.sqrt(d)
    q = _normalize_rows(_rng(seed, 2).standard_normal((nq, d))).astype(np.float32)
    return Workload("config4", None, q, M, 16, T_DEFAULT, codebook=cb,
                    packed_codes=packed, n=n)


def config5(n: int = 10_000_000, seed: int = 0) -> Workload:
    """4096-component mixture, sigma 0.4, d 256, normalised; M 128, 20 iterations."""
    means = _rng(seed, 1000).standard_normal((4096, 256))
    base = gaussian_mixture(n, 256, 4096, 0.4, seed, 1, means=means)
    return Workload("config5", base, None, 128, 16, T_DEFAULT, iterations=20, n=n)


def unpack_codes(packed: np.ndarray, M: int) -> np.ndarray:
    """4-bit packed rows (low nibble = even m) -> n x M uint32."""
    lo = packed & 15
    hi = packed >> 4
    out = np.empty((packed.shape[0], 2 * packed.shape[1]), np.uint32)
    out[:, 0::2] = lo
    out[:, 1::2] = hi
    return out[:, :M]


def pack_codes(codes: np.ndarray, row_bytes: Optional[int] = None) -> np.ndarray:
    codes = np.asarray(codes, np.uint8)
    n, M = codes.shape
    rb = row_bytes or ((M + 1) // 2 + 7) // 8 * 8
    out = np.zeros((n, rb), np.uint8)
    c = np.zeros((n, 2 * ((M + 1) // 2)), np.uint8)
    c[:, :M] = codes
    out[:, : c.shape[1] // 2] = c[:, 0::2] | (c[:, 1::2] << 4)
    return out
