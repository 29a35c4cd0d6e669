"""Shared fixtures for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np

from paper_1908_10396_b200 import workload as wl


def lognormal_rows(n: int, d: int, seed: int, sigma: float = 0.5) -> np.ndarray:
    """Config-3 distribution: directions uniform on the sphere, lognormal norms."""
    g = np.random.Generator(np.random.PCG64([seed, 77]))
    x = g.standard_normal((n, d))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    x *= np.exp(sigma * g.standard_normal(n))[:, None]
    return x.astype(np.float32)


def mixture_rows(n: int, d: int, seed: int, centers: int = 16, sigma: float = 0.3,
                 normalize: bool = True) -> np.ndarray:
    return wl.gaussian_mixture(n, d, centers, sigma, seed, 5, normalize=normalize)


def random_codebook(M: int, k: int, sd: int, seed: int, scale: float = 0.25) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64([seed, 99]))
    return g.standard_normal(M * k * sd) * scale


def threshold_hp_ho(x: np.ndarray, t: float, policy: int = 1):
    """CLI resolve_weights per point (anisoq_main.cpp:127-133) with the
    |x| <= T policy; computed by the oracle port."""
    from oracle import Port

    P = Port()
    norms = P.row_norms(np.asarray(x, np.float64))
    return P.threshold_weights(norms, x.shape[1], t, policy)
