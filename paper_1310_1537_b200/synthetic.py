"""Seeded synthetic inputs with the BASELINE configs' shapes and distributions.

These stand in for data (the reference's benchmarks are synthetic too,
glm.py:578-591, hb.py:89-107).  Every draw comes from one
`np.random.default_rng(seed)` in a fixed order, and row-chunked generation is
stream-identical to a single call, so large N is produced in chunks.
"""

from __future__ import annotations

import numpy as np
from scipy.special import expit

__all__ = ["baseline_design", "hb_design", "ising_spins", "potts_states"]


def baseline_design(n: int, k: int, seed: int = 0, intercept: bool = True, n_eval: int = 1,
                    chunk_rows: int | None = None, x_dtype=np.float64):
    """Configs 0-2: X[:,0]=1, X[:,1:]~N(0,1); beta_true~N(0,0.5^2); y~Bern(sigmoid(X beta_true));
    beta_eval~N(0,0.1^2) (n_eval rows).  Returns (x, y, beta_true, beta_eval)."""
    gen = np.random.default_rng(seed)
    x = np.empty((n, k), dtype=x_dtype)
    kz = k - 1 if intercept else k
    step = chunk_rows or max(1, (1 << 24) // max(kz, 1))
    for a in range(0, n, step):
        b = min(n, a + step)
        block = gen.standard_normal((b - a, kz))
        if intercept:
            x[a:b, 0] = 1.0
            x[a:b, 1:] = block
        else:
            x[a:b] = block
    beta_true = gen.normal(0.0, 0.5, k)
    u = gen.random(n)
    y = np.empty(n)
    for a in range(0, n, step):
        b = min(n, a + step)
        y[a:b] = (u[a:b] < expit(np.asarray(x[a:b], dtype=np.float64) @ beta_true)).astype(np.float64)
    beta_eval = gen.normal(0.0, 0.1, (n_eval, k)) if n_eval > 1 else gen.normal(0.0, 0.1, k)
    return x, y, beta_true, beta_eval


def baseline_design_rows(n: int, k: int, seed: int, row0: int, row1: int, n_eval: int = 1):
    """Rows [row0, row1) of baseline_design(n, k, seed, n_eval=n_eval) -- bit-identical (the
    generator stream is consumed chunk by chunk exactly as there; rows outside the range are
    drawn and dropped), holding only the requested rows in memory.  One rank's shard of
    the one global design."""
    gen = np.random.default_rng(seed)
    kz = k - 1
    step = max(1, (1 << 24) // max(kz, 1))
    x = np.empty((row1 - row0, k))
    for a in range(0, n, step):
        b = min(n, a + step)
        block = gen.standard_normal((b - a, kz))
        lo, hi = max(a, row0), min(b, row1)
        if lo < hi:
            x[lo - row0:hi - row0, 0] = 1.0
            x[lo - row0:hi - row0, 1:] = block[lo - a:hi - a]
    beta_true = gen.normal(0.0, 0.5, k)
    u = gen.random(n)[row0:row1]
    y = np.empty(row1 - row0)
    for a in range(0, row1 - row0, step):
        b = min(row1 - row0, a + step)
        y[a:b] = (u[a:b] < expit(x[a:b] @ beta_true)).astype(np.float64)
    beta_eval = gen.normal(0.0, 0.1, (n_eval, k)) if n_eval > 1 else gen.normal(0.0, 0.1, k)
    return x, y, beta_true, beta_eval


def hb_design(n_groups: int, k: int, seed: int = 0, mean_rows: int = 2000, tau: float = 0.3):
    """Config 3: n_g~Poisson(mean_rows) (>=1); mu~N(0,0.5^2); beta_g~N(mu,tau^2 I); X~N(0,1);
    y_g~Bern(sigmoid(X_g beta_g)); the evaluation point is a fresh beta_g~N(mu,tau^2 I).
    Returns (x, y, offsets, betas_eval, mu, tau)."""
    gen = np.random.default_rng(seed)
    rows = np.maximum(gen.poisson(mean_rows, n_groups), 1).astype(np.int64)
    mu = gen.normal(0.0, 0.5, k)
    betas_true = mu + tau * gen.standard_normal((n_groups, k))
    offsets = np.zeros(n_groups + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(rows)
    x = gen.standard_normal((int(offsets[-1]), k))
    u = gen.random(int(offsets[-1]))
    y = np.empty(int(offsets[-1]))
    for g in range(n_groups):
        a, b = offsets[g], offsets[g + 1]
        y[a:b] = (u[a:b] < expit(x[a:b] @ betas_true[g])).astype(np.float64)
    betas_eval = mu + tau * gen.standard_normal((n_groups, k))
    return x, y, offsets, betas_eval, mu, tau


def ising_spins(height: int, width: int, seed: int = 0) -> np.ndarray:
    """Config 4 initial state: iid uniform +-1 int8."""
    gen = np.random.default_rng(seed)
    return (gen.integers(0, 2, size=(height, width), dtype=np.int8) * 2 - 1).astype(np.int8)


def potts_states(height: int, width: int, seed: int = 0) -> np.ndarray:
    """Potts q=4 initial state: iid uniform 0..3 int8."""
    gen = np.random.default_rng(seed)
    return gen.integers(0, 4, size=(height, width), dtype=np.int8)
