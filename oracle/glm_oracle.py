"""CPU oracle for the logistic-GLM hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker or the timed CPU
baseline; the product (paper_1310_1537_b200/) never calls it.

A numpy restatement of the reference's algorithm, each function citing the
reference file:line it follows (/root/reference/pkg/src/parmcmc/...).  Pinned
against fixtures generated from the unmodified reference (tests/golden/,
made by tests/golden/make_golden.py) in tests/test_oracle.py.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.special import expit

_pools: dict[int, ThreadPoolExecutor] = {}


def partition(n: int, workers: int) -> list[tuple[int, int]]:
    """parallel.py:30-46: contiguous blocks, the first n % workers take one extra row."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    base, extra = divmod(n, workers)
    out, start = [], 0
    for w in range(workers):
        size = base + (1 if w < extra else 0)
        out.append((start, start + size))
        start += size
    return out


def _run(tasks):
    """parallel.py:66-73: one region, results in task order (threads release the GIL in numpy)."""
    if len(tasks) == 1:
        return [tasks[0]()]
    pool = _pools.get(len(tasks))
    if pool is None:
        pool = _pools[len(tasks)] = ThreadPoolExecutor(max_workers=len(tasks))
    futs = [pool.submit(t) for t in tasks]
    return [f.result() for f in futs]


def nll_sum(t: np.ndarray, y: np.ndarray) -> float:
    """glm.py:179-192 `_nll_sum`: -(sum t - y.t + 0.5(sum|t| - sum t) + sum log1p(exp(-|t|)))."""
    a = np.abs(t)
    s_abs = a.sum()
    np.negative(a, out=a)
    np.exp(a, out=a)
    np.log1p(a, out=a)
    s_t = t.sum()
    return -(s_t - np.dot(y, t) + 0.5 * (s_abs - s_t) + a.sum())


def block_fg(x: np.ndarray, y: np.ndarray, beta: np.ndarray):
    """glm.py:367-372 `_block_fg`: t = x@beta; f = _nll_sum; gf = y - expit(t); g = x.T@gf."""
    t = x @ beta
    f = nll_sum(t, y)
    gf = y - expit(t)
    return f, x.T @ gf


def loglike_grad(x, y, beta, workers: int = 1):
    """glm.py:418-436 `_grad_plf` + glm.py:243-250 `_merge_grad` (ascending worker order)."""
    beta = np.ascontiguousarray(beta, dtype=np.float64)

    def task(a, b):
        def run():
            if b <= a:
                return 0.0, np.zeros(x.shape[1])
            return block_fg(x[a:b], y[a:b], beta)
        return run

    parts = _run([task(a, b) for a, b in partition(x.shape[0], workers)])
    f, g = 0.0, np.zeros(x.shape[1])
    for pf, pg in parts:
        f += pf
        g += pg
    return f, g


def loglike(x, y, beta, workers: int = 1) -> float:
    """glm.py:314-329 `_loglike_plf` + glm.py:234-240 `_merge_scalar`."""
    beta = np.ascontiguousarray(beta, dtype=np.float64)

    def task(a, b):
        def run():
            return nll_sum(x[a:b] @ beta, y[a:b]) if b > a else 0.0
        return run

    acc = 0.0
    for p in _run([task(a, b) for a, b in partition(x.shape[0], workers)]):
        acc += p
    return acc


def prior_terms(beta, mu, sigma):
    """sampler.py:55-58 summed over k ascending, and the implied gradient -(beta-mu)/sigma^2."""
    f = 0.0
    for k in range(beta.size):
        z = (beta[k] - mu[k]) / sigma[k]
        f += -0.5 * z * z
    g = -(beta - mu) / (sigma * sigma)
    return f, g


def log_posterior_grad(x, y, beta, mu, sigma, workers: int = 1):
    """loglike_grad (glm.py:351) + sum_k GaussianPrior.logpdf_coord (sampler.py:55-58)."""
    f, g = loglike_grad(x, y, beta, workers)
    pf, pg = prior_terms(np.asarray(beta, dtype=np.float64), np.asarray(mu, dtype=np.float64),
                         np.asarray(sigma, dtype=np.float64))
    return f + pf, g + pg


def naive_loglike(x, y, beta) -> float:
    """tests/naive.py:16-29: scalar double loop (small inputs only)."""
    total = 0.0
    for n in range(x.shape[0]):
        t = 0.0
        for k in range(x.shape[1]):
            t += float(x[n, k]) * float(beta[k])
        lse = math.log1p(math.exp(-t)) if t >= 0 else -t + math.log1p(math.exp(t))
        total -= (1.0 - float(y[n])) * t + lse
    return total


def naive_grad(x, y, beta) -> np.ndarray:
    """tests/naive.py:32-47."""
    g = np.zeros(x.shape[1])
    for n in range(x.shape[0]):
        t = 0.0
        for k in range(x.shape[1]):
            t += float(x[n, k]) * float(beta[k])
        if t >= 0:
            p = 1.0 / (1.0 + math.exp(-t))
        else:
            e = math.exp(t)
            p = e / (1.0 + e)
        for k in range(x.shape[1]):
            g[k] += (float(y[n]) - p) * float(x[n, k])
    return g


def diff_loglike(xbeta, xk, y, delta, workers: int = 1) -> float:
    """glm.py:499-522: _nll_sum(xbeta + delta*xt[k], y) over the row partition."""
    def task(a, b):
        def run():
            return nll_sum(xbeta[a:b] + delta * xk[a:b], y[a:b]) if b > a else 0.0
        return run

    acc = 0.0
    for p in _run([task(a, b) for a, b in partition(xbeta.size, workers)]):
        acc += p
    return acc


def commit(xbeta, xk, delta) -> None:
    """glm.py:536-537: xbeta += delta * xt[k] (in place)."""
    if delta != 0.0:
        xbeta += delta * xk


def hb_log_posterior_grad(x, y, offsets, betas, mu=None, sigma=None):
    """hb.py:64-86/127-135: per-group loglike_grad + shared GaussianPrior (sampler.py:55-58)."""
    G = offsets.size - 1
    fs = np.empty(G)
    gs = np.empty((G, x.shape[1]))
    for g in range(G):
        a, b = int(offsets[g]), int(offsets[g + 1])
        f, gr = loglike_grad(x[a:b], y[a:b], betas[g])
        if mu is not None:
            pf, pg = prior_terms(betas[g], mu, sigma)
            f, gr = f + pf, gr + pg
        fs[g], gs[g] = f, gr
    return fs, gs
