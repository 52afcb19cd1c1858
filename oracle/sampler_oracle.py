"""CPU oracle for the slice-within-Gibbs chain (config 2) -- TEST INFRASTRUCTURE ONLY.

Only tests/ and bench.py's cpu_baseline leg may use it (as the checker / timed CPU
baseline).  A numpy restatement of the reference sampler:

  GaussianPrior.logpdf_coord   sampler.py:55-58
  log_posterior_coord          sampler.py:92-106 (diff path: glm.py:499-522)
  slice_sample_coord           sampler.py:112-167 (stepping-out + shrinkage, uniform order)
  run_chain                    sampler.py:170-200 (start at the prior mean, systematic scan)
  commit_update                glm.py:525-539
  DeviateBuffer UNIFORM01      rng.py:59-138 (numpy Philox(SeedSequence(seed)), capacity-invariant)

Pinned against the reference chain fixture (tests/golden/sampler.npz) in tests/test_oracle.py.
"""

from __future__ import annotations

import math

import numpy as np

from . import glm_oracle as gl

_MAX_SHRINK = 1000


class SliceWidenError(RuntimeError):
    pass


class UniformStream:
    """The DeviateBuffer UNIFORM01 stream: numpy Philox seeded by SeedSequence(seed, owner)."""

    def __init__(self, seed: int = 0, owner=(), block: int = 8192):
        self._gen = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=tuple(owner))))
        self._block = block
        self._buf = np.empty(0)
        self._i = 0

    def next(self) -> float:
        if self._i == self._buf.size:
            self._buf = self._gen.random(self._block)
            self._i = 0
        v = float(self._buf[self._i])
        self._i += 1
        return v


def run_chain(x, y, mu, sigma, n_iter, n_burnin=0, seed=0, slice_width=1.0, slice_max_steps=50,
              workers: int = 1, rng=None, beta0=None):
    """Returns (draws[n_iter-n_burnin, K], evals); the chain starts at beta0 (default mu)."""
    n, k = x.shape
    mu = np.asarray(mu, dtype=np.float64)
    sigma = np.asarray(sigma, dtype=np.float64)
    rng = rng if rng is not None else UniformStream(seed)
    beta = mu.copy() if beta0 is None else np.array(beta0, dtype=np.float64)
    xbeta = x @ beta                 # GlmWorkspace, glm.py:472
    xt = np.ascontiguousarray(x.T)   # glm.py:473
    evals = 0
    draws = np.empty((n_iter - n_burnin, k))

    def logprior(j, v):
        z = (v - mu[j]) / sigma[j]
        return -0.5 * z * z

    for it in range(n_iter):
        for j in range(k):
            x0 = float(beta[j])

            def logpost(xv):
                nonlocal evals
                evals += 1
                d = xv - x0
                return gl.diff_loglike(xbeta, xt[j], y, d, workers) + logprior(j, beta[j] + d)

            f0 = logpost(x0)
            level = f0 + math.log(1.0 - rng.next())
            width = slice_width
            r = rng.next()
            left = x0 - r * width
            right = left + width
            steps = 0
            while logpost(left) > level:
                left -= width
                steps += 1
                if steps > slice_max_steps:
                    raise SliceWidenError(j)
            steps = 0
            while logpost(right) > level:
                right += width
                steps += 1
                if steps > slice_max_steps:
                    raise SliceWidenError(j)
            for _ in range(_MAX_SHRINK):
                x1 = left + rng.next() * (right - left)
                if logpost(x1) > level:
                    break
                if x1 < x0:
                    left = x1
                else:
                    right = x1
                if right - left < 1e-12 * (1.0 + abs(x0)):
                    x1 = x0
                    break
            else:
                raise RuntimeError(j)
            gl.commit(xbeta, xt[j], x1 - x0)
            beta[j] += x1 - x0
        if it >= n_burnin:
            draws[it - n_burnin] = beta
    return draws, evals
