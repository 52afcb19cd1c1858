"""CPU restatement of the reference's batch-RNG samplers -- TEST INFRASTRUCTURE ONLY.

Only tests/ may use it, as the checker of the device samplers (include/pmb200.h
pm_rng_*).  Pinned against tests/golden/rng_batch.npz, which make_golden.py made
with the unmodified reference.

Streams are addressed by (Philox key, stream index), the device's view:
  * uniform i = numpy Philox4x64-10 output i, (w >> 11) * 2^-53 (rng.py:42-44, 86-90);
  * normal j = Box-Muller of uniform pair j // 2, cos for even j, sin for odd j
    (rng.py:47-56; the capacity-invariant order of the carry logic, rng.py:91-102).
Samplers follow rng.py:163-215 line by line (pure Python, small n).
"""

from __future__ import annotations

import math

import numpy as np

GAMMA_MAX_REJECT = 10_000  # rng.py:160


class DrainError(RuntimeError):
    pass


def _generator(key0: int, key1: int, pos: int) -> np.random.Generator:
    bg = np.random.Philox(key=np.array([key0, key1], dtype=np.uint64))
    st = bg.state
    ctr = np.zeros(4, dtype=np.uint64)
    ctr[0] = pos // 4
    st["state"]["counter"] = ctr
    st["buffer_pos"] = 4
    bg.state = st
    if pos % 4:
        bg.random_raw(pos % 4)
    return np.random.Generator(bg)


def uniforms(key0: int, key1: int, pos: int, n: int) -> np.ndarray:
    return _generator(key0, key1, pos).random(n)


def normals(key0: int, key1: int, pos: int, n: int) -> np.ndarray:
    """Normals pos .. pos+n-1 of the stream (rng.py:47-56)."""
    first = pos // 2
    pairs = (pos + n + 1) // 2 - first
    u = _generator(key0, key1, 2 * first).random((pairs, 2))
    r = np.sqrt(-2.0 * np.log1p(-u[:, 0]))
    th = (2.0 * np.pi) * u[:, 1]
    z = np.empty(2 * pairs)
    z[0::2] = r * np.cos(th)
    z[1::2] = r * np.sin(th)
    off = pos - 2 * first
    return z[off:off + n]


class _Src:
    """Sequential source over a stream from a start index (uniform or normal)."""

    def __init__(self, key, pos: int, normal: bool):
        self.k0, self.k1 = int(key[0]), int(key[1])
        self.pos = int(pos)
        self.normal = normal
        self._cache = np.empty(0)
        self._base = self.pos

    def next(self) -> float:
        i = self.pos - self._base
        if i >= self._cache.size:
            self._base = self.pos
            fn = normals if self.normal else uniforms
            self._cache = fn(self.k0, self.k1, self.pos, 256)
            i = 0
        self.pos += 1
        return float(self._cache[i])


def _gamma_std(alpha: float, u: _Src, z: _Src) -> float:
    """Marsaglia-Tsang squeeze rejection, alpha >= 1 (rng.py:163-178)."""
    d = alpha - 1.0 / 3.0
    c = 1.0 / math.sqrt(9.0 * d)
    for _ in range(GAMMA_MAX_REJECT):
        x = z.next()
        v = 1.0 + c * x
        if v <= 0.0:
            continue
        v = v * v * v
        uu = u.next()
        x2 = x * x
        if uu < 1.0 - 0.0331 * x2 * x2:
            return d * v
        if math.log(uu) < 0.5 * x2 + d * (1.0 - v + math.log(v)):
            return d * v
    raise DrainError("gamma rejection drained")


def _gamma_shape(alpha: float, u: _Src, z: _Src) -> float:
    """alpha < 1 boosted through Gamma(alpha+1) * U**(1/alpha) (rng.py:181-188)."""
    if alpha < 1.0:
        y = _gamma_std(alpha + 1.0, u, z)
        return y * u.next() ** (1.0 / alpha)
    return _gamma_std(alpha, u, z)


def gamma_draws(alpha, rate, n, ukey, upos, nkey, npos):
    """n sequential gamma_sample calls (rng.py:191-198) -> (draws, upos_end, npos_end)."""
    u, z = _Src(ukey, upos, False), _Src(nkey, npos, True)
    out = np.array([_gamma_shape(alpha, u, z) / rate for _ in range(n)])
    return out, u.pos, z.pos


def dirichlet_draws(alphas, n, ukey, upos, nkey, npos):
    """n sequential dirichlet_sample calls (rng.py:201-215) -> (draws[n, K], upos_end, npos_end)."""
    alphas = np.asarray(alphas, dtype=float)
    u, z = _Src(ukey, upos, False), _Src(nkey, npos, True)
    out = np.empty((n, alphas.size))
    for i in range(n):
        for _ in range(2):
            y = np.array([_gamma_shape(float(a), u, z) for a in alphas])
            total = y.sum()
            if total > 0.0:
                out[i] = y / total
                break
        else:
            raise DrainError("dirichlet underflow")
    return out, u.pos, z.pos
