"""ctypes wrapper of oracle/gibbs_oracle.c -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
it, as the checker / timed CPU baseline.  See gibbs_oracle.c for the reference
citations.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_int8, c_uint32, c_uint64

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libgibbs_oracle.so")
RNG_UNIFORMS, RNG_NUMPY_PHILOX, RNG_PHILOX4X32 = 0, 1, 2
_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", HERE], check=True, capture_output=True)
    lib = ctypes.CDLL(LIB)
    lib.oracle_philox4x64_10.argtypes = [POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64)]
    lib.oracle_philox4x32_10.argtypes = [POINTER(c_uint32), POINTER(c_uint32), POINTER(c_uint32)]
    lib.oracle_numpy_word.restype = c_uint64
    lib.oracle_numpy_word.argtypes = [c_uint64, c_uint64, c_uint64]
    lib.oracle_numpy_uniform.restype = c_double
    lib.oracle_numpy_uniform.argtypes = [c_uint64, c_uint64, c_uint64]
    lib.oracle_site_uniform.restype = c_double
    lib.oracle_site_uniform.argtypes = [c_uint64, c_uint64, c_uint64]
    lib.oracle_expit.restype = c_double
    lib.oracle_expit.argtypes = [c_double]
    lib.oracle_ising_sweeps.argtypes = [POINTER(c_int8), POINTER(c_double), c_int, c_int, c_double, c_int,
                                        c_int, c_int, c_uint64, c_uint64, c_uint64, POINTER(c_double)]
    lib.oracle_potts_sweeps.argtypes = [POINTER(c_int8), c_int, c_int, c_double, c_int, c_int, c_int,
                                        c_uint64, c_uint64, c_uint64, POINTER(c_double)]
    lib.oracle_potts_cdf.argtypes = [c_double, POINTER(c_int), POINTER(c_double)]
    _lib = lib
    return lib


def philox4x64(ctr, key) -> np.ndarray:
    c = (c_uint64 * 4)(*[int(v) for v in ctr])
    k = (c_uint64 * 2)(*[int(v) for v in key])
    o = (c_uint64 * 4)()
    load().oracle_philox4x64_10(c, k, o)
    return np.array(list(o), dtype=np.uint64)


def philox4x32(ctr, key) -> np.ndarray:
    c = (c_uint32 * 4)(*[int(v) for v in ctr])
    k = (c_uint32 * 2)(*[int(v) for v in key])
    o = (c_uint32 * 4)()
    load().oracle_philox4x32_10(c, k, o)
    return np.array(list(o), dtype=np.uint32)


def numpy_uniforms(key0: int, key1: int, start: int, n: int) -> np.ndarray:
    lib = load()
    return np.array([lib.oracle_numpy_uniform(start + i, key0, key1) for i in range(n)])


def site_uniforms(seed: int, sweep: int, n_sites: int) -> np.ndarray:
    """All uniforms of one sweep in stream order (colour 0 packed, then colour 1)."""
    lib = load()
    return np.array([lib.oracle_site_uniform(s, sweep, seed) for s in range(n_sites)])


def _dp(a):
    return None if a is None else a.ctypes.data_as(POINTER(c_double))


def ising_sweeps(s, b, w, periodic, n_sweeps, mode, key0=0, key1=0, pos=0, uniforms=None) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.int8).copy()
    H, W = s.shape
    b = None if b is None else np.ascontiguousarray(b, dtype=np.float64).ravel()
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
    load().oracle_ising_sweeps(s.ctypes.data_as(POINTER(c_int8)), _dp(b), H, W, float(w), int(periodic),
                               int(n_sweeps), int(mode), c_uint64(key0), c_uint64(key1), c_uint64(pos), _dp(u))
    return s


def potts_sweeps(s, coupling, periodic, n_sweeps, mode, key0=0, key1=0, pos=0, uniforms=None) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.int8).copy()
    H, W = s.shape
    u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
    load().oracle_potts_sweeps(s.ctypes.data_as(POINTER(c_int8)), H, W, float(coupling), int(periodic),
                               int(n_sweeps), int(mode), c_uint64(key0), c_uint64(key1), c_uint64(pos), _dp(u))
    return s


def potts_cdf(coupling: float, counts) -> np.ndarray:
    n = (c_int * 4)(*[int(v) for v in counts])
    out = (c_double * 3)()
    load().oracle_potts_cdf(float(coupling), n, out)
    return np.array(list(out))


def denoise(noisy01, w: float, bias_scale: float, sweeps: int, burnin: int, key0: int, key1: int):
    """CPU restatement of the reference denoiser (ising.py:257-290) on top of the
    oracle sweep: from_image spins/bias (ising.py:73-82), one free-boundary sweep
    at a time on the DeviateBuffer stream (H*W deviates per sweep), per-sweep
    flip counts (ising.py:283-284), sum of post-burn-in spins (ising.py:285-287)
    and the sign rule (acc >= 0, ties -> 1; kept == 0 -> input unchanged).
    Returns (restored uint8 image, flips int64[sweeps])."""
    img = np.asarray(noisy01)
    s = (2 * img.astype(np.int8) - 1).astype(np.int8)
    b = bias_scale * s.astype(np.float64)
    hw = s.size
    acc = np.zeros(s.shape, dtype=np.int64)
    flips = np.zeros(sweeps, dtype=np.int64)
    for t in range(sweeps):
        nxt = ising_sweeps(s, b, w, False, 1, RNG_NUMPY_PHILOX, key0, key1, t * hw)
        flips[t] = int(np.count_nonzero(nxt != s))
        s = nxt
        if t >= burnin:
            acc += s
    if sweeps - burnin <= 0:
        return img.astype(np.uint8).copy(), flips
    return (acc >= 0).astype(np.uint8), flips
