"""Uniform deviate streams consumed by the hot paths.

`DeviateBuffer` mirrors the reference's buffered Philox stream (rng.py:59-138)
with the exact stream contract: deviate i of a (seed, owner) stream is the i-th
output of numpy's Philox4x64-10 seeded by SeedSequence(seed, spawn_key=owner)
(rng.py:42-44), independent of buffer capacity.  The sampler's scalar control
flow consumes it on the host exactly as the reference does (sampler.py:131-153).

For the Gibbs kernels the stream is generated *on the device*: the kernel needs
only the Philox key and the stream position (`stream_key`, `position`), and the
buffer is then advanced past the consumed deviates with `skip` (O(1)).

`SitePhilox` is the (seed, sweep, site)-keyed Philox4x32-10 stream of BASELINE
config 4 (include/pmb200.h PM_RNG_PHILOX4X32); `site_uniforms` materialises
the uniforms of a sweep on the host for cross-checking.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import RngDrainError

__all__ = ["BufferKind", "DeviateBuffer", "SitePhilox", "philox_key_of", "RngDrainError", "GammaParams",
           "OneAtATimeUniform", "OneAtATimeNormal", "gamma_sample", "dirichlet_sample", "gamma_batch",
           "dirichlet_batch", "gamma_streams", "dirichlet_streams", "BenchDist", "BenchMode", "RngBenchRecord",
           "rng_bench", "write_rng_bench_csv"]


class BufferKind(Enum):
    UNIFORM01 = "uniform01"
    STD_NORMAL = "std_normal"


def _make_generator(seed: int, owner: Sequence[int]) -> np.random.Generator:
    ss = np.random.SeedSequence(seed, spawn_key=tuple(owner))
    return np.random.Generator(np.random.Philox(ss))


def _box_muller_pairs(gen: np.random.Generator, n_pairs: int) -> np.ndarray:
    """2*n_pairs standard normals from n_pairs uniform pairs (rng.py:47-56)."""
    u = gen.random((n_pairs, 2))
    r = np.sqrt(-2.0 * np.log1p(-u[:, 0]))
    theta = (2.0 * np.pi) * u[:, 1]
    out = np.empty(2 * n_pairs)
    out[0::2] = r * np.cos(theta)
    out[1::2] = r * np.sin(theta)
    return out


def _seek(gen: np.random.Generator, target: int) -> None:
    """Position a numpy Philox generator so its next output is stream word `target`."""
    bg = gen.bit_generator
    st = bg.state
    ctr = np.zeros(4, dtype=np.uint64)
    ctr[0] = target // 4          # numpy pre-increments before generating a block
    st["state"]["counter"] = ctr
    st["buffer_pos"] = 4
    st["has_uint32"] = 0
    bg.state = st
    if target % 4:
        bg.random_raw(target % 4)


def philox_key_of(gen_or_bitgen) -> tuple[int, int]:
    """The (key0, key1) of a numpy Philox generator, as the device kernels take it."""
    bg = getattr(gen_or_bitgen, "bit_generator", gen_or_bitgen)
    st = bg.state
    if st.get("bit_generator") != "Philox":
        raise TypeError("not a Philox bit generator")
    key = st["state"]["key"]
    return int(key[0]), int(key[1])


class DeviateBuffer:
    """Refillable block of pre-generated deviates with deterministic order (rng.py:59-138)."""

    def __init__(self, kind: BufferKind, capacity: int = 8192, seed: int = 0,
                 owner: Sequence[int] = ()):
        if capacity < 1:
            raise ValueError(f"capacity must be >= 1, got {capacity}")
        self.kind = kind
        self.capacity = int(capacity)
        self.data = np.empty(self.capacity)
        self.cursor = self.capacity
        self.refills = 0
        self.consumed = 0
        self._gen = _make_generator(seed, owner)
        self._carry: float | None = None
        self._gen_pos = 0                     # stream index of the generator's next output
        self._block_start = -self.capacity    # stream index of data[0] (no block yet)
        self._seek_to: int | None = None      # pending generator reposition (skip)

    def refill(self) -> None:
        """Fill data[0:capacity] with the next block of the base stream."""
        if self._seek_to is not None:
            self._apply_seek()
        self._block_start = self._gen_pos
        if self.kind is BufferKind.UNIFORM01:
            self.data[:] = self._gen.random(self.capacity)
            self._gen_pos += self.capacity
        else:
            pos = 0
            if self._carry is not None:
                self._block_start -= 1            # data[0] is the carried normal _gen_pos-1
                self.data[0] = self._carry
                self._carry = None
                pos = 1
            remaining = self.capacity - pos
            if remaining > 0:
                n_pairs = (remaining + 1) // 2
                block = _box_muller_pairs(self._gen, n_pairs)
                self.data[pos:] = block[:remaining]
                if 2 * n_pairs > remaining:
                    self._carry = float(block[remaining])
                self._gen_pos += 2 * n_pairs
        self.cursor = 0
        self.refills += 1

    def next(self) -> float:
        if self.cursor == self.capacity:
            self.refill()
        v = self.data[self.cursor]
        self.cursor += 1
        self.consumed += 1
        return float(v)

    def take(self, n: int) -> np.ndarray:
        out = np.empty(n)
        filled = 0
        while filled < n:
            if self.cursor == self.capacity:
                self.refill()
            m = min(n - filled, self.capacity - self.cursor)
            out[filled:filled + m] = self.data[self.cursor:self.cursor + m]
            self.cursor += m
            filled += m
        self.consumed += n
        return out

    @property
    def generated(self) -> int:
        """Deviates generated as the reference counts them (rng.py:129-138): a host consumer
        refills one block whenever it runs dry, so after `consumed` deviates it has filled
        ceil(consumed / capacity) blocks -- also when the device consumed them (skip)."""
        return max(self.refills, -(-self.consumed // self.capacity)) * self.capacity

    @property
    def waste_fraction(self) -> float:
        if self.generated == 0:
            return 0.0
        return (self.generated - self.consumed) / self.generated

    # ---- device-generation support -------------------------------------------------
    def stream_key(self) -> tuple[int, int]:
        """Philox key of this stream (for PM_RNG_NUMPY_PHILOX)."""
        return philox_key_of(self._gen)

    @property
    def position(self) -> int:
        """Stream index of the next deviate next()/take() would return."""
        return self._block_start + self.cursor

    def skip(self, n: int) -> None:
        """Advance past n deviates that were consumed elsewhere (on the device).

        Afterwards next()/take() continue exactly where n host calls would have left
        the stream (for STD_NORMAL including the carried sine half of a pair).
        """
        if n < 0:
            raise ValueError("n must be >= 0")
        if n == 0:
            return
        if n <= self.capacity - self.cursor:
            self.cursor += n
        else:
            # the generator is repositioned lazily, at the next refill (device paths skip
            # thousands of streams per call and most are never read on the host)
            target = self.position + n
            self._seek_to = target
            self._block_start = target - self.capacity
            self.cursor = self.capacity
        self.consumed += n

    def _apply_seek(self) -> None:
        target, self._seek_to = self._seek_to, None
        if self.kind is BufferKind.UNIFORM01:
            _seek(self._gen, target)
            self._carry = None
        else:
            # normal j is half of uniform pair j//2; an odd target starts on a carried sine
            _seek(self._gen, target - (target & 1))
            self._carry = float(_box_muller_pairs(self._gen, 1)[1]) if target & 1 else None
            target += target & 1
        self._gen_pos = target

    def take_device(self, n: int, device: int = 0) -> np.ndarray:
        """The next n deviates generated on the device (pm_rng_fill); advances the buffer
        exactly as take(n).  UNIFORM01 values are bit-identical to take(n); STD_NORMAL
        values agree to the rounding of CUDA's log1p/sincos (<= 2 ulp each)."""
        n = int(n)
        if n < 0:
            raise ValueError("n must be >= 0")
        out = np.empty(n)
        if n:
            k0, k1 = self.stream_key()
            kind = _lib.PM_RNG_KIND_UNIFORM01 if self.kind is BufferKind.UNIFORM01 else _lib.PM_RNG_KIND_STD_NORMAL
            _lib.require_device(device)
            _lib.call("pm_rng_fill", device, kind, ctypes.c_uint64(k0), ctypes.c_uint64(k1),
                      ctypes.c_uint64(self.position), n, out.ctypes.data, 0, None)
            self.skip(n)
        return out


class SitePhilox:
    """Philox4x32-10 keyed by (seed, sweep, site) (BASELINE config 4).

    Sweep t's uniform for stream site s (s = c*ceil(HW/2) + packed index) is
    word s%4 of Philox4x32_10(counter=(s/4 lo, s/4 hi, t lo, t hi),
    key=(seed lo, seed hi)) times 2^-32.  `sweep` is the next sweep number.
    """

    def __init__(self, seed: int = 0, sweep: int = 0):
        self.seed = int(seed) & ((1 << 64) - 1)
        self.sweep = int(sweep)

    def advance(self, n_sweeps: int) -> None:
        self.sweep += int(n_sweeps)


# ---------------------------------------------------------------------------------------
# per-call sources (rng.py:141-149 / 152-171 of the reference), positionable so the device
# samplers can consume them and hand them back advanced
# ---------------------------------------------------------------------------------------
class OneAtATimeUniform:
    """Per-call uniforms on the same stream as a UNIFORM01 buffer (rng.py:141-149)."""

    kind = BufferKind.UNIFORM01

    def __init__(self, seed: int = 0, owner: Sequence[int] = ()):
        self._gen = _make_generator(seed, owner)
        self.position = 0

    def next(self) -> float:
        self.position += 1
        return float(self._gen.random())

    def stream_key(self) -> tuple[int, int]:
        return philox_key_of(self._gen)

    def skip(self, n: int) -> None:
        self.position += int(n)
        _seek(self._gen, self.position)


class OneAtATimeNormal:
    """Per-call Box-Muller on the same stream as a STD_NORMAL buffer (rng.py:152-171)."""

    kind = BufferKind.STD_NORMAL

    def __init__(self, seed: int = 0, owner: Sequence[int] = ()):
        self._gen = _make_generator(seed, owner)
        self._carry: float | None = None
        self.position = 0

    def next(self) -> float:
        self.position += 1
        if self._carry is not None:
            v, self._carry = self._carry, None
            return v
        block = _box_muller_pairs(self._gen, 1)
        self._carry = float(block[1])
        return float(block[0])

    def stream_key(self) -> tuple[int, int]:
        return philox_key_of(self._gen)

    def skip(self, n: int) -> None:
        self.position += int(n)
        j = self.position
        _seek(self._gen, j - (j & 1))
        self._carry = float(_box_muller_pairs(self._gen, 1)[1]) if j & 1 else None


# ---------------------------------------------------------------------------------------
# Gamma / Dirichlet on the device (rng.py:152-215 of the reference)
# ---------------------------------------------------------------------------------------
@dataclass(frozen=True)
class GammaParams:
    """Shape/rate parameterisation; mean = alpha/rate, var = alpha/rate**2."""

    alpha: float
    rate: float

    def __post_init__(self):
        if not (self.alpha > 0 and self.rate > 0):
            raise ValueError(f"alpha and rate must be > 0, got {self.alpha}, {self.rate}")


def _stream(src, kind: BufferKind):
    """(key array, position array) of a positionable stream source of the given kind."""
    if getattr(src, "kind", None) is not kind or not hasattr(src, "stream_key") or not hasattr(src, "skip"):
        raise TypeError(f"device sampling needs a positionable {kind.value} stream "
                        "(DeviateBuffer / OneAtATime* of this package)")
    k0, k1 = src.stream_key()
    return np.array([k0, k1], dtype=np.uint64), np.array([src.position], dtype=np.uint64)


def _advance(src, old: int, new: int) -> None:
    src.skip(int(new) - int(old))


def _alphas(alphas) -> np.ndarray:
    a = np.asarray(alphas, dtype=float)
    if a.ndim != 1 or a.size < 1:
        raise ValueError("alphas must be a non-empty 1-D vector")
    if not np.all(a > 0):
        raise ValueError("all alphas must be > 0")
    return np.ascontiguousarray(a)


def gamma_batch(params: GammaParams, n: int, u_src, n_src, device: int = 0, timing: list | None = None) -> np.ndarray:
    """n Gamma(alpha, rate) draws == [gamma_sample(params, u_src, n_src) for _ in range(n)].

    Runs on the device (pm_rng_gamma): alpha >= 1 by the parallel two-scan form, alpha < 1
    (the U**(1/alpha) boost) sequentially on one thread.  Both sources are advanced past
    exactly the deviates the n sequential calls consume.  `timing`, if given, receives
    the device milliseconds.
    """
    if n < 0:
        raise ValueError("n must be >= 0")
    uk, up = _stream(u_src, BufferKind.UNIFORM01)
    nk, npos = _stream(n_src, BufferKind.STD_NORMAL)
    u0, n0 = int(up[0]), int(npos[0])
    out = np.empty(int(n))
    if n:
        _lib.require_device(device)
        ms = ctypes.c_float()
        _lib.call("pm_rng_gamma", device, float(params.alpha), float(params.rate), int(n), _lib.u64ptr(uk),
                  _lib.u64ptr(up), _lib.u64ptr(nk), _lib.u64ptr(npos), _lib.dptr(out), ctypes.byref(ms))
        if timing is not None:
            timing.append(float(ms.value))
    _advance(u_src, u0, up[0])
    _advance(n_src, n0, npos[0])
    return out


def dirichlet_batch(alphas, n: int, u_src, n_src, device: int = 0, timing: list | None = None) -> np.ndarray:
    """n Dirichlet(alphas) vectors == [dirichlet_sample(alphas, u_src, n_src) ...] (n x K)."""
    a = _alphas(alphas)
    if n < 0:
        raise ValueError("n must be >= 0")
    uk, up = _stream(u_src, BufferKind.UNIFORM01)
    nk, npos = _stream(n_src, BufferKind.STD_NORMAL)
    u0, n0 = int(up[0]), int(npos[0])
    out = np.empty((int(n), a.size))
    if n:
        _lib.require_device(device)
        ms = ctypes.c_float()
        _lib.call("pm_rng_dirichlet", device, _lib.dptr(a), a.size, int(n), _lib.u64ptr(uk), _lib.u64ptr(up),
                  _lib.u64ptr(nk), _lib.u64ptr(npos), _lib.dptr(out), ctypes.byref(ms))
        if timing is not None:
            timing.append(float(ms.value))
    _advance(u_src, u0, up[0])
    _advance(n_src, n0, npos[0])
    return out


def gamma_sample(params: GammaParams, u_src, n_src) -> float:
    """One Gamma(alpha, rate) deviate (rng.py:191-198) -- a device batch of one."""
    return float(gamma_batch(params, 1, u_src, n_src)[0])


def dirichlet_sample(alphas, u_src, n_src) -> np.ndarray:
    """Dirichlet(alphas) via normalised Gamma(alpha_i, 1) draws (rng.py:201-215)."""
    return dirichlet_batch(alphas, 1, u_src, n_src)[0]


def _streams(u_srcs, n_srcs):
    if len(u_srcs) != len(n_srcs):
        raise ValueError("need one normal source per uniform source")
    S = len(u_srcs)
    uk = np.empty((S, 2), dtype=np.uint64)
    nk = np.empty((S, 2), dtype=np.uint64)
    up = np.empty(S, dtype=np.uint64)
    npos = np.empty(S, dtype=np.uint64)
    for s in range(S):
        k, p = _stream(u_srcs[s], BufferKind.UNIFORM01)
        uk[s], up[s] = k, p[0]
        k, p = _stream(n_srcs[s], BufferKind.STD_NORMAL)
        nk[s], npos[s] = k, p[0]
    return S, uk, up, nk, npos


def gamma_streams(params: GammaParams, n_per: int, u_srcs, n_srcs, device: int = 0,
                  timing: list | None = None) -> np.ndarray:
    """S independent chains' draws: out[s] == gamma_batch(params, n_per, u_srcs[s], n_srcs[s]).

    One device thread per (uniform, normal) stream pair -- the reference's concurrency
    model of spawn-keyed owner streams (rng.py:7-9); each source is advanced.
    """
    S, uk, up, nk, npos = _streams(u_srcs, n_srcs)
    old_u, old_n = up.copy(), npos.copy()
    out = np.empty((S, int(n_per)))
    if S and n_per:
        _lib.require_device(device)
        ms = ctypes.c_float()
        _lib.call("pm_rng_gamma_streams", device, float(params.alpha), float(params.rate), S, int(n_per),
                  _lib.u64ptr(uk), _lib.u64ptr(up), _lib.u64ptr(nk), _lib.u64ptr(npos), _lib.dptr(out),
                  ctypes.byref(ms))
        if timing is not None:
            timing.append(float(ms.value))
    for s in range(S):
        _advance(u_srcs[s], old_u[s], up[s])
        _advance(n_srcs[s], old_n[s], npos[s])
    return out


def dirichlet_streams(alphas, n_per: int, u_srcs, n_srcs, device: int = 0, timing: list | None = None) -> np.ndarray:
    """S independent chains of Dirichlet(alphas) vectors, out[s, i, :]."""
    a = _alphas(alphas)
    S, uk, up, nk, npos = _streams(u_srcs, n_srcs)
    old_u, old_n = up.copy(), npos.copy()
    out = np.empty((S, int(n_per), a.size))
    if S and n_per:
        _lib.require_device(device)
        ms = ctypes.c_float()
        _lib.call("pm_rng_dirichlet_streams", device, _lib.dptr(a), a.size, S, int(n_per), _lib.u64ptr(uk),
                  _lib.u64ptr(up), _lib.u64ptr(nk), _lib.u64ptr(npos), _lib.dptr(out), ctypes.byref(ms))
        if timing is not None:
            timing.append(float(ms.value))
    for s in range(S):
        _advance(u_srcs[s], old_u[s], up[s])
        _advance(n_srcs[s], old_n[s], npos[s])
    return out


# ---------------------------------------------------------------------------------------
# generation benchmark (rng.py:218-300 of the reference), device mode
# ---------------------------------------------------------------------------------------
class BenchDist(Enum):
    UNIFORM = "uniform"
    NORMAL = "normal"
    GAMMA = "gamma"
    DIRICHLET = "dirichlet"


class BenchMode(Enum):
    ONE_AT_A_TIME = "oaat"
    BATCH = "batch"
    DEVICE = "device"


@dataclass
class RngBenchRecord:
    """One timed cell of the generation benchmark (CSV schema order, rng.py:233-241)."""

    dist: str
    mode: str
    n: int
    cycles_per_sample: float
    waste_fraction: float


NOMINAL_CLOCK_GHZ = 2.6
_BENCH_GAMMA = GammaParams(alpha=2.0, rate=3.0)
_BENCH_DIRICHLET_K = 100


def rng_bench(dist: BenchDist, mode: BenchMode, n: int, seed: int = 0, capacity: int = 8192,
              clock_ghz: float = NOMINAL_CLOCK_GHZ, device: int = 0) -> RngBenchRecord:
    """Time generating n deviates; cycles per sample at the nominal clock (rng.py:246-300).

    Compatibility-only (the batch-vs-one-at-a-time study is out of scope): kept
    so the reference's `rng-bench` command and tests run against the drop-in.

    DEVICE mode times the device generation with CUDA events on the same streams and
    workloads as the reference's cells (uniform / normal on one stream; Gamma(2, 3) on
    owner streams (0,), (1,); Dirichlet(1_100) normalised per Gamma component).  BATCH /
    ONE_AT_A_TIME time the host-side stream objects the reference compares (block-refilled
    DeviateBuffer vs a per-call source); their Gamma / Dirichlet cells draw one sample per
    device call (the per-call pattern the paper's batch RNG replaces).
    """
    if n < 1:
        raise ValueError("n must be >= 1")
    if mode is not BenchMode.DEVICE:
        return _rng_bench_per_call(dist, mode, n, seed, capacity, clock_ghz, device)
    ms: list[float] = []
    if dist in (BenchDist.UNIFORM, BenchDist.NORMAL):
        kind = BufferKind.UNIFORM01 if dist is BenchDist.UNIFORM else BufferKind.STD_NORMAL
        k0, k1 = DeviateBuffer(kind, seed=seed).stream_key()
        _lib.require_device(device)
        buf = _DeviceScratch(n)
        t = ctypes.c_float()
        code = _lib.PM_RNG_KIND_UNIFORM01 if kind is BufferKind.UNIFORM01 else _lib.PM_RNG_KIND_STD_NORMAL
        _lib.call("pm_rng_fill", device, code, ctypes.c_uint64(k0), ctypes.c_uint64(k1), ctypes.c_uint64(0), int(n),
                  buf.ptr, 1, ctypes.byref(t))
        buf.close()
        ms.append(float(t.value))
        samples = n
    else:
        u = DeviateBuffer(BufferKind.UNIFORM01, capacity, seed, owner=(0,))
        z = DeviateBuffer(BufferKind.STD_NORMAL, capacity, seed, owner=(1,))
        if dist is BenchDist.GAMMA:
            gamma_batch(_BENCH_GAMMA, n, u, z, device, timing=ms)
            samples = n
        else:
            dirichlet_batch(np.ones(_BENCH_DIRICHLET_K), n, u, z, device, timing=ms)
            samples = n * _BENCH_DIRICHLET_K
    wall = ms[0] * 1e-3
    return RngBenchRecord(dist.value, mode.value, n, wall * clock_ghz * 1e9 / samples, 0.0)


def _rng_bench_per_call(dist, mode, n, seed, capacity, clock_ghz, device) -> RngBenchRecord:
    import time
    batch = mode is BenchMode.BATCH
    waste = 0.0
    if dist in (BenchDist.UNIFORM, BenchDist.NORMAL):
        kind = BufferKind.UNIFORM01 if dist is BenchDist.UNIFORM else BufferKind.STD_NORMAL
        acc = 0.0
        if batch:
            src = DeviateBuffer(kind, capacity=capacity, seed=seed)
            t0 = time.perf_counter()
            for lo in range(0, n, capacity):
                acc += float(src.take(min(capacity, n - lo))[-1])
            wall = time.perf_counter() - t0
            waste = src.waste_fraction
        else:
            src = OneAtATimeUniform(seed) if kind is BufferKind.UNIFORM01 else OneAtATimeNormal(seed)
            t0 = time.perf_counter()
            for _ in range(n):
                acc += src.next()
            wall = time.perf_counter() - t0
        samples = n
    else:
        if batch:
            u = DeviateBuffer(BufferKind.UNIFORM01, capacity, seed, owner=(0,))
            z = DeviateBuffer(BufferKind.STD_NORMAL, capacity, seed, owner=(1,))
        else:
            u, z = OneAtATimeUniform(seed, owner=(0,)), OneAtATimeNormal(seed, owner=(1,))
        alphas = np.ones(_BENCH_DIRICHLET_K)
        t0 = time.perf_counter()
        for _ in range(n):
            if dist is BenchDist.GAMMA:
                gamma_batch(_BENCH_GAMMA, 1, u, z, device)
            else:
                dirichlet_batch(alphas, 1, u, z, device)
        wall = time.perf_counter() - t0
        samples = n if dist is BenchDist.GAMMA else n * _BENCH_DIRICHLET_K
        if batch:
            gen = u.generated + z.generated
            waste = (gen - u.consumed - z.consumed) / gen if gen else 0.0
    return RngBenchRecord(dist.value, mode.value, n, wall * clock_ghz * 1e9 / samples, waste)


class _DeviceScratch:
    """A device buffer of n doubles (cudaMalloc through torch's allocator-free path)."""

    def __init__(self, n: int):
        import torch  # plumbing only: device memory
        self._t = torch.empty(int(n), dtype=torch.float64, device="cuda")
        self.ptr = self._t.data_ptr()

    def close(self) -> None:
        self._t = None


def write_rng_bench_csv(records: Sequence[RngBenchRecord], path) -> None:
    with open(path, "w") as fh:
        fh.write("dist,mode,n,cycles_per_sample,waste_fraction\n")
        for r in records:
            fh.write(f"{r.dist},{r.mode},{r.n},{r.cycles_per_sample:.6g},{r.waste_fraction:.6g}\n")
