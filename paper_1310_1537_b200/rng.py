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

from enum import Enum
from typing import Sequence

import numpy as np

__all__ = ["BufferKind", "DeviateBuffer", "SitePhilox", "philox_key_of"]


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

    def refill(self) -> None:
        """Fill data[0:capacity] with the next block of the base stream."""
        self._block_start = self._gen_pos
        if self.kind is BufferKind.UNIFORM01:
            self.data[:] = self._gen.random(self.capacity)
            self._gen_pos += self.capacity
        else:
            pos = 0
            if self._carry is not None:
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
        return self.refills * self.capacity

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
        """Advance past n deviates that were consumed elsewhere (on the device)."""
        if self.kind is not BufferKind.UNIFORM01:
            raise TypeError("skip is defined for UNIFORM01 streams")
        if n < 0:
            raise ValueError("n must be >= 0")
        if n == 0:
            return
        if n <= self.capacity - self.cursor:
            self.cursor += n
        else:
            # reposition the generator at the target index; the next use refills from there
            target = self.position + n
            bg = self._gen.bit_generator
            st = bg.state
            ctr = np.zeros(4, dtype=np.uint64)
            ctr[0] = target // 4          # numpy pre-increments before generating a block
            st["state"]["counter"] = ctr
            st["buffer_pos"] = 4
            bg.state = st
            if target % 4:
                bg.random_raw(target % 4)
            self._gen_pos = target
            self._block_start = target - self.capacity
            self.cursor = self.capacity
        self.consumed += n


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
