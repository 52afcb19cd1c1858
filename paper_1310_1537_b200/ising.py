"""Checkerboard Gibbs sampling of Ising and q=4 Potts lattices on B200.

Mirror of the reference `parmcmc.ising` sweep path (ising.py:47-187):
`IsingLattice`, `ColorPartition`/`color_lattice`, `conditional_prob` and
`gibbs_sweep(lat, part, rng_buffer, plan)` keep their signatures and semantics:

    P(s_i = +1 | rest) = expit(z_i),  z_i = b_i + w * sum_j s_j        (ising.py:11-16)

colour 0 ((i+j) even) updates against frozen colour 1, then colour 1, with the
uniform of each site pre-assigned by its packed (scan-order) index
(ising.py:175-187).  The sweep runs on the device (include/pmb200.h pm_lat_*);
`ColorPartition` owns the device-resident lattice state, as the reference's
partition owns the packed spin arrays between sweeps (ising.py:101-150).

Uniform sources (the `rng_buffer` argument is duck-typed as in the reference):
  * a DeviateBuffer (this package's or the reference's, UNIFORM01): the numpy
    Philox4x64 stream is generated on the device at the buffer's position and
    the buffer is advanced -> bit-exact with the reference sweep;
  * a SitePhilox: Philox4x32-10 keyed by (seed, sweep, site) (BASELINE c4);
  * anything else with `.take(n)`: the uniforms are drawn on the host in the
    reference's order and shipped to the device.
Extensions beyond the reference: periodic boundaries and the Potts q=4 model.
"""

from __future__ import annotations

import ctypes

import numpy as np
from scipy.special import expit

from . import _lib
from .images import flip_noise, read_pbm, synthetic_binary_image, write_pbm
from .rng import BufferKind, DeviateBuffer, SitePhilox, philox_key_of

__all__ = [
    "IsingLattice", "PottsLattice", "ColorPartition", "conditional_prob", "color_lattice",
    "gibbs_sweep", "gibbs_sweeps", "potts_sweeps", "ising_prob_table", "potts_cdf_table",
    "ZCache", "gibbs_sweep_diff", "gibbs_sweeps_diff", "denoise",
    "read_pbm", "write_pbm", "synthetic_binary_image", "flip_noise",
]


def conditional_prob(z):
    """P(s_i = +1) = 1/(1+exp(-z)), overflow-safe; scalar or array (ising.py:96-98)."""
    return expit(z)


class IsingLattice:
    """Spin grid (int8 +-1), bias grid and uniform coupling (ising.py:47-93).

    `boundary` ("free" as the reference, or "periodic") is an extension.
    """

    def __init__(self, s, b, w: float, boundary: str = "free"):
        s = np.asarray(s)
        b = np.ascontiguousarray(b, dtype=np.float64)
        if s.ndim != 2 or s.size == 0:
            raise ValueError(f"spin grid must be non-empty 2-D, got shape {s.shape}")
        if b.shape != s.shape:
            raise ValueError(f"bias shape {b.shape} != spin shape {s.shape}")
        if not np.isin(s, (-1, 1)).all():
            raise ValueError("spins must be -1 or +1")
        if not np.isfinite(b).all() or not np.isfinite(w):
            raise ValueError("bias and coupling must be finite")
        if boundary not in ("free", "periodic"):
            raise ValueError("boundary must be 'free' or 'periodic'")
        if boundary == "periodic" and (s.shape[0] % 2 or s.shape[1] % 2):
            raise ValueError("periodic checkerboard needs even height and width")
        self.s = s.astype(np.int8)
        self.b = b
        self.w = float(w)
        self.boundary = boundary

    @property
    def height(self) -> int:
        return self.s.shape[0]

    @property
    def width(self) -> int:
        return self.s.shape[1]

    @classmethod
    def from_image(cls, image01, w: float, bias_scale: float) -> "IsingLattice":
        """{0,1} pixels -> {-1,+1} spins; bias = bias_scale * observed spin (ising.py:73-82)."""
        image01 = np.asarray(image01)
        if image01.size == 0:
            raise ValueError("empty image")
        if not np.isin(image01, (0, 1)).all():
            raise ValueError("image entries must be 0 or 1")
        spins = 2 * image01.astype(np.int8) - 1
        return cls(spins, bias_scale * spins.astype(np.float64), w)

    def log_weight(self, s=None) -> float:
        """Log of the unnormalised stationary probability of state s (ising.py:84-93):
        (b.s + w * sum over lattice edges of s_i s_j) / 2, whose single-site conditionals
        are expit(b_i + w * neighbour sum).  Periodic lattices include the wrap edges."""
        sf = (self.s if s is None else np.asarray(s)).astype(np.float64)
        edges = float(np.sum(sf[1:, :] * sf[:-1, :]) + np.sum(sf[:, 1:] * sf[:, :-1]))
        if self.boundary == "periodic":
            edges += float(np.sum(sf[0, :] * sf[-1, :]) + np.sum(sf[:, 0] * sf[:, -1]))
        return 0.5 * (float(np.sum(self.b * sf)) + self.w * edges)


class PottsLattice:
    """q=4 Potts lattice: states 0..3, P(a | rest) proportional to exp(coupling * n_a)."""

    def __init__(self, s, coupling: float, boundary: str = "periodic"):
        s = np.asarray(s)
        if s.ndim != 2 or s.size == 0:
            raise ValueError(f"state grid must be non-empty 2-D, got shape {s.shape}")
        if not np.isin(s, (0, 1, 2, 3)).all():
            raise ValueError("Potts states must be 0..3")
        if not np.isfinite(coupling):
            raise ValueError("coupling must be finite")
        if boundary not in ("free", "periodic"):
            raise ValueError("boundary must be 'free' or 'periodic'")
        if boundary == "periodic" and (s.shape[0] % 2 or s.shape[1] % 2):
            raise ValueError("periodic checkerboard needs even height and width")
        self.s = s.astype(np.int8)
        self.coupling = float(coupling)
        self.boundary = boundary

    @property
    def height(self) -> int:
        return self.s.shape[0]

    @property
    def width(self) -> int:
        return self.s.shape[1]


class LatticeDevice:
    """A pm_lat_t handle: the device-resident lattice state."""

    def __init__(self, height: int, width: int, boundary: str, model: int, device: int = 0):
        lib = _lib.load()
        _lib.require_device(device)
        h = ctypes.c_void_p()
        bnd = _lib.PM_BOUNDARY_PERIODIC if boundary == "periodic" else _lib.PM_BOUNDARY_FREE
        _lib.check(lib.pm_lat_create(device, int(height), int(width), bnd, model, ctypes.byref(h)),
                   "pm_lat_create")
        self._h = h
        self.height, self.width, self.model = height, width, model

    @property
    def handle(self):
        return self._h

    def set_spins(self, s: np.ndarray) -> None:
        s = np.ascontiguousarray(s, dtype=np.int8)
        _lib.call("pm_lat_set_spins", self._h, _lib.i8ptr(s))

    def get_spins(self, out: np.ndarray | None = None) -> np.ndarray:
        """The spins as an int8 grid, written straight into `out` when given (C-contiguous
        int8 of the lattice shape: a page-locked `out` makes the read one DMA)."""
        if out is None:
            out = np.empty((self.height, self.width), dtype=np.int8)
        elif out.dtype != np.int8 or not out.flags.c_contiguous or out.shape != (self.height, self.width):
            raise ValueError("out must be a C-contiguous int8 array of the lattice shape")
        _lib.call("pm_lat_get_spins", self._h, _lib.i8ptr(out))
        return out

    def stream(self) -> int:
        p = ctypes.c_void_p()
        _lib.call("pm_lat_stream", self._h, ctypes.byref(p))
        return p.value or 0

    def fast_path(self) -> bool:
        v = ctypes.c_int()
        _lib.call("pm_lat_packed", self._h, ctypes.byref(v))
        return bool(v.value)

    def sweeps(self, n: int, mode: int, key0: int = 0, key1: int = 0, pos: int = 0, uniforms=None) -> None:
        u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
        _lib.call("pm_lat_sweeps", self._h, int(n), int(mode), ctypes.c_uint64(key0),
                  ctypes.c_uint64(key1), ctypes.c_uint64(pos), _lib.dptr(u))

    def sweeps_acc(self, n: int, mode: int, key0: int = 0, key1: int = 0, pos: int = 0, uniforms=None,
                   acc_from: int = 0, acc: np.ndarray | None = None, want_flips: bool = True):
        """`sweeps` plus per-sweep flip counts and an in-place int32 post-`acc_from` accumulator."""
        u = None if uniforms is None else np.ascontiguousarray(uniforms, dtype=np.float64)
        flips = np.zeros(max(int(n), 0), dtype=np.int64) if want_flips else None
        accp = None
        if acc is not None:
            assert acc.dtype == np.int32 and acc.flags.c_contiguous and acc.size == self.height * self.width
            accp = acc.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        _lib.call("pm_lat_sweeps_acc", self._h, int(n), int(mode), ctypes.c_uint64(key0),
                  ctypes.c_uint64(key1), ctypes.c_uint64(pos), _lib.dptr(u), int(acc_from), accp,
                  None if flips is None else _lib.i64ptr(flips))
        return flips

    def time_sweeps(self, n: int, mode: int, key0: int = 0, key1: int = 0, pos: int = 0) -> float:
        """Device milliseconds of n sweeps with an in-kernel RNG (CUDA events, handle stream)."""
        ms = ctypes.c_float()
        _lib.call("pm_lat_time_sweeps", self._h, int(n), int(mode), ctypes.c_uint64(key0),
                  ctypes.c_uint64(key1), ctypes.c_uint64(pos), ctypes.byref(ms))
        return float(ms.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().pm_lat_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ColorPartition:
    """Checkerboard split (ising.py:101-150) owning the device-resident state.

    colors[c] are the flat indices of colour c in scan order (the packed order);
    the spins live on the device between sweeps and are unpacked into the
    lattice after every sweep call, as the reference's unpack_into does.
    """

    def __init__(self, lat, device: int = 0):
        h, w = lat.height, lat.width
        flat_color = (np.add.outer(np.arange(h), np.arange(w)) % 2).ravel()
        self.colors = [np.flatnonzero(flat_color == c) for c in (0, 1)]
        model = _lib.PM_MODEL_POTTS4 if isinstance(lat, PottsLattice) else _lib.PM_MODEL_ISING
        self._periodic = lat.boundary == "periodic"
        self.device = LatticeDevice(h, w, lat.boundary, model, device)
        # the bias is snapshotted here, as the reference's packed_b (ising.py:134-136); the
        # coupling is re-read before every sweep call (the reference reads lat.w on every
        # half-sweep, ising.py:184), see sync_coupling
        self._coupling = None
        if model == _lib.PM_MODEL_ISING:
            b = np.ascontiguousarray(lat.b, dtype=np.float64)
            uniform_b = bool(np.all(b == b.flat[0]))
            self._bias = None if (uniform_b and b.flat[0] == 0.0) else b.ravel().copy()
        self.sync_coupling(lat)
        self.pack_from(lat)

    def sync_coupling(self, lat) -> None:
        """Upload the probability tables again if the lattice's coupling changed since the
        last upload (e.g. an annealing schedule that sets lat.w between sweeps)."""
        if isinstance(lat, PottsLattice):
            c = float(lat.coupling)
            if c != self._coupling:
                _lib.call("pm_lat_set_potts", self.device.handle, c)
                self._coupling = c
        else:
            w = float(lat.w)
            if w != self._coupling:
                _lib.call("pm_lat_set_ising", self.device.handle, w, _lib.dptr(self._bias))
                self._coupling = w

    @property
    def n_sites(self) -> int:
        return self.colors[0].size + self.colors[1].size

    def pack_from(self, lat) -> None:
        self.device.set_spins(lat.s)

    def unpack_into(self, lat) -> None:
        s = lat.s
        if s.dtype == np.int8 and s.flags.c_contiguous and s.flags.writeable and s.shape == (lat.height, lat.width):
            self.device.get_spins(out=s)  # straight into the lattice's own buffer
        else:
            s[...] = self.device.get_spins()

    @property
    def packed_s(self) -> list[np.ndarray]:
        """Per-colour values in packed (scan) order, float64 (ising.py:134-136); a host copy
        of the device state."""
        flat = self.device.get_spins().ravel().astype(np.float64)
        return [flat[self.colors[c]] for c in (0, 1)]

    def neighbor_spin_sum(self, c: int) -> np.ndarray:
        """Exact neighbour sums of colour c's sites in packed order (ising.py:148-150), from
        the device state; 0 outside a free boundary, wrap-around when periodic."""
        s = self.device.get_spins()
        return _neighbour_sum_grid(s, self._periodic).ravel()[self.colors[c]]


def pin_lattice(lat) -> None:
    """Move lat.s into page-locked host memory (same values) so that pack_from /
    unpack_into -- the spin I/O of every sweep call -- are single DMA transfers instead of
    staged pageable copies.  Optional; the results do not depend on it."""
    import torch  # plumbing only: a page-locked host allocation
    owner = torch.empty(lat.s.shape, dtype=torch.int8, pin_memory=True)
    buf = owner.numpy()
    buf[...] = lat.s
    lat._pinned_owner = owner
    lat.s = buf


def color_lattice(lat, device: int = 0) -> ColorPartition:
    """Build the checkerboard partition and upload the lattice (ising.py:153-155)."""
    return ColorPartition(lat, device)


def _run(lat, part: ColorPartition, rng_buffer, n_sweeps: int, diag: dict | None = None):
    """Run n_sweeps device sweeps drawing from rng_buffer; returns per-sweep flips if diag."""
    if n_sweeps < 1:
        return np.zeros(0, dtype=np.int64) if diag is not None else None
    n0, n1 = part.colors[0].size, part.colors[1].size
    consumed = n_sweeps * (n0 + n1)
    dev = part.device
    part.sync_coupling(lat)
    if isinstance(rng_buffer, SitePhilox):
        mode, k0, k1, pos, u = _lib.PM_RNG_PHILOX4X32, rng_buffer.seed, 0, rng_buffer.sweep, None
        advance = lambda: rng_buffer.advance(n_sweeps)  # noqa: E731
    elif isinstance(rng_buffer, DeviateBuffer) and rng_buffer.kind is BufferKind.UNIFORM01:
        (k0, k1), pos, u = rng_buffer.stream_key(), rng_buffer.position, None
        mode = _lib.PM_RNG_NUMPY_PHILOX
        advance = lambda: rng_buffer.skip(consumed)  # noqa: E731
    elif _is_reference_uniform_buffer(rng_buffer):
        # the reference's own DeviateBuffer: same stream; generate on the device, then advance
        (k0, k1), pos, u = philox_key_of(rng_buffer._gen), _reference_position(rng_buffer), None
        mode = _lib.PM_RNG_NUMPY_PHILOX
        advance = lambda: rng_buffer.take(consumed)  # noqa: E731
    else:
        u = np.concatenate([np.asarray(rng_buffer.take(n), dtype=np.float64)
                            for _ in range(n_sweeps) for n in (n0, n1)])
        mode, k0, k1, pos = _lib.PM_RNG_UNIFORMS, 0, 0, 0
        advance = lambda: None  # noqa: E731
    flips = None
    if diag is None:
        dev.sweeps(n_sweeps, mode, k0, k1, pos, u)
    else:
        flips = dev.sweeps_acc(n_sweeps, mode, k0, k1, pos, u, diag.get("acc_from", 0), diag.get("acc"))
    advance()
    part.unpack_into(lat)
    return flips


def _is_reference_uniform_buffer(obj) -> bool:
    kind = getattr(obj, "kind", None)
    return (hasattr(obj, "_gen") and hasattr(obj, "refills") and hasattr(obj, "cursor")
            and getattr(kind, "value", None) == "uniform01")


def _reference_position(buf) -> int:
    """Stream index of the reference DeviateBuffer's next deviate (rng.py:86-127)."""
    if buf.refills == 0:
        return 0
    return (buf.refills - 1) * buf.capacity + buf.cursor


def gibbs_sweep(lat: IsingLattice, part: ColorPartition, rng_buffer, plan=None) -> None:
    """One full sweep: colour 0 against frozen colour 1, then colour 1 (ising.py:175-187).

    `plan` is accepted for signature compatibility (the device grid replaces the
    worker split, which the reference guarantees is exact, test_ising.py:140-149).
    """
    _run(lat, part, rng_buffer, 1)


def gibbs_sweeps(lat, part: ColorPartition, rng_buffer, n_sweeps: int, plan=None) -> None:
    """n_sweeps sweeps in one device call; identical to n_sweeps gibbs_sweep calls."""
    _run(lat, part, rng_buffer, n_sweeps)


def potts_sweeps(lat: PottsLattice, part: ColorPartition, rng_buffer, n_sweeps: int = 1) -> None:
    """Checkerboard heat-bath sweeps of the q=4 Potts model."""
    _run(lat, part, rng_buffer, n_sweeps)


def _neighbour_sum_grid(s: np.ndarray, periodic: bool) -> np.ndarray:
    """Sum of the 4 neighbours' values (0 outside a free boundary), as float64."""
    sf = s.astype(np.float64)
    if periodic:
        return (np.roll(sf, 1, 0) + np.roll(sf, -1, 0) + np.roll(sf, 1, 1) + np.roll(sf, -1, 1))
    out = np.zeros_like(sf)
    out[1:, :] += sf[:-1, :]
    out[:-1, :] += sf[1:, :]
    out[:, 1:] += sf[:, :-1]
    out[:, :-1] += sf[:, 1:]
    return out


class ZCache:
    """Neighbour-sum cache of the differential path (ising.py:190-229).

    The reference keeps per-colour neighbour sums and patches them by +-2 per
    flip so that a low flip rate saves the gather.  On B200 the gather is three
    coalesced row loads per 16 sites, cheaper than scattering cache updates, so
    the device sweep always recomputes the sums from the resident lattice and
    the "cache" is the lattice state the last differential sweep left behind:
    `nsum(c)` is derived from that snapshot (exact small integers in float64,
    as the reference's), `validate` compares it with a fresh gather of the
    current lattice and so still catches a lattice modified behind the
    cache's back (e.g. by a plain gibbs_sweep).
    """

    def __init__(self, lat: IsingLattice, part: ColorPartition):
        self._part = part
        self._periodic = getattr(lat, "boundary", "free") == "periodic"
        self._snap = lat.s.copy()
        self._nsum_cache = None
        self.flips_last_sweep = 0
        self.n_nodes = part.colors[0].size + part.colors[1].size

    def _resync(self, s: np.ndarray) -> None:
        self._snap = s.copy()
        self._nsum_cache = None

    def _grid(self) -> np.ndarray:
        if self._nsum_cache is None:
            self._nsum_cache = _neighbour_sum_grid(self._snap, self._periodic).ravel()
        return self._nsum_cache

    def nsum(self, c: int) -> np.ndarray:
        """Neighbour spin sums of colour c in packed (scan) order."""
        return self._grid()[self._part.colors[c]]

    def z_grid(self, lat: IsingLattice, part: ColorPartition) -> np.ndarray:
        """z_i = b_i + w * (neighbour spin sum), assembled on the grid (ising.py:210-215)."""
        out = np.empty(lat.height * lat.width)
        b = lat.b.ravel()
        for c in (0, 1):
            idx = part.colors[c]
            out[idx] = b[idx] + lat.w * self.nsum(c)
        return out.reshape(lat.height, lat.width)

    @property
    def flip_rate(self) -> float:
        return self.flips_last_sweep / self.n_nodes

    def validate(self, lat: IsingLattice, part: ColorPartition, tol: float = 1e-10) -> float:
        """Max |cached z - freshly gathered z|; raises AssertionError above tol (ising.py:221-229)."""
        fresh = _neighbour_sum_grid(lat.s, self._periodic).ravel()
        diff = np.abs(lat.w * (self._grid() - fresh))
        err = float(np.max(diff, initial=0.0))
        if err > tol:
            raise AssertionError(f"z cache desynchronized: max error {err:g} > {tol:g}")
        return err


def gibbs_sweep_diff(lat: IsingLattice, part: ColorPartition, zcache: ZCache, rng_buffer,
                     plan=None) -> None:
    """Differential sweep (ising.py:232-254): same trajectory as gibbs_sweep, plus
    zcache.flips_last_sweep counted on the device (integer atomics, exact)."""
    gibbs_sweeps_diff(lat, part, zcache, rng_buffer, 1)


def gibbs_sweeps_diff(lat: IsingLattice, part: ColorPartition, zcache: ZCache, rng_buffer,
                      n_sweeps: int) -> np.ndarray:
    """n_sweeps differential sweeps in one device call; returns the per-sweep flip counts."""
    flips = _run(lat, part, rng_buffer, n_sweeps, diag={})
    if n_sweeps >= 1:
        zcache.flips_last_sweep = int(flips[-1])
        zcache._resync(lat.s)
    return flips


def denoise(noisy_image, w: float = 1.0, bias_scale: float = 2.0, sweeps: int = 30, burnin: int = 10,
            seed: int = 0, use_diff: bool = False, plan=None, trace_out: list | None = None,
            device: int = 0) -> np.ndarray:
    """Posterior-mean-sign restoration of a {0,1} image (ising.py:257-290).

    All `sweeps` sweeps run in ONE device call (pm_lat_sweeps_acc): the
    post-burn-in spin sum is accumulated in an int32 grid on the device (exact,
    as the reference's float64 sum of +-1 values) and the per-sweep flip counts
    come back for `trace_out`.  The uniforms are the reference's
    DeviateBuffer(UNIFORM01, seed) stream, so the restored image is bit-identical.
    `use_diff` selects the same trajectory in the reference and is accepted for
    signature compatibility; `plan` likewise.
    """
    noisy_image = np.asarray(noisy_image)
    lat = IsingLattice.from_image(noisy_image, w=w, bias_scale=bias_scale)
    if sweeps < 0 or burnin < 0:
        raise ValueError("sweeps and burnin must be >= 0")
    kept = max(0, sweeps - burnin)
    if kept == 0 and trace_out is None:
        return noisy_image.astype(np.uint8).copy()
    part = color_lattice(lat, device)
    try:
        buf = DeviateBuffer(BufferKind.UNIFORM01, seed=seed)
        acc = np.zeros(lat.height * lat.width, dtype=np.int32)
        flips = _run(lat, part, buf, sweeps, diag={"acc_from": burnin, "acc": acc})
    finally:
        part.device.close()
    if trace_out is not None:
        trace_out.extend(float(f) / lat.s.size for f in flips)
    if kept == 0:
        return noisy_image.astype(np.uint8).copy()
    return (acc.reshape(lat.s.shape) >= 0).astype(np.uint8)


def ising_prob_table(w: float, b: float = 0.0) -> np.ndarray:
    """P(+1 | nsum) for nsum = -4..4 as the device uses it (host-built, exact expit)."""
    out = np.empty(9)
    _lib.call("pm_ising_prob_table", float(w), float(b), _lib.dptr(out))
    return out


def potts_cdf_table(coupling: float) -> np.ndarray:
    """cdf[idx, a] for idx = n0 + 5 n1 + 25 n2 + 125 n3, a = 0..2."""
    out = np.empty(625 * 3)
    _lib.call("pm_potts_cdf_table", float(coupling), _lib.dptr(out))
    return out.reshape(625, 3)
