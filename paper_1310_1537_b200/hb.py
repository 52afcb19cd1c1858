"""Hierarchical Bayesian logistic regression: batched per-group evaluation on B200.

The reference evaluates M groups sharing K with a Python loop of per-group
`loglike_grad` calls over `HbDataset.groups` (hb.py:64-86, 127-135), each group
under a fixed shared Gaussian prior (hb.py:110-124, sampler.py:36-58).  Here the
groups are CSR-batched (row offsets int64[G+1]) and one kernel launch returns
all G log-posteriors and the G x K gradient (include/pmb200.h pm_hb_*): one CTA
per group streams its rows through the same TMA ring as the flat kernel.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .glm import DesignMatrix, GradResult

__all__ = ["HbDataset", "CsrGroups", "HbDevice", "hb_log_posterior_grad", "MappingMode", "MappingPolicy",
           "HbState", "synthetic_hb_dataset", "hb_sweep", "hb_sweeps", "hb_benchmark"]


class HbDataset:
    """M design matrices sharing K; group sizes may differ (hb.py:64-86)."""

    def __init__(self, groups: list[DesignMatrix]):
        if not groups:
            raise ValueError("need at least one group")
        k = groups[0].n_cols
        for m, g in enumerate(groups):
            if g.n_cols != k:
                raise ValueError(f"group {m} has {g.n_cols} columns, expected {k}")
        self.groups = list(groups)
        self._csr = None

    @property
    def m_groups(self) -> int:
        return len(self.groups)

    @property
    def n_cols(self) -> int:
        return self.groups[0].n_cols

    @property
    def n_rows_total(self) -> int:
        return sum(g.n_rows for g in self.groups)

    def to_csr(self) -> "CsrGroups":
        if self._csr is None:
            x = np.concatenate([g.x for g in self.groups], axis=0)
            y = np.concatenate([g.y for g in self.groups])
            off = np.zeros(self.m_groups + 1, dtype=np.int64)
            off[1:] = np.cumsum([g.n_rows for g in self.groups])
            self._csr = CsrGroups(x, y, off)
        return self._csr


class CsrGroups:
    """Groups stored CSR-style: rows offsets[g]:offsets[g+1] of (x, y) are group g."""

    def __init__(self, x, y, offsets):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        if x.ndim != 2 or x.shape[1] < 1:
            raise ValueError("x must be 2-D with K >= 1")
        if off.ndim != 1 or off.size < 2 or off[0] != 0 or off[-1] != x.shape[0]:
            raise ValueError("offsets must start at 0 and end at N")
        if np.any(np.diff(off) < 1):
            raise ValueError("every group needs at least one row")
        if y.shape != (x.shape[0],):
            raise ValueError("y length must equal the row count")
        if not np.isfinite(x).all():
            raise ValueError("x contains non-finite entries")
        if not np.isin(y, (0.0, 1.0)).all():
            raise ValueError("y entries must be exactly 0 or 1")
        self.x, self.y, self.offsets = x, y, off
        self._dev = {}

    @property
    def m_groups(self) -> int:
        return self.offsets.size - 1

    @property
    def n_cols(self) -> int:
        return self.x.shape[1]

    @property
    def n_rows_total(self) -> int:
        return self.x.shape[0]

    def on_device(self, device: int = 0) -> "HbDevice":
        d = self._dev.get(device)
        if d is None:
            d = HbDevice(self, device)
            self._dev[device] = d
        return d


class HbDevice:
    """A pm_hb_t handle holding the CSR groups on one device."""

    def __init__(self, csr: CsrGroups, device: int = 0):
        lib = _lib.load()
        _lib.require_device(device)
        h = ctypes.c_void_p()
        _lib.check(lib.pm_hb_create(device, ctypes.byref(h)), "pm_hb_create")
        self._h = h
        self.G, self.K = csr.m_groups, csr.n_cols
        _lib.check(lib.pm_hb_upload(h, _lib.dptr(csr.x), _lib.dptr(csr.y), _lib.i64ptr(csr.offsets),
                                    self.G, self.K), "pm_hb_upload")
        # hot call through a prototype that takes raw addresses (no per-call POINTER objects)
        vp = ctypes.c_void_p
        self._eval_c = ctypes.CFUNCTYPE(ctypes.c_int, vp, vp, vp, vp, ctypes.c_int, vp, vp)(("pm_hb_eval", lib))

    def stream(self) -> int:
        p = ctypes.c_void_p()
        _lib.call("pm_hb_stream", self._h, ctypes.byref(p))
        return p.value or 0

    def eval(self, betas, mu=None, sigma=None, want_grad: bool = True):
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        if betas.shape != (self.G, self.K):
            raise ValueError(f"betas has shape {betas.shape}, expected ({self.G}, {self.K})")
        f = np.empty(self.G)
        g = np.empty((self.G, self.K)) if want_grad else None
        mu = None if mu is None else np.ascontiguousarray(mu, dtype=np.float64)
        sigma = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float64)
        if mu is not None and (mu.shape != (self.K,) or sigma is None or sigma.shape != (self.K,)):
            raise ValueError("prior dimension does not match dataset")
        addr = lambda a: None if a is None else a.__array_interface__["data"][0]  # noqa: E731
        rc = self._eval_c(self._h, addr(betas), addr(mu), addr(sigma), 1 if want_grad else 0, addr(f), addr(g))
        if rc:
            _lib.check(rc, "pm_hb_eval")
        return f, g

    def time_evals(self, betas, mu=None, sigma=None, n: int = 10, want_grad: bool = True) -> float:
        """Device milliseconds of n back-to-back launches (CUDA events on the handle stream)."""
        import ctypes as ct
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        mu = None if mu is None else np.ascontiguousarray(mu, dtype=np.float64)
        sigma = None if sigma is None else np.ascontiguousarray(sigma, dtype=np.float64)
        ms = ct.c_float()
        _lib.call("pm_hb_time_evals", self._h, _lib.dptr(betas), _lib.dptr(mu), _lib.dptr(sigma), int(want_grad),
                  int(n), ct.byref(ms))
        return float(ms.value)

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().pm_hb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hb_log_posterior_grad(data, betas, prior=None, device: int = 0, want_grad: bool = True):
    """Per-group log-posterior and gradient for all groups in one launch.

    data: HbDataset or CsrGroups; betas: (G, K); prior: GaussianPrior shared by all
    groups (None: likelihood only).  Returns a list of GradResult, one per group,
    each equal to loglike_grad(group, beta_g) plus the prior terms.
    """
    csr = data.to_csr() if isinstance(data, HbDataset) else data
    dev = csr.on_device(device)
    mu = None if prior is None else prior.mu
    sigma = None if prior is None else prior.sigma
    f, g = dev.eval(betas, mu, sigma, want_grad)
    return [GradResult(float(f[i]), None if g is None else g[i]) for i in range(dev.G)]


# ---------------------------------------------------------------------------------------
# hierarchical Gibbs sweep (hb.py:46-204 of the reference), device-resident
# ---------------------------------------------------------------------------------------
class MappingMode(Enum):
    """COARSE (workers across groups) / FINE (row-parallel per group), hb.py:46-49.

    On the device both mappings are the same launch -- one CTA per group, its rows
    split across the CTA's threads -- and, as in the reference, the draws never
    depend on the mapping.
    """

    COARSE = "coarse"
    FINE = "fine"


@dataclass(frozen=True)
class MappingPolicy:
    mode: MappingMode
    workers: int = 1
    neval: int = 1

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.neval < 1:
            raise ValueError("neval must be >= 1")


def synthetic_hb_dataset(m_groups: int, n_cols: int, navg: int, seed: int = 0, prior=None):
    """Uniform-size groups with beta_m drawn from the hyperprior (hb.py:89-107).

    Same SeedSequence(seed, spawn_key=(m,)) draws as the reference, so the data are
    identical.  Returns (HbDataset, betas_true (M, K)).
    """
    from .glm import synthetic_logistic
    from .sampler import GaussianPrior
    if prior is None:
        prior = GaussianPrior.isotropic(n_cols)
    groups, betas = [], np.empty((m_groups, n_cols))
    for m in range(m_groups):
        gen = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(m,)))
        beta_m = prior.mu + prior.sigma * gen.standard_normal(n_cols)
        child = int(gen.integers(2 ** 63))
        data, _ = synthetic_logistic(navg, n_cols, seed=child, beta=beta_m)
        groups.append(data)
        betas[m] = beta_m
    return HbDataset(groups), betas


class HbState:
    """Per-group workspaces and uniform streams persisting across sweeps (hb.py:110-124).

    The workspaces (xbeta, transposed X per group) live on the device in one pm_hbs_t
    handle; each group keeps the reference's stream DeviateBuffer(UNIFORM01,
    buffer_capacity, seed, owner=(m,)), advanced on the host after every device sweep
    past exactly the uniforms the group consumed.  Every group starts at prior.mu.
    """

    def __init__(self, ds: HbDataset, prior, seed: int = 0, buffer_capacity: int = 8192, device: int = 0):
        from .rng import BufferKind, DeviateBuffer
        if prior.mu.shape != (ds.n_cols,):
            raise ValueError("prior dimension does not match dataset")
        _lib.require_device(device)
        self.buffers = [DeviateBuffer(BufferKind.UNIFORM01, buffer_capacity, seed, owner=(m,))
                        for m in range(ds.m_groups)]
        self.total_evals = 0
        self.G, self.K = ds.m_groups, ds.n_cols
        self.device = device
        csr = ds.to_csr()
        self._rows = csr.n_rows_total
        keys = np.ascontiguousarray([b.stream_key() for b in self.buffers], dtype=np.uint64)
        pos = np.zeros(self.G, dtype=np.uint64)
        self._betas = np.ascontiguousarray(np.tile(prior.mu, (self.G, 1)))
        self._prior = (prior.mu.copy(), prior.sigma.copy())
        h = ctypes.c_void_p()
        _lib.call("pm_hbs_create", device, _lib.dptr(csr.x), _lib.dptr(csr.y), _lib.i64ptr(csr.offsets), self.G,
                  self.K, _lib.dptr(self._prior[0]), _lib.dptr(self._prior[1]), _lib.dptr(self._betas),
                  _lib.u64ptr(keys), _lib.u64ptr(pos), ctypes.byref(h))
        self._h = h
        self.last_kernel_ms = 0.0

    @property
    def betas(self) -> list[np.ndarray]:
        return [b.copy() for b in self._betas]

    def _use_prior(self, prior) -> None:
        if prior.mu.shape != (self.K,):
            raise ValueError("prior dimension does not match dataset")
        if not (np.array_equal(prior.mu, self._prior[0]) and np.array_equal(prior.sigma, self._prior[1])):
            _lib.call("pm_hbs_set_prior", self._h, _lib.dptr(prior.mu), _lib.dptr(prior.sigma))
            self._prior = (prior.mu.copy(), prior.sigma.copy())

    def sweeps(self, prior, n_sweeps: int, neval: int = 1, slice_width: float = 1.0,
               slice_max_steps: int = 50) -> None:
        """n_sweeps sweeps of every group in one device launch."""
        from .sampler import SliceWidenError
        self._use_prior(prior)
        pos = np.empty(self.G, dtype=np.uint64)
        evals = np.zeros(self.G, dtype=np.int64)
        fg, fk = ctypes.c_int32(-1), ctypes.c_int32(-1)
        ms = ctypes.c_float()
        start = np.array([b.position for b in self.buffers], dtype=np.int64)
        rc = _lib.load().pm_hbs_sweeps(self._h, int(n_sweeps), int(neval), float(slice_width), int(slice_max_steps),
                                       _lib.dptr(self._betas), _lib.u64ptr(pos), _lib.i64ptr(evals),
                                       ctypes.byref(fg), ctypes.byref(fk), ctypes.byref(ms))
        self.last_kernel_ms = float(ms.value)
        if rc == _lib.PM_OK or rc in (_lib.PM_ESLICE, _lib.PM_ESHRINK):
            for m, b in enumerate(self.buffers):
                b.skip(int(pos[m]) - int(start[m]))
            self.total_evals += int(evals.sum())
        if rc == _lib.PM_ESLICE:
            raise SliceWidenError(_lib.last_error())
        if rc == _lib.PM_ESHRINK:
            raise RuntimeError(_lib.last_error())
        _lib.check(rc, "pm_hbs_sweeps")

    def loglike(self) -> np.ndarray:
        """Per-group log-likelihood at the current coefficients (maintained xbeta)."""
        out = np.empty(self.G)
        _lib.call("pm_hbs_loglike", self._h, _lib.dptr(out))
        return out

    def xbeta(self) -> np.ndarray:
        """Maintained X_g beta_g for all groups, concatenated in row order."""
        out = np.empty(self._rows)
        _lib.call("pm_hbs_read_xbeta", self._h, _lib.dptr(out))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().pm_hbs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def hb_sweep(ds: HbDataset, state: HbState, prior, policy: MappingPolicy, slice_width: float = 1.0,
             slice_max_steps: int = 50) -> list[np.ndarray]:
    """One Gibbs sweep: every group's coefficient vector updated once (hb.py:138-168).

    Returns the post-sweep coefficient vectors (copies).
    """
    state.sweeps(prior, 1, policy.neval, slice_width, slice_max_steps)
    return state.betas


def hb_sweeps(ds: HbDataset, state: HbState, prior, policy: MappingPolicy, n_sweeps: int,
              slice_width: float = 1.0, slice_max_steps: int = 50) -> list[np.ndarray]:
    """n_sweeps hb_sweep calls fused into one launch (identical draws)."""
    state.sweeps(prior, n_sweeps, policy.neval, slice_width, slice_max_steps)
    return state.betas


def hb_benchmark(ds: HbDataset, prior, policies: list[MappingPolicy], n_sweeps: int = 3, reps: int = 3,
                 seed: int = 0, clock_ghz: float = 2.6, slice_width: float = 1.0):
    """Time n_sweeps sweeps under each policy; one BenchRecord per policy (hb.py:171-204).

    Compatibility-only (the CPU thread-mapping study is out of scope): kept so
    the reference's `hb-bench` command and tests run against the drop-in.  On the device
    the policy's mode / workers do not change the schedule (one CTA per group); only
    `neval` does.

    Each repetition restarts from a fresh state with the same seed; the wall time covers
    the n_sweeps sweeps (one device launch) and `evals` = n_sweeps * neval, so cpr is a
    cycles-per-group-row figure as in the reference.
    """
    import statistics
    import time

    from .perf import BenchRecord
    records = []
    for policy in policies:
        walls = []
        for _ in range(reps):
            state = HbState(ds, prior, seed=seed)
            t0 = time.perf_counter()
            state.sweeps(prior, n_sweeps, policy.neval, slice_width)
            walls.append(time.perf_counter() - t0)
            state.close()
        records.append(BenchRecord.from_wall(
            label=f"hb/{policy.mode.value}/neval{policy.neval}", n_rows=ds.n_rows_total, n_cols=ds.n_cols,
            workers=policy.workers, n_chunks=1, wall_seconds=statistics.median(walls),
            evals=n_sweeps * policy.neval, clock_ghz=clock_ghz))
    return records
