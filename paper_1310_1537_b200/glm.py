"""Logistic-regression log-likelihood / log-posterior and gradient on B200.

Drop-in mirror of the reference module `parmcmc.glm` (/root/reference/pkg/src/
parmcmc/glm.py): same classes, signatures, validation and exceptions, but every
evaluation is one fused sm_100a kernel launch through libpmb200.so
(include/pmb200.h).  There is no CPU path: without the library or a CUDA device
the calls raise.

    L(beta) = -sum_n [(1 - y_n) t_n + log(1 + exp(-t_n))],  t_n = x_n . beta
    g(beta) = X' (y - sigmoid(X beta))                        (glm.py:1-35)

The reference's `ExecPlan(strategy, workers, n_chunks)` is its operator/plugin
interface (glm.py:57-77): all of its strategies are accepted and run the same
single-pass device kernel (X read from HBM once; the CPU strategies only differ
in thread/cache layout, which the CUDA grid replaces).  `Strategy.B200` names
the device path explicitly.  ShardedMatrix shards are evaluated one per visible
device and merged in ascending shard order (glm.py:439-454).
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass
from enum import Enum

import numpy as np
from scipy.special import expit  # noqa: F401  (module attribute of the reference glm as well)

from . import _lib
from . import parallel
from .instrumentation import counters

__all__ = [
    "Strategy", "ExecPlan", "DesignMatrix", "Shard", "ShardedMatrix",
    "GradResult", "GlmWorkspace", "make_sharded", "loglike", "loglike_grad",
    "log_posterior_grad", "diff_loglike", "diff_loglike_multi", "commit_update",
    "load_design_csv", "synthetic_logistic",
]


class Strategy(Enum):
    SOM = "som"
    MOS = "mos"
    PLF = "plf"
    PLF_CHUNKED = "plf_chunked"
    SHARDED = "sharded"
    B200 = "b200"


@dataclass(frozen=True)
class ExecPlan:
    """How an evaluation maps onto the hardware (reference glm.py:65-77).

    `strategy`, `workers`, `n_chunks` keep the reference's meaning and
    validation; on the device they select nothing (one fused kernel serves
    all).  `device` picks the CUDA device; `x_storage` selects the HBM copy of X:
    "f64" (the reference's float64) or "f32" (fp32-X / fp64-accumulate variant).
    """

    strategy: Strategy = Strategy.PLF
    workers: int = 1
    n_chunks: int = 1
    device: int = 0
    x_storage: str = "f64"
    chain: str = "device"

    def __post_init__(self):
        if self.chain not in ("device", "host"):
            raise ValueError(f"chain must be 'device' or 'host', got {self.chain!r}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.n_chunks < 1:
            raise ValueError(f"n_chunks must be >= 1, got {self.n_chunks}")
        if self.device < 0:
            raise ValueError(f"device must be >= 0, got {self.device}")
        if self.x_storage not in ("f64", "f32"):
            raise ValueError(f"x_storage must be 'f64' or 'f32', got {self.x_storage!r}")


class GlmDevice:
    """One device-resident copy of (X, y): a pm_glm_t handle (include/pmb200.h)."""

    def __init__(self, x: np.ndarray, y: np.ndarray, device: int = 0, x_storage: str = "f64"):
        lib = _lib.load()
        _lib.require_device(device)
        h = ctypes.c_void_p()
        _lib.check(lib.pm_glm_create(device, ctypes.byref(h)), "pm_glm_create")
        self._h = h
        self.device = device
        self.x_storage = x_storage
        self.n_rows, self.n_cols = x.shape
        if x_storage == "f32":
            xs = np.ascontiguousarray(x, dtype=np.float32)
            dtype = _lib.PM_X_F32
        else:
            xs = np.ascontiguousarray(x, dtype=np.float64)
            dtype = _lib.PM_X_F64
        y = np.ascontiguousarray(y, dtype=np.float64)
        _lib.check(lib.pm_glm_upload(h, xs.ctypes.data_as(ctypes.c_void_p), dtype, _lib.dptr(y),
                                     self.n_rows, self.n_cols), "pm_glm_upload")
        self._prior_key = None
        self.lock = threading.Lock()
        self.grid = self.geometry()["grid"]
        # hot call: pm_glm_eval through a prototype that takes raw addresses (no per-call
        # POINTER objects) and a reusable result slot for f (guarded by self.lock)
        self._eval_c = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_void_p, ctypes.c_void_p)(("pm_glm_eval", lib))
        self._f_slot = ctypes.c_double()
        self._f_addr = ctypes.addressof(self._f_slot)

    @property
    def handle(self):
        return self._h

    def geometry(self) -> dict:
        g, t, s, k = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        sm = ctypes.c_size_t()
        _lib.call("pm_glm_geometry", self._h, ctypes.byref(g), ctypes.byref(t), ctypes.byref(s),
                  ctypes.byref(sm), ctypes.byref(k))
        return {"grid": g.value, "threads": t.value, "stages": s.value, "smem_bytes": sm.value,
                "kernel": {1: "stream", 2: "wide", 3: "rows"}.get(k.value, "none")}

    def stream(self) -> int:
        p = ctypes.c_void_p()
        _lib.call("pm_glm_stream", self._h, ctypes.byref(p))
        return p.value or 0

    def set_prior(self, mu, sigma) -> None:
        if mu is None:
            if self._prior_key is not None:
                _lib.call("pm_glm_set_prior", self._h, None, None)
                self._prior_key = None
            return
        ready = (isinstance(mu, np.ndarray) and isinstance(sigma, np.ndarray) and mu.dtype == np.float64
                 and sigma.dtype == np.float64 and mu.flags.c_contiguous and sigma.flags.c_contiguous)
        if not ready:  # _prior_arrays hands over validated contiguous float64 arrays
            mu = np.ascontiguousarray(mu, dtype=np.float64)
            sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        key = (mu.tobytes(), sigma.tobytes())
        if key != self._prior_key:
            _lib.call("pm_glm_set_prior", self._h, _lib.dptr(mu), _lib.dptr(sigma))
            self._prior_key = key

    def launch(self, beta: np.ndarray, with_prior: bool, want_grad: bool) -> None:
        _lib.call("pm_glm_launch", self._h, _lib.dptr(beta), int(with_prior), int(want_grad))

    def wait(self, want_grad: bool):
        f = ctypes.c_double()
        g = np.empty(self.n_cols) if want_grad else None
        _lib.call("pm_glm_wait", self._h, ctypes.byref(f), _lib.dptr(g))
        return f.value, g

    def time_launches(self, betas: np.ndarray, with_prior: bool, want_grad: bool) -> float:
        """Device milliseconds of len(betas) back-to-back evaluations (CUDA events)."""
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        ms = ctypes.c_float()
        with self.lock:
            _lib.call("pm_glm_time_launches", self._h, _lib.dptr(betas), int(betas.shape[0]), int(with_prior),
                      int(want_grad), ctypes.byref(ms))
        return float(ms.value)

    def time_cold(self, betas: np.ndarray, with_prior: bool, want_grad: bool) -> float:
        """Device milliseconds summed over len(betas) launches, each after an L2 scrub on the
        handle stream (pm_glm_time_cold: cold inputs, no host launch latency)."""
        betas = np.ascontiguousarray(betas, dtype=np.float64)
        ms = ctypes.c_float()
        with self.lock:
            _lib.call("pm_glm_time_cold", self._h, _lib.dptr(betas), int(betas.shape[0]), int(with_prior),
                      int(want_grad), ctypes.byref(ms))
        return float(ms.value)

    def eval(self, beta: np.ndarray, with_prior: bool, want_grad: bool):
        """One evaluation, one C call (pm_glm_eval holds the handle across launch + wait)."""
        g = np.empty(self.n_cols) if want_grad else None
        rc = self._eval_c(self._h, beta.__array_interface__["data"][0], 1 if with_prior else 0,
                          1 if want_grad else 0, self._f_addr,
                          g.__array_interface__["data"][0] if want_grad else None)
        if rc:
            _lib.check(rc, "pm_glm_eval")
        return self._f_slot.value, g

    def eval_device(self, beta: np.ndarray, want_grad: bool, dev_out_ptr: int, stream: int = 0,
                    with_prior: bool = False) -> None:
        """(f, g) as K+1 doubles into device memory on `stream`, no synchronisation."""
        _lib.call("pm_glm_eval_device", self._h, _lib.dptr(beta), int(with_prior), int(want_grad),
                  ctypes.c_void_p(dev_out_ptr), ctypes.c_void_p(stream or None))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.load().pm_glm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DesignMatrix:
    """Row-major N x K observation matrix with a binary response vector.

    Same validation as the reference (glm.py:87-103).  Immutable, so the device
    copy is uploaded on first use and cached per (device, storage).
    """

    def __init__(self, x, y):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        if x.ndim != 2:
            raise ValueError(f"x must be 2-D, got shape {x.shape}")
        if x.shape[0] < 1 or x.shape[1] < 1:
            raise ValueError(f"need N >= 1 and K >= 1, got shape {x.shape}")
        if y.shape != (x.shape[0],):
            raise ValueError(f"y has shape {y.shape}, expected ({x.shape[0]},)")
        if not np.isfinite(x).all():
            raise ValueError("x contains non-finite entries")
        if not np.isin(y, (0.0, 1.0)).all():
            raise ValueError("y entries must be exactly 0 or 1")
        self.x = x
        self.y = y
        self.x.setflags(write=False)
        self.y.setflags(write=False)
        self._devices: dict[tuple[int, str], GlmDevice] = {}
        self._dev_lock = threading.Lock()

    @property
    def n_rows(self) -> int:
        return self.x.shape[0]

    @property
    def n_cols(self) -> int:
        return self.x.shape[1]

    def on_device(self, device: int = 0, x_storage: str = "f64") -> GlmDevice:
        key = (device, x_storage)
        with self._dev_lock:
            dev = self._devices.get(key)
            if dev is None:
                dev = GlmDevice(self.x, self.y, device, x_storage)
                self._devices[key] = dev
            return dev

    def release_device(self) -> None:
        with self._dev_lock:
            for d in self._devices.values():
                d.close()
            self._devices.clear()


@dataclass(frozen=True)
class Shard:
    """One contiguous row block, privately allocated (glm.py:114-120)."""

    x: np.ndarray
    y: np.ndarray
    row_offset: int


class ShardedMatrix:
    """Row partition of a DesignMatrix into per-shard private copies (glm.py:123-140).

    Each shard is evaluated on device `shard_index % device_count`.
    """

    def __init__(self, shards: list[Shard], n_cols: int):
        self.shards = shards
        self._n_cols = n_cols
        self._designs: list[DesignMatrix | None] = [None] * len(shards)

    @property
    def n_shards(self) -> int:
        return len(self.shards)

    @property
    def n_rows(self) -> int:
        return sum(s.x.shape[0] for s in self.shards)

    @property
    def n_cols(self) -> int:
        return self._n_cols

    def shard_design(self, i: int) -> DesignMatrix:
        d = self._designs[i]
        if d is None:
            d = DesignMatrix(self.shards[i].x, self.shards[i].y)
            self._designs[i] = d
        return d


def make_sharded(data: DesignMatrix, n_shards: int) -> ShardedMatrix:
    """Copy contiguous near-equal row blocks into per-shard allocations (glm.py:143-158)."""
    if not 1 <= n_shards <= data.n_rows:
        raise ValueError(f"n_shards must be in [1, {data.n_rows}], got {n_shards}")
    shards = []
    for start, stop in parallel.partition(data.n_rows, n_shards):
        shards.append(Shard(x=data.x[start:stop].copy(), y=data.y[start:stop].copy(),
                            row_offset=start))
    return ShardedMatrix(shards, data.n_cols)


@dataclass
class GradResult:
    """Log-likelihood (or log-posterior) value and its gradient."""

    f: float
    g: np.ndarray


# analytic flops per row, as the reference counts them (glm.py:173-176)
_TR_FLOPS = 6
_TR_GRAD_FLOPS = 8
_DIFF_FLOPS = 8


def _check_beta(beta, n_cols: int, finite: bool = True) -> np.ndarray:
    """Shape and finiteness of beta (glm.py:210-216).  finite=False leaves the finiteness
    scan to the C entry the caller is about to invoke (pm_glm_eval / pm_glm_launch make the
    same check and raise the same ValueError), one pass instead of two per evaluation."""
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    if beta.shape != (n_cols,):
        raise ValueError(f"beta has shape {beta.shape}, expected ({n_cols},)")
    if finite and not np.isfinite(beta).all():
        raise ValueError("beta contains non-finite entries")
    return beta


def _prior_arrays(prior, n_cols: int):
    if prior is None:
        return None, None
    mu = np.ascontiguousarray(prior.mu, dtype=np.float64)
    sigma = np.ascontiguousarray(prior.sigma, dtype=np.float64)
    if mu.shape != (n_cols,):
        raise ValueError(f"prior has {mu.shape[0]} coordinates, data has {n_cols}")
    return mu, sigma


def _account(plan: ExecPlan, calls: int = 1, launches: int = 0, partials: int = 0, flops: int = 0) -> None:
    """The reference's region / merge accounting for `calls` evaluations under `plan`
    (instrumentation contract, read by its tests: SOM opens two regions -- the matvec and
    the transcendental pass, glm.py:277-295 / 375-396 -- every other strategy one, and the
    merge folds one partial per worker, glm.py:234-250), plus the device work of the call
    (kernel launches, partials folded on the device) -- one counter update in all."""
    regions = 2 if plan.strategy is Strategy.SOM else 1
    counters.account(parallel_regions=regions * calls, merge_events=plan.workers * calls,
                     kernel_launches=launches, device_partials=partials, flops=flops)


def _evaluate(data, beta, plan: ExecPlan, prior, want_grad: bool, flops: int = 0) -> GradResult:
    """Dispatch one evaluation to the device(s); `flops` (the caller's analytic count,
    glm.py:173-176) is accounted with the regions / merges once the evaluation succeeded."""
    mu, sigma = _prior_arrays(prior, data.n_cols)
    if isinstance(data, ShardedMatrix):
        return _evaluate_sharded(data, beta, plan, mu, sigma, want_grad, flops)
    dev = data.on_device(plan.device, plan.x_storage)
    with dev.lock:
        dev.set_prior(mu, sigma)
        f, g = dev.eval(beta, mu is not None, want_grad)
    _account(plan, launches=1, partials=dev.grid, flops=flops)
    return GradResult(f, g)


def _evaluate_sharded(view: ShardedMatrix, beta, plan: ExecPlan, mu, sigma, want_grad: bool,
                      flops: int = 0) -> GradResult:
    """One kernel per shard on device shard % n_devices, merged in ascending shard order."""
    n_dev = max(1, _lib.device_count())
    devs = []
    for i in range(view.n_shards):
        d = view.shard_design(i).on_device((plan.device + i) % n_dev, plan.x_storage)
        devs.append(d)
    # all shards in flight, then fold in shard order (glm.py:243-250)
    for i, d in enumerate(devs):
        d.lock.acquire()
    try:
        for i, d in enumerate(devs):
            with_prior = (i == 0) and mu is not None
            d.set_prior(mu if with_prior else None, sigma if with_prior else None)
            d.launch(beta, with_prior, want_grad)
        f = 0.0
        g = np.zeros(view.n_cols) if want_grad else None
        for d in devs:
            pf, pg = d.wait(want_grad)
            f += pf
            if want_grad:
                g += pg
    finally:
        for d in devs:
            d.lock.release()
    _account(plan, launches=len(devs), partials=len(devs), flops=flops)
    return GradResult(f, g)


def loglike(data, beta, plan: ExecPlan = ExecPlan()) -> float:
    """L(beta) (reference glm.py:257-274); one device pass, value plan-invariant."""
    beta = _check_beta(beta, data.n_cols, finite=False)
    return _evaluate(data, beta, plan, None, False, data.n_rows * (2 * data.n_cols + _TR_FLOPS)).f


def loglike_grad(data, beta, plan: ExecPlan = ExecPlan()) -> GradResult:
    """L(beta) and X'(y - sigmoid(X beta)) (reference glm.py:351-364) in one fused pass."""
    beta = _check_beta(beta, data.n_cols, finite=False)
    return _evaluate(data, beta, plan, None, True, data.n_rows * (4 * data.n_cols + _TR_GRAD_FLOPS))


def log_posterior_grad(data, beta, prior, plan: ExecPlan = ExecPlan(), want_grad: bool = True) -> GradResult:
    """Log-posterior L(beta) + sum_k -0.5((beta_k-mu_k)/sigma_k)^2 and its gradient.

    The one-call composite of loglike_grad (glm.py:351) and the prior terms of
    GaussianPrior.logpdf_coord (sampler.py:55-58, constants dropped); the prior
    is added on the device by the kernel's finalising CTA.
    """
    beta = _check_beta(beta, data.n_cols, finite=False)
    return _evaluate(data, beta, plan, prior, want_grad,
                     data.n_rows * (4 * data.n_cols + _TR_GRAD_FLOPS) + 4 * data.n_cols)


# ---------------------------------------------------------------------------
# differential update (glm.py:461-539)
# ---------------------------------------------------------------------------

class GlmWorkspace:
    """Device-resident X.beta_current plus the transposed copy of X (glm.py:461-489).

    `xbeta` reads the maintained vector back from the device; `beta_current`
    is the host copy of the coefficients.
    """

    def __init__(self, data: DesignMatrix, beta0, build_transpose: bool = True,
                 plan: ExecPlan = ExecPlan()):
        beta0 = _check_beta(beta0, data.n_cols)
        self.beta_current = beta0.copy()
        self._shape = (data.n_rows, data.n_cols)
        self._has_xt = bool(build_transpose)
        self._dev = data.on_device(plan.device, "f64")
        h = ctypes.c_void_p()
        _lib.check(_lib.load().pm_ws_create(self._dev.handle, _lib.dptr(beta0), ctypes.byref(h)),
                   "pm_ws_create")
        self._ws = h
        # hot call through a prototype that takes raw addresses (no per-call POINTER objects)
        vp = ctypes.c_void_p
        self._diff_c = ctypes.CFUNCTYPE(ctypes.c_int, vp, ctypes.c_int32, vp, ctypes.c_int32, vp)(
            ("pm_ws_diff_eval", _lib.load()))
        counters.add_launches(2)

    @property
    def n_rows(self) -> int:
        return self._shape[0]

    @property
    def n_cols(self) -> int:
        return self._shape[1]

    @property
    def xbeta(self) -> np.ndarray:
        out = np.empty(self.n_rows)
        _lib.call("pm_ws_read_xbeta", self._ws, _lib.dptr(out))
        return out

    @property
    def xt(self):
        """None when built without the transpose (the device copy is not exposed)."""
        return True if self._has_xt else None

    def validate(self, data: DesignMatrix, tol: float = 1e-10) -> float:
        """Max |xbeta - X.beta_current|, recomputed on the device; raises if above tol."""
        err = ctypes.c_double()
        beta = np.ascontiguousarray(self.beta_current)
        _lib.call("pm_ws_validate", self._ws, _lib.dptr(beta), ctypes.byref(err))
        counters.add_launches(2)
        if err.value > tol:
            raise AssertionError(f"workspace desynchronized: max error {err.value:g} > {tol:g}")
        return err.value

    def close(self) -> None:
        if getattr(self, "_ws", None):
            _lib.load().pm_ws_destroy(self._ws)
            self._ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check_coord(ws: GlmWorkspace, k: int) -> None:
    if not ws._has_xt:
        raise ValueError("workspace has no transposed copy; build with build_transpose=True")
    if not 0 <= k < ws.n_cols:
        raise IndexError(f"coordinate {k} out of range [0, {ws.n_cols})")


def diff_loglike(ws: GlmWorkspace, data: DesignMatrix, k: int, delta_beta_k: float,
                 plan: ExecPlan = ExecPlan()) -> float:
    """L at beta_current with coordinate k shifted by delta (glm.py:499-522), on the device."""
    return float(diff_loglike_multi(ws, data, k, [delta_beta_k], plan)[0])


def diff_loglike_multi(ws: GlmWorkspace, data: DesignMatrix, k: int, deltas,
                       plan: ExecPlan = ExecPlan()) -> np.ndarray:
    """L(beta_current + delta_m e_k) for up to 16 deltas in one pass over (xbeta, xt[k], y).

    Each value is bit-identical to a single-delta diff_loglike call.
    """
    _check_coord(ws, k)
    d = np.ascontiguousarray(deltas, dtype=np.float64).reshape(-1)
    if d.size < 1 or d.size > _lib.MAX_DELTAS:
        raise ValueError(f"between 1 and {_lib.MAX_DELTAS} deltas per pass")
    if data.n_rows != ws.n_rows or data.n_cols != ws.n_cols:
        raise ValueError("workspace/data shape mismatch")
    out = np.empty(d.size)
    # (the C entry rejects non-finite deltas with the reference's ValueError, glm.py:507-510)
    rc = ws._diff_c(ws._ws, int(k), d.__array_interface__["data"][0], int(d.size),
                    out.__array_interface__["data"][0])
    if rc:
        _lib.check(rc, "pm_ws_diff_eval")
    # glm.py:520-522: 8N flops, one PLF region and one merge per worker per evaluated delta
    counters.account(flops=ws.n_rows * _DIFF_FLOPS * d.size, parallel_regions=d.size,
                     merge_events=plan.workers * d.size, kernel_launches=1)
    return out


def commit_update(ws: GlmWorkspace, k: int, delta_beta_k: float,
                  plan: ExecPlan = ExecPlan()) -> None:
    """xbeta += delta * X_k on the device, beta_k += delta (glm.py:525-539)."""
    _check_coord(ws, k)
    if not math.isfinite(delta_beta_k):
        raise ValueError("delta_beta_k must be finite")
    if delta_beta_k != 0.0:
        _lib.call("pm_ws_commit", ws._ws, int(k), float(delta_beta_k))
        counters.add_launches(1)
    ws.beta_current[k] += delta_beta_k
    counters.add_flops(2 * ws.n_rows)


# ---------------------------------------------------------------------------------------
# data I/O and synthesis (host side, glm.py:546-591 of the reference)
# ---------------------------------------------------------------------------------------
def load_design_csv(path) -> DesignMatrix:
    """Plain CSV of K covariate columns followed by one 0/1 response column (glm.py:546-575).

    Blank lines are skipped; ValueError names the row/column of the first bad cell, a
    ragged row, a missing covariate column or a response outside {0, 1}.
    """
    import csv
    rows: list[list[float]] = []
    with open(path, newline="") as fh:
        for ln, row in enumerate(csv.reader(fh), start=1):
            if not any(c.strip() for c in row):
                continue
            parsed = []
            for col, cell in enumerate(row, start=1):
                try:
                    parsed.append(float(cell))
                except ValueError:
                    raise ValueError(f"{path}: row {ln}, column {col}: not a number: {cell!r}") from None
            rows.append(parsed)
    if not rows:
        raise ValueError(f"{path}: no data rows")
    width = len(rows[0])
    for ln, r in enumerate(rows, start=1):
        if len(r) != width:
            raise ValueError(f"{path}: row {ln}: expected {width} columns, got {len(r)}")
    if width < 2:
        raise ValueError(f"{path}: need at least one covariate column plus a response column")
    table = np.asarray(rows)
    resp = table[:, -1]
    bad = np.flatnonzero((resp != 0.0) & (resp != 1.0))
    if bad.size:
        raise ValueError(f"{path}: row {bad[0] + 1}, column {width}: response must be 0 or 1, got {resp[bad[0]]!r}")
    return DesignMatrix(table[:, :-1], resp)


def synthetic_logistic(n_rows: int, n_cols: int, seed: int = 0, beta=None, beta_scale: float = 1.0):
    """Seeded instance X ~ N(0,1), y ~ Bernoulli(sigmoid(X beta)) (glm.py:578-591).

    Same generator draws in the same order as the reference (X, then beta unless
    given, then the uniforms), so the instance is identical.  Returns (DesignMatrix, beta).
    """
    from scipy.special import expit
    gen = np.random.default_rng(seed)
    x = gen.standard_normal((n_rows, n_cols))
    beta = gen.normal(0.0, beta_scale, n_cols) if beta is None else _check_beta(beta, n_cols)
    y = (gen.random(n_rows) < expit(x @ beta)).astype(np.float64)
    return DesignMatrix(x, y), np.asarray(beta, dtype=np.float64)
