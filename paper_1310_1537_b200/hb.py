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

import numpy as np

from . import _lib
from .glm import DesignMatrix, GradResult

__all__ = ["HbDataset", "CsrGroups", "HbDevice", "hb_log_posterior_grad"]


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
        _lib.call("pm_hb_eval", self._h, _lib.dptr(betas), _lib.dptr(mu), _lib.dptr(sigma),
                  int(want_grad), _lib.dptr(f), _lib.dptr(g))
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
