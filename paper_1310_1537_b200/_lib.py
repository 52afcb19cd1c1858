"""ctypes binding of libpmb200.so, the sm_100a C ABI declared in include/pmb200.h.

There is no CPU fallback: if the shared library is missing, or no CUDA device is
visible, every hot-path call raises.  Error codes map to the exceptions the
reference raises at the same boundary (include/pmb200.h header comment):
PM_EINVAL -> ValueError, PM_ERANGE -> IndexError, PM_ENOMEM -> MemoryError,
PM_EDEVICE / PM_ESTATE -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from ctypes import (POINTER, c_char_p, c_double, c_int, c_int8, c_int32, c_int64,
                    c_size_t, c_uint64, c_void_p)

import numpy as np

PM_OK, PM_EINVAL, PM_ERANGE, PM_EDEVICE, PM_ENOMEM, PM_ESTATE, PM_ESLICE, PM_ESHRINK, PM_EDRAIN = range(9)
PM_RNG_KIND_UNIFORM01, PM_RNG_KIND_STD_NORMAL = 0, 1
PM_X_F64, PM_X_F32 = 0, 1
PM_BOUNDARY_FREE, PM_BOUNDARY_PERIODIC = 0, 1
PM_MODEL_ISING, PM_MODEL_POTTS4 = 0, 1
PM_RNG_UNIFORMS, PM_RNG_NUMPY_PHILOX, PM_RNG_PHILOX4X32 = 0, 1, 2
KIND_STREAM, KIND_WIDE, KIND_ROWS = 1, 2, 3
MAX_DELTAS = 16

LIB_NAME = "libpmb200.so"
# PM_LIB_PATH selects an A/B build variant of the same ABI (csrc/Makefile LIB=...)
LIB_PATH = os.environ.get("PM_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

_dp = POINTER(c_double)
_i64p = POINTER(c_int64)
_i8p = POINTER(c_int8)
_ip = POINTER(c_int)
_u64p = POINTER(c_uint64)
_fp = POINTER(ctypes.c_float)

# name -> (restype, argtypes); every symbol include/pmb200.h declares
SIGNATURES = {
    "pm_abi_version": (c_int, []),
    "pm_last_error": (c_char_p, []),
    "pm_device_count": (c_int, [_ip]),
    "pm_device_info": (c_int, [c_int, _ip, _ip, _ip, POINTER(c_size_t)]),
    "pm_tune_set": (c_int, [c_char_p, c_int, c_int]),
    "pm_tune_get": (c_int, [c_char_p, _ip, _ip]),
    "pm_glm_create": (c_int, [c_int, POINTER(c_void_p)]),
    "pm_glm_destroy": (c_int, [c_void_p]),
    "pm_glm_upload": (c_int, [c_void_p, c_void_p, c_int, _dp, c_int64, c_int32]),
    "pm_glm_set_prior": (c_int, [c_void_p, _dp, _dp]),
    "pm_glm_eval": (c_int, [c_void_p, _dp, c_int, c_int, _dp, _dp]),
    "pm_glm_launch": (c_int, [c_void_p, _dp, c_int, c_int]),
    "pm_glm_wait": (c_int, [c_void_p, _dp, _dp]),
    "pm_glm_eval_device": (c_int, [c_void_p, _dp, c_int, c_int, c_void_p, c_void_p]),
    "pm_fold_rows": (c_int, [c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    "pm_xchg_create": (c_int, [c_int, c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "pm_xchg_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "pm_xchg_open_peer": (c_int, [c_void_p, c_int32, c_void_p]),
    "pm_xchg_mailbox": (c_int, [c_void_p, POINTER(c_void_p)]),
    "pm_xchg_set_peer_ptr": (c_int, [c_void_p, c_int32, c_void_p]),
    "pm_xchg_status": (c_int, [c_void_p, POINTER(c_int32)]),
    "pm_xchg_destroy": (c_int, [c_void_p]),
    "pm_glm_eval_xchg": (c_int, [c_void_p, _dp, c_int, c_void_p, c_void_p, c_void_p]),
    "pm_glm_eval_xchg_phase": (c_int, [c_void_p, _dp, c_int, c_void_p, c_int, c_void_p, c_void_p]),
    "pm_glm_time_launches": (c_int, [c_void_p, _dp, c_int32, c_int, c_int, POINTER(ctypes.c_float)]),
    "pm_glm_time_cold": (c_int, [c_void_p, _dp, c_int32, c_int, c_int, POINTER(ctypes.c_float)]),
    "pm_glm_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "pm_glm_geometry": (c_int, [c_void_p, _ip, _ip, _ip, POINTER(c_size_t), _ip]),
    "pm_ws_create": (c_int, [c_void_p, _dp, POINTER(c_void_p)]),
    "pm_ws_destroy": (c_int, [c_void_p]),
    "pm_ws_diff_eval": (c_int, [c_void_p, c_int32, _dp, c_int32, _dp]),
    "pm_ws_commit": (c_int, [c_void_p, c_int32, c_double]),
    "pm_ws_read_xbeta": (c_int, [c_void_p, _dp]),
    "pm_ws_validate": (c_int, [c_void_p, _dp, _dp]),
    "pm_ws_run_chain": (c_int, [c_void_p, _dp, _dp, c_int32, c_int32, c_double, c_int32, c_uint64, c_uint64,
                                c_uint64, _dp, _dp, POINTER(c_uint64), POINTER(c_int64), POINTER(c_int32)]),
    "pm_chain_last_kernel_ms": (c_int, [POINTER(ctypes.c_float)]),
    "pm_hb_create": (c_int, [c_int, POINTER(c_void_p)]),
    "pm_hb_destroy": (c_int, [c_void_p]),
    "pm_hb_upload": (c_int, [c_void_p, _dp, _dp, _i64p, c_int32, c_int32]),
    "pm_hb_eval": (c_int, [c_void_p, _dp, _dp, _dp, c_int, _dp, _dp]),
    "pm_hb_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "pm_hb_time_evals": (c_int, [c_void_p, _dp, _dp, _dp, c_int, c_int32, POINTER(ctypes.c_float)]),
    "pm_hbs_create": (c_int, [c_int, _dp, _dp, _i64p, c_int32, c_int32, _dp, _dp, _dp, _u64p, _u64p,
                              POINTER(c_void_p)]),
    "pm_hbs_destroy": (c_int, [c_void_p]),
    "pm_hbs_sweeps": (c_int, [c_void_p, c_int32, c_int32, c_double, c_int32, _dp, _u64p, _i64p,
                              POINTER(c_int32), POINTER(c_int32), _fp]),
    "pm_hbs_set_prior": (c_int, [c_void_p, _dp, _dp]),
    "pm_hbs_loglike": (c_int, [c_void_p, _dp]),
    "pm_hbs_read_xbeta": (c_int, [c_void_p, _dp]),
    "pm_lat_create": (c_int, [c_int, c_int32, c_int32, c_int, c_int, POINTER(c_void_p)]),
    "pm_lat_destroy": (c_int, [c_void_p]),
    "pm_lat_set_spins": (c_int, [c_void_p, _i8p]),
    "pm_lat_get_spins": (c_int, [c_void_p, _i8p]),
    "pm_lat_set_ising": (c_int, [c_void_p, c_double, _dp]),
    "pm_lat_set_potts": (c_int, [c_void_p, c_double]),
    "pm_lat_sweeps": (c_int, [c_void_p, c_int32, c_int, c_uint64, c_uint64, c_uint64, _dp]),
    "pm_lat_time_sweeps": (c_int, [c_void_p, c_int32, c_int, c_uint64, c_uint64, c_uint64,
                                   POINTER(ctypes.c_float)]),
    "pm_lat_sweeps_acc": (c_int, [c_void_p, c_int32, c_int, c_uint64, c_uint64, c_uint64, _dp, c_int32,
                                  POINTER(c_int32), _i64p]),
    "pm_lat_stream": (c_int, [c_void_p, POINTER(c_void_p)]),
    "pm_lat_packed": (c_int, [c_void_p, _ip]),
    "pm_lat_create_strip": (c_int, [c_int, c_int32, c_int32, c_int32, c_int32, c_int, POINTER(c_void_p)]),
    "pm_lat_strip_half_sweep": (c_int, [c_void_p, c_int, c_uint64, c_uint64, c_void_p]),
    "pm_lat_strip_row": (c_int, [c_void_p, c_int, c_int32, POINTER(c_void_p)]),
    "pm_lat_strip_xchg_create": (c_int, [c_void_p, POINTER(c_void_p)]),
    "pm_lat_strip_xchg_ipc_handle": (c_int, [c_void_p, c_void_p]),
    "pm_lat_strip_xchg_set_peers": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "pm_lat_strip_xchg_start": (c_int, [c_void_p, c_void_p]),
    "pm_lat_strip_xchg_status": (c_int, [c_void_p, POINTER(c_int32)]),
    "pm_rng_fill": (c_int, [c_int, c_int, c_uint64, c_uint64, c_uint64, c_int64, c_void_p, c_int, _fp]),
    "pm_rng_gamma": (c_int, [c_int, c_double, c_double, c_int64, _u64p, _u64p, _u64p, _u64p, _dp, _fp]),
    "pm_rng_dirichlet": (c_int, [c_int, _dp, c_int32, c_int64, _u64p, _u64p, _u64p, _u64p, _dp, _fp]),
    "pm_rng_gamma_streams": (c_int, [c_int, c_double, c_double, c_int32, c_int64, _u64p, _u64p, _u64p, _u64p,
                                     _dp, _fp]),
    "pm_rng_dirichlet_streams": (c_int, [c_int, _dp, c_int32, c_int32, c_int64, _u64p, _u64p, _u64p, _u64p,
                                         _dp, _fp]),
    "pm_row_terms_host": (c_int, [_dp, _dp, c_int64, _dp, _dp]),
    "pm_ising_prob_table": (c_int, [c_double, c_double, _dp]),
    "pm_potts_cdf_table": (c_int, [c_double, _dp]),
}

_lock = threading.Lock()
_lib = None


class NativeLibraryMissing(RuntimeError):
    """libpmb200.so is not built or cannot be loaded; there is no CPU fallback."""


class RngDrainError(RuntimeError):
    """A bounded rejection loop exhausted its iteration cap (rng.py:36-37); PM_EDRAIN."""


def load() -> ctypes.CDLL:
    """Load libpmb200.so (once) and bind every declared symbol."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(make -C paper_1310_1537_b200/csrc); the B200 path has no CPU fallback")
        try:
            lib = ctypes.CDLL(LIB_PATH)
        except OSError as exc:
            raise NativeLibraryMissing(f"cannot load {LIB_PATH}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().pm_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str = "") -> None:
    """Raise the reference-equivalent exception for a non-zero status."""
    if rc == PM_OK:
        return
    msg = last_error() or what
    if rc == PM_EINVAL:
        raise ValueError(msg)
    if rc == PM_ERANGE:
        raise IndexError(msg)
    if rc == PM_ENOMEM:
        raise MemoryError(msg)
    if rc == PM_EDRAIN:
        raise RngDrainError(msg)
    raise RuntimeError(f"libpmb200: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def set_tune(name: str, value: int | None) -> None:
    """Override one kernel-dispatch knob (pm_tune_set); None restores the default."""
    call("pm_tune_set", name.encode(), 0 if value is None else int(value), int(value is None))


class tuned:
    """Context manager: `with tuned(glm_rows=1): ...` sets knobs and restores them after."""

    def __init__(self, **knobs):
        self.knobs = knobs
        self.saved = {}

    def __enter__(self):
        for k, v in self.knobs.items():
            val, is_set = c_int(), c_int()
            call("pm_tune_get", k.encode(), ctypes.byref(val), ctypes.byref(is_set))
            self.saved[k] = val.value if is_set.value else None
            set_tune(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            set_tune(k, v)
        return False


def device_count() -> int:
    n = c_int(0)
    rc = load().pm_device_count(ctypes.byref(n))
    if rc != PM_OK:
        return 0
    return n.value


def require_device(device: int = 0) -> None:
    """Fail loudly when no CUDA device is visible (no CPU fallback exists)."""
    n = device_count()
    if n == 0:
        raise RuntimeError("no CUDA device visible: the paper_1310_1537_b200 hot path runs only on B200 (sm_100a)")
    if not 0 <= device < n:
        raise IndexError(f"device {device} out of range [0, {n})")


def dptr(a: np.ndarray):
    """double* of a C-contiguous float64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(_i64p)


def u64ptr(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


def i8ptr(a: np.ndarray):
    assert a.dtype == np.int8 and a.flags.c_contiguous
    return a.ctypes.data_as(_i8p)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)
