"""CPU checks of the C ABI boundary: libpmb200.so loads, exports exactly what
include/pmb200.h declares, and its host-side table builders are bit-exact.
No compute kernel is launched (there is no GPU here)."""

import os
import re
import subprocess

import numpy as np
import pytest
from scipy.special import expit

from conftest import ROOT
from oracle import gibbs_oracle as go
from paper_1310_1537_b200 import _lib

HEADER = os.path.join(ROOT, "include", "pmb200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^PM_API\s+[\w\s\*]+?\b(pm_\w+)\s*\(", text, flags=re.M)))


def test_library_loads_and_reports_abi():
    lib = _lib.load()
    assert lib.pm_abi_version() == 1


def test_every_declared_symbol_is_exported_and_bound():
    names = declared_symbols()
    assert len(names) >= 30
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (pm_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    assert set(names) == set(_lib.exported_symbols())


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_ising_probability_table_is_scipy_expit_bitwise():
    gen = np.random.default_rng(0)
    for w, b in [(0.8814, 0.0), (1.0, 1.5), (1.0, -1.5), (0.0, 0.3)] + [
            (float(gen.normal()), float(gen.normal(0, 2))) for _ in range(200)]:
        got = np.empty(9)
        _lib.check(_lib.load().pm_ising_prob_table(w, b, _lib.dptr(got)))
        nsum = np.arange(-4, 5, dtype=np.float64)
        ref = expit(b + w * nsum)  # ising.py:184 then :98
        np.testing.assert_array_equal(got, ref)


def test_ising_probability_table_matches_c_oracle():
    for w, b in [(0.8814, 0.0), (2.5, -0.7), (-1.0, 0.25)]:
        got = np.empty(9)
        _lib.check(_lib.load().pm_ising_prob_table(w, b, _lib.dptr(got)))
        for n in range(-4, 5):
            wn = w * float(n)
            assert got[n + 4] == go.load().oracle_expit(b + wn)


@pytest.mark.parametrize("coupling", [0.4407, 1.0986, 0.0, 2.0])
def test_potts_cdf_table_matches_c_oracle_bitwise(coupling):
    tab = np.empty(625 * 3)
    _lib.check(_lib.load().pm_potts_cdf_table(coupling, _lib.dptr(tab)))
    tab = tab.reshape(625, 3)
    for idx in range(625):
        counts = (idx % 5, (idx // 5) % 5, (idx // 25) % 5, (idx // 125) % 5)
        np.testing.assert_array_equal(tab[idx], go.potts_cdf(coupling, counts))


def test_lean_math_accuracy():
    """The kernels' per-row softplus / sigmoid (pm_math.cuh, evaluated on the host with the
    same fused-multiply-add arithmetic the device runs) against glibc, <= 4 ulp."""
    import ctypes
    import math
    lib = _lib.load()
    rng = np.random.default_rng(1)
    t = np.concatenate([rng.uniform(0, 1, 20000), rng.uniform(0, 5, 20000), rng.uniform(0, 45, 20000),
                        rng.uniform(0, 708, 5000), np.abs(rng.normal(0, 1e-6, 500)),
                        [0.0, 1e-300, 0.5, math.log(2.0), 1.0, 2.0, 36.7, 708.0]])
    nll, w = np.empty_like(t), np.empty_like(t)
    ones = np.ones_like(t)
    _lib.check(lib.pm_row_terms_host(_lib.dptr(t), _lib.dptr(ones), t.size, _lib.dptr(nll), _lib.dptr(w)))
    sp = np.array([math.log1p(math.exp(-v)) for v in t])  # y = 1, t >= 0: nll = softplus(-t)
    assert np.max(np.abs(nll - sp) / np.spacing(sp)) <= 4
    sig = np.array([1.0 / (1.0 + math.exp(-v)) for v in t])
    assert np.max(np.abs((1.0 - w) - sig) / sig) < 1e-15
    tn, zeros = -t, np.zeros_like(t)
    _lib.check(lib.pm_row_terms_host(_lib.dptr(tn), _lib.dptr(zeros), t.size, _lib.dptr(nll), _lib.dptr(w)))
    sig_n = np.array([math.exp(-v) / (1.0 + math.exp(-v)) for v in t])
    m = sig_n > 1e-300
    assert np.max(np.abs(-w[m] - sig_n[m]) / sig_n[m]) < 1e-15
    # y = 0, t < 0: nll = (1-0)t + (-t) + softplus = softplus(-|t|)
    assert np.max(np.abs(nll - sp) / np.spacing(sp)) <= 4


def test_error_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.PM_EINVAL)
    with pytest.raises(IndexError):
        _lib.check(_lib.PM_ERANGE)
    with pytest.raises(MemoryError):
        _lib.check(_lib.PM_ENOMEM)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.PM_EDEVICE)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.PM_ESTATE)


def test_null_arguments_are_rejected_without_a_device():
    lib = _lib.load()
    assert lib.pm_glm_create(0, None) == _lib.PM_EINVAL
    assert lib.pm_ising_prob_table(1.0, 0.0, None) == _lib.PM_EINVAL
    assert "null" in _lib.last_error()
    assert lib.pm_glm_destroy(None) == _lib.PM_OK


def test_dispatch_is_not_read_from_the_environment():
    """Kernel choice must not depend on the user's environment: the dispatchers consult
    only the pm_tune_set table (A/B experiments and layout tests set it explicitly)."""
    csrc = os.path.join(ROOT, "paper_1310_1537_b200", "csrc")
    for name in os.listdir(csrc):
        if name.endswith((".cu", ".cuh")):
            assert "getenv" not in open(os.path.join(csrc, name)).read(), name
    lib = _lib.load()
    assert lib.pm_tune_set(b"no_such_knob", 1, 0) == _lib.PM_EINVAL
    with _lib.tuned(glm_rows=0, gibbs_ng=2):
        v, s = _lib.c_int(), _lib.c_int()
        _lib.call("pm_tune_get", b"gibbs_ng", _lib.ctypes.byref(v), _lib.ctypes.byref(s))
        assert (v.value, s.value) == (2, 1)
    _lib.call("pm_tune_get", b"gibbs_ng", _lib.ctypes.byref(v), _lib.ctypes.byref(s))
    assert s.value == 0
