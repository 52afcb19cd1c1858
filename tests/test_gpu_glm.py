"""Device parity of the GLM hot path (fused log-posterior + gradient kernel).

Bar (BASELINE north_star): fp64 within relative 1e-10 of the reference CPU path,
|df|/max(|f|,1) and max_k |dg_k|/max(|g_k|,1); fp32-X within 1e-5 of the fp64
oracle (and 1e-10 of the oracle run on the fp32-rounded X).
"""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import glm_oracle as gl
from paper_1310_1537_b200 import glm
from paper_1310_1537_b200.glm import DesignMatrix, ExecPlan, Strategy
from paper_1310_1537_b200.instrumentation import counters
from paper_1310_1537_b200.sampler import GaussianPrior
from paper_1310_1537_b200.synthetic import baseline_design

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1.0)


def grel(g, ref):
    return float(np.max(np.abs(g - ref) / np.maximum(np.abs(ref), 1.0)))


def test_golden_reference_cases(gpu):
    z = golden("glm.npz")
    for i in range(int(z["n_cases"])):
        d = DesignMatrix(z[f"x{i}"], z[f"y{i}"])
        beta = z[f"beta{i}"]
        r = glm.loglike_grad(d, beta)
        assert rel(r.f, float(z[f"f{i}"])) < TOL, (i, r.f, float(z[f"f{i}"]))
        assert grel(r.g, z[f"g{i}"]) < TOL, i
        assert rel(glm.loglike(d, beta), float(z[f"fl{i}"])) < TOL, i
        prior = GaussianPrior(z[f"mu{i}"], z[f"sigma{i}"])
        lp = glm.log_posterior_grad(d, beta, prior)
        assert rel(lp.f, float(z[f"lp{i}"])) < TOL, i
        _, pg = gl.prior_terms(beta, prior.mu, prior.sigma)
        assert grel(lp.g, z[f"g{i}"] + pg) < TOL, i


def test_config0_shape_fixture(gpu):
    z = golden("glm.npz")
    d = DesignMatrix(z["c0_x"], z["c0_y"])
    r = glm.log_posterior_grad(d, z["c0_beta"], GaussianPrior.isotropic(32, 0.0, 10.0))
    assert rel(r.f, float(z["c0_lp"])) < TOL
    _, pg = gl.prior_terms(z["c0_beta"], np.zeros(32), np.full(32, 10.0))
    assert grel(r.g, z["c0_g"] + pg) < TOL


def test_known_answers(gpu):
    x = np.random.default_rng(0).standard_normal((37, 4))
    y = (np.arange(37) % 2).astype(float)
    d = DesignMatrix(x, y)
    r = glm.loglike_grad(d, np.zeros(4))
    assert r.f == pytest.approx(-37 * math.log(2), rel=1e-12)
    np.testing.assert_allclose(r.g, x.T @ (y - 0.5), rtol=1e-12)
    d1 = DesignMatrix([[1.0, 2.0]], [1.0])
    r1 = glm.loglike_grad(d1, np.zeros(2))
    assert r1.f == pytest.approx(-math.log(2), rel=1e-14)
    np.testing.assert_allclose(r1.g, [0.5, 1.0], rtol=1e-14)
    assert glm.loglike(DesignMatrix([[1.0]], [1.0]), np.zeros(1)) == pytest.approx(-math.log(2), rel=1e-14)


@pytest.mark.parametrize("n,k", [(1, 1), (31, 1), (32, 32), (33, 33), (95, 31), (1000, 63), (4097, 64),
                                 (777, 100), (513, 128), (64, 160), (300, 255), (300, 256), (200, 257),
                                 (100, 512), (9, 2000)])
def test_ragged_shapes_against_oracle(gpu, n, k):
    gen = np.random.default_rng(n * 1000 + k)
    x = gen.standard_normal((n, k)) * gen.uniform(0.5, 2.0)
    y = (gen.random(n) < 0.5).astype(float)
    beta = gen.normal(0, 1.0 / math.sqrt(k), k)
    d = DesignMatrix(x, y)
    r = glm.loglike_grad(d, beta)
    f, g = gl.loglike_grad(x, y, beta)
    assert rel(r.f, f) < TOL and grel(r.g, g) < TOL
    assert rel(glm.loglike(d, beta), f) < TOL


def test_extreme_linear_predictors(gpu):
    # saturated sigmoids on both sides: the stable split must hold (glm.py:182-192)
    x = np.array([[800.0], [-800.0], [40.0], [-40.0], [1e-300], [0.0]])
    y = np.array([1.0, 0.0, 0.0, 1.0, 1.0, 0.0])
    for b in (1.0, -1.0, 0.5):
        r = glm.loglike_grad(DesignMatrix(x, y), np.array([b]))
        f, g = gl.loglike_grad(x, y, np.array([b]))
        assert np.isfinite(r.f) and rel(r.f, f) < TOL and grel(r.g, g) < TOL


def test_fixed_plan_is_bit_deterministic_and_plan_invariant(gpu):
    z = golden("glm.npz")
    d = DesignMatrix(z["x4"], z["y4"])
    beta = z["beta4"]
    first = glm.loglike_grad(d, beta)
    for strategy in Strategy:
        for workers in (1, 4):
            r = glm.loglike_grad(d, beta, ExecPlan(strategy, workers=workers, n_chunks=3))
            assert r.f == first.f and np.array_equal(r.g, first.g)


def test_sharded_view_matches_flat(gpu):
    z = golden("glm.npz")
    d = DesignMatrix(z["x5"], z["y5"])
    beta = z["beta5"]
    v = glm.make_sharded(d, 4)
    a, b = glm.loglike_grad(v, beta), glm.loglike_grad(d, beta)
    assert rel(a.f, b.f) < 1e-12 and grel(a.g, b.g) < 1e-12
    assert rel(glm.loglike(v, beta), b.f) < 1e-12
    prior = GaussianPrior.isotropic(d.n_cols, 0.1, 2.0)
    assert rel(glm.log_posterior_grad(v, beta, prior).f, glm.log_posterior_grad(d, beta, prior).f) < 1e-12


def test_fp32_storage_variant(gpu):
    x, y, _, beta = baseline_design(20000, 100, seed=5)
    d = DesignMatrix(x, y)
    r32 = glm.loglike_grad(d, beta, ExecPlan(x_storage="f32"))
    x32 = x.astype(np.float32).astype(np.float64)
    f32, g32 = gl.loglike_grad(x32, y, beta)
    assert rel(r32.f, f32) < TOL and grel(r32.g, g32) < TOL  # accumulation is fp64
    f64, g64 = gl.loglike_grad(x, y, beta)
    assert rel(r32.f, f64) < 1e-5 and grel(r32.g, g64) < 1e-5


def test_counters_follow_reference_contract(gpu):
    z = golden("glm.npz")
    d = DesignMatrix(z["x4"], z["y4"])
    counters.reset()
    glm.loglike_grad(d, z["beta4"])
    snap = counters.snapshot()
    assert snap.flops == d.n_rows * (4 * d.n_cols + 8)  # glm.py:354
    assert snap.parallel_regions == 1 and snap.kernel_launches == 1 and snap.merge_events == 1
    assert snap.device_partials >= 1
    for strategy, regions in ((Strategy.PLF, 1), (Strategy.SOM, 2), (Strategy.MOS, 1)):
        counters.reset()
        glm.loglike_grad(d, z["beta4"], ExecPlan(strategy, workers=4))
        snap = counters.snapshot()
        assert (snap.parallel_regions, snap.merge_events, snap.kernel_launches) == (regions, 4, 1)
    counters.reset()
    glm.loglike(d, z["beta4"])
    assert counters.snapshot().flops == d.n_rows * (2 * d.n_cols + 6)  # glm.py:264


def test_beta_validation(gpu):
    d = DesignMatrix(np.ones((5, 3)), np.ones(5))
    with pytest.raises(ValueError):
        glm.loglike(d, np.zeros(4))
    with pytest.raises(ValueError):
        glm.loglike_grad(d, np.array([0.0, np.inf, 0.0]))


def test_config0_full_size_against_oracle(gpu):
    x, y, _, beta = baseline_design(100_000, 32, seed=0)
    d = DesignMatrix(x, y)
    prior = GaussianPrior.isotropic(32, 0.0, 10.0)
    r = glm.log_posterior_grad(d, beta, prior)
    f, g = gl.log_posterior_grad(x, y, beta, prior.mu, prior.sigma, workers=4)
    assert rel(r.f, f) < TOL and grel(r.g, g) < TOL


def test_config1_shape_against_oracle(gpu):
    # config 1's K=100 at 2e6 rows (the oracle finishes in seconds); full-size checks below
    x, y, _, betas = baseline_design(2_000_000, 100, seed=1, n_eval=3)
    d = DesignMatrix(x, y)
    prior = GaussianPrior.isotropic(100, 0.0, 10.0)
    for beta in betas:
        r = glm.log_posterior_grad(d, beta, prior)
        f, g = gl.log_posterior_grad(x, y, beta, prior.mu, prior.sigma, workers=8)
        assert rel(r.f, f) < TOL and grel(r.g, g) < TOL
    r32 = glm.loglike_grad(d, betas[0], ExecPlan(x_storage="f32"))
    f, g = gl.loglike_grad(x, y, betas[0], workers=8)
    assert rel(r32.f, f) < 1e-5 and grel(r32.g, g) < 1e-5


def _cores():
    import os
    return max(1, len(os.sched_getaffinity(0)))


def test_config1_full_size_against_oracle(gpu):
    """BASELINE config 1 at its exact size (N=1e7, K=100, the bench's seed-7 design), three
    fresh beta ~ N(0, 0.1^2) with the N(0, 10^2) prior, against the CPU oracle over all host
    cores: fp64 within 1e-10 (f and every g_k); fp32-X within 1e-10 of the oracle on the
    fp32-rounded X and within 1e-5 of the fp64 oracle (the north-star tolerances)."""
    n, k = 10_000_000, 100
    x, y, _, betas = baseline_design(n, k, seed=7, n_eval=3)
    d = DesignMatrix(x, y)
    prior = GaussianPrior.isotropic(k, 0.0, 10.0)
    refs = []
    for beta in betas:
        r = glm.log_posterior_grad(d, beta, prior)
        f, g = gl.log_posterior_grad(x, y, beta, prior.mu, prior.sigma, workers=_cores())
        refs.append((f, g))
        assert rel(r.f, f) < TOL, (r.f, f)
        assert grel(r.g, g) < TOL
    d.release_device()
    plan32 = ExecPlan(x_storage="f32")
    got32 = [glm.log_posterior_grad(d, beta, prior, plan32) for beta in betas]
    d.release_device()
    x32 = x.astype(np.float32).astype(np.float64)
    del x
    for beta, r32, (f64, g64) in zip(betas, got32, refs):
        f, g = gl.log_posterior_grad(x32, y, beta, prior.mu, prior.sigma, workers=_cores())
        assert rel(r32.f, f) < TOL and grel(r32.g, g) < TOL
        assert rel(r32.f, f64) < 1e-5 and grel(r32.g, g64) < 1e-5


def test_config1_full_size_properties(gpu):
    """N=1e7, K=100 fp64 (8 GB): size-independent properties -- L(0) = -N ln 2 and
    g(0) = X'(y - 1/2) checked against cuBLAS fp64 (torch) -- and linearity of the
    row-sharded sum (two half-designs add up to the whole)."""
    import torch
    n, k = 10_000_000, 100
    x, y, _, beta = baseline_design(n, k, seed=11)
    d = DesignMatrix(x, y)
    r0 = glm.loglike_grad(d, np.zeros(k))
    assert rel(r0.f, -n * math.log(2)) < 1e-12
    xt = torch.from_numpy(x).cuda()
    g_ref = (xt.T @ (torch.from_numpy(y).cuda() - 0.5)).cpu().numpy()
    del xt
    torch.cuda.empty_cache()
    assert grel(r0.g, g_ref) < TOL
    r = glm.loglike_grad(d, beta)
    half = n // 2
    d.release_device()
    a = glm.loglike_grad(DesignMatrix(x[:half], y[:half]), beta)
    b = glm.loglike_grad(DesignMatrix(x[half:], y[half:]), beta)
    assert rel(r.f, a.f + b.f) < TOL and grel(r.g, a.g + b.g) < TOL
    assert abs(r.f) > 0 and np.all(np.isfinite(r.g))


@pytest.mark.parametrize("k", [2, 4, 6, 20, 22, 30, 32])
@pytest.mark.parametrize("n", [1, 33, 64, 1000, 250_007])
def test_row_per_lane_kernel_against_oracle_and_stream_kernel(gpu, n, k, tune):
    # fp64 with even K <= 32 runs the row-per-lane kernel (KIND_ROWS): equal contiguous tile
    # ranges per CTA, two tiles per stage; compare with the oracle and the column kernel
    tune(glm_rows=1)  # forced: the default picks it only for K <= 30 at large N
    gen = np.random.default_rng(n + k)
    x = gen.standard_normal((n, k))
    y = (gen.random(n) < 0.4).astype(float)
    beta = gen.normal(0, 0.3, k)
    prior = GaussianPrior(gen.normal(0, 0.5, k), np.full(k, 2.0))
    d = DesignMatrix(x, y)
    r = glm.log_posterior_grad(d, beta, prior)
    assert d.on_device(0).geometry()["kernel"] == "rows"
    f_ref, g_ref = gl.log_posterior_grad(x, y, beta, prior.mu, prior.sigma)
    assert rel(r.f, f_ref) < TOL and grel(r.g, g_ref) < TOL
    assert glm.loglike(d, beta) == glm.loglike_grad(d, beta).f
    again = glm.log_posterior_grad(d, beta, prior)
    assert again.f == r.f and np.array_equal(again.g, r.g)
    tune(glm_rows=0)
    d2 = DesignMatrix(x, y)
    r2 = glm.log_posterior_grad(d2, beta, prior)
    assert d2.on_device(0).geometry()["kernel"] == "stream"
    assert rel(r.f, r2.f) < TOL and grel(r.g, r2.g) < TOL


@pytest.mark.parametrize("pairs", ["2", "1", "0"])
def test_fp32_storage_all_layouts(gpu, tune, pairs):
    """fp32-X over K values that select every stream-kernel consumer layout (column per lane,
    column pairs with XOR-permuted rows, 7 or 15 consumer warps, the wide kernel), f only and
    f + g, against the oracle on the fp32-rounded X (1e-10)."""
    tune(f32_pairs=int(pairs))
    gen = np.random.default_rng(77)
    for k in (1, 2, 31, 40, 64, 66, 100, 128, 130, 192, 256, 300):
        n = 3001 + 37 * k
        x = gen.standard_normal((n, k))
        x[:, 0] = 1.0
        y = (gen.random(n) < 0.4).astype(np.float64)
        beta = gen.normal(0, 0.3, k)
        d = DesignMatrix(x, y)
        plan = ExecPlan(x_storage="f32")
        x32 = x.astype(np.float32).astype(np.float64)
        f, g = gl.loglike_grad(x32, y, beta)
        r = glm.loglike_grad(d, beta, plan)
        assert rel(r.f, f) < TOL and grel(r.g, g) < TOL, k
        assert rel(glm.loglike(d, beta, plan), f) < TOL, k
        d.release_device()


def test_fp32_widening_edge_values(gpu):
    """The fp32-X kernels widen X with integer ops (x * 2^-896, beta * 2^896): zeros, signed
    zeros, fp32 subnormals, the extreme normals and a beta too large for the scaling (routed
    to the wide kernel) all match the oracle on the fp32-rounded X."""
    gen = np.random.default_rng(5)
    n, k = 4099, 100
    x = gen.standard_normal((n, k)).astype(np.float32)
    x[:, 0] = 1.0
    x[::7, 3] = 0.0
    x[1::7, 4] = -0.0
    x[::5, 5] = np.float32(1e-42)  # subnormal
    x[1::5, 6] = -np.float32(3e-39)  # subnormal
    x[2::5, 7] = np.float32(1.17549435e-38)  # smallest normal
    x[3::11, 8] = np.float32(3.0e38)
    x[4::11, 9] = -np.float32(3.0e38)
    y = (gen.random(n) < 0.5).astype(np.float64)
    x64 = x.astype(np.float64)
    d = DesignMatrix(x64, y)
    plan = ExecPlan(x_storage="f32")
    for beta in (gen.normal(0, 0.1, k) * (np.arange(k) < 8),
                 np.r_[gen.normal(0, 1e-40, 10), np.zeros(k - 10)],
                 np.r_[np.zeros(10), 2.0 ** 110, np.zeros(k - 11)]):
        f, g = gl.loglike_grad(x64, y, beta)
        r = glm.loglike_grad(d, beta, plan)
        assert rel(r.f, f) < TOL and grel(r.g, g) < TOL


@pytest.mark.parametrize("pairs", ["1", "0"])
def test_fp64_stream_layouts(gpu, tune, pairs):
    """fp64 X through the stream kernel's two consumer layouts (column pairs with 16-byte
    loads and XOR-permuted rows, or column per lane), f only and f + g, odd and even N,
    against the oracle (1e-10)."""
    tune(f64_pairs=int(pairs))
    tune(glm_rows=0)
    gen = np.random.default_rng(78)
    for k in (2, 40, 64, 66, 100, 128, 192, 256):
        n = 2999 + 41 * k
        x = gen.standard_normal((n, k))
        x[:, 0] = 1.0
        y = (gen.random(n) < 0.6).astype(np.float64)
        beta = gen.normal(0, 0.3, k)
        d = DesignMatrix(x, y)
        f, g = gl.loglike_grad(x, y, beta)
        r = glm.loglike_grad(d, beta)
        assert rel(r.f, f) < TOL and grel(r.g, g) < TOL, k
        assert rel(glm.loglike(d, beta), f) < TOL, k
        d.release_device()


def test_handle_shared_by_threads_c_abi(gpu):
    """include/pmb200.h promises that calls on one handle are serialised, so one handle
    can serve pool threads (the reference's HB COARSE mapping, hb.py:152-161).  8 threads
    x 100 pm_glm_eval calls straight through the C ABI on ONE handle, each with its own
    beta: every result equals that beta's single-thread value bit for bit, and a second
    pm_glm_launch before pm_glm_wait is refused (PM_ESTATE)."""
    import ctypes
    import threading

    from paper_1310_1537_b200 import _lib
    x, y, _, _ = baseline_design(60_013, 32, seed=11)
    d = DesignMatrix(x, y)
    dev = d.on_device(0)
    prior = GaussianPrior.isotropic(32, 0.0, 10.0)
    dev.set_prior(prior.mu, prior.sigma)
    lib = _lib.load()
    gen = np.random.default_rng(12)
    n_threads, n_evals = 8, 100
    betas = gen.normal(0, 0.1, (n_threads, 4, 32))  # 4 distinct betas per thread, cycled
    ref = {}
    for t in range(n_threads):
        for j in range(4):
            f = ctypes.c_double()
            g = np.empty(32)
            _lib.check(lib.pm_glm_eval(dev.handle, _lib.dptr(betas[t, j]), 1, 1, ctypes.byref(f), _lib.dptr(g)),
                       "pm_glm_eval")
            ref[t, j] = (f.value, g)
    errors = []

    def worker(t):
        try:
            for i in range(n_evals):
                j = i % 4
                f = ctypes.c_double()
                g = np.empty(32)
                rc = lib.pm_glm_eval(dev.handle, _lib.dptr(betas[t, j]), 1, 1, ctypes.byref(f), _lib.dptr(g))
                if rc != 0:
                    errors.append((t, i, "rc", rc))
                elif f.value != ref[t, j][0] or not np.array_equal(g, ref[t, j][1]):
                    errors.append((t, i, "mismatch"))
        except Exception as e:  # pragma: no cover - reported below
            errors.append((t, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(n_threads)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[:5]
    # one evaluation in flight per handle
    _lib.check(lib.pm_glm_launch(dev.handle, _lib.dptr(betas[0, 0]), 1, 1), "pm_glm_launch")
    assert lib.pm_glm_launch(dev.handle, _lib.dptr(betas[0, 1]), 1, 1) == _lib.PM_ESTATE
    f = ctypes.c_double()
    _lib.check(lib.pm_glm_wait(dev.handle, ctypes.byref(f), None), "pm_glm_wait")
    assert f.value == ref[0, 0][0]
