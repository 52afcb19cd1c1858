"""Device batch RNG (include/pmb200.h pm_rng_*) against the reference's streams and samplers.

Uniforms are bit-exact; normals and Gamma/Dirichlet draws agree to rounding (CUDA's
log1p / sincos / log / pow vs the host libm) while the stream CONSUMPTION -- which
deviates every draw used -- must match the reference exactly.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import rng_oracle as ro
from paper_1310_1537_b200 import rng
from paper_1310_1537_b200.rng import (BufferKind, DeviateBuffer, GammaParams, OneAtATimeNormal, OneAtATimeUniform,
                                      dirichlet_batch, gamma_batch)
from test_rng_oracle import DIRICHLET_CASES, GAMMA_CASES, key

pytestmark = pytest.mark.gpu

NORMAL_RTOL, NORMAL_ATOL = 1e-13, 1e-14


def sources(seed, owner_u=(0,), owner_n=(1,), cap=8192):
    return (DeviateBuffer(BufferKind.UNIFORM01, cap, seed, owner=owner_u),
            DeviateBuffer(BufferKind.STD_NORMAL, cap, seed, owner=owner_n))


@pytest.mark.parametrize("cap", [1, 3, 8192])
def test_uniform_fill_is_bit_exact_and_advances(gpu, cap):
    a = DeviateBuffer(BufferKind.UNIFORM01, cap, seed=17, owner=(3,))
    b = DeviateBuffer(BufferKind.UNIFORM01, cap, seed=17, owner=(3,))
    for n in (1, 5, 4096, 3, 100003):
        np.testing.assert_array_equal(a.take_device(n), b.take(n))
        np.testing.assert_array_equal(a.take(3), b.take(3))


def test_normal_fill_matches_reference_stream(gpu):
    z = golden("rng_batch.npz")
    a = DeviateBuffer(BufferKind.STD_NORMAL, 4096, seed=8)
    np.testing.assert_allclose(a.take_device(4099), z["normal_n8"], rtol=NORMAL_RTOL, atol=NORMAL_ATOL)
    b = DeviateBuffer(BufferKind.STD_NORMAL, 3, seed=10, owner=(1,))
    got = np.concatenate([b.take_device(1), b.take(2), b.take_device(501), b.take(497)])
    np.testing.assert_allclose(got, z["normal_n10"], rtol=NORMAL_RTOL, atol=NORMAL_ATOL)
    # large range against the oracle, odd start
    k = key(8, ())
    c = DeviateBuffer(BufferKind.STD_NORMAL, seed=8)
    c.skip(12345)
    np.testing.assert_allclose(c.take_device(2_000_001), ro.normals(*k, 12345, 2_000_001),
                               rtol=NORMAL_RTOL, atol=NORMAL_ATOL)


@pytest.mark.parametrize("i", range(len(GAMMA_CASES)))
def test_gamma_batch_matches_reference(gpu, i):
    z = golden("rng_batch.npz")
    alpha, rate, seed, n = GAMMA_CASES[i]
    u, nb = sources(seed)
    draws = gamma_batch(GammaParams(alpha, rate), n, u, nb)
    np.testing.assert_allclose(draws, z[f"gamma_{i}"], rtol=1e-12)
    assert [u.position, nb.position] == list(z[f"gamma_used_{i}"])
    # the buffers continue where the reference's would
    u2, n2 = sources(seed)
    u2.skip(int(z[f"gamma_used_{i}"][0]))
    n2.skip(int(z[f"gamma_used_{i}"][1]))
    np.testing.assert_array_equal(u.take(5), u2.take(5))
    np.testing.assert_array_equal(nb.take(5), n2.take(5))


@pytest.mark.parametrize("i", range(len(DIRICHLET_CASES)))
def test_dirichlet_batch_matches_reference(gpu, i):
    z = golden("rng_batch.npz")
    alphas, seed, n = DIRICHLET_CASES[i]
    u, nb = sources(seed)
    draws = dirichlet_batch(alphas, n, u, nb)
    np.testing.assert_allclose(draws, z[f"dir_{i}"], rtol=1e-11, atol=1e-300)
    assert [u.position, nb.position] == list(z[f"dir_used_{i}"])


def test_streams_match_reference(gpu):
    z = golden("rng_batch.npz")
    us = [DeviateBuffer(BufferKind.UNIFORM01, seed=21, owner=(2 * s,)) for s in range(8)]
    ns = [DeviateBuffer(BufferKind.STD_NORMAL, seed=21, owner=(2 * s + 1,)) for s in range(8)]
    got = rng.gamma_streams(GammaParams(0.7, 1.5), 50, us, ns)
    np.testing.assert_allclose(got, z["gstreams"], rtol=1e-12)
    assert [[u.position, n.position] for u, n in zip(us, ns)] == z["gstreams_used"].tolist()
    us = [DeviateBuffer(BufferKind.UNIFORM01, seed=22, owner=(2 * s,)) for s in range(5)]
    ns = [DeviateBuffer(BufferKind.STD_NORMAL, seed=22, owner=(2 * s + 1,)) for s in range(5)]
    got = rng.dirichlet_streams([0.5, 1.0, 2.0], 20, us, ns)
    np.testing.assert_allclose(got, z["dstreams"], rtol=1e-11)
    assert [[u.position, n.position] for u, n in zip(us, ns)] == z["dstreams_used"].tolist()


def test_scan_form_split_calls_and_oracle(gpu):
    # the parallel two-scan form continues exactly across calls and windows
    p = GammaParams(2.0, 3.0)
    u1, n1 = sources(31)
    whole = gamma_batch(p, 50_000, u1, n1)
    u2, n2 = sources(31)
    parts = np.concatenate([gamma_batch(p, m, u2, n2) for m in (1, 2, 7, 20_000, 29_990)])
    np.testing.assert_array_equal(whole, parts)
    assert (u1.position, n1.position) == (u2.position, n2.position)
    ref, up, npos = ro.gamma_draws(2.0, 3.0, 20_000, key(31, (0,)), 0, key(31, (1,)), 0)
    np.testing.assert_allclose(whole[:20_000], ref, rtol=1e-12)
    # consumption of the first 20000 draws
    u3, n3 = sources(31)
    gamma_batch(p, 20_000, u3, n3)
    assert (u3.position, n3.position) == (up, npos)


def test_gamma_many_windows_moments(gpu):
    # 40M draws span two scan windows (2^25 attempts each); moments of Gamma(2, 3)
    u, nb = sources(41)
    d = gamma_batch(GammaParams(2.0, 3.0), 40_000_000, u, nb)
    assert abs(d.mean() - 2.0 / 3.0) < 5e-4 and abs(d.var() - 2.0 / 9.0) < 1e-3
    assert nb.position >= 40_000_000 and u.position >= 40_000_000
    assert u.position <= nb.position
    # a second device call equals the tail of one long one
    u2, n2 = sources(41)
    a = gamma_batch(GammaParams(2.0, 3.0), 39_999_000, u2, n2)
    b = gamma_batch(GammaParams(2.0, 3.0), 1_000, u2, n2)
    np.testing.assert_array_equal(np.concatenate([a, b]), d)


def test_one_at_a_time_sources_and_sample_api(gpu):
    u, n = OneAtATimeUniform(seed=9, owner=(0,)), OneAtATimeNormal(seed=9, owner=(1,))
    ub, nb = sources(9)
    for _ in range(5):
        assert rng.gamma_sample(GammaParams(2.0, 3.0), u, n) == rng.gamma_sample(GammaParams(2.0, 3.0), ub, nb)
    assert u.next() == ub.next() and n.next() == nb.next()
    v = rng.dirichlet_sample([2.0, 3.0, 5.0], ub, nb)
    assert v.shape == (3,) and abs(v.sum() - 1.0) < 1e-12


def test_rng_bench_device_records(gpu, tmp_path):
    recs = [rng.rng_bench(d, rng.BenchMode.DEVICE, n, seed=9)
            for d, n in ((rng.BenchDist.UNIFORM, 1 << 20), (rng.BenchDist.NORMAL, 1 << 20),
                         (rng.BenchDist.GAMMA, 100_000), (rng.BenchDist.DIRICHLET, 1000))]
    assert all(r.cycles_per_sample > 0 and r.mode == "device" for r in recs)
    path = tmp_path / "rng.csv"
    rng.write_rng_bench_csv(recs, path)
    assert path.read_text().splitlines()[0] == "dist,mode,n,cycles_per_sample,waste_fraction"
