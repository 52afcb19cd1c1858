"""Pin the batch-RNG oracle (oracle/rng_oracle.py) against reference fixtures (CPU only).

tests/golden/rng_batch.npz holds the unmodified reference's normal streams and its
Gamma / Dirichlet draws with their stream consumption (make_golden.py,
rng_batch_fixture); the stream-consumption counts must match exactly, the values to
rounding (numpy's log1p is SIMD-dispatched per host CPU).
"""

import numpy as np
import pytest

from conftest import golden
from oracle import rng_oracle as ro
from paper_1310_1537_b200 import rng
from paper_1310_1537_b200.rng import BufferKind, DeviateBuffer, GammaParams

# make_golden.py GAMMA_CASES / DIRICHLET_CASES
GAMMA_CASES = [(2.0, 3.0, 9, 3000), (1.0, 1.0, 4, 2000), (0.3, 2.0, 5, 1500), (5.5, 0.7, 6, 1000),
               (1.0000001, 1.0, 7, 500), (50.0, 2.0, 1, 500), (0.999, 1.0, 2, 400)]
DIRICHLET_CASES = [([2.0, 3.0, 5.0], 11, 500), ([1.0] * 100, 12, 40), ([0.1, 0.5, 1.0, 2.0], 13, 300), ([1.0], 14, 20),
                   ([0.05] * 5, 15, 200), ([3.0] * 7, 16, 150), ([1.5] * 130, 17, 10)]


def key(seed, owner):
    k = np.random.Philox(np.random.SeedSequence(seed, spawn_key=owner)).state["state"]["key"]
    return np.array(k, dtype=np.uint64)


def test_normal_stream_oracle_matches_reference():
    z = golden("rng_batch.npz")
    np.testing.assert_allclose(ro.normals(*key(8, ()), 0, 4099), z["normal_n8"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(ro.normals(*key(10, (1,)), 0, 1001), z["normal_n10"], rtol=1e-14, atol=1e-15)
    # an odd start (a carried sine) and a window
    np.testing.assert_allclose(ro.normals(*key(8, ()), 37, 100), z["normal_n8"][37:137], rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("i", range(len(GAMMA_CASES)))
def test_gamma_oracle_matches_reference(i):
    z = golden("rng_batch.npz")
    alpha, rate, seed, n = GAMMA_CASES[i]
    draws, up, npos = ro.gamma_draws(alpha, rate, n, key(seed, (0,)), 0, key(seed, (1,)), 0)
    np.testing.assert_allclose(draws, z[f"gamma_{i}"], rtol=1e-13)
    assert [up, npos] == list(z[f"gamma_used_{i}"])


@pytest.mark.parametrize("i", range(len(DIRICHLET_CASES)))
def test_dirichlet_oracle_matches_reference(i):
    z = golden("rng_batch.npz")
    alphas, seed, n = DIRICHLET_CASES[i]
    draws, up, npos = ro.dirichlet_draws(alphas, n, key(seed, (0,)), 0, key(seed, (1,)), 0)
    np.testing.assert_allclose(draws, z[f"dir_{i}"], rtol=1e-12, atol=1e-300)
    assert [up, npos] == list(z[f"dir_used_{i}"])


def test_host_api_validation_needs_no_device():
    with pytest.raises(ValueError):
        GammaParams(0.0, 1.0)
    with pytest.raises(ValueError):
        GammaParams(1.0, -2.0)
    u = DeviateBuffer(BufferKind.UNIFORM01, seed=1)
    zb = DeviateBuffer(BufferKind.STD_NORMAL, seed=1)
    with pytest.raises(ValueError):
        rng.dirichlet_batch([], 3, u, zb)
    with pytest.raises(ValueError):
        rng.dirichlet_batch([1.0, 0.0], 3, u, zb)
    with pytest.raises(ValueError):
        rng.dirichlet_batch(np.ones((2, 2)), 3, u, zb)
    with pytest.raises(TypeError):
        rng.gamma_batch(GammaParams(2.0, 1.0), 3, zb, u)   # swapped stream kinds
    with pytest.raises(ValueError):
        rng.rng_bench(rng.BenchDist.UNIFORM, rng.BenchMode.DEVICE, 0)
    # zero-size requests touch no device
    assert rng.gamma_batch(GammaParams(2.0, 1.0), 0, u, zb).shape == (0,)
    assert rng.dirichlet_batch([1.0, 2.0], 0, u, zb).shape == (0, 2)


@pytest.mark.parametrize("kind", [BufferKind.UNIFORM01, BufferKind.STD_NORMAL])
@pytest.mark.parametrize("capacity", [1, 2, 3, 7, 8192])
def test_skip_continues_the_stream_exactly(kind, capacity):
    # skip(n) must leave the buffer where take(n) would (capacity-invariant, rng.py:1-19)
    a = DeviateBuffer(kind, capacity=capacity, seed=5)
    b = DeviateBuffer(kind, capacity=capacity, seed=5)
    for k in (5, 3, 0, 11, 1, 4097, 2):
        assert a.position == b.position
        a.skip(k)
        b.take(k)
        assert a.position == b.position
        np.testing.assert_array_equal(a.take(7), b.take(7))
