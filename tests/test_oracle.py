"""Pin the CPU oracle (oracle/) against fixtures generated from the unmodified reference.

CPU only.  The fixtures come from tests/golden/make_golden.py (reference parmcmc
called through its public API); the Philox4x32 generator, which no reference
ships, is pinned by the Random123 known-answer vectors; Potts and periodic Ising
are pinned by exact enumeration (TV distance) as the reference pins its own
sweep (test_ising.py:176-199).
"""

import math

import numpy as np
import pytest

from conftest import golden
from oracle import gibbs_oracle as go
from oracle import glm_oracle as gl


def rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1.0)


# ------------------------------------------------------------------ GLM
def test_glm_oracle_matches_reference_fixtures():
    z = golden("glm.npz")
    for i in range(int(z["n_cases"])):
        x, y, beta = z[f"x{i}"], z[f"y{i}"], z[f"beta{i}"]
        f, g = gl.loglike_grad(x, y, beta)
        assert rel(f, float(z[f"f{i}"])) < 1e-13, i
        scale = np.maximum(np.abs(z[f"g{i}"]), 1.0)
        assert np.max(np.abs(g - z[f"g{i}"]) / scale) < 1e-13, i
        assert rel(gl.loglike(x, y, beta), float(z[f"fl{i}"])) < 1e-13
        lp, _ = gl.log_posterior_grad(x, y, beta, z[f"mu{i}"], z[f"sigma{i}"])
        assert rel(lp, float(z[f"lp{i}"])) < 1e-13


def test_glm_oracle_config0_shape_fixture():
    z = golden("glm.npz")
    f, g = gl.loglike_grad(z["c0_x"], z["c0_y"], z["c0_beta"])
    assert rel(f, float(z["c0_f"])) < 1e-13
    np.testing.assert_allclose(g, z["c0_g"], rtol=1e-12)
    lp, _ = gl.log_posterior_grad(z["c0_x"], z["c0_y"], z["c0_beta"], np.zeros(32), np.full(32, 10.0))
    assert rel(lp, float(z["c0_lp"])) < 1e-13


@pytest.mark.parametrize("workers", [1, 2, 3, 8])
def test_glm_oracle_worker_invariance_and_naive(workers):
    z = golden("glm.npz")
    x, y, beta = z["x1"], z["y1"], z["beta1"]
    f, g = gl.loglike_grad(x, y, beta, workers)
    assert rel(f, gl.naive_loglike(x, y, beta)) < 1e-12
    np.testing.assert_allclose(g, gl.naive_grad(x, y, beta), rtol=1e-10)


def test_glm_oracle_known_answers():
    x = np.random.default_rng(0).standard_normal((37, 4))
    y = (np.arange(37) % 2).astype(float)
    f, g = gl.loglike_grad(x, y, np.zeros(4))
    assert f == pytest.approx(-37 * math.log(2), rel=1e-12)
    np.testing.assert_allclose(g, x.T @ (y - 0.5), rtol=1e-12)
    f, g = gl.loglike_grad(np.array([[1.0, 2.0]]), np.array([1.0]), np.zeros(2))
    assert f == pytest.approx(-math.log(2), rel=1e-14)
    np.testing.assert_allclose(g, [0.5, 1.0], rtol=1e-14)


def test_diff_oracle_replays_reference_ops():
    z = golden("diff.npz")
    x, y, beta = z["x"], z["y"], z["beta"]
    xbeta = x @ beta
    xt = np.ascontiguousarray(x.T)
    for (op, k, d), v in zip(z["ops"], z["vals"]):
        k = int(k)
        if op == 0:
            assert rel(gl.diff_loglike(xbeta, xt[k], y, d), v) < 1e-13
        else:
            gl.commit(xbeta, xt[k], d)
    np.testing.assert_allclose(xbeta, z["xbeta"], rtol=0, atol=1e-12)


def test_sampler_oracle_matches_reference_chain():
    from oracle import sampler_oracle as so
    z = golden("sampler.npz")
    draws, evals = so.run_chain(z["x"], z["y"], np.zeros(4), np.full(4, 5.0), 30, 5, seed=77)
    np.testing.assert_array_equal(draws, z["draws"])
    assert evals == int(z["evals"])
    draws2, evals2 = so.run_chain(z["x2"], z["y2"], np.zeros(5), np.full(5, 5.0), 40, 0, seed=31)
    np.testing.assert_array_equal(draws2, z["draws2"])
    assert evals2 == int(z["evals2"])


def test_hb_oracle_matches_reference():
    z = golden("hb.npz")
    f, g = gl.hb_log_posterior_grad(z["x"], z["y"], z["offsets"], z["betas"], z["mu"], z["sigma"])
    np.testing.assert_allclose(f, z["f"], rtol=1e-13)
    np.testing.assert_allclose(g, z["g"], rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ RNG
def test_numpy_philox_stream_matches_reference_buffer():
    z = golden("rng.npz")
    for seed in (0, 5, 33):
        key = z[f"key{seed}"]
        u = go.numpy_uniforms(int(key[0]), int(key[1]), 0, 1000)
        np.testing.assert_array_equal(u, z[f"u{seed}"])
    key = z["key17_3"]
    np.testing.assert_array_equal(go.numpy_uniforms(int(key[0]), int(key[1]), 0, 100), z["u17_3"])


def test_philox4x32_known_answer_vectors():
    # Random123 kat_vectors, philox4x32_10
    assert [int(v) for v in go.philox4x32([0, 0, 0, 0], [0, 0])] == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert [int(v) for v in go.philox4x32([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2)] == [
        0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert [int(v) for v in go.philox4x32([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344],
                                          [0xA4093822, 0x299F31D0])] == [0xD16CFE09, 0x94FDCCEB, 0x5001E420,
                                                                          0x24126EA1]


def test_philox4x64_matches_numpy_bit_generator():
    bg = np.random.Philox(key=np.array([123456789, 987654321], dtype=np.uint64))
    raw = bg.random_raw(12)
    for i in range(12):
        w = go.load().oracle_numpy_word(i, 123456789, 987654321)
        assert w == int(raw[i])


def test_site_uniforms_are_fair():
    u = go.site_uniforms(seed=7, sweep=3, n_sites=40000)
    assert abs(u.mean() - 0.5) < 0.01 and u.min() >= 0.0 and u.max() < 1.0
    assert len(np.unique(u)) > 39000


# ------------------------------------------------------------------ Gibbs
def test_ising_oracle_matches_reference_sweeps():
    z = golden("ising.npz")
    zr = golden("rng.npz")  # noqa: F841
    for i in range(int(z["n_cases"])):
        h, w, sweeps, seed = (int(v) for v in z[f"meta_{i}"])
        bg = np.random.Philox(np.random.SeedSequence(seed))
        k0, k1 = (int(v) for v in bg.state["state"]["key"])
        got = go.ising_sweeps(z[f"s0_{i}"], z[f"b_{i}"], float(z[f"w_{i}"]), False, sweeps, go.RNG_NUMPY_PHILOX,
                              k0, k1, 0)
        np.testing.assert_array_equal(got, z[f"s1_{i}"], err_msg=f"case {i}")


def test_ising_oracle_image_bias_matches_reference():
    z = golden("ising.npz")
    bg = np.random.Philox(np.random.SeedSequence(9))
    k0, k1 = (int(v) for v in bg.state["state"]["key"])
    got = go.ising_sweeps(z["img_s0"], z["img_b"], 1.0, False, 60, go.RNG_NUMPY_PHILOX, k0, k1, 0)
    np.testing.assert_array_equal(got, z["img_s1"])


def test_periodic_ising_oracle_matches_reference_with_wrapped_table():
    z = golden("periodic.npz")
    for i in range(int(z["n_cases"])):
        h, w, sweeps, seed = (int(v) for v in z[f"meta_{i}"])
        cw, cb = (float(v) for v in z[f"wb_{i}"])
        got = go.ising_sweeps(z[f"s0_{i}"], np.full((h, w), cb), cw, True, sweeps, go.RNG_PHILOX4X32, seed, 0, 0)
        np.testing.assert_array_equal(got, z[f"s1_{i}"], err_msg=f"case {i}")


def test_ising_oracle_uniform_mode_equals_stream_mode():
    gen = np.random.default_rng(4)
    s = gen.choice([-1, 1], size=(6, 10)).astype(np.int8)
    b = gen.normal(0, 0.5, size=(6, 10))
    u = go.site_uniforms(11, 0, 60)
    u = np.concatenate([u, go.site_uniforms(11, 1, 60)])
    a = go.ising_sweeps(s, b, 0.7, True, 2, go.RNG_UNIFORMS, uniforms=u)
    c = go.ising_sweeps(s, b, 0.7, True, 2, go.RNG_PHILOX4X32, 11, 0, 0)
    np.testing.assert_array_equal(a, c)


def _neighbours(h, w, periodic):
    out = []
    for i in range(h):
        for j in range(w):
            nb = []
            for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                a, b = i + di, j + dj
                if periodic:
                    a, b = a % h, b % w
                elif not (0 <= a < h and 0 <= b < w):
                    continue
                nb.append(a * w + b)
            out.append(nb)
    return out


def _tv(counts, p):
    emp = counts / counts.sum()
    return 0.5 * float(np.abs(emp - p).sum())


def test_periodic_ising_oracle_total_variation():
    h, w, cw = 2, 4, 0.5
    nb = _neighbours(h, w, True)
    n = h * w
    states = ((np.arange(1 << n)[:, None] >> np.arange(n)) & 1) * 2 - 1
    logw = np.zeros(1 << n)
    for i in range(n):
        for j in nb[i]:
            logw += 0.25 * cw * states[:, i] * states[:, j]  # 1/2 * w * sum over directed pairs / 2
    p = np.exp(logw - logw.max())
    p /= p.sum()
    s = np.ones((h, w), dtype=np.int8)
    counts = np.zeros(1 << n)
    sweeps = 100000
    for t in range(sweeps):
        s = go.ising_sweeps(s, None, cw, True, 1, go.RNG_PHILOX4X32, 99, 0, t)
        code = int(((s.ravel() > 0) * (1 << np.arange(n))).sum())
        counts[code] += 1
    assert _tv(counts, p) < 0.05


@pytest.mark.parametrize("periodic", [False, True])
def test_potts_oracle_total_variation(periodic):
    h, w, K = 2, 2, 0.7
    nb = _neighbours(h, w, periodic)
    n = h * w
    states = (np.arange(4 ** n)[:, None] // (4 ** np.arange(n))) % 4
    logw = np.zeros(4 ** n)
    for i in range(n):
        for j in nb[i]:
            logw += 0.5 * K * (states[:, i] == states[:, j])
    p = np.exp(logw - logw.max())
    p /= p.sum()
    s = np.zeros((h, w), dtype=np.int8)
    counts = np.zeros(4 ** n)
    sweeps = 100000
    for t in range(sweeps):
        s = go.potts_sweeps(s, K, periodic, 1, go.RNG_PHILOX4X32, 5, 0, t)
        counts[int((s.ravel().astype(np.int64) * 4 ** np.arange(n)).sum())] += 1
    assert _tv(counts, p) < 0.05


def test_potts_cdf_is_normalised_and_monotone():
    for counts in ((4, 0, 0, 0), (1, 1, 1, 1), (0, 2, 2, 0), (0, 0, 0, 4), (1, 0, 3, 0)):
        c = go.potts_cdf(1.0986, counts)
        assert 0.0 <= c[0] <= c[1] <= c[2] <= 1.0
        e = np.exp(1.0986 * np.array(counts, dtype=float))
        np.testing.assert_allclose(c, np.cumsum(e)[:3] / e.sum(), rtol=1e-15)


# ------------------------------------------------------------------ denoise (ising.py:257-290)
def test_denoise_oracle_matches_reference_fixture():
    z = golden("denoise.npz")
    for i in range(int(z["n_cases"])):
        w, bscale, sweeps, burnin, _ = z[f"par_{i}"]
        key = z[f"key_{i}"]
        noisy = z[f"noisy_{i}"]
        out, flips = go.denoise(noisy, float(w), float(bscale), int(sweeps), int(burnin), int(key[0]), int(key[1]))
        np.testing.assert_array_equal(out, z[f"out_{i}"], err_msg=f"case {i}")
        np.testing.assert_array_equal(flips / noisy.size, z[f"trace_{i}"], err_msg=f"case {i}")


# ------------------------------------------------------------------ HB sweep (hb.py:110-168)
@pytest.mark.parametrize("c", [0, 1])
def test_hb_sweep_fixture_is_per_group_run_chain(c):
    # the reference's own equivalence (hb.py:14-17): group m's chain == run_chain on owner (m,)
    from oracle import sampler_oracle as so
    z = golden("hb_sweep.npz")
    x, y, off = z[f"x_{c}"], z[f"y_{c}"], z[f"off_{c}"]
    mu, sigma = z[f"prior_{c}"]
    seed, _, _, sweeps = (int(v) for v in z[f"meta_{c}"])
    total = 0
    for m in range(off.size - 1):
        a, b = off[m], off[m + 1]
        draws, evals = so.run_chain(x[a:b], y[a:b], mu, sigma, sweeps, 0, seed=seed,
                                    rng=so.UniformStream(seed, owner=(m,)))
        total += evals
        np.testing.assert_allclose(draws, z[f"betas_{c}"][:, m, :], rtol=1e-12, atol=1e-14)
    assert total == int(z[f"evals_{c}"])
