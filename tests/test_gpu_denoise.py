"""Device parity of the differential sweep and the denoising pipeline (ising.py:190-290).

Reference fixtures (tests/golden/denoise.npz, made by the unmodified reference)
pin the restored images, per-sweep flip traces, flips_last_sweep and the cached
neighbour sums; the oracle pins larger cases; the reference's own denoise tests
(test_ising.py:206-304) are restated on the device path.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import gibbs_oracle as go
from paper_1310_1537_b200 import ising
from paper_1310_1537_b200.images import flip_noise, synthetic_binary_image
from paper_1310_1537_b200.ising import (IsingLattice, ZCache, color_lattice, denoise, gibbs_sweep,
                                        gibbs_sweep_diff, gibbs_sweeps_diff)
from paper_1310_1537_b200.rng import BufferKind, DeviateBuffer, SitePhilox
from paper_1310_1537_b200.synthetic import ising_spins

pytestmark = pytest.mark.gpu


def test_denoise_matches_reference_fixture(gpu):
    z = golden("denoise.npz")
    for i in range(int(z["n_cases"])):
        w, bscale, sweeps, burnin, seed = z[f"par_{i}"]
        for use_diff in (False, True):
            trace = []
            out = denoise(z[f"noisy_{i}"], w=float(w), bias_scale=float(bscale), sweeps=int(sweeps),
                          burnin=int(burnin), seed=int(seed), use_diff=use_diff, trace_out=trace)
            np.testing.assert_array_equal(out, z[f"out_{i}"], err_msg=f"case {i}")
            assert out.dtype == np.uint8
            np.testing.assert_array_equal(np.array(trace), z[f"trace_{i}"], err_msg=f"case {i}")


def test_diff_sweeps_match_reference_flips_and_cache(gpu):
    z = golden("denoise.npz")
    lat = IsingLattice.from_image(z["diff_img"], 1.0, 1.5)
    part = color_lattice(lat)
    zc = ZCache(lat, part)
    buf = DeviateBuffer(BufferKind.UNIFORM01, seed=9)
    for t in range(len(z["diff_flips"])):
        gibbs_sweep_diff(lat, part, zc, buf)
        assert zc.flips_last_sweep == int(z["diff_flips"][t])
        np.testing.assert_array_equal(np.concatenate([zc.nsum(0), zc.nsum(1)]), z["diff_nsum"][t])
        assert zc.flip_rate == z["diff_flips"][t] / lat.s.size
    np.testing.assert_array_equal(lat.s, z["diff_s1"])
    np.testing.assert_array_equal(zc.z_grid(lat, part), z["diff_z"])
    assert zc.validate(lat, part) == 0.0


def test_diff_sweep_matches_plain_sweep_exactly(gpu):
    img = flip_noise(synthetic_binary_image(20, 24), 0.15, seed=2)
    lat_a, lat_b = IsingLattice.from_image(img, 1.0, 1.5), IsingLattice.from_image(img, 1.0, 1.5)
    pa, pb = color_lattice(lat_a), color_lattice(lat_b)
    zc = ZCache(lat_b, pb)
    ba, bb = DeviateBuffer(BufferKind.UNIFORM01, seed=9), DeviateBuffer(BufferKind.UNIFORM01, seed=9)
    for _ in range(60):
        gibbs_sweep(lat_a, pa, ba)
        gibbs_sweep_diff(lat_b, pb, zc, bb)
        np.testing.assert_array_equal(lat_a.s, lat_b.s)
    zc.validate(lat_b, pb)
    assert ba.position == bb.position


def test_diff_zero_flips_and_desync_detection(gpu):
    lat = IsingLattice(np.ones((6, 6), dtype=np.int8), 50.0 * np.ones((6, 6)), 0.0)
    part = color_lattice(lat)
    zc = ZCache(lat, part)
    before = [zc.nsum(c).copy() for c in (0, 1)]
    gibbs_sweep_diff(lat, part, zc, DeviateBuffer(BufferKind.UNIFORM01, seed=3))
    assert zc.flips_last_sweep == 0 and zc.flip_rate == 0.0
    for c in (0, 1):
        np.testing.assert_array_equal(zc.nsum(c), before[c])
    # a plain sweep behind the cache's back desynchronises it (ising.py:195-196)
    lat2 = IsingLattice(ising_spins(10, 10, seed=1), np.zeros((10, 10)), 0.2)
    p2 = color_lattice(lat2)
    zc2 = ZCache(lat2, p2)
    gibbs_sweep(lat2, p2, DeviateBuffer(BufferKind.UNIFORM01, seed=4))
    with pytest.raises(AssertionError):
        zc2.validate(lat2, p2)


def test_flip_counts_equal_changed_sites_many_sweeps(gpu):
    # per-sweep flips against the oracle's trajectory, generic + periodic Philox4x32 lattice
    s0 = ising_spins(64, 96, seed=5)
    lat = IsingLattice(s0, np.full(s0.shape, 0.1), 0.44, boundary="periodic")
    part = color_lattice(lat)
    zc = ZCache(lat, part)
    flips = gibbs_sweeps_diff(lat, part, zc, SitePhilox(seed=77), 8)
    s = s0
    for t in range(8):
        nxt = go.ising_sweeps(s, np.full(s0.shape, 0.1), 0.44, True, 1, go.RNG_PHILOX4X32, 77, 0, t)
        assert flips[t] == np.count_nonzero(nxt != s), t
        s = nxt
    np.testing.assert_array_equal(lat.s, s)
    assert zc.validate(lat, part) == 0.0


def test_denoise_against_oracle_larger(gpu):
    noisy = flip_noise(synthetic_binary_image(200, 301), 0.12, seed=21)
    buf = DeviateBuffer(BufferKind.UNIFORM01, seed=22)
    k0, k1 = buf.stream_key()
    trace = []
    out = denoise(noisy, w=0.9, bias_scale=1.7, sweeps=14, burnin=5, seed=22, trace_out=trace)
    ref, flips = go.denoise(noisy, 0.9, 1.7, 14, 5, k0, k1)
    np.testing.assert_array_equal(out, ref)
    np.testing.assert_array_equal(np.array(trace) * noisy.size, flips)


def test_denoise_reference_behaviour(gpu):
    # test_ising.py:260-297 restated on the device path
    img = synthetic_binary_image(24, 24)
    np.testing.assert_array_equal(denoise(img, w=1.0, bias_scale=8.0, sweeps=12, burnin=4, seed=1), img)
    img = synthetic_binary_image(64, 64)
    noisy = flip_noise(img, 0.1, seed=3)
    trace = []
    out = denoise(noisy, w=1.0, bias_scale=2.0, sweeps=30, burnin=10, seed=4, trace_out=trace)
    assert float((out != img).mean()) < float((noisy != img).mean())
    assert len(trace) == 30 and max(trace[10:]) < 0.25
    ones = synthetic_binary_image(48, 48, kind="all_ones")
    out = denoise(flip_noise(ones, 0.1, seed=7), w=1.0, bias_scale=2.0, sweeps=25, burnin=8, seed=8)
    assert float((out != ones).mean()) < 0.01


def test_denoise_full_size_properties(gpu):
    # 2048 x 2048: ties go to +1, flips equal the number of changed sites, output in {0,1}
    img = synthetic_binary_image(2048, 2048)
    noisy = flip_noise(img, 0.1, seed=31)
    trace = []
    out = denoise(noisy, sweeps=6, burnin=2, seed=32, trace_out=trace)
    assert out.shape == img.shape and set(np.unique(out)) <= {0, 1}
    assert float((out != img).mean()) < 0.5 * float((noisy != img).mean())
    assert len(trace) == 6 and all(0.0 < t < 0.5 for t in trace)


def test_sweeps_acc_accumulates_states(gpu):
    # the accumulator sums the new values of every sweep >= acc_from (Ising and Potts)
    s0 = ising_spins(32, 32, seed=9)
    lat = IsingLattice(s0, np.zeros(s0.shape), 0.3, boundary="periodic")
    part = color_lattice(lat)
    acc = np.zeros(s0.size, dtype=np.int32)
    flips = part.device.sweeps_acc(5, 2, 11, 0, 0, None, 2, acc)
    s, ref = s0, np.zeros(s0.shape, dtype=np.int64)
    for t in range(5):
        nxt = go.ising_sweeps(s, None, 0.3, True, 1, go.RNG_PHILOX4X32, 11, 0, t)
        assert flips[t] == np.count_nonzero(nxt != s)
        if t >= 2:
            ref += nxt
        s = nxt
    np.testing.assert_array_equal(acc.reshape(s0.shape), ref)
    part.device.close()
