"""Device parity of the checkerboard Gibbs sweep: bit-exact spins given the same uniforms."""

import numpy as np
import pytest

from conftest import golden
from oracle import gibbs_oracle as go
from paper_1310_1537_b200 import ising
from paper_1310_1537_b200.ising import IsingLattice, PottsLattice, color_lattice, gibbs_sweep, gibbs_sweeps
from paper_1310_1537_b200.rng import BufferKind, DeviateBuffer, SitePhilox
from paper_1310_1537_b200.synthetic import ising_spins, potts_states

pytestmark = pytest.mark.gpu


def test_free_boundary_matches_reference_sweeps(gpu):
    z = golden("ising.npz")
    for i in range(int(z["n_cases"])):
        h, w, sweeps, seed = (int(v) for v in z[f"meta_{i}"])
        lat = IsingLattice(z[f"s0_{i}"], z[f"b_{i}"], float(z[f"w_{i}"]))
        part = color_lattice(lat)
        buf = DeviateBuffer(BufferKind.UNIFORM01, seed=seed)
        for _ in range(sweeps):
            gibbs_sweep(lat, part, buf)
        np.testing.assert_array_equal(lat.s, z[f"s1_{i}"], err_msg=f"case {i}")
        assert buf.position == sweeps * h * w


def test_batched_sweeps_equal_single_sweeps_and_buffer_continues(gpu):
    z = golden("ising.npz")
    lat = IsingLattice(z["s0_7"], z["b_7"], float(z["w_7"]))
    part = color_lattice(lat)
    buf = DeviateBuffer(BufferKind.UNIFORM01, seed=77, capacity=100)
    gibbs_sweeps(lat, part, buf, 30)
    np.testing.assert_array_equal(lat.s, z["s1_7"])
    ref = DeviateBuffer(BufferKind.UNIFORM01, seed=77).take(30 * 16 * 12 + 5)
    np.testing.assert_array_equal(buf.take(5), ref[-5:])


def test_image_bias_matches_reference(gpu):
    z = golden("ising.npz")
    lat = IsingLattice(z["img_s0"], z["img_b"], 1.0)
    part = color_lattice(lat)
    buf = DeviateBuffer(BufferKind.UNIFORM01, seed=9)
    gibbs_sweeps(lat, part, buf, 60)
    np.testing.assert_array_equal(lat.s, z["img_s1"])


class _HostUniforms:
    """Duck-typed buffer (only .take) -> PM_RNG_UNIFORMS path."""

    def __init__(self, seed):
        self.buf = DeviateBuffer(BufferKind.UNIFORM01, seed=seed)

    def take(self, n):
        return self.buf.take(n)


def test_host_uniform_path_matches_reference(gpu):
    z = golden("ising.npz")
    for i in (0, 5, 8):
        h, w, sweeps, seed = (int(v) for v in z[f"meta_{i}"])
        lat = IsingLattice(z[f"s0_{i}"], z[f"b_{i}"], float(z[f"w_{i}"]))
        part = color_lattice(lat)
        src = _HostUniforms(seed)
        for _ in range(sweeps):
            gibbs_sweep(lat, part, src)
        np.testing.assert_array_equal(lat.s, z[f"s1_{i}"])


def test_periodic_matches_reference_with_wrapped_table(gpu):
    z = golden("periodic.npz")
    for i in range(int(z["n_cases"])):
        h, w, sweeps, seed = (int(v) for v in z[f"meta_{i}"])
        cw, cb = (float(v) for v in z[f"wb_{i}"])
        lat = IsingLattice(z[f"s0_{i}"], np.full((h, w), cb), cw, boundary="periodic")
        part = color_lattice(lat)
        gibbs_sweeps(lat, part, SitePhilox(seed), sweeps)
        np.testing.assert_array_equal(lat.s, z[f"s1_{i}"], err_msg=f"case {i}")


@pytest.mark.parametrize("shape", [(32, 32), (64, 96), (2, 32), (512, 512)])
def test_packed_fast_path_matches_c_oracle(gpu, shape):
    s0 = ising_spins(*shape, seed=3)
    sweeps = 1000 if shape == (512, 512) else 50
    lat = IsingLattice(s0, np.zeros(shape), 0.8814, boundary="periodic")
    part = color_lattice(lat)
    assert part.device.fast_path()
    gibbs_sweeps(lat, part, SitePhilox(2024), sweeps)
    ref = go.ising_sweeps(s0, None, 0.8814, True, sweeps, go.RNG_PHILOX4X32, 2024, 0, 0)
    np.testing.assert_array_equal(lat.s, ref)


def test_fast_and_generic_paths_agree(gpu):
    # biased lattice forces the generic kernel; compare against the fast path at b == 0
    s0 = ising_spins(64, 64, seed=4)
    a = IsingLattice(s0, np.zeros((64, 64)), 0.6, boundary="periodic")
    pa = color_lattice(a)
    assert pa.device.fast_path()
    gibbs_sweeps(a, pa, SitePhilox(5, sweep=7), 20)
    b = IsingLattice(s0, np.zeros((64, 64)), 0.6, boundary="periodic")
    pb = color_lattice(b)
    u = np.concatenate([go.site_uniforms(5, 7 + t, 64 * 64) for t in range(20)])
    pb.device.sweeps(20, 0, uniforms=u)  # PM_RNG_UNIFORMS on the generic kernel
    pb.unpack_into(b)
    np.testing.assert_array_equal(a.s, b.s)


def test_odd_width_and_random_bias_against_oracle(gpu):
    gen = np.random.default_rng(8)
    for shape in ((7, 9), (13, 1), (1, 13), (31, 33)):
        s0 = gen.choice([-1, 1], size=shape).astype(np.int8)
        b = gen.normal(0, 0.8, size=shape)
        lat = IsingLattice(s0, b, 0.9)
        part = color_lattice(lat)
        buf = DeviateBuffer(BufferKind.UNIFORM01, seed=42)
        k0, k1 = buf.stream_key()
        gibbs_sweeps(lat, part, buf, 17)
        ref = go.ising_sweeps(s0, b, 0.9, False, 17, go.RNG_NUMPY_PHILOX, k0, k1, 0)
        np.testing.assert_array_equal(lat.s, ref)


# packed fast path: (32, 32) -> 16-site groups NG=1, (96, 64) -> NG=2, (64, 128) -> NG=4;
# coupling 40 puts thresholds at 2^32 (cdf rounds to 1), so the 64-bit threshold table is used
@pytest.mark.parametrize("periodic,shape,coupling", [(True, (32, 32), 1.0986), (True, (64, 128), 1.0986),
                                                     (True, (96, 64), 1.0986), (False, (9, 11), 1.0986),
                                                     (True, (6, 10), 1.0986), (False, (32, 64), 1.0986),
                                                     (True, (64, 128), 40.0), (True, (96, 64), 40.0)])
def test_potts_matches_c_oracle(gpu, periodic, shape, coupling):
    s0 = potts_states(*shape, seed=1)
    lat = PottsLattice(s0, coupling, boundary="periodic" if periodic else "free")
    part = color_lattice(lat)
    ising.potts_sweeps(lat, part, SitePhilox(77), 40)
    ref = go.potts_sweeps(s0, coupling, periodic, 40, go.RNG_PHILOX4X32, 77, 0, 0)
    np.testing.assert_array_equal(lat.s, ref)


def test_config4_lattice_first_sweeps_against_oracle(gpu):
    """BASELINE config 4 exactly: 8192^2 periodic Ising, w = 2 x 0.4407 (J=1), h=0,
    Philox4x32 keyed by (seed, sweep, site): the first 10 sweeps bit-exact against the C
    oracle given the same uniforms, checked after sweep 1, 3 and 10."""
    s0 = ising_spins(8192, 8192, seed=0)
    lat = IsingLattice(s0, np.zeros((8192, 8192)), 0.8814, boundary="periodic")
    part = color_lattice(lat)
    assert part.device.fast_path()
    rng = SitePhilox(1)
    ref = s0
    done = 0
    for upto in (1, 3, 10):
        gibbs_sweeps(lat, part, rng, upto - done)
        ref = go.ising_sweeps(ref, None, 0.8814, True, upto - done, go.RNG_PHILOX4X32, 1, 0, done)
        done = upto
        np.testing.assert_array_equal(lat.s, ref, err_msg=f"after sweep {upto}")


def test_potts_config4_first_sweeps_against_oracle(gpu):
    """The config-4 Potts q=4 variant at its exact shape (8192^2 periodic, coupling 0.4407):
    the first 2 sweeps bit-exact against the C oracle (and one sweep at 2048^2)."""
    for shape, sweeps in (((2048, 2048), 1), ((8192, 8192), 2)):
        s0 = potts_states(*shape, seed=2)
        lat = PottsLattice(s0, 0.4407)
        part = color_lattice(lat)
        assert part.device.fast_path()
        ising.potts_sweeps(lat, part, SitePhilox(3), sweeps)
        ref = go.potts_sweeps(s0, 0.4407, True, sweeps, go.RNG_PHILOX4X32, 3, 0, 0)
        np.testing.assert_array_equal(lat.s, ref, err_msg=str(shape))


def test_single_node_and_zero_coupling(gpu):
    lat = IsingLattice([[1]], [[0.3]], 0.5)
    part = color_lattice(lat)
    gibbs_sweep(lat, part, DeviateBuffer(BufferKind.UNIFORM01, seed=0))
    assert lat.s[0, 0] in (-1, 1)
    lat = IsingLattice(np.ones((16, 16), dtype=np.int8), np.zeros((16, 16)), 0.0)
    part = color_lattice(lat)
    total = 0.0
    buf = DeviateBuffer(BufferKind.UNIFORM01, seed=30)
    for _ in range(200):
        gibbs_sweeps(lat, part, buf, 10)
        total += float(lat.s.sum())
    assert abs(total / (200 * 256)) < 0.05


def _local_exchange(strips, colour):
    """In-process halo exchange between strips on one GPU (the NCCL schedule's data flow)."""
    n = len(strips)
    for k, s in enumerate(strips):
        up, down = strips[(k - 1) % n], strips[(k + 1) % n]
        s.row(colour, 0).copy_(up.row(colour, up.rows))
        s.row(colour, s.rows + 1).copy_(down.row(colour, 1))


@pytest.mark.parametrize("n_strips,model", [(1, "ising"), (2, "ising"), (3, "ising"), (4, "potts"), (5, "ising")])
def test_strips_match_single_lattice(gpu, n_strips, model):
    import torch
    from paper_1310_1537_b200.dist import LatticeStrip, strip_bounds
    H, W, sweeps, seed = 96, 64, 20, 31
    full = ising_spins(H, W, seed=6) if model == "ising" else potts_states(H, W, seed=6)
    strips = []
    for k in range(n_strips):
        a, b = strip_bounds(H, n_strips, k)
        s = LatticeStrip(H, W, a, b - a, 0, model=model, w=0.8814, coupling=1.0986)
        s.set_spins(full[a:b])
        strips.append(s)
    for c in (0, 1):
        _local_exchange(strips, c)
    for t in range(sweeps):
        for c in (0, 1):
            for s in strips:
                s.half_sweep(c, seed, t)
            _local_exchange(strips, c)
    torch.cuda.synchronize()
    got = np.concatenate([s.get_spins() for s in strips], axis=0)
    if model == "ising":
        ref = go.ising_sweeps(full, None, 0.8814, True, sweeps, go.RNG_PHILOX4X32, seed, 0, 0)
    else:
        ref = go.potts_sweeps(full, 1.0986, True, sweeps, go.RNG_PHILOX4X32, seed, 0, 0)
    np.testing.assert_array_equal(got, ref)


def test_partition_accessors_match_reference(gpu):
    # ColorPartition.packed_s / neighbor_spin_sum (ising.py:134-150) after the reference's
    # 60-sweep image trajectory, read back from the device state
    z = golden("ising.npz")
    lat = IsingLattice(z["img_s0"], z["img_b"], 1.0)
    part = color_lattice(lat)
    buf = DeviateBuffer(BufferKind.UNIFORM01, seed=9)
    gibbs_sweeps(lat, part, buf, 60)
    np.testing.assert_array_equal(lat.s, z["img_s1"])
    np.testing.assert_array_equal(part.neighbor_spin_sum(0), z["img_nsum0"])
    np.testing.assert_array_equal(part.neighbor_spin_sum(1), z["img_nsum1"])
    np.testing.assert_array_equal(part.packed_s[0], z["img_packed0"])
    np.testing.assert_array_equal(part.packed_s[1], z["img_packed1"])
    assert lat.log_weight() == float(z["img_logw"])


@pytest.mark.parametrize("n_strips,model", [(1, "ising"), (2, "ising"), (3, "potts"), (5, "ising")])
def test_strips_peer_halo_exchange_match_single_lattice(gpu, n_strips, model):
    """Strips exchanging halo rows through peer memory (the half-sweep kernels store their
    boundary rows into the neighbours' double-buffered mailboxes and raise flags; no host
    copies): here all strips live on one GPU with same-process mailbox pointers.  A
    half-sweep waits only for the neighbours' deposits of the previous half-sweep, so all
    strips' launches go in order on ONE stream (kernels that wait on a running kernel must
    not share a GPU).  Bit-identical to one lattice, and no wait timed out."""
    import torch
    from paper_1310_1537_b200.dist import LatticeStrip, strip_bounds
    H, W, sweeps, seed = 96, 128, 20, 41
    full = ising_spins(H, W, seed=8) if model == "ising" else potts_states(H, W, seed=8)
    strips = []
    for k in range(n_strips):
        a, b = strip_bounds(H, n_strips, k)
        s = LatticeStrip(H, W, a, b - a, 0, model=model, w=0.8814, coupling=1.0986)
        s.set_spins(full[a:b])
        strips.append(s)
    st = torch.cuda.Stream(device=0)
    boxes = [s.xchg_mailbox() for s in strips]
    for k, s in enumerate(strips):
        s.xchg_set_peers(up=boxes[(k - 1) % n_strips], down=boxes[(k + 1) % n_strips])
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for s in strips:
            s.xchg_start()
        for t in range(sweeps):
            for c in (0, 1):
                for s in strips:
                    s.half_sweep(c, seed, t)
    torch.cuda.synchronize()
    assert not any(s.xchg_timed_out() for s in strips)
    got = np.concatenate([s.get_spins() for s in strips], axis=0)
    if model == "ising":
        ref = go.ising_sweeps(full, None, 0.8814, True, sweeps, go.RNG_PHILOX4X32, seed, 0, 0)
    else:
        ref = go.potts_sweeps(full, 1.0986, True, sweeps, go.RNG_PHILOX4X32, seed, 0, 0)
    np.testing.assert_array_equal(got, ref)
    for s in strips:
        s.close()


@pytest.mark.parametrize("model", ["ising", "potts"])
def test_set_spins_rejects_invalid_values_on_device(gpu, model):
    """pm_lat_set_spins validates on the device before touching the lattice: an invalid
    value raises ValueError (the reference's check, ising.py:64-70) and the state stays."""
    if model == "ising":
        s0 = ising_spins(64, 96, seed=4)
        lat = IsingLattice(s0, np.zeros(s0.shape), 0.5, boundary="periodic")
    else:
        s0 = potts_states(64, 96, seed=4)
        lat = PottsLattice(s0, 0.7, boundary="periodic")
    part = color_lattice(lat)
    dev = part.device
    dev.set_spins(s0)
    invalid = (0, 5, -2) if model == "ising" else (-1, 5, 4)
    for pos, v in zip(((0, 0), (63, 95), (17, 33)), invalid):
        bad = s0.copy()
        bad[pos] = v
        with pytest.raises(ValueError):
            dev.set_spins(bad)
        np.testing.assert_array_equal(dev.get_spins(), s0)


@pytest.mark.parametrize("model", ["ising", "potts"])
def test_coupling_change_between_sweeps_is_used(gpu, model):
    """The reference reads lat.w on every half-sweep (ising.py:184; the bias is the
    partition's packed_b snapshot), so an annealing caller that changes the coupling between
    sweep calls must see the new value: 4 sweeps at one coupling, then 5 at another, bit-exact
    against the oracle run in the same two segments (periodic packed path and free-boundary
    generic path)."""
    for periodic in (True, False):
        bnd = "periodic" if periodic else "free"
        if model == "ising":
            s0 = ising_spins(64, 128, seed=12)
            b = np.random.default_rng(2).normal(0, 0.3, s0.shape) if not periodic else np.zeros(s0.shape)
            lat = IsingLattice(s0, b, 0.3, boundary=bnd)
        else:
            s0 = potts_states(64, 128, seed=12)
            lat = PottsLattice(s0, 0.4, boundary=bnd)
        part = color_lattice(lat)
        rng = SitePhilox(99)
        gibbs_sweeps(lat, part, rng, 4)
        if model == "ising":
            lat.w = 1.2
            ref = go.ising_sweeps(s0, None if periodic else b, 0.3, periodic, 4, go.RNG_PHILOX4X32, 99, 0, 0)
            ref = go.ising_sweeps(ref, None if periodic else b, 1.2, periodic, 5, go.RNG_PHILOX4X32, 99, 0, 4)
        else:
            lat.coupling = 1.3
            ref = go.potts_sweeps(s0, 0.4, periodic, 4, go.RNG_PHILOX4X32, 99, 0, 0)
            ref = go.potts_sweeps(ref, 1.3, periodic, 5, go.RNG_PHILOX4X32, 99, 0, 4)
        gibbs_sweeps(lat, part, rng, 5)
        np.testing.assert_array_equal(lat.s, ref, err_msg=bnd)


@pytest.mark.parametrize("model", ["ising", "potts"])
def test_smem_staged_half_sweep_bit_exact(gpu, tune, model):
    """The shared-memory neighbour-staging A/B variant (tune gibbs_smem=1: 8-row CTAs stage
    the other colour's rows once) gives the same spins as the oracle, incl. the periodic
    wrap of the staged rows / edge bytes and a row count that is not a multiple of 8."""
    tune(gibbs_smem=1)
    for shape in ((68, 256), (64, 2048)):
        s0 = ising_spins(*shape, seed=6) if model == "ising" else potts_states(*shape, seed=6)
        lat = (IsingLattice(s0, np.zeros(shape), 0.8814, boundary="periodic") if model == "ising"
               else PottsLattice(s0, 0.4407))
        part = color_lattice(lat)
        assert part.device.fast_path()
        gibbs_sweeps(lat, part, SitePhilox(13), 6)
        ref = (go.ising_sweeps(s0, None, 0.8814, True, 6, go.RNG_PHILOX4X32, 13, 0, 0) if model == "ising"
               else go.potts_sweeps(s0, 0.4407, True, 6, go.RNG_PHILOX4X32, 13, 0, 0))
        np.testing.assert_array_equal(lat.s, ref, err_msg=str(shape))
