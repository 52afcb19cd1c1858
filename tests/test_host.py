"""CPU tests of the host-side mirror of the reference interface (validation,
layouts, streams, error behaviour).  No kernel is launched."""

import numpy as np
import pytest

from conftest import golden
from paper_1310_1537_b200 import _lib
from paper_1310_1537_b200.glm import DesignMatrix, ExecPlan, Strategy, make_sharded
from paper_1310_1537_b200.ising import IsingLattice, PottsLattice
from paper_1310_1537_b200.parallel import partition
from paper_1310_1537_b200.rng import BufferKind, DeviateBuffer, SitePhilox
from paper_1310_1537_b200.sampler import ChainConfig, GaussianPrior
from paper_1310_1537_b200.synthetic import baseline_design, hb_design


def test_partition_rule_matches_reference():
    # parallel.py:30-46: first n % workers blocks take one extra element
    assert partition(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert partition(2, 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    with pytest.raises(ValueError):
        partition(5, 0)


def test_design_matrix_validation():
    with pytest.raises(ValueError):
        DesignMatrix([[1.0]], [2.0])
    with pytest.raises(ValueError):
        DesignMatrix([[np.nan]], [1.0])
    with pytest.raises(ValueError):
        DesignMatrix(np.empty((0, 2)), [])
    with pytest.raises(ValueError):
        DesignMatrix([[1.0], [2.0]], [1.0])
    d = DesignMatrix([[1.0, 2.0]], [1.0])
    assert not d.x.flags.writeable and not d.y.flags.writeable


def test_exec_plan_validation():
    with pytest.raises(ValueError):
        ExecPlan(workers=0)
    with pytest.raises(ValueError):
        ExecPlan(n_chunks=0)
    with pytest.raises(ValueError):
        ExecPlan(x_storage="f16")
    assert ExecPlan(Strategy.B200).strategy is Strategy.B200


def test_make_sharded_layout():
    x = np.arange(10.0).reshape(5, 2)
    d = DesignMatrix(x, [0, 1, 0, 1, 1])
    v = make_sharded(d, 2)
    assert [s.x.shape[0] for s in v.shards] == [3, 2]
    assert [s.row_offset for s in v.shards] == [0, 3]
    assert not np.shares_memory(v.shards[0].x, d.x)
    with pytest.raises(ValueError):
        make_sharded(d, 6)


def test_prior_and_chain_config_validation():
    with pytest.raises(ValueError):
        GaussianPrior(np.zeros(2), np.array([1.0, 0.0]))
    for bad in (dict(n_iter=0, n_burnin=0), dict(n_iter=5, n_burnin=5),
                dict(n_iter=5, n_burnin=0, slice_width=0.0), dict(n_iter=5, n_burnin=0, slice_max_steps=0)):
        with pytest.raises(ValueError):
            ChainConfig(**bad)
    p = GaussianPrior.isotropic(3, 1.0, 2.0)
    assert p.logpdf_coord(0, 3.0) == -0.5


def test_deviate_buffer_stream_matches_reference_fixture():
    z = golden("rng.npz")
    for seed in (0, 5, 33):
        for cap in (1, 7, 64, 4096):
            buf = DeviateBuffer(BufferKind.UNIFORM01, capacity=cap, seed=seed)
            np.testing.assert_array_equal(buf.take(1000), z[f"u{seed}"])
        key = DeviateBuffer(BufferKind.UNIFORM01, seed=seed).stream_key()
        assert key == tuple(int(v) for v in z[f"key{seed}"])
    buf = DeviateBuffer(BufferKind.UNIFORM01, capacity=16, seed=17, owner=(3,))
    np.testing.assert_array_equal(buf.take(100), z["u17_3"])


@pytest.mark.parametrize("cap", [1, 5, 64, 8192])
def test_deviate_buffer_skip_and_position(cap):
    ref = DeviateBuffer(BufferKind.UNIFORM01, capacity=4096, seed=3).take(5000)
    buf = DeviateBuffer(BufferKind.UNIFORM01, capacity=cap, seed=3)
    pos = 0
    for n_skip, n_take in ((0, 3), (7, 1), (1000, 9), (2, 50), (3001, 4)):
        buf.skip(n_skip)
        pos += n_skip
        assert buf.position == pos
        np.testing.assert_array_equal(buf.take(n_take), ref[pos:pos + n_take])
        pos += n_take
        assert buf.position == pos
    assert buf.next() == ref[pos]


def test_site_philox_advances():
    s = SitePhilox(seed=2 ** 64 + 5, sweep=3)
    assert s.seed == 5
    s.advance(10)
    assert s.sweep == 13


def test_lattice_validation():
    with pytest.raises(ValueError):
        IsingLattice(np.zeros((2, 2)), np.zeros((2, 2)), 1.0)
    with pytest.raises(ValueError):
        IsingLattice(np.ones((3, 4)), np.zeros((3, 4)), 1.0, boundary="periodic")
    with pytest.raises(ValueError):
        IsingLattice(np.ones((2, 2)), np.zeros((2, 3)), 1.0)
    with pytest.raises(ValueError):
        PottsLattice(np.full((2, 2), 4), 1.0)
    lat = IsingLattice.from_image(np.array([[0, 1], [1, 1]]), 1.0, 2.0)
    assert lat.s.tolist() == [[-1, 1], [1, 1]] and lat.b[0, 0] == -2.0


def test_baseline_generators_follow_survey_recipe():
    x, y, bt, be = baseline_design(100, 5, seed=1)
    assert np.all(x[:, 0] == 1.0) and set(np.unique(y)) <= {0.0, 1.0}
    # chunked generation is stream-identical to a single call
    x2, y2, _, _ = baseline_design(100, 5, seed=1, chunk_rows=7)
    np.testing.assert_array_equal(x, x2)
    np.testing.assert_array_equal(y, y2)
    xs, ys, off, betas, mu, tau = hb_design(20, 4, seed=3, mean_rows=50)
    assert off[0] == 0 and off[-1] == xs.shape[0] and betas.shape == (20, 4) and tau == 0.3


def test_device_calls_fail_loudly_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("a device is visible")
    d = DesignMatrix([[1.0, 2.0]], [1.0])
    from paper_1310_1537_b200.glm import loglike_grad
    with pytest.raises(RuntimeError, match="no CUDA device"):
        loglike_grad(d, np.zeros(2))


def test_log_weight_matches_reference_fixture():
    # IsingLattice.log_weight (ising.py:84-93) on the reference's own trajectories
    from paper_1310_1537_b200.ising import IsingLattice
    z = golden("ising.npz")
    for i in range(int(z["n_cases"])):
        lat = IsingLattice(z[f"s1_{i}"], z[f"b_{i}"], float(z[f"w_{i}"]))
        assert lat.log_weight() == pytest.approx(float(z["logw_cases"][i]), rel=1e-14, abs=1e-12)
    lat = IsingLattice(z["img_s1"], z["img_b"], 1.0)
    assert lat.log_weight() == pytest.approx(float(z["img_logw"]), rel=1e-14)
    # explicit state argument and a periodic lattice counting the wrap edges
    s = np.array([[1, -1], [1, 1]], dtype=np.int8)
    per = IsingLattice(s, np.zeros((2, 2)), 0.5, boundary="periodic")
    assert per.log_weight() == 0.5 * 0.5 * (2 * (1 * 1 + (-1) * 1) + 2 * (1 * -1 + 1 * 1))


def test_potts_compact_code_sums_are_unique():
    """The packed Potts kernel indexes its threshold table by the sum of per-neighbour codes
    {0, 1, 5, 21}[state] (ising.cu kPottsCodeBytes; the packed arrays store these codes): the 35 neighbour multisets of q=4 states
    over 4 neighbours must give distinct sums that fit one byte and the 85-entry table."""
    import itertools
    codes = (0, 1, 5, 21)
    sums = {}
    for ms in itertools.combinations_with_replacement(range(4), 4):
        e = sum(codes[a] for a in ms)
        assert e not in sums, (ms, sums.get(e))
        sums[e] = ms
    assert len(sums) == 35 and max(sums) == 84
    # the byte constant holds the codes in state order
    assert [(0x15050100 >> (8 * a)) & 0xFF for a in range(4)] == list(codes)
