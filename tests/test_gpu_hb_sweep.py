"""Device-resident hierarchical Gibbs sweep (pm_hbs_*) against the reference's hb_sweep.

tests/golden/hb_sweep.npz holds the unmodified reference's trajectories (HbState +
hb_sweep, hb.py:110-168); the oracle's run_chain on each group's owner stream is the
reference's own equivalence ("a single group's chain reproduces sampler.run_chain run
on the same stream", hb.py:14-17) and checks larger ragged cases.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import sampler_oracle as so
from paper_1310_1537_b200.glm import DesignMatrix
from paper_1310_1537_b200.hb import (HbDataset, HbState, MappingMode, MappingPolicy, hb_benchmark,
                                     hb_log_posterior_grad, hb_sweep, hb_sweeps, synthetic_hb_dataset)
from paper_1310_1537_b200.sampler import GaussianPrior, SliceWidenError

pytestmark = pytest.mark.gpu

DRAW_RTOL = 1e-9


def dataset(x, y, off):
    return HbDataset([DesignMatrix(x[off[g]:off[g + 1]], y[off[g]:off[g + 1]]) for g in range(off.size - 1)])


@pytest.mark.parametrize("c", [0, 1])
def test_hb_sweep_matches_reference_trajectory(gpu, c):
    z = golden("hb_sweep.npz")
    ds = dataset(z[f"x_{c}"], z[f"y_{c}"], z[f"off_{c}"])
    prior = GaussianPrior(z[f"prior_{c}"][0], z[f"prior_{c}"][1])
    seed, cap, neval, sweeps = (int(v) for v in z[f"meta_{c}"])
    st = HbState(ds, prior, seed=seed, buffer_capacity=cap)
    pol = MappingPolicy(MappingMode.COARSE, workers=1, neval=neval)
    for s in range(sweeps):
        betas = np.array(hb_sweep(ds, st, prior, pol))
        np.testing.assert_allclose(betas, z[f"betas_{c}"][s], rtol=DRAW_RTOL, atol=1e-12, err_msg=f"sweep {s}")
    assert st.total_evals == int(z[f"evals_{c}"])
    assert [b.consumed for b in st.buffers] == z[f"used_{c}"].tolist()
    assert [b.position for b in st.buffers] == z[f"used_{c}"].tolist()
    st.close()


def test_fused_sweeps_equal_single_sweeps_and_modes_agree(gpu):
    ds, _ = synthetic_hb_dataset(9, 4, 300, seed=2)
    prior = GaussianPrior.isotropic(4, sigma=2.0)
    a = HbState(ds, prior, seed=3)
    b = HbState(ds, prior, seed=3)
    for _ in range(4):
        ba = hb_sweep(ds, a, prior, MappingPolicy(MappingMode.COARSE, workers=4))
    bb = hb_sweeps(ds, b, prior, MappingPolicy(MappingMode.FINE, workers=2, neval=2), 4)
    np.testing.assert_array_equal(np.array(ba), np.array(bb))
    assert a.total_evals == b.total_evals
    assert [x.position for x in a.buffers] == [x.position for x in b.buffers]


def test_ragged_groups_against_oracle_chains(gpu):
    rng = np.random.default_rng(7)
    sizes = [1, 2, 31, 32, 33, 500, 2999, 64, 128, 1000]
    k = 5
    groups = []
    for n in sizes:
        x = rng.standard_normal((n, k))
        y = (rng.random(n) < 1 / (1 + np.exp(-x @ rng.normal(0, 0.7, k)))).astype(float)
        groups.append(DesignMatrix(x, y))
    ds = HbDataset(groups)
    prior = GaussianPrior(np.zeros(k), np.full(k, 1.5))
    st = HbState(ds, prior, seed=11)
    traj = [np.array(hb_sweep(ds, st, prior, MappingPolicy(MappingMode.FINE))) for _ in range(3)]
    total = 0
    for m, g in enumerate(groups):
        draws, evals = so.run_chain(g.x, g.y, prior.mu, prior.sigma, 3, 0, seed=11,
                                    rng=so.UniformStream(11, owner=(m,)))
        total += evals
        np.testing.assert_allclose(np.array([t[m] for t in traj]), draws, rtol=DRAW_RTOL, atol=1e-12,
                                   err_msg=f"group {m}")
    assert st.total_evals == total


def test_config3_scale_sweep_keeps_xbeta_consistent(gpu):
    # G=1000 groups of ~2000 rows, K=20 (config-3 shape): the maintained xbeta after a sweep
    # must reproduce the batched kernel's fresh likelihood at the returned coefficients
    ds, _ = synthetic_hb_dataset(1000, 20, 2000, seed=3)
    prior = GaussianPrior.isotropic(20, sigma=1.0)
    st = HbState(ds, prior, seed=4)
    st.sweeps(prior, 2)
    betas = np.array(st.betas)
    assert np.isfinite(betas).all()
    fresh = hb_log_posterior_grad(ds, betas, None, want_grad=False)
    f_fresh = np.array([r.f for r in fresh])
    np.testing.assert_allclose(st.loglike(), f_fresh, rtol=1e-10)
    assert st.last_kernel_ms > 0
    evals_per_update = st.total_evals / (2 * 1000 * 20)
    assert 4.0 < evals_per_update < 12.0


def test_errors_and_validation(gpu):
    ds, _ = synthetic_hb_dataset(3, 2, 40, seed=1)
    prior = GaussianPrior.isotropic(2)
    st = HbState(ds, prior, seed=1)
    with pytest.raises(SliceWidenError):
        hb_sweep(ds, st, prior, MappingPolicy(MappingMode.COARSE), slice_width=1e-9, slice_max_steps=1)
    with pytest.raises(ValueError):
        HbState(ds, GaussianPrior.isotropic(3))
    with pytest.raises(ValueError):
        MappingPolicy(MappingMode.FINE, workers=0)
    with pytest.raises(ValueError):
        st.sweeps(prior, 1, neval=0)
    # a new prior is taken up by the next sweep
    st2 = HbState(ds, prior, seed=2)
    other = GaussianPrior(np.array([0.5, -0.5]), np.array([0.05, 0.05]))
    betas = np.array(hb_sweep(ds, st2, other, MappingPolicy(MappingMode.COARSE)))
    for m, g in enumerate(ds.groups):
        draws, _ = so.run_chain(g.x, g.y, other.mu, other.sigma, 1, 0, rng=so.UniformStream(2, owner=(m,)),
                                beta0=prior.mu)
        np.testing.assert_allclose(betas[m], draws[0], rtol=DRAW_RTOL, atol=1e-12)


def test_hb_benchmark_records(gpu):
    ds, _ = synthetic_hb_dataset(20, 5, 500, seed=0)
    prior = GaussianPrior.isotropic(5)
    recs = hb_benchmark(ds, prior, [MappingPolicy(MappingMode.COARSE), MappingPolicy(MappingMode.FINE, neval=2)],
                        n_sweeps=2, reps=2)
    assert [r.label for r in recs] == ["hb/coarse/neval1", "hb/fine/neval2"]
    assert all(r.cpr > 0 and r.n_rows == 10_000 for r in recs)
