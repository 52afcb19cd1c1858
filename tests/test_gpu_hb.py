"""Device parity of the batched hierarchical (per-group) log-posterior + gradient."""

import numpy as np
import pytest

from conftest import golden
from oracle import glm_oracle as gl
from paper_1310_1537_b200.glm import DesignMatrix
from paper_1310_1537_b200.hb import CsrGroups, HbDataset, hb_log_posterior_grad
from paper_1310_1537_b200.sampler import GaussianPrior
from paper_1310_1537_b200.synthetic import hb_design

pytestmark = pytest.mark.gpu
TOL = 1e-10


def check(f, g, fr, gr):
    assert np.max(np.abs(f - fr) / np.maximum(np.abs(fr), 1.0)) < TOL
    assert np.max(np.abs(g - gr) / np.maximum(np.abs(gr), 1.0)) < TOL


def test_reference_fixture(gpu):
    z = golden("hb.npz")
    csr = CsrGroups(z["x"], z["y"], z["offsets"])
    res = hb_log_posterior_grad(csr, z["betas"], GaussianPrior(z["mu"], z["sigma"]))
    check(np.array([r.f for r in res]), np.stack([r.g for r in res]), z["f"], z["g"])


def test_dataset_of_design_matrices(gpu):
    gen = np.random.default_rng(0)
    groups = [DesignMatrix(gen.standard_normal((n, 6)), (gen.random(n) < 0.4).astype(float))
              for n in (1, 31, 32, 33, 100, 7)]
    ds = HbDataset(groups)
    betas = gen.normal(0, 0.5, (6, 6))
    res = hb_log_posterior_grad(ds, betas)
    for m, grp in enumerate(groups):
        f, g = gl.loglike_grad(grp.x, grp.y, betas[m])
        assert abs(res[m].f - f) / max(abs(f), 1) < TOL
        assert np.max(np.abs(res[m].g - g) / np.maximum(np.abs(g), 1)) < TOL


def test_config3_shape_against_oracle(gpu):
    x, y, off, betas, mu, tau = hb_design(1000, 20, seed=3)
    csr = CsrGroups(x, y, off)
    prior = GaussianPrior(mu, np.full(20, tau))
    res = hb_log_posterior_grad(csr, betas, prior)
    f, g = gl.hb_log_posterior_grad(x, y, off, betas, mu, np.full(20, tau))
    check(np.array([r.f for r in res]), np.stack([r.g for r in res]), f, g)
    again = hb_log_posterior_grad(csr, betas, prior)
    assert all(a.f == b.f and np.array_equal(a.g, b.g) for a, b in zip(res, again))


def test_wide_k_and_validation(gpu):
    x, y, off, betas, mu, tau = hb_design(7, 100, seed=4, mean_rows=90)
    csr = CsrGroups(x, y, off)
    res = hb_log_posterior_grad(csr, betas)
    f, g = gl.hb_log_posterior_grad(x, y, off, betas)
    check(np.array([r.f for r in res]), np.stack([r.g for r in res]), f, g)
    with pytest.raises(ValueError):
        hb_log_posterior_grad(csr, betas[:3])
    with pytest.raises(ValueError):
        CsrGroups(x, y, np.array([0, 5, 5, x.shape[0]]))


@pytest.mark.parametrize("k", [2, 4, 20, 22, 32])
@pytest.mark.parametrize("layout", ["tiny_groups", "huge_groups", "single"])
def test_row_per_lane_path_segments(gpu, k, layout, tune):
    # even K <= 32 takes the row-per-lane kernel with balanced tile ranges: groups split across
    # CTAs (huge), many groups inside one CTA's range (tiny), one group over the whole grid
    gen = np.random.default_rng(k)
    sizes = {"tiny_groups": gen.integers(1, 40, 5000), "huge_groups": [100_000, 37, 250_001],
             "single": [77_777]}[layout]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    x = gen.standard_normal((int(off[-1]), k))
    y = (gen.random(int(off[-1])) < 0.45).astype(float)
    betas = gen.normal(0, 0.3, (len(sizes), k))
    mu, sigma = gen.normal(0, 0.5, k), np.full(k, 0.7)
    prior = GaussianPrior(mu, sigma)
    res = hb_log_posterior_grad(CsrGroups(x, y, off), betas, prior)
    f = np.array([r.f for r in res])
    g = np.stack([r.g for r in res])
    fr, gr = gl.hb_log_posterior_grad(x, y, off, betas, mu, sigma)
    check(f, g, fr, gr)
    res_f = hb_log_posterior_grad(CsrGroups(x, y, off), betas, prior, want_grad=False)
    np.testing.assert_array_equal(np.array([r.f for r in res_f]), f)
    # the column-per-lane kernel agrees to rounding
    tune(hb_rows=0)
    res0 = hb_log_posterior_grad(CsrGroups(x, y, off), betas, prior)
    check(np.array([r.f for r in res0]), np.stack([r.g for r in res0]), f, g)
