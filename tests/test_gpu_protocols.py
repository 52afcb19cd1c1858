"""Hand-rolled device protocols without compute-sanitizer (the tool is closed on this GPU
pool, profiles/r02_sanitizer.txt): every kernel family with an mbarrier ring, an acq_rel
ticket or system-scope flags runs at small sizes against the oracle
(tools/sanitize_subset.py, the subset the sanitizer was meant to run), and the stream
kernel is repeated many times per consumer layout / stage geometry -- a stage released
too early or a mis-ordered flag shows up as run-to-run different bits (that is how the
r01 stage-reuse race was found)."""

import os
import sys

import numpy as np
import pytest

from paper_1310_1537_b200 import _lib, glm
from paper_1310_1537_b200.glm import DesignMatrix, ExecPlan
from paper_1310_1537_b200.sampler import GaussianPrior
from paper_1310_1537_b200.synthetic import baseline_design

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(ROOT, "tools"))


@pytest.mark.parametrize("family", ["glm_cases", "hb_cases", "gibbs_cases", "strip_cases", "xchg_cases",
                                    "chain_cases"])
def test_protocol_subset_against_oracle(gpu, family):
    import sanitize_subset
    getattr(sanitize_subset, family)()


@pytest.mark.parametrize("k,n,xs,knobs", [
    (32, 100_000, "f64", {}),                      # config 0: 2-tile units, producer thread
    (75, 260_000, "f64", {}),                      # odd K: column consumer, KC = 3, ring reuse
    (32, 100_000, "f64", {"stream_tps": 1}),       # single interleaved tiles
    (32, 700_001, "f64", {"stream_tps": 2}),       # ring reuse with 2-tile units, ragged tail
    (20, 300_000, "f64", {"glm_rows": 0}),         # narrow design through the column kernel
    (100, 300_000, "f64", {}),                     # pairs layout, ring reuse
    (100, 300_000, "f32", {}),                     # fp32-X row-dot consumer, 16 self-producing warps
    (100, 300_000, "f32", {"f32_selfprod": 1}),    # ... 15 self-producing warps, warp 0 idle
    (100, 300_000, "f32", {"f32_selfprod": 0}),    # ... with the producer thread
    (100, 300_000, "f32", {"stream_ncw": 7}),      # ... 8 warps, two stages each
    (100, 300_000, "f32", {"f32_pairs": 4}),       # row-dot by warp pairs (named barriers, count-2 release)
    (100, 300_000, "f32", {"f32_pairs": 1}),       # sub-tile pairs consumer
    (36, 150_001, "f32", {}),                      # row-dot, KC = 2, ragged tail
    (124, 90_000, "f32", {}),                      # row-dot, one stage per warp
    (64, 200_000, "f32", {"stream_tps": 4}),       # fp32-X, 4-tile units
    (33, 150_000, "f32", {}),                      # fp32-X column consumer (odd K)
])
def test_stream_kernel_repeats_bitwise(gpu, k, n, xs, knobs):
    from oracle import glm_oracle as gl
    with _lib.tuned(**knobs):
        x, y, _, betas = baseline_design(n, k, seed=n % 97 + k, n_eval=2)
        d = DesignMatrix(x, y)
        prior = GaussianPrior.isotropic(k, 0.0, 10.0)
        plan = ExecPlan(x_storage=xs)
        first = glm.log_posterior_grad(d, betas[0], prior, plan)
        xr = x.astype(np.float32).astype(np.float64) if xs == "f32" else x
        f, g = gl.log_posterior_grad(xr, y, betas[0], prior.mu, prior.sigma)
        assert abs(first.f - f) / max(abs(f), 1.0) < 1e-10
        assert np.max(np.abs(first.g - g) / np.maximum(np.abs(g), 1.0)) < 1e-10
        for i in range(60):
            other = glm.log_posterior_grad(d, betas[1], prior, plan)  # a different beta in between
            again = glm.log_posterior_grad(d, betas[0], prior, plan)
            assert again.f == first.f and np.array_equal(again.g, first.g), i
            assert other.f != first.f
        d.release_device()
