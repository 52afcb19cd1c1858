"""The NCCL evaluation path of DistributedDesign on one GPU (a 1-rank process group).

Multi-GPU runs are not available here; this exercises the exact device code path of a
rank -- rank-0 prior in the kernel, NCCL all-gather, the pm_fold_rows launch -- and
checks it against the single-GPU evaluation bit for bit (the fold of one partial is
that partial).  The multi-rank collective logic is covered by tests/test_dist_gloo.py.
"""

import os
import socket

import numpy as np
import pytest

from oracle import glm_oracle as gl
from paper_1310_1537_b200 import glm
from paper_1310_1537_b200.glm import DesignMatrix
from paper_1310_1537_b200.sampler import GaussianPrior

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_single_rank_matches_single_gpu_path(gpu):
    import torch
    import torch.distributed as dist
    from paper_1310_1537_b200 import _lib
    from paper_1310_1537_b200.dist import DistributedDesign
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        gen = np.random.default_rng(3)
        for n, k in ((1000, 7), (200_000, 20), (50_001, 100)):
            x = gen.standard_normal((n, k))
            y = (gen.random(n) < 0.4).astype(float)
            beta = gen.normal(0, 0.2, k)
            prior = GaussianPrior(gen.normal(0, 0.5, k), np.full(k, 3.0))
            d = DesignMatrix(x, y)
            single = glm.log_posterior_grad(d, beta, prior)
            dd = DistributedDesign(d, device=0)
            res = dd.log_posterior_grad(beta, prior)
            assert res.f == single.f and np.array_equal(res.g, single.g)
            f_ref, g_ref = gl.log_posterior_grad(x, y, beta, prior.mu, prior.sigma)
            assert abs(res.f - f_ref) / max(abs(f_ref), 1) < 1e-10
            no_prior = dd.log_posterior_grad(beta, None)
            assert no_prior.f == glm.loglike_grad(d, beta).f
        # the fold launch itself: ascending-row sum of a (world, width) device block
        blk = torch.randn(5, 33, dtype=torch.float64, device="cuda:0")
        out = torch.empty(33, dtype=torch.float64, device="cuda:0")
        _lib.call("pm_fold_rows", blk.data_ptr(), 5, 33, out.data_ptr(), None)
        torch.cuda.synchronize()
        ref = blk[0].clone()
        for r in range(1, 5):
            ref += blk[r]
        assert torch.equal(out, ref)
    finally:
        dist.destroy_process_group()


def test_nccl_single_rank_back_to_back_and_strip(gpu):
    # many evaluations queued back to back on torch's (legacy default) stream must each see
    # their own kernel's partial: the C ABI gets cudaStreamLegacy, not NULL (= handle stream)
    import torch
    import torch.distributed as dist
    from paper_1310_1537_b200.dist import DistributedDesign, LatticeStrip, strip_sweeps
    from paper_1310_1537_b200.ising import IsingLattice, color_lattice, gibbs_sweeps
    from paper_1310_1537_b200.rng import SitePhilox
    from paper_1310_1537_b200.synthetic import ising_spins
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        gen = np.random.default_rng(5)
        n, k = 2_000_000, 100
        x = gen.standard_normal((n, k))
        y = (gen.random(n) < 0.5).astype(float)
        d = DesignMatrix(x, y)
        dd = DistributedDesign(d, device=0)
        prior = GaussianPrior.isotropic(k, 0.0, 10.0)
        betas = gen.normal(0, 0.1, (12, k))
        outs = [dd.log_posterior_grad_device(b, prior) for b in betas]   # queued, no host sync
        torch.cuda.synchronize()
        for b, o in zip(betas, outs):
            single = glm.log_posterior_grad(d, b, prior)
            o = o.cpu().numpy()
            assert o[0] == single.f and np.array_equal(o[1:], single.g)
        # a 1-rank strip: half-sweeps and the wrap-around halo copies on torch's stream
        s0 = ising_spins(64, 128, seed=3)
        strip = LatticeStrip(64, 128, 0, 64, 0, model="ising", w=0.6)
        strip.set_spins(s0)
        strip_sweeps(strip, 25, 77, 0, 0, 1)
        lat = IsingLattice(s0, np.zeros(s0.shape), 0.6, boundary="periodic")
        gibbs_sweeps(lat, color_lattice(lat), SitePhilox(77), 25)
        np.testing.assert_array_equal(strip.get_spins(), lat.s)
        strip.close()
    finally:
        dist.destroy_process_group()
