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
