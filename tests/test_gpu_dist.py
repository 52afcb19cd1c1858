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


def _xchg(device, world, rank, width):
    import ctypes

    from paper_1310_1537_b200 import _lib
    h = ctypes.c_void_p()
    _lib.check(_lib.load().pm_xchg_create(device, world, rank, width, ctypes.byref(h)), "pm_xchg_create")
    return h


def _mailbox(h):
    import ctypes

    from paper_1310_1537_b200 import _lib
    p = ctypes.c_void_p()
    _lib.call("pm_xchg_mailbox", h, ctypes.byref(p))
    return p.value


def test_peer_exchange_single_rank_matches_single_gpu_path(gpu):
    """pm_glm_eval_xchg with world 1: the finishing CTA deposits into its own mailbox, raises
    its flag, waits and folds -- bit-identical to the plain evaluation, over many epochs
    (both mailbox parities), with and without the prior."""
    import ctypes

    import torch
    from paper_1310_1537_b200 import _lib
    gen = np.random.default_rng(8)
    n, k = 70_001, 100
    x = gen.standard_normal((n, k))
    y = (gen.random(n) < 0.5).astype(float)
    d = DesignMatrix(x, y)
    dev = d.on_device(0)
    prior = GaussianPrior(gen.normal(0, 0.5, k), np.full(k, 2.0))
    dev.set_prior(prior.mu, prior.sigma)
    xh = _xchg(0, 1, 0, k + 1)
    out = torch.empty(k + 1, dtype=torch.float64, device="cuda:0")
    try:
        for i in range(7):
            beta = gen.normal(0, 0.2, k)
            wp = i % 2 == 0
            if wp:  # the reference evaluations below reset the shared handle's prior
                dev.set_prior(prior.mu, prior.sigma)
            _lib.call("pm_glm_eval_xchg", dev.handle, _lib.dptr(beta), int(wp), xh,
                      ctypes.c_void_p(out.data_ptr()), None)  # the handle's own stream
            torch.cuda.synchronize()
            got = out.cpu().numpy()
            ref = glm.log_posterior_grad(d, beta, prior) if wp else glm.loglike_grad(d, beta)
            assert got[0] == ref.f and np.array_equal(got[1:], ref.g), i
        st = ctypes.c_int32()
        _lib.call("pm_xchg_status", xh, ctypes.byref(st))
        assert st.value == 0
    finally:
        _lib.load().pm_xchg_destroy(xh)


def test_peer_exchange_two_ranks_one_process(gpu):
    """Two row shards on one GPU, each with its own design handle and mailbox, exchanging
    through peer memory (same-process mailbox pointers).  Kernels that wait on one another
    must not share a GPU (nothing guarantees they are co-resident), so the split form is
    used: both ranks' phase-1 launches (stream + deposit + flags), then both phase-2
    launches (wait -- already satisfied -- and fold), all in order on one stream.  Both
    ranks must hold the ascending-rank fold of the two partials, bit-identical to the NCCL
    path's pm_fold_rows and within 1e-10 of the oracle."""
    import ctypes

    import torch
    from paper_1310_1537_b200 import _lib
    from paper_1310_1537_b200.parallel import partition
    gen = np.random.default_rng(9)
    n, k = 300_007, 100
    x = gen.standard_normal((n, k))
    y = (gen.random(n) < 0.5).astype(float)
    prior = GaussianPrior(gen.normal(0, 0.5, k), np.full(k, 2.0))
    shards = [DesignMatrix(x[a:b], y[a:b]) for a, b in partition(n, 2)]
    devs = [s.on_device(0) for s in shards]
    devs[0].set_prior(prior.mu, prior.sigma)
    xs = [_xchg(0, 2, r, k + 1) for r in range(2)]
    boxes = [_mailbox(h) for h in xs]
    for r in range(2):
        _lib.call("pm_xchg_set_peer_ptr", xs[r], 1 - r, ctypes.c_void_p(boxes[1 - r]))
    stream = torch.cuda.Stream(device=0)
    outs = [torch.empty(k + 1, dtype=torch.float64, device="cuda:0") for _ in range(2)]
    part = [torch.empty(k + 1, dtype=torch.float64, device="cuda:0") for _ in range(2)]
    try:
        # phase 2 before phase 1, and phase 1 twice, are refused
        beta = gen.normal(0, 0.2, k)
        with pytest.raises(RuntimeError):
            _lib.call("pm_glm_eval_xchg_phase", devs[0].handle, _lib.dptr(beta), 1, xs[0], 2,
                      ctypes.c_void_p(outs[0].data_ptr()), ctypes.c_void_p(stream.cuda_stream))
        for i in range(6):
            beta = gen.normal(0, 0.2, k)
            for phase in (1, 2):
                for r in range(2):
                    _lib.call("pm_glm_eval_xchg_phase", devs[r].handle, _lib.dptr(beta), int(r == 0), xs[r], phase,
                              ctypes.c_void_p(outs[r].data_ptr() if phase == 2 else None),
                              ctypes.c_void_p(stream.cuda_stream))
                if phase == 1 and i == 0:
                    with pytest.raises(RuntimeError):
                        _lib.call("pm_glm_eval_xchg_phase", devs[0].handle, _lib.dptr(beta), 1, xs[0], 1,
                                  None, ctypes.c_void_p(stream.cuda_stream))
            torch.cuda.synchronize()
            a, b = outs[0].cpu().numpy(), outs[1].cpu().numpy()
            assert np.array_equal(a, b), i
            # the NCCL path's fold of the same partials
            for r in range(2):
                devs[r].eval_device(beta, True, part[r].data_ptr(), 0, with_prior=(r == 0))
            torch.cuda.synchronize()
            blk = torch.stack(part)
            fold = torch.empty(k + 1, dtype=torch.float64, device="cuda:0")
            _lib.call("pm_fold_rows", blk.data_ptr(), 2, k + 1, fold.data_ptr(), None)
            torch.cuda.synchronize()
            assert np.array_equal(a, fold.cpu().numpy()), i
            f_ref, g_ref = gl.log_posterior_grad(x, y, beta, prior.mu, prior.sigma)
            assert abs(a[0] - f_ref) / max(abs(f_ref), 1) < 1e-10
            assert np.max(np.abs(a[1:] - g_ref) / np.maximum(np.abs(g_ref), 1)) < 1e-10
        for h in xs:
            st = ctypes.c_int32()
            _lib.call("pm_xchg_status", h, ctypes.byref(st))
            assert st.value == 0
    finally:
        for h in xs:
            _lib.load().pm_xchg_destroy(h)
