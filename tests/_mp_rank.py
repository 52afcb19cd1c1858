"""One rank of tests/test_gpu_multiproc.py: a separate PROCESS on cuda:0 that drives the
real cross-process exchange -- CUDA IPC mailboxes opened from handles all-gathered over a
gloo side channel (NCCL refuses two ranks on one GPU).

Ranks that share one GPU are time-sliced, so no kernel may wait on a kernel that is still
running (B200_PROFILING.md: such ranks raised Xid 109).  The launches are therefore ordered
from the host:
  * GLM: pm_glm_eval_xchg_phase 1 (stream + deposit + flags), synchronise, gloo barrier,
    phase 2 (the same evaluation, then acquire the flags -- already raised -- and fold);
  * strips: each half-sweep kernel waits only for the neighbours' deposits of the PREVIOUS
    half-sweep, so a synchronise + barrier after every half-sweep is enough.
Writes its results to <out>/rank<r>.npz for the parent test to compare.

usage: python tests/_mp_rank.py <rank> <world> <port> <out_dir>
"""

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

N_ROWS, K, N_EVALS = 200_003, 100, 50
H, W, SWEEPS, SEED = 96, 128, 20, 41


def glm_betas():
    return np.random.default_rng(1234).normal(0, 0.2, (N_EVALS, K))


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    import torch
    import torch.distributed as dist

    from paper_1310_1537_b200 import _lib
    from paper_1310_1537_b200.dist import LatticeStrip, PeerExchange, start_peer_halos, strip_bounds
    from paper_1310_1537_b200.glm import DesignMatrix
    from paper_1310_1537_b200.parallel import partition
    from paper_1310_1537_b200.sampler import GaussianPrior
    from paper_1310_1537_b200.synthetic import baseline_design, ising_spins, potts_states

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    res = {}
    try:
        # ---- row-sharded log-posterior + gradient, in-kernel exchange over IPC ----
        x, y, _, _ = baseline_design(N_ROWS, K, seed=5)
        a, b = partition(N_ROWS, world)[rank]
        dev = DesignMatrix(x[a:b], y[a:b]).on_device(0)
        prior = GaussianPrior.isotropic(K, 0.0, 10.0)
        if rank == 0:
            dev.set_prior(prior.mu, prior.sigma)
        px = PeerExchange(0, K + 1, group=None)
        assert px.ok, px.error
        o = torch.empty(K + 1, dtype=torch.float64, device="cuda:0")
        stream = torch.cuda.current_stream(0).cuda_stream or 1
        outs = []
        for beta in glm_betas():
            px.eval_phase(dev, beta, rank == 0, 1, 0, stream)
            torch.cuda.synchronize()
            dist.barrier()
            px.eval_phase(dev, beta, rank == 0, 2, o.data_ptr(), stream)
            torch.cuda.synchronize()
            outs.append(o.cpu().numpy().copy())
        res["glm"] = np.stack(outs)
        res["glm_timed_out"] = np.int32(px.timed_out())
        px.close()
        dist.barrier()

        # ---- lattice strips, in-kernel halo exchange over IPC ----
        for model in ("ising", "potts"):
            full = ising_spins(H, W, seed=8) if model == "ising" else potts_states(H, W, seed=8)
            r0, r1 = strip_bounds(H, world, rank)
            strip = LatticeStrip(H, W, r0, r1 - r0, 0, model=model, w=0.8814, coupling=1.0986)
            strip.set_spins(full[r0:r1])
            assert start_peer_halos(strip, rank, world)
            torch.cuda.synchronize()
            dist.barrier()
            for t in range(SWEEPS):
                for c in (0, 1):
                    strip.half_sweep(c, SEED, t)
                    torch.cuda.synchronize()
                    dist.barrier()
            res[f"strip_{model}"] = strip.get_spins()
            res[f"strip_{model}_timed_out"] = np.int32(strip.xchg_timed_out())
            strip.close()
            dist.barrier()
        _lib.load()
    finally:
        dist.destroy_process_group()
    np.savez(os.path.join(out, f"rank{rank}.npz"), **res)


if __name__ == "__main__":
    main()
