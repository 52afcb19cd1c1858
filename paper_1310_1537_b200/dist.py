"""Row sharding across ranks (one process per GPU, torch.distributed over NCCL).

The reference splits rows across worker threads and per-shard private copies
(parallel.py:30-46, glm.py:143-158, 439-454) and merges the (f, g) partials in
ascending worker order (glm.py:243-250).  Here each rank holds the rows
`partition(N, world)[rank]` on its own GPU; one evaluation is

    rank-local fused kernel -> (K+1) doubles on the device
    -> NCCL all-gather of the partials (one exchange step)
    -> sum in ascending rank order (bitwise identical on every rank)
    -> + prior terms (sampler.py:55-58), once.

`ordered_sum` and `gather_partials` are the collective logic; they are exercised
with the gloo backend on CPU tensors in tests/test_dist_gloo.py.
"""

from __future__ import annotations

import numpy as np

from .glm import DesignMatrix, GradResult, _check_beta
from .parallel import partition

__all__ = ["shard_bounds", "ordered_sum", "gather_partials", "DistributedDesign"]


def shard_bounds(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Rows owned by `rank` (parallel.py:30-46: the first n % world ranks get one extra)."""
    return partition(n_rows, world)[rank]


def ordered_sum(gathered):
    """Sum the rows of a (world, K+1) tensor in ascending rank order (fixed association)."""
    acc = gathered[0].clone()
    for r in range(1, gathered.shape[0]):
        acc += gathered[r]
    return acc


def gather_partials(part, group=None):
    """All-gather every rank's (K+1) partial and fold them in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(part.shape), dtype=part.dtype, device=part.device)
        dist.all_gather_into_tensor(out, part.contiguous(), group=group)
    else:
        parts = [torch.empty_like(part) for _ in range(world)]
        dist.all_gather(parts, part.contiguous(), group=group)
        out = torch.stack(parts)
    return ordered_sum(out)


def prior_terms_torch(beta_t, mu_t, sigma_t):
    z = (beta_t - mu_t) / sigma_t
    f = -0.5 * (z * z)
    # ascending-k sequential sum, like the device finaliser (glm_kernels.cuh)
    fsum = f[0].clone()
    for k in range(1, f.shape[0]):
        fsum += f[k]
    return fsum, -(beta_t - mu_t) / (sigma_t * sigma_t)


class DistributedDesign:
    """This rank's row shard on its GPU, evaluated with one NCCL exchange per call."""

    def __init__(self, local: DesignMatrix, device: int, x_storage: str = "f64", group=None):
        import torch
        self.local = local
        self.device = device
        self.group = group
        self.dev = local.on_device(device, x_storage)
        self.k = local.n_cols
        self._buf = torch.empty(self.k + 1, dtype=torch.float64, device=f"cuda:{device}")

    def _partial(self, beta: np.ndarray):
        import torch
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self.dev.eval_device(beta, True, self._buf.data_ptr(), stream)
        return self._buf

    def log_posterior_grad_device(self, beta, prior=None):
        """(f, g) as a device tensor of K+1 doubles, identical on every rank."""
        import torch
        beta = _check_beta(beta, self.k)
        tot = gather_partials(self._partial(beta), self.group)
        if prior is not None:
            dev = tot.device
            bt = torch.from_numpy(beta).to(dev, non_blocking=True)
            pf, pg = prior_terms_torch(bt, torch.from_numpy(prior.mu).to(dev), torch.from_numpy(prior.sigma).to(dev))
            tot[0] += pf
            tot[1:] += pg
        return tot

    def log_posterior_grad(self, beta, prior=None) -> GradResult:
        out = self.log_posterior_grad_device(beta, prior).cpu().numpy()
        return GradResult(float(out[0]), out[1:].copy())
