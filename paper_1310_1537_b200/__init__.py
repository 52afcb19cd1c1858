"""B200-native (sm_100a) drop-in for the two SIMD hot paths of arXiv 1310.1537.

Mirrors the reference package `parmcmc` (/root/reference/pkg/src/parmcmc/
__init__.py:18-32) for the hot-path modules:

* `glm`      logistic log-likelihood / log-posterior and gradient (fused single-pass
             kernel), the differential-update workspace
* `sampler`  slice-within-Gibbs chains driven by the device evaluations
* `hb`       hierarchical per-group evaluation in one CSR-batched launch
* `ising`    checkerboard Gibbs sweeps (Ising, q=4 Potts) on the device
* `rng`      the Philox uniform streams the kernels consume
* `dist`     torch.distributed (NCCL) row sharding across ranks

Every hot call goes through libpmb200.so (include/pmb200.h); there is no CPU
fallback.
"""

from .glm import (DesignMatrix, ExecPlan, GlmWorkspace, GradResult, ShardedMatrix, Strategy,
                  commit_update, diff_loglike, diff_loglike_multi, log_posterior_grad, loglike,
                  loglike_grad, make_sharded)
from .hb import CsrGroups, HbDataset, hb_log_posterior_grad
from .ising import (ColorPartition, IsingLattice, PottsLattice, color_lattice, conditional_prob,
                    gibbs_sweep, gibbs_sweeps, potts_sweeps)
from .rng import BufferKind, DeviateBuffer, SitePhilox
from .sampler import (ChainConfig, ChainOutput, GaussianPrior, SliceWidenError,
                      log_posterior_coord, run_chain, slice_sample_coord)

__version__ = "0.1.0"
