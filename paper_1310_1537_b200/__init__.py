"""B200-native (sm_100a) drop-in for the two SIMD hot paths of arXiv 1310.1537.

Mirrors the reference package `parmcmc` (/root/reference/pkg/src/parmcmc/
__init__.py:18-32):

* `glm`      logistic log-likelihood / log-posterior and gradient (fused single-pass
             kernel), the differential-update workspace, CSV / synthetic data
* `sampler`  slice-within-Gibbs chains (device-resident `run_chain`)
* `hb`       hierarchical models: batched per-group evaluation in one launch and the
             device-resident `hb_sweep` (one CTA per group)
* `ising`    checkerboard Gibbs sweeps (Ising, q=4 Potts), `ZCache`, `gibbs_sweep_diff`,
             `denoise`
* `images`   PBM I/O and test images for the denoiser
* `rng`      the Philox streams, device batch generation, Gamma / Dirichlet samplers
* `perf`     CPR grid runner with a B200 device model; `cli` the command line
* `dist`     torch.distributed (NCCL) row shards and lattice strips across ranks

Every hot call goes through libpmb200.so (include/pmb200.h); there is no CPU
fallback.
"""

from .glm import (DesignMatrix, ExecPlan, GlmWorkspace, GradResult, ShardedMatrix, Strategy,
                  commit_update, diff_loglike, diff_loglike_multi, load_design_csv, log_posterior_grad,
                  loglike, loglike_grad, make_sharded, synthetic_logistic)
from .hb import (CsrGroups, HbDataset, HbState, MappingMode, MappingPolicy, hb_benchmark,
                 hb_log_posterior_grad, hb_sweep, synthetic_hb_dataset)
from .images import flip_noise, read_pbm, synthetic_binary_image, write_pbm
from .ising import (ColorPartition, IsingLattice, PottsLattice, ZCache, color_lattice, conditional_prob,
                    denoise, gibbs_sweep, gibbs_sweep_diff, gibbs_sweeps, potts_sweeps)
from .rng import (BufferKind, DeviateBuffer, GammaParams, RngDrainError, SitePhilox, dirichlet_sample,
                  gamma_sample)
from .sampler import (ChainConfig, ChainOutput, GaussianPrior, SliceWidenError,
                      log_posterior_coord, run_chain, slice_sample_coord, write_draws_csv)

__version__ = "0.2.0"
