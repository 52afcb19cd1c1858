/*
 * pmb200.h -- C ABI of libpmb200.so, the B200 (sm_100a) implementation of the two
 * SIMD hot paths of arXiv 1310.1537 as shipped in the reference package `parmcmc`
 * (/root/reference/pkg/src/parmcmc).
 *
 * Every entry point below replaces one reference Python call (file:line cited per
 * function).  The reference's "plugin" boundary is the ExecPlan argument each hot
 * function dispatches on (glm.py:57-77, 257-274, 351-364); the Python mirror in
 * paper_1310_1537_b200/ binds these symbols with ctypes and keeps the reference's
 * signatures (INTEGRATION.md shows the binding a reference maintainer would add).
 *
 * Conventions
 *   - every function returns int: PM_OK (0) or an error code; pm_last_error()
 *     returns a thread-local message for the last failing call on this thread.
 *       PM_EINVAL  -> ValueError      (shape / non-finite / validation; glm.py:74-99,210-216)
 *       PM_ERANGE  -> IndexError      (coordinate out of range; glm.py:495-496)
 *       PM_EDEVICE -> RuntimeError    (CUDA failure)
 *       PM_ENOMEM  -> MemoryError
 *       PM_ESTATE  -> RuntimeError    (call order: e.g. eval before upload)
 *   - host pointers are borrowed for the duration of the call only;
 *   - calls are synchronous unless the name ends in _launch/_async;
 *   - a handle is bound to one device and owns one CUDA stream; calls on one handle
 *     are serialised by a per-handle mutex, so handles may be used from pool threads
 *     (the reference's HB COARSE mapping calls kernels from workers, hb.py:152-161);
 *   - results are bitwise repeatable for a fixed handle and input (the reference's
 *     fixed-plan determinism, test_glm.py:107-114): every reduction has a fixed order
 *     and no floating-point atomics are used.
 */
#ifndef PMB200_H
#define PMB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PM_ABI_VERSION 1

#if defined(__GNUC__)
#define PM_API __attribute__((visibility("default")))
#else
#define PM_API
#endif

enum pm_status {
  PM_OK = 0,
  PM_EINVAL = 1,
  PM_ERANGE = 2,
  PM_EDEVICE = 3,
  PM_ENOMEM = 4,
  PM_ESTATE = 5,
  PM_ESLICE = 6,   /* -> SliceWidenError (sampler.py:32-33, 141-150) */
  PM_ESHRINK = 7,  /* -> RuntimeError "slice shrinkage failed" (sampler.py:163-164) */
  PM_EDRAIN = 8    /* -> RngDrainError (rng.py:36-37, 178, 214) */
};

/* storage type of the design matrix on the device */
enum pm_xtype { PM_X_F64 = 0, PM_X_F32 = 1 };

/* ------------------------------------------------------------------ library */
PM_API int pm_abi_version(void);
PM_API const char* pm_last_error(void);
PM_API int pm_device_count(int* n);
PM_API int pm_device_info(int device, int* sm_count, int* cc_major, int* cc_minor, size_t* total_mem);
/* Kernel-dispatch overrides for A/B experiments and the layout tests (names and defaults
 * in csrc/pm_common.cu: glm_rows, f32_pairs, f64_pairs, stream_ncw, hb_rows, pdl,
 * gibbs_ng, ...).  The library never reads the environment: without these calls its
 * dispatch is fixed.  reset != 0 restores the default; unknown names -> PM_EINVAL.
 * Process-wide; a design / lattice handle reads them when it is created or uploaded. */
PM_API int pm_tune_set(const char* name, int value, int reset);
PM_API int pm_tune_get(const char* name, int* value, int* is_set);

/* ------------------------------------------------------------------ GLM
 * One device-resident logistic design: X row-major [N][K] (stored padded to a
 * multiple of 32 rows with zero rows; the padding never contributes), y in {0,1}.
 * Replaces the numpy arrays of DesignMatrix (glm.py:80-111), which the reference
 * declares immutable and shareable, so they are uploaded once and cached.
 */
typedef struct pm_glm_s* pm_glm_t;

PM_API int pm_glm_create(int device, pm_glm_t* out);
PM_API int pm_glm_destroy(pm_glm_t h);

/* X: host, row-major, n_rows*n_cols elements of double (PM_X_F64) or float (PM_X_F32);
 * y: host double[n_rows], each exactly 0 or 1 (glm.py:96-99). */
PM_API int pm_glm_upload(pm_glm_t h, const void* X, int x_dtype, const double* y,
                  int64_t n_rows, int32_t n_cols);

/* Diagonal Gaussian prior N(mu_k, sigma_k^2) (sampler.py:36-58); mu == sigma == NULL clears. */
PM_API int pm_glm_set_prior(pm_glm_t h, const double* mu, const double* sigma);

/* One fused pass over X (glm.py:351-372 loglike_grad -> _block_fg; glm.py:257 loglike):
 *   f = L(beta) [+ sum_k -0.5 ((beta_k-mu_k)/sigma_k)^2 if with_prior]
 *   g = X'(y - sigmoid(X beta)) [- (beta-mu)/sigma^2 if with_prior]   (if want_grad)
 * beta: host double[K]; f_out: host double*; g_out: host double[K] or NULL. */
PM_API int pm_glm_eval(pm_glm_t h, const double* beta, int with_prior, int want_grad,
                double* f_out, double* g_out);

/* Split form of pm_glm_eval for several handles in flight (the reference's
 * SHARDED strategy, glm.py:439-454, one shard per device): _launch enqueues the
 * kernel on the handle's stream, _wait returns the result as soon as the kernel's
 * finishing CTA has published it (it polls a completion word the kernel stores, system
 * scope, after (f, g) in mapped host memory; the stream itself drains a few microseconds
 * later and every later call on the handle is ordered after it).
 * One evaluation may be in flight per handle: _launch returns PM_ESTATE until the
 * matching _wait.  pm_glm_eval holds the handle's mutex across both halves, so
 * threads sharing one handle each get their own (f, g). */
PM_API int pm_glm_launch(pm_glm_t h, const double* beta, int with_prior, int want_grad);
PM_API int pm_glm_wait(pm_glm_t h, double* f_out, double* g_out);

/* Device-output form for collectives: writes (f, g[K]) as K+1 doubles to the device
 * buffer dev_out on `stream` (a cudaStream_t, NULL = the handle's own stream) without
 * synchronising; the caller reduces the partials across ranks (NCCL).  with_prior adds the
 * handle's prior terms in the kernel (exactly one rank does, so the fold holds it once). */
PM_API int pm_glm_eval_device(pm_glm_t h, const double* beta, int with_prior, int want_grad, double* dev_out,
                       void* stream);
/* Peer-memory exchange for row-sharded evaluations (one process per GPU, one NVLink/NVSwitch
 * node).  Replaces dist.py's NCCL all-gather + pm_fold_rows (the reference's ascending-worker
 * merge of per-worker partials, glm.py:243-250 / _grad_sharded 439-454) by ONE kernel launch:
 * the finishing CTA of every rank stores its (K+1) partial into all ranks' mailboxes (P2P),
 * raises its flag there, waits for every rank's flag and folds in ascending rank order, so
 * dev_out holds the world total with identical bits on every rank.  Setup: each rank creates
 * its mailbox, exports pm_xchg_ipc_handle (64 bytes), and opens every peer's handle with
 * pm_xchg_open_peer.  All ranks must call pm_glm_eval_xchg the same number of times (SPMD).
 * A rank missing for ~10 s ends the wait with NaN results and pm_xchg_status() = 1. */
typedef struct pm_xchg_s* pm_xchg_t;
PM_API int pm_xchg_create(int device, int32_t world, int32_t rank, int32_t width, pm_xchg_t* out);
PM_API int pm_xchg_ipc_handle(pm_xchg_t x, void* handle_out /* 64 bytes */);
PM_API int pm_xchg_open_peer(pm_xchg_t x, int32_t peer, const void* handle /* 64 bytes */);
/* Same-process peers (one process driving several GPUs with peer access, or tests): the
 * local mailbox address, and a peer's mailbox address used directly instead of an IPC map. */
PM_API int pm_xchg_mailbox(pm_xchg_t x, void** ptr);
PM_API int pm_xchg_set_peer_ptr(pm_xchg_t x, int32_t peer, void* mailbox);
PM_API int pm_xchg_status(pm_xchg_t x, int32_t* timed_out);
PM_API int pm_xchg_destroy(pm_xchg_t x);
PM_API int pm_glm_eval_xchg(pm_glm_t h, const double* beta, int with_prior, pm_xchg_t x, double* dev_out,
                            void* stream);
/* Split form of pm_glm_eval_xchg: phase 1 = stream + deposit + raise the flags (no wait,
 * dev_out untouched), phase 2 = the same evaluation again, then wait for every rank's flag
 * and fold (no deposit; same epoch), phase 3 = pm_glm_eval_xchg.  Phase 1 and 2 alternate
 * per handle (PM_ESTATE otherwise).  With a host barrier between every rank's phase 1 and
 * any rank's phase 2 no kernel ever waits on a kernel that is still running, so ranks that
 * SHARE one GPU (processes time-sliced on it) can drive the real IPC exchange. */
PM_API int pm_glm_eval_xchg_phase(pm_glm_t h, const double* beta, int with_prior, pm_xchg_t x, int phase,
                                  double* dev_out, void* stream);
/* out[c] = in[0][c] + in[1][c] + ... + in[world-1][c] in ascending row order (the reference's
 * ascending-worker merge, glm.py:243-250), c < width; device pointers, one launch on `stream`
 * (NULL = the legacy default stream).  Bitwise identical on every rank given the same input. */
PM_API int pm_fold_rows(const double* in_dev, int32_t world, int32_t width, double* out_dev, void* stream);

/* Benchmark helper: n back-to-back launches (beta row i of betas[n][K]) bracketed by CUDA
 * events on the handle's stream; *total_ms = elapsed device time. */
PM_API int pm_glm_time_launches(pm_glm_t h, const double* betas, int32_t n, int with_prior,
                                int want_grad, float* total_ms);
/* Cold-cache variant: before each of the n launches the L2 is scrubbed on the same stream
 * (512 MiB write + 256 MiB clean read); *total_ms = sum of the n launches' own event
 * intervals (device time with inputs in HBM, not host launch latency). */
PM_API int pm_glm_time_cold(pm_glm_t h, const double* betas, int32_t n, int with_prior,
                            int want_grad, float* total_ms);

/* The handle's CUDA stream (cudaStream_t), for event timing by the caller. */
PM_API int pm_glm_stream(pm_glm_t h, void** stream);
/* Launch geometry actually used (for the bench roofline and tests). */
PM_API int pm_glm_geometry(pm_glm_t h, int* grid, int* threads, int* stages, size_t* smem_bytes,
                    int* kernel_kind);

/* ------------------------------------------------------------------ differential update
 * Replaces GlmWorkspace / diff_loglike / commit_update (glm.py:461-539): a
 * device-resident xbeta[N] = X beta_current and the transposed copy xt[K][N].
 */
typedef struct pm_ws_s* pm_ws_t;

PM_API int pm_ws_create(pm_glm_t h, const double* beta0, pm_ws_t* out);
PM_API int pm_ws_destroy(pm_ws_t ws);
/* f_out[m] = L(beta_current + deltas[m] e_k), m < n_deltas (glm.py:499-522), one pass
 * over (xbeta, xt[k], y) for all deltas; never mutates the workspace. */
PM_API int pm_ws_diff_eval(pm_ws_t ws, int32_t k, const double* deltas, int32_t n_deltas,
                    double* f_out);
/* xbeta += delta * xt[k] (glm.py:525-539; bit-identical to numpy's two roundings). */
PM_API int pm_ws_commit(pm_ws_t ws, int32_t k, double delta);
PM_API int pm_ws_read_xbeta(pm_ws_t ws, double* out);
/* max_n |xbeta_n - (X beta_current)_n| recomputed on the device (GlmWorkspace.validate,
 * glm.py:484-489). */
PM_API int pm_ws_validate(pm_ws_t ws, const double* beta_current, double* max_abs_err);

/* Device-resident run_chain (sampler.py:170-200) from the workspace's current xbeta and
 * beta_inout[K] (in: start point, out: final point), prior N(mu, sigma^2), on the numpy
 * Philox4x64 UNIFORM01 stream with key (key0, key1) starting at deviate stream_pos (the
 * reference's consumption order, sampler.py:131-153).  One cooperative kernel; every
 * conditional evaluation is one grid-wide pass.  draws_out: (n_iter-n_burnin) x K;
 * *stream_pos_out = position after the chain; *evals_out = the reference's evaluation
 * count; on PM_ESLICE / PM_ESHRINK *fail_coord = the coordinate. */
PM_API int pm_ws_run_chain(pm_ws_t ws, const double* mu, const double* sigma, int32_t n_iter, int32_t n_burnin,
                           double slice_width, int32_t slice_max_steps, uint64_t key0, uint64_t key1,
                           uint64_t stream_pos, double* draws_out, double* beta_inout, uint64_t* stream_pos_out,
                           int64_t* evals_out, int32_t* fail_coord);

/* Device time (CUDA events around the cooperative kernel) of this thread's last
 * pm_ws_run_chain call, in milliseconds. */
PM_API int pm_chain_last_kernel_ms(float* ms);

/* ------------------------------------------------------------------ hierarchical GLM
 * Replaces the per-group loop of loglike_grad over HbDataset.groups (hb.py:64-86,
 * 127-135) with one launch over CSR-batched groups sharing K.
 */
typedef struct pm_hb_s* pm_hb_t;

PM_API int pm_hb_create(int device, pm_hb_t* out);
PM_API int pm_hb_destroy(pm_hb_t h);
/* X: host double[offsets[G]][K] row-major, y: host double[offsets[G]], offsets int64[G+1]
 * (offsets[0] == 0, non-decreasing, every group non-empty). */
PM_API int pm_hb_upload(pm_hb_t h, const double* X, const double* y, const int64_t* offsets,
                 int32_t n_groups, int32_t n_cols);
/* betas: host double[G][K]; mu, sigma: host double[K] shared prior or NULL (no prior);
 * f_out: host double[G]; g_out: host double[G][K] or NULL. */
PM_API int pm_hb_eval(pm_hb_t h, const double* betas, const double* mu, const double* sigma,
               int want_grad, double* f_out, double* g_out);
PM_API int pm_hb_stream(pm_hb_t h, void** stream);
/* Benchmark helper: n back-to-back kernel launches on device-resident betas (uploaded once),
 * bracketed by CUDA events on the handle's stream; *total_ms = elapsed device time. */
PM_API int pm_hb_time_evals(pm_hb_t h, const double* betas, const double* mu, const double* sigma,
                            int want_grad, int32_t n, float* total_ms);

/* Hierarchical Gibbs sweep state (replaces HbState + hb_sweep, hb.py:110-168): per-group
 * workspaces (xbeta, transposed X) and per-group numpy Philox uniform streams
 * (DeviateBuffer(UNIFORM01, seed, owner=(g,)), hb.py:118-119).  Groups are CSR rows
 * offsets[g]..offsets[g+1] of X (row-major N x K) and y; beta0 [G][K] is the start point
 * (the reference starts every group at prior.mu); keys [G][2], pos [G] the streams. */
typedef struct pm_hbs_s* pm_hbs_t;
PM_API int pm_hbs_create(int device, const double* X, const double* y, const int64_t* offsets, int32_t G,
                         int32_t K, const double* mu, const double* sigma, const double* beta0,
                         const uint64_t* keys, const uint64_t* pos, pm_hbs_t* out);
PM_API int pm_hbs_destroy(pm_hbs_t h);
/* n_sweeps Gibbs sweeps of every group in ONE launch (one CTA per group; slice-within-Gibbs
 * per coordinate, sampler.py:112-167; neval-1 extra full evaluations per group and sweep,
 * hb.py:130-131).  Out: betas [G][K], stream positions [G], evaluation counts of this call
 * [G].  PM_ESLICE / PM_ESHRINK name the first failing group and coordinate. */
PM_API int pm_hbs_sweeps(pm_hbs_t h, int32_t n_sweeps, int32_t neval, double slice_width, int32_t max_steps,
                         double* betas_out, uint64_t* pos_out, int64_t* evals_out, int32_t* fail_group,
                         int32_t* fail_coord, float* ms);
/* Replace the shared hyperprior N(mu, sigma^2) used by later sweeps. */
PM_API int pm_hbs_set_prior(pm_hbs_t h, const double* mu, const double* sigma);
/* Per-group log-likelihood at the current state (from the maintained xbeta). */
PM_API int pm_hbs_loglike(pm_hbs_t h, double* ll_out);
/* Maintained xbeta, concatenated in CSR row order (N doubles). */
PM_API int pm_hbs_read_xbeta(pm_hbs_t h, double* out);

/* ------------------------------------------------------------------ lattice Gibbs
 * Replaces IsingLattice/ColorPartition/gibbs_sweep (ising.py:47-187) and adds the
 * periodic boundary and the q=4 Potts model.  Colour c = (i+j)%2; colour 0 updates
 * against frozen colour 1, then colour 1 (ising.py:175-187).
 */
enum pm_boundary { PM_BOUNDARY_FREE = 0, PM_BOUNDARY_PERIODIC = 1 };
enum pm_model { PM_MODEL_ISING = 0, PM_MODEL_POTTS4 = 1 };
enum pm_rng {
  /* caller-supplied doubles in the reference's consumption order: per sweep, colour 0
   * in packed (scan) order then colour 1 (ising.py:185, rng.py:115-127) */
  PM_RNG_UNIFORMS = 0,
  /* numpy Philox4x64-10 DeviateBuffer stream (rng.py:42-44,86-90): deviate i uses
   * counter i/4+1, word i%4, u = (word>>11)*2^-53; key = (key0, key1) */
  PM_RNG_NUMPY_PHILOX = 1,
  /* Philox4x32-10 keyed by (seed, sweep, site): key = (key0 lo32, key0 hi32), counter
   * = (s/4 lo32, s/4 hi32, sweep lo32, sweep hi32), word s%4, u = word*2^-32, where
   * s = c*ceil(HW/2) + (i*W+j)/2 is the site's position in the sweep's stream */
  PM_RNG_PHILOX4X32 = 2
};

typedef struct pm_lat_s* pm_lat_t;

PM_API int pm_lat_create(int device, int32_t height, int32_t width, int boundary, int model,
                  pm_lat_t* out);
PM_API int pm_lat_destroy(pm_lat_t h);
/* spins: host int8[H*W] row-major; Ising values +-1, Potts values 0..3. */
PM_API int pm_lat_set_spins(pm_lat_t h, const int8_t* spins);
PM_API int pm_lat_get_spins(pm_lat_t h, int8_t* spins);
/* Ising field: P(s=+1) = expit(b_ij + w * sum of neighbour spins) (ising.py:11-16, 184);
 * bias: host double[H*W] or NULL for b == 0.  The host builds the exact probability
 * table with the reference's own arithmetic (b + w*nsum, then 1/(1+exp(-z)), as
 * scipy.special.expit), so the device compare u < p is bit-identical. */
PM_API int pm_lat_set_ising(pm_lat_t h, double w, const double* bias);
/* Potts q=4: P(a) proportional to exp(coupling * n_a), n_a = neighbours in state a;
 * a = #{a' < 3 : u >= cdf[a']} with the cdf built on the host in ascending a. */
PM_API int pm_lat_set_potts(pm_lat_t h, double coupling);
/* Run n_sweeps full sweeps.  stream_pos: PM_RNG_NUMPY_PHILOX -> index of the next
 * deviate of the buffer's stream; PM_RNG_PHILOX4X32 -> sweep number of the first sweep.
 * uniforms: host double[n_sweeps*H*W] for PM_RNG_UNIFORMS, else NULL. */
PM_API int pm_lat_sweeps(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1,
                  uint64_t stream_pos, const double* uniforms);
/* pm_lat_sweeps plus the diagnostics of the differential path and the denoiser
 * (replaces ZCache.flips_last_sweep, ising.py:204/253, and the post-burn-in
 * spin accumulator of denoise, ising.py:275-287):
 *   flips_out: host int64[n_sweeps] or NULL; flips_out[t] = sites whose value
 *              changed in sweep t (each site is updated once per sweep, so this
 *              is also count_nonzero(s_after != s_before), ising.py:284).
 *   acc_inout: host int32[H*W] or NULL; for every sweep t >= acc_from the new
 *              spins (Ising) / states (Potts) are added in, row-major.
 * Same trajectory as pm_lat_sweeps; runs on the generic kernel. */
PM_API int pm_lat_sweeps_acc(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1,
                      uint64_t stream_pos, const double* uniforms, int32_t acc_from, int32_t* acc_inout,
                      int64_t* flips_out);
/* Benchmark helper: pm_lat_sweeps for an in-kernel RNG mode, bracketed by CUDA events on the
 * handle's stream; *total_ms = elapsed device time of the n_sweeps sweeps. */
PM_API int pm_lat_time_sweeps(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1,
                              uint64_t stream_pos, float* total_ms);
PM_API int pm_lat_stream(pm_lat_t h, void** stream);
/* 1 if sweeps run on the red-black packed fast path (periodic, even H and W). */
PM_API int pm_lat_packed(pm_lat_t h, int* packed);

/* Strip of a periodic H x W lattice for multi-GPU sweeps: this handle owns
 * global rows [row0, row0+rows) and keeps one halo row of each colour above and below.
 * Requires even H, W and W % 32 == 0; spins via pm_lat_set/get_spins (rows x W); the
 * field via pm_lat_set_ising (uniform) / pm_lat_set_potts.  Site colours and RNG site
 * indices use global coordinates, so any strip decomposition gives the single-GPU spins. */
PM_API int pm_lat_create_strip(int device, int32_t height, int32_t width, int32_t row0, int32_t rows,
                               int model, pm_lat_t* out);
/* Update colour `colour` of the own rows (Philox4x32 keyed by (seed, sweep, site)) on
 * `stream` (cudaStream_t, NULL = handle stream) reading the other colour's halo rows.
 * The caller then exchanges this colour's first/last own rows with the neighbours. */
PM_API int pm_lat_strip_half_sweep(pm_lat_t h, int colour, uint64_t seed, uint64_t sweep, void* stream);
/* Device pointer of packed row `array_row` of colour `colour` (W/2 bytes): 0 = top halo,
 * 1..rows = own rows, rows+1 = bottom halo. */
PM_API int pm_lat_strip_row(pm_lat_t h, int colour, int32_t array_row, void** dev_ptr);
/* Peer-memory halo exchange (replaces the caller's per-half-sweep exchange, e.g. NCCL
 * send/recv): each strip owns a mailbox of double-buffered halo rows + flags; the
 * half-sweep kernel stores its first / last own rows straight into the up neighbour's
 * "row below" / the down neighbour's "row above" (P2P over NVLink/NVSwitch), its last CTA
 * raises their flags, and the rows that need a halo wait for it (acquire, ~10 s timeout ->
 * pm_lat_strip_xchg_status = 1).  Setup: pm_lat_strip_xchg_create (returns the mailbox
 * address), pm_lat_strip_xchg_ipc_handle (64 bytes, for other processes), set_peers with a
 * same-process mailbox pointer or an IPC handle per neighbour (up = the strip above, rows
 * row0-1..., periodic), then pm_lat_strip_xchg_start after pm_lat_set_spins.  Every strip
 * must then run the same half-sweep sequence (SPMD). */
PM_API int pm_lat_strip_xchg_create(pm_lat_t h, void** mailbox);
PM_API int pm_lat_strip_xchg_ipc_handle(pm_lat_t h, void* handle_out /* 64 bytes */);
PM_API int pm_lat_strip_xchg_set_peers(pm_lat_t h, void* up, const void* up_ipc, void* down, const void* down_ipc);
PM_API int pm_lat_strip_xchg_start(pm_lat_t h, void* stream);
PM_API int pm_lat_strip_xchg_status(pm_lat_t h, int32_t* timed_out);

/* ---------------------------------------------------------------- batch RNG
 * Device generation of the reference's deviate streams (rng.py:42-138) and its Gamma /
 * Dirichlet samplers (rng.py:152-215).  A stream is numpy Philox4x64-10 with key
 * (key[0], key[1]) (SeedSequence(seed, spawn_key=owner), rng.py:42-44); positions are
 * stream indices: uniform index for UNIFORM01 streams, normal index for STD_NORMAL
 * streams (normal j = Box-Muller of uniform pair j/2, cos for even j, sin for odd j,
 * rng.py:47-56 -- the capacity-invariant order of DeviateBuffer's carry logic 91-102).
 * All outputs are host arrays; ms (nullable) receives the device time (CUDA events). */
enum pm_rng_kind { PM_RNG_KIND_UNIFORM01 = 0, PM_RNG_KIND_STD_NORMAL = 1 };
/* out[i] = deviate pos+i of the stream, i < n (DeviateBuffer.take, rng.py:115-127).
 * out_is_device: out is a device pointer on `device`. */
PM_API int pm_rng_fill(int device, int kind, uint64_t key0, uint64_t key1, uint64_t pos, int64_t n, double* out,
                int out_is_device, float* ms);
/* n draws of gamma_sample(GammaParams(alpha, rate), u_src, n_src) (rng.py:191-198) from
 * the uniform stream ukey at *upos and the normal stream nkey at *npos; both positions
 * advance past exactly the deviates n sequential calls consume.  PM_EDRAIN after 10000
 * rejections in one draw (rng.py:178). */
PM_API int pm_rng_gamma(int device, double alpha, double rate, int64_t n, const uint64_t* ukey, uint64_t* upos,
                 const uint64_t* nkey, uint64_t* npos, double* out, float* ms);
/* n draws of dirichlet_sample(alphas[kd], u_src, n_src) (rng.py:201-215), out[n][kd]. */
PM_API int pm_rng_dirichlet(int device, const double* alphas, int32_t kd, int64_t n, const uint64_t* ukey,
                     uint64_t* upos, const uint64_t* nkey, uint64_t* npos, double* out, float* ms);
/* S independent stream pairs (owner spawn keys, rng.py:7-9), n_per draws each:
 * ukeys/nkeys [S][2], upos/npos [S] in/out, out [S][n_per] (gamma) / [S][n_per][kd]. */
PM_API int pm_rng_gamma_streams(int device, double alpha, double rate, int32_t S, int64_t n_per,
                         const uint64_t* ukeys, uint64_t* upos, const uint64_t* nkeys, uint64_t* npos,
                         double* out, float* ms);
PM_API int pm_rng_dirichlet_streams(int device, const double* alphas, int32_t kd, int32_t S, int64_t n_per,
                             const uint64_t* ukeys, uint64_t* upos, const uint64_t* nkeys, uint64_t* npos,
                             double* out, float* ms);

/* Host evaluation of the kernels' per-row logistic terms (the same pm_math.cuh code the
 * device runs, bit for bit): nll = (1-y)t + softplus(-t), w = y - sigmoid(t).  For tests. */
PM_API int pm_row_terms_host(const double* t, const double* y, int64_t n, double* nll_out, double* w_out);

/* Host-side table builders, exported so tests can check them against the oracle. */
PM_API int pm_ising_prob_table(double w, double b, double* p_out /*9: nsum=-4..4*/);
PM_API int pm_potts_cdf_table(double coupling, double* cdf_out /*625*3*/);

#ifdef __cplusplus
}
#endif
#endif /* PMB200_H */
