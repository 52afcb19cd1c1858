// Device code for the callers of the GLM hot path:
//   K3 diff_eval   (glm.py:499-522)  multi-delta conditional log-likelihood, one pass
//   K4 commit      (glm.py:525-539)  xbeta += delta * xt[k]
//   workspace init (glm.py:469-474)  xbeta = X beta0, xt = X^T
//   K5 hb segmented (hb.py:64-86, 127-135) one CTA per group over CSR-batched groups
#pragma once

#include "glm_kernels.cuh"

namespace pm {

constexpr int kMaxDeltas = 16;

struct DeltaPack {
  double d[kMaxDeltas];
};

struct DiffArgs {
  const double* xbeta;
  const double* xk;   // xt + k*n_pad
  const double* y;
  int64_t n;
  double* partials;   // [kMaxDeltas][grid]
  unsigned int* counter;
  double* out;        // [M]
  unsigned long long* done;     // completion word after `out` in mapped memory (see GlmArgs::done)
  unsigned long long done_seq;
};

// Rounding identical to numpy's `xbeta + delta*xk` (glm.py:517): product rounded, then sum.

// Grid-stride over elements; per-thread sums for each delta in the same order for every M,
// so f for a given delta is bit-identical whether it is evaluated alone or in a batch.
template <int M>
__global__ void __launch_bounds__(256) diff_eval_kernel(DiffArgs a, DeltaPack dp) {
  __shared__ double red[8][M];
  __shared__ int flag;
  double acc[M];
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const double xb = __ldg(a.xbeta + i);
    const double xk = __ldg(a.xk + i);
    const double yy = __ldg(a.y + i);
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] += row_nll(shifted_t(xb, dp.d[m], xk), yy);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const double s = warp_sum(acc[m]);
    if (lane == 0) red[warp][m] = s;
  }
  __syncthreads();
  if (threadIdx.x < M) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w][threadIdx.x];
    a.partials[size_t(threadIdx.x) * gridDim.x + blockIdx.x] = s;  // [m][cta]: coalesced fold
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // one acq_rel ticket publishes / acquires the CTA partials (see K1)
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(a.counter) : "memory");
    flag = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!flag) return;
  // warp w folds delta m = w, w + 8, ...: lane-strided CTA partials (loads in flight
  // together), then the fixed butterfly -- the order does not depend on M
  for (int m = warp; m < M; m += blockDim.x >> 5) {
    const double s = warp_sum(fold_lane(a.partials + size_t(m) * gridDim.x, 1, gridDim.x, lane));
    if (lane == 0) a.out[m] = -s;
  }
  if (threadIdx.x == 0) *a.counter = 0u;
  if (a.done) {
    __syncthreads();  // every warp's result store, then one system-scope fence + release store
    if (threadIdx.x == 0) {
      asm volatile("fence.sc.sys;" ::: "memory");
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.done), "l"(a.done_seq) : "memory");
    }
  }
}

__global__ void __launch_bounds__(256) commit_kernel(double* __restrict__ xbeta, const double* __restrict__ xk,
                                                     double d, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    xbeta[i] = __dadd_rn(xbeta[i], __dmul_rn(d, xk[i]));
}

// xbeta[r] = X[r,:] . beta  (one warp per row; GlmWorkspace construction and validate)
template <typename XT>
__global__ void __launch_bounds__(256) xbeta_kernel(const XT* __restrict__ X, const double* __restrict__ beta,
                                                    int K, int64_t n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    double acc = 0.0;
    for (int k = lane; k < K; k += 32) acc = fma(ld_x(X + r * K + k), __ldg(beta + k), acc);
    acc = warp_sum(acc);
    if (lane == 0) out[r] = acc;
  }
}

// max |a - b| over n (validate, glm.py:484-489): per-block max then single atomicMax on bits
// (non-negative doubles order like their bit patterns, so this is exact and order-free).
__global__ void __launch_bounds__(256) maxabs_diff_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                          int64_t n, unsigned long long* out_bits) {
  double m = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    m = fmax(m, fabs(a[i] - b[i]));
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, s));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, (unsigned long long)__double_as_longlong(m));
}

// X [n][K] (row-major, XT) -> xt [K][ld] f64, 32x32 tiles through shared memory.
template <typename XT>
__global__ void __launch_bounds__(256) transpose_kernel(const XT* __restrict__ X, int64_t n, int K,
                                                        double* __restrict__ xt, int64_t ld) {
  __shared__ double tile[32][33];
  const int64_t r0 = int64_t(blockIdx.x) * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i;
    const int c = c0 + tx;
    tile[i][tx] = (r < n && c < K) ? ld_x(X + r * K + c) : 0.0;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int c = c0 + i;
    const int64_t r = r0 + tx;
    if (c < K && r < n) xt[int64_t(c) * ld + r] = tile[tx][i];
  }
}

__global__ void __launch_bounds__(256) f64_to_f32_kernel(const double* __restrict__ src, float* __restrict__ dst,
                                                         int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = __double2float_rn(src[i]);
}

// ---------------------------------------------------------------- K5 hierarchical
struct HbArgs {
  const double* X;        // padded per group: group g occupies rows [poff[g], poff[g+1])
  const double* y;
  const int64_t* poff;    // [G+1] padded row offsets (multiples of 32)
  const int64_t* nrows;   // [G] real rows per group
  int K;
  int stages;
  const double* betas;    // [G][K]
  const double* mu;       // [K] or null
  const double* sigma;    // [K] or null
  double* out_f;          // [G]
  double* out_g;          // [G][K]
};

// One CTA per group: the group's tiles stream through the same TMA ring as K1; the CTA
// reduces its warps in fixed order and adds the shared group prior.  No cross-CTA step.
// Groups are short (~63 tiles), so several CTAs per SM hide latency: smaller register
// sub-tiles (HbRows) keep the footprint under the 3-CTAs/SM register budget.
template <int KC, bool GRAD>
struct HbRows {
  static constexpr int value = !GRAD ? 32 : (KC == 1 ? 16 : (KC == 2 ? 8 : 4));
};

template <int KC, bool GRAD, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 3) hb_kernel(HbArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = a.K;
  const int S = a.stages;
  const StreamSmem sm = carve_stream_smem(smem_raw, K, sizeof(double), S, NCW);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int grp = blockIdx.x;
  const double* bg = a.betas + size_t(grp) * K;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    fence_mbar_init();
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) sm.sbeta[k] = bg[k];
  __syncthreads();
  double breg[KC], g[KC];
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    const int c = lane + 32 * j;
    breg[j] = (c < K) ? sm.sbeta[c] : 0.0;
    g[j] = 0.0;
  }
  double nll = 0.0;
  const int64_t p0 = a.poff[grp], p1 = a.poff[grp + 1];
  stream_tiles<double, KC, GRAD, NCW, HbRows<KC, GRAD>::value>(a.X, a.y, K, p0 / kTileRows, p1 / kTileRows, 1,
                                                               p0 + a.nrows[grp], S, sm, breg, g, nll, false);
  if (warp > 0) {
    const int cw = warp - 1;
    const double wsum = warp_sum(nll);
    if (lane == 0) sm.wf[cw] = -wsum;
    if (GRAD) {
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        const int c = lane + 32 * j;
        if (c < K) sm.wg[size_t(cw) * K + c] = g[j];
      }
    }
  }
  __syncthreads();
  const bool prior = a.mu != nullptr;
  for (int c = threadIdx.x; c <= K; c += blockDim.x) {
    if (c == 0) {
      double f = 0.0;
      for (int w = 0; w < NCW; ++w) f += sm.wf[w];
      if (prior) {
        for (int k = 0; k < K; ++k) {
          const double z = (sm.sbeta[k] - a.mu[k]) / a.sigma[k];
          f += -0.5 * z * z;
        }
      }
      a.out_f[grp] = f;
    } else if (GRAD) {
      const int k = c - 1;
      double gk = 0.0;
      for (int w = 0; w < NCW; ++w) gk += sm.wg[size_t(w) * K + k];
      if (prior) {
        const double sg = a.sigma[k];
        gk -= (sm.sbeta[k] - a.mu[k]) / (sg * sg);
      }
      a.out_g[size_t(grp) * K + k] = gk;
    }
  }
}

// ---------------------------------------------------------------- small-K hierarchical path
// For even K <= 32 the column-per-lane layout leaves lanes idle (K=20: 12 of 32) and pays a
// transpose-reduce per row; here each lane owns one ROW of a 32-row tile: its K values come
// from shared memory as 16-byte loads, the dot product runs in two interleaved chains, the
// logistic terms are computed once per row, and the gradient accumulates in K registers.
// The padded tiles of all groups are split into equal contiguous ranges, one per CTA
// (1 CTA/SM), so no wave quantisation; a CTA's range covers pieces ("segments") of a few
// groups.  Every consumer warp writes one (nll, g[K]) partial per segment (zeros if it had
// no tile there) and hb_fold_kernel sums the partials of each group in a fixed order
// (segment, warp) and adds the prior: deterministic for a given device.
struct HbRowsArgs {
  const double* X;
  const double* y;
  const int64_t* poff;   // [G+1] padded row offsets (multiples of 32)
  const int64_t* nrows;  // [G]
  const int* seg_base;   // [grid+1] first segment of each CTA
  int G, K, stages, tps;
  int contig;            // 1: contiguous unit range per consumer warp; 0: round-robin
  int fused;             // 1: fold in the same launch (per-group tickets); 0: hb_fold_kernel
  int selfprod;          // 1: every consumer warp issues the bulk copies of its own units (no producer thread)
  int64_t n_tiles;       // poff[G] / 32
  const double* betas;   // [G][K]
  double* part;          // [nseg][NCW][K+1]
  const int* cta_g0;     // [grid] first group of each CTA's tile range
  const int* gseg;       // [G+1] first segment of each group
  unsigned* gcount;      // [G] tickets, zero between launches
  const double* mu;      // fused fold: prior (nullable) and outputs
  const double* sigma;
  double* out_f;
  double* out_g;
};

// b: this warp's copy of the group's beta in shared memory (all lanes read the same address:
// broadcast), so only x[] and g[] occupy registers and 15 consumer warps fit per SM.
// `dep` accumulates a value computed from every shared load of the tile; the caller releases
// the stage with mbar_arrive_after(dep) once all of the stage's tiles are consumed.
//
// Bank conflicts: lane l reads its row in 16-byte chunks; with Q = K/2 chunks per row, the
// 8 lanes of a 128-byte wavefront start Q chunks apart.  When Q is a multiple of 8 (K = 16,
// 32) they all hit the same bank group (8-way conflict; measured 2x slower), so those
// shapes XOR-swizzle: register slot q holds chunk q ^ sw with sw = lane & 7 (a permutation
// inside each aligned group of 8 chunks), and rows_unrotate() maps the gradient slots back.
// Other even K keep static offsets (2- and 4-way conflicts measured harmless).
// KMAX is the exact (even) K of the instantiation; the runtime K must equal it.
template <int KMAX>
struct RowsSwizzle {
  static constexpr bool value = (KMAX / 2) % 8 == 0;
};

template <int KMAX, bool GRAD>
__device__ __forceinline__ void consume_tile_rows(const double* xs, const double* ys, int K, int sw, int lane,
                                                  int64_t row0, int64_t row_limit, const double* b,
                                                  double (&g)[KMAX], double& nll_acc, double& dep) {
  constexpr bool SW = RowsSwizzle<KMAX>::value;
  const double2* xr = reinterpret_cast<const double2*>(xs + lane * KMAX);  // 16-byte aligned rows
  const double2* b2 = reinterpret_cast<const double2*>(b);
  double x[KMAX];
  double t0 = 0.0, t1 = 0.0;
#pragma unroll
  for (int q = 0; q < KMAX / 2; ++q) {
    const int c = SW ? (q ^ sw) : q;
    const double2 v = xr[c];
    const double2 bb = b2[c];
    x[2 * q] = v.x;
    x[2 * q + 1] = v.y;
    t0 = fma(v.x, bb.x, t0);
    t1 = fma(v.y, bb.y, t1);
  }
  const double yv = ys[lane];
  dep += t0 + t1 + yv;  // t0, t1, yv consume every load of this tile
  double nll, w;
  row_terms(t0 + t1, yv, nll, w);
  const bool valid = row0 + lane < row_limit;
  nll_acc += valid ? nll : 0.0;
  if (GRAD) {
    w = valid ? w : 0.0;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) g[k] = fma(w, x[k], g[k]);
  }
}

// Column totals of the swizzled per-lane gradient slots: column pair (2c, 2c+1) sits in slot
// c ^ sw; a select over the 8 slots of c's group picks it, then the fixed butterfly sums the
// lanes.  out(k, v) receives column k's warp total in every lane.
template <int KMAX, class Out>
__device__ __forceinline__ void rows_unrotate(const double (&g)[KMAX], int K, int sw, Out out) {
  if constexpr (!RowsSwizzle<KMAX>::value) {
#pragma unroll
    for (int k = 0; k < KMAX; ++k) out(k, warp_sum(g[k]));
  } else {
#pragma unroll
    for (int cc = 0; cc < KMAX / 2; ++cc) {
      const int s = cc ^ sw;
      double v0 = 0.0, v1 = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int q = (cc & ~7) | j;
        if (q == s) {
          v0 = g[2 * q];
          v1 = g[2 * q + 1];
        }
      }
      out(2 * cc, warp_sum(v0));
      out(2 * cc + 1, warp_sum(v1));
    }
  }
}

__device__ __forceinline__ int group_of_tile(const int64_t* poff, int G, int64_t tile) {
  // largest g with poff[g] / 32 <= tile
  int lo = 0, hi = G - 1;
  const int64_t row = tile * kTileRows;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (poff[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Per group: fold the partials of its segments (gseg[g] .. gseg[g+1]-1) and warps in that
// order, add the prior (sampler.py:55-58), write f and g.  Threads tid, tid+nt, ... take the
// columns; shared by hb_fold_kernel and the fused tail of hb_rows_kernel (identical bits).
template <bool GRAD, bool CG>
__device__ __forceinline__ void hb_fold_group(const double* part, const int* gseg, int nw, int K,
                                              const double* betas, const double* mu, const double* sigma,
                                              double* out_f, double* out_g, int grp, int tid, int nt) {
  const int s0 = gseg[grp], s1 = gseg[grp + 1];
  for (int c = tid; c <= K; c += nt) {
    if (c > 0 && !GRAD) break;
    double acc = 0.0;
    for (int s = s0; s < s1; ++s)
      for (int w = 0; w < nw; ++w) {
        const double* p = part + (size_t(s) * nw + w) * (K + 1) + c;
        acc += CG ? __ldcg(p) : *p;
      }
    if (c == 0) {
      double f = -acc;
      if (mu) {
        for (int k = 0; k < K; ++k) {
          const double z = (betas[size_t(grp) * K + k] - mu[k]) / sigma[k];
          f += -0.5 * z * z;
        }
      }
      out_f[grp] = f;
    } else {
      const int k = c - 1;
      double gk = acc;
      if (mu) {
        const double sg = sigma[k];
        gk -= (betas[size_t(grp) * K + k] - mu[k]) / (sg * sg);
      }
      out_g[size_t(grp) * K + k] = gk;
    }
  }
}

// first group of the tile range starting at `tile`, searched inside [lo, hi]
__device__ __forceinline__ int group_of_tile_in(const int64_t* poff, int lo, int hi, int64_t tile) {
  const int64_t row = tile * kTileRows;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (poff[mid] <= row) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// NCW odd (7, 15): warp 0 is the producer (or idle when the consumers produce for themselves);
// NCW even (8): every warp of the CTA consumes and produces for itself (a.selfprod required).
template <int NCW>
struct HbRowsThreads {
  static constexpr bool all = NCW % 2 == 0;
  static constexpr int value = (all ? NCW : NCW + 1) * 32;
};
template <int KMAX, bool GRAD, int NCW>
__global__ void __launch_bounds__(HbRowsThreads<NCW>::value, 1) hb_rows_kernel(HbRowsArgs a) {
  constexpr bool ALL = HbRowsThreads<NCW>::all;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = a.K;
  const int S = a.stages;
  const int TPS = a.tps;  // 32-row tiles per stage: one bulk copy moves TPS consecutive tiles
  // carve S*TPS tile slots (stage s = slots s*TPS ..): contiguous, since 32*K*8 is a multiple
  // of 128 for even K; only the first S barrier pairs are used.  wg: per-warp beta copies.
  const StreamSmem sm = carve_stream_smem(smem_raw, K, sizeof(double), S * TPS, NCW);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t C = gridDim.x, c = blockIdx.x;
  const int64_t t0 = c * a.n_tiles / C, t1 = (c + 1) * a.n_tiles / C;
  if (t0 >= t1) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t n_mine = t1 - t0;
  const int64_t n_units = (n_mine + TPS - 1) / TPS;
  const uint32_t tile_bytes = uint32_t(kTileRows) * K * sizeof(double);
  const size_t stage_pitch = size_t(tile_bytes) * TPS;
  const int nact = S < NCW ? S : NCW;
  const int spw = S / nact;  // stages per consumer warp: warp w owns stages w, w + nact, ...
  // Each consumer warp takes a CONTIGUOUS share of the CTA's units (a.contig = 1), so a warp
  // crosses ~1-2 group boundaries per launch instead of every group of the CTA (each crossing
  // costs a partial flush and a beta reload); a.contig = 0: round-robin, unit w + m*nact.
  const int64_t q = n_units / nact;
  const int rr = int(n_units - q * nact);
  const int cw = ALL ? warp : warp - 1;
  // this consumer warp's units (pure arithmetic on the arguments: no global loads, so a
  // self-producing warp can start its first copies before the PDL wait)
  const int64_t u_first = a.contig ? int64_t(cw) * q + (int64_t(cw) * rr) / nact : cw;
  const int64_t n_w = a.contig ? int64_t(cw + 1) * q + (int64_t(cw + 1) * rr) / nact - u_first
                               : q + (cw < rr ? 1 : 0);
  const int64_t u_step = a.contig ? 1 : nact;
  // Self-producing consumers (a.selfprod): warp w refills its own stages, unit m + spw into
  // the stage unit m has just left -- no producer thread to serialise on (~100 ns per copy,
  // 2 copies per 10 KB unit: ~44 us of one thread's time per config-3 launch) and no `empty`
  // barriers.
  auto issue_unit = [&](int64_t m, int s) {  // lane 0 of consumer warp cw
    const int64_t tile = t0 + (u_first + m * u_step) * TPS;
    const uint32_t nt = uint32_t(t1 - tile < TPS ? t1 - tile : TPS);
    mbar_arrive_expect_tx(&sm.full[s], nt * (tile_bytes + 32 * sizeof(double)));
    bulk_g2s(sm.xs + size_t(s) * stage_pitch, a.X + tile * int64_t(kTileRows) * K, nt * tile_bytes, &sm.full[s]);
    bulk_g2s(sm.ys + size_t(s) * 32 * TPS, a.y + tile * kTileRows, nt * 32 * sizeof(double), &sm.full[s]);
  };
  if (a.selfprod && (ALL || warp > 0) && cw < nact && lane == 0) {
    for (int m = 0; m < spw; ++m)
      if (m < n_w) issue_unit(m, cw + nact * m);
  }
  if (!ALL && warp == 0 && !a.selfprod) {
    if (lane == 0) {
      // the single producer thread is on the critical path: no divisions and no dependent
      // global loads before its first copy (the per-warp first unit / count are rebuilt
      // incrementally, Bresenham style)
      const int64_t m_max = (n_units + nact - 1) / nact;
      const int64_t step = a.contig ? 1 : nact;
      int ms = 0;       // m % spw
      uint32_t n = 0;   // m / spw
      for (int64_t m = 0; m < m_max; ++m) {
        int64_t u0 = 0;
        int acc = 0;
        for (int w = 0; w < nact; ++w) {
          int64_t first, cnt;
          if (a.contig) {
            int64_t nxt = u0 + q;
            acc += rr;
            if (acc >= nact) {
              acc -= nact;
              ++nxt;
            }
            first = u0;
            cnt = nxt - u0;
            u0 = nxt;
          } else {
            first = w;
            cnt = q + (w < rr ? 1 : 0);
          }
          if (m >= cnt) continue;
          const int64_t u = first + m * step;
          const int s = w + nact * ms;
          if (n > 0) mbar_wait(&sm.empty[s], (n - 1) & 1);
          const int64_t tile = t0 + u * TPS;
          const uint32_t nt = uint32_t(t1 - tile < TPS ? t1 - tile : TPS);
          mbar_arrive_expect_tx(&sm.full[s], nt * (tile_bytes + 32 * sizeof(double)));
          bulk_g2s(sm.xs + size_t(s) * stage_pitch, a.X + tile * int64_t(kTileRows) * K, nt * tile_bytes,
                   &sm.full[s]);
          bulk_g2s(sm.ys + size_t(s) * 32 * TPS, a.y + tile * kTileRows, nt * 32 * sizeof(double), &sm.full[s]);
        }
        if (++ms == spw) {
          ms = 0;
          ++n;
        }
      }
    }
  }
  // PDL: the copies above only read X and y (never written by a kernel); the consumers and
  // the fold below read beta and write the partials / tickets the previous launch uses
  if (threadIdx.x == 0) pdl_trigger();
  if (ALL || warp > 0) pdl_wait();
  // the CTA's groups and segments (host-computed; loaded after the producer started)
  const int g_first = a.cta_g0[c];
  const int seg0 = a.seg_base[c];
  const int g_last = g_first + (a.seg_base[c + 1] - seg0) - 1;
  if ((ALL || warp > 0) && cw < nact) {
    double* b = sm.wg + size_t(cw) * K;
    double g[KMAX];
    double nll = 0.0;
    auto load_beta = [&](int grp) {
      __syncwarp();  // previous group's reads of b are done
      for (int k = lane; k < K; k += 32) b[k] = __ldg(a.betas + int64_t(grp) * K + k);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < KMAX; ++k) g[k] = 0.0;
      nll = 0.0;
    };
    // partial of group `grp` (this warp's share of segment seg0 + grp - g_first)
    const int q0 = RowsSwizzle<KMAX>::value ? (lane & 7) : 0;  // chunk swizzle (consume_tile_rows)
    auto slot = [&](int grp) { return a.part + (size_t(seg0 + grp - g_first) * NCW + cw) * (K + 1); };
    auto flush = [&](int grp) {
      double* dst = slot(grp);
      const double ns = warp_sum(nll);
      if (lane == 0) dst[0] = ns;
      if (GRAD)
        rows_unrotate<KMAX>(g, K, q0, [&](int k, double v) {
          if (lane == 0) dst[1 + k] = v;
        });
    };
    auto zero_fill = [&](int grp) {  // a segment of the CTA this warp has no rows of
      double* dst = slot(grp);
      for (int k = lane; k <= K; k += 32) dst[k] = 0.0;
    };
    if (n_w <= 0) {
      for (int grp = g_first; grp <= g_last; ++grp) zero_fill(grp);
    } else {
      int cur = group_of_tile_in(a.poff, g_first, g_last, t0 + u_first * TPS);
      for (int grp = g_first; grp < cur; ++grp) zero_fill(grp);
      load_beta(cur);
      int s = cw;
      uint32_t n = 0;
      int64_t next_start = a.poff[cur + 1], row_limit = a.poff[cur] + a.nrows[cur];
      for (int64_t m = 0; m < n_w; ++m) {
        const int64_t u = u_first + m * u_step;
        const int64_t tile0 = t0 + u * TPS;
        const int nt = int(t1 - tile0 < TPS ? t1 - tile0 : TPS);
        mbar_wait(&sm.full[s], n & 1);
        const double* xst = reinterpret_cast<const double*>(sm.xs + size_t(s) * stage_pitch);
        const double* yst = sm.ys + size_t(s) * 32 * TPS;
        double dep = 0.0;
        for (int j = 0; j < nt; ++j) {
          const int64_t row0 = (tile0 + j) * kTileRows;
          while (row0 >= next_start) {
            flush(cur);
            load_beta(++cur);
            next_start = a.poff[cur + 1];
            row_limit = a.poff[cur] + a.nrows[cur];
          }
          consume_tile_rows<KMAX, GRAD>(xst + size_t(j) * kTileRows * K, yst + 32 * j, K, q0, lane, row0,
                                        row_limit, b, g, nll, dep);
        }
        mbar_arrive_after(a.selfprod ? nullptr : &sm.empty[s], dep, lane, const_cast<double*>(xst));
        if (a.selfprod && lane == 0 && m + spw < n_w) issue_unit(m + spw, s);  // the stage is quiescent
        s += nact;
        if (s >= nact * spw) {
          s = cw;
          ++n;
        }
      }
      flush(cur);
      for (int grp = cur + 1; grp <= g_last; ++grp) zero_fill(grp);  // segments after this warp's rows
    }
  }
  if (!a.fused) return;
  pdl_wait();  // (the producer thread: its ticket writes below follow the previous launch)
  // Fused fold: one acq_rel ticket per group this CTA touched (thread i takes groups
  // g_first + i, ...; the CTA barrier before it orders every warp's partial stores, PTX
  // fences being cumulative); the CTA that completes a group (count = its segments, one per
  // CTA overlapping it) folds it, warp per group, in hb_fold_kernel's order.  Replaces the
  // second launch.  The list of groups to fold reuses the (drained) stage memory.
  int* list = reinterpret_cast<int*>(sm.xs);  // <= blockDim.x entries per chunk
  int* nlist = list + blockDim.x;
  for (int gc = g_first; gc <= g_last; gc += blockDim.x) {
    __syncthreads();  // partial stores done (first chunk) / previous chunk's list consumed
    if (threadIdx.x == 0) *nlist = 0;
    __syncthreads();
    const int grp = gc + threadIdx.x;
    if (grp <= g_last) {
      const unsigned need = unsigned(a.gseg[grp + 1] - a.gseg[grp]);
      unsigned t;
      asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(a.gcount + grp) : "memory");
      if (t + 1 == need) {
        a.gcount[grp] = 0u;  // re-arm for the next launch (kernel boundary orders it)
        list[atomicAdd(nlist, 1)] = grp;
      }
    }
    __syncthreads();
    const int nl = *nlist;
    for (int i = warp; i < nl; i += blockDim.x >> 5)
      hb_fold_group<GRAD, true>(a.part, a.gseg, NCW, K, a.betas, a.mu, a.sigma, a.out_f, a.out_g, list[i], lane,
                                32);
  }
}

// ---------------------------------------------------------------- K1 small-K row-per-lane variant
// The flat evaluation (glm.py:367-372) for fp64 X with even K <= 32: each CTA streams an
// equal contiguous range of the padded tiles, TPS tiles per stage, and every consumer lane
// owns one row (consume_tile_rows; beta broadcast from shared memory).  Per-warp partials
// go through the same deterministic CTA fold and last-CTA finish as glm_stream_kernel.
template <int KMAX, bool GRAD, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) glm_rows_kernel(GlmArgs a, BetaPack<1> beta, int tps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = a.K;
  const int S = a.stages;
  const int TPS = tps;
  const StreamSmem sm = carve_stream_smem(smem_raw, K, sizeof(double), S * TPS, NCW);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], 1);
    }
    fence_mbar_init();
  }
  for (int k = threadIdx.x; k < K; k += blockDim.x) sm.sbeta[k] = beta.v[k];
  __syncthreads();
  if (blockIdx.x == 0 && a.with_prior && warp == NCW) prior_precompute(a, sm.sbeta, lane);
  const int64_t C = gridDim.x, c = blockIdx.x;
  const int64_t t0 = c * a.n_tiles / C, t1 = (c + 1) * a.n_tiles / C;
  const int64_t n_units = (t1 - t0 + TPS - 1) / TPS;
  const uint32_t tile_bytes = uint32_t(kTileRows) * K * sizeof(double);
  const size_t stage_pitch = size_t(tile_bytes) * TPS;
  const int nact = S < NCW ? S : NCW;
  const int Se = S - S % nact;
  const double* X = static_cast<const double*>(a.X);
  const int q0 = RowsSwizzle<KMAX>::value ? (lane & 7) : 0;  // chunk swizzle (consume_tile_rows)
  double g[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) g[k] = 0.0;
  double nll = 0.0;
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int s = 0;
      uint32_t n = 0;
      for (int64_t i = 0; i < n_units; ++i) {
        if (n > 0) mbar_wait(&sm.empty[s], (n - 1) & 1);
        const int64_t tile = t0 + i * TPS;
        const uint32_t nt = uint32_t(t1 - tile < TPS ? t1 - tile : TPS);
        mbar_arrive_expect_tx(&sm.full[s], nt * (tile_bytes + 32 * sizeof(double)));
        if (a.evict_first)
          bulk_g2s_hint(sm.xs + size_t(s) * stage_pitch, X + tile * int64_t(kTileRows) * K, nt * tile_bytes,
                        &sm.full[s], pol);
        else
          bulk_g2s(sm.xs + size_t(s) * stage_pitch, X + tile * int64_t(kTileRows) * K, nt * tile_bytes, &sm.full[s]);
        bulk_g2s(sm.ys + size_t(s) * 32 * TPS, a.y + tile * kTileRows, nt * 32 * sizeof(double), &sm.full[s]);
        if (++s == Se) {
          s = 0;
          ++n;
        }
      }
    }
  } else if (warp - 1 < nact) {
    const int cw = warp - 1;
    int s = cw;
    uint32_t n = 0;
    for (int64_t i = cw; i < n_units; i += nact) {
      const int64_t tile0 = t0 + i * TPS;
      const int nt = int(t1 - tile0 < TPS ? t1 - tile0 : TPS);
      mbar_wait(&sm.full[s], n & 1);
      const double* xst = reinterpret_cast<const double*>(sm.xs + size_t(s) * stage_pitch);
      const double* yst = sm.ys + size_t(s) * 32 * TPS;
      double dep = 0.0;
      for (int j = 0; j < nt; ++j)
        consume_tile_rows<KMAX, GRAD>(xst + size_t(j) * kTileRows * K, yst + 32 * j, K, q0, lane,
                                      (tile0 + j) * kTileRows, a.n_rows, sm.sbeta, g, nll, dep);
      mbar_arrive_after(&sm.empty[s], dep, lane, const_cast<double*>(xst));
      s += nact;
      if (s >= Se) {
        s = cw;
        ++n;
      }
    }
  }
  if (warp > 0) {  // every consumer warp (idle ones write zeros): fixed-order butterflies
    const int cw = warp - 1;
    const double ws = warp_sum(nll);
    if (lane == 0) sm.wf[cw] = -ws;
    if (GRAD)
      rows_unrotate<KMAX>(g, K, q0, [&](int k, double v) {
        if (lane == 0) sm.wg[size_t(cw) * K + k] = v;
      });
  }
  cta_reduce_finalize(a, sm, NCW, GRAD);
}

// Per group: fold the partials of its segments (gseg[g] .. gseg[g+1]-1) and warps in order.
template <bool GRAD>
__global__ void hb_fold_kernel(const double* part, const int* gseg, int nw, int K, const double* betas,
                               const double* mu, const double* sigma, double* out_f, double* out_g) {
  pdl_trigger();  // the next evaluation's rows kernel may start streaming X meanwhile
  pdl_wait();     // the rows kernel's partials are complete
  hb_fold_group<GRAD, false>(part, gseg, nw, K, betas, mu, sigma, out_f, out_g, blockIdx.x, threadIdx.x, blockDim.x);
}

}  // namespace pm
