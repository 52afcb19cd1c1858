// Device-resident slice-within-Gibbs chain.
//
// One cooperative persistent kernel runs run_chain (sampler.py:170-200) end to end:
//   * every thread replays the reference's scalar control flow of slice_sample_coord
//     (sampler.py:112-167) identically -- stepping-out, shrinkage, degenerate-slice exit,
//     SliceWidenError / shrink-failure -- with explicit __dmul_rn/__dadd_rn/__dsub_rn so the
//     interval arithmetic rounds exactly like the host (no FMA contraction);
//   * the uniforms are the numpy Philox4x64-10 DeviateBuffer stream (rng.py:42-44), generated
//     on the device at the buffer's position, consumed in the reference's order;
//   * each conditional evaluation is one grid-wide pass over (xbeta, xt[k], y)
//     (glm.py:499-522) with a fixed-order reduction and ONE grid sync (partials double-buffered);
//     f0 and the first stepping-out interval are evaluated in one 3-delta pass;
//   * commit_update (glm.py:525-539) is fused into the next pass: each thread owns a fixed set
//     of rows, so it applies xbeta += delta*xt[k] to its rows right before reading them.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "glm_kernels.cuh"
#include "philox.cuh"

namespace cg = cooperative_groups;
using namespace pm;

namespace {

constexpr int kChainThreads = 256;
constexpr int kChainMaxM = 9;  // deltas per pass (3 + kSpecFirst)

struct ChainArgs {
  double* xbeta;
  const double* xt;      // [K][ld]
  const double* y;
  int64_t n, ld;
  int K;
  const double* mu;
  const double* sigma;
  int n_iter, n_burnin, max_steps;
  double width;
  uint64_t key0, key1, pos0;
  double* beta;          // [K] in/out
  double* draws;         // [n_iter - n_burnin][K]
  unsigned long long* bar;  // grid barrier arrival count (zero at launch); null: cg grid sync
  double* partials;      // [2][kChainMaxM][grid] (coalesced fold: every CTA reads all of a delta's partials)
  unsigned long long* out_pos;
  long long* out_evals;
  int* status;           // [0] = 0 ok / 1 widen / 2 shrink, [1] = coordinate
};

__device__ __forceinline__ double uniform_at(const ChainArgs& a, uint64_t idx) {
  return double(numpy_philox_word(idx, a.key0, a.key1) >> 11) * 0x1p-53;
}

// GaussianPrior.logpdf_coord(k, v) (sampler.py:55-58)
__device__ __forceinline__ double logprior(const ChainArgs& a, int k, double v) {
  const double z = __ddiv_rn(__dsub_rn(v, a.mu[k]), a.sigma[k]);
  return __dmul_rn(__dmul_rn(-0.5, z), z);
}

// U: rows per ILP batch; SF: shrink candidates evaluated with f0/left/right in the first pass;
// SN: shrink candidates per later pass
template <int U, int SF, int SN>
__global__ void __launch_bounds__(kChainThreads) chain_kernel(ChainArgs a) {
  constexpr int kSpecFirst = SF;
  constexpr int kSpecNext = SN;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sbeta[];  // [K]
  __shared__ double red[kChainThreads / 32][kChainMaxM];
  __shared__ double tot_s[kChainMaxM];
  __shared__ double ubuf[32];        // uniforms of stream indices ubase .. ubase+31
  __shared__ uint64_t ubase_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  unsigned long long bar_target = 0;  // thread 0: arrivals expected after this CTA's next barrier
  for (int k = tid; k < a.K; k += blockDim.x) sbeta[k] = a.beta[k];
  if (tid == 0) ubase_s = ~0ull;
  __syncthreads();

  uint64_t pos = a.pos0;
  long long evals = 0;
  int parity = 0;
  int pend_k = -1;
  double pend_d = 0.0;
  const int64_t stride = int64_t(G) * blockDim.x;
  const int64_t i0 = int64_t(blockIdx.x) * blockDim.x + tid;

  // Uniform of stream index idx (numpy Philox DeviateBuffer stream).  Every thread of the CTA
  // calls this with the same idx at the same point; warp 0 refills 32 consecutive uniforms.
  auto getu = [&](uint64_t idx) -> double {
    const uint64_t base = ubase_s;
    if (base == ~0ull || idx < base || idx >= base + 32) {
      __syncthreads();
      if (warp == 0) ubuf[lane] = uniform_at(a, idx + lane);
      if (tid == 0) ubase_s = idx;
      __syncthreads();
      return ubuf[0];
    }
    return ubuf[idx - base];
  };

  // One conditional log-likelihood pass for M deltas of coordinate k: out[m] = L(beta + d_m e_k).
  auto pass = [&](auto mtag, int k, const double* d, double* out) {
    constexpr int M = decltype(mtag)::value;
    double acc[M];
#pragma unroll
    for (int m = 0; m < M; ++m) acc[m] = 0.0;
    double dm[M];
#pragma unroll
    for (int m = 0; m < M; ++m) dm[m] = d[m];
    const double* xk = a.xt + int64_t(k) * a.ld;
    const double* xp = pend_k >= 0 ? a.xt + int64_t(pend_k) * a.ld : nullptr;
    // U rows per step: all loads first, then U independent transcendental chains (ILP);
    // the per-thread summation order is the same for every M (rows in ascending order)
    int64_t i = i0;
    for (; i + (U - 1) * stride < a.n; i += U * stride) {
      double xb[U], xv[U], yy[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t r = i + u * stride;
        xb[u] = a.xbeta[r];
        xv[u] = xk[r];
        yy[u] = a.y[r];
        if (xp) xb[u] = __dadd_rn(xb[u], __dmul_rn(pend_d, xp[r]));  // fused commit_update, glm.py:537
      }
      if (xp) {
#pragma unroll
        for (int u = 0; u < U; ++u) a.xbeta[i + u * stride] = xb[u];
      }
#pragma unroll
      for (int m = 0; m < M; ++m) {
        double t[U];
#pragma unroll
        for (int u = 0; u < U; ++u) t[u] = row_nll(shifted_t(xb[u], dm[m], xv[u]), yy[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc[m] += t[u];
      }
    }
    for (; i < a.n; i += stride) {
      double xb = a.xbeta[i];
      if (xp) {
        xb = __dadd_rn(xb, __dmul_rn(pend_d, xp[i]));
        a.xbeta[i] = xb;
      }
      const double xv = xk[i], yy = a.y[i];
#pragma unroll
      for (int m = 0; m < M; ++m) acc[m] += row_nll(shifted_t(xb, dm[m], xv), yy);
    }
    pend_k = -1;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const double s = warp_sum(acc[m]);
      if (lane == 0) red[warp][m] = s;
    }
    __syncthreads();
    if (tid < M) {
      double s = 0.0;
      for (int w = 0; w < kChainThreads / 32; ++w) s += red[w][tid];
      a.partials[(size_t(parity) * kChainMaxM + tid) * G + blockIdx.x] = s;  // [parity][m][cta]: the fold reads rows
    }
    // grid-wide barrier (the launch is cooperative: all CTAs are resident).  One release
    // add by thread 0 after the CTA barrier publishes this CTA's partials (PTX fences are
    // cumulative over writes ordered before them by bar.sync); the acquire spin on the
    // monotonic arrival count orders every other CTA's before the fold's loads.  Replaces
    // cg::grid_group::sync (two extra fences and CTA barriers per pass).
    if (a.bar) {
      __syncthreads();
      if (tid == 0) {
        bar_target += G;
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(a.bar) : "memory");
        unsigned long long seen;
        do {
          asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(seen) : "l"(a.bar) : "memory");
        } while (seen < bar_target);
      }
      __syncthreads();
    } else {
      grid.sync();
    }
    // every CTA folds all CTA partials in the same fixed order: warp w folds delta m = w, w+8..
    for (int m = warp; m < M; m += kChainThreads / 32) {
      const double p = warp_sum(fold_lane(a.partials + (size_t(parity) * kChainMaxM + m) * G, 1, G, lane));
      if (lane == 0) tot_s[m] = -p;
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < M; ++m) out[m] = tot_s[m];
    __syncthreads();
    parity ^= 1;
  };

  int status = 0, fail_k = -1;
  for (int it = 0; it < a.n_iter && !status; ++it) {
    for (int k = 0; k < a.K && !status; ++k) {
      const double x0 = sbeta[k];
      const double tiny = __dmul_rn(1e-12, __dadd_rn(1.0, fabs(x0)));
      // log_posterior_coord(ws, data, prior, k, x - x0) = ll + logpdf(k, beta_k + (x - x0))
      auto post = [&](double x, double ll) { return __dadd_rn(ll, logprior(a, k, __dadd_rn(x0, __dsub_rn(x, x0)))); };
      // Shrink candidates from (L, R) starting at stream index p, each assuming the previous
      // one was rejected: after a rejection the new interval depends only on x1 < x0
      // (sampler.py:156-162), so the sequence is known before any comparison.
      auto build = [&](double L, double R, uint64_t p, int nmax, double* cand) -> int {
        int n = 0;
        while (n < nmax) {
          const double x1 = __dadd_rn(L, __dmul_rn(getu(p + n), __dsub_rn(R, L)));
          cand[n++] = x1;
          if (x1 < x0) L = x1; else R = x1;
          if (__dsub_rn(R, L) < tiny) break;  // the scan ends here whatever the outcome
        }
        return n;
      };
      const double u_level = getu(pos);
      const double w = a.width;
      const double r = getu(pos + 1);
      pos += 2;
      double left = __dsub_rn(x0, __dmul_rn(r, w));
      double right = __dadd_rn(left, w);
      // pass 1: f0, left_0, right_0 and kSpecFirst shrink candidates (assuming no stepping-out)
      double cand[kSpecFirst > kSpecNext ? kSpecFirst : kSpecNext];
      const int n1 = build(left, right, pos, kSpecFirst, cand);
      double d1[3 + kSpecFirst], ll1[3 + kSpecFirst];
      d1[0] = 0.0;
      d1[1] = __dsub_rn(left, x0);
      d1[2] = __dsub_rn(right, x0);
      for (int j = 0; j < kSpecFirst; ++j) d1[3 + j] = j < n1 ? __dsub_rn(cand[j], x0) : 0.0;
      pass(std::integral_constant<int, 3 + kSpecFirst>{}, k, d1, ll1);
      const double f0 = post(x0, ll1[0]);
      evals += 1;
      const double level = __dadd_rn(f0, log(__dsub_rn(1.0, u_level)));
      // stepping out (sampler.py:138-150)
      bool stepped = false;
      double fl = post(left, ll1[1]);
      evals += 1;
      int steps = 0;
      while (fl > level) {
        stepped = true;
        left = __dsub_rn(left, w);
        if (++steps > a.max_steps) {
          status = 1;
          fail_k = k;
          break;
        }
        double dd = __dsub_rn(left, x0), ll;
        pass(std::integral_constant<int, 1>{}, k, &dd, &ll);
        fl = post(left, ll);
        evals += 1;
      }
      if (status) break;
      double fr = post(right, ll1[2]);
      evals += 1;
      steps = 0;
      while (fr > level) {
        stepped = true;
        right = __dadd_rn(right, w);
        if (++steps > a.max_steps) {
          status = 1;
          fail_k = k;
          break;
        }
        double dd = __dsub_rn(right, x0), ll;
        pass(std::integral_constant<int, 1>{}, k, &dd, &ll);
        fr = post(right, ll);
        evals += 1;
      }
      if (status) break;
      // shrinkage (sampler.py:152-164), candidates consumed in order from speculative batches
      int avail = stepped ? 0 : n1, j = 0;
      double llc[kSpecFirst > kSpecNext ? kSpecFirst : kSpecNext];
      for (int q = 0; q < n1; ++q) llc[q] = ll1[3 + q];
      double x1 = x0;
      bool accepted = false;
      for (int s = 0; s < 1000; ++s) {
        if (j == avail) {  // next batch from the current interval
          avail = build(left, right, pos, kSpecNext, cand);
          double dn[kSpecNext];
          for (int q = 0; q < kSpecNext; ++q) dn[q] = q < avail ? __dsub_rn(cand[q], x0) : 0.0;
          pass(std::integral_constant<int, kSpecNext>{}, k, dn, llc);
          j = 0;
        }
        x1 = cand[j];
        const double f1 = post(x1, llc[j]);
        ++j;
        ++pos;
        evals += 1;
        if (f1 > level) {
          accepted = true;
          break;
        }
        if (x1 < x0)
          left = x1;
        else
          right = x1;
        if (__dsub_rn(right, left) < tiny) {
          x1 = x0;  // degenerate slice; keep the current point
          accepted = true;
          break;
        }
      }
      if (!accepted) {
        status = 2;
        fail_k = k;
        break;
      }
      // commit_update(ws, k, x1 - x0): beta_k += delta; xbeta update deferred to the next pass
      const double delta = __dsub_rn(x1, x0);
      if (delta != 0.0) {
        pend_k = k;
        pend_d = delta;
      }
      __syncthreads();
      if (tid == 0) sbeta[k] = __dadd_rn(x0, delta);
      __syncthreads();
    }
    if (!status && it >= a.n_burnin && blockIdx.x == 0) {
      for (int k = tid; k < a.K; k += blockDim.x) a.draws[int64_t(it - a.n_burnin) * a.K + k] = sbeta[k];
    }
  }
  // flush the last pending commit (no reduction needed)
  if (pend_k >= 0) {
    const double* xp = a.xt + int64_t(pend_k) * a.ld;
    for (int64_t i = i0; i < a.n; i += stride) a.xbeta[i] = __dadd_rn(a.xbeta[i], __dmul_rn(pend_d, xp[i]));
  }
  if (blockIdx.x == 0) {
    for (int k = tid; k < a.K; k += blockDim.x) a.beta[k] = sbeta[k];
    if (tid == 0) {
      *a.out_pos = pos;
      *a.out_evals = evals;
      a.status[0] = status;
      a.status[1] = fail_k;
    }
  }
}

thread_local float g_last_chain_ms = 0.f;

}  // namespace

extern "C" {

int pm_chain_last_kernel_ms(float* ms) {
  if (!ms) return fail(PM_EINVAL, "null argument");
  *ms = g_last_chain_ms;
  return PM_OK;
}

int pm_ws_run_chain(pm_ws_t ws, const double* mu, const double* sigma, int32_t n_iter, int32_t n_burnin,
                    double slice_width, int32_t slice_max_steps, uint64_t key0, uint64_t key1, uint64_t stream_pos,
                    double* draws_out, double* beta_inout, uint64_t* stream_pos_out, int64_t* evals_out,
                    int32_t* fail_coord) {
  if (!ws || !mu || !sigma || !beta_inout || !stream_pos_out || !evals_out) return fail(PM_EINVAL, "null argument");
  if (n_iter < 1 || n_burnin < 0 || n_burnin >= n_iter) return fail(PM_EINVAL, "need 0 <= n_burnin < n_iter");
  if (!(slice_width > 0) || !std::isfinite(slice_width)) return fail(PM_EINVAL, "slice_width must be > 0");
  if (slice_max_steps < 1) return fail(PM_EINVAL, "slice_max_steps must be >= 1");
  if ((n_iter - n_burnin) > 0 && !draws_out) return fail(PM_EINVAL, "draws_out is null");
  pm_ws_view v;
  int rc = pm_ws_internal_view(ws, &v);
  if (rc) return rc;
  for (int k = 0; k < v.K; ++k)
    if (!(sigma[k] > 0) || !std::isfinite(mu[k]) || !std::isfinite(beta_inout[k]))
      return fail(PM_EINVAL, "prior / beta must be finite with sigma > 0");
  pm_ws_internal_lock(ws, 1);
  struct Unlock {
    pm_ws_t w;
    ~Unlock() { pm_ws_internal_lock(w, 0); }
  } unlock{ws};
  DeviceGuard g(v.device);
  cudaStream_t st = static_cast<cudaStream_t>(v.stream);
  const size_t smem = sizeof(double) * size_t(v.K);
  // tuning knobs (defaults measured on B200): rows per ILP batch and CTAs per SM
  const int unroll = tune("chain_unroll", 2);
  const int want_per_sm = std::max(1, tune("chain_blocks_per_sm", 2));
  const int spec = tune("chain_spec", 4);  // speculative shrink candidates in the first pass
  void* kfn;
  if (spec >= 6) kfn = unroll >= 2 ? reinterpret_cast<void*>(chain_kernel<2, 6, 4>) : reinterpret_cast<void*>(chain_kernel<1, 6, 4>);
  else if (spec >= 4) kfn = unroll >= 2 ? reinterpret_cast<void*>(chain_kernel<2, 4, 3>) : reinterpret_cast<void*>(chain_kernel<1, 4, 3>);
  else if (spec >= 2) kfn = unroll >= 2 ? reinterpret_cast<void*>(chain_kernel<2, 2, 2>) : reinterpret_cast<void*>(chain_kernel<1, 2, 2>);
  else kfn = unroll >= 2 ? reinterpret_cast<void*>(chain_kernel<2, 1, 1>) : reinterpret_cast<void*>(chain_kernel<1, 1, 1>);
  int per_sm = 0;
  PM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kChainThreads, smem));
  if (per_sm < 1) return fail(PM_EDEVICE, "chain kernel cannot be resident");
  const int grid = std::max(1, std::min(v.sms * std::min(per_sm, want_per_sm),
                                        int((v.n + kChainThreads - 1) / kChainThreads)));
  const int kept = n_iter - n_burnin;
  double* dbuf = nullptr;
  const size_t nd = size_t(3) * v.K + size_t(kept) * v.K + size_t(2) * grid * kChainMaxM;
  // stream-ordered allocation: no device-wide synchronisation of cudaMalloc/cudaFree
  pm::retain_pool(v.device);
  PM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dbuf), sizeof(double) * nd + 64, st));
  struct Free {
    void* p;
    cudaStream_t s;
    ~Free() { cudaFreeAsync(p, s); }
  } fr{dbuf, st};
  double* d_mu = dbuf;
  double* d_sigma = d_mu + v.K;
  double* d_beta = d_sigma + v.K;
  double* d_draws = d_beta + v.K;
  double* d_part = d_draws + size_t(kept) * v.K;
  unsigned long long* d_pos = reinterpret_cast<unsigned long long*>(d_part + size_t(2) * grid * kChainMaxM);
  long long* d_evals = reinterpret_cast<long long*>(d_pos + 1);
  int* d_status = reinterpret_cast<int*>(d_evals + 1);
  PM_CUDA(cudaMemcpyAsync(d_mu, mu, sizeof(double) * v.K, cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemcpyAsync(d_sigma, sigma, sizeof(double) * v.K, cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemcpyAsync(d_beta, beta_inout, sizeof(double) * v.K, cudaMemcpyHostToDevice, st));
  ChainArgs a;
  a.xbeta = v.xbeta;
  a.xt = v.xt;
  a.y = v.y;
  a.n = v.n;
  a.ld = v.ld;
  a.K = v.K;
  a.mu = d_mu;
  a.sigma = d_sigma;
  a.n_iter = n_iter;
  a.n_burnin = n_burnin;
  a.max_steps = slice_max_steps;
  a.width = slice_width;
  a.key0 = key0;
  a.key1 = key1;
  a.pos0 = stream_pos;
  a.beta = d_beta;
  a.draws = d_draws;
  a.partials = d_part;
  a.bar = tune("chain_own_barrier", 0) != 0 ? d_pos + 4 : nullptr;  // inside the 64 trailing bytes
  PM_CUDA(cudaMemsetAsync(d_pos + 4, 0, sizeof(unsigned long long), st));
  a.out_pos = d_pos;
  a.out_evals = d_evals;
  a.status = d_status;
  void* kargs[] = {&a};
  // the kernel is always bracketed by CUDA events (pm_chain_last_kernel_ms)
  cudaEvent_t te0 = nullptr, te1 = nullptr;
  PM_CUDA(cudaEventCreate(&te0));
  PM_CUDA(cudaEventCreate(&te1));
  PM_CUDA(cudaEventRecord(te0, st));
  PM_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(grid), dim3(kChainThreads), kargs, smem, st));
  PM_CUDA(cudaEventRecord(te1, st));
  PM_CUDA(cudaEventSynchronize(te1));
  PM_CUDA(cudaEventElapsedTime(&g_last_chain_ms, te0, te1));
  cudaEventDestroy(te0);
  cudaEventDestroy(te1);
  unsigned long long pos = 0;
  long long evals = 0;
  int status[2] = {0, -1};
  PM_CUDA(cudaMemcpyAsync(&pos, d_pos, sizeof(pos), cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaMemcpyAsync(&evals, d_evals, sizeof(evals), cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaMemcpyAsync(status, d_status, sizeof(status), cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaMemcpyAsync(beta_inout, d_beta, sizeof(double) * v.K, cudaMemcpyDeviceToHost, st));
  if (kept > 0)
    PM_CUDA(cudaMemcpyAsync(draws_out, d_draws, sizeof(double) * size_t(kept) * v.K, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  *stream_pos_out = pos;
  *evals_out = evals;
  if (fail_coord) *fail_coord = status[1];
  if (status[0] == 1)
    return fail(PM_ESLICE, "stepping-out exceeded " + std::to_string(slice_max_steps) + " steps (coordinate " +
                               std::to_string(status[1]) + ")");
  if (status[0] == 2)
    return fail(PM_ESHRINK, "slice shrinkage failed to accept (coordinate " + std::to_string(status[1]) + ")");
  return PM_OK;
}

}  // extern "C"
