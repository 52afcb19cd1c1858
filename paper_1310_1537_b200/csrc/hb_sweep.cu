// Device-resident hierarchical Gibbs sweep (hb_sweep, hb.py:110-168).
//
// With the hyperprior fixed the G group coefficient vectors are conditionally independent
// (hb.py:1-22), so every group's chain runs in its own CTA: the slice-within-Gibbs update
// of each coordinate (sampler.py:112-167, the same control flow as chain.cu, replayed by
// every thread with explicit _rn arithmetic) evaluates its conditionals with CTA-wide
// passes over the group's rows -- no grid synchronisation, no host round trip.  n_sweeps
// sweeps of all groups are one launch; a group's uniforms are its own numpy Philox stream
// (DeviateBuffer(UNIFORM01, seed, owner=(m,)), hb.py:118-119) generated on the device.
//
// Layout: rows of group g live at padded offset poff[g] (a multiple of 32) of
//   xt [K][ld] (transposed X, the GlmWorkspace.xt of glm.py:468-472), xbeta [ld], y [ld];
// each CTA thread owns rows r = tid, tid + blockDim, ... of its group, so the deferred
// commit_update (xbeta += delta * xt[k], glm.py:525-539) is applied by the thread that
// reads those rows in the next pass.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "glm_kernels.cuh"
#include "philox.cuh"

using namespace pm;

namespace {

constexpr int kHbsThreads = 128;
constexpr int kHbsMaxM = 8;

struct HbsArgs {
  double* xbeta;
  const double* xt;   // [K][ld]
  const double* y;
  const int64_t* poff;   // [G] padded row offset
  const int64_t* nrows;  // [G]
  int64_t ld;
  int G, K;
  const double* mu;
  const double* sigma;
  double* beta;          // [G][K] in/out
  const uint64_t* keys;  // [G][2]
  uint64_t* pos;         // [G] in/out
  long long* evals;      // [G] out (this call)
  int* status;           // [G]: 0 ok, 1 widen, 2 shrink (coordinate in status_k)
  int* status_k;
  int n_sweeps, neval, max_steps;
  double width;
};

__device__ __forceinline__ double hb_logprior(const HbsArgs& a, int k, double v) {
  const double z = __ddiv_rn(__dsub_rn(v, a.mu[k]), a.sigma[k]);
  return __dmul_rn(__dmul_rn(-0.5, z), z);
}

template <int SF, int SN, int MINB>
__global__ void __launch_bounds__(kHbsThreads, MINB) hb_sweep_kernel(HbsArgs a) {
  constexpr int NW = kHbsThreads / 32;
  extern __shared__ double sbeta[];  // [K]
  __shared__ double red[NW][kHbsMaxM];
  __shared__ double tot_s[kHbsMaxM];
  __shared__ double ubuf[32];
  __shared__ uint64_t ubase_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  for (int g = blockIdx.x; g < a.G; g += gridDim.x) {
    const int64_t off = a.poff[g], n = a.nrows[g];
    double* xbeta = a.xbeta + off;
    const double* y = a.y + off;
    const uint64_t k0 = a.keys[2 * g], k1 = a.keys[2 * g + 1];
    __syncthreads();
    for (int k = tid; k < a.K; k += blockDim.x) sbeta[k] = a.beta[int64_t(g) * a.K + k];
    if (tid == 0) ubase_s = ~0ull;
    __syncthreads();
    uint64_t pos = a.pos[g];
    long long evals = 0;
    int pend_k = -1;
    double pend_d = 0.0;

    auto getu = [&](uint64_t idx) -> double {
      const uint64_t base = ubase_s;
      if (base == ~0ull || idx < base || idx >= base + 32) {
        __syncthreads();
        if (warp == 0) ubuf[lane] = double(numpy_philox_word(idx + lane, k0, k1) >> 11) * 0x1p-53;
        if (tid == 0) ubase_s = idx;
        __syncthreads();
        return ubuf[0];
      }
      return ubuf[idx - base];
    };

    // out[m] = L_g(beta + d_m e_k) over the group's rows; applies the pending commit first
    auto pass = [&](auto mtag, int k, const double* d, double* out) {
      constexpr int M = decltype(mtag)::value;
      double acc[M], dm[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        acc[m] = 0.0;
        dm[m] = d[m];
      }
      const double* xk = a.xt + int64_t(k) * a.ld + off;
      const double* xp = pend_k >= 0 ? a.xt + int64_t(pend_k) * a.ld + off : nullptr;
      for (int64_t i = tid; i < n; i += kHbsThreads) {
        double xb = xbeta[i];
        if (xp) {
          xb = __dadd_rn(xb, __dmul_rn(pend_d, xp[i]));
          xbeta[i] = xb;
        }
        const double xv = xk[i], yy = y[i];
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
#pragma unroll
        for (int w = 0; w < NW; ++w) s += red[w][tid];
        tot_s[tid] = -s;
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < M; ++m) out[m] = tot_s[m];
      __syncthreads();
    };

    int status = 0, fail_k = -1;
    for (int sw = 0; sw < a.n_sweeps && !status; ++sw) {
      // neval - 1 extra full evaluations before the update (hb.py:130-131): data reuse only
      for (int e = 1; e < a.neval; ++e) {
        double d0 = 0.0, ll;
        pass(std::integral_constant<int, 1>{}, 0, &d0, &ll);
      }
      for (int k = 0; k < a.K && !status; ++k) {
        const double x0 = sbeta[k];
        const double tiny = __dmul_rn(1e-12, __dadd_rn(1.0, fabs(x0)));
        auto post = [&](double x, double ll) { return __dadd_rn(ll, hb_logprior(a, k, __dadd_rn(x0, __dsub_rn(x, x0)))); };
        auto build = [&](double L, double R, uint64_t p, int nmax, double* cand) -> int {
          int c = 0;
          while (c < nmax) {
            const double x1 = __dadd_rn(L, __dmul_rn(getu(p + c), __dsub_rn(R, L)));
            cand[c++] = x1;
            if (x1 < x0) L = x1; else R = x1;
            if (__dsub_rn(R, L) < tiny) break;
          }
          return c;
        };
        const double u_level = getu(pos);
        const double w = a.width;
        const double r = getu(pos + 1);
        pos += 2;
        double left = __dsub_rn(x0, __dmul_rn(r, w));
        double right = __dadd_rn(left, w);
        constexpr int SC = SF > SN ? SF : SN;
        double cand[SC];
        const int n1 = build(left, right, pos, SF, cand);
        double d1[3 + SF], ll1[3 + SF];
        d1[0] = 0.0;
        d1[1] = __dsub_rn(left, x0);
        d1[2] = __dsub_rn(right, x0);
        for (int j = 0; j < SF; ++j) d1[3 + j] = j < n1 ? __dsub_rn(cand[j], x0) : 0.0;
        pass(std::integral_constant<int, 3 + SF>{}, k, d1, ll1);
        const double f0 = post(x0, ll1[0]);
        evals += 1;
        const double level = __dadd_rn(f0, log(__dsub_rn(1.0, u_level)));
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
        int avail = stepped ? 0 : n1, j = 0;
        double llc[SC];
        for (int q = 0; q < n1; ++q) llc[q] = ll1[3 + q];
        double x1 = x0;
        bool accepted = false;
        for (int s = 0; s < 1000; ++s) {
          if (j == avail) {
            avail = build(left, right, pos, SN, cand);
            double dn[SN];
            for (int q = 0; q < SN; ++q) dn[q] = q < avail ? __dsub_rn(cand[q], x0) : 0.0;
            pass(std::integral_constant<int, SN>{}, k, dn, llc);
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
            x1 = x0;
            accepted = true;
            break;
          }
        }
        if (!accepted) {
          status = 2;
          fail_k = k;
          break;
        }
        const double delta = __dsub_rn(x1, x0);
        if (delta != 0.0) {
          pend_k = k;
          pend_d = delta;
        }
        __syncthreads();
        if (tid == 0) sbeta[k] = __dadd_rn(x0, delta);
        __syncthreads();
      }
    }
    if (pend_k >= 0) {
      const double* xp = a.xt + int64_t(pend_k) * a.ld + off;
      for (int64_t i = tid; i < n; i += kHbsThreads) xbeta[i] = __dadd_rn(xbeta[i], __dmul_rn(pend_d, xp[i]));
    }
    __syncthreads();
    for (int k = tid; k < a.K; k += blockDim.x) a.beta[int64_t(g) * a.K + k] = sbeta[k];
    if (tid == 0) {
      a.pos[g] = pos;
      a.evals[g] = evals;
      a.status[g] = status;
      a.status_k[g] = fail_k;
    }
  }
}

// xbeta = X beta0 per group (GlmWorkspace.__init__, glm.py:468-472), fixed column order
__global__ void hbs_xbeta_kernel(double* xbeta, const double* xt, const int64_t* poff, const int64_t* nrows,
                                 int64_t ld, int K, const double* beta) {
  const int g = blockIdx.x;
  const int64_t off = poff[g], n = nrows[g];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = __dadd_rn(s, __dmul_rn(xt[int64_t(k) * ld + off + i], beta[int64_t(g) * K + k]));
    xbeta[off + i] = s;
  }
}

// Full log-likelihood per group from xbeta (for validate / diagnostics)
__global__ void hbs_loglike_kernel(const double* xbeta, const double* y, const int64_t* poff, const int64_t* nrows,
                                   double* out) {
  const int g = blockIdx.x;
  const int64_t off = poff[g], n = nrows[g];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += row_nll(xbeta[off + i], y[off + i]);
  __shared__ double red[kHbsThreads / 32];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kHbsThreads / 32; ++w) s += red[w];
    out[g] = -s;
  }
}

__global__ void hbs_transpose_kernel(const double* x, int64_t n, int K, const int64_t* src_off,
                                     const int64_t* poff, const int64_t* nrows, double* xt, int64_t ld) {
  const int g = blockIdx.y;
  const int64_t nn = nrows[g];
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nn * K; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / K;
    const int k = int(i % K);
    xt[int64_t(k) * ld + poff[g] + r] = x[(src_off[g] + r) * K + k];
  }
}

}  // namespace

struct pm_hbs_s {
  int device = 0;
  int G = 0, K = 0;
  int64_t ld = 0, n = 0;
  cudaStream_t stream = nullptr;
  double* xt = nullptr;
  double* xbeta = nullptr;
  double* y = nullptr;
  int64_t* poff = nullptr;
  int64_t* nrows = nullptr;
  double* mu = nullptr;
  double* sigma = nullptr;
  double* beta = nullptr;
  uint64_t* keys = nullptr;
  uint64_t* pos = nullptr;
  long long* evals = nullptr;
  int* status = nullptr;
  std::mutex mu_lock;
  float last_ms = 0.f;
};

namespace {
void hbs_free(pm_hbs_s* h) {
  void* ps[] = {h->xt, h->xbeta, h->y, h->poff, h->nrows, h->mu, h->sigma, h->beta, h->keys, h->pos, h->evals, h->status};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (h->stream) cudaStreamDestroy(h->stream);
}
}  // namespace

extern "C" {

int pm_hbs_create(int device, const double* X, const double* y, const int64_t* offsets, int32_t G, int32_t K,
                  const double* mu, const double* sigma, const double* beta0, const uint64_t* keys,
                  const uint64_t* pos, pm_hbs_t* out) {
  if (!X || !y || !offsets || !mu || !sigma || !beta0 || !keys || !pos || !out) return fail(PM_EINVAL, "null argument");
  if (G < 1 || K < 1) return fail(PM_EINVAL, "need G >= 1 and K >= 1");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(PM_EDEVICE, "no CUDA device visible");
  if (device < 0 || device >= ndev) return fail(PM_ERANGE, "device index out of range");
  if (offsets[0] != 0) return fail(PM_EINVAL, "offsets[0] must be 0");
  std::vector<int64_t> poff(G), nrows(G);
  int64_t ld = 0;
  for (int g = 0; g < G; ++g) {
    const int64_t m = offsets[g + 1] - offsets[g];
    if (m < 1) return fail(PM_EINVAL, "every group needs >= 1 row");
    poff[g] = ld;
    nrows[g] = m;
    ld += (m + 31) / 32 * 32;
  }
  const int64_t N = offsets[G];
  for (int k = 0; k < K; ++k)
    if (!(sigma[k] > 0) || !std::isfinite(mu[k])) return fail(PM_EINVAL, "prior must be finite with sigma > 0");
  DeviceGuard dg(device);
  auto* h = new pm_hbs_s;
  h->device = device;
  h->G = G;
  h->K = K;
  h->ld = ld;
  h->n = N;
  auto bail = [&](cudaError_t e, const char* what) {
    hbs_free(h);
    delete h;
    return cuda_fail(e, what);
  };
#define HBS_TRY(call)                       \
  do {                                      \
    cudaError_t _e = (call);                \
    if (_e != cudaSuccess) return bail(_e, #call); \
  } while (0)
  HBS_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  HBS_TRY(cudaMalloc(&h->xt, sizeof(double) * size_t(K) * ld));
  HBS_TRY(cudaMalloc(&h->xbeta, sizeof(double) * ld));
  HBS_TRY(cudaMalloc(&h->y, sizeof(double) * ld));
  HBS_TRY(cudaMalloc(&h->poff, sizeof(int64_t) * G));
  HBS_TRY(cudaMalloc(&h->nrows, sizeof(int64_t) * G));
  HBS_TRY(cudaMalloc(&h->mu, sizeof(double) * K));
  HBS_TRY(cudaMalloc(&h->sigma, sizeof(double) * K));
  HBS_TRY(cudaMalloc(&h->beta, sizeof(double) * size_t(G) * K));
  HBS_TRY(cudaMalloc(&h->keys, sizeof(uint64_t) * 2 * G));
  HBS_TRY(cudaMalloc(&h->pos, sizeof(uint64_t) * G));
  HBS_TRY(cudaMalloc(&h->evals, sizeof(long long) * G));
  HBS_TRY(cudaMalloc(&h->status, sizeof(int) * 2 * G));
  cudaStream_t st = h->stream;
  HBS_TRY(cudaMemsetAsync(h->xt, 0, sizeof(double) * size_t(K) * ld, st));
  HBS_TRY(cudaMemsetAsync(h->y, 0, sizeof(double) * ld, st));
  // y into padded positions
  for (int g = 0; g < G; ++g)
    HBS_TRY(cudaMemcpyAsync(h->y + poff[g], y + offsets[g], sizeof(double) * nrows[g], cudaMemcpyHostToDevice, st));
  HBS_TRY(cudaMemcpyAsync(h->poff, poff.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, st));
  HBS_TRY(cudaMemcpyAsync(h->nrows, nrows.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, st));
  HBS_TRY(cudaMemcpyAsync(h->mu, mu, sizeof(double) * K, cudaMemcpyHostToDevice, st));
  HBS_TRY(cudaMemcpyAsync(h->sigma, sigma, sizeof(double) * K, cudaMemcpyHostToDevice, st));
  HBS_TRY(cudaMemcpyAsync(h->beta, beta0, sizeof(double) * size_t(G) * K, cudaMemcpyHostToDevice, st));
  HBS_TRY(cudaMemcpyAsync(h->keys, keys, sizeof(uint64_t) * 2 * G, cudaMemcpyHostToDevice, st));
  HBS_TRY(cudaMemcpyAsync(h->pos, pos, sizeof(uint64_t) * G, cudaMemcpyHostToDevice, st));
  // X (row-major, CSR rows) -> per-group transposed columns, in bounded chunks of groups
  {
    std::vector<int64_t> src_off(offsets, offsets + G);
    int64_t* d_src = nullptr;
    HBS_TRY(cudaMalloc(&d_src, sizeof(int64_t) * G));
    HBS_TRY(cudaMemcpyAsync(d_src, src_off.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, st));
    double* d_x = nullptr;
    HBS_TRY(cudaMalloc(&d_x, sizeof(double) * size_t(N) * K));
    HBS_TRY(cudaMemcpyAsync(d_x, X, sizeof(double) * size_t(N) * K, cudaMemcpyHostToDevice, st));
    hbs_transpose_kernel<<<dim3(64, G), 256, 0, st>>>(d_x, N, K, d_src, h->poff, h->nrows, h->xt, ld);
    HBS_TRY(cudaGetLastError());
    HBS_TRY(cudaStreamSynchronize(st));
    cudaFree(d_x);
    cudaFree(d_src);
  }
  hbs_xbeta_kernel<<<G, kHbsThreads, 0, st>>>(h->xbeta, h->xt, h->poff, h->nrows, ld, K, h->beta);
  HBS_TRY(cudaGetLastError());
  HBS_TRY(cudaStreamSynchronize(st));
#undef HBS_TRY
  *out = h;
  return PM_OK;
}

int pm_hbs_destroy(pm_hbs_t h) {
  if (!h) return PM_OK;
  {
    DeviceGuard dg(h->device);
    hbs_free(h);
  }
  delete h;
  return PM_OK;
}

int pm_hbs_sweeps(pm_hbs_t h, int32_t n_sweeps, int32_t neval, double slice_width, int32_t max_steps,
                  double* betas_out, uint64_t* pos_out, int64_t* evals_out, int32_t* fail_group, int32_t* fail_coord,
                  float* ms) {
  if (!h || !betas_out || !pos_out || !evals_out) return fail(PM_EINVAL, "null argument");
  if (n_sweeps < 0) return fail(PM_EINVAL, "n_sweeps must be >= 0");
  if (neval < 1) return fail(PM_EINVAL, "neval must be >= 1");
  if (!(slice_width > 0) || !std::isfinite(slice_width)) return fail(PM_EINVAL, "slice_width must be > 0");
  if (max_steps < 1) return fail(PM_EINVAL, "slice_max_steps must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu_lock);
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  HbsArgs a;
  a.xbeta = h->xbeta;
  a.xt = h->xt;
  a.y = h->y;
  a.poff = h->poff;
  a.nrows = h->nrows;
  a.ld = h->ld;
  a.G = h->G;
  a.K = h->K;
  a.mu = h->mu;
  a.sigma = h->sigma;
  a.beta = h->beta;
  a.keys = h->keys;
  a.pos = h->pos;
  a.evals = h->evals;
  a.status = h->status;
  a.status_k = h->status + h->G;
  a.n_sweeps = n_sweeps;
  a.neval = neval;
  a.max_steps = max_steps;
  a.width = slice_width;
  const int spec = tune("hbs_spec", 1);  // measured on B200 (tools/ab_hbs.sh): no speculation, 8 CTAs/SM
  const size_t smem = sizeof(double) * size_t(h->K);
  // CTAs per SM the register budget must allow (1000 groups fit one wave at >= 7 per SM)
  const int minb = tune("hbs_minb", 8);
  void (*kfn)(HbsArgs);
  if (spec >= 4) kfn = hb_sweep_kernel<4, 3, 4>;
  else if (spec >= 2) kfn = minb >= 8 ? hb_sweep_kernel<2, 2, 8> : minb >= 7 ? hb_sweep_kernel<2, 2, 7> : hb_sweep_kernel<2, 2, 4>;
  else kfn = minb >= 8 ? hb_sweep_kernel<1, 1, 8> : hb_sweep_kernel<1, 1, 4>;
  int per_sm = 0;
  PM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kHbsThreads, smem));
  if (per_sm < 1) return fail(PM_EDEVICE, "hb sweep kernel cannot be resident");
  const int grid = std::max(1, std::min(h->G, sm_count(h->device) * per_sm));
  cudaEvent_t e0, e1;
  PM_CUDA(cudaEventCreate(&e0));
  PM_CUDA(cudaEventCreate(&e1));
  PM_CUDA(cudaEventRecord(e0, st));
  if (n_sweeps > 0) kfn<<<grid, kHbsThreads, smem, st>>>(a);
  PM_CUDA(cudaGetLastError());
  PM_CUDA(cudaEventRecord(e1, st));
  PM_CUDA(cudaEventSynchronize(e1));
  PM_CUDA(cudaEventElapsedTime(&h->last_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (ms) *ms = h->last_ms;
  std::vector<long long> ev(h->G, 0);
  std::vector<int> stat(2 * size_t(h->G), 0);
  PM_CUDA(cudaMemcpyAsync(betas_out, h->beta, sizeof(double) * size_t(h->G) * h->K, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaMemcpyAsync(pos_out, h->pos, sizeof(uint64_t) * h->G, cudaMemcpyDeviceToHost, st));
  if (n_sweeps > 0) {
    PM_CUDA(cudaMemcpyAsync(ev.data(), h->evals, sizeof(long long) * h->G, cudaMemcpyDeviceToHost, st));
    PM_CUDA(cudaMemcpyAsync(stat.data(), h->status, sizeof(int) * 2 * h->G, cudaMemcpyDeviceToHost, st));
  }
  PM_CUDA(cudaStreamSynchronize(st));
  for (int g = 0; g < h->G; ++g) evals_out[g] = ev[g];
  for (int g = 0; g < h->G; ++g) {
    if (stat[g]) {
      if (fail_group) *fail_group = g;
      if (fail_coord) *fail_coord = stat[h->G + g];
      if (stat[g] == 1)
        return fail(PM_ESLICE, "stepping-out exceeded " + std::to_string(max_steps) + " steps (group " +
                                   std::to_string(g) + ", coordinate " + std::to_string(stat[h->G + g]) + ")");
      return fail(PM_ESHRINK, "slice shrinkage failed to accept (group " + std::to_string(g) + ", coordinate " +
                                  std::to_string(stat[h->G + g]) + ")");
    }
  }
  return PM_OK;
}

int pm_hbs_set_prior(pm_hbs_t h, const double* mu, const double* sigma) {
  if (!h || !mu || !sigma) return fail(PM_EINVAL, "null argument");
  for (int k = 0; k < h->K; ++k)
    if (!(sigma[k] > 0) || !std::isfinite(mu[k])) return fail(PM_EINVAL, "prior must be finite with sigma > 0");
  std::lock_guard<std::mutex> lk(h->mu_lock);
  DeviceGuard dg(h->device);
  PM_CUDA(cudaMemcpyAsync(h->mu, mu, sizeof(double) * h->K, cudaMemcpyHostToDevice, h->stream));
  PM_CUDA(cudaMemcpyAsync(h->sigma, sigma, sizeof(double) * h->K, cudaMemcpyHostToDevice, h->stream));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  return PM_OK;
}

int pm_hbs_loglike(pm_hbs_t h, double* ll_out) {
  if (!h || !ll_out) return fail(PM_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(h->mu_lock);
  DeviceGuard dg(h->device);
  cudaStream_t st = h->stream;
  double* d = nullptr;
  PM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), sizeof(double) * h->G, st));
  hbs_loglike_kernel<<<h->G, kHbsThreads, 0, st>>>(h->xbeta, h->y, h->poff, h->nrows, d);
  PM_CUDA(cudaGetLastError());
  PM_CUDA(cudaMemcpyAsync(ll_out, d, sizeof(double) * h->G, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaFreeAsync(d, st));
  PM_CUDA(cudaStreamSynchronize(st));
  return PM_OK;
}

int pm_hbs_read_xbeta(pm_hbs_t h, double* out) {
  if (!h || !out) return fail(PM_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(h->mu_lock);
  DeviceGuard dg(h->device);
  std::vector<int64_t> poff(h->G), nrows(h->G);
  PM_CUDA(cudaMemcpy(poff.data(), h->poff, sizeof(int64_t) * h->G, cudaMemcpyDeviceToHost));
  PM_CUDA(cudaMemcpy(nrows.data(), h->nrows, sizeof(int64_t) * h->G, cudaMemcpyDeviceToHost));
  int64_t o = 0;
  for (int g = 0; g < h->G; ++g) {
    PM_CUDA(cudaMemcpy(out + o, h->xbeta + poff[g], sizeof(double) * nrows[g], cudaMemcpyDeviceToHost));
    o += nrows[g];
  }
  return PM_OK;
}

}  // extern "C"
