// Host side of the GLM hot path: handles, geometry, dispatch and the C ABI
// (include/pmb200.h).  Kernels live in glm_kernels.cuh / glm_aux_kernels.cuh.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "glm_aux_kernels.cuh"

using namespace pm;

namespace {

// consumer warps of the streaming kernel: 7 + 1 producer = 8 warps = 2 per SMSP, which lets
// ptxas give each thread up to 255 registers (9 warps put 3 on one SMSP -> 168 max)
constexpr int kNCW = 7;
constexpr int kStreamThreads = (kNCW + 1) * 32;
constexpr int kMaxStages = 16;
constexpr int kHbNCW = 4;
constexpr int kHbThreads = (kHbNCW + 1) * 32;
constexpr int kHbMaxStages = 6;
constexpr int kHbRowsNCW = 15;                        // small-K row-per-lane path (1 CTA/SM)
constexpr int kHbRowsThreads = (kHbRowsNCW + 1) * 32;
constexpr int kWideThreads = 256;
constexpr int kMaxKC = 8;                    // stream kernel handles K <= 256

enum KernelKind { KIND_NONE = 0, KIND_STREAM = 1, KIND_WIDE = 2, KIND_ROWS = 3 };

int max_optin_smem(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  return v;
}

// finite <=> exponent field not all ones; branch-free so the host compiler vectorises it
// (an early-exit isfinite loop costs ~7 us per 20,000 doubles: every HB evaluation)
bool all_finite(const double* p, int64_t n) {
  constexpr uint64_t kExp = 0x7ff0000000000000ull;
  uint64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t b;
    std::memcpy(&b, p + i, sizeof(b));
    bad |= uint64_t((b & kExp) == kExp);
  }
  return bad == 0;
}

// dst[0..n) = src[0..n) and the same finiteness test in one pass over the data
bool copy_check_finite(double* dst, const double* src, int64_t n) {
  constexpr uint64_t kExp = 0x7ff0000000000000ull;
  uint64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    uint64_t b;
    std::memcpy(&b, src + i, sizeof(b));
    bad |= uint64_t((b & kExp) == kExp);
    std::memcpy(dst + i, &b, sizeof(b));
  }
  return bad == 0;
}

template <typename T>
__global__ void count_nonfinite(const T* __restrict__ p, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    c += isfinite(p[i]) ? 0ull : 1ull;
  for (int s = 16; s >= 1; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

}  // namespace

struct pm_glm_s {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  std::mutex mu;
  // data
  void* X = nullptr;
  double* y = nullptr;
  int xtype = PM_X_F64;
  int64_t n_rows = 0, n_pad = 0, n_tiles = 0;
  int K = 0;
  // prior
  double* prior_mu = nullptr;
  double* prior_sigma = nullptr;
  double* prior_terms = nullptr;  // [K+1] scratch of the kernels' prior_precompute
  bool has_prior = false;
  // scratch
  double* partials = nullptr;
  int partials_cap = 0;
  unsigned int* counter = nullptr;
  double* out_host = nullptr;   // mapped pinned [K+2]: (f, g[K]) and the completion word
  unsigned long long seq = 0;   // evaluations launched through pm_glm_launch / pm_glm_eval
  double* out_dev = nullptr;    // device alias of out_host
  double* beta_dev = nullptr;   // [K] (wide kernel)
  double* beta_pinned = nullptr;
  double* xt_cache = nullptr;   // [K][n_pad] transposed X, shared by the workspaces
  // geometry
  int kind = KIND_NONE;
  int grid = 0, threads = 0, stages = 0, tps = 1, ncw = 7;
  int pairs = 0;  // fp32-X consumer layout (glm_stream_kernel PAIRS)
  int selfprod = 0;  // row-dot consumer: 1 consumer warps issue their own copies, 3 + warp 0 consumes too
  size_t smem = 0;
  bool launched = false;
  int last_want_grad = 1;
};

namespace {

void free_glm_data(pm_glm_s* h) {
  if (h->X) cudaFree(h->X);
  if (h->y) cudaFree(h->y);
  if (h->partials) cudaFree(h->partials);
  if (h->beta_dev) cudaFree(h->beta_dev);
  if (h->out_host) cudaFreeHost(h->out_host);
  if (h->beta_pinned) cudaFreeHost(h->beta_pinned);
  if (h->prior_mu) cudaFree(h->prior_mu);
  if (h->prior_sigma) cudaFree(h->prior_sigma);
  if (h->prior_terms) cudaFree(h->prior_terms);
  if (h->xt_cache) cudaFree(h->xt_cache);
  h->xt_cache = nullptr;
  h->X = nullptr;
  h->y = nullptr;
  h->partials = nullptr;
  h->beta_dev = nullptr;
  h->out_host = nullptr;
  h->out_dev = nullptr;
  h->beta_pinned = nullptr;
  h->prior_mu = h->prior_sigma = h->prior_terms = nullptr;
  h->has_prior = false;
  h->K = 0;
  h->n_rows = h->n_pad = h->n_tiles = 0;
  h->kind = KIND_NONE;
}

// ---- stream kernel dispatch table ------------------------------------------------
using StreamLaunch = cudaError_t (*)(const GlmArgs&, const double*, int, size_t, cudaStream_t);

template <typename XT, int KC, bool GRAD, int PAIRS = 0>
cudaError_t launch_stream(const GlmArgs& a, const double* beta, int grid, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto kern = glm_stream_kernel<XT, KC, GRAD, kNCW, SubRows<KC, GRAD>::value, kTileRows, PAIRS>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), attr);
  if (e != cudaSuccess) return e;
  BetaPack<KC> bp;
  for (int k = 0; k < 32 * KC; ++k) bp.v[k] = (k < a.K) ? beta[k] : 0.0;
  kern<<<grid, kStreamThreads, smem, st>>>(a, bp);
  return cudaGetLastError();
}

template <typename XT, bool GRAD>
StreamLaunch pick_stream(int kc) {
  switch (kc) {
    case 1: return launch_stream<XT, 1, GRAD>;
    case 2: return launch_stream<XT, 2, GRAD>;
    case 3: return launch_stream<XT, 3, GRAD>;
    case 4: return launch_stream<XT, 4, GRAD>;
    case 5: return launch_stream<XT, 5, GRAD>;
    case 6: return launch_stream<XT, 6, GRAD>;
    case 7: return launch_stream<XT, 7, GRAD>;
    case 8: return launch_stream<XT, 8, GRAD>;
  }
  return nullptr;
}

template <bool GRAD>
StreamLaunch pick_stream_pairs_f64(int kc) {  // fp64 X, pairs layout (even kc)
  switch (kc) {
    case 2: return launch_stream<double, 2, GRAD, 1>;
    case 4: return launch_stream<double, 4, GRAD, 1>;
    case 6: return launch_stream<double, 6, GRAD, 1>;
    case 8: return launch_stream<double, 8, GRAD, 1>;
  }
  return nullptr;
}

template <bool GRAD>
StreamLaunch pick_stream_pairs(int kc, int pairs) {  // fp32-X, pairs layouts (even kc)
  if (pairs == 2) {
    if (kc == 2) return launch_stream<float, 2, GRAD, 2>;
    if (kc == 4) return launch_stream<float, 4, GRAD, 2>;
    return nullptr;
  }
  if (pairs == 3) {
    if (kc == 2) return launch_stream<float, 2, GRAD, 3>;
    if (kc == 4) return launch_stream<float, 4, GRAD, 3>;
    return nullptr;
  }
  switch (kc) {
    case 2: return launch_stream<float, 2, GRAD, 1>;
    case 4: return launch_stream<float, 4, GRAD, 1>;
    case 6: return launch_stream<float, 6, GRAD, 1>;
    case 8: return launch_stream<float, 8, GRAD, 1>;
  }
  return nullptr;
}

StreamLaunch pick_stream_any(int xtype, int kc, bool grad, int pairs) {
  if (xtype == PM_X_F64 && pairs) return grad ? pick_stream_pairs_f64<true>(kc) : pick_stream_pairs_f64<false>(kc);
  if (xtype == PM_X_F64) return grad ? pick_stream<double, true>(kc) : pick_stream<double, false>(kc);
  if (pairs) return grad ? pick_stream_pairs<true>(kc, pairs) : pick_stream_pairs<false>(kc, pairs);
  return grad ? pick_stream<float, true>(kc) : pick_stream<float, false>(kc);
}

// 15 consumer warps (512 threads, <= 128 registers) with half-height register sub-tiles:
// twice the warps to hide the latency chains of the compute-bound fp32-X variant.
constexpr int kNCW15 = 15;
template <typename XT, int KC, bool GRAD, int PAIRS>
cudaError_t launch_stream15(const GlmArgs& a, const double* beta, int grid, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  constexpr int R = !GRAD ? 16 : (KC <= 2 ? 16 : 8);
  auto kern = glm_stream_kernel<XT, KC, GRAD, kNCW15, R, kTileRows, PAIRS>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), attr);
  if (e != cudaSuccess) return e;
  BetaPack<KC> bp;
  for (int k = 0; k < 32 * KC; ++k) bp.v[k] = (k < a.K) ? beta[k] : 0.0;
  kern<<<grid, (kNCW15 + 1) * 32, smem, st>>>(a, bp);
  return cudaGetLastError();
}

StreamLaunch pick_stream15(int kc, bool grad, int pairs) {  // fp32-X only
  if (pairs == 3) {
    if (kc == 2) return grad ? launch_stream15<float, 2, true, 3> : launch_stream15<float, 2, false, 3>;
    if (kc == 4) return grad ? launch_stream15<float, 4, true, 3> : launch_stream15<float, 4, false, 3>;
    return nullptr;
  }
  if (pairs) {
    if (kc == 2) return grad ? launch_stream15<float, 2, true, 1> : launch_stream15<float, 2, false, 1>;
    if (kc == 4) return grad ? launch_stream15<float, 4, true, 1> : launch_stream15<float, 4, false, 1>;
    return nullptr;
  }
  switch (kc) {
    case 1: return grad ? launch_stream15<float, 1, true, 0> : launch_stream15<float, 1, false, 0>;
    case 2: return grad ? launch_stream15<float, 2, true, 0> : launch_stream15<float, 2, false, 0>;
    case 3: return grad ? launch_stream15<float, 3, true, 0> : launch_stream15<float, 3, false, 0>;
    case 4: return grad ? launch_stream15<float, 4, true, 0> : launch_stream15<float, 4, false, 0>;
  }
  return nullptr;
}

// fp32-X row-dot consumer with a PAIR of warps per tile (consume_tile_rowdot2): 14 consumer
// warps = 7 pairs, 480 threads, <= 136 registers.
constexpr int kNCW14 = 14;
template <bool GRAD>
cudaError_t launch_stream14(const GlmArgs& a, const double* beta, int grid, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto kern = glm_stream_kernel<float, 4, GRAD, kNCW14, 8, kTileRows, 4>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), attr);
  if (e != cudaSuccess) return e;
  BetaPack<4> bp;
  for (int k = 0; k < 128; ++k) bp.v[k] = (k < a.K) ? beta[k] : 0.0;
  kern<<<grid, (kNCW14 + 1) * 32, smem, st>>>(a, bp);
  return cudaGetLastError();
}

template <typename XT, bool GRAD>
cudaError_t launch_wide(const GlmArgs& a, int grid, int threads, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto kern = glm_wide_kernel<XT, GRAD>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), attr);
  if (e != cudaSuccess) return e;
  kern<<<grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

// ---- small-K row-per-lane kernel (fp64, even K <= 32) -----------------------------
using RowsLaunch = cudaError_t (*)(const GlmArgs&, const double*, int, size_t, int, int, cudaStream_t);

template <int KMAX, bool GRAD, int NCW>
cudaError_t launch_rows_n(const GlmArgs& a, const double* beta, int grid, size_t smem, int tps, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto kern = glm_rows_kernel<KMAX, GRAD, NCW>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), attr);
  if (e != cudaSuccess) return e;
  BetaPack<1> bp;
  for (int k = 0; k < 32; ++k) bp.v[k] = (k < a.K) ? beta[k] : 0.0;
  kern<<<grid, (NCW + 1) * 32, smem, st>>>(a, bp, tps);
  return cudaGetLastError();
}

// ncw = consumer warps: 15 (512 threads, <= 128 registers) for K <= 16, where the per-row
// transcendental chain rather than HBM bounds the kernel, else 7
template <int KMAX, bool GRAD>
cudaError_t launch_rows(const GlmArgs& a, const double* beta, int grid, size_t smem, int tps, int ncw,
                        cudaStream_t st) {
  if constexpr (KMAX <= 16) {
    if (ncw == 15) return launch_rows_n<KMAX, GRAD, 15>(a, beta, grid, smem, tps, st);
  }
  return launch_rows_n<KMAX, GRAD, kNCW>(a, beta, grid, smem, tps, st);
}

template <bool GRAD>
RowsLaunch pick_rows(int K) {
  switch (K) {  // exact even K: the row loops and the swizzle are compile-time
    case 2: return launch_rows<2, GRAD>;
    case 4: return launch_rows<4, GRAD>;
    case 6: return launch_rows<6, GRAD>;
    case 8: return launch_rows<8, GRAD>;
    case 10: return launch_rows<10, GRAD>;
    case 12: return launch_rows<12, GRAD>;
    case 14: return launch_rows<14, GRAD>;
    case 16: return launch_rows<16, GRAD>;
    case 18: return launch_rows<18, GRAD>;
    case 20: return launch_rows<20, GRAD>;
    case 22: return launch_rows<22, GRAD>;
    case 24: return launch_rows<24, GRAD>;
    case 26: return launch_rows<26, GRAD>;
    case 28: return launch_rows<28, GRAD>;
    case 30: return launch_rows<30, GRAD>;
    case 32: return launch_rows<32, GRAD>;
  }
  return nullptr;
}

int choose_geometry(pm_glm_s* h) {
  const int xs = (h->xtype == PM_X_F64) ? 8 : 4;
  const int kc = (h->K + 31) / 32;
  const int budget = std::min(max_optin_smem(h->device), 232448) - 1024;
  h->kind = KIND_NONE;
  h->pairs = 0;
  h->selfprod = 0;
  h->tps = 1;
  const int t_rows = tune("glm_rows", -1);
  // row-per-lane kernel: fp64, even K <= 30, and enough tiles to fill the machine (measured on
  // B200, tools/ab_rows_k.py: 1.3-2x faster than the column kernel at N = 1e7 for K <= 30; at
  // K = 32 and at N ~ 1e5 the column kernel is as fast or faster).  tune glm_rows=0/1 forces.
  const bool rows_forced = t_rows == 1;
  const bool rows_ok = h->xtype == PM_X_F64 && h->K % 2 == 0 && h->K <= 32;
  if (rows_ok && t_rows != 0 &&
      (rows_forced || (h->K <= 30 && h->n_tiles >= int64_t(32) * h->sms))) {
    // 7 consumer warps (15 measured slower at every K); stages of ~8 KB (TPS tiles per bulk
    // copy: the single producer thread's per-copy cost bounds small-K shapes otherwise)
    const int ncw = (tune("rows_ncw", kNCW) == 15 && h->K <= 16) ? 15 : kNCW;
    // measured (tools/ab_rows_tps.py, profiles/r01_ab_rows_tps.txt): 1 tile per copy halves
    // the throughput; >= 4 tiles reach the HBM bound for K >= 12.  Prefer 2 stages per warp
    // with >= 4 tiles each, else 1 stage per warp with as many tiles (<= 16) as fit.
    const int t_tps = tune("rows_tps", -1);
    auto fits = [&](int stages, int t) { return stream_smem_bytes(h->K, 8, stages * t, ncw) <= size_t(budget); };
    int tps = 16;
    while (tps > 1 && !fits(2 * ncw, tps)) --tps;
    if (tps < 4) {
      tps = 16;
      while (tps > 1 && !fits(ncw, tps)) --tps;
    }
    if (t_tps > 0) tps = std::min(16, t_tps);
    while (tps > 1 && !fits(ncw, tps)) --tps;
    int S = 4 * ncw;
    while (S > ncw && stream_smem_bytes(h->K, 8, S * tps, ncw) > size_t(budget)) S -= ncw;
    if (stream_smem_bytes(h->K, 8, S * tps, ncw) <= size_t(budget)) {
      h->kind = KIND_ROWS;
      h->stages = S;
      h->tps = tps;
      h->ncw = ncw;
      h->threads = (ncw + 1) * 32;
      h->smem = stream_smem_bytes(h->K, 8, S * tps, ncw);
      h->grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->sms, h->n_tiles));
      return PM_OK;
    }
  }
  if (kc <= kMaxKC) {
    // fp32-X, even K with an even register count: the pairs consumer layout
    // (consume_tile_pairs; tune f32_pairs=0 disables for A/B)
    // 1 = sub-tile pairs (default; +5.5 % over columns at c1f32), 2 = whole-tile consumer
    // (KC 2 or 4, 7 warps; measured 11 % slower than pairs at K=100: the re-read stage is held
    // for the whole tile and 2 stages per warp expose the refill latency), 0 = columns
    // default (-1): the row-dot consumer where it applies (below), else sub-tile pairs
    const int pmode_t = tune("f32_pairs", -1);
    const bool rowdot_ok = h->xtype == PM_X_F32 && h->K % 4 == 0 && (h->K / 4) % 2 == 1 && (kc == 2 || kc == 4);
    const int pmode = pmode_t >= 0 ? pmode_t : (rowdot_ok ? 3 : 1);
    int pairs = 0;
    if (h->xtype == PM_X_F32 && h->K % 2 == 0 && kc % 2 == 0 && pmode > 0) pairs = (pmode == 2 && kc <= 4) ? 2 : 1;
    // 3 = row-dot consumer (consume_tile_rowdot): K % 4 == 0 with K/4 odd (conflict-free
    // 16-byte row loads), KC 2 or 4; 15 (+1) consumer warps, or 7 (+1) with tune stream_ncw=7.
    // c1f32: 1406 evals/s vs 1272 with the sub-tile pairs consumer (profiles/r02_ab_f32_rowdot.txt)
    if (pmode == 3 && rowdot_ok) pairs = 3;
    // 4 = row-dot consumer, two warps per tile (consume_tile_rowdot2): KC == 4 only
    if (h->xtype == PM_X_F32 && pmode == 4 && h->K % 4 == 0 && (h->K / 4) % 2 == 1 && kc == 4) pairs = 4;
    // fp64 X: the same pairs layout with 16-byte loads (tune f64_pairs=0 disables for A/B)
    if (h->xtype == PM_X_F64 && h->K % 2 == 0 && kc % 2 == 0 && tune("f64_pairs", 1) != 0) pairs = 1;
    // Tiles per stage U (one bulk copy each), column-per-lane consumers only: a 32-row tile of
    // a narrow design is small (8 KB at K = 32 fp64) and the single producer thread's ~200 ns
    // per copy then bounds the pipeline, so stages of ~24 KB hold U consecutive tiles of a
    // contiguous per-CTA tile range (tune stream_tps=1 restores single interleaved tiles).
    const size_t tile_b = size_t(kTileRows) * h->K * xs;
    int U = int(std::min<size_t>(8, std::max<size_t>(1, (24 * 1024) / tile_b)));
    const int t_u = tune("stream_tps", -1);
    if (t_u >= 1) U = std::min(t_u, 16);
    // at least two units per consumer warp, so a warp computes on one while the next lands
    // (config 0, 22 tiles per CTA: U = 1 / 2 / 3 / 4 -> 19.2 / 19.8 / 20.6 / 21.4 us cold and
    // 16.5 / 15.8 / 15.5 / 16.1 us warm; N = 1e6: 70.1 / 58.1 / 58.5 / 64.6 us cold)
    const int64_t per_cta = (h->n_tiles + h->sms - 1) / std::max(1, h->sms);
    U = int(std::max<int64_t>(1, std::min<int64_t>(U, (per_cta + 2 * kNCW - 1) / (2 * kNCW))));
    if (pairs != 0) U = 1;
    const int tr = U * kTileRows;
    const size_t fixed = stream_smem_bytes(h->K, xs, 0, kNCW, tr);
    const size_t per_stage = stream_smem_bytes(h->K, xs, 1, 0, tr) - stream_smem_bytes(h->K, xs, 0, 0, tr);
    int S = int((budget - (long)fixed) / (long)per_stage);
    S = std::min(S, kMaxStages);
    if (S >= 1) S -= S % std::min(S, kNCW);  // each stage owned by one consumer warp
    if (S >= 2) {
      h->kind = KIND_STREAM;
      h->stages = S;
      h->tps = U;
      h->pairs = pairs;
      h->threads = kStreamThreads;
      h->ncw = kNCW;
      h->smem = stream_smem_bytes(h->K, xs, S, kNCW, tr);
      h->grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->sms, h->n_tiles));
    }
    // fp32-X, K <= 128: 15 consumer warps, one 32-row stage each (tune stream_ncw=7 disables;
    // measured: 16-row stages, 2 per warp, are 26 % slower -- per-stage overheads dominate)
    // (the pairs consumer runs 7 warps: its two unrolled sub-tiles need the registers)
    if (h->kind == KIND_STREAM && h->xtype == PM_X_F32 && kc <= 4 &&
        ((h->pairs == 0 || h->pairs == 3) && tune("stream_ncw", 15) != 7)) {
      const size_t fixed15 = stream_smem_bytes(h->K, xs, 0, kNCW15);
      const size_t per_stage1 = stream_smem_bytes(h->K, xs, 1, 0) - stream_smem_bytes(h->K, xs, 0, 0);
      int S15 = int((budget - (long)fixed15) / (long)per_stage1);
      S15 -= S15 % kNCW15;
      if (S15 >= kNCW15) {
        h->stages = std::min(S15, 2 * kNCW15);
        h->tps = 1;  // single interleaved tiles
        h->ncw = kNCW15;
        h->threads = (kNCW15 + 1) * 32;
        h->smem = stream_smem_bytes(h->K, xs, h->stages, kNCW15);
      }
    }
  }
#ifdef PM_AB_STREAM_SELFPROD
  if (h->kind == KIND_STREAM && h->pairs == 0 && h->ncw == kNCW && tune("stream_selfprod", 0) != 0) {
    // column consumers: all 8 warps consume and issue their own bulk copies (no producer
    // thread); stages a multiple of 8
    const int nw = kNCW + 1, tr = h->tps * kTileRows;
    int S = std::min(kMaxStages, 2 * nw);
    while (S > nw && stream_smem_bytes(h->K, xs, S, nw, tr) > size_t(budget)) S -= nw;
    if (stream_smem_bytes(h->K, xs, S, nw, tr) <= size_t(budget)) {
      h->selfprod = 3;
      h->stages = S;
      h->smem = stream_smem_bytes(h->K, xs, S, nw, tr);
    }
  }
#endif
  if (h->kind == KIND_STREAM && h->pairs == 3) {
    // row-dot consumer: self-producing consumer warps (tune f32_selfprod: 0 = producer thread,
    // 1 = consumer warps issue their own copies, 3 (default) = and warp 0 consumes as well:
    // ncw + 1 consumer warps with one stage each, or two when they fit)
    h->selfprod = tune("f32_selfprod", 3);
    if (h->selfprod == 3) {
      const int nw = h->ncw + 1;
      int S = 2 * nw;
      if (stream_smem_bytes(h->K, xs, S, nw) > size_t(budget)) S = nw;
      if (stream_smem_bytes(h->K, xs, S, nw) <= size_t(budget)) {
        h->stages = S;
        h->smem = stream_smem_bytes(h->K, xs, S, nw);
      } else {
        h->selfprod = 1;
      }
    }
  }
  if (h->kind == KIND_STREAM && h->pairs == 4) {
    // 7 warp pairs, two stages each when they fit (else one)
    int S14 = 14;
    if (stream_smem_bytes(h->K, xs, S14, kNCW14) > size_t(budget)) S14 = 7;
    if (stream_smem_bytes(h->K, xs, S14, kNCW14) <= size_t(budget)) {
      h->stages = S14;
      h->tps = 1;
      h->ncw = kNCW14;
      h->threads = (kNCW14 + 1) * 32;
      h->smem = stream_smem_bytes(h->K, xs, S14, kNCW14);
    } else {
      h->pairs = 1;  // does not fit: the sub-tile pairs consumer
    }
  }
  if (h->kind == KIND_NONE) {
    int nw = kWideThreads / 32;
    while (nw > 1 && stream_smem_bytes(h->K, xs, 0, nw) > (size_t)budget) --nw;
    if (stream_smem_bytes(h->K, xs, 0, nw) > (size_t)budget)
      return fail(PM_EINVAL, "n_cols too large for the device (K=" + std::to_string(h->K) + ")");
    h->kind = KIND_WIDE;
    h->stages = 0;
    h->threads = nw * 32;
    h->smem = stream_smem_bytes(h->K, xs, 0, nw);
    const int64_t warps_needed = (h->n_rows + 0);
    const int64_t blocks = (warps_needed + nw - 1) / nw;
    h->grid = (int)std::max<int64_t>(1, std::min<int64_t>(int64_t(h->sms) * 2, blocks));
  }
  return PM_OK;
}

GlmArgs make_args(pm_glm_s* h, bool with_prior, double* out) {
  GlmArgs a;
  a.X = h->X;
  a.y = h->y;
  a.n_rows = h->n_rows;
  a.n_tiles = h->n_tiles;
  a.K = h->K;
  a.stages = h->stages;
  a.tps = h->kind == KIND_STREAM ? h->tps : 1;
  a.selfprod = h->kind == KIND_STREAM ? h->selfprod : 0;
  a.with_prior = with_prior ? 1 : 0;
  a.evict_first = 1;
  a.prior_mu = h->prior_mu;
  a.prior_sigma = h->prior_sigma;
  a.prior_terms = h->prior_terms;
  a.partials = h->partials;
  a.counter = h->counter;
  a.out = out;
  a.beta_dev = h->beta_dev;
  a.xw = 0;  // no peer exchange (pm_glm_eval_xchg sets these)
  a.xrank = 0;
  a.xphase = 3;
  a.xepoch = 0;
  for (int p = 0; p < kMaxXchgRanks; ++p) a.xpeer[p] = nullptr;
  a.xstatus = nullptr;
  a.done = nullptr;
  a.done_seq = 0;
#ifdef PM_AB_PHASES
  static unsigned long long* stamps = nullptr;
  if (!stamps) {
    cudaMalloc(&stamps, sizeof(unsigned long long) * 8 * 4096);
    cudaMemset(stamps, 0, sizeof(unsigned long long) * 8 * 4096);
  }
  a.stamps = stamps;
#endif
  return a;
}

int check_beta(pm_glm_s* h, const double* beta) {
  if (!beta) return fail(PM_EINVAL, "beta is null");
  if (!all_finite(beta, h->K)) return fail(PM_EINVAL, "beta contains non-finite entries");
  return PM_OK;
}

// enqueue one evaluation writing (f, g) to `out` on stream `st` (caller holds the mutex)
struct XchgLaunch {  // peer exchange fields of one evaluation (pm_glm_eval_xchg)
  int world = 0, rank = 0, phase = 3;
  unsigned long long epoch = 0;
  double* peer[kMaxXchgRanks] = {};
  unsigned* status = nullptr;
};

int enqueue_eval(pm_glm_s* h, const double* beta, bool with_prior, bool grad, double* out, cudaStream_t st,
                 const XchgLaunch* xl = nullptr, unsigned long long done_seq = 0) {
  GlmArgs a = make_args(h, with_prior, out);
  if (done_seq) {  // results go to the handle's mapped buffer: completion word right after them
    a.done = reinterpret_cast<unsigned long long*>(h->out_dev + h->K + 1);
    a.done_seq = done_seq;
  }
  if (xl) {
    a.xw = xl->world;
    a.xrank = xl->rank;
    a.xphase = xl->phase;
    a.xepoch = xl->epoch;
    for (int p = 0; p < kMaxXchgRanks; ++p) a.xpeer[p] = xl->peer[p];
    a.xstatus = xl->status;
  }
  cudaError_t e;
  // the fp32-X stream kernel widens X by integer ops to x * 2^-896 and scales beta by 2^896
  // (glm_kernels.cuh ld_x_scaled); a beta that large would overflow, so it takes the wide
  // kernel (plain conversions) instead -- same results, slower, never hit by real chains
  bool wide_fallback = false;
  if (h->kind == KIND_STREAM && h->xtype == PM_X_F32) {
    for (int k = 0; k < h->K; ++k) wide_fallback |= !(std::fabs(beta[k]) < 0x1p100);
  }
  if (h->kind == KIND_STREAM && !wide_fallback) {
    StreamLaunch fn = h->ncw == kNCW14 ? (grad ? launch_stream14<true> : launch_stream14<false>)
                      : h->ncw == kNCW15 ? pick_stream15((h->K + 31) / 32, grad, h->pairs)
                                         : pick_stream_any(h->xtype, (h->K + 31) / 32, grad, h->pairs);
    e = fn(a, beta, h->grid, h->smem, st);
  } else if (h->kind == KIND_ROWS) {
    RowsLaunch fn = grad ? pick_rows<true>(h->K) : pick_rows<false>(h->K);
    e = fn(a, beta, h->grid, h->smem, h->tps, h->ncw, st);
  } else {
    int grid = h->grid, threads = h->threads;
    size_t smem = h->smem;
    if (wide_fallback) {
      const int nw = kWideThreads / 32;
      grid = (int)std::max<int64_t>(1, std::min<int64_t>(int64_t(h->sms) * 2, (h->n_rows + nw - 1) / nw));
      threads = nw * 32;
      smem = stream_smem_bytes(h->K, 4, 0, nw);  // K <= 256 here: always fits
    }
    std::memcpy(h->beta_pinned, beta, sizeof(double) * h->K);
    e = cudaMemcpyAsync(h->beta_dev, h->beta_pinned, sizeof(double) * h->K, cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      if (h->xtype == PM_X_F64)
        e = grad ? launch_wide<double, true>(a, grid, threads, smem, st)
                 : launch_wide<double, false>(a, grid, threads, smem, st);
      else
        e = grad ? launch_wide<float, true>(a, grid, threads, smem, st)
                 : launch_wide<float, false>(a, grid, threads, smem, st);
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "glm kernel launch");
  return PM_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int pm_glm_create(int device, pm_glm_t* out) {
  if (!out) return fail(PM_EINVAL, "pm_glm_create: null output");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(PM_ERANGE, "device index out of range");
  pm_glm_s* h = new pm_glm_s();
  h->device = device;
  DeviceGuard g(device);
  h->sms = sm_count(device);
  e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMalloc(&h->counter, sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(h->counter, 0, sizeof(unsigned int));
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(e, "pm_glm_create");
  }
  *out = h;
  return PM_OK;
}

int pm_glm_destroy(pm_glm_t h) {
  if (!h) return PM_OK;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard g(h->device);
    cudaStreamSynchronize(h->stream);
    free_glm_data(h);
    if (h->counter) cudaFree(h->counter);
    if (h->ev_a) cudaEventDestroy(h->ev_a);
    if (h->ev_b) cudaEventDestroy(h->ev_b);
    if (h->stream) cudaStreamDestroy(h->stream);
  }
  delete h;
  return PM_OK;
}

int pm_glm_upload(pm_glm_t h, const void* X, int x_dtype, const double* y, int64_t n_rows, int32_t n_cols) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (!X || !y) return fail(PM_EINVAL, "X and y must be non-null");
  if (n_rows < 1 || n_cols < 1)
    return fail(PM_EINVAL, "need N >= 1 and K >= 1, got shape (" + std::to_string(n_rows) + ", " +
                               std::to_string(n_cols) + ")");
  if (x_dtype != PM_X_F64 && x_dtype != PM_X_F32) return fail(PM_EINVAL, "x_dtype must be PM_X_F64 or PM_X_F32");
  for (int64_t i = 0; i < n_rows; ++i)
    if (!(y[i] == 0.0 || y[i] == 1.0)) return fail(PM_EINVAL, "y entries must be exactly 0 or 1");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  cudaStreamSynchronize(h->stream);
  free_glm_data(h);
  h->xtype = x_dtype;
  h->n_rows = n_rows;
  h->K = n_cols;
  h->n_pad = (n_rows + kTileRows - 1) / kTileRows * kTileRows;
  h->n_tiles = h->n_pad / kTileRows;
  const size_t xs = (x_dtype == PM_X_F64) ? 8 : 4;
  const size_t xbytes = size_t(h->n_pad) * n_cols * xs;
  const size_t real_bytes = size_t(n_rows) * n_cols * xs;
  PM_CUDA(cudaMalloc(&h->X, xbytes));
  PM_CUDA(cudaMalloc(&h->y, sizeof(double) * h->n_pad));
  PM_CUDA(cudaMemsetAsync(static_cast<char*>(h->X) + real_bytes, 0, xbytes - real_bytes, h->stream));
  PM_CUDA(cudaMemsetAsync(h->y + n_rows, 0, sizeof(double) * (h->n_pad - n_rows), h->stream));
  PM_CUDA(cudaMemcpyAsync(h->y, y, sizeof(double) * n_rows, cudaMemcpyHostToDevice, h->stream));
  unsigned long long* bad = nullptr;
  PM_CUDA(cudaMalloc(&bad, sizeof(unsigned long long)));
  PM_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), h->stream));
  if (x_dtype == PM_X_F64) {
    PM_CUDA(cudaMemcpyAsync(h->X, X, real_bytes, cudaMemcpyHostToDevice, h->stream));
    count_nonfinite<double><<<h->sms * 4, 256, 0, h->stream>>>(static_cast<const double*>(h->X),
                                                               int64_t(n_rows) * n_cols, bad);
  } else {
    // X arrives as float (the caller rounded the reference's float64 X, glm.py:88)
    PM_CUDA(cudaMemcpyAsync(h->X, X, real_bytes, cudaMemcpyHostToDevice, h->stream));
    count_nonfinite<float><<<h->sms * 4, 256, 0, h->stream>>>(static_cast<const float*>(h->X),
                                                              int64_t(n_rows) * n_cols, bad);
  }
  unsigned long long nbad = 0;
  PM_CUDA(cudaMemcpyAsync(&nbad, bad, sizeof(nbad), cudaMemcpyDeviceToHost, h->stream));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  cudaFree(bad);
  if (nbad) {
    free_glm_data(h);
    return fail(PM_EINVAL, "x contains non-finite entries");
  }
  int rc = choose_geometry(h);
  if (rc != PM_OK) {
    free_glm_data(h);
    return rc;
  }
  h->partials_cap = std::max(std::max(h->grid, 1), 2 * h->sms);  // the fp32 wide fallback uses 2 x SMs
  PM_CUDA(cudaMalloc(&h->partials, sizeof(double) * size_t(h->partials_cap) * (n_cols + 1)));
  PM_CUDA(cudaMalloc(&h->beta_dev, sizeof(double) * (n_cols + 1)));  // +1: PM_AB_OUT_DEVICE scratch
  PM_CUDA(cudaHostAlloc(&h->out_host, sizeof(double) * (n_cols + 2), cudaHostAllocMapped | cudaHostAllocPortable));
  std::memset(h->out_host, 0, sizeof(double) * (n_cols + 2));
  h->seq = 0;
  PM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->out_dev), h->out_host, 0));
  PM_CUDA(cudaHostAlloc(&h->beta_pinned, sizeof(double) * n_cols, cudaHostAllocPortable));
  return PM_OK;
}

int pm_glm_set_prior(pm_glm_t h, const double* mu, const double* sigma) {
  if (!h) return fail(PM_EINVAL, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  if (h->K == 0) return fail(PM_ESTATE, "upload data before setting the prior");
  if (!mu && !sigma) {
    h->has_prior = false;
    return PM_OK;
  }
  if (!mu || !sigma) return fail(PM_EINVAL, "mu and sigma must both be given");
  for (int k = 0; k < h->K; ++k) {
    if (!std::isfinite(mu[k]) || !std::isfinite(sigma[k])) return fail(PM_EINVAL, "prior must be finite");
    if (!(sigma[k] > 0)) return fail(PM_EINVAL, "all prior sigmas must be > 0");
  }
  cudaStreamSynchronize(h->stream);
  if (!h->prior_mu) PM_CUDA(cudaMalloc(&h->prior_mu, sizeof(double) * h->K));
  if (!h->prior_sigma) PM_CUDA(cudaMalloc(&h->prior_sigma, sizeof(double) * h->K));
  if (!h->prior_terms) PM_CUDA(cudaMalloc(&h->prior_terms, sizeof(double) * (h->K + 1)));
  PM_CUDA(cudaMemcpy(h->prior_mu, mu, sizeof(double) * h->K, cudaMemcpyHostToDevice));
  PM_CUDA(cudaMemcpy(h->prior_sigma, sigma, sizeof(double) * h->K, cudaMemcpyHostToDevice));
  h->has_prior = true;
  return PM_OK;
}

}  // extern "C"

namespace {
// launch / wait bodies; the caller holds h->mu.  pm_glm_eval holds it across both so two
// threads sharing a handle cannot interleave (one's (f, g) read out of the other's launch).
int glm_launch_locked(pm_glm_s* h, const double* beta, int with_prior, int want_grad) {
  if (h->K == 0) return fail(PM_ESTATE, "no data uploaded");
  if (h->launched) return fail(PM_ESTATE, "an evaluation is already in flight (pm_glm_wait first)");
  if (with_prior && !h->has_prior) return fail(PM_ESTATE, "with_prior set but no prior configured");
  int rc = check_beta(h, beta);
  if (rc) return rc;
  DeviceGuard g(h->device);
  rc = enqueue_eval(h, beta, with_prior != 0, want_grad != 0, h->out_dev, h->stream, nullptr, ++h->seq);
  if (rc) return rc;
  h->launched = true;
  h->last_want_grad = want_grad;
  return PM_OK;
}

int glm_wait_locked(pm_glm_s* h, double* f_out, double* g_out) {
  if (!h->launched) return fail(PM_ESTATE, "pm_glm_wait without a launch");
  DeviceGuard g(h->device);
  h->launched = false;
  // The finishing CTA stores (f, g), then the launch's sequence number (system-scope release)
  // into the mapped buffer: poll that word instead of cudaStreamSynchronize -- the results
  // are readable a few microseconds before the driver reports the stream idle (kernel
  // teardown + completion processing).  The stream is queried now and then so that a failed
  // launch ends the wait; tune glm_poll=0 restores the synchronise.
  bool seen = false;
  if (tune("glm_poll", 1) != 0) {
    volatile unsigned long long* word = reinterpret_cast<volatile unsigned long long*>(h->out_host + h->K + 1);
    for (unsigned spins = 1;; ++spins) {
      if (*word == h->seq) {
        seen = true;
        break;
      }
      if ((spins & 0x3ff) == 0 && cudaStreamQuery(h->stream) != cudaErrorNotReady) break;
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  }
  if (!seen) PM_CUDA(cudaStreamSynchronize(h->stream));
  if (f_out) *f_out = h->out_host[0];
  if (g_out && h->last_want_grad) std::memcpy(g_out, h->out_host + 1, sizeof(double) * h->K);
  return PM_OK;
}
}  // namespace

extern "C" {

int pm_glm_launch(pm_glm_t h, const double* beta, int with_prior, int want_grad) {
  if (!h) return fail(PM_EINVAL, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  return glm_launch_locked(h, beta, with_prior, want_grad);
}

int pm_glm_wait(pm_glm_t h, double* f_out, double* g_out) {
  if (!h) return fail(PM_EINVAL, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  return glm_wait_locked(h, f_out, g_out);
}

int pm_glm_eval(pm_glm_t h, const double* beta, int with_prior, int want_grad, double* f_out, double* g_out) {
  if (!h) return fail(PM_EINVAL, "null handle");
  std::lock_guard<std::mutex> lk(h->mu);
  int rc = glm_launch_locked(h, beta, with_prior, want_grad);
  if (rc) return rc;
  return glm_wait_locked(h, f_out, g_out);
}

// ---- peer-memory exchange of row-sharded ranks (replaces NCCL all-gather + fold) ----
struct pm_xchg_s {
  int device = 0, world = 0, rank = 0, width = 0;
  char* mailbox = nullptr;          // local, cudaMalloc'd, IPC-exported
  double* peer[kMaxXchgRanks] = {};  // every rank's mailbox in this process (self = mailbox)
  bool opened[kMaxXchgRanks] = {};   // IPC mappings to close
  unsigned* status = nullptr;       // device u32: 1 after a wait timeout
  unsigned long long epoch = 0;
  bool half_open = false;           // split form: a phase-1 launch awaits its phase-2 launch
  std::mutex mu;
};

int pm_xchg_create(int device, int32_t world, int32_t rank, int32_t width, pm_xchg_t* out) {
  if (!out) return fail(PM_EINVAL, "null output");
  if (world < 1 || world > kMaxXchgRanks) return fail(PM_EINVAL, "world must be in 1..16");
  if (rank < 0 || rank >= world) return fail(PM_ERANGE, "rank out of range");
  if (width < 1) return fail(PM_EINVAL, "width must be >= 1");
  DeviceGuard g(device);
  pm_xchg_s* x = new pm_xchg_s();
  x->device = device;
  x->world = world;
  x->rank = rank;
  x->width = width;
  const size_t bytes = xchg_bytes(world, width);
  cudaError_t e = cudaMalloc(&x->mailbox, bytes);
  if (e == cudaSuccess) e = cudaMemset(x->mailbox, 0, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&x->status, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(x->status, 0, sizeof(unsigned));
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    if (x->mailbox) cudaFree(x->mailbox);
    if (x->status) cudaFree(x->status);
    delete x;
    return cuda_fail(e, "pm_xchg_create");
  }
  x->peer[rank] = reinterpret_cast<double*>(x->mailbox);
  *out = x;
  return PM_OK;
}

int pm_xchg_ipc_handle(pm_xchg_t x, void* handle_out) {
  if (!x || !handle_out) return fail(PM_EINVAL, "null argument");
  DeviceGuard g(x->device);
  cudaIpcMemHandle_t hd;
  PM_CUDA(cudaIpcGetMemHandle(&hd, x->mailbox));
  std::memcpy(handle_out, &hd, sizeof(hd));
  return PM_OK;
}

int pm_xchg_open_peer(pm_xchg_t x, int32_t peer, const void* handle) {
  if (!x || !handle) return fail(PM_EINVAL, "null argument");
  if (peer < 0 || peer >= x->world) return fail(PM_ERANGE, "peer out of range");
  if (peer == x->rank) return PM_OK;
  std::lock_guard<std::mutex> lk(x->mu);
  if (x->opened[peer]) return fail(PM_ESTATE, "peer already opened");
  DeviceGuard g(x->device);
  cudaIpcMemHandle_t hd;
  std::memcpy(&hd, handle, sizeof(hd));
  void* p = nullptr;
  PM_CUDA(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
  x->peer[peer] = static_cast<double*>(p);
  x->opened[peer] = true;
  return PM_OK;
}

int pm_xchg_mailbox(pm_xchg_t x, void** ptr) {
  if (!x || !ptr) return fail(PM_EINVAL, "null argument");
  *ptr = x->mailbox;
  return PM_OK;
}

int pm_xchg_set_peer_ptr(pm_xchg_t x, int32_t peer, void* mailbox) {
  if (!x || !mailbox) return fail(PM_EINVAL, "null argument");
  if (peer < 0 || peer >= x->world) return fail(PM_ERANGE, "peer out of range");
  std::lock_guard<std::mutex> lk(x->mu);
  if (x->opened[peer]) return fail(PM_ESTATE, "peer was opened through IPC");
  x->peer[peer] = static_cast<double*>(mailbox);
  return PM_OK;
}

int pm_xchg_status(pm_xchg_t x, int32_t* timed_out) {
  if (!x || !timed_out) return fail(PM_EINVAL, "null argument");
  DeviceGuard g(x->device);
  unsigned v = 0;
  PM_CUDA(cudaMemcpy(&v, x->status, sizeof(v), cudaMemcpyDeviceToHost));
  *timed_out = int(v);
  return PM_OK;
}

int pm_xchg_destroy(pm_xchg_t x) {
  if (!x) return PM_OK;
  {
    DeviceGuard g(x->device);
    cudaDeviceSynchronize();
    for (int p = 0; p < x->world; ++p)
      if (x->opened[p]) cudaIpcCloseMemHandle(x->peer[p]);
    if (x->mailbox) cudaFree(x->mailbox);
    if (x->status) cudaFree(x->status);
  }
  delete x;
  return PM_OK;
}

int pm_glm_eval_xchg_phase(pm_glm_t h, const double* beta, int with_prior, pm_xchg_t x, int phase, double* dev_out,
                           void* stream) {
  if (!h || !x) return fail(PM_EINVAL, "null handle");
  if (!dev_out && phase != 1) return fail(PM_EINVAL, "dev_out is null");
  if (phase < 1 || phase > 3) return fail(PM_EINVAL, "phase must be 1, 2 or 3");
  std::lock_guard<std::mutex> lk(h->mu);
  std::lock_guard<std::mutex> lx(x->mu);
  if (h->K == 0) return fail(PM_ESTATE, "no data uploaded");
  if (x->width != h->K + 1) return fail(PM_EINVAL, "exchange width must be n_cols + 1");
  if (x->device != h->device) return fail(PM_EINVAL, "exchange and design on different devices");
  for (int p = 0; p < x->world; ++p)
    if (!x->peer[p]) return fail(PM_ESTATE, "peer mailbox not opened (pm_xchg_open_peer)");
  if ((phase == 2) != x->half_open)
    return fail(PM_ESTATE, phase == 2 ? "phase 2 without a phase-1 launch" : "phase-1 launch awaits its phase 2");
  int rc = check_beta(h, beta);
  if (rc) return rc;
  if (with_prior && !h->has_prior) return fail(PM_ESTATE, "no prior set (pm_glm_set_prior)");
  DeviceGuard g(h->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
  if (st != h->stream) {
    PM_CUDA(cudaEventRecord(h->ev_a, h->stream));
    PM_CUDA(cudaStreamWaitEvent(st, h->ev_a, 0));
  }
  XchgLaunch xl;
  xl.world = x->world;
  xl.rank = x->rank;
  xl.phase = phase;
  xl.epoch = phase == 2 ? x->epoch : x->epoch + 1;  // phase 2 folds the epoch phase 1 deposited
  for (int p = 0; p < x->world; ++p) xl.peer[p] = x->peer[p];
  xl.status = x->status;
  rc = enqueue_eval(h, beta, with_prior != 0, true, dev_out, st, &xl);
  if (rc) return rc;
  x->epoch = xl.epoch;
  x->half_open = phase == 1;
  if (st != h->stream) {
    PM_CUDA(cudaEventRecord(h->ev_b, st));
    PM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_b, 0));
  }
  return PM_OK;
}

int pm_glm_eval_xchg(pm_glm_t h, const double* beta, int with_prior, pm_xchg_t x, double* dev_out, void* stream) {
  return pm_glm_eval_xchg_phase(h, beta, with_prior, x, 3, dev_out, stream);
}

int pm_glm_eval_device(pm_glm_t h, const double* beta, int with_prior, int want_grad, double* dev_out,
                       void* stream) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (!dev_out) return fail(PM_EINVAL, "dev_out is null");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->K == 0) return fail(PM_ESTATE, "no data uploaded");
  int rc = check_beta(h, beta);
  if (rc) return rc;
  if (with_prior && !h->has_prior) return fail(PM_ESTATE, "no prior set (pm_glm_set_prior)");
  DeviceGuard g(h->device);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
  if (st != h->stream) {  // order against earlier work on the handle (shared scratch)
    PM_CUDA(cudaEventRecord(h->ev_a, h->stream));
    PM_CUDA(cudaStreamWaitEvent(st, h->ev_a, 0));
  }
  rc = enqueue_eval(h, beta, with_prior != 0, want_grad != 0, dev_out, st);
  if (rc) return rc;
  if (st != h->stream) {
    PM_CUDA(cudaEventRecord(h->ev_b, st));
    PM_CUDA(cudaStreamWaitEvent(h->stream, h->ev_b, 0));
  }
  return PM_OK;
}

}  // extern "C"

namespace {
__global__ void fold_rows_kernel(const double* __restrict__ in, int world, int width, double* __restrict__ out) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < width; c += gridDim.x * blockDim.x) {
    double acc = in[c];
    for (int r = 1; r < world; ++r) acc += in[size_t(r) * width + c];
    out[c] = acc;
  }
}
}  // namespace

extern "C" {

int pm_fold_rows(const double* in_dev, int32_t world, int32_t width, double* out_dev, void* stream) {
  if (!in_dev || !out_dev) return fail(PM_EINVAL, "null argument");
  if (world < 1 || width < 1) return fail(PM_EINVAL, "need world >= 1 and width >= 1");
  const int threads = 128;
  const int blocks = std::min(1024, (width + threads - 1) / threads);
  fold_rows_kernel<<<blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(in_dev, world, width, out_dev);
  PM_CUDA(cudaGetLastError());
  return PM_OK;
}

int pm_glm_time_launches(pm_glm_t h, const double* betas, int32_t n, int with_prior, int want_grad,
                         float* total_ms) {
  if (!h || !betas || !total_ms) return fail(PM_EINVAL, "null argument");
  if (n < 1) return fail(PM_EINVAL, "n must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->K == 0) return fail(PM_ESTATE, "no data uploaded");
  if (with_prior && !h->has_prior) return fail(PM_ESTATE, "with_prior set but no prior configured");
  for (int i = 0; i < n; ++i) {
    int rc = check_beta(h, betas + size_t(i) * h->K);
    if (rc) return rc;
  }
  DeviceGuard g(h->device);
  cudaEvent_t e0, e1;
  PM_CUDA(cudaEventCreate(&e0));
  PM_CUDA(cudaEventCreate(&e1));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  PM_CUDA(cudaEventRecord(e0, h->stream));
#ifdef PM_AB_OUT_DEVICE  // A/B timing experiment only: results to device memory, not mapped host memory
  double* out_t = h->beta_dev;  // K doubles; the A/B build only times, never reads it
#else
  double* out_t = h->out_dev;
#endif
  for (int i = 0; i < n; ++i) {
    int rc = enqueue_eval(h, betas + size_t(i) * h->K, with_prior != 0, want_grad != 0, out_t, h->stream);
    if (rc) return rc;
  }
  PM_CUDA(cudaEventRecord(e1, h->stream));
  PM_CUDA(cudaEventSynchronize(e1));
  PM_CUDA(cudaEventElapsedTime(total_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  h->last_want_grad = want_grad;
#ifdef PM_AB_PHASES
  {  // phases of the LAST launch, ns relative to the first CTA's entry
    GlmArgs a = make_args(h, false, nullptr);
    const int G = h->grid;
    std::vector<unsigned long long> st(size_t(G) * 8);
    cudaMemcpy(st.data(), a.stamps, sizeof(unsigned long long) * st.size(), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, e_max = 0, p_max = 0, s_min = ~0ull, s_max = 0, k_max = 0, f_last = 0, c5 = 0, c6 = 0;
    for (int b = 0; b < G; ++b) {
      const unsigned long long* s = &st[size_t(b) * 8];
      t0 = std::min(t0, s[0]);
      e_max = std::max(e_max, s[0]);
      p_max = std::max(p_max, s[1]);
      s_min = std::min(s_min, s[2]);
      s_max = std::max(s_max, s[2]);
      k_max = std::max(k_max, s[3]);
      f_last = std::max(f_last, s[4]);
      c5 = std::max(c5, s[5]);
      c6 = std::max(c6, s[6]);
    }
    std::fprintf(stderr,
                 "[phases] grid %d: entry spread %.2f us, prologue done %.2f, stream done first %.2f last %.2f, "
                 "tickets done %.2f, chunk sums %.2f, totals %.2f, finish done %.2f (event %.2f us per launch)\n",
                 G, (e_max - t0) * 1e-3, (p_max - t0) * 1e-3, (s_min - t0) * 1e-3, (s_max - t0) * 1e-3,
                 (k_max - t0) * 1e-3, (c5 - t0) * 1e-3, (c6 - t0) * 1e-3, (f_last - t0) * 1e-3, *total_ms * 1e3 / n);
    cudaMemset(a.stamps, 0, sizeof(unsigned long long) * st.size());
  }
#endif
  return PM_OK;
}

int pm_glm_time_cold(pm_glm_t h, const double* betas, int32_t n, int with_prior, int want_grad,
                     float* total_ms) {
  if (!h || !betas || !total_ms) return fail(PM_EINVAL, "null argument");
  if (n < 1) return fail(PM_EINVAL, "n must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->K == 0) return fail(PM_ESTATE, "no data uploaded");
  if (with_prior && !h->has_prior) return fail(PM_ESTATE, "with_prior set but no prior configured");
  for (int i = 0; i < n; ++i) {
    int rc = check_beta(h, betas + size_t(i) * h->K);
    if (rc) return rc;
  }
  DeviceGuard g(h->device);
  std::vector<cudaEvent_t> ev(2 * size_t(n), nullptr);
  for (auto& e : ev) PM_CUDA(cudaEventCreate(&e));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  // per launch: scrub L2 on the SAME stream, then events around the launch alone -- the GPU
  // goes straight from the scrub to the evaluation, so the interval is device time with cold
  // inputs, not the host's launch latency
  for (int i = 0; i < n; ++i) {
    PM_CUDA(l2_scrub(h->device, h->stream));
    PM_CUDA(cudaEventRecord(ev[2 * i], h->stream));
    int rc = enqueue_eval(h, betas + size_t(i) * h->K, with_prior != 0, want_grad != 0, h->out_dev, h->stream);
    if (rc) return rc;
    PM_CUDA(cudaEventRecord(ev[2 * i + 1], h->stream));
  }
  PM_CUDA(cudaStreamSynchronize(h->stream));
  float tot = 0.f;
  for (int i = 0; i < n; ++i) {
    float ms = 0.f;
    PM_CUDA(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
    tot += ms;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  *total_ms = tot;
  h->last_want_grad = want_grad;
  return PM_OK;
}

int pm_glm_stream(pm_glm_t h, void** stream) {
  if (!h || !stream) return fail(PM_EINVAL, "null argument");
  *stream = h->stream;
  return PM_OK;
}

int pm_glm_geometry(pm_glm_t h, int* grid, int* threads, int* stages, size_t* smem_bytes, int* kernel_kind) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (grid) *grid = h->grid;
  if (threads) *threads = h->threads;
  if (stages) *stages = h->stages;
  if (smem_bytes) *smem_bytes = h->smem;
  if (kernel_kind) *kernel_kind = h->kind;
  return PM_OK;
}

}  // extern "C"

// ====================================================================== workspace
struct pm_ws_s {
  pm_glm_s* h = nullptr;
  double* xbeta = nullptr;
  double* xt = nullptr;
  double* tmp = nullptr;
  double* beta_dev = nullptr;
  double* partials = nullptr;
  unsigned int* counter = nullptr;
  unsigned long long* maxbits = nullptr;
  double* out_host = nullptr;
  double* out_dev = nullptr;
  unsigned long long seq = 0;  // differential evaluations launched (completion word value)
  int grid = 0;
  std::mutex mu;
};

namespace {

template <int M>
cudaError_t launch_diff(const DiffArgs& a, const DeltaPack& dp, int grid, cudaStream_t st) {
  diff_eval_kernel<M><<<grid, 256, 0, st>>>(a, dp);
  return cudaGetLastError();
}

void free_ws(pm_ws_s* w) {
  if (w->xbeta) cudaFree(w->xbeta);  // w->xt is the handle's shared transposed copy
  if (w->tmp) cudaFree(w->tmp);
  if (w->beta_dev) cudaFree(w->beta_dev);
  if (w->partials) cudaFree(w->partials);
  if (w->counter) cudaFree(w->counter);
  if (w->maxbits) cudaFree(w->maxbits);
  if (w->out_host) cudaFreeHost(w->out_host);
}

cudaError_t launch_xbeta(pm_glm_s* h, const double* beta_dev, double* out) {
  const int grid = std::max(1, std::min(h->sms * 8, int((h->n_rows * 32 + 255) / 256)));
  if (h->xtype == PM_X_F64)
    xbeta_kernel<double><<<grid, 256, 0, h->stream>>>(static_cast<const double*>(h->X), beta_dev, h->K, h->n_rows,
                                                      out);
  else
    xbeta_kernel<float><<<grid, 256, 0, h->stream>>>(static_cast<const float*>(h->X), beta_dev, h->K, h->n_rows, out);
  return cudaGetLastError();
}

}  // namespace

extern "C" {

int pm_ws_create(pm_glm_t h, const double* beta0, pm_ws_t* out) {
  if (!h || !out) return fail(PM_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->K == 0) return fail(PM_ESTATE, "no data uploaded");
  int rc = check_beta(h, beta0);
  if (rc) return rc;
  DeviceGuard g(h->device);
  pm_ws_s* w = new pm_ws_s();
  w->h = h;
  const int64_t n = h->n_rows, np = h->n_pad;
  const int K = h->K;
  cudaError_t e = cudaSuccess;
  auto chk = [&](cudaError_t x) {
    if (e == cudaSuccess) e = x;
  };
  chk(cudaMalloc(&w->xbeta, sizeof(double) * np));
  chk(cudaMalloc(&w->tmp, sizeof(double) * np));
  // X^T (GlmWorkspace.xt, glm.py:473) depends only on the immutable design: built once per
  // handle and shared read-only by all of its workspaces (repeat chains skip the transpose)
  const bool build_xt = h->xt_cache == nullptr;
  if (build_xt) chk(cudaMalloc(&h->xt_cache, sizeof(double) * size_t(K) * np));
  w->xt = h->xt_cache;
  chk(cudaMalloc(&w->beta_dev, sizeof(double) * K));
  w->grid = (int)std::max<int64_t>(1, std::min<int64_t>(int64_t(h->sms) * 4, (n + 255) / 256));
  chk(cudaMalloc(&w->partials, sizeof(double) * size_t(w->grid) * kMaxDeltas));
  chk(cudaMalloc(&w->counter, sizeof(unsigned int)));
  chk(cudaMalloc(&w->maxbits, sizeof(unsigned long long)));
  chk(cudaHostAlloc(&w->out_host, sizeof(double) * (kMaxDeltas + 1), cudaHostAllocMapped | cudaHostAllocPortable));
  if (w->out_host) std::memset(w->out_host, 0, sizeof(double) * (kMaxDeltas + 1));
  if (e != cudaSuccess) {
    free_ws(w);
    delete w;
    return cuda_fail(e, "pm_ws_create alloc");
  }
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&w->out_dev), w->out_host, 0);
  chk(cudaMemsetAsync(w->counter, 0, sizeof(unsigned int), h->stream));
  chk(cudaMemsetAsync(w->xbeta, 0, sizeof(double) * np, h->stream));
  chk(cudaMemcpyAsync(w->beta_dev, beta0, sizeof(double) * K, cudaMemcpyHostToDevice, h->stream));
  chk(launch_xbeta(h, w->beta_dev, w->xbeta));
  dim3 tg(unsigned((n + 31) / 32), unsigned((K + 31) / 32));
  if (build_xt && e == cudaSuccess) {
    chk(cudaMemsetAsync(h->xt_cache, 0, sizeof(double) * size_t(K) * np, h->stream));  // padding rows
    if (h->xtype == PM_X_F64)
      transpose_kernel<double><<<tg, 256, 0, h->stream>>>(static_cast<const double*>(h->X), n, K, w->xt, np);
    else
      transpose_kernel<float><<<tg, 256, 0, h->stream>>>(static_cast<const float*>(h->X), n, K, w->xt, np);
  }
  chk(cudaGetLastError());
  chk(cudaStreamSynchronize(h->stream));
  if (e != cudaSuccess) {
    free_ws(w);
    delete w;
    return cuda_fail(e, "pm_ws_create init");
  }
  *out = w;
  return PM_OK;
}

int pm_ws_destroy(pm_ws_t w) {
  if (!w) return PM_OK;
  {
    std::lock_guard<std::mutex> lk(w->h->mu);
    DeviceGuard g(w->h->device);
    cudaStreamSynchronize(w->h->stream);
    free_ws(w);
  }
  delete w;
  return PM_OK;
}

int pm_ws_diff_eval(pm_ws_t w, int32_t k, const double* deltas, int32_t n_deltas, double* f_out) {
  if (!w || !deltas || !f_out) return fail(PM_EINVAL, "null argument");
  pm_glm_s* h = w->h;
  if (k < 0 || k >= h->K)
    return fail(PM_ERANGE, "coordinate " + std::to_string(k) + " out of range [0, " + std::to_string(h->K) + ")");
  if (n_deltas < 1 || n_deltas > kMaxDeltas)
    return fail(PM_EINVAL, "n_deltas must be in [1, " + std::to_string(kMaxDeltas) + "]");
  if (!all_finite(deltas, n_deltas)) return fail(PM_EINVAL, "delta_beta_k must be finite");
  std::lock_guard<std::mutex> lk(w->mu);
  std::lock_guard<std::mutex> lk2(h->mu);
  DeviceGuard g(h->device);
  DiffArgs a;
  a.xbeta = w->xbeta;
  a.xk = w->xt + size_t(k) * h->n_pad;
  a.y = h->y;
  a.n = h->n_rows;
  a.partials = w->partials;
  a.counter = w->counter;
  a.out = w->out_dev;
  a.done = reinterpret_cast<unsigned long long*>(w->out_dev + kMaxDeltas);
  a.done_seq = ++w->seq;
  DeltaPack dp;
  for (int m = 0; m < kMaxDeltas; ++m) dp.d[m] = m < n_deltas ? deltas[m] : 0.0;
  cudaError_t e;
  if (n_deltas == 1) e = launch_diff<1>(a, dp, w->grid, h->stream);
  else if (n_deltas == 2) e = launch_diff<2>(a, dp, w->grid, h->stream);
  else if (n_deltas <= 4) e = launch_diff<4>(a, dp, w->grid, h->stream);
  else if (n_deltas <= 8) e = launch_diff<8>(a, dp, w->grid, h->stream);
  else e = launch_diff<16>(a, dp, w->grid, h->stream);
  if (e != cudaSuccess) return cuda_fail(e, "diff_eval launch");
  // completion: poll the word the finishing CTA stores after the results (as pm_glm_wait)
  bool seen = false;
  if (tune("glm_poll", 1) != 0) {
    volatile unsigned long long* word = reinterpret_cast<volatile unsigned long long*>(w->out_host + kMaxDeltas);
    for (unsigned spins = 1;; ++spins) {
      if (*word == w->seq) {
        seen = true;
        break;
      }
      if ((spins & 0x3ff) == 0 && cudaStreamQuery(h->stream) != cudaErrorNotReady) break;
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  }
  if (!seen) PM_CUDA(cudaStreamSynchronize(h->stream));
  std::memcpy(f_out, w->out_host, sizeof(double) * n_deltas);
  return PM_OK;
}

int pm_ws_commit(pm_ws_t w, int32_t k, double delta) {
  if (!w) return fail(PM_EINVAL, "null workspace");
  pm_glm_s* h = w->h;
  if (k < 0 || k >= h->K)
    return fail(PM_ERANGE, "coordinate " + std::to_string(k) + " out of range [0, " + std::to_string(h->K) + ")");
  if (!std::isfinite(delta)) return fail(PM_EINVAL, "delta_beta_k must be finite");
  if (delta == 0.0) return PM_OK;  // glm.py:536
  std::lock_guard<std::mutex> lk(w->mu);
  std::lock_guard<std::mutex> lk2(h->mu);
  DeviceGuard g(h->device);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(int64_t(h->sms) * 4, (h->n_rows + 255) / 256));
  commit_kernel<<<grid, 256, 0, h->stream>>>(w->xbeta, w->xt + size_t(k) * h->n_pad, delta, h->n_rows);
  PM_CUDA(cudaGetLastError());
  return PM_OK;
}

int pm_ws_internal_view(pm_ws_t w, pm_ws_view* v) {
  if (!w || !v) return fail(PM_EINVAL, "null argument");
  pm_glm_s* h = w->h;
  v->xbeta = w->xbeta;
  v->xt = w->xt;
  v->y = h->y;
  v->n = h->n_rows;
  v->ld = h->n_pad;
  v->K = h->K;
  v->device = h->device;
  v->sms = h->sms;
  v->stream = h->stream;
  return PM_OK;
}

int pm_ws_internal_lock(pm_ws_t w, int lock) {
  if (lock) {
    w->mu.lock();
    w->h->mu.lock();
  } else {
    w->h->mu.unlock();
    w->mu.unlock();
  }
  return PM_OK;
}

int pm_ws_read_xbeta(pm_ws_t w, double* out) {
  if (!w || !out) return fail(PM_EINVAL, "null argument");
  pm_glm_s* h = w->h;
  std::lock_guard<std::mutex> lk(w->mu);
  std::lock_guard<std::mutex> lk2(h->mu);
  DeviceGuard g(h->device);
  PM_CUDA(cudaMemcpyAsync(out, w->xbeta, sizeof(double) * h->n_rows, cudaMemcpyDeviceToHost, h->stream));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  return PM_OK;
}

int pm_ws_validate(pm_ws_t w, const double* beta_current, double* max_abs_err) {
  if (!w || !beta_current || !max_abs_err) return fail(PM_EINVAL, "null argument");
  pm_glm_s* h = w->h;
  std::lock_guard<std::mutex> lk(w->mu);
  std::lock_guard<std::mutex> lk2(h->mu);
  DeviceGuard g(h->device);
  PM_CUDA(cudaMemcpyAsync(w->beta_dev, beta_current, sizeof(double) * h->K, cudaMemcpyHostToDevice, h->stream));
  PM_CUDA(launch_xbeta(h, w->beta_dev, w->tmp));
  PM_CUDA(cudaMemsetAsync(w->maxbits, 0, sizeof(unsigned long long), h->stream));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(int64_t(h->sms) * 4, (h->n_rows + 255) / 256));
  maxabs_diff_kernel<<<grid, 256, 0, h->stream>>>(w->xbeta, w->tmp, h->n_rows, w->maxbits);
  PM_CUDA(cudaGetLastError());
  unsigned long long bits = 0;
  PM_CUDA(cudaMemcpyAsync(&bits, w->maxbits, sizeof(bits), cudaMemcpyDeviceToHost, h->stream));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  double v;
  std::memcpy(&v, &bits, sizeof(v));
  *max_abs_err = v;
  return PM_OK;
}

}  // extern "C"

// ====================================================================== hierarchical
struct pm_hb_s {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  double* X = nullptr;
  double* y = nullptr;
  int64_t* poff = nullptr;
  int64_t* nrows = nullptr;
  int G = 0, K = 0;
  int stages = 0;
  size_t smem = 0;
  double* betas = nullptr;
  double* mu_dev = nullptr;
  double* sigma_dev = nullptr;
  double* out_f = nullptr;
  double* out_g = nullptr;
  double* pin_in = nullptr;    // G*K + 2K (mapped: the kernels can read it in place, tune hb_mapped_in)
  double* pin_in_dev = nullptr;  // device alias of pin_in
  double* pin_out = nullptr;   // G + G*K (mapped)
  double* pin_out_dev = nullptr;  // device alias of pin_out
  // small-K row-per-lane path (even K <= 32): balanced tile ranges + segment fold
  bool rows = false;
  int rows_grid = 0, rows_stages = 0, rows_ncw = 7, rows_tps = 1;
  int rows_contig = 1, rows_fused = 0, rows_pdl = 1;  // PM_HB_CONTIG / _FUSED / PM_PDL = 0 for A/B
  int* cta_g0 = nullptr;        // [rows_grid] first group of each CTA
  unsigned* gcount = nullptr;   // [G] fused-fold tickets
  size_t rows_smem = 0;
  int64_t n_tiles = 0;
  int* seg_base = nullptr;     // [rows_grid + 1]
  int* gseg = nullptr;         // [G + 1]
  double* part = nullptr;      // [nseg][kHbRowsNCW][K+1]
};

namespace {

void free_hb(pm_hb_s* h) {
  for (void* p : {(void*)h->X, (void*)h->y, (void*)h->poff, (void*)h->nrows, (void*)h->betas,
                  (void*)h->out_f, (void*)h->seg_base, (void*)h->gseg,
                  (void*)h->part, (void*)h->cta_g0, (void*)h->gcount})
    if (p) cudaFree(p);
  h->seg_base = h->gseg = h->cta_g0 = nullptr;
  h->gcount = nullptr;
  h->part = nullptr;
  h->rows = false;
  if (h->pin_in) cudaFreeHost(h->pin_in);
  if (h->pin_out) cudaFreeHost(h->pin_out);
  h->X = h->y = nullptr;
  h->poff = h->nrows = nullptr;
  h->betas = h->mu_dev = h->sigma_dev = h->out_f = h->out_g = nullptr;
  h->pin_in = h->pin_out = h->pin_out_dev = nullptr;
  h->G = h->K = 0;
}

using HbLaunch = cudaError_t (*)(const HbArgs&, int, size_t, cudaStream_t);

template <int KC, bool GRAD>
cudaError_t launch_hb(const HbArgs& a, int grid, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto kern = hb_kernel<KC, GRAD, kHbNCW>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), attr);
  if (e != cudaSuccess) return e;
  kern<<<grid, kHbThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int KMAX, bool GRAD, int NCW>
cudaError_t launch_hb_rows_n(const pm_hb_s* h, const HbArgs& a, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};
  auto kern = hb_rows_kernel<KMAX, GRAD, NCW>;
  cudaError_t e = ensure_smem_attr(reinterpret_cast<const void*>(kern), attr);
  if (e != cudaSuccess) return e;
  HbRowsArgs r;
  r.X = a.X;
  r.y = a.y;
  r.poff = a.poff;
  r.nrows = a.nrows;
  r.seg_base = h->seg_base;
  r.G = h->G;
  r.K = h->K;
  r.stages = h->rows_stages;
  r.tps = h->rows_tps;
  r.contig = h->rows_contig;
  r.selfprod = tune("hb_selfprod", 1) != 0 ? 1 : 0;
  r.fused = h->rows_fused;
  r.n_tiles = h->n_tiles;
  r.betas = a.betas;
  r.part = h->part;
  r.cta_g0 = h->cta_g0;
  r.gseg = h->gseg;
  r.gcount = h->gcount;
  r.mu = a.mu;
  r.sigma = a.sigma;
  r.out_f = a.out_f;
  r.out_g = a.out_g;
  if (HbRowsThreads<NCW>::all) r.selfprod = 1;  // no producer warp in that geometry
  e = launch_pdl(h->rows_pdl != 0, kern, dim3(h->rows_grid), dim3(HbRowsThreads<NCW>::value), h->rows_smem, st, r);
  if (e != cudaSuccess || h->rows_fused) return e;
  return launch_pdl(h->rows_pdl != 0, hb_fold_kernel<GRAD>, dim3(h->G), dim3(64), 0, st, (const double*)h->part,
                    (const int*)h->gseg, int(NCW), h->K, a.betas, a.mu, a.sigma, a.out_f, a.out_g);
}

template <int KMAX, bool GRAD>
cudaError_t launch_hb_rows(const pm_hb_s* h, const HbArgs& a, cudaStream_t st) {
  if (h->rows_ncw == 8) return launch_hb_rows_n<KMAX, GRAD, 8>(h, a, st);
  return h->rows_ncw == 7 ? launch_hb_rows_n<KMAX, GRAD, 7>(h, a, st) : launch_hb_rows_n<KMAX, GRAD, 15>(h, a, st);
}

using HbRowsLaunch = cudaError_t (*)(const pm_hb_s*, const HbArgs&, cudaStream_t);

template <bool GRAD>
HbLaunch pick_hb(int kc);

template <bool GRAD>
HbRowsLaunch pick_hb_rows(int K) {
  switch (K) {  // exact even K: the row loops and the swizzle are compile-time
    case 2: return launch_hb_rows<2, GRAD>;
    case 4: return launch_hb_rows<4, GRAD>;
    case 6: return launch_hb_rows<6, GRAD>;
    case 8: return launch_hb_rows<8, GRAD>;
    case 10: return launch_hb_rows<10, GRAD>;
    case 12: return launch_hb_rows<12, GRAD>;
    case 14: return launch_hb_rows<14, GRAD>;
    case 16: return launch_hb_rows<16, GRAD>;
    case 18: return launch_hb_rows<18, GRAD>;
    case 20: return launch_hb_rows<20, GRAD>;
    case 22: return launch_hb_rows<22, GRAD>;
    case 24: return launch_hb_rows<24, GRAD>;
    case 26: return launch_hb_rows<26, GRAD>;
    case 28: return launch_hb_rows<28, GRAD>;
    case 30: return launch_hb_rows<30, GRAD>;
    case 32: return launch_hb_rows<32, GRAD>;
  }
  return nullptr;
}

// one launch of whichever HB path the handle uses
cudaError_t launch_hb_any(const pm_hb_s* h, const HbArgs& a, bool grad) {
  if (h->rows) {
    HbRowsLaunch fn = grad ? pick_hb_rows<true>(h->K) : pick_hb_rows<false>(h->K);
    return fn(h, a, h->stream);
  }
  HbLaunch fn = grad ? pick_hb<true>((h->K + 31) / 32) : pick_hb<false>((h->K + 31) / 32);
  return fn(a, h->G, h->smem, h->stream);
}

template <bool GRAD>
HbLaunch pick_hb(int kc) {
  switch (kc) {
    case 1: return launch_hb<1, GRAD>;
    case 2: return launch_hb<2, GRAD>;
    case 3: return launch_hb<3, GRAD>;
    case 4: return launch_hb<4, GRAD>;
    case 5: return launch_hb<5, GRAD>;
    case 6: return launch_hb<6, GRAD>;
    case 7: return launch_hb<7, GRAD>;
    case 8: return launch_hb<8, GRAD>;
  }
  return nullptr;
}

}  // namespace

extern "C" {

int pm_hb_create(int device, pm_hb_t* out) {
  if (!out) return fail(PM_EINVAL, "null output");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(PM_ERANGE, "device index out of range");
  pm_hb_s* h = new pm_hb_s();
  h->device = device;
  DeviceGuard g(device);
  h->sms = sm_count(device);
  e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete h;
    return cuda_fail(e, "cudaStreamCreate");
  }
  *out = h;
  return PM_OK;
}

int pm_hb_destroy(pm_hb_t h) {
  if (!h) return PM_OK;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard g(h->device);
    cudaStreamSynchronize(h->stream);
    free_hb(h);
    cudaStreamDestroy(h->stream);
  }
  delete h;
  return PM_OK;
}

int pm_hb_upload(pm_hb_t h, const double* X, const double* y, const int64_t* offsets, int32_t G, int32_t K) {
  if (!h || !X || !y || !offsets) return fail(PM_EINVAL, "null argument");
  if (G < 1) return fail(PM_EINVAL, "need at least one group");
  if (K < 1) return fail(PM_EINVAL, "need K >= 1");
  if ((K + 31) / 32 > kMaxKC) return fail(PM_EINVAL, "hierarchical path supports K <= 256");
  if (offsets[0] != 0) return fail(PM_EINVAL, "offsets[0] must be 0");
  for (int g = 0; g < G; ++g)
    if (offsets[g + 1] <= offsets[g]) return fail(PM_EINVAL, "every group needs >= 1 row (group " + std::to_string(g) + ")");
  const int64_t N = offsets[G];
  for (int64_t i = 0; i < N; ++i)
    if (!(y[i] == 0.0 || y[i] == 1.0)) return fail(PM_EINVAL, "y entries must be exactly 0 or 1");
  for (int64_t i = 0; i < N * K; ++i)
    if (!std::isfinite(X[i])) return fail(PM_EINVAL, "x contains non-finite entries");
  std::vector<int64_t> poff(G + 1), nr(G);
  poff[0] = 0;
  for (int g = 0; g < G; ++g) {
    nr[g] = offsets[g + 1] - offsets[g];
    poff[g + 1] = poff[g] + (nr[g] + kTileRows - 1) / kTileRows * kTileRows;
  }
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard gd(h->device);
  cudaStreamSynchronize(h->stream);
  free_hb(h);
  h->G = G;
  h->K = K;
  const int64_t NP = poff[G];
  PM_CUDA(cudaMalloc(&h->X, sizeof(double) * size_t(NP) * K));
  PM_CUDA(cudaMalloc(&h->y, sizeof(double) * NP));
  PM_CUDA(cudaMemsetAsync(h->X, 0, sizeof(double) * size_t(NP) * K, h->stream));
  PM_CUDA(cudaMemsetAsync(h->y, 0, sizeof(double) * NP, h->stream));
  for (int g = 0; g < G; ++g) {
    PM_CUDA(cudaMemcpyAsync(h->X + size_t(poff[g]) * K, X + size_t(offsets[g]) * K, sizeof(double) * nr[g] * K,
                            cudaMemcpyHostToDevice, h->stream));
    PM_CUDA(cudaMemcpyAsync(h->y + poff[g], y + offsets[g], sizeof(double) * nr[g], cudaMemcpyHostToDevice,
                            h->stream));
  }
  PM_CUDA(cudaMalloc(&h->poff, sizeof(int64_t) * (G + 1)));
  PM_CUDA(cudaMalloc(&h->nrows, sizeof(int64_t) * G));
  PM_CUDA(cudaMemcpyAsync(h->poff, poff.data(), sizeof(int64_t) * (G + 1), cudaMemcpyHostToDevice, h->stream));
  PM_CUDA(cudaMemcpyAsync(h->nrows, nr.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, h->stream));
  // betas, mu, sigma contiguous on the device (one H2D copy per evaluation from pin_in)
  PM_CUDA(cudaMalloc(&h->betas, sizeof(double) * (size_t(G) * K + 2 * K)));
  h->mu_dev = h->betas + size_t(G) * K;
  h->sigma_dev = h->mu_dev + K;
  // f then g, contiguous: pm_hb_eval reads both back with one D2H copy
  PM_CUDA(cudaMalloc(&h->out_f, sizeof(double) * (size_t(G) + size_t(G) * K)));
  h->out_g = h->out_f + G;
  PM_CUDA(cudaHostAlloc(&h->pin_in, sizeof(double) * (size_t(G) * K + 2 * K), cudaHostAllocPortable | cudaHostAllocMapped));
  PM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->pin_in_dev), h->pin_in, 0));
  // mapped, so the fold can also write (f, g) straight into host memory (tune hb_mapped_out=1)
  PM_CUDA(cudaHostAlloc(&h->pin_out, sizeof(double) * (size_t(G) + size_t(G) * K),
                        cudaHostAllocPortable | cudaHostAllocMapped));
  PM_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->pin_out_dev), h->pin_out, 0));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  const size_t fixed = stream_smem_bytes(K, 8, 0, kHbNCW);
  const size_t per_stage = stream_smem_bytes(K, 8, 1, 0) - stream_smem_bytes(K, 8, 0, 0);
  int S = kHbMaxStages;
  const size_t cap = 60 * 1024;
  while (S > 2 && fixed + S * per_stage > cap) --S;
  h->stages = S;
  h->smem = stream_smem_bytes(K, 8, S, kHbNCW);
  // small-K path: equal contiguous tile ranges, one CTA per SM
  if (K % 2 == 0 && K <= 32 && tune("hb_rows", 1) != 0) {
    const int C = h->sms;
    const int64_t T = NP / kTileRows;
    auto group_of = [&](int64_t tile) {
      return int(std::upper_bound(poff.begin(), poff.end(), tile * kTileRows) - poff.begin()) - 1;
    };
    std::vector<int> seg_base(C + 1, 0), gseg(G + 1, -1), cta_g0(C, 0);
    int nseg = 0;
    for (int c = 0; c < C; ++c) {
      seg_base[c] = nseg;
      const int64_t t0 = int64_t(c) * T / C, t1 = int64_t(c + 1) * T / C;
      if (t0 >= t1) continue;
      const int gf = group_of(t0), gl = group_of(t1 - 1);
      cta_g0[c] = gf;
      for (int g2 = gf; g2 <= gl; ++g2) {
        if (gseg[g2] < 0) gseg[g2] = nseg;
        ++nseg;
      }
    }
    seg_base[C] = nseg;
    gseg[G] = nseg;
    // consumer warps (7 or 15), tiles per stage, stages (a multiple of the consumer count,
    // at least two per warp when they fit): tune hb_rows_ncw / _tps / _stages for A/B
    // (8: every warp consumes and issues its own bulk copies -- the default; 7 / 15: + a
    // producer warp, which idles under hb_selfprod=1)
    const int t_ncw = tune("hb_rows_ncw", tune("hb_selfprod", 1) != 0 ? 8 : 7);
    const int ncw = t_ncw == 15 ? 15 : (t_ncw == 8 ? 8 : 7);
    int tps = std::max(1, std::min(8, tune("hb_rows_tps", 2)));
    const int t_st = tune("hb_rows_stages", -1);
    const size_t cap = 200 * 1024;
    while (tps > 1 && stream_smem_bytes(K, 8, ncw * tps, ncw) > cap) --tps;
    int Sr = 4 * ncw;
    while (Sr > ncw && stream_smem_bytes(K, 8, Sr * tps, ncw) > cap) Sr -= ncw;
    if (t_st > 0) Sr = std::max(ncw, std::min(Sr, t_st / ncw * ncw));
    PM_CUDA(cudaMalloc(&h->seg_base, sizeof(int) * (C + 1)));
    PM_CUDA(cudaMalloc(&h->gseg, sizeof(int) * (G + 1)));
    PM_CUDA(cudaMalloc(&h->part, sizeof(double) * size_t(nseg) * ncw * (K + 1)));
    PM_CUDA(cudaMemcpy(h->seg_base, seg_base.data(), sizeof(int) * (C + 1), cudaMemcpyHostToDevice));
    PM_CUDA(cudaMemcpy(h->gseg, gseg.data(), sizeof(int) * (G + 1), cudaMemcpyHostToDevice));
    PM_CUDA(cudaMalloc(&h->cta_g0, sizeof(int) * C));
    PM_CUDA(cudaMemcpy(h->cta_g0, cta_g0.data(), sizeof(int) * C, cudaMemcpyHostToDevice));
    PM_CUDA(cudaMalloc(&h->gcount, sizeof(unsigned) * G));
    PM_CUDA(cudaMemset(h->gcount, 0, sizeof(unsigned) * G));
    h->rows_contig = tune("hb_contig", 1) != 0 ? 1 : 0;
    // fold fused into the rows launch (per-group tickets) by default: with the self-producing
    // 8-warp kernel it beats the separate PDL-overlapped fold launch, 61.5 vs 64.4 us
    // (profiles/r02_ab_hb_selfprod.txt); with the r01 producer-thread kernel it was the other
    // way round (68.3 vs 71.2 us, profiles/r01_ab_hb_pdl.txt).  tune hb_fused=0 separates it.
    h->rows_fused = tune("hb_fused", 1) == 1 ? 1 : 0;
    h->rows_pdl = tune("pdl", 1) != 0 ? 1 : 0;
    h->rows = true;
    h->rows_grid = C;
    h->rows_ncw = ncw;
    h->rows_tps = tps;
    h->rows_stages = Sr;
    h->rows_smem = stream_smem_bytes(K, 8, Sr * tps, ncw);
    h->n_tiles = T;
  }
  return PM_OK;
}

}  // extern "C"

// validate, stage betas/prior on the device and build the kernel arguments (mutex held)
static int hb_stage(pm_hb_t h, const double* betas, const double* mu, const double* sigma, HbArgs& a) {
  if (h->G == 0) return fail(PM_ESTATE, "no data uploaded");
  const int G = h->G, K = h->K;
  const bool prior = mu != nullptr;
  if (prior != (sigma != nullptr)) return fail(PM_EINVAL, "mu and sigma must both be given");
  if (prior) {
    for (int k = 0; k < K; ++k)
      if (!(sigma[k] > 0) || !std::isfinite(mu[k]) || !std::isfinite(sigma[k]))
        return fail(PM_EINVAL, "prior must be finite with sigma > 0");
  }
  // staged and validated in one pass (a rejected call leaves stale staging bytes, nothing else)
  if (!copy_check_finite(h->pin_in, betas, int64_t(G) * K)) return fail(PM_EINVAL, "betas contain non-finite entries");
  if (prior) {
    std::memcpy(h->pin_in + size_t(G) * K, mu, sizeof(double) * K);
    std::memcpy(h->pin_in + size_t(G) * K + K, sigma, sizeof(double) * K);
  }
  // hb_mapped_in=1 (A/B): no H2D copy -- the kernels read betas / mu / sigma in place from the
  // mapped staging buffer (one 8K-byte read per warp and group over PCIe instead of a DMA
  // before the launch); default: one copy, betas then mu and sigma (contiguous on both sides)
  const bool mapped_in = tune("hb_mapped_in", 0) == 1;
  if (!mapped_in)
    PM_CUDA(cudaMemcpyAsync(h->betas, h->pin_in, sizeof(double) * (size_t(G) * K + (prior ? 2 * K : 0)),
                            cudaMemcpyHostToDevice, h->stream));
  a.X = h->X;
  a.y = h->y;
  a.poff = h->poff;
  a.nrows = h->nrows;
  a.K = K;
  a.stages = h->stages;
  const double* src = mapped_in ? h->pin_in_dev : h->betas;
  a.betas = src;
  a.mu = prior ? src + size_t(G) * K : nullptr;
  a.sigma = prior ? src + size_t(G) * K + K : nullptr;
  a.out_f = h->out_f;
  a.out_g = h->out_g;
  return PM_OK;
}

extern "C" {

int pm_hb_eval(pm_hb_t h, const double* betas, const double* mu, const double* sigma, int want_grad, double* f_out,
               double* g_out) {
  if (!h || !betas || !f_out) return fail(PM_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard gd(h->device);
  HbArgs a;
  int rc = hb_stage(h, betas, mu, sigma, a);
  if (rc) return rc;
  const int G = h->G, K = h->K;
  const bool grad = want_grad != 0 && g_out != nullptr;
  // default (hb_mapped_out=1): the fold's stores go straight into mapped host memory;
  // hb_mapped_out=0: the fold writes (f, g) to device memory and one DMA brings them back
  // (168 KB at config 3).  Re-measured in r02 after the host path was trimmed: 110.1 vs 117.1 us
  // per call end to end (profiles/r02_ab_hb_selfprod.txt); in r01 the copy had won.
  const bool mapped = tune("hb_mapped_out", 1) == 1;
  if (mapped) {
    a.out_f = h->pin_out_dev;
    a.out_g = h->pin_out_dev + G;
  }
  cudaError_t e = launch_hb_any(h, a, grad);
  if (e != cudaSuccess) return cuda_fail(e, "hb kernel launch");
  if (!mapped)
    PM_CUDA(cudaMemcpyAsync(h->pin_out, h->out_f, sizeof(double) * (size_t(G) + (grad ? size_t(G) * K : 0)),
                            cudaMemcpyDeviceToHost, h->stream));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  std::memcpy(f_out, h->pin_out, sizeof(double) * G);
  if (grad) std::memcpy(g_out, h->pin_out + G, sizeof(double) * size_t(G) * K);
  return PM_OK;
}

int pm_hb_stream(pm_hb_t h, void** stream) {
  if (!h || !stream) return fail(PM_EINVAL, "null argument");
  *stream = h->stream;
  return PM_OK;
}

int pm_hb_time_evals(pm_hb_t h, const double* betas, const double* mu, const double* sigma, int want_grad,
                     int32_t n, float* total_ms) {
  if (!h || !betas || !total_ms) return fail(PM_EINVAL, "null argument");
  if (n < 1) return fail(PM_EINVAL, "n must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard gd(h->device);
  HbArgs a;
  int rc = hb_stage(h, betas, mu, sigma, a);
  if (rc) return rc;
  cudaEvent_t e0, e1;
  PM_CUDA(cudaEventCreate(&e0));
  PM_CUDA(cudaEventCreate(&e1));
  PM_CUDA(cudaEventRecord(e0, h->stream));
  for (int i = 0; i < n; ++i) {
    cudaError_t e = launch_hb_any(h, a, want_grad != 0);
    if (e != cudaSuccess) return cuda_fail(e, "hb kernel launch");
  }
  PM_CUDA(cudaEventRecord(e1, h->stream));
  PM_CUDA(cudaEventSynchronize(e1));
  PM_CUDA(cudaEventElapsedTime(total_ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return PM_OK;
}

}  // extern "C"
