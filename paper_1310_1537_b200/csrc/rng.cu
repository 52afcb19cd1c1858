// Batch deviate generation on the device: the reference's buffered
// streams and its Gamma / Dirichlet samplers (rng.py:42-56, 59-138, 165-215).
//
// Stream contract (rng.py:1-19): a (seed, owner) stream is numpy's Philox4x64-10; uniform
// i is word i%4 of block counter i/4+1, (w >> 11) * 2^-53 (philox.cuh).  Standard normals
// are Box-Muller on consecutive uniform pairs: normal j comes from pair p = j/2 (uniforms
// 2p, 2p+1, always in Philox block p/2), r cos(theta) for even j, r sin(theta) for odd j
// (rng.py:47-56, carry logic 91-102).  Every deviate is therefore a pure function of its
// stream index, and one thread per Philox block fills any index range.
//
// Gamma / Dirichlet (rng.py:165-215) consume the two streams sequentially with
// rejection.  Two device forms:
//   * pm_rng_gamma_streams / pm_rng_dirichlet_streams: S independent (uniform, normal)
//     stream pairs -- the reference's concurrency model (owner spawn keys, rng.py:7-9) --
//     one thread each, running the reference's exact control flow.
//   * pm_rng_gamma / pm_rng_dirichlet on ONE stream pair with a homogeneous shape >= 1
//     (no U^(1/alpha) boost, so every attempt costs exactly one normal and, when
//     1 + c x > 0, one uniform): attempt i's uniform index is the number of valid
//     attempts before it (an exclusive scan), its acceptance is then a pure function of
//     i, and draw k is the k-th accepted attempt (a second scan).  Three parallel passes
//     replace the sequential loop and consume exactly the same deviates.  Other shapes
//     run the sequential form on one thread.
// Arithmetic follows the reference's Python evaluation order with explicit _rn
// intrinsics (no FMA contraction); transcendental functions are CUDA's (log, log1p,
// sincos, pow: <= 2 ulp), so normals and draws match numpy to rounding, not bitwise.

#include <cub/device/device_scan.cuh>
#include <math.h>

#include <vector>

#include "philox.cuh"
#include "pm_internal.cuh"

namespace {

using pm::U64x4;

constexpr int kGammaMaxReject = 10000;  // _GAMMA_MAX_REJECT (rng.py:160)
constexpr double kTwoPi = 6.283185307179586;  // 2.0 * np.pi (rng.py:52)

__device__ __forceinline__ double u53(uint64_t w) { return double(w >> 11) * 0x1.0p-53; }

__device__ __forceinline__ U64x4 philox_block(uint64_t b, uint64_t k0, uint64_t k1) {
  U64x4 c;
  c.v[0] = b + 1;
  c.v[1] = 0;
  c.v[2] = 0;
  c.v[3] = 0;
  return pm::philox4x64_10(c, k0, k1);
}

// r cos / r sin of one uniform pair (rng.py:50-55): 1-u in (0,1] keeps log finite.
__device__ __forceinline__ void box_muller(double u0, double u1, double& zc, double& zs) {
  const double r = sqrt(__dmul_rn(-2.0, log1p(-u0)));
  const double th = __dmul_rn(kTwoPi, u1);
  double s, c;
  sincos(th, &s, &c);
  zc = __dmul_rn(r, c);
  zs = __dmul_rn(r, s);
}

// Sequential cursor over a uniform stream (one Philox block cached).
struct UCursor {
  uint64_t k0, k1, idx, blk;
  U64x4 w;
  bool have;
  __device__ void init(uint64_t a, uint64_t b, uint64_t pos) {
    k0 = a;
    k1 = b;
    idx = pos;
    have = false;
  }
  __device__ double next() {
    const uint64_t b = idx >> 2;
    if (!have || b != blk) {
      w = philox_block(b, k0, k1);
      blk = b;
      have = true;
    }
    const double u = u53(w.v[idx & 3]);
    ++idx;
    return u;
  }
};

// Sequential cursor over a normal stream (one pair cached).
struct NCursor {
  uint64_t k0, k1, idx, pair;
  double z0, z1;
  bool have;
  __device__ void init(uint64_t a, uint64_t b, uint64_t pos) {
    k0 = a;
    k1 = b;
    idx = pos;
    have = false;
  }
  __device__ double next() {
    const uint64_t p = idx >> 1;
    if (!have || p != pair) {
      const U64x4 w = philox_block(p >> 1, k0, k1);
      const int o = int(p & 1) * 2;
      box_muller(u53(w.v[o]), u53(w.v[o + 1]), z0, z1);
      pair = p;
      have = true;
    }
    const double z = (idx & 1) ? z1 : z0;
    ++idx;
    return z;
  }
};

// Per-shape constants computed on the host in Python's order (rng.py:165-166, 184-188).
struct Shape {
  double d, c;      // for the Marsaglia-Tsang core (shape alpha or alpha+1)
  double inv;       // 1/alpha when boosted
  int boost;        // alpha < 1
};

Shape make_shape(double alpha) {
  Shape s;
  s.boost = alpha < 1.0;
  const double a = s.boost ? alpha + 1.0 : alpha;
  s.d = a - 1.0 / 3.0;
  s.c = 1.0 / sqrt(9.0 * s.d);
  s.inv = s.boost ? 1.0 / alpha : 1.0;
  return s;
}

// _gamma_std (rng.py:163-178); returns false when the rejection loop drains.
__device__ bool gamma_std(const Shape& sh, UCursor& U, NCursor& N, double& out) {
  for (int r = 0; r < kGammaMaxReject; ++r) {
    const double x = N.next();
    double v = __dadd_rn(1.0, __dmul_rn(sh.c, x));
    if (v <= 0.0) continue;
    v = __dmul_rn(__dmul_rn(v, v), v);
    const double u = U.next();
    const double x2 = __dmul_rn(x, x);
    if (u < __dsub_rn(1.0, __dmul_rn(__dmul_rn(0.0331, x2), x2))) {
      out = __dmul_rn(sh.d, v);
      return true;
    }
    if (log(u) < __dadd_rn(__dmul_rn(0.5, x2), __dmul_rn(sh.d, __dadd_rn(__dsub_rn(1.0, v), log(v))))) {
      out = __dmul_rn(sh.d, v);
      return true;
    }
  }
  return false;
}

// _gamma_shape (rng.py:181-188)
__device__ bool gamma_shape(const Shape& sh, UCursor& U, NCursor& N, double& out) {
  double y;
  if (!gamma_std(sh, U, N, y)) return false;
  if (sh.boost) {
    const double u = U.next();
    y = __dmul_rn(y, pow(u, sh.inv));
  }
  out = y;
  return true;
}

// numpy's pairwise summation of a contiguous float64 vector (np.sum / ndarray.sum):
// n < 8 plain loop from 0.0; n <= 128 eight interleaved partial sums combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) plus the tail; above, split at n/2 rounded down to
// a multiple of 8 and recurse.
__device__ double pairwise_block(const double* a, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

__device__ double pairwise_sum(const double* a, int n) {
  if (n <= 128) return pairwise_block(a, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pairwise_sum(a, n2), pairwise_sum(a + n2, n - n2));
}

// ---------------------------------------------------------------- fill
__global__ void fill_kernel(int kind, uint64_t k0, uint64_t k1, uint64_t pos, int64_t n, double* out) {
  const uint64_t b0 = pos >> 2, b1 = (pos + uint64_t(n) - 1) >> 2;
  const uint64_t nb = b1 - b0 + 1;
  for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nb; t += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t b = b0 + t;
    const U64x4 w = philox_block(b, k0, k1);
    double v[4];
    if (kind == PM_RNG_KIND_UNIFORM01) {
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = u53(w.v[q]);
    } else {
      box_muller(u53(w.v[0]), u53(w.v[1]), v[0], v[1]);
      box_muller(u53(w.v[2]), u53(w.v[3]), v[2], v[3]);
    }
    const uint64_t first = b * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t i = first + q;
      if (i >= pos && i < pos + uint64_t(n)) out[i - pos] = v[q];
    }
  }
}

// ---------------------------------------------------------------- independent streams
struct StreamArgs {
  const uint64_t* ukeys;  // [S][2]
  const uint64_t* nkeys;
  uint64_t* upos;         // [S] in/out
  uint64_t* npos;
  const Shape* shapes;    // [kd]
  int kd;                 // 0 -> gamma with shapes[0], else Dirichlet dimension
  double rate;
  int S;
  int64_t n_per;
  double* out;            // gamma: [S][n_per]; Dirichlet: [S][n_per][kd]
  double* scratch;        // Dirichlet: [S][kd]
  int* drained;
};

__global__ void streams_kernel(StreamArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  UCursor U;
  NCursor N;
  U.init(a.ukeys[2 * s], a.ukeys[2 * s + 1], a.upos[s]);
  N.init(a.nkeys[2 * s], a.nkeys[2 * s + 1], a.npos[s]);
  bool ok = true;
  if (a.kd == 0) {
    const Shape sh = a.shapes[0];
    for (int64_t i = 0; i < a.n_per && ok; ++i) {
      double g;
      ok = gamma_shape(sh, U, N, g);
      if (ok) a.out[int64_t(s) * a.n_per + i] = __ddiv_rn(g, a.rate);
    }
  } else {
    double* y = a.scratch + int64_t(s) * a.kd;
    for (int64_t i = 0; i < a.n_per && ok; ++i) {
      bool done = false;
      for (int attempt = 0; attempt < 2 && ok && !done; ++attempt) {  // rng.py:207-213
        for (int k = 0; k < a.kd && ok; ++k) ok = gamma_shape(a.shapes[k], U, N, y[k]);
        if (!ok) break;
        const double total = pairwise_sum(y, a.kd);
        if (total > 0.0) {
          double* o = a.out + (int64_t(s) * a.n_per + i) * a.kd;
          for (int k = 0; k < a.kd; ++k) o[k] = __ddiv_rn(y[k], total);
          done = true;
        }
      }
      if (ok && !done) ok = false;
    }
  }
  if (!ok) atomicExch(a.drained, 1);
  a.upos[s] = U.idx;
  a.npos[s] = N.idx;
}

// ---------------------------------------------------------------- one stream, parallel scans
// Pass 1: attempt i uses normal npos+i; v = 1 + c x; valid = v > 0.
__global__ void attempt_normals_kernel(uint64_t k0, uint64_t k1, uint64_t npos, int64_t W, double c,
                                       double* xv, int* valid) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < W; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = npos + uint64_t(i);
    const uint64_t p = j >> 1;
    const U64x4 w = philox_block(p >> 1, k0, k1);
    const int o = int(p & 1) * 2;
    double zc, zs;
    box_muller(u53(w.v[o]), u53(w.v[o + 1]), zc, zs);
    const double x = (j & 1) ? zs : zc;
    xv[i] = x;
    valid[i] = __dadd_rn(1.0, __dmul_rn(c, x)) > 0.0 ? 1 : 0;
  }
}

// Pass 2: valid attempt i takes uniform upos + vex[i]; accept test (rng.py:170-177).
__global__ void attempt_accept_kernel(uint64_t k0, uint64_t k1, uint64_t upos, int64_t W, double c, double d,
                                      const double* xv, const int* valid, const int* vex, double* val,
                                      int* acc) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < W; i += int64_t(gridDim.x) * blockDim.x) {
    int ok = 0;
    double g = 0.0;
    if (valid[i]) {
      const double x = xv[i];
      double v = __dadd_rn(1.0, __dmul_rn(c, x));
      v = __dmul_rn(__dmul_rn(v, v), v);
      const uint64_t ui = upos + uint64_t(vex[i]);
      const U64x4 w = philox_block(ui >> 2, k0, k1);
      const double u = u53(w.v[ui & 3]);
      const double x2 = __dmul_rn(x, x);
      if (u < __dsub_rn(1.0, __dmul_rn(__dmul_rn(0.0331, x2), x2)) ||
          log(u) < __dadd_rn(__dmul_rn(0.5, x2), __dmul_rn(d, __dadd_rn(__dsub_rn(1.0, v), log(v))))) {
        ok = 1;
        g = __dmul_rn(d, v);
      }
    }
    acc[i] = ok;
    val[i] = g;
  }
}

// Pass 3: scatter the first `need` accepted values; remember where the last one was.
__global__ void attempt_scatter_kernel(int64_t W, int64_t need, double rate, const int* acc, const int* aex,
                                       const double* val, double* out, int64_t* where, int64_t* last_i) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < W; i += int64_t(gridDim.x) * blockDim.x) {
    if (!acc[i]) continue;
    const int64_t k = aex[i];
    if (k >= need) continue;
    out[k] = rate == 1.0 ? val[i] : __ddiv_rn(val[i], rate);
    where[k] = i;
    if (k == need - 1) *last_i = i;
  }
}

// Drain check: consecutive accepted attempts more than kGammaMaxReject apart.
__global__ void gap_kernel(int64_t m, int64_t prev, const int64_t* where, int* drained) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t before = k == 0 ? prev : where[k - 1];
    if (where[k] - before > kGammaMaxReject) atomicExch(drained, 1);
  }
}

// Dirichlet normalisation of homogeneous gamma components: y / pairwise_sum(y).
__global__ void normalise_kernel(int64_t n, int kd, const double* y, double* out, int* underflow) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double* yi = y + i * kd;
    const double total = pairwise_sum(yi, kd);
    if (!(total > 0.0)) atomicExch(underflow, 1);
    for (int k = 0; k < kd; ++k) out[i * kd + k] = __ddiv_rn(yi[k], total);
  }
}

int grid_for(int device, int64_t work, int threads) {
  const int64_t cap = int64_t(pm::sm_count(device)) * 8;
  int64_t g = (work + threads - 1) / threads;
  if (g > cap) g = cap;
  return int(g < 1 ? 1 : g);
}

struct Timer {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  cudaStream_t s;
  float* ms;
  Timer(cudaStream_t st, float* out) : s(st), ms(out) {
    if (ms) {
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0, s);
    }
  }
  void stop() {
    if (ms) {
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(ms, e0, e1);
    }
  }
  ~Timer() {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  }
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  cudaStream_t s;
  explicit DevBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t n) { return cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * (n ? n : 1), s); }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

int check_device(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return pm::fail(PM_EDEVICE, "no CUDA device visible");
  if (device < 0 || device >= n) return pm::fail(PM_ERANGE, "device index out of range");
  pm::retain_pool(device);
  return PM_OK;
}

// Single stream pair, homogeneous shape >= 1: the scan form.  Writes `need` gamma draws
// (divided by rate) to dev_out and advances *upos / *npos past exactly the consumed deviates.
int gamma_scan(int device, cudaStream_t st, double alpha, double rate, int64_t need, uint64_t uk0, uint64_t uk1,
               uint64_t* upos, uint64_t nk0, uint64_t nk1, uint64_t* npos, double* dev_out) {
  const Shape sh = make_shape(alpha);
  // attempts per draw ~ 1/acceptance (<= 1.05 for alpha >= 1); window with slack
  const int64_t Wmax = int64_t(1) << 25;
  int64_t W = need + need / 8 + 4096;
  if (W > Wmax) W = Wmax;
  DevBuf<double> xv(st), val(st);
  DevBuf<int> valid(st), vex(st), acc(st), aex(st), drained(st);
  DevBuf<int64_t> where(st), last(st);
  DevBuf<unsigned char> tmp(st);
  PM_CUDA(xv.alloc(W));
  PM_CUDA(val.alloc(W));
  PM_CUDA(valid.alloc(W));
  PM_CUDA(vex.alloc(W));
  PM_CUDA(acc.alloc(W));
  PM_CUDA(aex.alloc(W));
  PM_CUDA(drained.alloc(1));
  PM_CUDA(last.alloc(1));
  PM_CUDA(where.alloc(W));
  size_t tmp_bytes = 0;
  PM_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, valid.p, vex.p, int(W), st));
  PM_CUDA(tmp.alloc(tmp_bytes));
  PM_CUDA(cudaMemsetAsync(drained.p, 0, sizeof(int), st));
  int64_t done = 0, prev_acc = -1;  // prev_acc: attempt index (relative) of the last accept
  uint64_t un = *upos, nn = *npos;
  while (done < need) {
    const int64_t want = need - done;
    const int g = grid_for(device, W, 256);
    attempt_normals_kernel<<<g, 256, 0, st>>>(nk0, nk1, nn, W, sh.c, xv.p, valid.p);
    PM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, valid.p, vex.p, int(W), st));
    attempt_accept_kernel<<<g, 256, 0, st>>>(uk0, uk1, un, W, sh.c, sh.d, xv.p, valid.p, vex.p, val.p, acc.p);
    PM_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, acc.p, aex.p, int(W), st));
    const int64_t minus1 = -1;
    PM_CUDA(cudaMemcpyAsync(last.p, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    attempt_scatter_kernel<<<g, 256, 0, st>>>(W, want, rate, acc.p, aex.p, val.p, dev_out + done, where.p, last.p);
    PM_CUDA(cudaGetLastError());
    int tails[4];
    int64_t last_i = -1;
    PM_CUDA(cudaMemcpyAsync(&tails[0], vex.p + (W - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    PM_CUDA(cudaMemcpyAsync(&tails[1], valid.p + (W - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    PM_CUDA(cudaMemcpyAsync(&tails[2], aex.p + (W - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    PM_CUDA(cudaMemcpyAsync(&tails[3], acc.p + (W - 1), sizeof(int), cudaMemcpyDeviceToHost, st));
    PM_CUDA(cudaMemcpyAsync(&last_i, last.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PM_CUDA(cudaStreamSynchronize(st));
    const int64_t n_valid = int64_t(tails[0]) + tails[1];
    const int64_t n_acc = int64_t(tails[2]) + tails[3];
    const int64_t got = n_acc < want ? n_acc : want;
    // gaps between consecutive accepts within the window (prev carried in relative terms)
    if (got > 0) gap_kernel<<<grid_for(device, got, 256), 256, 0, st>>>(got, prev_acc, where.p, drained.p);
    if (got == want) {
      // consumed: attempts 0..last_i; uniforms = valid attempts among them
      int v_last = 0;
      PM_CUDA(cudaMemcpyAsync(&v_last, vex.p + last_i, sizeof(int), cudaMemcpyDeviceToHost, st));
      PM_CUDA(cudaStreamSynchronize(st));
      nn += uint64_t(last_i + 1);
      un += uint64_t(v_last + 1);
      done += got;
    } else {
      int64_t last_rel = -1;
      if (got > 0) {
        PM_CUDA(cudaMemcpyAsync(&last_rel, where.p + (got - 1), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        PM_CUDA(cudaStreamSynchronize(st));
      }
      // the whole window is consumed; the next window's attempt 0 follows attempt W-1
      prev_acc = (got > 0 ? last_rel : prev_acc) - W;
      // attempts since the last accept: -prev_acc - 1; the reference gives up at 10000
      if (-prev_acc - 1 >= int64_t(kGammaMaxReject))
        return pm::fail(PM_EDRAIN, "gamma rejection failed to accept after 10000 rounds");
      nn += uint64_t(W);
      un += uint64_t(n_valid);
      done += got;
    }
  }
  int h_drained = 0;
  PM_CUDA(cudaMemcpyAsync(&h_drained, drained.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  if (h_drained)
    return pm::fail(PM_EDRAIN, "gamma rejection failed to accept after 10000 rounds");
  *upos = un;
  *npos = nn;
  return PM_OK;
}

int run_streams(int device, cudaStream_t st, const std::vector<Shape>& shapes, int kd, double rate, int32_t S,
                int64_t n_per, const uint64_t* ukeys, uint64_t* upos, const uint64_t* nkeys, uint64_t* npos,
                double* dev_out) {
  DevBuf<uint64_t> d_uk(st), d_nk(st), d_up(st), d_np(st);
  DevBuf<Shape> d_sh(st);
  DevBuf<double> d_scr(st);
  DevBuf<int> d_dr(st);
  PM_CUDA(d_uk.alloc(2 * size_t(S)));
  PM_CUDA(d_nk.alloc(2 * size_t(S)));
  PM_CUDA(d_up.alloc(S));
  PM_CUDA(d_np.alloc(S));
  PM_CUDA(d_sh.alloc(shapes.size()));
  PM_CUDA(d_scr.alloc(size_t(S) * (kd > 0 ? kd : 1)));
  PM_CUDA(d_dr.alloc(1));
  PM_CUDA(cudaMemcpyAsync(d_uk.p, ukeys, sizeof(uint64_t) * 2 * S, cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemcpyAsync(d_nk.p, nkeys, sizeof(uint64_t) * 2 * S, cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemcpyAsync(d_up.p, upos, sizeof(uint64_t) * S, cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemcpyAsync(d_np.p, npos, sizeof(uint64_t) * S, cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemcpyAsync(d_sh.p, shapes.data(), sizeof(Shape) * shapes.size(), cudaMemcpyHostToDevice, st));
  PM_CUDA(cudaMemsetAsync(d_dr.p, 0, sizeof(int), st));
  StreamArgs a;
  a.ukeys = d_uk.p;
  a.nkeys = d_nk.p;
  a.upos = d_up.p;
  a.npos = d_np.p;
  a.shapes = d_sh.p;
  a.kd = kd;
  a.rate = rate;
  a.S = S;
  a.n_per = n_per;
  a.out = dev_out;
  a.scratch = d_scr.p;
  a.drained = d_dr.p;
  streams_kernel<<<(S + 127) / 128, 128, 0, st>>>(a);
  PM_CUDA(cudaGetLastError());
  int dr = 0;
  PM_CUDA(cudaMemcpyAsync(&dr, d_dr.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaMemcpyAsync(upos, d_up.p, sizeof(uint64_t) * S, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaMemcpyAsync(npos, d_np.p, sizeof(uint64_t) * S, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  if (dr) return pm::fail(PM_EDRAIN, "gamma rejection failed to accept after 10000 rounds");
  return PM_OK;
}

int validate_shape(double a) {
  if (!(a > 0.0) || !isfinite(a)) return pm::fail(PM_EINVAL, "gamma shape must be finite and > 0");
  return PM_OK;
}

}  // namespace

extern "C" {

int pm_rng_fill(int device, int kind, uint64_t key0, uint64_t key1, uint64_t pos, int64_t n, double* out,
                int out_is_device, float* ms) {
  if (int rc = check_device(device)) return rc;
  if (kind != PM_RNG_KIND_UNIFORM01 && kind != PM_RNG_KIND_STD_NORMAL) return pm::fail(PM_EINVAL, "unknown kind");
  if (n < 0) return pm::fail(PM_EINVAL, "n must be >= 0");
  if (n == 0) return PM_OK;
  if (!out) return pm::fail(PM_EINVAL, "out is NULL");
  pm::DeviceGuard g(device);
  cudaStream_t st = cudaStreamPerThread;
  DevBuf<double> tmp(st);
  double* dst = out;
  if (!out_is_device) {
    PM_CUDA(tmp.alloc(size_t(n)));
    dst = tmp.p;
  }
  Timer t(st, ms);
  const int64_t blocks = ((int64_t(pos & 3) + n) + 3) / 4;
  fill_kernel<<<grid_for(device, blocks, 256), 256, 0, st>>>(kind, key0, key1, pos, n, dst);
  PM_CUDA(cudaGetLastError());
  t.stop();
  if (!out_is_device) PM_CUDA(cudaMemcpyAsync(out, dst, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  return PM_OK;
}

int pm_rng_gamma(int device, double alpha, double rate, int64_t n, const uint64_t* ukey, uint64_t* upos,
                 const uint64_t* nkey, uint64_t* npos, double* out, float* ms) {
  if (int rc = check_device(device)) return rc;
  if (int rc = validate_shape(alpha)) return rc;
  if (!(rate > 0.0)) return pm::fail(PM_EINVAL, "rate must be > 0");
  if (n < 0) return pm::fail(PM_EINVAL, "n must be >= 0");
  if (n == 0) return PM_OK;
  pm::DeviceGuard g(device);
  cudaStream_t st = cudaStreamPerThread;
  DevBuf<double> d_out(st);
  PM_CUDA(d_out.alloc(size_t(n)));
  Timer t(st, ms);
  int rc;
  if (alpha >= 1.0) {
    rc = gamma_scan(device, st, alpha, rate, n, ukey[0], ukey[1], upos, nkey[0], nkey[1], npos, d_out.p);
  } else {
    rc = run_streams(device, st, {make_shape(alpha)}, 0, rate, 1, n, ukey, upos, nkey, npos, d_out.p);
  }
  t.stop();
  if (rc) return rc;
  PM_CUDA(cudaMemcpyAsync(out, d_out.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  return PM_OK;
}

int pm_rng_dirichlet(int device, const double* alphas, int32_t kd, int64_t n, const uint64_t* ukey, uint64_t* upos,
                     const uint64_t* nkey, uint64_t* npos, double* out, float* ms) {
  if (int rc = check_device(device)) return rc;
  if (kd < 1) return pm::fail(PM_EINVAL, "alphas must be a non-empty 1-D vector");
  std::vector<Shape> shapes(kd);
  bool homogeneous = true;
  for (int k = 0; k < kd; ++k) {
    if (!(alphas[k] > 0.0)) return pm::fail(PM_EINVAL, "all alphas must be > 0");
    shapes[k] = make_shape(alphas[k]);
    homogeneous = homogeneous && alphas[k] == alphas[0];
  }
  if (n < 0) return pm::fail(PM_EINVAL, "n must be >= 0");
  if (n == 0) return PM_OK;
  pm::DeviceGuard g(device);
  cudaStream_t st = cudaStreamPerThread;
  DevBuf<double> d_out(st), d_y(st);
  DevBuf<int> d_uf(st);
  PM_CUDA(d_out.alloc(size_t(n) * kd));
  Timer t(st, ms);
  int rc;
  if (homogeneous && alphas[0] >= 1.0) {
    // components are consecutive Gamma(alpha, 1) draws of one stream; the sum of
    // Gamma(alpha >= 1) draws is > 0, so the underflow retry (rng.py:207-213) never fires
    PM_CUDA(d_y.alloc(size_t(n) * kd));
    PM_CUDA(d_uf.alloc(1));
    PM_CUDA(cudaMemsetAsync(d_uf.p, 0, sizeof(int), st));
    rc = gamma_scan(device, st, alphas[0], 1.0, n * kd, ukey[0], ukey[1], upos, nkey[0], nkey[1], npos, d_y.p);
    if (rc == PM_OK) {
      normalise_kernel<<<grid_for(device, n, 128), 128, 0, st>>>(n, kd, d_y.p, d_out.p, d_uf.p);
      int uf = 0;
      PM_CUDA(cudaMemcpyAsync(&uf, d_uf.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      PM_CUDA(cudaStreamSynchronize(st));
      if (uf) rc = pm::fail(PM_EDRAIN, "dirichlet gamma components underflowed");
    }
  } else {
    rc = run_streams(device, st, shapes, kd, 1.0, 1, n, ukey, upos, nkey, npos, d_out.p);
  }
  t.stop();
  if (rc) return rc;
  PM_CUDA(cudaMemcpyAsync(out, d_out.p, sizeof(double) * n * kd, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  return PM_OK;
}

int pm_rng_gamma_streams(int device, double alpha, double rate, int32_t S, int64_t n_per, const uint64_t* ukeys,
                         uint64_t* upos, const uint64_t* nkeys, uint64_t* npos, double* out, float* ms) {
  if (int rc = check_device(device)) return rc;
  if (int rc = validate_shape(alpha)) return rc;
  if (!(rate > 0.0)) return pm::fail(PM_EINVAL, "rate must be > 0");
  if (S < 0 || n_per < 0) return pm::fail(PM_EINVAL, "S and n_per must be >= 0");
  if (S == 0 || n_per == 0) return PM_OK;
  pm::DeviceGuard g(device);
  cudaStream_t st = cudaStreamPerThread;
  DevBuf<double> d_out(st);
  PM_CUDA(d_out.alloc(size_t(S) * n_per));
  Timer t(st, ms);
  const int rc = run_streams(device, st, {make_shape(alpha)}, 0, rate, S, n_per, ukeys, upos, nkeys, npos, d_out.p);
  t.stop();
  if (rc) return rc;
  PM_CUDA(cudaMemcpyAsync(out, d_out.p, sizeof(double) * S * n_per, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  return PM_OK;
}

int pm_rng_dirichlet_streams(int device, const double* alphas, int32_t kd, int32_t S, int64_t n_per,
                             const uint64_t* ukeys, uint64_t* upos, const uint64_t* nkeys, uint64_t* npos, double* out,
                             float* ms) {
  if (int rc = check_device(device)) return rc;
  if (kd < 1) return pm::fail(PM_EINVAL, "alphas must be a non-empty 1-D vector");
  std::vector<Shape> shapes(kd);
  for (int k = 0; k < kd; ++k) {
    if (!(alphas[k] > 0.0)) return pm::fail(PM_EINVAL, "all alphas must be > 0");
    shapes[k] = make_shape(alphas[k]);
  }
  if (S < 0 || n_per < 0) return pm::fail(PM_EINVAL, "S and n_per must be >= 0");
  if (S == 0 || n_per == 0) return PM_OK;
  pm::DeviceGuard g(device);
  cudaStream_t st = cudaStreamPerThread;
  DevBuf<double> d_out(st);
  PM_CUDA(d_out.alloc(size_t(S) * n_per * kd));
  Timer t(st, ms);
  const int rc = run_streams(device, st, shapes, kd, 1.0, S, n_per, ukeys, upos, nkeys, npos, d_out.p);
  t.stop();
  if (rc) return rc;
  PM_CUDA(cudaMemcpyAsync(out, d_out.p, sizeof(double) * S * n_per * kd, cudaMemcpyDeviceToHost, st));
  PM_CUDA(cudaStreamSynchronize(st));
  return PM_OK;
}

}  // extern "C"
