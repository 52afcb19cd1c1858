// Device code of the logistic-GLM hot path, sm_100a.
//
// Reference semantics (all /root/reference/pkg/src/parmcmc):
//   _block_fg            glm.py:367-372   t = x@beta; f = _nll_sum(t,y); gf = y - expit(t); g = x.T@gf
//   _nll_sum             glm.py:179-192   -sum[(1-y)t + max(-t,0) + log1p(exp(-|t|))]
//   _merge_grad          glm.py:243-250   fixed-order sum of partials
//   GaussianPrior        sampler.py:55-58 -0.5*((v-mu)/sigma)^2, constants dropped
//   diff_loglike         glm.py:499-522   _nll_sum(xbeta + delta*xt[k], y)
//   commit_update        glm.py:525-539   xbeta += delta*xt[k]
//
// Layout in HBM: X row-major [n_pad][K] with n_pad = roundup(N, 32) (zero rows), y f64 [n_pad].
// One tile = 32 consecutive rows = 32*K*sizeof(XT) contiguous bytes, moved by one TMA bulk
// copy (cp.async.bulk -> SASS UBLKCP) into a shared-memory ring guarded by mbarriers.
// X is read from HBM exactly once per evaluation.
#pragma once

#include <type_traits>

#include "pm_internal.cuh"
#include "pm_math.cuh"

namespace pm {

constexpr int kTileRows = 32;

template <int KC>
struct BetaPack {
  double v[32 * KC];
};

// Per-row stable terms, identical algebra to _nll_sum (glm.py:186-192) and expit.
//   nll = (1-y) t + max(-t,0) + log1p(exp(-|t|))       (the reference's f is -sum nll)
//   w   = y - sigmoid(t)                                (glm.py:371)
// (lean fp64 exp/log1p/reciprocal of pm_math.cuh: <= 2 ulp, no special-case paths)
__device__ __forceinline__ void row_terms(double t, double y, double& nll, double& w) {
  pm_row_terms(t, y, nll, w);
}

// Rounding identical to numpy's `xbeta + delta*xk` (glm.py:517/537): product rounded, then sum.
__device__ __forceinline__ double shifted_t(double xb, double d, double xk) {
  return __dadd_rn(xb, __dmul_rn(d, xk));
}

// nll term only (diff_loglike, glm.py:499-522)
__device__ __forceinline__ double row_nll(double t, double y) { return pm_row_nll(t, y); }

// v[r] holds this lane's partial dot product for sub-tile row r (R rows).  Returns, in lane l,
// the full (all-lane) dot product of row l & (R-1): log2(R) transpose-halving steps, then a
// plain butterfly over the remaining lane bits (so every lane of a row group holds the same
// bits).  R = 32 costs 31 shuffles per 32 rows.
template <int R>
__device__ __forceinline__ double transpose_reduce(double (&v)[R], int lane) {
#pragma unroll
  for (int s = R / 2; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int i = 0; i < s; ++i) {
      const double send = upper ? v[i] : v[i + s];
      const double keep = upper ? v[i + s] : v[i];
      v[i] = keep + shfl_xor_d(send, s);
    }
  }
  double t = v[0];
#pragma unroll
  for (int m = R; m < 32; m <<= 1) t += shfl_xor_d(t, m);
  return t;
}

template <typename XT>
__device__ __forceinline__ double ld_x(const XT* p) {
  return static_cast<double>(*p);
}

// fp32-X widening without F2F.F64.F32 (an XU-pipe op at a quarter of the ALU rate, the
// measured limiter of the fp32-X stream kernel): the fp32 bit pattern s|e8|m23 becomes the
// fp64 words hi = s|000|e8|m[22:3], lo = m[2:0] << 29, i.e. exactly x * 2^-896 for EVERY
// finite x (zero and subnormals included: an fp32 subnormal lands on the fp64 subnormal of
// the same scaled value).  Two ALU ops + one shift.  The caller multiplies beta and the
// per-row residual by 2^896 (exact), so x'beta' = x beta and w' x' = w x bit for bit: the
// results are identical to the F2F form.  Used when |beta| < 2^100 (host-checked).
constexpr double kF32Unscale = 0x1p896;
__device__ __forceinline__ double ld_x_scaled(const float* p) {
  const uint32_t b = *reinterpret_cast<const uint32_t*>(p);
  const uint32_t hi = uint32_t(int32_t(b) >> 3) & 0x8FFFFFFFu;
  return __hiloint2double(int(hi), int(b << 29));
}
__device__ __forceinline__ double ld_x_scaled(const double* p) { return *p; }

template <typename XT>
struct XScale {  // factor applied to beta and to the row residual for scaled loads
  static constexpr double value = 1.0;
};
template <>
struct XScale<float> {
#ifdef PM_F32_F2F
  static constexpr double value = 1.0;
#else
  static constexpr double value = kF32Unscale;
#endif
};

template <typename XT>
__device__ __forceinline__ double ld_x_stream(const XT* p) {
  if constexpr (XScale<XT>::value != 1.0) return ld_x_scaled(p);
  return ld_x(p);
}

// Rows per register-resident sub-tile: x[R][KC] stays in registers from the dot product to
// the gradient update, so shared memory is read once; R*KC <= 64 doubles per lane.
template <int KC, bool GRAD>
struct SubRows {
  static constexpr int value = !GRAD ? 32 : (KC <= 2 ? 32 : (KC <= 4 ? 16 : 8));
};

// One warp consumes one 32-row tile resident in shared memory, R rows at a time.
// Lane l owns columns l + 32 j (j < KC): beta and the gradient accumulators live in
// registers.  The tile is read from HBM once (TMA) and from shared memory once.
// Each row's transcendental terms are computed by 32/R lanes; only lane < R counts f.
// `empty` (the stage's release barrier) is arrived on as soon as the last sub-tile's values
// are in registers, so the producer can refill the stage while this warp still computes.
// Self-producing consumers pass a RefillWhen: at the release point the warp quiesces its reads
// of the stage and, when `active` (the unit's last tile), issues its own next copies (fn).
struct NoRefill {};
template <class F>
struct RefillWhen {
  bool active;
  F fn;
};
template <typename XT, int KC, bool GRAD, int R = SubRows<KC, GRAD>::value, int TR = kTileRows,
          class Refill = NoRefill>
__device__ __forceinline__ void consume_tile(const XT* xs, const double* ys, int K, int lane, int64_t row0,
                                             int64_t row_limit, const double (&breg)[KC], double (&g)[KC],
                                             double& nll_acc, uint64_t* empty, Refill refill = Refill()) {
#pragma unroll 1
  for (int sub = 0; sub < TR / R; ++sub) {
    const XT* xb = xs + (sub * R) * K + lane;
    double x[R][KC];
    double v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        x[r][j] = (j < KC - 1 || lane + 32 * j < K) ? ld_x_stream(xb + r * K + 32 * j) : 0.0;
        // first term as a product: rn(x*b) == fma(x, b, 0) up to the sign of a zero (which
        // cannot change f or g), and it saves zeroing the accumulator pair (CS2R) per row
        acc = j == 0 ? __dmul_rn(x[r][0], breg[0]) : fma(x[r][j], breg[j], acc);
      }
      v[r] = acc;
    }
    const int rr = sub * R + (lane & (R - 1));
    const double yv = ys[rr];
    if (sub == TR / R - 1) {
      // the last sub-tile's loads feed v[] and yv (earlier sub-tiles were consumed before)
      double dep = yv;
#pragma unroll
      for (int r = 0; r < R; ++r) dep += v[r];
      if constexpr (!std::is_same<Refill, NoRefill>::value) {
        if (refill.active) {
          mbar_arrive_after(nullptr, dep, lane, const_cast<XT*>(xs));  // quiesce only
          refill.fn();
        }
      } else if (empty) {
        mbar_arrive_after(empty, dep, lane, const_cast<XT*>(xs));
      }
    }
    const double t = transpose_reduce<R>(v, lane);
    double nll, w;
    row_terms(t, yv, nll, w);
    const bool valid = row0 + rr < row_limit;
    nll_acc += (valid && lane < R) ? nll : 0.0;
    if (GRAD) {
      w = valid ? w : 0.0;
      if constexpr (XScale<XT>::value != 1.0) w *= XScale<XT>::value;  // exact (power of two)
      // NS interleaved accumulator sets so at least ~8 independent DFMA chains are in flight
      // (one set of KC chains would serialise on DFMA latency at small KC)
      constexpr int NS = KC >= 8 ? 1 : ((8 / KC) < R ? (8 / KC) : R);
      double ga[NS > 1 ? NS - 1 : 1][KC];
#pragma unroll
      for (int s = 0; s + 1 < NS; ++s)
#pragma unroll
        for (int j = 0; j < KC; ++j) ga[s][j] = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double wr = shfl_d(w, r);
        if (r % NS == 0) {
#pragma unroll
          for (int j = 0; j < KC; ++j) g[j] = fma(wr, x[r][j], g[j]);
        } else {
#pragma unroll
          for (int j = 0; j < KC; ++j) ga[r % NS - 1][j] = fma(wr, x[r][j], ga[r % NS - 1][j]);
        }
      }
#pragma unroll
      for (int s = 0; s + 1 < NS; ++s)
#pragma unroll
        for (int j = 0; j < KC; ++j) g[j] += ga[s][j];
    }
  }
}

// fp32-X consumer: column PAIRS per lane and XOR-permuted rows (K even, ceil(K/32) even).
// Lane l owns columns 64c + 2l + e (c < KC/2, e < 2): one 8-byte shared load per (row, c)
// instead of two 4-byte ones.  Slot r of lane l holds row r ^ (l & (R-1)) of the sub-tile
// (a per-lane row offset, roff[r]), so the transpose-reduce needs no selects: at level s a
// lane keeps slots [0, s) and adds the partner's (lane ^ s) slots [s, 2s), which hold exactly
// the same rows.  Lane l ends with the dot product of row l & (R-1); the residual of the row
// in slot r lives in lane l ^ r.  Bitwise deterministic for a fixed geometry; the per-row
// arithmetic (product + sum orders) differs from consume_tile only in the lane summation tree.
// (fp64 X: the same layout with 16-byte loads of two doubles, no widening.)
template <typename XT, int KC, bool GRAD, int R, int TR>
__device__ __forceinline__ void consume_tile_pairs(const XT* xs, const double* ys, int K, int lane, int64_t row0,
                                                   int64_t row_limit, const double (&breg)[KC], double (&g)[KC],
                                                   double& nll_acc, uint64_t* empty, const uint32_t (&roff)[R]) {
  static_assert(KC % 2 == 0, "pairs layout needs an even register count");
  constexpr int KP = KC / 2;
  const bool last_ok = 64 * (KP - 1) + 2 * lane < K;
  // fp32-X: the two sub-tiles of a tile are unrolled so the compiler interleaves their
  // latency chains (+4.5 % at c1f32 with 7 consumer warps, profiles/r01_ab_unroll.txt);
  // fp64 keeps one sub-tile at a time (HBM-bound; unrolling measured no gain)
  constexpr int kSubUnroll = std::is_same<XT, float>::value ? 2 : 1;
#pragma unroll kSubUnroll
  for (int sub = 0; sub < TR / R; ++sub) {
    const char* xb = reinterpret_cast<const char*>(xs) + size_t(sub) * R * K * sizeof(XT);
    double x[R][KC];
    double v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
      if constexpr (std::is_same<XT, double>::value) {
        const double2* pr = reinterpret_cast<const double2*>(xb + roff[r]);
#pragma unroll
        for (int c = 0; c < KP; ++c) {
          double2 u = make_double2(0.0, 0.0);
          if (c < KP - 1 || last_ok) u = pr[32 * c];
          x[r][2 * c] = u.x;
          x[r][2 * c + 1] = u.y;
          acc = c == 0 ? __dmul_rn(x[r][0], breg[0]) : fma(x[r][2 * c], breg[2 * c], acc);
          acc = fma(x[r][2 * c + 1], breg[2 * c + 1], acc);
        }
        v[r] = acc;
        continue;
      }
      const uint2* pr = reinterpret_cast<const uint2*>(xb + roff[r]);
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        uint2 u = make_uint2(0u, 0u);
        if (c < KP - 1 || last_ok) u = pr[32 * c];
#if defined(PM_F32_F2F)
        x[r][2 * c] = double(__uint_as_float(u.x));
        x[r][2 * c + 1] = double(__uint_as_float(u.y));
#else
        x[r][2 * c] = ld_x_scaled(reinterpret_cast<const float*>(&u.x));
        x[r][2 * c + 1] = ld_x_scaled(reinterpret_cast<const float*>(&u.y));
#endif
        acc = c == 0 ? __dmul_rn(x[r][0], breg[0]) : fma(x[r][2 * c], breg[2 * c], acc);
        acc = fma(x[r][2 * c + 1], breg[2 * c + 1], acc);
      }
      v[r] = acc;
    }
    const int rr = sub * R + (lane & (R - 1));
    const double yv = ys[rr];
    if (sub == TR / R - 1) {
      double dep = yv;
#pragma unroll
      for (int r = 0; r < R; ++r) dep += v[r];
      mbar_arrive_after(empty, dep, lane, const_cast<XT*>(xs));
    }
#pragma unroll
    for (int st = R / 2; st >= 1; st >>= 1) {
#pragma unroll
      for (int i = 0; i < st; ++i) v[i] += shfl_xor_d(v[i + st], st);
    }
    double t = v[0];
#pragma unroll
    for (int m = R; m < 32; m <<= 1) t += shfl_xor_d(t, m);
    double nll, w;
    row_terms(t, yv, nll, w);
    const bool valid = row0 + rr < row_limit;
    nll_acc += (valid && lane < R) ? nll : 0.0;
    if (GRAD) {
      w = valid ? w : 0.0;
      w *= XScale<XT>::value;  // exact (power of two)
      constexpr int NS = KC >= 8 ? 1 : ((8 / KC) < R ? (8 / KC) : R);
      double ga[NS > 1 ? NS - 1 : 1][KC];
#pragma unroll
      for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
        for (int j = 0; j < KC; ++j) ga[s2][j] = 0.0;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double wr = r == 0 ? w : shfl_xor_d(w, r);
        if (r % NS == 0) {
#pragma unroll
          for (int j = 0; j < KC; ++j) g[j] = fma(wr, x[r][j], g[j]);
        } else {
#pragma unroll
          for (int j = 0; j < KC; ++j) ga[r % NS - 1][j] = fma(wr, x[r][j], ga[r % NS - 1][j]);
        }
      }
#pragma unroll
      for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
        for (int j = 0; j < KC; ++j) g[j] += ga[s2][j];
    }
  }
}

// fp32-X whole-tile consumer (pairs layout, KC in {2, 4}, 7 consumer warps, 2 stages per
// warp).  A tile's 32 rows are taken as 4 blocks of 8 XOR-permuted rows (as in
// consume_tile_pairs); the 8-lane partial sums of the 4 blocks are then reduced across lane
// bits 3 and 4 with a select transpose, so lane l ends with the full dot product of tile row
// l: the logistic terms are evaluated ONCE per row (32 distinct rows per warp evaluation,
// instead of 32/R lanes repeating each row -- that latency chain bounded the sub-tile
// consumers).  HOLD (KC = 2): the raw fp32 words stay in registers and the stage is released
// right after the dot products; otherwise (KC = 4, the registers do not fit) the gradient
// pass re-reads the stage and releases it afterwards.  Widening: integer ops for the dot
// products (x * 2^-896 against beta * 2^896), F2F for a re-read gradient pass (balances the
// ALU and XU pipes; both exact, so the results do not depend on the choice).
template <int KC, bool GRAD>
__device__ __forceinline__ void consume_tile_f32full(const float* xs, const double* ys, int K, int lane,
                                                     int64_t row0, int64_t row_limit, const double (&breg)[KC],
                                                     double (&g)[KC], double& nll_acc, uint64_t* empty,
                                                     const uint32_t (&roff)[8]) {
  static_assert(KC == 2 || KC == 4, "whole-tile fp32 consumer: KC 2 or 4");
  constexpr int KP = KC / 2;
  constexpr bool HOLD = KC == 2;
  const bool last_ok = 64 * (KP - 1) + 2 * lane < K;
  const int b = lane & 7;
  const char* xb = reinterpret_cast<const char*>(xs);
  const uint32_t blk = uint32_t(8 * K * sizeof(float));
  auto load = [&](int s, int r, int c) -> uint2 {
    uint2 u = make_uint2(0u, 0u);
    if (c < KP - 1 || last_ok) u = reinterpret_cast<const uint2*>(xb + s * blk + roff[r])[32 * c];
    return u;
  };
  uint2 xr[HOLD ? 4 : 1][8][KP];
  if constexpr (HOLD) {
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < KP; ++c) xr[s][r][c] = load(s, r, c);
  }
  const double yv = ys[lane];
  double vs[4];
  double dep = yv;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int c = 0; c < KP; ++c) {
        const uint2 u = HOLD ? xr[HOLD ? s : 0][r][c] : load(s, r, c);
        acc = fma(ld_x_scaled(reinterpret_cast<const float*>(&u.x)), breg[2 * c], acc);
        acc = fma(ld_x_scaled(reinterpret_cast<const float*>(&u.y)), breg[2 * c + 1], acc);
      }
      v[r] = acc;
      dep += acc;
    }
#pragma unroll
    for (int st = 4; st >= 1; st >>= 1) {
#pragma unroll
      for (int i = 0; i < st; ++i) v[i] += shfl_xor_d(v[i + st], st);
    }
    vs[s] = v[0];  // block s, row 8s + b, summed over the 8 lanes sharing lane bits 3-4
  }
  if (HOLD || !GRAD) mbar_arrive_after(empty, dep, lane, const_cast<float*>(xs));  // all words consumed
  // across lane bits 4 then 3: lane l keeps block (l >> 3), i.e. tile row l
  {
    const bool up = (lane & 16) != 0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const double send = up ? vs[i] : vs[i + 2];
      const double keep = up ? vs[i + 2] : vs[i];
      vs[i] = keep + shfl_xor_d(send, 16);
    }
    const bool up1 = (lane & 8) != 0;
    const double send = up1 ? vs[0] : vs[1];
    const double keep = up1 ? vs[1] : vs[0];
    vs[0] = keep + shfl_xor_d(send, 8);
  }
  const double t = vs[0];
  double nll, w;
  row_terms(t, yv, nll, w);
  const bool valid = row0 + lane < row_limit;
  nll_acc += valid ? nll : 0.0;
  if (GRAD) {
    // HOLD widens by integer ops (x * 2^-896): scale w by 2^896 (exact); else F2F (unscaled)
    w = valid ? (HOLD ? w * kF32Unscale : w) : 0.0;
    constexpr int NS = KC == 2 ? 4 : 2;
    double ga[NS - 1][KC];
#pragma unroll
    for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
      for (int j = 0; j < KC; ++j) ga[s2][j] = 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const double wr = __shfl_sync(0xffffffffu, w, 8 * s + (r ^ b));
        const int set = (8 * s + r) % NS;
#pragma unroll
        for (int c = 0; c < KP; ++c) {
          double x0, x1;
          if constexpr (HOLD) {
            x0 = ld_x_scaled(reinterpret_cast<const float*>(&xr[s][r][c].x));
            x1 = ld_x_scaled(reinterpret_cast<const float*>(&xr[s][r][c].y));
          } else {
            const uint2 u = load(s, r, c);
            x0 = double(__uint_as_float(u.x));
            x1 = double(__uint_as_float(u.y));
          }
          if (set == 0) {
            g[2 * c] = fma(wr, x0, g[2 * c]);
            g[2 * c + 1] = fma(wr, x1, g[2 * c + 1]);
          } else {
            ga[set - 1][2 * c] = fma(wr, x0, ga[set - 1][2 * c]);
            ga[set - 1][2 * c + 1] = fma(wr, x1, ga[set - 1][2 * c + 1]);
          }
        }
      }
#pragma unroll
    for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
      for (int j = 0; j < KC; ++j) g[j] += ga[s2][j];
    if constexpr (!HOLD) {
      double dg = 0.0;
#pragma unroll
      for (int j = 0; j < KC; ++j) dg += g[j];  // depends on every re-read word
      mbar_arrive_after(empty, dg, lane, const_cast<float*>(xs));
    }
  }
}

// fp32-X "row-dot" consumer (PAIRS == 3; K % 4 == 0 and K/4 odd, so the 16-byte row loads of
// a quarter-warp fall in distinct bank groups).
// Phase A: lane l owns ROW l of the 32-row tile: its dot product over all K columns with
//   16-byte shared loads of the row, beta broadcast from shared memory (every lane reads the
//   same address), 4 interleaved DFMA chains and F2F widening (XU pipe, otherwise idle) --
//   no shuffles, no transpose -- then the logistic terms ONCE per row.
// Phase B: the gradient in the pairs layout (lane l owns columns 64c + 2l, 64c + 2l + 1): the
//   tile is re-read row by row with 8-byte loads, widened by integer ops (x * 2^-896 against
//   w * 2^896, exact), w_r broadcast from lane r.
// Against consume_tile_pairs at K = 100: ~33 instead of ~45 warp instructions per row, 64
// instead of 124 shuffles per tile, and x never lives in registers across the two phases
// (the pairs consumer keeps 16 x 4 doubles = 128 registers per sub-tile in flight).
// PM_ROWDOT_F2F_PAIRS: leading column pairs of every gradient-phase row widened by F2F (XU
// pipe) instead of integer ops (ALU pipe); A/B builds override it (-DPM_ROWDOT_F2F_PAIRS=0|1|2)
#ifndef PM_ROWDOT_F2F_PAIRS
#define PM_ROWDOT_F2F_PAIRS 1
#endif
template <int KC, bool GRAD>
__device__ __forceinline__ void consume_tile_rowdot(const float* xs, const double* ys, int K, int lane,
                                                    int64_t row0, int64_t row_limit, const double* sbeta,
                                                    double (&g)[KC], double& nll_acc, uint64_t* empty) {
  static_assert(KC % 2 == 0, "row-dot consumer: pairs layout in the gradient phase");
  constexpr int KP = KC / 2;
  const float* xr = xs + size_t(lane) * K;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int nq = K >> 2;
#pragma unroll 5
  for (int q = 0; q < nq; ++q) {
    const float4 xv = *reinterpret_cast<const float4*>(xr + 4 * q);
    const double2 b01 = *reinterpret_cast<const double2*>(sbeta + 4 * q);
    const double2 b23 = *reinterpret_cast<const double2*>(sbeta + 4 * q + 2);
    a0 = fma(double(xv.x), b01.x, a0);
    a1 = fma(double(xv.y), b01.y, a1);
    a2 = fma(double(xv.z), b23.x, a2);
    a3 = fma(double(xv.w), b23.y, a3);
  }
  const double t = (a0 + a1) + (a2 + a3);
  const double yv = ys[lane];
  double nll, w;
  row_terms(t, yv, nll, w);
  const bool valid = row0 + lane < row_limit;
  nll_acc += valid ? nll : 0.0;
  if constexpr (!GRAD) {
    mbar_arrive_after(empty, t + yv, lane, const_cast<float*>(xs));
    return;
  }
  w = valid ? w * kF32Unscale : 0.0;  // exact (power of two)
  const bool last_ok = 64 * (KP - 1) + 2 * lane < K;
  const char* xb = reinterpret_cast<const char*>(xs) + 2 * lane * sizeof(float);
  const uint32_t row_bytes = uint32_t(K) * sizeof(float);
  constexpr int NS = KC >= 8 ? 1 : 8 / KC;
  double ga[NS > 1 ? NS - 1 : 1][KC];
#pragma unroll
  for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
    for (int j = 0; j < KC; ++j) ga[s2][j] = 0.0;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const double wr = __shfl_sync(0xffffffffu, w, r);
    // the first pair of every row is widened by F2F against the unscaled residual (one
    // exact DMUL per row), the others by integer ops against the scaled one: the products
    // are the same real numbers, so the sums do not depend on the split -- it balances the
    // XU pipe (F2F) against the ALU pipe (3 integer ops per element)
    [[maybe_unused]] const double wr_u = wr * (1.0 / kF32Unscale);
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      uint2 u = make_uint2(0u, 0u);
      if (c < KP - 1 || last_ok) u = *reinterpret_cast<const uint2*>(xb + r * row_bytes + 256 * c);
      const bool f2f = c < PM_ROWDOT_F2F_PAIRS;
      const double x0 = f2f ? double(__uint_as_float(u.x)) : ld_x_scaled(reinterpret_cast<const float*>(&u.x));
      const double x1 = f2f ? double(__uint_as_float(u.y)) : ld_x_scaled(reinterpret_cast<const float*>(&u.y));
      const double ww = f2f ? wr_u : wr;
      if (r % NS == 0) {
        g[2 * c] = fma(ww, x0, g[2 * c]);
        g[2 * c + 1] = fma(ww, x1, g[2 * c + 1]);
      } else {
        ga[r % NS - 1][2 * c] = fma(ww, x0, ga[r % NS - 1][2 * c]);
        ga[r % NS - 1][2 * c + 1] = fma(ww, x1, ga[r % NS - 1][2 * c + 1]);
      }
    }
  }
#pragma unroll
  for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
    for (int j = 0; j < KC; ++j) g[j] += ga[s2][j];
  double dg = 0.0;
#pragma unroll
  for (int j = 0; j < KC; ++j) dg += g[j];  // depends on every re-read word
  mbar_arrive_after(empty, dg, lane, const_cast<float*>(xs));
}

// fp32-X row-dot consumer run by a PAIR of warps per tile (PAIRS == 4; KC == 4, K % 4 == 0,
// K/4 odd).  A single warp per tile holds its stage for the whole two-phase tile time, and 15
// such warps with one stage each left the consumers waiting on their refills for 42 % of the
// samples (profiles/r02_ncu_rowdot15_*: by Little's law ~6 tiles must be in flight per SM on
// top of the ones being computed, and 21 stages of 13 KB do not fit).  Two warps per tile
// halve the hold time: 7 pairs x 2 stages = 14 stages, double-buffered, 14 consumer warps.
//   phase A: warp `sub` of the pair takes the 16-byte column chunks [q_lo, q_hi) of ALL 32
//     rows (lane = row); the two partial dot products meet through shared memory (`xch`,
//     double-buffered by tile parity) at a 64-thread named barrier; both warps evaluate the
//     logistic terms (each needs w for its rows below; only sub 0 counts f).
//   phase B: warp `sub` adds rows [16 sub, 16 sub + 16) into its own gradient partial (pairs
//     layout, integer widening), then both warps arrive on the stage's release barrier
//     (initialised with count 2); each writes its dependency word into its OWN half of the
//     stage (the partner may still be reading the other half).
template <int KC, bool GRAD>
__device__ __forceinline__ void consume_tile_rowdot2(const float* xs, const double* ys, int K, int lane, int sub,
                                                     int pair, uint32_t parity, int64_t row0, int64_t row_limit,
                                                     const double* sbeta, double* xch, double (&g)[KC],
                                                     double& nll_acc, uint64_t* empty) {
  static_assert(KC % 2 == 0, "row-dot consumer: pairs layout in the gradient phase");
  constexpr int KP = KC / 2;
  const float* xr = xs + size_t(lane) * K;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int nq = K >> 2, nh = (nq + 1) >> 1;
  const int q_lo = sub ? nh : 0, q_hi = sub ? nq : nh;
#pragma unroll 4
  for (int q = q_lo; q < q_hi; ++q) {
    const float4 xv = *reinterpret_cast<const float4*>(xr + 4 * q);
    const double2 b01 = *reinterpret_cast<const double2*>(sbeta + 4 * q);
    const double2 b23 = *reinterpret_cast<const double2*>(sbeta + 4 * q + 2);
    a0 = fma(double(xv.x), b01.x, a0);
    a1 = fma(double(xv.y), b01.y, a1);
    a2 = fma(double(xv.z), b23.x, a2);
    a3 = fma(double(xv.w), b23.y, a3);
  }
  const double tpart = (a0 + a1) + (a2 + a3);
  double* box = xch + ((size_t(pair) * 2 + parity) * 2) * 32;  // [pair][parity][sub][lane]
  box[sub * 32 + lane] = tpart;
  asm volatile("bar.sync %0, 64;" ::"r"(pair + 1) : "memory");
  const double other = box[(sub ^ 1) * 32 + lane];
  const double t = sub ? other + tpart : tpart + other;  // t_0 + t_1 in both warps
  const double yv = ys[lane];
  double nll, w;
  row_terms(t, yv, nll, w);
  const bool valid = row0 + lane < row_limit;
  nll_acc += (valid && sub == 0) ? nll : 0.0;
  float* mine = const_cast<float*>(xs) + size_t(16 * sub) * K;  // this warp's half of the stage
  if constexpr (!GRAD) {
    mbar_arrive_after(empty, t + yv, lane, mine);
    return;
  }
  w = valid ? w * kF32Unscale : 0.0;  // exact (power of two)
  const bool last_ok = 64 * (KP - 1) + 2 * lane < K;
  const char* xb = reinterpret_cast<const char*>(mine) + 2 * lane * sizeof(float);
  const uint32_t row_bytes = uint32_t(K) * sizeof(float);
  constexpr int NS = KC >= 8 ? 1 : 8 / KC;
  double ga[NS > 1 ? NS - 1 : 1][KC];
#pragma unroll
  for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
    for (int j = 0; j < KC; ++j) ga[s2][j] = 0.0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const double wr = __shfl_sync(0xffffffffu, w, 16 * sub + r);
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      uint2 u = make_uint2(0u, 0u);
      if (c < KP - 1 || last_ok) u = *reinterpret_cast<const uint2*>(xb + r * row_bytes + 256 * c);
      const double x0 = ld_x_scaled(reinterpret_cast<const float*>(&u.x));
      const double x1 = ld_x_scaled(reinterpret_cast<const float*>(&u.y));
      if (r % NS == 0) {
        g[2 * c] = fma(wr, x0, g[2 * c]);
        g[2 * c + 1] = fma(wr, x1, g[2 * c + 1]);
      } else {
        ga[r % NS - 1][2 * c] = fma(wr, x0, ga[r % NS - 1][2 * c]);
        ga[r % NS - 1][2 * c + 1] = fma(wr, x1, ga[r % NS - 1][2 * c + 1]);
      }
    }
  }
#pragma unroll
  for (int s2 = 0; s2 + 1 < NS; ++s2)
#pragma unroll
    for (int j = 0; j < KC; ++j) g[j] += ga[s2][j];
  double dg = 0.0;
#pragma unroll
  for (int j = 0; j < KC; ++j) dg += g[j];  // depends on every re-read word
  mbar_arrive_after(empty, dg, lane, mine);
}

// Column owned by register j of `lane` in the two consumer layouts.
template <bool PAIRS>
__device__ __forceinline__ int lane_col(int lane, int j) {
  return PAIRS ? 64 * (j >> 1) + 2 * lane + (j & 1) : lane + 32 * j;
}

// Shared-memory carve-up of the streaming kernels.
struct StreamSmem {
  unsigned char* xs;  // [S][tile_bytes]
  double* ys;         // [S][32]
  uint64_t* full;     // [S]
  uint64_t* empty;    // [S]
  double* sbeta;      // [K]
  double* wg;         // [nw][K]
  double* wf;         // [nw]
  int* flag;
};

__host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// tr = rows per stage (a 32-row tile, or half of one for the 2-stages-per-warp fp32-X variant)
__host__ __device__ inline size_t stream_smem_bytes(int K, int xsize, int S, int nw, int tr = kTileRows) {
  size_t tile = size_t(tr) * K * xsize;
  size_t b = align_up(tile, 128) * S;
  b += size_t(S) * tr * sizeof(double);
  b += size_t(2 * S) * sizeof(uint64_t);
  b += align_up(size_t(K) * sizeof(double), 16);
  b += size_t(nw) * K * sizeof(double);
  b += align_up(size_t(nw) * sizeof(double), 16) + 16;
  return b;
}

__device__ inline StreamSmem carve_stream_smem(unsigned char* base, int K, int xsize, int S, int nw,
                                               int tr = kTileRows) {
  StreamSmem s;
  size_t tile = align_up(size_t(tr) * K * xsize, 128);
  unsigned char* p = base;
  s.xs = p;
  p += tile * S;
  s.ys = reinterpret_cast<double*>(p);
  p += size_t(S) * tr * sizeof(double);
  s.full = reinterpret_cast<uint64_t*>(p);
  p += size_t(S) * sizeof(uint64_t);
  s.empty = reinterpret_cast<uint64_t*>(p);
  p += size_t(S) * sizeof(uint64_t);
  s.sbeta = reinterpret_cast<double*>(p);
  p += align_up(size_t(K) * sizeof(double), 16);
  s.wg = reinterpret_cast<double*>(p);
  p += size_t(nw) * K * sizeof(double);
  s.wf = reinterpret_cast<double*>(p);
  p += align_up(size_t(nw) * sizeof(double), 16);
  s.flag = reinterpret_cast<int*>(p);
  return s;
}

// Producer/consumer ring over "units" of tiles (a tile = TR consecutive rows).
//   U == 1: unit i is the single tile tile_begin + i*stride (< tile_end): tiles interleaved
//           across CTAs (stride = grid) or a contiguous range (stride = 1).
//   U  > 1: the caller's range [tile_begin, tile_end) is contiguous (stride must be 1) and
//           unit i is the U consecutive tiles from tile_begin + i*U (the last unit may be
//           shorter): ONE bulk copy of X and one of y per unit.  For small tiles (K <= ~64
//           fp64) the single producer thread's ~200 ns per copy bounds the pipeline
//           otherwise (profiles/r02_c0_breakdown.txt).
// A stage holds one unit; warp 0 lane 0 issues the TMA bulk copies; warps 1..NCW consume
// units round-robin.  Rows with global (padded) index >= row_limit are masked (padding).
// MULTI (compile time): U > 1 is only compiled into the column-per-lane consumers of the
// 8-warp kernels (the narrow designs that need it); the pairs consumers keep the plain
// single-tile loop (a per-tile release condition inside their unrolled sub-tile pair cost
// the fp32-X kernel 9 %, r02 pass C).
template <typename XT, int KC, bool GRAD, int NCW, int R = SubRows<KC, GRAD>::value, int TR = kTileRows,
          int PAIRS = 0>
__device__ __forceinline__ void stream_tiles(const XT* __restrict__ X, const double* __restrict__ y, int K,
                                             int64_t tile_begin, int64_t tile_end, int64_t stride,
                                             int64_t row_limit, int S, const StreamSmem& sm,
                                             const double (&breg)[KC], double (&g)[KC], double& nll_acc,
                                             bool evict_first, int U_arg = 1, int selfprod = 0) {
  constexpr bool MULTI = PAIRS == 0 && NCW <= 8;
  const int U = MULTI ? U_arg : 1;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t tile_elems = uint32_t(TR) * K;
  const uint32_t tile_bytes = tile_elems * sizeof(XT);
  const size_t tile_pitch = align_up(size_t(U) * tile_bytes, 128);  // stage pitch
  const int64_t n_tiles_mine = tile_end > tile_begin ? (tile_end - tile_begin + stride - 1) / stride : 0;
  const int64_t n_mine = (n_tiles_mine + U - 1) / U;  // units
  // Every stage must belong to exactly one consumer warp, which uses it in order: an
  // mbarrier parity wait cannot tell phase n from phase n+2, so a stage shared by two
  // warps could let one of them run a phase ahead.  nact consumers, Se = multiple of nact.
  constexpr int CW = PAIRS == 4 ? 2 : 1;  // warps per consumer unit (a stage's owner)
  constexpr int NCU = NCW / CW;           // consumer units
  const int nact = S < NCU ? S : NCU;
  const int Se = S - S % nact;

  if constexpr (PAIRS == 3) {
    // Self-producing consumers (row-dot consumer, runtime flag): every consumer warp issues
    // the bulk copies of its OWN next tile into the stage it has just finished reading, so
    // there is no producer thread to serialise on (~100 ns per copy, in stage order: with one
    // stage per warp a warp that finishes out of order waits behind the producer's head of
    // line) and no `empty` barrier: the refill starts the moment the stage is quiescent.
    if (selfprod) {
      // mode 3: the (now idle) producer warp consumes as well: NCW + 1 consumer warps
      const bool all = selfprod == 3;
      if (!all && warp == 0) return;
      const int cw = all ? warp : warp - 1;
      const int nact = all ? (S < NCW + 1 ? S : NCW + 1) : (S < NCW ? S : NCW);
      const int Se = S - S % nact;
      if (cw >= nact) return;
      const int spw = Se / nact;  // stages per warp
      const uint64_t pol = l2_policy_evict_first();
      auto issue_one = [&](int64_t i, int s) {  // lane 0
        const int64_t tile = tile_begin + i * stride;
        mbar_arrive_expect_tx(&sm.full[s], tile_bytes + TR * uint32_t(sizeof(double)));
        const XT* src = X + tile * int64_t(tile_elems);
        if (evict_first) {
          bulk_g2s_hint(sm.xs + size_t(s) * tile_pitch, src, tile_bytes, &sm.full[s], pol);
        } else {
          bulk_g2s(sm.xs + size_t(s) * tile_pitch, src, tile_bytes, &sm.full[s]);
        }
        bulk_g2s(sm.ys + size_t(s) * TR, y + tile * TR, TR * uint32_t(sizeof(double)), &sm.full[s]);
      };
      if (lane == 0) {
        for (int m = 0; m < spw; ++m) {
          const int64_t i = cw + int64_t(m) * nact;
          if (i < n_mine) issue_one(i, cw + m * nact);
        }
      }
      int m = 0;        // stage slot of this warp
      uint32_t n = 0;   // use count of the slot
      for (int64_t i = cw; i < n_mine; i += nact) {
        const int s = cw + m * nact;
        mbar_wait(&sm.full[s], n & 1);
        consume_tile_rowdot<KC, GRAD>(reinterpret_cast<const float*>(sm.xs + size_t(s) * tile_pitch),
                                      sm.ys + size_t(s) * TR, K, lane, (tile_begin + i * stride) * TR, row_limit,
                                      sm.sbeta, g, nll_acc, nullptr);
        const int64_t nxt = i + int64_t(spw) * nact;  // the stage is quiescent: refill it
        if (lane == 0 && nxt < n_mine) issue_one(nxt, s);
        if (++m == spw) {
          m = 0;
          ++n;
        }
      }
      return;
    }
  }
#ifdef PM_AB_STREAM_SELFPROD  // A/B build only (-DPM_AB_STREAM_SELFPROD + tune stream_selfprod=1): compiled into
                              // the default library, the extra path cost the config-0 kernel ~1 us per launch
  if constexpr (MULTI) {
    // Self-producing column consumers (selfprod == 3: all NCW + 1 warps consume and issue the
    // bulk copies of their own units; narrow / small designs, where the single producer
    // thread's ~100 ns per copy delays the last warp's first data by more than a microsecond
    // and an eighth consumer shortens the per-warp chain of tiles).
    if (selfprod == 3) {
      const int cw = warp;
      const int nact = S < NCW + 1 ? S : NCW + 1;
      const int Se = S - S % nact;
      if (cw >= nact) return;
      const int spw = Se / nact;
      const uint64_t pol = l2_policy_evict_first();
      auto issue_unit = [&](int64_t i, int s) {  // lane 0
        const int64_t tile = tile_begin + i * U * stride;
        const int64_t left = n_tiles_mine - i * U;
        const uint32_t cnt = uint32_t(left < U ? left : U);
        mbar_arrive_expect_tx(&sm.full[s], cnt * (tile_bytes + TR * uint32_t(sizeof(double))));
        const XT* src = X + tile * int64_t(tile_elems);
        if (evict_first) {
          bulk_g2s_hint(sm.xs + size_t(s) * tile_pitch, src, cnt * tile_bytes, &sm.full[s], pol);
        } else {
          bulk_g2s(sm.xs + size_t(s) * tile_pitch, src, cnt * tile_bytes, &sm.full[s]);
        }
        bulk_g2s(sm.ys + size_t(s) * U * TR, y + tile * TR, cnt * TR * uint32_t(sizeof(double)), &sm.full[s]);
      };
      if (lane == 0) {
        for (int m = 0; m < spw; ++m) {
          const int64_t i = cw + int64_t(m) * nact;
          if (i < n_mine) issue_unit(i, cw + m * nact);
        }
      }
      int m = 0;
      uint32_t n = 0;
      for (int64_t i = cw; i < n_mine; i += nact) {
        const int s = cw + m * nact;
        mbar_wait(&sm.full[s], n & 1);
        const int64_t tile0 = tile_begin + i * U * stride;
        const int64_t left = n_tiles_mine - i * U;
        const int cnt = int(left < U ? left : U);
        const unsigned char* xstage = sm.xs + size_t(s) * tile_pitch;
        const double* ystage = sm.ys + size_t(s) * U * TR;
        const int64_t nxt = i + int64_t(spw) * nact;
        auto refill = [&]() {
          if (lane == 0 && nxt < n_mine) issue_unit(nxt, s);
        };
        for (int j = 0; j < cnt; ++j) {
          consume_tile<XT, KC, GRAD, R, TR>(reinterpret_cast<const XT*>(xstage + size_t(j) * tile_bytes),
                                            ystage + j * TR, K, lane, (tile0 + j) * TR, row_limit, breg, g, nll_acc,
                                            nullptr, RefillWhen<decltype(refill)>{j == cnt - 1, refill});
        }
        if (++m == spw) {
          m = 0;
          ++n;
        }
      }
      return;
    }
  }
#endif
  if (warp == 0) {
    const uint64_t pol = l2_policy_evict_first();
    int s = 0;        // stage = i % Se
    uint32_t n = 0;   // use count of the stage = i / Se
    int64_t tile = tile_begin;
    int64_t left = n_tiles_mine;
    auto issue = [&](int64_t i_end) {  // lane 0 only
      for (int64_t i = int64_t(n) * Se + s; i < i_end; ++i) {
        if (n > 0) mbar_wait(&sm.empty[s], (n - 1) & 1);
        const uint32_t cnt = uint32_t(left < U ? left : U);
        mbar_arrive_expect_tx(&sm.full[s], cnt * (tile_bytes + TR * uint32_t(sizeof(double))));
        const XT* src = X + tile * int64_t(tile_elems);
        if (evict_first) {
          bulk_g2s_hint(sm.xs + size_t(s) * tile_pitch, src, cnt * tile_bytes, &sm.full[s], pol);
        } else {
          bulk_g2s(sm.xs + size_t(s) * tile_pitch, src, cnt * tile_bytes, &sm.full[s]);
        }
        bulk_g2s(sm.ys + size_t(s) * U * TR, y + tile * TR, cnt * TR * uint32_t(sizeof(double)), &sm.full[s]);
        tile += U * stride;
        left -= U;
        if (++s == Se) {
          s = 0;
          ++n;
        }
      }
    };
    if (lane == 0) issue(n_mine);
    return;
  }
  const int cw = (warp - 1) / CW;
  [[maybe_unused]] const int sub = (warp - 1) % CW;
  if (cw >= nact) return;
  int s = cw;       // i % Se for i = cw + m*nact (Se is a multiple of nact)
  uint32_t n = 0;   // i / Se
  constexpr int RO = PAIRS == 2 ? 8 : (PAIRS == 1 ? R : 1);
  uint32_t roff[RO];  // pairs layouts: byte offset of slot r's row + this lane's pair
  if constexpr (PAIRS == 1 || PAIRS == 2) {
#pragma unroll
    for (int r = 0; r < RO; ++r) roff[r] = uint32_t(((r ^ (lane & (RO - 1))) * K + 2 * lane) * sizeof(XT));
  }
  for (int64_t i = cw; i < n_mine; i += nact) {
    mbar_wait(&sm.full[s], n & 1);
    const int64_t tile0 = tile_begin + i * U * stride;
    const int64_t left = n_tiles_mine - i * U;
    const int cnt = int(left < U ? left : U);
    const unsigned char* xstage = sm.xs + size_t(s) * tile_pitch;
    const double* ystage = sm.ys + size_t(s) * U * TR;
#ifdef PM_AB_NO_COMPUTE  // A/B timing experiment only: the TMA pipeline without the consumers' math
    {
      const double dep = ystage[lane];
      nll_acc += dep;
      mbar_arrive_after(&sm.empty[s], dep, lane, const_cast<unsigned char*>(xstage));
      s += nact;
      if (s >= Se) {
        s = cw;
        ++n;
      }
      continue;
    }
#endif
    if constexpr (!MULTI) {
      const int64_t row0 = tile0 * TR;
      if constexpr (PAIRS == 4) {
        // xch: the pair's exchange boxes live in the (still unused) per-warp gradient area
        consume_tile_rowdot2<KC, GRAD>(reinterpret_cast<const float*>(xstage), ystage, K, lane, sub, cw,
                                       uint32_t((i / nact) & 1), row0, row_limit, sm.sbeta, sm.wg, g, nll_acc,
                                       &sm.empty[s]);
      } else if constexpr (PAIRS == 3) {
        consume_tile_rowdot<KC, GRAD>(reinterpret_cast<const float*>(xstage), ystage, K, lane, row0, row_limit,
                                      sm.sbeta, g, nll_acc, &sm.empty[s]);
      } else if constexpr (PAIRS == 2) {
        consume_tile_f32full<KC, GRAD>(reinterpret_cast<const float*>(xstage), ystage, K, lane, row0, row_limit,
                                       breg, g, nll_acc, &sm.empty[s], roff);
      } else if constexpr (PAIRS == 1) {
        consume_tile_pairs<XT, KC, GRAD, R, TR>(reinterpret_cast<const XT*>(xstage), ystage, K, lane, row0,
                                                row_limit, breg, g, nll_acc, &sm.empty[s], roff);
      } else {
        consume_tile<XT, KC, GRAD, R, TR>(reinterpret_cast<const XT*>(xstage), ystage, K, lane, row0, row_limit,
                                          breg, g, nll_acc, &sm.empty[s]);
      }
    } else {
      for (int j = 0; j < cnt; ++j) {
        uint64_t* rel = (j == cnt - 1) ? &sm.empty[s] : nullptr;  // release with the unit's last tile
        consume_tile<XT, KC, GRAD, R, TR>(reinterpret_cast<const XT*>(xstage + size_t(j) * tile_bytes),
                                          ystage + j * TR, K, lane, (tile0 + j) * TR, row_limit, breg, g, nll_acc,
                                          rel);
      }
    }
    s += nact;
    if (s >= Se) {
      s = cw;
      ++n;
    }
  }
}

constexpr int kMaxXchgRanks = 16;

// Mailbox of the peer exchange (one per rank, device memory, IPC-shared):
//   data  [2][world][width] doubles (double-buffered by epoch parity: a rank can be at most one
//         evaluation ahead of the slowest reader, see pm_glm_eval_xchg)
//   flags [world] u64 = latest epoch rank r deposited here
__host__ __device__ inline size_t xchg_flags_offset(int world, int width) {
  return (size_t(2) * world * width * sizeof(double) + 127) / 128 * 128;
}
__host__ __device__ inline size_t xchg_bytes(int world, int width) {
  return xchg_flags_offset(world, width) + size_t(world) * sizeof(unsigned long long);
}

struct GlmArgs {
  const void* X;
  const double* y;
  int64_t n_rows;
  int64_t n_tiles;
  int K;
  int stages;
  int tps;                    // stream kernel: tiles per stage (1 = interleaved single tiles)
  int selfprod;               // row-dot consumer: consumer warps issue their own bulk copies
  int with_prior;
  int evict_first;
  const double* prior_mu;     // device [K]
  const double* prior_sigma;  // device [K]
  double* prior_terms;        // device [K+1] scratch: prior_precompute -> cta_reduce_finalize
  double* partials;           // [grid][K+1]
  unsigned int* counter;      // zero between launches
  double* out;                // [K+1]  (f, g)
  const double* beta_dev;     // wide kernel only
  // peer-memory exchange of row-sharded ranks (xw > 0; pm_glm_eval_xchg): the finishing CTA
  // deposits this rank's (K+1) partial into every rank's mailbox over NVLink, raises its flag
  // there, waits for all ranks' flags in its own mailbox and folds in ascending rank order
  int xw, xrank;
  int xphase;                 // 3: deposit + wait/fold (one launch); 1 / 2: one half only (split form)
  unsigned long long xepoch;  // >= 1, +1 per evaluation, identical on every rank
  double* xpeer[kMaxXchgRanks];  // mailbox base of every rank, mapped into this process
  unsigned* xstatus;          // local: set to 1 on a wait timeout
  // completion word (nullable): written with done_seq, system-scope release, after the
  // results -- pm_glm_wait polls it in mapped host memory instead of synchronising the stream
  unsigned long long* done;
  unsigned long long done_seq;
#ifdef PM_AB_PHASES  // A/B timing experiment only: %globaltimer stamps per CTA, 8 slots each
  unsigned long long* stamps;
#endif
};

__device__ __forceinline__ void ab_stamp(const GlmArgs& a, int slot, int tid = 0) {
#ifdef PM_AB_PHASES
  if (threadIdx.x == tid) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.stamps[blockIdx.x * 8 + slot] = t;
  }
#else
  (void)a;
  (void)slot;
#endif
}

// Peer exchange, second half (the finishing CTA only): publish this rank's deposits, wait for
// every rank's, fold them in ascending rank order (dist.ordered_sum / pm_fold_rows: identical
// bits on every rank).  Thread 0: one system-scope fence after the CTA barrier covers every
// thread's P2P stores (PTX fences are cumulative over writes ordered before them by
// bar.sync), then a release store of the epoch into each rank's flag slot; the acquire loads
// of the local flags order the peers' deposits before the fold's reads.  A rank that never
// arrives (dead peer) ends the wait after ~10 s with *xstatus = 1 and NaN results, instead of
// hanging the GPU.
// `flag`: a free shared int (the finisher's last-CTA flag; the kernels reserve all dynamic
// shared memory, so no static __shared__ here)
__device__ inline void xchg_finish(const GlmArgs& a, int ncols, int* flag) {
  const int width = a.K + 1;
  volatile int& timed_out = *flag;
  __syncthreads();
  if (threadIdx.x == 0) {
    timed_out = 0;
    const size_t fo = xchg_flags_offset(a.xw, width);
    if (a.xphase & 1) {
      asm volatile("fence.sc.sys;" ::: "memory");
      for (int p = 0; p < a.xw; ++p) {
        unsigned long long* f =
            reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(a.xpeer[p]) + fo) + a.xrank;
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(a.xepoch) : "memory");
      }
    }
    const unsigned long long* mine =
        reinterpret_cast<const unsigned long long*>(reinterpret_cast<const char*>(a.xpeer[a.xrank]) + fo);
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int r = 0; r < ((a.xphase & 2) ? a.xw : 0); ++r) {
      while (true) {
        unsigned long long e;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(e) : "l"(mine + r) : "memory");
        if (e >= a.xepoch) break;
        unsigned long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 10000000000ull) {
          timed_out = 1;
          *a.xstatus = 1u;
          break;
        }
        __nanosleep(64);
      }
      if (timed_out) break;
    }
  }
  __syncthreads();
  if (!(a.xphase & 2)) return;
  const double* data = a.xpeer[a.xrank] + size_t(a.xepoch & 1) * a.xw * width;
  for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
    double acc = __ldcv(data + c);
    for (int r = 1; r < a.xw; ++r) acc += __ldcv(data + size_t(r) * width + c);
    a.out[c] = timed_out ? __longlong_as_double(0x7ff8000000000000ll) : acc;
  }
}

// Prior terms of the log-posterior (sampler.py:55-58, constants dropped), computed by ONE warp
// of CTA 0 at the start of the launch, off the critical path (they depend only on beta, mu,
// sigma): terms[0] = sum_k -0.5 ((beta_k - mu_k) / sigma_k)^2 (lane-strided partials, then
// the fixed butterfly), terms[1+k] = (beta_k - mu_k) / sigma_k^2.  Ordered before CTA 0's
// release ticket in cta_reduce_finalize, so the finishing CTA (acquire) reads them from L2;
// in the tail they cost two loads instead of K dependent divisions (~2 us of a c0 launch).
template <class BetaAt>
__device__ __forceinline__ void prior_precompute_from(const GlmArgs& a, BetaAt beta_at, int lane) {
  double f = 0.0;
  for (int k = lane; k < a.K; k += 32) {
    const double mu = a.prior_mu[k], sg = a.prior_sigma[k];
    const double d = beta_at(k) - mu;
    const double z = d / sg;
    f += -0.5 * z * z;
    a.prior_terms[1 + k] = d / (sg * sg);
  }
  f = warp_sum(f);
  if (lane == 0) a.prior_terms[0] = f;
}
__device__ inline void prior_precompute(const GlmArgs& a, const double* sbeta, int lane) {
  prior_precompute_from(a, [sbeta](int k) { return sbeta[k]; }, lane);
}

// Deterministic cross-CTA finish: CTA partial -> partials[blockIdx]; the last CTA to
// arrive sums all partials in ascending CTA order (the reference's ascending-worker merge,
// glm.py:243-250), adds the prior (sampler.py:55-58) and writes (f, g).
template <int CU = 5>
__device__ inline void cta_reduce_finalize(const GlmArgs& a, const StreamSmem& sm, int nw, bool grad) {
  const int K = a.K;
  const int tid = threadIdx.x;
  __syncthreads();
  double* mine = a.partials + size_t(blockIdx.x) * (K + 1);
  for (int c = tid; c <= K; c += blockDim.x) {
    double acc = 0.0;
    if (c == 0) {
      for (int w = 0; w < nw; ++w) acc += sm.wf[w];
    } else if (grad) {
      for (int w = 0; w < nw; ++w) acc += sm.wg[size_t(w) * K + (c - 1)];
    }
    mine[c] = acc;
  }
#ifdef PM_AB_NO_FINALIZE  // A/B timing experiment only: CTA partials, no cross-CTA finish
  return;
#endif
  // One acq_rel ticket by thread 0 after the CTA barrier publishes the whole CTA's partial
  // (PTX fences are cumulative over writes ordered before them by bar.sync) and, in the last
  // CTA, acquires every other CTA's; replaces two per-thread __threadfence() (MEMBAR +
  // L1 invalidation), measured ~4 us of a c0 launch.
  __syncthreads();
  ab_stamp(a, 2);
  if (tid == 0) {
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(a.counter) : "memory");
    *sm.flag = (t == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  ab_stamp(a, 3);
  if (*sm.flag == 0) return;
  const int G = gridDim.x;
  const int lane = tid & 31, wid = tid >> 5, nwarps = blockDim.x >> 5;
  // Column totals in a fixed order, coalesced: lanes = 32 consecutive columns (one 256-byte
  // row segment of a CTA's partial per warp load, every fetched sector fully used), warps =
  // (column group, one of 4 chunks of consecutive CTAs).  A lane sums its chunk's CTAs in ascending
  // order with up to BU loads in flight (one L2 round trip for 148 CTAs split over >= 4
  // chunks), chunk sums go through shared memory and are added in ascending chunk order:
  // the reference's ascending-worker merge (glm.py:243-250), bracketed by chunk.
  // (r02 phase stamps: the previous lane-per-CTA form read 8 bytes of every 32-byte sector,
  // 6400 sector requests from one SM: 3.8-4.8 us at K = 32 on 148 CTAs.)
  constexpr int BU = CU >= 5 ? 40 : 20;
  constexpr int nchunk = 4;  // fixed: a column's summation order depends on the grid only (f of
                             // a GRAD=false launch is bit-identical to f of a GRAD=true one)
  const int ncols = grad ? K + 1 : 1;
  const int ncg = (ncols + 31) >> 5;
  double* scratch = (size_t(nw) * K >= size_t(nchunk) * ncols) ? sm.wg : reinterpret_cast<double*>(sm.xs);
  const double prior_c = (a.with_prior && tid < ncols) ? __ldcg(a.prior_terms + tid) : 0.0;  // in flight
  for (int item = wid; item < ncg * nchunk; item += nwarps) {
    const int cg = item / nchunk, chunk = item - cg * nchunk;
    const int b_lo = int(int64_t(G) * chunk / nchunk), b_hi = int(int64_t(G) * (chunk + 1) / nchunk);
    const int c = cg * 32 + lane;
    double acc = 0.0;
    for (int b0 = b_lo; b0 < b_hi; b0 += BU) {
      double v[BU];
#pragma unroll
      for (int i = 0; i < BU; ++i)
        v[i] = (b0 + i < b_hi && c < ncols) ? __ldcg(a.partials + size_t(b0 + i) * (K + 1) + c) : 0.0;
#pragma unroll
      for (int i = 0; i < BU; ++i)
        if (b0 + i < b_hi) acc += v[i];
    }
    if (c < ncols) scratch[size_t(chunk) * ncols + c] = acc;
  }
  ab_stamp(a, 5);
  __syncthreads();
  for (int c = tid; c < ncols; c += blockDim.x) {
    double tot = scratch[c];
    for (int ch = 1; ch < nchunk; ++ch) tot += scratch[size_t(ch) * ncols + c];
    // partials hold -sum(nll) = L and the gradient; + the prior terms of prior_precompute
    double v = tot;
    if (a.with_prior) {
      const double pr = c == tid ? prior_c : __ldcg(a.prior_terms + c);
      v = c == 0 ? tot + pr : tot - pr;
    }
    if (a.xw == 0) {
      a.out[c] = v;
    } else if (a.xphase & 1) {  // deposit into slot [parity][xrank] of every rank's mailbox (P2P stores)
      const size_t o = (size_t(a.xepoch & 1) * a.xw + a.xrank) * size_t(K + 1) + c;
      for (int p = 0; p < a.xw; ++p) a.xpeer[p][o] = v;
    }
  }
  ab_stamp(a, 6);
  if (tid == 0) *a.counter = 0u;  // re-arm for the next launch (kernel boundary orders it)
  if (a.done && a.xw == 0) {
    __syncthreads();  // every thread's result stores, then one system-scope fence + release store
    if (tid == 0) {
      asm volatile("fence.sc.sys;" ::: "memory");
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.done), "l"(a.done_seq) : "memory");
    }
  }
#ifdef PM_AB_PHASES
  __syncthreads();
  ab_stamp(a, 4);
#endif
  if (a.xw > 0) xchg_finish(a, ncols, sm.flag);
}

// K1 + K2: persistent fused single-pass kernel, one CTA per SM.
// R: rows per register sub-tile (SubRows default; smaller R frees registers for more warps)
// TR: rows per stage (32, or 16 so that 15 consumer warps can own 2 stages each)
// PAIRS: fp32-X consumer layouts -- 1: consume_tile_pairs, 2: consume_tile_f32full
template <typename XT, int KC, bool GRAD, int NCW, int R = SubRows<KC, GRAD>::value, int TR = kTileRows,
          int PAIRS = 0>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    glm_stream_kernel(GlmArgs a, BetaPack<KC> beta) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  ab_stamp(a, 0);
#ifdef PM_AB_EMPTY  // A/B timing experiment only: launch + exit of the same grid / smem footprint
  if (threadIdx.x == 0 && blockIdx.x == 0) a.out[0] = 0.0;
  return;
#endif
  const int K = a.K;
  const int S = a.stages;
  const int U = a.tps;  // tiles per stage (> 1: contiguous tile range per CTA, one copy per unit)
  const int nw = ((PAIRS == 3 || (PAIRS == 0 && NCW <= 8)) && a.selfprod == 3) ? NCW + 1 : NCW;  // warps holding a partial
  const StreamSmem sm = carve_stream_smem(smem_raw, K, sizeof(XT), S, nw, TR * U);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // Thread 0 initialises the mbarriers; the CTA barrier follows at once, so the producer's
  // first copies are in flight while the consumers fetch beta from the parameter bank (the
  // first touch misses the constant cache) and CTA 0 computes the prior terms.
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&sm.full[s], 1);
      mbar_init(&sm.empty[s], PAIRS == 4 ? 2 : 1);  // released by every warp of the owning unit
    }
    fence_mbar_init();
  }
  if constexpr (PAIRS >= 3) {  // the row-dot consumers read all of beta from shared memory
    for (int k = threadIdx.x; k < K; k += blockDim.x) sm.sbeta[k] = beta.v[k];
  }
  __syncthreads();
  ab_stamp(a, 1);
  double breg[KC], g[KC];
#pragma unroll
  for (int j = 0; j < KC; ++j) {
    const int c = lane_col<PAIRS != 0>(lane, j);
    breg[j] = ((warp > 0 || nw > NCW) && c < K) ? beta.v[c] * XScale<XT>::value : 0.0;  // exact (power of two)
    g[j] = 0.0;
  }
  if (blockIdx.x == 0 && a.with_prior && warp == NCW)
    prior_precompute_from(a, [&beta](int k) { return beta.v[k]; }, lane);
  double nll = 0.0;
  int64_t tb, te, stride;
  const int64_t nt = a.n_tiles * (kTileRows / TR);
  if (U > 1) {  // contiguous, near-equal tile ranges
    tb = nt * blockIdx.x / gridDim.x;
    te = nt * (blockIdx.x + 1) / gridDim.x;
    stride = 1;
  } else {  // tiles interleaved across the CTAs
    tb = blockIdx.x;
    te = nt;
    stride = gridDim.x;
  }
  stream_tiles<XT, KC, GRAD, NCW, R, TR, PAIRS>(static_cast<const XT*>(a.X), a.y, K, tb, te, stride, a.n_rows, S, sm,
                                                breg, g, nll, a.evict_first != 0, U, a.selfprod);
  if constexpr (PAIRS == 4) __syncthreads();  // the pairs' exchange boxes share sm.wg: all tiles done first
  if (warp > 0 || nw > NCW) {
    const int cw = nw > NCW ? warp : warp - 1;
    const double wsum = warp_sum(nll);
    if (lane == 0) sm.wf[cw] = -wsum;
    if (GRAD) {
#pragma unroll
      for (int j = 0; j < KC; ++j) {
        const int c = lane_col<PAIRS != 0>(lane, j);
        if (c < K) sm.wg[size_t(cw) * K + c] = g[j];
      }
    }
  }
  cta_reduce_finalize<(NCW > 8 ? 3 : 5)>(a, sm, nw, GRAD);
}

// Wide-K kernel (K > 256): one warp per row, lanes stride the columns, X read once from
// HBM (the gradient pass re-reads the row from L1), per-warp gradient accumulators in smem.
template <typename XT, bool GRAD>
__global__ void __launch_bounds__(256) glm_wide_kernel(GlmArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int K = a.K;
  const int nw = blockDim.x >> 5;
  StreamSmem sm = carve_stream_smem(smem_raw, K, sizeof(XT), 0, nw);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < K; k += blockDim.x) sm.sbeta[k] = a.beta_dev[k];
  double* ga = sm.wg + size_t(warp) * K;
  for (int k = lane; k < K; k += 32) ga[k] = 0.0;
  __syncthreads();
  if (blockIdx.x == 0 && a.with_prior && warp == nw - 1) prior_precompute(a, sm.sbeta, lane);
  const XT* X = static_cast<const XT*>(a.X);
  double nll = 0.0;
  const int64_t total_warps = int64_t(gridDim.x) * nw;
  for (int64_t row = int64_t(blockIdx.x) * nw + warp; row < a.n_rows; row += total_warps) {
    const XT* xr = X + row * K;
    double acc = 0.0;
    for (int k = lane; k < K; k += 32) acc = fma(ld_x(xr + k), sm.sbeta[k], acc);
    const double t = warp_sum(acc);
    double r_nll, w;
    row_terms(t, __ldg(a.y + row), r_nll, w);
    nll += r_nll;  // identical in every lane
    if (GRAD) {
      for (int k = lane; k < K; k += 32) ga[k] = fma(w, ld_x(xr + k), ga[k]);
    }
  }
  if (lane == 0) sm.wf[warp] = -nll;
  cta_reduce_finalize(a, sm, nw, GRAD);
}

}  // namespace pm
