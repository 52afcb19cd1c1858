// Red-black (checkerboard) Gibbs sweeps for Ising and q=4 Potts lattices.
//
// Reference semantics (ising.py):
//   colour c = (i+j)%2; packed index = scan order within the colour          ising.py:101-131
//   z = b + w * sum(neighbour spins), missing free-boundary neighbours = 0    ising.py:119-131,184
//   s = +1 iff u < expit(z), u pre-assigned by packed index                   ising.py:158-172,185
//   colour 0 against frozen colour 1, then colour 1                           ising.py:183-187
// The host builds exact probability tables with the reference's arithmetic, so the device does
// only integer neighbour sums and an exact compare (double compare, or the equivalent integer
// compare word < ceil(p * 2^32) on the packed fast path).
//
// Layouts in HBM:
//   W even : red-black packed, two int8 arrays [H][W/2]; colour c of row i sits at column
//            j = 2q + ((i+c)&1).  A half-sweep reads the other colour and writes its own.
//   W odd  : plain int8 grid [H][W] (colours are the parity of the flat index).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "philox.cuh"
#include "pm_internal.cuh"

using namespace pm;

namespace {

bool pdl_default() { return tune("pdl", 1) != 0; }

// Resident CTAs per SM the packed kernel is register-budgeted for (NG >= 2): Ising 4
// (64 registers), Potts 3 (80 registers, no spills): profiles/r01_ab_gibbs_minb.txt
#ifndef PM_GIBBS_MINB_ISING
#define PM_GIBBS_MINB_ISING 4
#endif
#ifndef PM_GIBBS_MINB_POTTS
#define PM_GIBBS_MINB_POTTS 3
#endif

constexpr int kPottsIdx = 625;  // n0 + 5 n1 + 25 n2 + 125 n3, n_a in 0..4
// Packed fast path: a neighbour in state a contributes code {0, 1, 5, 21}[a]; the 35
// neighbour multisets (n0 + n1 + n2 + n3 = 4) have distinct code sums n1 + 5 n2 + 21 n3 <= 84,
// so one byte per site indexes an 85-entry threshold table.
constexpr int kPottsCodes = 85;
constexpr uint32_t kPottsCodeBytes = 0x15050100u;  // bytes {0, 1, 5, 21}

// Packed colour arrays store an encoding of each site's value so that the packed kernel's
// neighbour statistic is a plain byte-wise sum of 4 words (no masks, no per-byte lookups):
//   enc 1 (Ising): e = 1 - s (0x00 for +1, 0x02 for -1): the sum is 2 x (number of -1's);
//   enc 2 (Potts q=4): e = {0, 1, 5, 21}[state], the compact code (kPottsCodeBytes).
// pack/unpack and LatView convert; unpacked grids (odd W) are stored as is (enc 0).
// (branch-free: a select chain here compiled to a slow per-byte lookup in pack/unpack)
__host__ __device__ __forceinline__ int8_t enc_site(int8_t v, int enc) {
  const int code = int((kPottsCodeBytes >> (8 * (v & 3))) & 0xFFu);
  return enc == 1 ? int8_t(1 - v) : enc == 2 ? int8_t(code) : v;
}
__host__ __device__ __forceinline__ int8_t dec_site(int8_t e, int enc) {
  const int state = int(e > 0) + int(e > 1) + int(e > 5);
  return enc == 1 ? int8_t(1 - e) : enc == 2 ? int8_t(state) : e;
}

struct LatView {
  int8_t* pk0;  // packed colour 0  (W even) or grid (W odd)
  int8_t* pk1;  // packed colour 1  (W even)
  int H, W, W2;
  int packed;

  int enc;     // packed byte encoding (enc_site / dec_site)

  __device__ __forceinline__ int8_t get(int i, int j) const {
    if (packed) {
      const int8_t v = ((i + j) & 1 ? pk1 : pk0)[int64_t(i) * W2 + (j >> 1)];
      return dec_site(v, enc);
    }
    return pk0[int64_t(i) * W + j];
  }
  __device__ __forceinline__ void set(int i, int j, int8_t v) const {
    if (packed)
      ((i + j) & 1 ? pk1 : pk0)[int64_t(i) * W2 + (j >> 1)] = enc_site(v, enc);
    else
      pk0[int64_t(i) * W + j] = v;
  }
};

struct GenericArgs {
  LatView lat;
  int periodic;
  int model;            // PM_MODEL_*
  int rng;              // PM_RNG_*
  int colour;
  int64_t n0;           // ceil(HW/2): sites of colour 0
  int64_t n_c;          // sites of this colour
  const int32_t* cls;   // [H*W] class per site, or null (class 0)
  const double* ptab;   // Ising: [n_class][9] P(+1) for nsum = -4..4
  const double* cdf;    // Potts: [625][3]
  uint64_t key0, key1;
  uint64_t base;        // numpy: stream index of this half-sweep's first deviate
  uint64_t sweep;       // philox4x32: sweep number
  const double* uni;    // uniforms of this half-sweep (n_c), PM_RNG_UNIFORMS
  // optional diagnostics (gibbs_sweep_diff / denoise, ising.py:232-290)
  unsigned long long* flips;  // += number of sites whose value changed (integer atomics: exact)
  int32_t* acc;               // [H*W] row-major running sum of the new values, or null
};

__device__ __forceinline__ double uniform_for(const GenericArgs& a, int64_t p) {
  if (a.rng == PM_RNG_UNIFORMS) return a.uni[p];
  if (a.rng == PM_RNG_NUMPY_PHILOX) {
    const uint64_t w = numpy_philox_word(a.base + uint64_t(p), a.key0, a.key1);
    return double(w >> 11) * 0x1p-53;
  }
  const uint64_t s = uint64_t(a.colour) * uint64_t(a.n0) + uint64_t(p);
  const U32x4 blk = site_philox_block(s >> 2, a.sweep, a.key0);
  return double(blk.v[s & 3]) * 0x1p-32;
}

// One thread per site of colour c, any shape / boundary / model / RNG mode.
__global__ void __launch_bounds__(256) gibbs_generic_kernel(GenericArgs a) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int H = a.lat.H, W = a.lat.W;
  unsigned int nflip = 0;
  for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < a.n_c; p += stride) {
    int i, j;
    if ((W & 1) == 0) {
      const int W2 = W >> 1;
      i = int(p / W2);
      j = 2 * int(p % W2) + ((i + a.colour) & 1);
    } else {
      const int64_t f = 2 * p + a.colour;
      i = int(f / W);
      j = int(f % W);
    }
    const int di[4] = {-1, 1, 0, 0};
    const int dj[4] = {0, 0, -1, 1};
    int nsum = 0, pidx = 0;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      int ni = i + di[d], nj = j + dj[d];
      if (a.periodic) {
        ni = (ni + H) % H;
        nj = (nj + W) % W;
      } else if (ni < 0 || ni >= H || nj < 0 || nj >= W) {
        continue;  // free boundary: sentinel 0 (ising.py:121-131)
      }
      const int v = a.lat.get(ni, nj);
      if (a.model == PM_MODEL_ISING) {
        nsum += v;
      } else {
        pidx += (v == 0) ? 1 : (v == 1) ? 5 : (v == 2) ? 25 : 125;
      }
    }
    const double u = uniform_for(a, p);
    int8_t ns;
    if (a.model == PM_MODEL_ISING) {
      const int cl = a.cls ? a.cls[int64_t(i) * W + j] : 0;
      const double pp = a.ptab[cl * 9 + nsum + 4];
      ns = (u < pp) ? int8_t(1) : int8_t(-1);
    } else {
      const double* c3 = a.cdf + pidx * 3;
      ns = int8_t((u >= c3[0]) + (u >= c3[1]) + (u >= c3[2]));
    }
    if (a.flips) nflip += (a.lat.get(i, j) != ns) ? 1u : 0u;
    if (a.acc) a.acc[int64_t(i) * W + j] += ns;
    a.lat.set(i, j, ns);
  }
  if (a.flips) {
    for (int s = 16; s >= 1; s >>= 1) nflip += __shfl_xor_sync(0xffffffffu, nflip, s);
    if ((threadIdx.x & 31) == 0 && nflip) atomicAdd(a.flips, (unsigned long long)nflip);
  }
}

// ---------------------------------------------------------------- packed fast path
// Periodic, even H and W, W/2 % 16 == 0, uniform bias, Philox4x32 (seed, sweep, site).
// Thread = 16 consecutive packed sites of one row: 3 x 16-byte loads of the other colour
// (rows i-1, i, i+1) + 2 edge bytes, 4 Philox4x32 blocks, one 16-byte store.
struct PackedArgs {
  const int8_t* other;
  int8_t* mine;
  int H, W2;                  // global lattice height, packed width
  int colour;
  int64_t n0;                 // global sites of colour 0
  uint64_t sweep;
  uint64_t seed;
  Philox32Keys rk;            // key schedule of seed (host-computed)
  unsigned long long thr[9];  // Ising: ceil(P(+1 | nsum) * 2^32), nsum = -4..4
  // strip decomposition: own rows are global rows row0 .. row0+rows-1, stored at array rows
  // halo .. halo+rows-1; with halo = 1 the arrays carry one halo row above and below
  // (filled by the caller's exchange) and there is no vertical wrap inside the strip.
  int row0, rows, halo;
  // peer-memory halo exchange (xmb != null; pm_lat_strip_xchg_*): this strip's mailbox and
  // its up / down neighbours' mailboxes (CUDA IPC or same-process pointers).  The halo rows
  // of the colour read here come from xmb (parity rpar), waiting for flag >= kread; the own
  // first / last rows computed here are also stored into the up neighbour's DOWN halo / the
  // down neighbour's UP halo (parity wpar), and the last CTA raises their flags to kwrite.
  int8_t* xmb;
  int8_t* xup;
  int8_t* xdown;
  int rpar, wpar;
  unsigned long long kread, kwrite;
  unsigned* ticket;
  unsigned* status;
};

// Strip mailbox: halos [parity 2][colour 2][side 2: 0 = row above the strip, 1 = row below]
// [W2] bytes, then flags [colour 2][side 2] u64 = latest deposit number in that halo.
__host__ __device__ inline size_t lat_xchg_halo(int par, int colour, int side, int W2) {
  return (size_t(par) * 4 + colour * 2 + side) * W2;
}
__host__ __device__ inline size_t lat_xchg_flags(int W2) { return (size_t(8) * W2 + 127) / 128 * 128; }
__host__ __device__ inline size_t lat_xchg_bytes(int W2) { return lat_xchg_flags(W2) + 4 * sizeof(unsigned long long); }

// wait (acquire, system scope) until *flag >= k; ~10 s then *status = 1
__device__ inline void lat_wait_flag(const unsigned long long* flag, unsigned long long k, unsigned* status) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned long long e;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(e) : "l"(flag) : "memory");
    if (e >= k) return;
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 10000000000ull) {
      *status = 1u;
      return;
    }
    __nanosleep(100);
  }
}

__device__ __forceinline__ uint4 ld16(const int8_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

__device__ __forceinline__ uint32_t w_of(const uint4& v, int m) {
  return m == 0 ? v.x : m == 1 ? v.y : m == 2 ? v.z : v.w;
}



__device__ __forceinline__ uint32_t lane_id() {
  uint32_t l;
  asm("mov.u32 %0, %%laneid;" : "=r"(l));
  return l;
}

// prmt.b32 without __byte_perm's selector masking (selector nibbles here are 0..7)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}


// Threshold tables in shared memory.  T32: every threshold ceil(p*2^32) is < 2^32 (checked on
// the host), so the exact test u < p is the 32-bit compare word < T; otherwise 64-bit.
template <int MODEL, bool T32>
struct GibbsTables {
  // Ising: by number of -1 neighbours nd = 0..4 (nsum = 4 - 2 nd)
  // Potts T32: by the compact code sum e (0..84), threshold a of entry e replicated per lane at
  //   word (3e + a) * 32 + lane, so every lane reads its own bank (random e, no conflicts)
  // Potts 64-bit: by the compact code sum e, entry 3e + a (no lane replication: rare path)
#ifdef PM_AB_GIBBS_BORROW
  using IsingT = unsigned long long;  // 2^64 - T
#else
  using IsingT = typename std::conditional<T32, uint32_t, unsigned long long>::type;
#endif
  typename std::conditional<MODEL == PM_MODEL_ISING, IsingT[8],
                            typename std::conditional<T32, uint32_t[kPottsCodes * 3 * 32],
                                                      unsigned long long[kPottsCodes * 3]>::type>::type t;
};

// Thread = NG consecutive 16-site groups of one packed row (setup amortised over 16*NG sites).
// sm != null (STAGE): the other colour's rows r-1, r, r+1 come from the CTA's shared-memory
// stage (sm = this thread's first byte of row r there, rows `pitch` bytes apart, >= 16
// staged bytes on either side for the edge neighbours) instead of three L2 loads each.
template <int MODEL, bool T32, int NG, bool XCHG>
__device__ __forceinline__ void gibbs_packed_row(const PackedArgs& a, const GibbsTables<MODEL, T32>& tb, int r,
                                                 int q0, const int8_t* sm = nullptr, int pitch = 0);

__device__ inline void lat_xchg_publish(const PackedArgs& a);

// XCHG: the strip peer-memory halo exchange (PackedArgs xmb ...) is compiled in.
// STAGE (A/B, tune gibbs_smem=1; periodic whole lattices only): each CTA covers blockDim.y
// rows and stages the other colour's rows above / below / inside (+ 16 edge bytes either
// side) in shared memory once, so every row is read from L2 (blockDim.y + 2) / blockDim.y
// times instead of 3 -- the north-star's neighbour-sum staging.
template <int MODEL, bool T32, int NG, int RPT>
__device__ __forceinline__ void gibbs_packed_rows(const PackedArgs& a, const GibbsTables<MODEL, T32>& tb, int r0,
                                                  int q0);

// RPT: consecutive rows per thread (gibbs_packed_rows; 1 = one row per thread, the only form
// of the peer-exchanging and staged kernels)
template <int MODEL, bool T32, int NG, bool XCHG, bool STAGE = false, int RPT = 1>
__global__ void __launch_bounds__(256, NG == 1 ? 6 : MODEL == PM_MODEL_ISING ? PM_GIBBS_MINB_ISING : PM_GIBBS_MINB_POTTS)
    gibbs_packed_kernel(PackedArgs a, const unsigned long long* __restrict__ pthr, const uint32_t* __restrict__ pcomp) {
  __shared__ GibbsTables<MODEL, T32> tb;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if constexpr (MODEL == PM_MODEL_ISING) {
    // static indices into the parameter array (a dynamic index would copy the params to local memory)
    if (tid == 0) {
#pragma unroll
#ifdef PM_AB_GIBBS_BORROW
      for (int k = 0; k < 5; ++k) tb.t[k] = 0ull - a.thr[8 - 2 * k];
#else
      for (int k = 0; k < 5; ++k) tb.t[k] = a.thr[8 - 2 * k];
#endif
    }
  } else if constexpr (T32) {
    // replicate the compact table (85 x 3 words) across the 32 lanes: 4 lanes per 16-byte store
    uint4* dst = reinterpret_cast<uint4*>(&tb.t[0]);
    for (int t = tid; t < kPottsCodes * 3 * 8; t += blockDim.x * blockDim.y) {
      const uint32_t v = __ldg(pcomp + (t >> 3));
      dst[t] = make_uint4(v, v, v, v);
    }
  } else {
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(&tb.t[0]);
    for (int t = tid; t < kPottsCodes * 3; t += blockDim.x * blockDim.y) dst[t] = pthr[t];
  }
  __syncthreads();
  // PDL: the tables above are host-built (memcpy); the lattice is written by the previous
  // half-sweep, so wait for it here -- the launch and block scheduling overlap its tail
  pdl_trigger();
  pdl_wait();
  // 2-D grid of 2-D blocks: x = (16*NG)-site column groups of a row, y = rows
  const int per_row = a.W2 / (16 * NG);
  const int cgrp = blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (STAGE) {
    extern __shared__ __align__(16) int8_t stage[];
    const int span = blockDim.x * 16 * NG;  // packed bytes of a row covered by the CTA
    const int pitch = span + 32;
    const int nchunk = pitch / 16, nrow = blockDim.y + 2;
    const int cbase = blockIdx.x * span;
    const int nthr = blockDim.x * blockDim.y;
    for (int rb = blockIdx.y * blockDim.y; rb < a.rows; rb += gridDim.y * blockDim.y) {
      for (int t = tid; t < nrow * nchunk; t += nthr) {
        const int rr = t / nchunk, cc = t - rr * nchunk;
        int gr = rb - 1 + rr;
        gr = gr < 0 ? gr + a.rows : (gr >= a.rows ? gr - a.rows : gr);
        int gc = cbase - 16 + cc * 16;
        gc = gc < 0 ? gc + a.W2 : (gc >= a.W2 ? gc - a.W2 : gc);
        *reinterpret_cast<uint4*>(stage + rr * pitch + cc * 16) = ld16(a.other + int64_t(gr) * a.W2 + gc);
      }
      __syncthreads();
      const int r = rb + threadIdx.y;
      if (r < a.rows && cgrp < per_row)
        gibbs_packed_row<MODEL, T32, NG, XCHG>(a, tb, r, cgrp * 16 * NG,
                                               stage + (threadIdx.y + 1) * pitch + 16 + threadIdx.x * 16 * NG, pitch);
      __syncthreads();
    }
  } else if (cgrp < per_row) {
    if constexpr (RPT > 1 && !XCHG) {
      for (int rg = blockIdx.y * blockDim.y + threadIdx.y; rg * RPT < a.rows; rg += gridDim.y * blockDim.y)
        gibbs_packed_rows<MODEL, T32, NG, RPT>(a, tb, rg * RPT, cgrp * 16 * NG);
    } else {
      for (int r = blockIdx.y * blockDim.y + threadIdx.y; r < a.rows; r += gridDim.y * blockDim.y) {
        gibbs_packed_row<MODEL, T32, NG, XCHG>(a, tb, r, cgrp * 16 * NG);
      }
    }
  }
  if constexpr (XCHG) lat_xchg_publish(a);
}

// New packed words of one row chunk: U / D / M = the other colour's rows above / below / at the
// row, `edge` the one byte beyond the chunk on the side given by o, g0 the chunk's first
// Philox block.
template <int MODEL, bool T32, int NG>
__device__ __forceinline__ void gibbs_packed_words(const PackedArgs& a, const GibbsTables<MODEL, T32>& tb,
                                                   const uint32_t (&U)[4 * NG], const uint32_t (&D)[4 * NG],
                                                   const uint32_t (&M)[4 * NG], uint32_t edge, int o, uint32_t g0,
                                                   uint32_t (&res)[4 * NG]) {
  constexpr int NW = 4 * NG;
#pragma unroll
  for (int m = 0; m < NW; ++m) {
    const uint32_t cur = M[m];
    // byte b of `sh` = the other horizontal neighbour of site 4m+b (funnel shift across words)
    const uint32_t sh = o == 0 ? __funnelshift_l(m == 0 ? (edge << 24) : M[m - 1], cur, 8)
                               : __funnelshift_r(cur, m == NW - 1 ? edge : M[m + 1], 8);
    const U32x4 blk = site_philox_block_rk(g0 + uint32_t(m), a.sweep, a.rk);
    uint32_t out = 0;
    if constexpr (MODEL == PM_MODEL_ISING) {
      // packed bytes are 1 - s (0x02 for -1, 0x00 for +1), so the plain 4-way byte sum is
      // 2 x (number of -1 neighbours) <= 8 per byte (no carries, no masks); scaled to the
      // table's byte offset (x4 for u32 thresholds, x8 for u64) it is the LDS address offset
#ifdef PM_AB_GIBBS_BORROW
      // A/B build only: the compare on the FMA pipe.  tb.t holds 2^64 - T per entry (8 bytes);
      // word + (2^64 - T) as one IMAD.WIDE: the high word is all ones iff word < T.  One
      // IMAD.WIDE + one LOP3 per site instead of ISETP + a predicated add (both ALU).
      const uint32_t off = (U[m] + D[m] + cur + sh) << 2;
      const char* tbase = reinterpret_cast<const char*>(&tb.t[0]);
      uint32_t plus_bits = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t o = __byte_perm(off, 0u, 0x4440u + b);
        const unsigned long long neg = *reinterpret_cast<const unsigned long long*>(tbase + o);
        unsigned long long w;
        asm("mad.wide.u32 %0, %1, 1, %2;" : "=l"(w) : "r"(blk.v[b]), "l"(neg));
        plus_bits |= uint32_t(w >> 32) & (1u << (8 * b));
      }
      out = 0x02020202u - 2u * plus_bits;
#else
      constexpr int SH = T32 ? 1 : 2;
      const uint32_t off = (U[m] + D[m] + cur + sh) << SH;
      const char* tbase = reinterpret_cast<const char*>(&tb.t[0]);
      uint32_t plus_bits = 0;  // bit 8b set <=> site b becomes +1
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t o = __byte_perm(off, 0u, 0x4440u + b);
        bool plus;
        if constexpr (T32) {
          plus = blk.v[b] < *reinterpret_cast<const uint32_t*>(tbase + o);
        } else {
          plus = uint64_t(blk.v[b]) < *reinterpret_cast<const unsigned long long*>(tbase + o);
        }
        plus_bits |= plus ? (1u << (8 * b)) : 0u;
      }
      out = 0x02020202u - 2u * plus_bits;  // per byte: 0x00 (+1) or 0x02 (-1), no borrows
#endif
    } else {
      if constexpr (T32) {
        // packed bytes hold the codes already (enc 2): code sums <= 84 per byte, no carries
        const uint32_t e4 = U[m] + D[m] + cur + sh;
        const uint32_t* lt = &tb.t[0] + lane_id();
        uint32_t st[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint32_t* t3 = lt + prmt(e4, 0u, 0x4440u + b) * 96;
          const uint32_t w = blk.v[b];
          st[b] = uint32_t(w >= t3[0]) + uint32_t(w >= t3[32]) + uint32_t(w >= t3[64]);
        }
        // new states as PRMT selector nibbles, then their codes in one lookup
        out = prmt(kPottsCodeBytes, 0u, st[0] | (st[1] << 4) | (st[2] << 8) | (st[3] << 12));
      } else {
        const uint32_t e4 = U[m] + D[m] + cur + sh;  // code sums, as in the 32-bit path
        const unsigned long long* tt = reinterpret_cast<const unsigned long long*>(&tb.t[0]);
        uint32_t st[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const unsigned long long* t3 = tt + prmt(e4, 0u, 0x4440u + b) * 3;
          const uint64_t w = blk.v[b];
          st[b] = uint32_t(w >= t3[0]) + uint32_t(w >= t3[1]) + uint32_t(w >= t3[2]);
        }
        out = prmt(kPottsCodeBytes, 0u, st[0] | (st[1] << 4) | (st[2] << 8) | (st[3] << 12));
      }
    }
    res[m] = out;
  }
}

// RPT consecutive rows of one column group per thread (whole lattices and NCCL-exchanged
// strips; the peer-exchanging and staged forms keep one row per thread): row r + 1's rows
// above / at are row r's rows at / below, so each further row costs ONE new 16-byte load per
// group instead of three, and the per-thread set-up (parameters, addresses, table base) is
// paid once per RPT rows.
template <int MODEL, bool T32, int NG, int RPT>
__device__ __forceinline__ void gibbs_packed_rows(const PackedArgs& a, const GibbsTables<MODEL, T32>& tb, int r0,
                                                  int q0) {
  constexpr int NW = 4 * NG;
  auto load_row = [&](int arow, uint32_t (&w)[NW]) {
    const int8_t* p = a.other + int64_t(arow) * a.W2 + q0;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      const uint4 v = ld16(p + 16 * g);
      w[4 * g] = v.x, w[4 * g + 1] = v.y, w[4 * g + 2] = v.z, w[4 * g + 3] = v.w;
    }
  };
  const int li0 = r0 + a.halo;
  const int iu0 = a.halo ? li0 - 1 : (li0 == 0 ? a.rows - 1 : li0 - 1);
  uint32_t U[NW], M[NW], D[NW];
  load_row(iu0, U);
  load_row(li0, M);
  // not unrolled: a fully unrolled RPT = 4 body needs more than the 64 (Ising) / 80 (Potts)
  // registers of the occupancy these kernels run at (152 / 296 bytes of spills); rolled, the
  // window advances by 2 x NW register moves per row
#pragma unroll 1
  for (int j = 0; j < RPT; ++j) {
    const int r = r0 + j;
    if (r >= a.rows) break;
    const int li = r + a.halo;
    const int i = a.row0 + r;
    const int id = a.halo ? li + 1 : (li == a.rows - 1 ? 0 : li + 1);
    load_row(id, D);
    const int o = (i + a.colour) & 1;
    const int qe = o ? ((q0 + 16 * NG == a.W2) ? 0 : q0 + 16 * NG) : ((q0 == 0) ? a.W2 - 1 : q0 - 1);
    const uint32_t edge = uint32_t(uint8_t(__ldg(a.other + int64_t(li) * a.W2 + qe)));
    const uint32_t g0 = uint32_t((uint64_t(a.colour) * uint64_t(a.n0) + uint64_t(i) * a.W2 + q0) >> 2);
    uint32_t res[NW];
    gibbs_packed_words<MODEL, T32, NG>(a, tb, U, D, M, edge, o, g0, res);
#pragma unroll
    for (int g = 0; g < NG; ++g)
      *reinterpret_cast<uint4*>(a.mine + int64_t(li) * a.W2 + q0 + 16 * g) =
          make_uint4(res[4 * g], res[4 * g + 1], res[4 * g + 2], res[4 * g + 3]);
#pragma unroll
    for (int m = 0; m < NW; ++m) {  // next row: above = this row, at = the row below
      U[m] = M[m];
      M[m] = D[m];
    }
  }
}

template <int MODEL, bool T32, int NG, bool XCHG>
__device__ __forceinline__ void gibbs_packed_row(const PackedArgs& a, const GibbsTables<MODEL, T32>& tb, int r,
                                                 int q0, const int8_t* sm, int pitch) {
  constexpr int NW = 4 * NG;   // 32-bit words (4 sites each) handled by this thread
  const int li = r + a.halo;   // array row
  const int i = a.row0 + r;    // global row: colour parity and RNG site index
  const int iu = a.halo ? li - 1 : (li == 0 ? a.rows - 1 : li - 1);
  const int id = a.halo ? li + 1 : (li == a.rows - 1 ? 0 : li + 1);
  const int8_t* orow = a.other + int64_t(li) * a.W2;
  const int8_t* urow = a.other + int64_t(iu) * a.W2;
  const int8_t* drow = a.other + int64_t(id) * a.W2;
  if constexpr (XCHG) {  // halo rows of the other colour from the mailbox, once the neighbours delivered
    const int oc = a.colour ^ 1;
    const unsigned long long* fl = reinterpret_cast<const unsigned long long*>(a.xmb + lat_xchg_flags(a.W2));
    if (r == 0) {
      lat_wait_flag(fl + oc * 2 + 0, a.kread, a.status);
      urow = a.xmb + lat_xchg_halo(a.rpar, oc, 0, a.W2);
    }
    if (r == a.rows - 1) {
      lat_wait_flag(fl + oc * 2 + 1, a.kread, a.status);
      drow = a.xmb + lat_xchg_halo(a.rpar, oc, 1, a.W2);
    }
  }
  uint32_t U[NW], D[NW], M[NW];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    uint4 u4, d4, m4;
    if (sm) {
      u4 = *reinterpret_cast<const uint4*>(sm - pitch + 16 * g);
      d4 = *reinterpret_cast<const uint4*>(sm + pitch + 16 * g);
      m4 = *reinterpret_cast<const uint4*>(sm + 16 * g);
    } else {
      u4 = ld16(urow + q0 + 16 * g), d4 = ld16(drow + q0 + 16 * g), m4 = ld16(orow + q0 + 16 * g);
    }
    U[4 * g] = u4.x, U[4 * g + 1] = u4.y, U[4 * g + 2] = u4.z, U[4 * g + 3] = u4.w;
    D[4 * g] = d4.x, D[4 * g + 1] = d4.y, D[4 * g + 2] = d4.z, D[4 * g + 3] = d4.w;
    M[4 * g] = m4.x, M[4 * g + 1] = m4.y, M[4 * g + 2] = m4.z, M[4 * g + 3] = m4.w;
  }
  // o = 0: horizontal neighbours of packed site q are q-1 and q; o = 1: q and q+1
  const int o = (i + a.colour) & 1;
  const int qe = o ? ((q0 + 16 * NG == a.W2) ? 0 : q0 + 16 * NG) : ((q0 == 0) ? a.W2 - 1 : q0 - 1);
  const uint32_t edge = sm ? uint32_t(uint8_t(o ? sm[16 * NG] : sm[-1])) : uint32_t(uint8_t(__ldg(orow + qe)));
  // Philox block of the first word.  The packed path only runs on lattices with fewer than
  // 2^34 - 256 sites (packed_blocks_fit), so every block index of the half-sweep fits 32 bits:
  // the counter's high word is 0 and g0 + m is a 32-bit add (no carry chain per word)
  const uint32_t g0 = uint32_t((uint64_t(a.colour) * uint64_t(a.n0) + uint64_t(i) * a.W2 + q0) >> 2);
  uint32_t res[NW];
  gibbs_packed_words<MODEL, T32, NG>(a, tb, U, D, M, edge, o, g0, res);
#pragma unroll
  for (int g = 0; g < NG; ++g)
    *reinterpret_cast<uint4*>(a.mine + int64_t(li) * a.W2 + q0 + 16 * g) =
        make_uint4(res[4 * g], res[4 * g + 1], res[4 * g + 2], res[4 * g + 3]);
  if constexpr (XCHG) {  // own boundary rows into the neighbours' halos (P2P stores over NVLink)
    if (r == 0) {
#pragma unroll
      for (int g = 0; g < NG; ++g)
        *reinterpret_cast<uint4*>(a.xup + lat_xchg_halo(a.wpar, a.colour, 1, a.W2) + q0 + 16 * g) =
            make_uint4(res[4 * g], res[4 * g + 1], res[4 * g + 2], res[4 * g + 3]);
    }
    if (r == a.rows - 1) {
#pragma unroll
      for (int g = 0; g < NG; ++g)
        *reinterpret_cast<uint4*>(a.xdown + lat_xchg_halo(a.wpar, a.colour, 0, a.W2) + q0 + 16 * g) =
            make_uint4(res[4 * g], res[4 * g + 1], res[4 * g + 2], res[4 * g + 3]);
    }
  }
}

// Completion of a peer-exchanging half-sweep: the last CTA (acq_rel ticket after a CTA
// barrier and a system-scope fence covering the CTA's P2P stores) raises the neighbours'
// flags for this colour: up neighbour's "row below" flag, down neighbour's "row above" flag.
__device__ inline void lat_xchg_publish(const PackedArgs& a) {
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    asm volatile("fence.sc.sys;" ::: "memory");
    unsigned t;
    asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(a.ticket) : "memory");
    last = (t == gridDim.x * gridDim.y - 1) ? 1 : 0;
    if (last) {
      *a.ticket = 0u;  // re-arm (kernel boundary orders it)
      asm volatile("fence.sc.sys;" ::: "memory");
      unsigned long long* fu = reinterpret_cast<unsigned long long*>(a.xup + lat_xchg_flags(a.W2)) + a.colour * 2 + 1;
      unsigned long long* fd = reinterpret_cast<unsigned long long*>(a.xdown + lat_xchg_flags(a.W2)) + a.colour * 2 + 0;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fu), "l"(a.kwrite) : "memory");
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fd), "l"(a.kwrite) : "memory");
    }
  }
}

// ---------------------------------------------------------------- layout conversion
// grid [H][W] <-> packed colour arrays.  par0 = global row of grid row 0 (colour parity),
// aoff = array row of grid row 0 (1 for strips, whose arrays start with a halo row).
// One thread per (row, pair of columns): the two sites of a pair have opposite colours, so
// the thread moves one byte to each colour array (no 64-bit division per site).
__global__ void pack_kernel(const int8_t* __restrict__ grid, int H, int W, int8_t* pk0, int8_t* pk1, int par0,
                            int aoff, int enc) {
  const int W2 = W >> 1;
  const int64_t n = int64_t(H) * W2;
  for (int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < n; f += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(f / W2), q = int(f - int64_t(i) * W2);
    const char2 v = reinterpret_cast<const char2*>(grid + int64_t(i) * W)[q];
    const int8_t* src = reinterpret_cast<const int8_t*>(&v);
    const int c0 = (par0 + i) & 1;  // colour of column 2q
    const int64_t o = int64_t(i + aoff) * W2 + q;
    (c0 ? pk1 : pk0)[o] = enc_site(src[0], enc);
    (c0 ? pk0 : pk1)[o] = enc_site(src[1], enc);
  }
}
__global__ void unpack_kernel(int8_t* __restrict__ grid, int H, int W, const int8_t* pk0, const int8_t* pk1,
                              int par0, int aoff, int enc) {
  const int W2 = W >> 1;
  const int64_t n = int64_t(H) * W2;
  for (int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < n; f += int64_t(gridDim.x) * blockDim.x) {
    const int i = int(f / W2), q = int(f - int64_t(i) * W2);
    const int c0 = (par0 + i) & 1;
    const int64_t o = int64_t(i + aoff) * W2 + q;
    char2 v;
    v.x = dec_site((c0 ? pk1 : pk0)[o], enc);
    v.y = dec_site((c0 ? pk0 : pk1)[o], enc);
    reinterpret_cast<char2*>(grid + int64_t(i) * W)[q] = v;
  }
}
// count of invalid values (Ising: not +-1; Potts: not 0..3) in n bytes, 16 at a time
__global__ void count_invalid_spins_kernel(const int8_t* __restrict__ s, int64_t n, int potts,
                                           unsigned long long* bad) {
  unsigned long long local = 0;
  const int64_t n16 = n / 16;
  for (int64_t f = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < n16; f += int64_t(gridDim.x) * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(s)[f];
    for (uint32_t w : {v.x, v.y, v.z, v.w}) {
      for (int b = 0; b < 4; ++b) {
        const int8_t x = int8_t(w >> (8 * b));
        local += potts ? !(x >= 0 && x <= 3) : !(x == 1 || x == -1);
      }
    }
  }
  for (int64_t f = n16 * 16 + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; f < n;
       f += int64_t(gridDim.x) * blockDim.x) {
    const int8_t x = s[f];
    local += potts ? !(x >= 0 && x <= 3) : !(x == 1 || x == -1);
  }
  if (local) atomicAdd(bad, local);
}

// ---------------------------------------------------------------- host tables
// P(+1) = expit(b + w*nsum) with the reference's two roundings (ising.py:184: numpy computes
// w*nsum, then adds b) and scipy's expit 1/(1+exp(-z)).  Compiled with -ffp-contract=off.
void ising_probs(double w, double b, double* p) {
  for (int n = -4; n <= 4; ++n) {
    volatile double wn = w * double(n);
    volatile double z = b + wn;
    p[n + 4] = 1.0 / (1.0 + std::exp(-z));
  }
}

void potts_cdf(double coupling, double* cdf) {
  for (int idx = 0; idx < kPottsIdx; ++idx) {
    int n[4] = {idx % 5, (idx / 5) % 5, (idx / 25) % 5, (idx / 125) % 5};
    double e[4];
    for (int a = 0; a < 4; ++a) {
      volatile double x = coupling * double(n[a]);
      e[a] = std::exp(x);
    }
    volatile double s0 = e[0];
    volatile double s1 = s0 + e[1];
    volatile double s2 = s1 + e[2];
    volatile double z = s2 + e[3];
    cdf[idx * 3 + 0] = s0 / z;
    cdf[idx * 3 + 1] = s1 / z;
    cdf[idx * 3 + 2] = s2 / z;
  }
}

// u = w * 2^-32 < p  <=>  w < ceil(p * 2^32)   (p * 2^32 is exact; w integer)
unsigned long long thr32(double p) {
  const double t = std::ceil(p * 4294967296.0);
  if (t <= 0.0) return 0ull;
  if (t >= 4294967296.0) return 4294967296ull;
  return (unsigned long long)t;
}

}  // namespace

struct pm_lat_s {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  int H = 0, W = 0, boundary = 0, model = 0;   // H = own rows for a strip
  int packed = 0;
  // strip of a periodic global lattice (multi-GPU, §8e): own rows are global rows
  // row0 .. row0+H-1, arrays hold H+2 rows (halo above and below)
  int strip = 0, row0 = 0, H_global = 0;
  int8_t* pk0 = nullptr;
  int8_t* pk1 = nullptr;
  int8_t* scratch = nullptr;  // H*W staging for set/get
  // Ising
  bool has_field = false;
  double w = 0.0;
  int n_class = 0;
  int32_t* cls = nullptr;
  double* ptab = nullptr;
  unsigned long long thr[9] = {0};
  // Potts
  bool has_potts = false;
  double* cdf = nullptr;
  unsigned long long* pthr = nullptr;  // Potts packed path, 64-bit thresholds: [85][3] by code sum
  uint32_t* pthr32 = nullptr;  // Potts packed path: [85][3] thresholds by code sum, when all < 2^32
  bool pdl = pdl_default();   // packed half-sweeps launched with PDL (PM_PDL=0 disables)
  bool t32 = false;           // every threshold of the active model fits 32 bits
  // uniforms staging
  double* uni = nullptr;
  size_t uni_cap = 0;
  // strip peer-memory halo exchange (pm_lat_strip_xchg_*)
  int8_t* xmb = nullptr;                   // own mailbox (IPC-exported)
  int8_t* xup = nullptr;                   // up / down neighbours' mailboxes in this process
  int8_t* xdown = nullptr;
  bool xup_ipc = false, xdown_ipc = false;  // mappings to close
  unsigned* xticket = nullptr;             // [0] ticket, [1] status
  unsigned long long xcount[2] = {0, 0};   // deposits made per colour (identical on every rank)
  bool xready = false;                     // initial deposit done: half-sweeps use the mailbox
  cudaEvent_t strip_done = nullptr;        // recorded after each strip half-sweep on the caller's
                                           // stream; spin I/O on h->stream waits for it
};

namespace {

void free_lat(pm_lat_s* h) {
  if (h->xup_ipc && h->xup) cudaIpcCloseMemHandle(h->xup);
  if (h->xdown_ipc && h->xdown && !(h->xup_ipc && h->xdown == h->xup)) cudaIpcCloseMemHandle(h->xdown);
  h->xup = h->xdown = nullptr;
  h->xup_ipc = h->xdown_ipc = false;
  for (void* p : {(void*)h->pk0, (void*)h->pk1, (void*)h->scratch, (void*)h->cls, (void*)h->ptab, (void*)h->cdf,
                  (void*)h->pthr, (void*)h->pthr32, (void*)h->uni, (void*)h->xmb, (void*)h->xticket})
    if (p) cudaFree(p);
  h->xmb = nullptr;
  h->xticket = nullptr;
  h->xready = false;
  h->pthr32 = nullptr;
  h->pk0 = h->pk1 = h->scratch = nullptr;
  h->cls = nullptr;
  h->ptab = h->cdf = h->uni = nullptr;
  h->pthr = nullptr;
  h->uni_cap = 0;
}

LatView view_of(pm_lat_s* h) {
  LatView v;
  v.pk0 = h->pk0;
  v.pk1 = h->pk1;
  v.H = h->H;
  v.W = h->W;
  v.W2 = h->W / 2;
  v.packed = h->packed;
  v.enc = h->packed ? (h->model == PM_MODEL_ISING ? 1 : 2) : 0;
  return v;
}

// Philox4x32 block indices (site / 4) of a whole lattice fit 32 bits with margin for a
// thread's words: the packed kernel's 32-bit counter arithmetic
bool packed_blocks_fit(int64_t H, int64_t W) { return H * W / 4 < (int64_t(1) << 32) - 64; }

bool fast_path_ok(pm_lat_s* h) {
  return h->packed && h->boundary == PM_BOUNDARY_PERIODIC && (h->H % 2 == 0) && ((h->W / 2) % 16 == 0) &&
         packed_blocks_fit(h->strip ? h->H_global : h->H, h->W) &&
         (h->model == PM_MODEL_POTTS4 || h->n_class == 1);
}

int grid_for(pm_lat_s* h, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(int64_t(h->sms) * 16, (n + 255) / 256));
}

}  // namespace

extern "C" {

int pm_ising_prob_table(double w, double b, double* p_out) {
  if (!p_out) return fail(PM_EINVAL, "null output");
  ising_probs(w, b, p_out);
  return PM_OK;
}

int pm_potts_cdf_table(double coupling, double* cdf_out) {
  if (!cdf_out) return fail(PM_EINVAL, "null output");
  potts_cdf(coupling, cdf_out);
  return PM_OK;
}

int pm_lat_create(int device, int32_t H, int32_t W, int boundary, int model, pm_lat_t* out) {
  if (!out) return fail(PM_EINVAL, "null output");
  if (H < 1 || W < 1) return fail(PM_EINVAL, "spin grid must be non-empty 2-D");
  if (boundary != PM_BOUNDARY_FREE && boundary != PM_BOUNDARY_PERIODIC) return fail(PM_EINVAL, "bad boundary");
  if (model != PM_MODEL_ISING && model != PM_MODEL_POTTS4) return fail(PM_EINVAL, "bad model");
  if (boundary == PM_BOUNDARY_PERIODIC && ((H % 2) || (W % 2)))
    return fail(PM_EINVAL, "periodic checkerboard needs even height and width");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(PM_ERANGE, "device index out of range");
  pm_lat_s* h = new pm_lat_s();
  h->device = device;
  h->H = H;
  h->W = W;
  h->boundary = boundary;
  h->model = model;
  h->packed = (W % 2 == 0) ? 1 : 0;
  DeviceGuard g(device);
  h->sms = sm_count(device);
  const size_t n_sites = size_t(H) * W;
  e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) {
    if (h->packed) {
      e = cudaMalloc(&h->pk0, n_sites / 2 + 16);
      if (e == cudaSuccess) e = cudaMalloc(&h->pk1, n_sites / 2 + 16);
    } else {
      e = cudaMalloc(&h->pk0, n_sites + 16);
    }
  }
  if (e == cudaSuccess) e = cudaMalloc(&h->scratch, n_sites + 16);
  if (e != cudaSuccess) {
    free_lat(h);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return cuda_fail(e, "pm_lat_create");
  }
  *out = h;
  return PM_OK;
}

int pm_lat_destroy(pm_lat_t h) {
  if (!h) return PM_OK;
  {
    std::lock_guard<std::mutex> lk(h->mu);
    DeviceGuard g(h->device);
    if (h->strip_done) {
      cudaEventSynchronize(h->strip_done);
      cudaEventDestroy(h->strip_done);
    }
    cudaStreamSynchronize(h->stream);
    free_lat(h);
    cudaStreamDestroy(h->stream);
  }
  delete h;
  return PM_OK;
}

int pm_lat_set_spins(pm_lat_t h, const int8_t* s) {
  if (!h || !s) return fail(PM_EINVAL, "null argument");
  const int64_t n = int64_t(h->H) * h->W;
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  // the neighbours' mailboxes hold this strip's boundary rows from the initial deposit:
  // repacking the own rows now would leave those halos stale
  if (h->strip && h->xready) return fail(PM_ESTATE, "set_spins after pm_lat_strip_xchg_start");
  if (h->strip_done) PM_CUDA(cudaStreamWaitEvent(h->stream, h->strip_done, 0));
  // validated on the device (the reference checks the values, ising.py:64-70) before the
  // lattice state is touched: upload to the staging buffer, count invalid values, then pack
  if (!h->scratch) PM_CUDA(cudaMalloc(&h->scratch, size_t(n) + 16));
  unsigned long long* bad = nullptr;
  PM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(unsigned long long), h->stream));
  PM_CUDA(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), h->stream));
  PM_CUDA(cudaMemcpyAsync(h->scratch, s, n, cudaMemcpyHostToDevice, h->stream));
  count_invalid_spins_kernel<<<grid_for(h, n / 16 + 1), 256, 0, h->stream>>>(h->scratch, n,
                                                                             h->model == PM_MODEL_POTTS4, bad);
  unsigned long long nbad = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&nbad, bad, sizeof(nbad), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaFreeAsync(bad, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess) return cuda_fail(e, "pm_lat_set_spins");
  if (nbad) return fail(PM_EINVAL, h->model == PM_MODEL_ISING ? "spins must be -1 or +1" : "Potts states must be 0..3");
  if (h->packed) {
    pack_kernel<<<grid_for(h, n / 2), 256, 0, h->stream>>>(h->scratch, h->H, h->W, h->pk0, h->pk1, h->row0,
                                                          h->strip, h->model == PM_MODEL_ISING ? 1 : 2);
  } else {
    PM_CUDA(cudaMemcpyAsync(h->pk0, h->scratch, n, cudaMemcpyDeviceToDevice, h->stream));
  }
  PM_CUDA(cudaGetLastError());
  PM_CUDA(cudaStreamSynchronize(h->stream));
  return PM_OK;
}

int pm_lat_get_spins(pm_lat_t h, int8_t* s) {
  if (!h || !s) return fail(PM_EINVAL, "null argument");
  const int64_t n = int64_t(h->H) * h->W;
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  if (h->strip_done) PM_CUDA(cudaStreamWaitEvent(h->stream, h->strip_done, 0));
  if (h->packed) {
    unpack_kernel<<<grid_for(h, n / 2), 256, 0, h->stream>>>(h->scratch, h->H, h->W, h->pk0, h->pk1, h->row0,
                                                             h->strip, h->model == PM_MODEL_ISING ? 1 : 2);
    PM_CUDA(cudaGetLastError());
    PM_CUDA(cudaMemcpyAsync(s, h->scratch, n, cudaMemcpyDeviceToHost, h->stream));
  } else {
    PM_CUDA(cudaMemcpyAsync(s, h->pk0, n, cudaMemcpyDeviceToHost, h->stream));
  }
  PM_CUDA(cudaStreamSynchronize(h->stream));
  return PM_OK;
}

int pm_lat_set_ising(pm_lat_t h, double w, const double* bias) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (h->model != PM_MODEL_ISING) return fail(PM_ESTATE, "lattice is not an Ising model");
  if (!std::isfinite(w)) return fail(PM_EINVAL, "bias and coupling must be finite");
  const int64_t n = int64_t(h->H) * h->W;
  std::vector<double> uniq;
  std::vector<int32_t> cls;
  if (bias) {
    for (int64_t f = 0; f < n; ++f)
      if (!std::isfinite(bias[f])) return fail(PM_EINVAL, "bias and coupling must be finite");
    uniq.assign(bias, bias + n);
    std::sort(uniq.begin(), uniq.end());
    // -0.0 and +0.0 merge: both give the same z and the same expit
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    if (uniq.size() > 1) {
      cls.resize(n);
      for (int64_t f = 0; f < n; ++f)
        cls[f] = int32_t(std::lower_bound(uniq.begin(), uniq.end(), bias[f]) - uniq.begin());
    }
  } else {
    uniq.push_back(0.0);
  }
  std::vector<double> tab(uniq.size() * 9);
  for (size_t c = 0; c < uniq.size(); ++c) ising_probs(w, uniq[c], tab.data() + 9 * c);
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  cudaStreamSynchronize(h->stream);
  if (h->cls) cudaFree(h->cls);
  if (h->ptab) cudaFree(h->ptab);
  h->cls = nullptr;
  h->ptab = nullptr;
  PM_CUDA(cudaMalloc(&h->ptab, sizeof(double) * tab.size()));
  PM_CUDA(cudaMemcpy(h->ptab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
  if (!cls.empty()) {
    PM_CUDA(cudaMalloc(&h->cls, sizeof(int32_t) * n));
    PM_CUDA(cudaMemcpy(h->cls, cls.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  }
  h->n_class = int(cls.empty() ? 1 : uniq.size());
  h->w = w;
  h->t32 = true;
  for (int t = 0; t < 9; ++t) {
    h->thr[t] = thr32(tab[t]);
    if (h->thr[t] > 0xFFFFFFFFull) h->t32 = false;  // p == 1: the 32-bit compare cannot express it
  }
  h->has_field = true;
  return PM_OK;
}

int pm_lat_set_potts(pm_lat_t h, double coupling) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (h->model != PM_MODEL_POTTS4) return fail(PM_ESTATE, "lattice is not a Potts model");
  if (!std::isfinite(coupling)) return fail(PM_EINVAL, "coupling must be finite");
  std::vector<double> cdf(kPottsIdx * 3);
  potts_cdf(coupling, cdf.data());
  std::vector<unsigned long long> thr(kPottsIdx * 3);
  bool fits = true;
  for (int t = 0; t < kPottsIdx * 3; ++t) {
    thr[t] = thr32(cdf[t]);
    if (thr[t] > 0xFFFFFFFFull) fits = false;
  }
  // compact table of the packed path: entry n1 + 5 n2 + 21 n3 of the multiset (n0, n1, n2, n3)
  std::vector<uint32_t> tc(kPottsCodes * 3, 0u);
  std::vector<unsigned long long> tc64(kPottsCodes * 3, 0ull);
  for (int idx = 0; idx < kPottsIdx; ++idx) {
    const int n0 = idx % 5, n1 = (idx / 5) % 5, n2 = (idx / 25) % 5, n3 = idx / 125;
    if (n0 + n1 + n2 + n3 != 4) continue;
    const int e = n1 + 5 * n2 + 21 * n3;
    for (int a = 0; a < 3; ++a) {
      tc[3 * e + a] = uint32_t(thr[3 * idx + a]);
      tc64[3 * e + a] = thr[3 * idx + a];
    }
  }
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  cudaStreamSynchronize(h->stream);
  if (!h->cdf) PM_CUDA(cudaMalloc(&h->cdf, sizeof(double) * kPottsIdx * 3));
  if (!h->pthr) PM_CUDA(cudaMalloc(&h->pthr, sizeof(unsigned long long) * kPottsCodes * 3));
  if (!h->pthr32) PM_CUDA(cudaMalloc(&h->pthr32, sizeof(uint32_t) * kPottsCodes * 3));
  PM_CUDA(cudaMemcpy(h->cdf, cdf.data(), sizeof(double) * kPottsIdx * 3, cudaMemcpyHostToDevice));
  PM_CUDA(cudaMemcpy(h->pthr, tc64.data(), sizeof(unsigned long long) * kPottsCodes * 3, cudaMemcpyHostToDevice));
  PM_CUDA(cudaMemcpy(h->pthr32, tc.data(), sizeof(uint32_t) * kPottsCodes * 3, cudaMemcpyHostToDevice));
  h->t32 = fits;
  h->has_potts = true;
  return PM_OK;
}

static int lat_sweeps_impl(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1,
                           uint64_t stream_pos, const double* uniforms, float* total_ms, int32_t acc_from = 0,
                           int32_t* acc_out = nullptr, int64_t* flips_out = nullptr);

// One half-sweep (colour c) of the packed fast path; for a strip, the own rows of the strip.
static cudaError_t launch_packed(pm_lat_s* h, int c, uint64_t sweep, uint64_t seed, cudaStream_t st) {
  const int Hg = h->strip ? h->H_global : h->H;
  PackedArgs pa;
  pa.other = c == 0 ? h->pk1 : h->pk0;
  pa.mine = c == 0 ? h->pk0 : h->pk1;
  pa.H = Hg;
  pa.W2 = h->W / 2;
  pa.colour = c;
  pa.n0 = int64_t(Hg) * (h->W / 2);
  pa.sweep = sweep;
  pa.seed = seed;
  pa.rk = philox4x32_keys(seed);
  for (int k = 0; k < 9; ++k) pa.thr[k] = h->thr[k];
  pa.row0 = h->row0;
  pa.rows = h->H;
  pa.halo = h->strip;
  pa.xmb = pa.xup = pa.xdown = nullptr;
  pa.rpar = pa.wpar = 0;
  pa.kread = pa.kwrite = 0;
  pa.ticket = pa.status = nullptr;
  if (h->strip && h->xready) {
    // read the other colour's latest deposit, write this colour's next one
    // (xcount[c] advances only once the launch succeeded: a failed launch must not desync the
    // deposit numbers the neighbours wait for)
    const unsigned long long kr = h->xcount[c ^ 1], kw = h->xcount[c] + 1;
    pa.xmb = h->xmb;
    pa.xup = h->xup;
    pa.xdown = h->xdown;
    pa.rpar = int(kr & 1);
    pa.wpar = int(kw & 1);
    pa.kread = kr;
    pa.kwrite = kw;
    pa.ticket = h->xticket;
    pa.status = h->xticket + 1;
  }
  const int W2 = h->W / 2;
  // 16-site groups per thread: Ising 2, Potts 4 (profiles/r01_ab_gibbs_minb.txt);
  // tune gibbs_ng=1|2|4 overrides (A/B knob)
  const int ng_t = tune("gibbs_ng", 0);
  const int ng_env = (ng_t == 1 || ng_t == 2 || ng_t == 4) ? ng_t : 0;
  const int ng_cap = ng_env ? ng_env : (h->model == PM_MODEL_ISING ? 2 : 4);
  const int ng = (W2 % 64 == 0 && ng_cap >= 4) ? 4 : (W2 % 32 == 0 && ng_cap >= 2) ? 2 : 1;  // 16-site groups per thread
  const int per_row = W2 / (16 * ng);
  const int bx = std::min(256, per_row);
  const int by = std::max(1, 256 / bx);
  const dim3 block(bx, by);
  const dim3 grid((per_row + bx - 1) / bx, std::min((h->H + by - 1) / by, 65535));
  const bool ising = h->model == PM_MODEL_ISING;
  cudaError_t e = cudaSuccess;  // a failed launch is also the thread's last error (callers check it)
  // A/B (tune gibbs_smem=1): shared-memory staging of the other colour's rows, 8-row CTAs
  if (tune("gibbs_smem", 0) == 1 && !pa.xmb && !h->strip && h->t32 &&
      ((ising && ng == 2) || (!ising && ng == 4))) {
    const int sbx = std::min(32, per_row), sby = 8;
    const dim3 sblock(sbx, sby);
    const dim3 sgrid((per_row + sbx - 1) / sbx, std::min((h->H + sby - 1) / sby, 65535));
    const size_t smem = size_t(sby + 2) * (sbx * 16 * ng + 32);
    if (!ising) {  // 32.6 KB static table + the stage exceed the 48 KB default
      e = cudaFuncSetAttribute(gibbs_packed_kernel<PM_MODEL_POTTS4, true, 4, false, true>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      if (e != cudaSuccess) return e;
    }
    e = ising ? launch_pdl(h->pdl, gibbs_packed_kernel<PM_MODEL_ISING, true, 2, false, true>, sgrid, sblock, smem, st,
                           pa, (const unsigned long long*)h->pthr, (const uint32_t*)h->pthr32)
              : launch_pdl(h->pdl, gibbs_packed_kernel<PM_MODEL_POTTS4, true, 4, false, true>, sgrid, sblock, smem,
                           st, pa, (const unsigned long long*)h->pthr, (const uint32_t*)h->pthr32);
    return e;
  }
  // rows per thread without the in-kernel exchange (tune gibbs_rpt = 1 | 2 | 4; default 1: measured no gain, profiles/r02_ab_gibbs_rpt.txt):
  // the grid's y extent shrinks accordingly
  const int t_rpt = tune("gibbs_rpt", 1);
  const int rpt = pa.xmb ? 1 : (t_rpt >= 4 ? 4 : (t_rpt >= 2 ? 2 : 1));
  const dim3 grid_r(grid.x, std::min(((h->H + rpt - 1) / rpt + by - 1) / by, 65535));
#define PM_LAUNCH_PACKED(M, T, N)                                                                      \
  e = pa.xmb ? launch_pdl(h->pdl, gibbs_packed_kernel<M, T, N, true>, grid, block, 0, st, pa,          \
                          (const unsigned long long*)h->pthr, (const uint32_t*)h->pthr32)                 \
      : rpt == 4 ? launch_pdl(h->pdl, gibbs_packed_kernel<M, T, N, false, false, 4>, grid_r, block, 0, st, pa, \
                              (const unsigned long long*)h->pthr, (const uint32_t*)h->pthr32)             \
      : rpt == 2 ? launch_pdl(h->pdl, gibbs_packed_kernel<M, T, N, false, false, 2>, grid_r, block, 0, st, pa, \
                              (const unsigned long long*)h->pthr, (const uint32_t*)h->pthr32)             \
                 : launch_pdl(h->pdl, gibbs_packed_kernel<M, T, N, false>, grid, block, 0, st, pa,     \
                              (const unsigned long long*)h->pthr, (const uint32_t*)h->pthr32)
#define PM_LAUNCH_NG(M, T)            \
  do {                                \
    if (ng == 4)                      \
      PM_LAUNCH_PACKED(M, T, 4);      \
    else if (ng == 2)                 \
      PM_LAUNCH_PACKED(M, T, 2);      \
    else                              \
      PM_LAUNCH_PACKED(M, T, 1);      \
  } while (0)
  if (ising && h->t32) PM_LAUNCH_NG(PM_MODEL_ISING, true);
  else if (ising) PM_LAUNCH_NG(PM_MODEL_ISING, false);
  else if (h->t32) PM_LAUNCH_NG(PM_MODEL_POTTS4, true);
  else PM_LAUNCH_NG(PM_MODEL_POTTS4, false);
#undef PM_LAUNCH_NG
#undef PM_LAUNCH_PACKED
  if (e == cudaSuccess && pa.xmb) h->xcount[c] = pa.kwrite;
  return e;
}

int pm_lat_create_strip(int device, int32_t height, int32_t width, int32_t row0, int32_t rows, int model,
                        pm_lat_t* out) {
  if (!out) return fail(PM_EINVAL, "null output");
  if (height < 2 || width < 2 || (height % 2) || (width % 2))
    return fail(PM_EINVAL, "periodic checkerboard needs even height and width");
  if ((width / 2) % 16) return fail(PM_EINVAL, "strips need width % 32 == 0 (16-site packed groups)");
  if (rows < 1 || row0 < 0 || row0 + rows > height) return fail(PM_ERANGE, "strip rows out of range");
  if (model != PM_MODEL_ISING && model != PM_MODEL_POTTS4) return fail(PM_EINVAL, "bad model");
  if (!packed_blocks_fit(height, width)) return fail(PM_EINVAL, "strips need a lattice of fewer than 2^34 sites");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
  if (device < 0 || device >= n) return fail(PM_ERANGE, "device index out of range");
  pm_lat_s* h = new pm_lat_s();
  h->device = device;
  h->H = rows;
  h->W = width;
  h->boundary = PM_BOUNDARY_PERIODIC;
  h->model = model;
  h->packed = 1;
  h->strip = 1;
  h->row0 = row0;
  h->H_global = height;
  DeviceGuard g(device);
  h->sms = sm_count(device);
  const size_t arr = size_t(rows + 2) * (width / 2) + 16;
  e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&h->pk0, arr);
  if (e == cudaSuccess) e = cudaMalloc(&h->pk1, arr);
  if (e == cudaSuccess) e = cudaMemset(h->pk0, 0, arr);
  if (e == cudaSuccess) e = cudaMemset(h->pk1, 0, arr);
  if (e == cudaSuccess) e = cudaMalloc(&h->scratch, size_t(rows) * width + 16);
  if (e != cudaSuccess) {
    free_lat(h);
    if (h->stream) cudaStreamDestroy(h->stream);
    delete h;
    return cuda_fail(e, "pm_lat_create_strip");
  }
  *out = h;
  return PM_OK;
}

int pm_lat_strip_half_sweep(pm_lat_t h, int colour, uint64_t seed, uint64_t sweep, void* stream) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (!h->strip) return fail(PM_ESTATE, "not a strip handle");
  if (colour != 0 && colour != 1) return fail(PM_EINVAL, "colour must be 0 or 1");
  if (h->model == PM_MODEL_ISING && !h->has_field) return fail(PM_ESTATE, "call pm_lat_set_ising first");
  if (h->model == PM_MODEL_POTTS4 && !h->has_potts) return fail(PM_ESTATE, "call pm_lat_set_potts first");
  if (h->model == PM_MODEL_ISING && h->n_class != 1) return fail(PM_EINVAL, "strips need a uniform field");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  const cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
  PM_CUDA(launch_packed(h, colour, sweep, seed, st));
  if (st != h->stream) {  // order later spin I/O (h->stream) after this half-sweep
    if (!h->strip_done) PM_CUDA(cudaEventCreateWithFlags(&h->strip_done, cudaEventDisableTiming));
    PM_CUDA(cudaEventRecord(h->strip_done, st));
  }
  return PM_OK;
}

int pm_lat_strip_row(pm_lat_t h, int colour, int32_t array_row, void** dev_ptr) {
  if (!h || !dev_ptr) return fail(PM_EINVAL, "null argument");
  if (!h->strip) return fail(PM_ESTATE, "not a strip handle");
  if (colour != 0 && colour != 1) return fail(PM_EINVAL, "colour must be 0 or 1");
  if (array_row < 0 || array_row > h->H + 1) return fail(PM_ERANGE, "array row out of range");
  *dev_ptr = (colour ? h->pk1 : h->pk0) + size_t(array_row) * (h->W / 2);
  return PM_OK;
}

int pm_lat_strip_xchg_create(pm_lat_t h, void** mailbox) {
  if (!h || !mailbox) return fail(PM_EINVAL, "null argument");
  if (!h->strip) return fail(PM_ESTATE, "not a strip handle");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  if (!h->xmb) {
    const size_t bytes = lat_xchg_bytes(h->W / 2);
    PM_CUDA(cudaMalloc(&h->xmb, bytes));
    PM_CUDA(cudaMemset(h->xmb, 0, bytes));
    PM_CUDA(cudaMalloc(&h->xticket, 2 * sizeof(unsigned)));
    PM_CUDA(cudaMemset(h->xticket, 0, 2 * sizeof(unsigned)));
    PM_CUDA(cudaDeviceSynchronize());
  }
  *mailbox = h->xmb;
  return PM_OK;
}

int pm_lat_strip_xchg_ipc_handle(pm_lat_t h, void* handle_out) {
  if (!h || !handle_out) return fail(PM_EINVAL, "null argument");
  if (!h->xmb) return fail(PM_ESTATE, "call pm_lat_strip_xchg_create first");
  DeviceGuard g(h->device);
  cudaIpcMemHandle_t hd;
  PM_CUDA(cudaIpcGetMemHandle(&hd, h->xmb));
  std::memcpy(handle_out, &hd, sizeof(hd));
  return PM_OK;
}

int pm_lat_strip_xchg_set_peers(pm_lat_t h, void* up, const void* up_ipc, void* down, const void* down_ipc) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (!h->xmb) return fail(PM_ESTATE, "call pm_lat_strip_xchg_create first");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->xup || h->xdown) return fail(PM_ESTATE, "peers already set");
  DeviceGuard g(h->device);
  auto map = [&](void* ptr, const void* ipc, int8_t** out, bool* opened) -> int {
    if (ptr) {
      *out = static_cast<int8_t*>(ptr);
      return PM_OK;
    }
    if (!ipc) return fail(PM_EINVAL, "need a pointer or an IPC handle for each neighbour");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, ipc, sizeof(hd));
    void* p = nullptr;
    PM_CUDA(cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess));
    *out = static_cast<int8_t*>(p);
    *opened = true;
    return PM_OK;
  };
  int rc = map(up, up_ipc, &h->xup, &h->xup_ipc);
  if (rc) return rc;
  // world 2: both neighbours are the same rank (map it once)
  if (!down && down_ipc && up_ipc && std::memcmp(up_ipc, down_ipc, sizeof(cudaIpcMemHandle_t)) == 0) {
    h->xdown = h->xup;
    return PM_OK;
  }
  rc = map(down, down_ipc, &h->xdown, &h->xdown_ipc);
  if (rc) {
    if (h->xup_ipc) cudaIpcCloseMemHandle(h->xup);
    h->xup = nullptr;
    h->xup_ipc = false;
  }
  return rc;
}

int pm_lat_strip_xchg_status(pm_lat_t h, int32_t* timed_out) {
  if (!h || !timed_out) return fail(PM_EINVAL, "null argument");
  if (!h->xticket) return fail(PM_ESTATE, "no exchange");
  DeviceGuard g(h->device);
  unsigned v[2] = {0, 0};
  PM_CUDA(cudaMemcpy(v, h->xticket, sizeof(v), cudaMemcpyDeviceToHost));
  *timed_out = int(v[1]);
  return PM_OK;
}

}  // extern "C"

namespace {
// Initial deposit: this strip's first / last rows of both colours into the neighbours' halos
// (deposit number 1 of each colour, parity 1), then their flags.
__global__ void lat_xchg_init_kernel(const int8_t* pk0, const int8_t* pk1, int rows, int W2, int8_t* up,
                                     int8_t* down) {
  for (int c = 0; c < 2; ++c) {
    const int8_t* pk = c ? pk1 : pk0;
    for (int q = threadIdx.x; q < W2; q += blockDim.x) {
      up[lat_xchg_halo(1, c, 1, W2) + q] = pk[size_t(1) * W2 + q];       // my first row: below `up`
      down[lat_xchg_halo(1, c, 0, W2) + q] = pk[size_t(rows) * W2 + q];  // my last row: above `down`
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.sc.sys;" ::: "memory");
    for (int c = 0; c < 2; ++c) {
      unsigned long long* fu = reinterpret_cast<unsigned long long*>(up + lat_xchg_flags(W2)) + c * 2 + 1;
      unsigned long long* fd = reinterpret_cast<unsigned long long*>(down + lat_xchg_flags(W2)) + c * 2 + 0;
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fu), "l"(1ull) : "memory");
      asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fd), "l"(1ull) : "memory");
    }
  }
}
}  // namespace

extern "C" {

int pm_lat_strip_xchg_start(pm_lat_t h, void* stream) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (!h->xmb || !h->xup || !h->xdown) return fail(PM_ESTATE, "exchange peers not set");
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  if (h->xcount[0] || h->xcount[1]) return fail(PM_ESTATE, "exchange already started");
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : h->stream;
  lat_xchg_init_kernel<<<1, 256, 0, st>>>(h->pk0, h->pk1, h->H, h->W / 2, h->xup, h->xdown);
  PM_CUDA(cudaGetLastError());
  h->xcount[0] = h->xcount[1] = 1;
  h->xready = true;
  return PM_OK;
}

int pm_lat_sweeps(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1, uint64_t stream_pos,
                  const double* uniforms) {
  return lat_sweeps_impl(h, n_sweeps, rng_mode, key0, key1, stream_pos, uniforms, nullptr);
}

int pm_lat_time_sweeps(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1,
                       uint64_t stream_pos, float* total_ms) {
  if (!total_ms) return fail(PM_EINVAL, "null argument");
  if (rng_mode == PM_RNG_UNIFORMS) return fail(PM_EINVAL, "timing needs an in-kernel RNG mode");
  return lat_sweeps_impl(h, n_sweeps, rng_mode, key0, key1, stream_pos, nullptr, total_ms);
}

int pm_lat_sweeps_acc(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1,
                      uint64_t stream_pos, const double* uniforms, int32_t acc_from, int32_t* acc_inout,
                      int64_t* flips_out) {
  if (acc_from < 0) return fail(PM_EINVAL, "acc_from must be >= 0");
  return lat_sweeps_impl(h, n_sweeps, rng_mode, key0, key1, stream_pos, uniforms, nullptr, acc_from, acc_inout,
                         flips_out);
}

static int lat_sweeps_impl(pm_lat_t h, int32_t n_sweeps, int rng_mode, uint64_t key0, uint64_t key1,
                           uint64_t stream_pos, const double* uniforms, float* total_ms, int32_t acc_from,
                           int32_t* acc_out, int64_t* flips_out) {
  if (!h) return fail(PM_EINVAL, "null handle");
  if (n_sweeps < 0) return fail(PM_EINVAL, "n_sweeps must be >= 0");
  if (rng_mode != PM_RNG_UNIFORMS && rng_mode != PM_RNG_NUMPY_PHILOX && rng_mode != PM_RNG_PHILOX4X32)
    return fail(PM_EINVAL, "bad rng mode");
  if (rng_mode == PM_RNG_UNIFORMS && !uniforms && n_sweeps > 0) return fail(PM_EINVAL, "uniforms required");
  if (h->model == PM_MODEL_ISING && !h->has_field) return fail(PM_ESTATE, "call pm_lat_set_ising first");
  if (h->model == PM_MODEL_POTTS4 && !h->has_potts) return fail(PM_ESTATE, "call pm_lat_set_potts first");
  if (h->strip) return fail(PM_ESTATE, "strip handles sweep with pm_lat_strip_half_sweep + halo exchange");
  if (n_sweeps == 0) return PM_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  DeviceGuard g(h->device);
  const int64_t HW = int64_t(h->H) * h->W;
  const int64_t n0 = (HW + 1) / 2, n1 = HW / 2;
  if (rng_mode == PM_RNG_UNIFORMS) {
    const size_t need = size_t(n_sweeps) * HW;
    if (need > h->uni_cap) {
      if (h->uni) cudaFree(h->uni);
      h->uni = nullptr;
      h->uni_cap = 0;
      PM_CUDA(cudaMalloc(&h->uni, sizeof(double) * need));
      h->uni_cap = need;
    }
    PM_CUDA(cudaMemcpyAsync(h->uni, uniforms, sizeof(double) * need, cudaMemcpyHostToDevice, h->stream));
  }
  const bool diag = acc_out || flips_out;   // diagnostics run on the generic kernel
  const bool fast = rng_mode == PM_RNG_PHILOX4X32 && fast_path_ok(h) && !diag;
  int32_t* d_acc = nullptr;
  unsigned long long* d_flips = nullptr;
  struct FreeDiag {
    void* a;
    void* b;
    cudaStream_t s;
    ~FreeDiag() {
      if (a) cudaFreeAsync(a, s);
      if (b) cudaFreeAsync(b, s);
    }
  } free_diag{nullptr, nullptr, h->stream};
  if (acc_out) {
    PM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_acc), sizeof(int32_t) * HW, h->stream));
    free_diag.a = d_acc;
    PM_CUDA(cudaMemcpyAsync(d_acc, acc_out, sizeof(int32_t) * HW, cudaMemcpyHostToDevice, h->stream));
  }
  if (flips_out) {
    PM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_flips), sizeof(unsigned long long) * n_sweeps, h->stream));
    free_diag.b = d_flips;
    PM_CUDA(cudaMemsetAsync(d_flips, 0, sizeof(unsigned long long) * n_sweeps, h->stream));
  }
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (total_ms) {
    PM_CUDA(cudaEventCreate(&e0));
    PM_CUDA(cudaEventCreate(&e1));
    PM_CUDA(cudaEventRecord(e0, h->stream));
  }
  for (int t = 0; t < n_sweeps; ++t) {
    for (int c = 0; c < 2; ++c) {
      const int64_t nc = c == 0 ? n0 : n1;
      if (nc == 0) continue;
      if (fast) {
        PM_CUDA(launch_packed(h, c, stream_pos + uint64_t(t), key0, h->stream));
      } else {
        GenericArgs a;
        a.lat = view_of(h);
        a.periodic = h->boundary == PM_BOUNDARY_PERIODIC;
        a.model = h->model;
        a.rng = rng_mode;
        a.colour = c;
        a.n0 = n0;
        a.n_c = nc;
        a.cls = h->cls;
        a.ptab = h->ptab;
        a.cdf = h->cdf;
        a.key0 = key0;
        a.key1 = key1;
        a.base = stream_pos + uint64_t(t) * HW + (c == 0 ? 0 : n0);
        a.sweep = stream_pos + uint64_t(t);
        a.uni = rng_mode == PM_RNG_UNIFORMS ? h->uni + size_t(t) * HW + (c == 0 ? 0 : n0) : nullptr;
        a.flips = d_flips ? d_flips + t : nullptr;
        a.acc = (d_acc && t >= acc_from) ? d_acc : nullptr;
        gibbs_generic_kernel<<<grid_for(h, nc), 256, 0, h->stream>>>(a);
      }
      PM_CUDA(cudaGetLastError());
    }
  }
  if (total_ms) {
    PM_CUDA(cudaEventRecord(e1, h->stream));
    PM_CUDA(cudaEventSynchronize(e1));
    PM_CUDA(cudaEventElapsedTime(total_ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (d_acc) PM_CUDA(cudaMemcpyAsync(acc_out, d_acc, sizeof(int32_t) * HW, cudaMemcpyDeviceToHost, h->stream));
  if (d_flips)
    PM_CUDA(cudaMemcpyAsync(flips_out, d_flips, sizeof(int64_t) * n_sweeps, cudaMemcpyDeviceToHost, h->stream));
  PM_CUDA(cudaStreamSynchronize(h->stream));
  return PM_OK;
}

int pm_lat_stream(pm_lat_t h, void** stream) {
  if (!h || !stream) return fail(PM_EINVAL, "null argument");
  *stream = h->stream;
  return PM_OK;
}

int pm_lat_packed(pm_lat_t h, int* packed) {
  if (!h || !packed) return fail(PM_EINVAL, "null argument");
  *packed = fast_path_ok(h) ? 1 : 0;
  return PM_OK;
}

}  // extern "C"
