// Counter-based Philox generators (Salmon et al., SC'11), host + device.
//   philox4x64_10: numpy.random.Philox's generator (rng.py:42-44 builds it from a
//                  SeedSequence); numpy pre-increments the 256-bit counter before each
//                  4-word block, so stream deviate i comes from counter i/4+1, word i%4,
//                  and a uniform double is (word >> 11) * 2^-53.
//   philox4x32_10: the (seed, sweep, site)-keyed generator of BASELINE config 4.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define PM_HD __host__ __device__ __forceinline__
#else
#define PM_HD inline
#endif

namespace pm {

struct U64x4 {
  uint64_t v[4];
};
struct U32x4 {
  uint32_t v[4];
};

PM_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#if defined(__CUDA_ARCH__)
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  const unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

PM_HD void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
#if defined(__CUDA_ARCH__) && defined(PM_PHILOX_HILO)
  // A/B: IMAD.HI + IMAD instead of one IMAD.WIDE
  hi = __umulhi(a, b);
  lo = a * b;
#elif defined(__CUDA_ARCH__)
  // one IMAD.WIDE.U32 (the C++ form leaves an extra add of zero on the high word)
  asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}"
      : "=r"(lo), "=r"(hi)
      : "r"(a), "r"(b));
#else
  const uint64_t p = (uint64_t)a * b;
  lo = (uint32_t)p;
  hi = (uint32_t)(p >> 32);
#endif
}

PM_HD U64x4 philox4x64_10(U64x4 c, uint64_t k0, uint64_t k1) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(M0, c.v[0], hi0, lo0);
    mulhilo64(M1, c.v[2], hi1, lo1);
    U64x4 o;
    o.v[0] = hi1 ^ c.v[1] ^ k0;
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ k1;
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

PM_HD U32x4 philox4x32_10(U32x4 c, uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(M0, c.v[0], hi0, lo0);
    mulhilo32(M1, c.v[2], hi1, lo1);
    U32x4 o;
    o.v[0] = hi1 ^ c.v[1] ^ k0;
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ k1;
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

// Deviate `idx` of numpy's Philox stream with key (k0,k1), fresh counter: the raw word.
PM_HD uint64_t numpy_philox_word(uint64_t idx, uint64_t k0, uint64_t k1) {
  U64x4 c;
  c.v[0] = idx / 4 + 1;  // numpy increments before generating (no carry below 2^64 blocks)
  c.v[1] = 0;
  c.v[2] = 0;
  c.v[3] = 0;
  const U64x4 o = philox4x64_10(c, k0, k1);
  return o.v[idx % 4];
}

// Key schedule of philox4x32_10 for a 64-bit seed: k[2r] = k0 + r W0, k[2r+1] = k1 + r W1.
struct Philox32Keys {
  uint32_t k[20];
};

PM_HD Philox32Keys philox4x32_keys(uint64_t seed) {
  Philox32Keys rk;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    rk.k[2 * r] = k0;
    rk.k[2 * r + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return rk;
}

// site_philox_block for a 32-bit group index with the key schedule precomputed on the host
// (kernel parameters: each round's key XOR takes its operand straight from the constant bank,
// no per-thread key additions).  Bit-identical to site_philox_block(group, sweep, seed).
PM_HD U32x4 site_philox_block_rk(uint32_t group, uint64_t sweep, const Philox32Keys& rk) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  U32x4 c;
  c.v[0] = group;
  c.v[1] = 0u;
  c.v[2] = (uint32_t)sweep;
  c.v[3] = (uint32_t)(sweep >> 32);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(M0, c.v[0], hi0, lo0);
    mulhilo32(M1, c.v[2], hi1, lo1);
    U32x4 o;
    o.v[0] = hi1 ^ c.v[1] ^ rk.k[2 * r];
    o.v[1] = lo1;
    o.v[2] = hi0 ^ c.v[3] ^ rk.k[2 * r + 1];
    o.v[3] = lo0;
    c = o;
  }
  return c;
}

// The 4 words of the (seed, sweep, group) Philox4x32 block holding stream sites 4g..4g+3.
PM_HD U32x4 site_philox_block(uint64_t group, uint64_t sweep, uint64_t seed) {
  U32x4 c;
  c.v[0] = (uint32_t)group;
  c.v[1] = (uint32_t)(group >> 32);
  c.v[2] = (uint32_t)sweep;
  c.v[3] = (uint32_t)(sweep >> 32);
  return philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
}

}  // namespace pm
