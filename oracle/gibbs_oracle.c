/*
 * CPU oracle for the checkerboard Gibbs hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library (as the checker or the timed CPU baseline);
 * the product (paper_1310_1537_b200/) never links it.
 *
 * Plain-C restatement of the reference sweep (/root/reference/pkg/src/parmcmc/ising.py):
 *   colours, packed (scan) order          ising.py:101-131
 *   z = b + w * nsum, free-boundary 0s    ising.py:119-131, 148-150, 184
 *   s = +1 iff u < expit(z)               ising.py:96-98, 158-172 (scipy expit = 1/(1+exp(-z)))
 *   colour 0 then colour 1                ising.py:175-187
 *   uniforms taken in packed order        ising.py:185, rng.py:115-127
 * and of numpy's Philox4x64-10 uniform stream (rng.py:42-44, 86-90: numpy pre-increments
 * the counter, so deviate i is word i%4 of counter i/4+1, u = (word>>11) * 2^-53).
 *
 * Extensions with no reference implementation (parity for these is pinned by the
 * Random123 known-answer vector for Philox4x32-10, by exact enumeration tests and by
 * the reference sweep fed the same uniforms; see tests/test_oracle.py):
 *   periodic boundary  -- neighbour (i+-1)%H, (j+-1)%W
 *   Potts q=4          -- P(a) ~ exp(coupling * n_a); a = #{a' < 3 : u >= cdf_a'}
 *   Philox4x32-10 keyed by (seed, sweep, site) (include/pmb200.h PM_RNG_PHILOX4X32)
 *
 * Build: make -C oracle  (gcc -O2 -ffp-contract=off; no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { RNG_UNIFORMS = 0, RNG_NUMPY_PHILOX = 1, RNG_PHILOX4X32 = 2 };

static void mulhilo64(uint64_t a, uint64_t b, uint64_t* hi, uint64_t* lo) {
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
}

void oracle_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ull, c0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ull, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1, n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* numpy Philox stream: the raw 64-bit word of deviate idx (fresh counter 0). */
uint64_t oracle_numpy_word(uint64_t idx, uint64_t key0, uint64_t key1) {
  uint64_t ctr[4] = {idx / 4 + 1, 0, 0, 0}, key[2] = {key0, key1}, out[4];
  oracle_philox4x64_10(ctr, key, out);
  return out[idx % 4];
}

double oracle_numpy_uniform(uint64_t idx, uint64_t key0, uint64_t key1) {
  return (double)(oracle_numpy_word(idx, key0, key1) >> 11) * (1.0 / 9007199254740992.0);
}

/* (seed, sweep, site) Philox4x32 uniform: site s of the sweep's stream. */
double oracle_site_uniform(uint64_t s, uint64_t sweep, uint64_t seed) {
  uint64_t g = s >> 2;
  uint32_t ctr[4] = {(uint32_t)g, (uint32_t)(g >> 32), (uint32_t)sweep, (uint32_t)(sweep >> 32)};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)}, out[4];
  oracle_philox4x32_10(ctr, key, out);
  return (double)out[s & 3] * (1.0 / 4294967296.0);
}

double oracle_expit(double z) { return 1.0 / (1.0 + exp(-z)); }

/* packed index of flat site f within its colour = count of same-colour sites before it */
static int64_t packed_index(int64_t f) { return f / 2; }

typedef struct {
  int mode;
  uint64_t key0, key1, pos;   /* numpy: stream index of the first deviate; philox32: sweep */
  const double* uniforms;
} rng_t;

static double draw(const rng_t* r, int64_t t, int c, int64_t n0, int64_t HW, int64_t p) {
  switch (r->mode) {
    case RNG_UNIFORMS:
      return r->uniforms[t * HW + (c ? n0 : 0) + p];
    case RNG_NUMPY_PHILOX:
      return oracle_numpy_uniform(r->pos + (uint64_t)(t * HW + (c ? n0 : 0) + p), r->key0, r->key1);
    default:
      return oracle_site_uniform((uint64_t)(c ? n0 : 0) + (uint64_t)p, r->pos + (uint64_t)t, r->key0);
  }
}

static int nbr(int H, int W, int periodic, int i, int j, int d, int* ni, int* nj) {
  static const int di[4] = {-1, 1, 0, 0}, dj[4] = {0, 0, -1, 1};
  int a = i + di[d], b = j + dj[d];
  if (periodic) {
    a = (a + H) % H;
    b = (b + W) % W;
  } else if (a < 0 || a >= H || b < 0 || b >= W) {
    return 0;
  }
  *ni = a;
  *nj = b;
  return 1;
}

/* n_sweeps Ising sweeps in place on s[H*W] (int8 +-1); b[H*W] bias (NULL = 0). */
int oracle_ising_sweeps(int8_t* s, const double* b, int H, int W, double w, int periodic, int n_sweeps,
                        int mode, uint64_t key0, uint64_t key1, uint64_t pos, const double* uniforms) {
  const int64_t HW = (int64_t)H * W, n0 = (HW + 1) / 2;
  rng_t r = {mode, key0, key1, pos, uniforms};
  for (int64_t t = 0; t < n_sweeps; ++t) {
    for (int c = 0; c < 2; ++c) {
      for (int64_t f = 0; f < HW; ++f) {
        const int i = (int)(f / W), j = (int)(f % W);
        if (((i + j) & 1) != c) continue;
        double nsum = 0.0; /* float64 sum of neighbour spins, sentinel 0 (ising.py:150) */
        for (int d = 0; d < 4; ++d) {
          int ni, nj;
          if (nbr(H, W, periodic, i, j, d, &ni, &nj)) nsum += (double)s[(int64_t)ni * W + nj];
        }
        volatile double wn = w * nsum;           /* lat.w * neighbor_spin_sum  */
        volatile double z = (b ? b[f] : 0.0) + wn; /* packed_b[c] + ...          */
        const double u = draw(&r, t, c, n0, HW, packed_index(f));
        s[f] = (u < oracle_expit(z)) ? 1 : -1;
      }
    }
  }
  return 0;
}

/* cdf of the q=4 heat-bath conditional for neighbour counts n[4] (ascending a). */
void oracle_potts_cdf(double coupling, const int n[4], double cdf[3]) {
  double e[4];
  for (int a = 0; a < 4; ++a) {
    volatile double x = coupling * (double)n[a];
    e[a] = exp(x);
  }
  volatile double s0 = e[0];
  volatile double s1 = s0 + e[1];
  volatile double s2 = s1 + e[2];
  volatile double z = s2 + e[3];
  cdf[0] = s0 / z;
  cdf[1] = s1 / z;
  cdf[2] = s2 / z;
}

/* n_sweeps Potts q=4 sweeps in place on s[H*W] (int8 0..3). */
int oracle_potts_sweeps(int8_t* s, int H, int W, double coupling, int periodic, int n_sweeps, int mode,
                        uint64_t key0, uint64_t key1, uint64_t pos, const double* uniforms) {
  const int64_t HW = (int64_t)H * W, n0 = (HW + 1) / 2;
  rng_t r = {mode, key0, key1, pos, uniforms};
  for (int64_t t = 0; t < n_sweeps; ++t) {
    for (int c = 0; c < 2; ++c) {
      for (int64_t f = 0; f < HW; ++f) {
        const int i = (int)(f / W), j = (int)(f % W);
        if (((i + j) & 1) != c) continue;
        int n[4] = {0, 0, 0, 0};
        for (int d = 0; d < 4; ++d) {
          int ni, nj;
          if (nbr(H, W, periodic, i, j, d, &ni, &nj)) n[s[(int64_t)ni * W + nj]]++;
        }
        double cdf[3];
        oracle_potts_cdf(coupling, n, cdf);
        const double u = draw(&r, t, c, n0, HW, packed_index(f));
        s[f] = (int8_t)((u >= cdf[0]) + (u >= cdf[1]) + (u >= cdf[2]));
      }
    }
  }
  return 0;
}
