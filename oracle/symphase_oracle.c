/* TEST INFRASTRUCTURE ONLY — see symphase_oracle.h for scope and pinning. */
#include "symphase_oracle.h"

#include <string.h>

uint64_t orc_mix64(uint64_t x) {
  /* SplitMix64 finalizer — sampler.hpp:14-19 */
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t orc_keyed_draw(uint64_t seed, uint64_t group, uint64_t shot) {
  /* sampler.hpp:24-26 */
  return orc_mix64(orc_mix64(orc_mix64(seed) ^ group) ^ shot);
}

double orc_unit_double(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; } /* sampler.hpp:28 */

unsigned orc_group_bits(int dist, double param, uint64_t u) {
  /* fill_group — sampler.cpp:11-44. Each statement is a separately rounded
   * IEEE double operation (no contraction: compiled without -ffast-math and
   * with -ffp-contract=off semantics for C11 on x86-64 SSE2). */
  switch (dist) {
    case ORC_CONST:
      return 1u; /* sampler.cpp:15-16 */
    case ORC_COIN:
      return (unsigned)(u & 1u); /* sampler.cpp:18-19 */
    case ORC_BERNOULLI:
      return orc_unit_double(u) < param ? 1u : 0u; /* sampler.cpp:21-22 */
    case ORC_DEP1: {
      double v = orc_unit_double(u);
      double keep = 1.0 - param;
      if (v < keep) return 0u; /* sampler.cpp:26 */
      double r = (v - keep) / param;
      double t = r * 3.0;
      int k = (int)t;
      int pattern = 1 + (k < 2 ? k : 2); /* sampler.cpp:28 */
      return (unsigned)pattern;          /* bit0 -> x symbol, bit1 -> z symbol */
    }
    case ORC_DEP2: {
      double v = orc_unit_double(u);
      double keep = 1.0 - param;
      if (v < keep) return 0u; /* sampler.cpp:35 */
      double r = (v - keep) / param;
      double t = r * 15.0;
      int k = (int)t;
      int pattern = 1 + (k < 14 ? k : 14); /* sampler.cpp:37 */
      return (unsigned)pattern;            /* bit b -> symbol first+b */
    }
    default:
      return 0u;
  }
}

int orc_draw_assignments(uint64_t n_groups, const uint8_t* dist, const double* param,
                         const uint32_t* first, const uint32_t* arity, uint64_t n_sym,
                         uint64_t n_shots, uint64_t seed, uint64_t* S, uint64_t ldS) {
  return orc_draw_assignments_range(n_groups, dist, param, first, arity, n_sym, 0, n_shots, seed,
                                    S, ldS);
}

int orc_draw_assignments_range(uint64_t n_groups, const uint8_t* dist, const double* param,
                               const uint32_t* first, const uint32_t* arity, uint64_t n_sym,
                               uint64_t shot_begin, uint64_t n_shots, uint64_t seed, uint64_t* S,
                               uint64_t ldS) {
  if (n_shots == 0) return -2; /* sampler.cpp:50 */
  memset(S, 0, (size_t)(n_sym * ldS) * sizeof(uint64_t));
  for (uint64_t shot = 0; shot < n_shots; ++shot) {
    uint64_t bit = 1ull << (shot & 63);
    uint64_t w = shot >> 6;
    if (n_sym > 0) S[w] |= bit; /* row 0 = constant symbol, sampler.cpp:53 */
    for (uint64_t g = 1; g < n_groups; ++g) {
      uint64_t u = orc_keyed_draw(seed, g, shot_begin + shot); /* order-insensitive keys, sampler.hpp:21-26 */
      unsigned bits = orc_group_bits(dist[g], param[g], u);
      for (uint32_t b = 0; b < arity[g] && bits; ++b, bits >>= 1) {
        if (bits & 1u) S[(uint64_t)(first[g] + b) * ldS + w] |= bit;
      }
    }
  }
  return 0;
}

int orc_sample_sparse(uint64_t n_meas, const uint64_t* row_ptr, const uint32_t* sym_idx,
                      uint64_t n_sym, uint64_t n_shots, const uint64_t* S, uint64_t ldS,
                      uint64_t* out, uint64_t ld) {
  /* Range check first, as sampler.cpp:63-67 does before any work. */
  for (uint64_t i = 0; i < row_ptr[n_meas]; ++i)
    if (sym_idx[i] >= n_sym) return -1;
  uint64_t words = (n_shots + 63) / 64;
  uint64_t tail = n_shots & 63 ? (1ull << (n_shots & 63)) - 1 : ~0ull;
  for (uint64_t k = 0; k < n_meas; ++k) {
    uint64_t* o = out + k * ld;
    memset(o, 0, (size_t)ld * sizeof(uint64_t));
    for (uint64_t i = row_ptr[k]; i < row_ptr[k + 1]; ++i) {
      const uint64_t* s = S + (uint64_t)sym_idx[i] * ldS;
      for (uint64_t w = 0; w < words; ++w) o[w] ^= s[w];
    }
    if (words) o[words - 1] &= tail; /* edge-tile padding stays zero (bit_matrix.hpp:62-66) */
  }
  return 0;
}

uint64_t orc_encode(uint64_t n_meas, uint64_t n_shots, const uint64_t* m, uint64_t ld,
                    int fmt, uint8_t* out) {
  uint64_t p = 0;
  if (fmt == 0) { /* sampler.cpp:122-128 */
    for (uint64_t j = 0; j < n_shots; ++j) {
      for (uint64_t k = 0; k < n_meas; ++k)
        out[p++] = ((m[k * ld + (j >> 6)] >> (j & 63)) & 1) ? '1' : '0';
      out[p++] = '\n';
    }
  } else { /* sampler.cpp:129-138: ceil(n_m/8) bytes, measurement k at bit k%8 of byte k/8 */
    uint64_t stride = (n_meas + 7) / 8;
    for (uint64_t j = 0; j < n_shots; ++j) {
      for (uint64_t b = 0; b < stride; ++b) {
        uint8_t byte = 0;
        for (uint64_t t = 0; t < 8; ++t) {
          uint64_t k = b * 8 + t;
          if (k < n_meas && ((m[k * ld + (j >> 6)] >> (j & 63)) & 1)) byte |= (uint8_t)(1u << t);
        }
        out[p++] = byte;
      }
    }
  }
  return p;
}
