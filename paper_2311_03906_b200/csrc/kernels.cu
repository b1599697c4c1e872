// sm_100a kernels for the SymPhase sampling hot path.
//
//   K1  fused sampler      draw (Philox4x32-10, geometric skip) + GF(2) product +
//                          record write, one persistent kernel (replaces
//                          draw_assignments + sample, sampler.cpp:48-112)
//   K4  fused, compat RNG  bit-exact keyed_draw/fill_group (sampler.hpp:14-28,
//                          sampler.cpp:11-44) + product
//   D   draw               the assignment matrix S of K1/K4 (draw_assignments)
//   K2  explicit-S product sample(expressions, batch) / gf2_multiply_sparse
//                          (sampler.cpp:61-112, bit_matrix.cpp:314-328)
//   K3  encode             encode_shots '01' / 'b8' (sampler.cpp:118-140)
//
// All of this is integer/bitwise and HBM-bound work: LOP3 XOR accumulation,
// shared-memory tiles, coalesced u64 stores. There is no binary MMA on sm_100a
// worth using, so no tensor-core path.
#include "kernels.cuh"

#include <algorithm>

namespace symphase {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kFusedThreads = 512;

// ---- random numbers -------------------------------------------------------

// Philox4x32-10 (Salmon et al., SC'11), counter-based: one call -> 4 words.
__device__ __forceinline__ uint4 philox10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Exponential(1) variate -ln(u), u = k * 2^-24 with k = (r >> 8) + 1 in
// [1, 2^24] (so P(u <= x) is exact to 2^-24). Near u = 1 the series of
// -ln(1 - x) keeps full relative precision where lg2.approx would not.
__device__ __forceinline__ float exp1_from_bits(uint32_t r) {
  const uint32_t k = (r >> 8) + 1u;
  const float ux = static_cast<float>(0x1000000u - k) * 0x1.0p-24f;  // 1 - u, exact
  if (ux < 0.03125f) return ux * (1.f + ux * (0.5f + ux * (0.33333334f + ux * 0.25f)));
  return -__log2f(static_cast<float>(k) * 0x1.0p-24f) * 0.6931471806f;
}

// SplitMix64 finalizer and keyed draw — sampler.hpp:14-26.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t keyed_draw(uint64_t seed_mix, uint64_t group, uint64_t shot) {
  return mix64(mix64(seed_mix ^ group) ^ shot);  // seed_mix = mix64(seed)
}

// fill_group (sampler.cpp:11-44) as symbol bits: bit b = symbol first+b.
// Every double operation is an explicitly rounded intrinsic, so no FMA
// contraction can change a comparison against the reference.
__device__ __forceinline__ uint32_t group_bits_compat(uint32_t dist, double p, uint64_t u) {
  switch (dist) {
    case 0: return 1u;
    case 2: return static_cast<uint32_t>(u & 1u);
    case 1: return __dmul_rn(__ull2double_rn(u >> 11), 0x1.0p-53) < p ? 1u : 0u;
    case 3: case 4: {
      const double v = __dmul_rn(__ull2double_rn(u >> 11), 0x1.0p-53);
      const double keep = __dsub_rn(1.0, p);
      if (v < keep) return 0u;
      const double r = __ddiv_rn(__dsub_rn(v, keep), p);
      const int n = dist == 3 ? 3 : 15;
      const int k = __double2int_rz(__dmul_rn(r, static_cast<double>(n)));
      return 1u + static_cast<uint32_t>(min(n - 1, k));
    }
    default: return 0u;
  }
}

__device__ __forceinline__ uint32_t pattern_of(uint32_t dist, uint32_t r) {
  // Given that the channel fired: Bernoulli -> its one symbol; DEPOLARIZE1 ->
  // X, Z, Y uniformly (bits x=1, z=2); DEPOLARIZE2 -> one of 15 non-identity
  // Paulis uniformly (sampler.cpp:24-42 pattern encoding).
  if (dist == 3) return 1u + __umulhi(r, 3u);
  if (dist == 4) return 1u + __umulhi(r, 15u);
  return 1u;
}

// Runs one geometric-skip chain over its slice [lo, hi) of a class's
// flattened (group, shot) trial space for global tile gtile, calling
// emit(group_id, shot_in_tile, pattern) for each firing channel.
template <class Emit>
__device__ __forceinline__ void run_chain(const DevPlan& P, uint32_t c, uint64_t gtile,
                                          uint32_t k0, uint32_t k1, Emit&& emit) {
  const uint32_t cls = P.ch_class[c];
  uint64_t pos = P.ch_lo[c];
  const uint64_t hi = P.ch_hi[c];
  const float inv = P.cls_inv[cls];
  const uint32_t dist = P.cls_dist[cls];
  const uint32_t* groups = P.cls_groups + P.cls_goff[cls];
  const uint32_t tmask = (1u << P.t_log2) - 1u;
  uint4 ctr = make_uint4(c, 0u, static_cast<uint32_t>(gtile),
                         (static_cast<uint32_t>(gtile >> 32) & 0xFFFFFFu) | (kDomChain << 24));
  for (;;) {
    const uint4 r = philox10(ctr, k0, k1);
    ctr.y++;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float sf = exp1_from_bits(h ? r.z : r.x) * inv;
      // Chain slices are <= 2^24 trials, so (float)rem is exact.
      if (!(sf < static_cast<float>(hi - pos))) return;
      pos += static_cast<uint64_t>(sf);
      if (pos >= hi) return;
      emit(groups[pos >> P.t_log2], static_cast<uint32_t>(pos) & tmask,
           pattern_of(dist, h ? r.w : r.y));
      ++pos;
    }
  }
}

// Output pass shared by K1/K4: tile (+ const + dense coins) -> HBM.
template <bool kCounts>
__device__ __forceinline__ void store_tile(const DevPlan& P, const uint32_t* tile,
                                           const uint32_t* coin, const uint32_t* row_const,
                                           bool use_dense, uint64_t t_local, uint64_t n_shots,
                                           uint64_t* __restrict__ out, uint64_t ld,
                                           unsigned long long* cnt) {
  const uint32_t tw2_log2 = P.t_log2 - 6, tw2 = 1u << tw2_log2;
  const uint64_t T = 1ull << P.t_log2;
  const uint64_t first = t_local * T;
  const uint64_t valid = min(T, n_shots - first);
  const uint32_t vw = static_cast<uint32_t>((valid + 63) >> 6);
  const uint64_t tail = (valid & 63) ? ((1ull << (valid & 63)) - 1) : ~0ull;
  const uint2* t2 = reinterpret_cast<const uint2*>(tile);
  const uint2* c2 = reinterpret_cast<const uint2*>(coin);
  const uint32_t items = P.n_meas << tw2_log2;
  for (uint32_t i = threadIdx.x; i < items; i += blockDim.x) {
    const uint32_t k = i >> tw2_log2, p = i & (tw2 - 1);
    if (p >= vw) continue;
    uint2 v = t2[i];
    if ((row_const[k >> 5] >> (k & 31)) & 1u) { v.x = ~v.x; v.y = ~v.y; }
    if (use_dense) {
      for (uint32_t j = P.drow_ptr[k], e = P.drow_ptr[k + 1]; j < e; ++j) {
        const uint2 c = c2[(P.drow_slot[j] << tw2_log2) + p];
        v.x ^= c.x;
        v.y ^= c.y;
      }
    }
    uint64_t w = (static_cast<uint64_t>(v.y) << 32) | v.x;
    if (p == vw - 1) w &= tail;
    out[static_cast<uint64_t>(k) * ld + (first >> 6) + p] = w;
    if (kCounts) atomicAdd(&cnt[k], static_cast<unsigned long long>(__popcll(w)));
  }
}

// ---- K1: fused Philox sampler --------------------------------------------
template <bool kCounts>
__global__ void __launch_bounds__(kFusedThreads)
k1_fused(const DevPlan P, uint64_t seed, uint64_t tile0, uint32_t n_tiles, uint64_t n_shots,
         uint64_t* __restrict__ out, uint64_t ld, unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t tw = P.tw;
  uint32_t* tile = smem;                                  // [n_meas][tw]
  uint32_t* coin = tile + static_cast<size_t>(P.n_meas) * tw;  // [n_dense_live][tw]
  unsigned long long* cnt =
      reinterpret_cast<unsigned long long*>(coin + static_cast<size_t>(P.n_dense_live) * tw);
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  if (kCounts)
    for (uint32_t i = threadIdx.x; i < P.n_meas; i += blockDim.x) cnt[i] = 0;

  const uint32_t tw4_log2 = P.t_log2 - 7, tw4 = 1u << tw4_log2;
  for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t gtile = tile0 + t;
    // Phase 0: clear the accumulation tile.
    uint4* t4 = reinterpret_cast<uint4*>(tile);
    for (uint32_t i = threadIdx.x; i < (P.n_meas << tw4_log2); i += blockDim.x)
      t4[i] = make_uint4(0, 0, 0, 0);
    // Phase 1: bit-sliced fair-coin words, keyed by (symbol, global 128-shot quad).
    uint4* c4 = reinterpret_cast<uint4*>(coin);
    for (uint32_t i = threadIdx.x; i < (P.n_dense_live << tw4_log2); i += blockDim.x) {
      const uint32_t slot = i >> tw4_log2, q = i & (tw4 - 1);
      const uint64_t gq = (gtile << tw4_log2) + q;
      c4[i] = philox10(make_uint4(P.dense_sym[slot], static_cast<uint32_t>(gq),
                                  (static_cast<uint32_t>(gq >> 32) & 0xFFFFFFu) | (kDomCoin << 24),
                                  0u),
                       k0, k1);
    }
    __syncthreads();
    // Phase 2: sparse channels — geometric-skip chains, XOR the fired
    // symbols' M_sym columns into the tile (one bit per measurement row).
    for (uint32_t c = threadIdx.x; c < P.n_chains_live; c += blockDim.x) {
      run_chain(P, c, gtile, k0, k1, [&](uint32_t gid, uint32_t shot, uint32_t pat) {
        const uint32_t bit = 1u << (shot & 31), wofs = shot >> 5;
        uint32_t s = P.g_first[gid];
        for (; pat; pat >>= 1, ++s) {
          if (!(pat & 1u)) continue;
          for (uint64_t j = P.col_ptr[s], e = P.col_ptr[s + 1]; j < e; ++j)
            atomicXor(&tile[P.col_rows[j] * tw + wofs], bit);
        }
      });
    }
    __syncthreads();
    // Phase 3: constant + dense terms, coalesced u64 stores.
    store_tile<kCounts>(P, tile, coin, P.row_const, true, t, n_shots, out, ld, cnt);
    __syncthreads();
  }
  if (kCounts)
    for (uint32_t i = threadIdx.x; i < P.n_meas; i += blockDim.x)
      if (cnt[i]) atomicAdd(&counts[i], cnt[i]);
}

// ---- K4: fused sampler with the reference's keyed_draw -------------------
template <bool kCounts>
__global__ void __launch_bounds__(kFusedThreads)
k4_fused_compat(const DevPlan P, uint64_t seed_mix, uint64_t tile0, uint32_t n_tiles,
                uint64_t n_shots, uint64_t* __restrict__ out, uint64_t ld,
                unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) uint32_t smem[];
  const uint32_t tw = P.tw, tw_log2 = P.t_log2 - 5;
  uint32_t* tile = smem;
  unsigned long long* cnt =
      reinterpret_cast<unsigned long long*>(tile + static_cast<size_t>(P.n_meas) * tw);
  if (kCounts)
    for (uint32_t i = threadIdx.x; i < P.n_meas; i += blockDim.x) cnt[i] = 0;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t gshot0 = (tile0 + t) << P.t_log2;
    uint4* t4 = reinterpret_cast<uint4*>(tile);
    for (uint32_t i = threadIdx.x; i < (P.n_meas << (P.t_log2 - 7)); i += blockDim.x)
      t4[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const uint32_t tasks = P.n_live_groups << tw_log2;
    for (uint32_t task = warp; task < tasks; task += nwarps) {
      const uint32_t gid = P.live_groups[task >> tw_log2], w = task & (tw - 1);
      const uint64_t shot = gshot0 + (w << 5) + lane;
      const uint32_t bits =
          group_bits_compat(P.g_dist[gid], P.g_param[gid], keyed_draw(seed_mix, gid, shot));
      const uint32_t first = P.g_first[gid], arity = P.g_arity[gid];
      for (uint32_t b = 0; b < arity; ++b) {
        const uint32_t word = __ballot_sync(kFull, (bits >> b) & 1u);
        if (!word) continue;
        const uint32_t s = first + b;
        for (uint64_t j = P.col_ptr[s] + lane, e = P.col_ptr[s + 1]; j < e; j += 32)
          atomicXor(&tile[P.col_rows[j] * tw + w], word);
      }
    }
    __syncthreads();
    store_tile<kCounts>(P, tile, nullptr, P.row_const_compat, false, t, n_shots, out, ld, cnt);
    __syncthreads();
  }
  if (kCounts)
    for (uint32_t i = threadIdx.x; i < P.n_meas; i += blockDim.x)
      if (cnt[i]) atomicAdd(&counts[i], cnt[i]);
}

// ---- D: draw_assignments -------------------------------------------------
__global__ void d_fill_ones(const uint32_t* syms, uint32_t n, uint64_t* S, uint64_t ldS,
                            uint64_t n_words, uint64_t tail) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n * n_words;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / n_words, w = i - r * n_words;
    S[static_cast<uint64_t>(syms[r]) * ldS + w] = (w == n_words - 1) ? tail : ~0ull;
  }
}

__global__ void d_coins(const DevPlan P, uint64_t seed, uint64_t quad0, uint64_t n_quads,
                        uint64_t n_words32, uint32_t last_mask, uint32_t* S32, uint64_t ld32) {
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const uint64_t total = P.n_dense_all * n_quads;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t slot = i / n_quads, q = i - slot * n_quads;
    const uint64_t gq = quad0 + q;
    const uint32_t sym = P.dense_sym[slot];
    const uint4 r = philox10(make_uint4(sym, static_cast<uint32_t>(gq),
                                        (static_cast<uint32_t>(gq >> 32) & 0xFFFFFFu) |
                                            (kDomCoin << 24),
                                        0u),
                             k0, k1);
    const uint32_t v[4] = {r.x, r.y, r.z, r.w};
    uint32_t* row = S32 + sym * ld32;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t w = q * 4 + j;
      if (w < n_words32) row[w] = (w == n_words32 - 1) ? (v[j] & last_mask) : v[j];
    }
  }
}

__global__ void d_chains(const DevPlan P, uint64_t seed, uint64_t tile0, uint32_t n_tiles,
                         uint64_t n_shots, uint32_t* S32, uint64_t ld32) {
  const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  const uint64_t total = static_cast<uint64_t>(P.n_chains_all) * n_tiles;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t = static_cast<uint32_t>(i / P.n_chains_all);
    const uint32_t c = static_cast<uint32_t>(i - static_cast<uint64_t>(t) * P.n_chains_all);
    const uint64_t base = static_cast<uint64_t>(t) << P.t_log2;
    run_chain(P, c, tile0 + t, k0, k1, [&](uint32_t gid, uint32_t shot, uint32_t pat) {
      const uint64_t j = base + shot;
      if (j >= n_shots) return;
      uint32_t s = P.g_first[gid];
      for (; pat; pat >>= 1, ++s)
        if (pat & 1u) atomicXor(&S32[s * ld32 + (j >> 5)], 1u << (j & 31));
    });
  }
}

__global__ void d_compat(const DevPlan P, uint64_t seed_mix, uint64_t shot0, uint64_t n_words32,
                         uint64_t n_shots, uint32_t* S32, uint64_t ld32) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t tasks = static_cast<uint64_t>(P.n_groups - 1) * n_words32;
  for (uint64_t task = warp; task < tasks; task += nwarps) {
    const uint32_t gid = 1u + static_cast<uint32_t>(task / n_words32);
    const uint64_t w = task % n_words32;
    const uint64_t j = (w << 5) + lane;
    const uint32_t bits =
        group_bits_compat(P.g_dist[gid], P.g_param[gid], keyed_draw(seed_mix, gid, shot0 + j));
    const uint32_t first = P.g_first[gid], arity = P.g_arity[gid];
    for (uint32_t b = 0; b < arity; ++b) {
      const uint32_t word = __ballot_sync(kFull, j < n_shots && ((bits >> b) & 1u));
      if (lane == 0) S32[(first + b) * ld32 + w] = word;
    }
  }
}

// ---- K2: explicit-S product ----------------------------------------------
// One warp per measurement row, 64 u64 words (4096 shots) per warp; the row's
// symbol list is warp-uniform. Rows vary fastest across blocks so the S
// window a wave touches stays L2-resident while every row consumes it.
constexpr int kK2Rows = 8;

__global__ void __launch_bounds__(kK2Rows * 32)
k2_sparse(const uint64_t* __restrict__ row_ptr, const uint32_t* __restrict__ sym_idx,
          uint32_t n_meas, const uint64_t* __restrict__ S, uint64_t ldS, uint64_t n_words,
          uint64_t tail, uint64_t* __restrict__ out, uint64_t ld) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t k = blockIdx.x * kK2Rows + (threadIdx.x >> 5);
  if (k >= n_meas) return;
  const uint64_t b = row_ptr[k], e = row_ptr[k + 1];
  for (uint64_t win = blockIdx.y; win * 64 < n_words; win += gridDim.y) {
    const uint64_t w0 = win * 64 + lane, w1 = w0 + 32;
    const bool v0 = w0 < n_words, v1 = w1 < n_words;
    uint64_t a0 = 0, a1 = 0, c0 = 0, c1 = 0;
    uint64_t i = b;
    for (; i + 2 <= e; i += 2) {
      const uint64_t* r0 = S + static_cast<uint64_t>(__ldg(sym_idx + i)) * ldS;
      const uint64_t* r1 = S + static_cast<uint64_t>(__ldg(sym_idx + i + 1)) * ldS;
      if (v0) { a0 ^= __ldg(r0 + w0); c0 ^= __ldg(r1 + w0); }
      if (v1) { a1 ^= __ldg(r0 + w1); c1 ^= __ldg(r1 + w1); }
    }
    if (i < e) {
      const uint64_t* r0 = S + static_cast<uint64_t>(__ldg(sym_idx + i)) * ldS;
      if (v0) a0 ^= __ldg(r0 + w0);
      if (v1) a1 ^= __ldg(r0 + w1);
    }
    a0 ^= c0;
    a1 ^= c1;
    if (v0) out[static_cast<uint64_t>(k) * ld + w0] = (w0 == n_words - 1) ? (a0 & tail) : a0;
    if (v1) out[static_cast<uint64_t>(k) * ld + w1] = (w1 == n_words - 1) ? (a1 & tail) : a1;
  }
}

// Dense variant: the row is read as packed M_sym words; set bits select S rows.
__global__ void __launch_bounds__(kK2Rows * 32)
k2_dense(const uint64_t* __restrict__ M, uint64_t ldm, uint64_t m_words, uint32_t n_meas,
         const uint64_t* __restrict__ S, uint64_t ldS, uint64_t n_words, uint64_t tail,
         uint64_t* __restrict__ out, uint64_t ld) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t k = blockIdx.x * kK2Rows + (threadIdx.x >> 5);
  if (k >= n_meas) return;
  const uint64_t* mrow = M + static_cast<uint64_t>(k) * ldm;
  for (uint64_t win = blockIdx.y; win * 64 < n_words; win += gridDim.y) {
    const uint64_t w0 = win * 64 + lane, w1 = w0 + 32;
    const bool v0 = w0 < n_words, v1 = w1 < n_words;
    uint64_t a0 = 0, a1 = 0;
    for (uint64_t mw = 0; mw < m_words; ++mw) {
      uint64_t m = __ldg(mrow + mw);
      while (m) {
        const uint64_t s = mw * 64 + __ffsll(static_cast<long long>(m)) - 1;
        m &= m - 1;
        const uint64_t* r = S + s * ldS;
        if (v0) a0 ^= __ldg(r + w0);
        if (v1) a1 ^= __ldg(r + w1);
      }
    }
    if (v0) out[static_cast<uint64_t>(k) * ld + w0] = (w0 == n_words - 1) ? (a0 & tail) : a0;
    if (v1) out[static_cast<uint64_t>(k) * ld + w1] = (w1 == n_words - 1) ? (a1 & tail) : a1;
  }
}

// ---- K3: encode ----------------------------------------------------------
// 32x32 bit transpose across a warp: in lane l bit b -> out lane b bit l.
__device__ __forceinline__ uint32_t transpose32(uint32_t x) {
  const uint32_t lane = threadIdx.x & 31;
  constexpr uint32_t kLow[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    const int j = 16 >> s;
    const uint32_t y = __shfl_xor_sync(kFull, x, j);
    const uint32_t low = kLow[s];
    x = (lane & j) ? ((x & ~low) | ((y & ~low) >> j)) : ((x & low) | ((y & low) << j));
  }
  return x;
}

// b8: ceil(n_m/8) bytes per shot, measurement k at bit k%8 of byte k/8.
// Each warp turns one 32-shot column into 32 records, staged in shared
// memory so the global write of the block's records is contiguous.
__global__ void k3_b8(const uint32_t* __restrict__ m32, uint64_t ld32, uint32_t n_meas,
                      uint64_t n_shots, uint32_t rec, uint8_t* __restrict__ out, bool staged) {
  extern __shared__ __align__(16) uint8_t stage[];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t n_words32 = (n_shots + 31) >> 5;
  const uint32_t kwords = (n_meas + 31) >> 5;
  const uint64_t shot0 = static_cast<uint64_t>(blockIdx.x) * nw * 32;
  const uint64_t col = (shot0 >> 5) + warp;
  const uint64_t my_shot = shot0 + warp * 32 + lane;
  for (uint32_t kw = 0; kw < kwords; ++kw) {
    const uint32_t k = kw * 32 + lane;
    uint32_t x = (k < n_meas && col < n_words32) ? m32[k * ld32 + col] : 0u;
    x = transpose32(x);
    uint8_t* dst = staged ? stage + static_cast<uint64_t>(warp * 32 + lane) * rec
                          : out + my_shot * rec;
    if (!staged && my_shot >= n_shots) continue;
#pragma unroll
    for (uint32_t b = 0; b < 4; ++b)
      if (kw * 4 + b < rec) dst[kw * 4 + b] = static_cast<uint8_t>(x >> (8 * b));
  }
  if (!staged) return;
  __syncthreads();
  const uint64_t shots = min(static_cast<uint64_t>(nw) * 32, n_shots - shot0);
  const uint64_t nbytes = shots * rec;
  uint8_t* dst = out + shot0 * rec;
  for (uint64_t i = threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = stage[i];
}

// '01': one line per shot, '0'/'1' per measurement then '\n'.
__global__ void k3_01(const uint32_t* __restrict__ m32, uint64_t ld32, uint32_t n_meas,
                      uint64_t n_shots, uint8_t* __restrict__ out) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t n_words32 = (n_shots + 31) >> 5;
  const uint64_t col = static_cast<uint64_t>(blockIdx.x) * nw + warp;
  if (col >= n_words32) return;
  const uint64_t shot = col * 32 + lane;
  const uint64_t line = static_cast<uint64_t>(n_meas) + 1;
  const uint32_t kwords = (n_meas + 31) >> 5;
  for (uint32_t kw = 0; kw < kwords; ++kw) {
    const uint32_t k = kw * 32 + lane;
    uint32_t x = k < n_meas ? m32[k * ld32 + col] : 0u;
    x = transpose32(x);
    if (shot < n_shots) {
      uint8_t* dst = out + shot * line + kw * 32;
      const uint32_t lim = min(32u, n_meas - kw * 32);
      for (uint32_t b = 0; b < lim; ++b) dst[b] = ((x >> b) & 1u) ? '1' : '0';
    }
  }
  if (shot < n_shots) out[shot * line + n_meas] = '\n';
}

__global__ void k_debug_philox(const uint32_t* in, uint32_t* out) {
  const uint4 r = philox10(make_uint4(in[0], in[1], in[2], in[3]), in[4], in[5]);
  out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}

int check_launch() { return cudaGetLastError() == cudaSuccess ? 0 : -1; }

uint64_t host_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <class K>
int persistent_grid(K kernel, const LaunchCfg& L, size_t smem, uint32_t n_tiles, int* grid) {
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kFusedThreads, smem) !=
          cudaSuccess ||
      per_sm < 1)
    return -1;
  *grid = static_cast<int>(std::min<uint64_t>(n_tiles, static_cast<uint64_t>(per_sm) * L.num_sms));
  return 0;
}

}  // namespace

size_t fused_smem_bytes(uint32_t n_meas, uint32_t n_dense, uint32_t tw, bool counts) {
  return (static_cast<size_t>(n_meas) + n_dense) * tw * 4 + (counts ? 8ull * n_meas : 0);
}

int launch_fused_sample(const DevPlan& P, const LaunchCfg& L, uint64_t seed, uint64_t tile0,
                        uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t* counts) {
  const uint64_t T = 1ull << P.t_log2;
  const uint32_t n_tiles = static_cast<uint32_t>((n_shots + T - 1) / T);
  const bool with_counts = counts != nullptr;
  const size_t smem = fused_smem_bytes(P.n_meas, P.n_dense_live, P.tw, with_counts);
  int grid = 0;
  auto* cnt = reinterpret_cast<unsigned long long*>(counts);
  if (with_counts) {
    if (persistent_grid(k1_fused<true>, L, smem, n_tiles, &grid)) return -1;
    k1_fused<true><<<grid, kFusedThreads, smem, L.stream>>>(P, seed, tile0, n_tiles, n_shots, out,
                                                            ld, cnt);
  } else {
    if (persistent_grid(k1_fused<false>, L, smem, n_tiles, &grid)) return -1;
    k1_fused<false><<<grid, kFusedThreads, smem, L.stream>>>(P, seed, tile0, n_tiles, n_shots,
                                                             out, ld, cnt);
  }
  return check_launch() ? -1 : 1;
}

int launch_fused_sample_compat(const DevPlan& P, const LaunchCfg& L, uint64_t seed,
                               uint64_t tile0, uint64_t n_shots, uint64_t* out, uint64_t ld,
                               uint64_t* counts) {
  const uint64_t T = 1ull << P.t_log2;
  const uint32_t n_tiles = static_cast<uint32_t>((n_shots + T - 1) / T);
  const bool with_counts = counts != nullptr;
  const size_t smem = fused_smem_bytes(P.n_meas, 0, P.tw, with_counts);
  int grid = 0;
  auto* cnt = reinterpret_cast<unsigned long long*>(counts);
  const uint64_t sm = host_mix64(seed);
  if (with_counts) {
    if (persistent_grid(k4_fused_compat<true>, L, smem, n_tiles, &grid)) return -1;
    k4_fused_compat<true><<<grid, kFusedThreads, smem, L.stream>>>(P, sm, tile0, n_tiles,
                                                                   n_shots, out, ld, cnt);
  } else {
    if (persistent_grid(k4_fused_compat<false>, L, smem, n_tiles, &grid)) return -1;
    k4_fused_compat<false><<<grid, kFusedThreads, smem, L.stream>>>(P, sm, tile0, n_tiles,
                                                                    n_shots, out, ld, cnt);
  }
  return check_launch() ? -1 : 1;
}

int launch_draw(const DevPlan& P, const LaunchCfg& L, bool compat, uint64_t seed, uint64_t tile0,
                uint64_t n_shots, uint64_t* S, uint64_t ldS) {
  int launches = 0;
  const uint64_t n_words = (n_shots + 63) / 64, n_words32 = (n_shots + 31) / 32;
  const uint64_t tail = (n_shots & 63) ? ((1ull << (n_shots & 63)) - 1) : ~0ull;
  if (cudaMemsetAsync(S, 0, static_cast<size_t>(P.n_sym) * ldS * 8, L.stream) != cudaSuccess)
    return -1;
  uint32_t* S32 = reinterpret_cast<uint32_t*>(S);
  const uint64_t ld32 = 2 * ldS;
  const int grid = L.num_sms * 8;
  // Rows that are identically one: s0 (sampler.cpp:53), plus Bernoulli(p>=1)
  // symbols in Philox mode (unit_double(u) < 1 always holds).
  const uint32_t n_ones = compat ? 1u : P.n_ones;
  if (n_ones) {
    d_fill_ones<<<grid, 256, 0, L.stream>>>(P.ones_syms, n_ones, S, ldS, n_words, tail);
    ++launches;
  }
  if (compat) {
    if (P.n_groups > 1) {
      d_compat<<<grid, 256, 0, L.stream>>>(P, host_mix64(seed), tile0 << P.t_log2, n_words32,
                                           n_shots, S32, ld32);
      ++launches;
    }
  } else {
    const uint64_t n_quads = (n_words32 + 3) / 4;
    const uint32_t last_mask = (n_shots & 31) ? ((1u << (n_shots & 31)) - 1) : ~0u;
    if (P.n_dense_all) {
      d_coins<<<grid, 256, 0, L.stream>>>(P, seed, (tile0 << P.t_log2) >> 7, n_quads, n_words32,
                                          last_mask, S32, ld32);
      ++launches;
    }
    const uint64_t T = 1ull << P.t_log2;
    const uint32_t n_tiles = static_cast<uint32_t>((n_shots + T - 1) / T);
    if (P.n_chains_all) {
      d_chains<<<grid, 256, 0, L.stream>>>(P, seed, tile0, n_tiles, n_shots, S32, ld32);
      ++launches;
    }
  }
  return check_launch() ? -1 : launches;
}

int launch_product(const DevPlan& P, const LaunchCfg& L, bool dense, const uint64_t* S,
                   uint64_t ldS, uint64_t n_shots, uint64_t* out, uint64_t ld) {
  const uint64_t n_words = (n_shots + 63) / 64;
  if (P.n_meas == 0 || n_words == 0) return 0;
  const uint64_t tail = (n_shots & 63) ? ((1ull << (n_shots & 63)) - 1) : ~0ull;
  const uint64_t windows = (n_words + 63) / 64;
  dim3 grid((P.n_meas + kK2Rows - 1) / kK2Rows, static_cast<unsigned>(std::min<uint64_t>(windows, 65535)));
  if (dense) {
    const uint64_t m_words = (P.n_sym + 63) / 64;
    k2_dense<<<grid, kK2Rows * 32, 0, L.stream>>>(P.dense, P.ldm, m_words, P.n_meas, S, ldS,
                                                  n_words, tail, out, ld);
  } else {
    k2_sparse<<<grid, kK2Rows * 32, 0, L.stream>>>(P.row_ptr, P.sym_idx, P.n_meas, S, ldS,
                                                   n_words, tail, out, ld);
  }
  return check_launch() ? -1 : 1;
}

int launch_encode(const LaunchCfg& L, const uint64_t* m, uint64_t ld, uint64_t n_meas,
                  uint64_t n_shots, int fmt, uint8_t* bytes) {
  if (n_shots == 0 || n_meas == 0) {
    if (fmt == 0 && n_shots) {  // n_meas == 0: one empty line per shot
      if (cudaMemsetAsync(bytes, '\n', n_shots, L.stream) != cudaSuccess) return -1;
    }
    return 0;
  }
  const uint32_t* m32 = reinterpret_cast<const uint32_t*>(m);
  const uint64_t n_words32 = (n_shots + 31) / 32;
  if (fmt == 0) {
    const uint64_t blocks = (n_words32 + 7) / 8;
    k3_01<<<static_cast<unsigned>(blocks), 256, 0, L.stream>>>(m32, 2 * ld,
                                                               static_cast<uint32_t>(n_meas),
                                                               n_shots, bytes);
  } else {
    const uint32_t rec = static_cast<uint32_t>((n_meas + 7) / 8);
    const size_t budget = 96 * 1024;
    uint32_t warps = static_cast<uint32_t>(std::min<size_t>(8, budget / (32ull * rec)));
    const bool staged = warps >= 1;
    if (!staged) warps = 8;
    const size_t smem = staged ? static_cast<size_t>(warps) * 32 * rec : 0;
    if (staged && cudaFuncSetAttribute(k3_b8, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)) != cudaSuccess)
      return -1;
    const uint64_t blocks = (n_words32 + warps - 1) / warps;
    k3_b8<<<static_cast<unsigned>(blocks), warps * 32, smem, L.stream>>>(
        m32, 2 * ld, static_cast<uint32_t>(n_meas), n_shots, rec, bytes, staged);
  }
  return check_launch() ? -1 : 1;
}

int launch_debug_philox(const LaunchCfg& L, const uint32_t* ctr_key_dev, uint32_t* out_dev) {
  k_debug_philox<<<1, 1, 0, L.stream>>>(ctr_key_dev, out_dev);
  return check_launch() ? -1 : 1;
}

}  // namespace symphase
