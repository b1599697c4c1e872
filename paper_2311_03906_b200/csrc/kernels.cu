// sm_100a kernels for the SymPhase sampling hot path.
//
//   K1  fused sampler      draw (Philox4x32-10, geometric skip) + GF(2) product +
//                          record write, one persistent warp-specialised kernel
//                          (replaces draw_assignments + sample, sampler.cpp:48-112)
//   K4  fused, compat RNG  bit-exact keyed_draw/fill_group (sampler.hpp:14-28,
//                          sampler.cpp:11-44) + product
//   D   draw               the assignment matrix S of K1/K4 (draw_assignments)
//   K2  explicit-S product sample(expressions, batch) / gf2_multiply_sparse
//                          (sampler.cpp:61-112, bit_matrix.cpp:314-328)
//   K3  encode             encode_shots '01' / 'b8' (sampler.cpp:118-140)
//
// All of this is integer/bitwise, HBM-write-bound work: shared-memory XOR
// tiles, LOP3 accumulation, coalesced 16-byte stores. sm_100a has no binary
// MMA worth using, so there is no tensor-core path.
#include "kernels.cuh"

#include <algorithm>
#include <type_traits>

#include "device_common.cuh"

namespace symphase {

RoundKeys expand_keys(uint64_t seed) {
  RoundKeys K{};
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int i = 0; i < 10; ++i) {
    K.k[2 * i] = k0;
    K.k[2 * i + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return K;
}

namespace {

// ---- K4: fused sampler with the reference's keyed_draw -------------------
// Validation path (bit-exact with the CPU reference): one 64-bit keyed draw
// per (group, shot), ballot into 32-shot symbol words, XOR into the tile.
template <bool kCounts>
__global__ void __launch_bounds__(kFusedThreads)
k4_fused_compat(const DevPlan P, uint64_t seed_mix, uint64_t tile0, uint32_t n_tiles,
                uint64_t n_shots, uint64_t* __restrict__ out, uint64_t ld,
                unsigned long long* __restrict__ counts) {
  extern __shared__ __align__(16) uint32_t smem_k4[];
  const uint32_t tw = P.tw, tw_log2 = P.t_log2 - 5;
  uint32_t* tile = smem_k4;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    const uint64_t gshot0 = (tile0 + t) << P.t_log2;
    for (uint32_t i = threadIdx.x; i < P.n_meas * tw; i += blockDim.x) tile[i] = 0;
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
    const uint64_t first = static_cast<uint64_t>(t) << P.t_log2;
    const uint64_t valid = min(static_cast<uint64_t>(1) << P.t_log2, n_shots - first);
    const uint32_t vw = static_cast<uint32_t>((valid + 63) >> 6);
    const uint64_t tail = (valid & 63) ? ((1ull << (valid & 63)) - 1) : ~0ull;
    const uint32_t tw2_log2 = P.t_log2 - 6;
    const uint2* t2 = reinterpret_cast<const uint2*>(tile);
    for (uint32_t i = threadIdx.x; i < (P.n_meas << tw2_log2); i += blockDim.x) {
      const uint32_t k = i >> tw2_log2, p = i & ((1u << tw2_log2) - 1);
      if (p >= vw) continue;
      uint2 v = t2[i];
      uint64_t w = (static_cast<uint64_t>(v.y) << 32) | v.x;
      if ((P.row_const_compat[k >> 5] >> (k & 31)) & 1u) w = ~w;
      if (p == vw - 1) w &= tail;
      out[static_cast<uint64_t>(k) * ld + (first >> 6) + p] = w;
      if (kCounts && w) atomicAdd(&counts[k], static_cast<unsigned long long>(__popcll(w)));
    }
    __syncthreads();
  }
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

__global__ void d_coins(const DevPlan P, const RoundKeys K, uint64_t quad0, uint64_t n_quads,
                        uint64_t n_words32, uint32_t last_mask, uint32_t* S32, uint64_t ld32) {
  const uint64_t total = P.n_dense_all * n_quads;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t slot = i / n_quads, q = i - slot * n_quads;
    const uint64_t gq = quad0 + q;
    const uint32_t sym = P.dense_sym[slot];
    if (sym >= P.n_sym) continue;  // a merged pseudo coin: not a symbol of S
    const uint4 r = philox10(make_uint4(sym, static_cast<uint32_t>(gq),
                                        (static_cast<uint32_t>(gq >> 32) & 0xFFFFFFu) |
                                            (kDomCoin << 24),
                                        0u),
                             K);
    const uint32_t v[4] = {r.x, r.y, r.z, r.w};
    uint32_t* row = S32 + sym * ld32;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t w = q * 4 + j;
      if (w < n_words32) row[w] = (w == n_words32 - 1) ? (v[j] & last_mask) : v[j];
    }
  }
}

// The j-th set bit (0-based) of a pattern mask, as a 1-based pattern.
__device__ __forceinline__ uint32_t nth_pattern(uint32_t mask, uint32_t j) {
  for (; j; --j) mask &= mask - 1;
  return static_cast<uint32_t>(__ffs(mask));
}

// Sparse symbols of S: the same slices (streams) as the fused kernel. Pass 0
// walks the live and dead classes; a firing of a thinned group's pseudo
// variable sets one of the group's non-null patterns (uniform, keyed by
// (group, global shot)). Pass 1 walks the null classes: a null event of a
// thinned group on a shot where the group did not fire sets one of its null
// patterns (the pass runs after pass 0, so the check sees every firing).
__global__ void d_segments(const DevPlan P, const RoundKeys K, uint64_t tile0, uint32_t n_tiles,
                           uint64_t n_shots, uint32_t* S32, uint64_t ld32, uint32_t pass) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint32_t seg0 = pass ? P.n_seg_all : 0u, n_seg = pass ? P.n_seg_null : P.n_seg_all;
  const uint32_t n_cls = P.n_cls_all + (pass ? P.n_cls_null : 0u);
  const uint64_t total = static_cast<uint64_t>(n_seg) * n_tiles;
  const uint64_t shot0 = tile0 << P.t_log2;
  for (uint64_t i = warp; i < total; i += nwarps) {
    const uint32_t t = static_cast<uint32_t>(i / n_seg);
    const uint32_t seg = seg0 + static_cast<uint32_t>(i - static_cast<uint64_t>(t) * n_seg);
    const uint64_t base = static_cast<uint64_t>(t) << P.t_log2;
    Segment sg;
    segment_init(sg, P.cls, n_cls, seg, P.t_log2);
    segment_walk(sg, K, tile0 + t, P.t_log2, lane, [&](auto, const Fired& f) {
      for (int k = 0; k < kSlots; ++k) {
        if (!((f.v >> k) & 1u)) continue;
        const uint64_t j = base + f.shot[k];
        if (j >= n_shots) continue;
        uint32_t gid = P.cls_groups[sg.goff + f.g[k]];
        uint32_t pat = f.pat[k];
        bool mech = false;
        if (pass == 0 && gid >= P.n_groups) {
          const uint32_t mp = P.mech_pat[gid - P.n_groups];
          gid = P.thin_src[gid - P.n_groups];
          if (gid == UINT32_MAX) continue;  // a merged pseudo group: not a symbol of S
          if (mp) {  // one mechanism (Pauli pattern) of its source group
            pat = mp;
            mech = true;
          }
        }
        const uint32_t first = P.g_first[gid];
        if (!mech && (pass == 1 || P.g_masks[gid] != 0)) {
          const uint64_t gj = shot0 + j;
          const uint32_t h = philox10(make_uint4(gid, static_cast<uint32_t>(gj),
                                                 (static_cast<uint32_t>(gj >> 32) & 0xFFFFFFu) |
                                                     (kDomThin << 24),
                                                 0u),
                                      K).x;
          const uint32_t mask = pass == 0 ? (P.g_masks[gid] & 0xFFFFu) : (P.g_masks[gid] >> 16);
          if (pass == 1) {
            // dropped when the group fired on this shot in pass 0
            bool fired = false;
            for (uint32_t b = 0; b < P.g_arity[gid]; ++b)
              fired |= (S32[(first + b) * ld32 + (j >> 5)] >> (j & 31)) & 1u;
            if (fired) continue;
          }
          pat = nth_pattern(mask, __umulhi(h, __popc(mask)));
        }
        uint32_t s = first;
        for (; pat; pat >>= 1, ++s)
          if (pat & 1u) atomicXor(&S32[s * ld32 + (j >> 5)], 1u << (j & 31));
      }
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

// CSR variant over a segment work list (long rows cut, see DevPlan): one
// warp per segment; a cut row's segments XOR their partial words into the
// (zeroed) output with 64-bit atomics.
__global__ void __launch_bounds__(kK2Rows * 32)
k2_sparse_seg(const uint64_t* __restrict__ seg_ptr, const uint32_t* __restrict__ seg_row,
              uint32_t n_seg, const uint32_t* __restrict__ sym_idx, const uint64_t* __restrict__ S,
              uint64_t ldS, uint64_t n_words, uint64_t tail, uint64_t* __restrict__ out,
              uint64_t ld) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t sgi = blockIdx.x * kK2Rows + (threadIdx.x >> 5);
  if (sgi >= n_seg) return;
  const uint32_t rw = seg_row[sgi];
  const uint32_t k = rw & 0x7FFFFFFFu;
  const bool split = (rw >> 31) != 0;
  const uint64_t b = seg_ptr[sgi], e = seg_ptr[sgi + 1];
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
    if (w0 == n_words - 1) a0 &= tail;
    if (w1 == n_words - 1) a1 &= tail;
    uint64_t* o = out + static_cast<uint64_t>(k) * ld;
    if (split) {
      if (v0 && a0) atomicXor(reinterpret_cast<unsigned long long*>(o + w0), a0);
      if (v1 && a1) atomicXor(reinterpret_cast<unsigned long long*>(o + w1), a1);
    } else {
      if (v0) o[w0] = a0;
      if (v1) o[w1] = a1;
    }
  }
}

__global__ void k2_zero_rows(const uint32_t* __restrict__ rows, uint32_t n_rows, uint64_t n_words,
                             uint64_t* __restrict__ out, uint64_t ld) {
  const uint64_t total = static_cast<uint64_t>(n_rows) * n_words;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[static_cast<uint64_t>(rows[i / n_words]) * ld + i % n_words] = 0;
}

// Dense variant: Method of Four Russians over shared-memory tables. A CTA
// owns 512 measurement rows x 2048 shots (32 u64 words: lane = word, 32 row
// accumulators per thread in registers). Symbols are taken 8 at a time: for
// group g the CTA builds T_g[b][w] = XOR of S[8g + i][w] over the set bits i
// of b (256 entries, Gray-code order, one XOR each), then every row XORs in
// T_g[byte g of its M_sym row]. The row bytes come group-major (one 4-byte
// shared broadcast serves four rows), S rows and bytes are staged 16 groups
// at a time with cp.async (double-buffered), and two tables alternate, so
// one barrier per group separates building T_g from reading it. Work is
// n_meas x words x ceil(n_sym / 8) lookups whatever the density, so it wins
// over the CSR walk for dense M_sym (abi.cpp picks it).
constexpr int kM4Rows = 512, kM4Words = 32, kM4Chunk = 16, kM4Threads = 512;
constexpr int kM4RowsPerWarp = kM4Rows / (kM4Threads / 32);  // 32
constexpr size_t kM4Smem = (2ull * 256 * kM4Words + 2ull * kM4Chunk * 8 * kM4Words) * 8 +
                           2ull * kM4Chunk * kM4Rows;

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(kM4Threads, 1)
k2_m4rm(const uint8_t* __restrict__ Mg, uint64_t gm_ld, uint32_t n_meas, uint32_t n_sym,
        const uint64_t* __restrict__ S, uint64_t ldS, uint64_t n_words, uint64_t tail,
        uint64_t* __restrict__ out, uint64_t ld) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(smem);                   // [2][256][32]
  uint64_t* ss = tab + 2 * 256 * kM4Words;                              // [2][128][32]
  uint8_t* mb = reinterpret_cast<uint8_t*>(ss + 2 * kM4Chunk * 8 * kM4Words);  // [2][16][512]
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t r0 = blockIdx.y * kM4Rows;
  const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * kM4Words;
  const uint32_t n_g = (n_sym + 7) / 8;
  const uint32_t n_chunks = (n_g + kM4Chunk - 1) / kM4Chunk;
  // Stage chunk c (groups 16c .. 16c+15) into buffer c & 1: S rows
  // [128c, 128c+128) x words [w0, w0+32), and the bytes of those groups for
  // the CTA's 512 rows. Out-of-range parts read as zero.
  auto stage = [&](uint32_t c) {
    const uint32_t buf = c & 1;
    const uint32_t ss_s =
        static_cast<uint32_t>(__cvta_generic_to_shared(ss + buf * kM4Chunk * 8 * kM4Words));
#pragma unroll
    for (int i = 0; i < (kM4Chunk * 8 * kM4Words) / kM4Threads; ++i) {
      const uint32_t e = t + i * kM4Threads;  // (row in chunk, word)
      const uint64_t j = static_cast<uint64_t>(c) * kM4Chunk * 8 + (e >> 5);
      const uint64_t w = w0 + (e & 31);
      const bool ok = j < n_sym && w < n_words;
      cp_async8(ss_s + e * 8, ok ? S + j * ldS + w : S, ok);
    }
    const uint32_t mb_s =
        static_cast<uint32_t>(__cvta_generic_to_shared(mb + buf * kM4Chunk * kM4Rows));
    {
      const uint32_t e = t;  // 16-byte piece: (group in chunk, 16 rows)
      const uint32_t gi = e / (kM4Rows / 16), rr = (e % (kM4Rows / 16)) * 16;
      const uint64_t g = static_cast<uint64_t>(c) * kM4Chunk + gi;
      const bool ok = g < n_g && r0 + rr < gm_ld;
      cp_async16(mb_s + e * 16, ok ? Mg + g * gm_ld + r0 + rr : Mg, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  uint64_t acc[kM4RowsPerWarp];
#pragma unroll
  for (int r = 0; r < kM4RowsPerWarp; ++r) acc[r] = 0;
  stage(0);
  // Phase g: rows look up group g-1, the CTA builds the table of group g.
  for (uint32_t g = 0; g <= n_g; ++g) {
    const uint32_t c = g / kM4Chunk, gi = g % kM4Chunk;
    if (gi == 0 && g < n_g) {  // chunk c must have landed
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    }
    if (gi == 1 && c + 1 < n_chunks) stage(c + 1);  // its buffer's last readers passed a barrier
    if (g > 0) {
      const uint32_t gp = g - 1;
      const uint64_t* T = tab + (gp & 1) * 256 * kM4Words + lane;
      const uint32_t* bytes4 = reinterpret_cast<const uint32_t*>(
          mb + ((gp / kM4Chunk) & 1) * kM4Chunk * kM4Rows + (gp % kM4Chunk) * kM4Rows +
          warp * kM4RowsPerWarp);
#pragma unroll
      for (int q = 0; q < kM4RowsPerWarp / 4; ++q) {
        const uint32_t v = bytes4[q];  // rows 4q .. 4q+3 of this warp (broadcast)
#pragma unroll
        for (int r = 0; r < 4; ++r) acc[4 * q + r] ^= T[((v >> (8 * r)) & 0xFFu) * kM4Words];
      }
    }
    if (g < n_g) {
      // entries b = 16h + l for this thread's word w and high nibble h:
      // start from the XOR of the high rows, then walk l in Gray order
      const uint32_t w = lane, h = warp;
      const uint64_t* srow = ss + (c & 1) * kM4Chunk * 8 * kM4Words + gi * 8 * kM4Words + w;
      uint64_t lo[4], e = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        lo[i] = srow[i * kM4Words];
        if ((h >> i) & 1u) e ^= srow[(4 + i) * kM4Words];
      }
      uint64_t* T = tab + (g & 1) * 256 * kM4Words + (h * 16) * kM4Words + w;
      T[0] = e;
#pragma unroll
      for (int l = 1; l < 16; ++l) {
        e ^= lo[l & 1 ? 0 : l & 2 ? 1 : l & 4 ? 2 : 3];  // lowest set bit of l
        T[(l ^ (l >> 1)) * kM4Words] = e;
      }
    }
    __syncthreads();
  }
  const uint64_t w = w0 + lane;
  if (w < n_words) {
#pragma unroll
    for (int r = 0; r < kM4RowsPerWarp; ++r) {
      const uint32_t k = r0 + warp * kM4RowsPerWarp + r;
      if (k < n_meas) out[static_cast<uint64_t>(k) * ld + w] = (w == n_words - 1) ? (acc[r] & tail) : acc[r];
    }
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
// memory so the global write of the block's records is contiguous (16-byte
// stores when aligned). Word (row k, 32-shot column c) of a
// measurement-major (tw_log2 < 0) or tiled (tw32 = 2^tw_log2 = T/32) array.
__device__ __forceinline__ uint64_t rec_word(uint32_t k, uint64_t c, uint64_t ld32,
                                             uint32_t n_meas, int tw_log2) {
  if (tw_log2 < 0) return k * ld32 + c;
  return ((c >> tw_log2) * n_meas + k << tw_log2) + (c & ((1u << tw_log2) - 1));
}

__global__ void k3_b8(const uint32_t* __restrict__ m32, uint64_t ld32, uint32_t n_meas,
                      uint64_t n_shots, uint32_t rec, uint8_t* __restrict__ out, bool staged,
                      int tw_log2) {
  extern __shared__ __align__(16) uint8_t stage[];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t n_words32 = (n_shots + 31) >> 5;
  const uint32_t kwords = (n_meas + 31) >> 5;
  const uint64_t shot0 = static_cast<uint64_t>(blockIdx.x) * nw * 32;
  const uint64_t col = (shot0 >> 5) + warp;
  const uint64_t my_shot = shot0 + warp * 32 + lane;
  for (uint32_t kw = 0; kw < kwords; ++kw) {
    const uint32_t k = kw * 32 + lane;
    uint32_t x = (k < n_meas && col < n_words32) ? m32[rec_word(k, col, ld32, n_meas, tw_log2)] : 0u;
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
  if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0 && (nbytes & 15) == 0) {
    const uint4* s4 = reinterpret_cast<const uint4*>(stage);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (uint64_t i = threadIdx.x; i < (nbytes >> 4); i += blockDim.x) d4[i] = s4[i];
  } else {
    for (uint64_t i = threadIdx.x; i < nbytes; i += blockDim.x) dst[i] = stage[i];
  }
}

// '01': one line per shot, '0'/'1' per measurement then '\n'.
__global__ void k3_01(const uint32_t* __restrict__ m32, uint64_t ld32, uint32_t n_meas,
                      uint64_t n_shots, uint8_t* __restrict__ out, int tw_log2) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t n_words32 = (n_shots + 31) >> 5;
  const uint64_t col = static_cast<uint64_t>(blockIdx.x) * nw + warp;
  if (col >= n_words32) return;
  const uint64_t shot = col * 32 + lane;
  const uint64_t line = static_cast<uint64_t>(n_meas) + 1;
  const uint32_t kwords = (n_meas + 31) >> 5;
  for (uint32_t kw = 0; kw < kwords; ++kw) {
    const uint32_t k = kw * 32 + lane;
    uint32_t x = k < n_meas ? m32[rec_word(k, col, ld32, n_meas, tw_log2)] : 0u;
    x = transpose32(x);
    if (shot < n_shots) {
      uint8_t* dst = out + shot * line + kw * 32;
      const uint32_t lim = min(32u, n_meas - kw * 32);
      for (uint32_t b = 0; b < lim; ++b) dst[b] = ((x >> b) & 1u) ? '1' : '0';
    }
  }
  if (shot < n_shots) out[shot * line + n_meas] = '\n';
}

// counts[k] += popcount of row k's first n_shots bits (one warp per row).
__global__ void k_row_counts(const uint64_t* __restrict__ m, uint64_t ld, uint32_t n_meas,
                             uint64_t n_words, uint64_t tail, unsigned long long* counts) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t k = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; k < n_meas;
       k += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    unsigned long long c = 0;
    for (uint64_t w = lane; w < n_words; w += 32)
      c += __popcll(w == n_words - 1 ? (m[k * ld + w] & tail) : m[k * ld + w]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
    if (lane == 0 && c) atomicAdd(&counts[k], c);
  }
}

// Tiled [tile][row][T/64] -> measurement-major [row][ld]; one thread per u64.
__global__ void k_untile(const uint64_t* __restrict__ in, uint32_t n_meas, uint32_t tw2,
                         uint64_t n_words, uint64_t total, uint64_t* __restrict__ out,
                         uint64_t ld) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t t = i / (static_cast<uint64_t>(n_meas) * tw2);
    const uint64_t r = i - t * n_meas * tw2;
    const uint64_t k = r / tw2, w = r - k * tw2;
    const uint64_t col = t * tw2 + w;
    if (col < n_words) out[k * ld + col] = in[i];
  }
}

__global__ void k_debug_philox(const uint32_t* in, uint32_t* out) {
  RoundKeys K;
  uint32_t k0 = in[4], k1 = in[5];
  for (int i = 0; i < 10; ++i) {
    K.k[2 * i] = k0;
    K.k[2 * i + 1] = k1;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const uint4 r = philox10(make_uint4(in[0], in[1], in[2], in[3]), K);
  out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}

}  // namespace

namespace k1 {
// Defined in k1_fused.cuh, instantiated in the k1_inst.cu variant units.
template <bool kStaged, bool kRowStaged, int kLp, bool kPadPred, int kEB>
int launch_k1(const DevPlan& P, const LaunchCfg& L, const RoundKeys& K, uint64_t tile0,
              uint32_t n_tiles, uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t tstride,
              unsigned long long* cnt, unsigned long long* det_cnt);
}  // namespace k1

namespace k7 {
// Defined in k7_queued.cuh, instantiated in k7_inst.cu. Returns 0 when the
// plan does not fit the variant (the caller runs K1).
template <int kThreads, bool kRowStaged, int kLp, int kEB>
int launch_k7(const DevPlan& P, const LaunchCfg& L, const RoundKeys& K, uint64_t tile0,
              uint32_t n_tiles, uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t tstride,
              unsigned long long* cnt, unsigned long long* det_cnt);
}  // namespace k7

size_t fused_smem_bytes(const DevPlan& P, uint32_t t_log2, bool staged, bool row_staged,
                        uint32_t n_buf) {
  const size_t tw = size_t{1} << (t_log2 - 5);
  size_t b = n_buf * (static_cast<size_t>(P.n_meas) * tw + spare_words(tw)) * 4;  // tiles + spare
  b += align16(4ull * P.n_meas * count_lanes(t_log2, n_buf)) + 16;  // counts, dispensers
  b += align16(4ull * (P.n_det + (P.n_det ? 1 : 0)) * count_lanes(t_log2, n_buf));  // detector counts + spare
  b += 16 * kMaxBufHost;                                               // tile mbarriers
  if (P.coins_staged)
    b += align16(4ull * (P.n_dense_live + 2)) + align16(4ull * P.n_dense_live) +
         align16(2ull * P.n_coin_rows);                                 // coin tables
  if (row_staged) {
    b += align16(4ull * (P.n_meas + 4));
    b += align16(4ull * (P.n_paths + 1));
    b += align16(4ull * P.n_paths);
    b += align16(2ull * P.n_keep);
  }
  if (staged) {
    b += align16(sizeof(ClassInfo) * P.n_cls_live);
    b += 16ull * P.n_desc_live;
    b += align16(P.n_colrow * 2);
  }
  return b;
}

int launch_fused_sample(const DevPlan& P, const LaunchCfg& L, uint64_t seed, uint64_t tile0,
                        uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t* counts,
                        bool tiled, uint64_t* det_counts) {
  const uint64_t T = 1ull << P.t_log2;
  const uint64_t tstride = tiled ? static_cast<uint64_t>(P.n_meas) * (T / 64) : T / 64;
  if (tiled) ld = T / 64;
  const uint32_t n_tiles = static_cast<uint32_t>((n_shots + T - 1) / T);
  const RoundKeys K = expand_keys(seed);
  auto* cnt = reinterpret_cast<unsigned long long*>(counts);
  auto* dcnt = reinterpret_cast<unsigned long long*>(det_counts);
  // K7: same records; the launch autotune decides per launch kind. Falls
  // through to K1 when the rings do not fit.
  const uint32_t kind = (tiled ? 2u : 0u) | (dcnt ? 1u : 0u);
  if (P.queued_ok && P.q_sel[kind]) {
    int r = 0;
    DevPlan PQ = P;
    if (!P.q_fixed_shape) PQ.q_walk = PQ.q_apply = P.q_shape[kind];
#define SP_K7T(th, lp, eb)                                                                      \
  (P.row_staged ? k7::launch_k7<th, true, lp, eb>(PQ, L, K, tile0, n_tiles, n_shots, out, ld,   \
                                                  tstride, cnt, dcnt)                           \
                : k7::launch_k7<th, false, lp, eb>(PQ, L, K, tile0, n_tiles, n_shots, out, ld,  \
                                                   tstride, cnt, dcnt))
#define SP_K7(lp, eb) (P.q_threads == 768 ? SP_K7T(768, lp, eb) : SP_K7T(1024, lp, eb))
    const uint32_t key = P.lp * 8 + P.entry_bytes;
    switch (key) {
      case 4 * 8 + 1: r = SP_K7(4, 1); break;
      case 8 * 8 + 1: r = SP_K7(8, 1); break;
      case 16 * 8 + 1: r = SP_K7(16, 1); break;
      case 4 * 8 + 2: r = SP_K7(4, 2); break;
      case 8 * 8 + 2: r = SP_K7(8, 2); break;
      case 4 * 8 + 4: r = SP_K7(4, 4); break;
      default: r = 0;
    }
#undef SP_K7
#undef SP_K7T
    if (r != 0) return r;
  }
#define SP_K1(st, rs, lp, pp, eb) \
  k1::launch_k1<st, rs, lp, pp, eb>(P, L, K, tile0, n_tiles, n_shots, out, ld, tstride, cnt, dcnt)
#define SP_K1R(lp, pp, eb) \
  (P.row_staged ? SP_K1(false, true, lp, pp, eb) : SP_K1(false, false, lp, pp, eb))
#define SP_K1P(lp, eb) (P.pad_pred ? SP_K1R(lp, true, eb) : SP_K1R(lp, false, eb))
#define SP_K1L(lp) \
  (P.entry_bytes == 1 ? SP_K1P(lp, 1) : P.entry_bytes == 2 ? SP_K1P(lp, 2) : SP_K1P(lp, 4))
  if (P.lp == 4) return SP_K1L(4);
  if (P.lp == 8) return SP_K1L(8);
  if (P.lp == 16) return SP_K1L(16);
  if (P.staged) return P.row_staged ? SP_K1(true, true, 0, false, 4) : SP_K1(true, false, 0, false, 4);
  return SP_K1R(0, false, 4);
#undef SP_K1
#undef SP_K1R
#undef SP_K1P
#undef SP_K1L
}

int launch_fused_sample_compat(const DevPlan& P, const LaunchCfg& L, uint64_t seed,
                               uint64_t tile0, uint64_t n_shots, uint64_t* out, uint64_t ld,
                               uint64_t* counts) {
  const uint64_t T = 1ull << P.t_log2;
  const uint32_t n_tiles = static_cast<uint32_t>((n_shots + T - 1) / T);
  const size_t smem = static_cast<size_t>(P.n_meas) * P.tw * 4;
  int grid = 0;
  auto* cnt = reinterpret_cast<unsigned long long*>(counts);
  const uint64_t sm = host_mix64(seed);
  if (counts) {
    if (persistent_grid(k4_fused_compat<true>, L, smem, n_tiles, 8, &grid)) return -1;
    k4_fused_compat<true><<<grid, kFusedThreads, smem, L.stream>>>(P, sm, tile0, n_tiles,
                                                                   n_shots, out, ld, cnt);
  } else {
    if (persistent_grid(k4_fused_compat<false>, L, smem, n_tiles, 8, &grid)) return -1;
    k4_fused_compat<false><<<grid, kFusedThreads, smem, L.stream>>>(P, sm, tile0, n_tiles,
                                                                    n_shots, out, ld, cnt);
  }
  return check_launch() ? -1 : 1;
}

int launch_draw(const DevPlan& P, const LaunchCfg& L, bool compat, uint64_t seed, uint64_t tile0,
                uint64_t n_shots, uint64_t* S, uint64_t ldS, bool segments) {
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
    const RoundKeys K = expand_keys(seed);
    const uint64_t n_quads = (n_words32 + 3) / 4;
    const uint32_t last_mask = (n_shots & 31) ? ((1u << (n_shots & 31)) - 1) : ~0u;
    if (P.n_dense_all) {
      d_coins<<<grid, 256, 0, L.stream>>>(P, K, (tile0 << P.t_log2) >> 7, n_quads, n_words32,
                                          last_mask, S32, ld32);
      ++launches;
    }
    const uint64_t T = 1ull << P.t_log2;
    const uint32_t n_tiles = static_cast<uint32_t>((n_shots + T - 1) / T);
    if (P.n_seg_all && segments) {
      d_segments<<<grid, 256, 0, L.stream>>>(P, K, tile0, n_tiles, n_shots, S32, ld32, 0u);
      ++launches;
    }
    if (P.n_seg_null && segments) {  // null patterns of thinned groups, after every firing is in S
      d_segments<<<grid, 256, 0, L.stream>>>(P, K, tile0, n_tiles, n_shots, S32, ld32, 1u);
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
  dim3 grid((P.n_meas + kK2Rows - 1) / kK2Rows,
            static_cast<unsigned>(std::min<uint64_t>(windows, 65535)));
  if (dense) {
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k2_m4rm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(kM4Smem)) != cudaSuccess)
        return -1;
      attr = true;
    }
    if (!P.dense_gm) return -1;
    const uint64_t row_blocks = (P.n_meas + kM4Rows - 1) / kM4Rows;
    const uint64_t slabs = (n_words + kM4Words - 1) / kM4Words;
    if (row_blocks > 65535 || slabs > 0x7FFFFFFFull) return -1;
    dim3 g4(static_cast<unsigned>(slabs), static_cast<unsigned>(row_blocks));
    k2_m4rm<<<g4, kM4Threads, kM4Smem, L.stream>>>(P.dense_gm, P.gm_ld, P.n_meas, P.n_sym, S, ldS,
                                                   n_words, tail, out, ld);
  } else if (P.k2_seg_ptr) {
    if (P.n_k2_split) {
      const uint64_t total = static_cast<uint64_t>(P.n_k2_split) * n_words;
      const int zb = static_cast<int>(std::min<uint64_t>((total + 255) / 256, 8ull * L.num_sms));
      k2_zero_rows<<<zb, 256, 0, L.stream>>>(P.k2_split_rows, P.n_k2_split, n_words, out, ld);
    }
    dim3 gs((P.n_k2_seg + kK2Rows - 1) / kK2Rows,
            static_cast<unsigned>(std::min<uint64_t>(windows, 65535)));
    k2_sparse_seg<<<gs, kK2Rows * 32, 0, L.stream>>>(P.k2_seg_ptr, P.k2_seg_row, P.n_k2_seg,
                                                     P.sym_idx, S, ldS, n_words, tail, out, ld);
  } else {
    k2_sparse<<<grid, kK2Rows * 32, 0, L.stream>>>(P.row_ptr, P.sym_idx, P.n_meas, S, ldS,
                                                   n_words, tail, out, ld);
  }
  return check_launch() ? -1 : 1;
}

int launch_encode(const LaunchCfg& L, const uint64_t* m, uint64_t ld, uint64_t n_meas,
                  uint64_t n_shots, int fmt, uint8_t* bytes, uint32_t tile_shots) {
  // tiled input: T/32 words per row per tile (T a power of two >= 128)
  int tw_log2 = -1;
  if (tile_shots) tw_log2 = __builtin_ctz(tile_shots / 32);
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
                                                               n_shots, bytes, tw_log2);
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
        m32, 2 * ld, static_cast<uint32_t>(n_meas), n_shots, rec, bytes, staged, tw_log2);
  }
  return check_launch() ? -1 : 1;
}

int launch_untile(const LaunchCfg& L, const uint64_t* in, uint64_t n_meas, uint32_t tile_shots,
                  uint64_t n_shots, uint64_t* out, uint64_t ld) {
  const uint64_t n_words = (n_shots + 63) / 64;
  if (!n_meas || !n_words) return 0;
  const uint64_t tiles = (n_shots + tile_shots - 1) / tile_shots;
  const uint64_t total = n_meas * tiles * (tile_shots / 64);
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 1u << 20));
  k_untile<<<blocks, 256, 0, L.stream>>>(in, static_cast<uint32_t>(n_meas), tile_shots / 64,
                                        n_words, total, out, ld);
  return check_launch() ? -1 : 1;
}

int launch_row_counts(const LaunchCfg& L, const uint64_t* m, uint64_t ld, uint64_t n_meas,
                      uint64_t n_shots, uint64_t* counts) {
  const uint64_t n_words = (n_shots + 63) / 64;
  if (!n_meas || !n_words) return 0;
  const uint64_t tail = (n_shots & 63) ? ((1ull << (n_shots & 63)) - 1) : ~0ull;
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((n_meas + 7) / 8, 65535));
  k_row_counts<<<blocks, 256, 0, L.stream>>>(m, ld, static_cast<uint32_t>(n_meas), n_words, tail,
                                            reinterpret_cast<unsigned long long*>(counts));
  return check_launch() ? -1 : 1;
}

int launch_debug_philox(const LaunchCfg& L, const uint32_t* ctr_key_dev, uint32_t* out_dev) {
  k_debug_philox<<<1, 1, 0, L.stream>>>(ctr_key_dev, out_dev);
  return check_launch() ? -1 : 1;
}

}  // namespace symphase
