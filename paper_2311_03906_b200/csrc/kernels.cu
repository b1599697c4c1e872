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

constexpr unsigned kFull = 0xFFFFFFFFu;

// Named barriers of the fused kernel (0 is __syncthreads).
constexpr uint32_t kBarFull0 = 1, kBarEmpty0 = 3, kBarDrain = 5;

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t{15}; }

// ---- random numbers -------------------------------------------------------

// Philox4x32-10 (Salmon et al., SC'11): one counter block -> 4 words. The
// key schedule is expanded on the host, so each round is 2 IMAD.WIDE + 2 LOP3
// with the round keys read straight from the parameter bank.
__device__ __forceinline__ uint4 philox10(uint4 c, const RoundKeys& K) {
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ K.k[2 * i], lo1, hi0 ^ c.w ^ K.k[2 * i + 1], lo0);
  }
  return c;
}

// Geometric skip floor(-ln(u) / -ln(1-p)) from 24 random bits: u = k * 2^-24
// with k = (r >> 8) + 1 in [1, 2^24] (so P(u <= x) is exact to 2^-24).
// Computed as lg2(u) * clg with clg = ln2 / ln(1-p) < 0. Near u = 1 the
// series of log2(1 - x) keeps full relative precision where lg2.approx would
// not. Clamped to 2^22 (segments are at most 2^22 trials, so a clamped skip
// still lands past the segment end, and 256 of them cannot overflow u32).
__device__ __forceinline__ uint32_t geo_skip(uint32_t r, float clg) {
  constexpr float kL = 1.4426950408889634f;  // 1 / ln 2
  const float u = static_cast<float>((r >> 8) + 1u) * 0x1.0p-24f;
  const float ux = 1.f - u;  // exact: both are multiples of 2^-24 in [0, 1]
  // log2(1 - x) = -(x + x^2/2 + x^3/3 + x^4/4 + ...) / ln 2
  const float series = ux * (-kL + ux * (-0.5f * kL + ux * (-kL / 3.f + ux * (-0.25f * kL))));
  float lg;  // u >= 2^-24 is a normal float, so the flush-to-zero form is exact
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(u));
  const float sf = (ux < 0.03125f ? series : lg) * clg;  // branch-free select
  return __float2uint_rz(fminf(sf, 4194304.f));
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

// ---- geometric-skip segments ----------------------------------------------
//
// A class's flattened (group, shot) trial space of one tile is cut into
// segments; each segment is one Bernoulli(p) process walked by ONE warp in
// lockstep. Every lane draws kBlocks Philox blocks per step: 4 skips per
// block (Bernoulli) or 3 skips + one word whose three base-n digits pick the
// non-identity Pauli of each firing (n = 3 for DEPOLARIZE1 -> X, Z, Y;
// n = 15 for DEPOLARIZE2) — the joint channel pmf of fill_group
// (sampler.cpp:24-42). Geometric gaps floor(Exp/-ln(1-p)) + 1 are laid
// end to end in lane order with a warp prefix sum, so one step yields up to
// 192-256 firing positions with no divergence. Streams are keyed by
// (segment, global tile), independent of which warp, CTA or GPU runs them.
struct Segment {
  uint32_t g0, s0;  // first trial = (class position g0, shot s0 in the tile)
  uint32_t len, seg, goff, dist, pbase, npat;
  float clg;
};

// Philox blocks each lane draws per walk step (independent counters, so the
// two ten-round chains interleave), and the firings one step can yield.
constexpr int kBlocks = 2;
constexpr int kSlots = 4 * kBlocks;

// Firings of one walk step on one lane (slot k valid iff v & (1<<k)).
struct Fired {
  uint32_t v;
  uint32_t g[kSlots], shot[kSlots], pat[kSlots];  // class position, shot in tile, pattern
};

__device__ __forceinline__ void segment_init(Segment& sg, const ClassInfo* cls, uint32_t n_cls,
                                             uint32_t seg, uint32_t t_log2) {
  uint32_t lo = 0, hi = n_cls;  // largest k with cls[k].seg_off <= seg
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (cls[mid].seg_off <= seg) lo = mid; else hi = mid;
  }
  const ClassInfo& ci = cls[lo];
  const uint64_t first = static_cast<uint64_t>(seg - ci.seg_off) * ci.L;
  sg.g0 = static_cast<uint32_t>(first >> t_log2);
  sg.s0 = static_cast<uint32_t>(first) & ((1u << t_log2) - 1u);
  sg.len = static_cast<uint32_t>(min(first + ci.L, ci.trials) - first);
  sg.seg = seg;
  sg.goff = ci.goff;
  sg.dist = ci.dist;
  sg.pbase = ci.pbase;
  sg.npat = ci.npat;
  sg.clg = ci.clg;
}

__device__ __forceinline__ uint4 segment_philox(const Segment& sg, const RoundKeys& K,
                                                uint64_t gtile, uint32_t step, int b,
                                                uint32_t lane) {
  const uint32_t c3 = (static_cast<uint32_t>(gtile >> 32) & 0xFFFFFFu) | (kDomChain << 24);
  return philox10(make_uint4(sg.seg, (step * kBlocks + b) * 32 + lane,
                             static_cast<uint32_t>(gtile), c3),
                  K);
}

// Walks one segment with the whole warp; r holds the Philox blocks of its
// first step. After each step's positions are known, pre(tag, f) runs
// (issue table loads), then the next step's Philox blocks are computed —
// independent work that hides those loads — and then emit(tag, f) runs on
// every lane (lanes may have no valid firing). On the last step next(sn)
// fetches the following segment, whose first blocks are computed in place
// of the next step's, so segment boundaries cost no exposed Philox latency.
// Returns whether sg/r now describe a following segment.
template <bool kBern, class Pre, class Emit, class Next>
__device__ __forceinline__ bool segment_walk_t(Segment& sg, uint4 (&r)[kBlocks],
                                               const RoundKeys& K, uint64_t gtile,
                                               uint32_t t_log2, uint32_t lane, Pre&& pre,
                                               Emit&& emit, Next&& next) {
  constexpr bool bern = kBern;
  const uint32_t n = sg.dist == 3 ? 3u : 15u;
  const uint32_t magic = n == 3 ? 0x5556u : 0x1112u;  // exact /n for values < n^3
  const uint32_t tmask = (1u << t_log2) - 1u;
  uint32_t pos = 0;  // trials consumed (warp-uniform), < len <= 2^22
  for (uint32_t draw = 0;; ++draw) {
    uint32_t incl[kSlots];
    uint32_t acc = 0;
#pragma unroll
    for (int b = 0; b < kBlocks; ++b) {
      const uint32_t w[4] = {r[b].x, r[b].y, r[b].z, r[b].w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k == 3 && !bern) { incl[4 * b + k] = acc; continue; }
        acc += geo_skip(w[k], sg.clg) + 1u;  // gap to the next firing
        incl[4 * b + k] = acc;
      }
    }
    uint32_t scan = acc;  // warp inclusive scan of the lanes' gap sums
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, scan, o);
      if (lane >= static_cast<uint32_t>(o)) scan += t;
    }
    const uint32_t total = __shfl_sync(kFull, scan, 31);
    // trial index (relative to the segment) of this lane's firings, minus 1
    const uint32_t base = pos + scan - acc - 1;
    const uint32_t sbase = sg.s0 + base;
    Fired f;
    f.v = 0;
#pragma unroll
    for (int b = 0; b < kBlocks; ++b) {
      uint32_t digits = bern ? 0u : __umulhi(r[b].w, n * n * n);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int sl = 4 * b + k;
        f.pat[sl] = 1u;
        f.g[sl] = 0;
        f.shot[sl] = 0;
        if (k == 3 && !bern) continue;
        if (!bern) {
          const uint32_t q = (digits * magic) >> 16;
          f.pat[sl] = 1u + digits - q * n;
          digits = q;
        }
        const uint32_t t = sbase + incl[sl];  // < 2^12 + 2^31: no overflow
        f.g[sl] = sg.g0 + (t >> t_log2);
        f.shot[sl] = t & tmask;
        f.v |= (base + incl[sl] < sg.len ? 1u : 0u) << sl;
      }
    }
    pos += total;
    const bool more = pos < sg.len;
    pre(std::integral_constant<bool, kBern>{}, f);
    // The next step's (or segment's) Philox blocks are independent of this
    // step's table loads and atomics: computing them first overlaps the two.
    Segment sn;
    bool have_next = false;
    if (more) {
#pragma unroll
      for (int b = 0; b < kBlocks; ++b) r[b] = segment_philox(sg, K, gtile, draw + 1, b, lane);
    } else {
      have_next = next(sn);
      if (have_next) {
#pragma unroll
        for (int b = 0; b < kBlocks; ++b) r[b] = segment_philox(sn, K, gtile, 0, b, lane);
      }
    }
    emit(std::integral_constant<bool, kBern>{}, f);
    if (!more) {
      if (have_next) sg = sn;
      return have_next;
    }
  }
}

// Bernoulli classes use all four words of a block as skips; DEPOLARIZE
// classes use three and draw patterns from the fourth. The two shapes are
// separate instantiations so neither pays for the other's slots.
template <class Pre, class Emit, class Next>
__device__ __forceinline__ bool segment_walk_chain(Segment& sg, uint4 (&r)[kBlocks],
                                                   const RoundKeys& K, uint64_t gtile,
                                                   uint32_t t_log2, uint32_t lane, Pre&& pre,
                                                   Emit&& emit, Next&& next) {
  if (sg.dist == 1) return segment_walk_t<true>(sg, r, K, gtile, t_log2, lane, pre, emit, next);
  return segment_walk_t<false>(sg, r, K, gtile, t_log2, lane, pre, emit, next);
}

// One segment on its own (the standalone draw kernel).
template <class Emit>
__device__ __forceinline__ void segment_walk(Segment sg, const RoundKeys& K, uint64_t gtile,
                                             uint32_t t_log2, uint32_t lane, Emit&& emit) {
  uint4 r[kBlocks];
#pragma unroll
  for (int b = 0; b < kBlocks; ++b) r[b] = segment_philox(sg, K, gtile, 0, b, lane);
  segment_walk_chain(sg, r, K, gtile, t_log2, lane, [](auto, const Fired&) {}, emit,
                     [](Segment&) { return false; });
}

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// 16-byte shared store of v (keep != 0) or of zeros, as two predicated
// stores instead of four selects.
__device__ __forceinline__ void sts_or_zero(uint32_t a, uint4 v, uint32_t keep) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %5, 0;\n\t"
      "@p st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n\t"
      "@!p st.shared.v4.u32 [%0], {%6, %6, %6, %6};\n\t}" ::"r"(a),
      "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(keep), "r"(0u)
      : "memory");
}

__device__ __forceinline__ uint4 xor4(uint4 a, uint4 b) {
  return make_uint4(a.x ^ b.x, a.y ^ b.y, a.z ^ b.z, a.w ^ b.w);
}

// ---- K1: fused, warp-specialised Philox sampler ---------------------------
//
// The planner rewrites M_sym = L·D (abi.cpp, chain transform): each row k has
// at most one earlier parent row p(k) and D row k = row k XOR row p(k), which
// for syndrome-extraction circuits is the detector-like difference of
// consecutive rounds — far fewer symbols per column. The kernel samples in
// D space and rebuilds M rows level by level (out[k] = d[k] ^ out[p(k)]).
//
// Per CTA: two shared-memory accumulation tiles [n_meas][T/32] u32 (double
// buffer) and two coin buffers [n_dense+1][T/32]. Generator warps walk the
// geometric-skip segments of tile i (warp-cooperative) and XOR each fired
// symbol's D column into tile[i&1] with shared atomics; drain warps
// meanwhile make tile i's fair-coin words, then — once the tile is complete
// — add dense terms and parents level by level, stream the records to HBM
// with 16-byte stores and zero the buffer for tile i+2. Named barriers
// FULL[b] / EMPTY[b] hand the buffers back and forth. Event tables and row
// tables are staged in shared memory when they fit.
template <bool kStaged, bool kRowStaged, int kLp, bool kPadPred, bool kU8>
__global__ void __launch_bounds__(kFusedThreads, 1)
k1_fused(const DevPlan P, const RoundKeys K, uint64_t tile0, uint32_t n_tiles, uint64_t n_shots,
         uint64_t* __restrict__ out, uint64_t ld, uint64_t tile_stride,
         unsigned long long* __restrict__ counts, bool vec) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t tw = P.tw, tw4_log2 = P.t_log2 - 7, tw4 = 1u << tw4_log2;
  // One spare row absorbs the XORs of padded flip-list entries (never read).
  const uint32_t tile_words = (P.n_meas + 1) * tw;
  const bool with_counts = counts != nullptr;
  uint32_t* tiles = reinterpret_cast<uint32_t*>(smem);
  uint8_t* p = reinterpret_cast<uint8_t*>(tiles + 2 * tile_words);
  // Flip counts: per (row, lane) partials when a warp walks one path per
  // 128-shot column group (T = 4096: no cross-lane reduction per row),
  // else one counter per row.
  const uint32_t cnt_lanes = tw4 >= 32 ? 32u : 1u;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(p);
  p += align16(4ull * P.n_meas * cnt_lanes);
  uint32_t* segctr = reinterpret_cast<uint32_t*>(p);  // per-buffer segment dispensers
  p += 16;

  const ClassInfo* CLS = P.cls;
  const uint4* DESC = P.desc;
  const uint16_t* COLROW = P.colrow;
  const uint4* PLIST = P.plist;
  const uint32_t* PROWS = P.path_rows;
  const uint32_t* PPTR = P.path_ptr;
  const int32_t* PPAR = P.path_par;
  const uint16_t* KEEP = P.keep_rows;
  if (kRowStaged) {
    uint32_t* s_prows = reinterpret_cast<uint32_t*>(p);
    p += align16(4ull * (P.n_meas + 1));
    uint32_t* s_pptr = reinterpret_cast<uint32_t*>(p);
    p += align16(4ull * (P.n_paths + 1));
    int32_t* s_ppar = reinterpret_cast<int32_t*>(p);
    p += align16(4ull * P.n_paths);
    uint16_t* s_keep = reinterpret_cast<uint16_t*>(p);
    p += align16(2ull * P.n_keep);
    for (uint32_t i = threadIdx.x; i <= P.n_meas; i += blockDim.x) s_prows[i] = P.path_rows[i];
    for (uint32_t i = threadIdx.x; i <= P.n_paths; i += blockDim.x) s_pptr[i] = P.path_ptr[i];
    for (uint32_t i = threadIdx.x; i < P.n_paths; i += blockDim.x) s_ppar[i] = P.path_par[i];
    for (uint32_t i = threadIdx.x; i < P.n_keep; i += blockDim.x) s_keep[i] = P.keep_rows[i];
    PROWS = s_prows;
    PPTR = s_pptr;
    PPAR = s_ppar;
    KEEP = s_keep;
  }
  if (kStaged) {
    ClassInfo* s_cls = reinterpret_cast<ClassInfo*>(p);
    p += align16(sizeof(ClassInfo) * P.n_cls_live);
    uint4* s_desc = reinterpret_cast<uint4*>(p);
    p += 16ull * P.n_desc_live;
    uint16_t* s_col = reinterpret_cast<uint16_t*>(p);
    {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(P.cls);
      uint32_t* dst = reinterpret_cast<uint32_t*>(s_cls);
      for (uint32_t i = threadIdx.x; i < P.n_cls_live * (sizeof(ClassInfo) / 4); i += blockDim.x)
        dst[i] = src[i];
    }
    for (uint32_t i = threadIdx.x; i < P.n_desc_live; i += blockDim.x) s_desc[i] = P.desc[i];
    for (uint64_t i = threadIdx.x; i < P.n_colrow; i += blockDim.x) s_col[i] = P.colrow[i];
    CLS = s_cls;
    DESC = s_desc;
    COLROW = s_col;
  }
  {
    uint4* t4 = reinterpret_cast<uint4*>(tiles);
    for (uint32_t i = threadIdx.x; i < (2 * tile_words) / 4; i += blockDim.x)
      t4[i] = make_uint4(0, 0, 0, 0);
    if (with_counts)
      for (uint32_t i = threadIdx.x; i < P.n_meas * cnt_lanes; i += blockDim.x) cnt[i] = 0;
    if (threadIdx.x < 2) segctr[threadIdx.x] = 0;
  }
  __syncthreads();

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_gen = P.gen_warps;
  const uint32_t n_my =
      n_tiles > blockIdx.x ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;

  if (warp < n_gen) {
    // ---------------- event generators ----------------
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint32_t b = i & 1;
      const uint64_t gtile = tile0 + blockIdx.x + static_cast<uint64_t>(i) * gridDim.x;
      long long tw0 = clock64();
      if (i >= 2) named_sync(kBarEmpty0 + b, blockDim.x);
      long long tw1 = clock64();
      uint32_t* tile = tiles + b * tile_words;
      const uint32_t tile_s = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
      // Fair-coin words of this tile (dense symbols), keyed by (symbol,
      // 128-shot quad), XORed word-wise into the D rows of the symbol's
      // column; the last slot is the constant term (all ones).
      for (uint32_t j = threadIdx.x; j < ((P.n_dense_live + 1) << tw4_log2); j += n_gen * 32) {
        const uint32_t slot = j >> tw4_log2, q = j & (tw4 - 1);
        uint32_t e = __ldg(P.coin_ptr + slot);
        const uint32_t e1 = __ldg(P.coin_ptr + slot + 1);
        if (e == e1) continue;
        uint4 c = make_uint4(kFull, kFull, kFull, kFull);
        if (slot < P.n_dense_live) {
          const uint64_t gq = (gtile << tw4_log2) + q;
          c = philox10(make_uint4(P.dense_sym[slot], static_cast<uint32_t>(gq),
                                  (static_cast<uint32_t>(gq >> 32) & 0xFFFFFFu) | (kDomCoin << 24),
                                  0u),
                       K);
        }
        for (; e < e1; ++e) {
          const uint32_t a = tile_s + ((static_cast<uint32_t>(__ldg(P.coin_rows + e)) + 4 * q) << 2);
          asm volatile(
              "red.shared.xor.b32 [%0], %1;\n\t"
              "red.shared.xor.b32 [%0+4], %2;\n\t"
              "red.shared.xor.b32 [%0+8], %3;\n\t"
              "red.shared.xor.b32 [%0+12], %4;" ::"r"(a),
              "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w)
              : "memory");
        }
      }
      const uint32_t spare = P.n_meas * tw;
      uint32_t seg = 0;
      Segment sg;
      // Exact flip list of (class position, pattern): kLp entries padded
      // with the spare row — u8 row indices when the tile has <= 256 rows
      // (kU8: a list is 4-16 bytes, so the table stays in L1), else u32
      // tile byte offsets (a flip is then one add + one shared XOR). Lists
      // are loaded before the next Philox blocks are computed (pre) where
      // registers allow, so the L1/L2 latency hides under that arithmetic;
      // the rest are issued at the start of emit. Invalid slots load the
      // all-padding list.
      constexpr int kWords = kLp > 0 ? (kU8 ? kLp / 4 : kLp) : 1;  // u32 words per list
      constexpr int kPre = kWords * kSlots <= 32 ? kSlots : (kWords <= 8 && !kPadPred) ? 4 : 0;
      const uint32_t spare_b = spare * 4u;
      const uint32_t row_b = tw * 4u;
      uint32_t lst[kSlots][kWords];
      auto load_lists = [&](auto bern_tag, const Fired& f, int k0, int k1) {
        constexpr bool kB = decltype(bern_tag)::value;
#pragma unroll
        for (int k = 0; k < kSlots; ++k) {
          if (k < k0 || k >= k1 || (!kB && (k & 3) == 3)) continue;
          const uint32_t li =
              ((f.v >> k) & 1u) ? sg.pbase + f.g[k] * sg.npat + f.pat[k] - 1 : P.plist_dummy;
          const uint32_t* src = reinterpret_cast<const uint32_t*>(PLIST) + static_cast<size_t>(li) * kWords;
          if constexpr (kWords == 1) {
            lst[k][0] = __ldg(src);
          } else if constexpr (kWords == 2) {
            const uint2 v = __ldg(reinterpret_cast<const uint2*>(src));
            lst[k][0] = v.x;
            lst[k][1] = v.y;
          } else {
#pragma unroll
            for (int h = 0; h < kWords / 4; ++h) {
              const uint4 v = __ldg(reinterpret_cast<const uint4*>(src) + h);
              lst[k][4 * h] = v.x;
              lst[k][4 * h + 1] = v.y;
              lst[k][4 * h + 2] = v.z;
              lst[k][4 * h + 3] = v.w;
            }
          }
        }
      };
      auto pre = [&](auto bern_tag, const Fired& f) {
        if constexpr (kLp > 0 && kPre > 0) {
          if (!(P.debug_mode & 1u)) load_lists(bern_tag, f, 0, kPre);
        }
      };
      auto emit = [&](auto bern_tag, const Fired& f) {
        constexpr bool kB = decltype(bern_tag)::value;
        if (P.debug_mode & 1u) {
          if (f.v == 0xFFFFFFFFu) tile[0] = f.g[0] ^ f.shot[1] ^ f.pat[2];  // keep the walk alive
          return;
        }
        if constexpr (kLp > 0) {
          if constexpr (kPre > 0 && kPre < kSlots) load_lists(bern_tag, f, kPre, kSlots);
#pragma unroll
          for (int half = 0; half < kSlots; half += 4) {
            if constexpr (kPre == 0) load_lists(bern_tag, f, half, half + 4);
#pragma unroll
            for (int k = half; k < half + 4; ++k) {
              if (!kB && (k & 3) == 3) continue;
              const uint32_t wb = tile_s + ((f.shot[k] >> 5) << 2);
              const uint32_t bit = ((f.v >> k) & 1u) << (f.shot[k] & 31);
#pragma unroll
              for (int e = 0; e < kLp; ++e) {
                uint32_t a;
                bool real;
                if constexpr (kU8) {
                  const uint32_t row = __byte_perm(lst[k][e >> 2], 0u, 0x4440u | (e & 3));
                  a = wb + row * row_b;
                  real = row != P.n_meas;
                } else {
                  a = wb + lst[k][e];
                  real = lst[k][e] != spare_b;
                }
                // kPadPred (many firings per shot): skip padding so the ATOMS
                // pipe only carries real flips; else padding XORs the spare
                // row (never read).
                if (!kPadPred || real)
                  asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(a), "r"(bit) : "memory");
              }
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < kSlots; ++k) {
            if (!kB && (k & 3) == 3) continue;
            if (!((f.v >> k) & 1u)) continue;
            const uint4 d = DESC[sg.goff + f.g[k]];
            const uint32_t bit = 1u << (f.shot[k] & 31);
            uint32_t* wb = tile + (f.shot[k] >> 5);
            uint32_t off = d.x;
            const uint32_t lens[4] = {d.y & 0xFFFFu, d.y >> 16, d.z & 0xFFFFu, d.z >> 16};
#pragma unroll
            for (int s = 0; s < 4; ++s) {
              if ((f.pat[k] >> s) & 1u)
                for (uint32_t j = 0; j < lens[s]; ++j) atomicXor(wb + COLROW[off + j], bit);
              off += lens[s];
            }
          }
        }
      };
      // Segments of this tile, taken from the tile's dispenser one after
      // another; each walk hands over to the next on its last step.
      auto next = [&](Segment& sn) {
        if (lane == 0) seg = atomicAdd(&segctr[b], 1u);
        seg = __shfl_sync(kFull, seg, 0);
        if (seg >= P.n_seg_live || (P.debug_mode & 2u)) return false;
        segment_init(sn, CLS, P.n_cls_live, seg, P.t_log2);
        return true;
      };
      uint4 r[kBlocks];
      bool have = next(sg);
      if (have) {
#pragma unroll
        for (int bb = 0; bb < kBlocks; ++bb) r[bb] = segment_philox(sg, K, gtile, 0, bb, lane);
      }
      while (have) have = segment_walk_chain(sg, r, K, gtile, P.t_log2, lane, pre, emit, next);
      if (P.timers && lane == 0) {  // gen: [0] waiting EMPTY, [1] working
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 0, tw1 - tw0);
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 1, clock64() - tw1);
      }
      named_arrive(kBarFull0 + b, blockDim.x);
    }
  } else {
    // ---------------- drain warps ----------------
    const uint32_t ct = threadIdx.x - n_gen * 32, nct = blockDim.x - n_gen * 32;
    const uint32_t cnt_s = static_cast<uint32_t>(__cvta_generic_to_shared(cnt));
    // row stride in bytes for the fast path's 32x32->64 address multiply
    const uint32_t ldb = ld < (1ull << 29) ? static_cast<uint32_t>(ld * 8) : 0u;
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint32_t b = i & 1;
      const uint64_t t_local = blockIdx.x + static_cast<uint64_t>(i) * gridDim.x;
      long long td0 = clock64();
      named_sync(kBarFull0 + b, blockDim.x);
      long long td1 = clock64();

      uint4* t4 = reinterpret_cast<uint4*>(tiles + b * tile_words);
      const uint32_t t4_s = static_cast<uint32_t>(__cvta_generic_to_shared(t4));
      const uint64_t first = t_local << P.t_log2;
      const uint64_t valid = min(static_cast<uint64_t>(1) << P.t_log2, n_shots - first);
      const uint32_t vq = static_cast<uint32_t>((valid + 127) >> 7);
      const uint32_t rem = static_cast<uint32_t>(valid & 127);
      const bool fast = vec && ldb != 0 && (valid == (static_cast<uint64_t>(1) << P.t_log2));
      // Rows along parent paths (heavy-path decomposition of the L forest):
      // one thread walks a path top-down for one 128-shot column, carrying
      // the running row value; a path's head waits only for its parent's
      // path, which ran in an earlier round.
      for (uint32_t rd = 0; rd < ((P.debug_mode & 8u) ? 0u : P.n_rounds); ++rd) {
        const uint32_t p0 = P.round_ptr[rd], p1 = P.round_ptr[rd + 1];
        const uint32_t tasks = (p1 - p0) << tw4_log2;
        const uint32_t tasks_rounded = (tasks + 31) & ~31u;
        for (uint32_t j = ct; j < tasks_rounded; j += nct) {
          const bool act = j < tasks;
          const uint32_t pth = act ? p0 + (j >> tw4_log2) : p0;
          const uint32_t q = j & (tw4 - 1);
          const int32_t par = act ? PPAR[pth] : -1;
          uint4 prev = par >= 0 ? t4[(static_cast<uint32_t>(par) << tw4_log2) + q]
                                : make_uint4(0, 0, 0, 0);
          const uint32_t xe = act ? PPTR[pth + 1] : 0;
          uint32_t x = act ? PPTR[pth] : 0;
          uint64_t* obase = out + t_local * tile_stride + 2 * q;
          uint8_t* obase_b = reinterpret_cast<uint8_t*>(obase);
          // One row of the path: row = tile word ^ parent row; keep or clear
          // the tile word, store 16 bytes to HBM, optionally count.
          auto row_step = [&](auto fast_tag, auto wp_tag, uint32_t e, uint4 c) {
            constexpr bool kFast = decltype(fast_tag)::value;  // full tile, aligned, ldb < 2^32
            constexpr bool kWarpPath = decltype(wp_tag)::value;  // a warp per path (T = 4096)
            const uint32_t k = e & 0xFFFFu;
            uint4 v = xor4(c, prev);
            // Rows with light children keep their final value for a later
            // round; all others are cleared for tile i+2 right away.
            sts_or_zero(t4_s + (((k << tw4_log2) + q) << 4), v, e >> 31);
            prev = v;
            uint32_t pc = 0;
            if constexpr (kFast) {
              *reinterpret_cast<uint4*>(obase_b + static_cast<uint64_t>(k) * ldb) = v;
              if (with_counts) pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            } else if (q < vq) {
              uint64_t* o = obase + static_cast<uint64_t>(k) * ld;
              bool two = true;  // whether the item's second u64 word is inside the tile
              if (q == vq - 1 && rem) {
                const uint32_t m[4] = {
                    rem >= 32 ? kFull : (1u << rem) - 1,
                    rem >= 64 ? kFull : rem > 32 ? (1u << (rem - 32)) - 1 : 0u,
                    rem >= 96 ? kFull : rem > 64 ? (1u << (rem - 64)) - 1 : 0u,
                    rem > 96 ? (1u << (rem - 96)) - 1 : 0u};
                v.x &= m[0]; v.y &= m[1]; v.z &= m[2]; v.w &= m[3];
                two = rem > 64;
              }
              const uint64_t w0 = (static_cast<uint64_t>(v.y) << 32) | v.x;
              const uint64_t w1 = (static_cast<uint64_t>(v.w) << 32) | v.z;
              if (vec && two) {
                *reinterpret_cast<ulonglong2*>(o) = make_ulonglong2(w0, w1);
              } else {
                o[0] = w0;
                if (two) o[1] = w1;
              }
              if (with_counts) pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            }
            if (with_counts) {
              if constexpr (kWarpPath) {  // per-lane partials, no reduction here
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnt_s + ((k * 32 + lane) << 2)),
                             "r"(pc)
                             : "memory");
              } else {
                if (pc) atomicAdd(&cnt[k], pc);
              }
            }
          };
          // Two rows per iteration with the next row's entry and tile word
          // prefetched (path_rows is padded, so x + 2 <= n_meas is readable).
          auto walk = [&](auto fast_tag, auto wp_tag) {
            uint32_t ea = PROWS[x];
            uint4 ca = t4[((ea & 0xFFFFu) << tw4_log2) + q];
            for (; x + 2 <= xe; x += 2) {
              const uint32_t eb = PROWS[x + 1];
              const uint4 cb = t4[((eb & 0xFFFFu) << tw4_log2) + q];
              row_step(fast_tag, wp_tag, ea, ca);
              ea = PROWS[x + 2];
              ca = t4[((ea & 0xFFFFu) << tw4_log2) + q];
              row_step(fast_tag, wp_tag, eb, cb);
            }
            if (x < xe) row_step(fast_tag, wp_tag, ea, ca);
          };
          if (tw4 >= 32) {
            if (fast) walk(std::true_type{}, std::true_type{});
            else walk(std::false_type{}, std::true_type{});
          } else {
            if (fast) walk(std::true_type{}, std::false_type{});
            else walk(std::false_type{}, std::false_type{});
          }
        }
        // A later round must not start before every row a light child
        // reads is final.
        if (rd + 1 < P.n_rounds) named_sync(kBarDrain, nct);
      }
      if (P.n_keep) {
        named_sync(kBarDrain, nct);  // all light children have read their parents
        for (uint32_t j = ct; j < (P.n_keep << tw4_log2); j += nct)
          t4[(static_cast<uint32_t>(KEEP[j >> tw4_log2]) << tw4_log2) + (j & (tw4 - 1))] =
              make_uint4(0, 0, 0, 0);
      }
      if (ct == 0) segctr[b] = 0;  // all generators are past tile i (FULL[b] completed)
      if (P.timers && lane == 0) {  // drain: [2] waiting FULL, [3] working
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 2, td1 - td0);
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 3, clock64() - td1);
      }
      if (i + 2 < n_my) named_arrive(kBarEmpty0 + b, blockDim.x);
    }
  }
  if (with_counts) {
    __syncthreads();
    if (cnt_lanes == 32) {  // one warp per row: sum the lane partials
      for (uint32_t k = threadIdx.x >> 5; k < P.n_meas; k += blockDim.x >> 5) {
        const uint32_t c = __reduce_add_sync(kFull, cnt[k * 32 + lane]);
        if (lane == 0 && c) atomicAdd(&counts[k], static_cast<unsigned long long>(c));
      }
    } else {
      for (uint32_t i = threadIdx.x; i < P.n_meas; i += blockDim.x)
        if (cnt[i]) atomicAdd(&counts[i], static_cast<unsigned long long>(cnt[i]));
    }
  }
}

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

__global__ void d_segments(const DevPlan P, const RoundKeys K, uint64_t tile0, uint32_t n_tiles,
                           uint64_t n_shots, uint32_t* S32, uint64_t ld32) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t total = static_cast<uint64_t>(P.n_seg_all) * n_tiles;
  for (uint64_t i = warp; i < total; i += nwarps) {
    const uint32_t t = static_cast<uint32_t>(i / P.n_seg_all);
    const uint32_t seg = static_cast<uint32_t>(i - static_cast<uint64_t>(t) * P.n_seg_all);
    const uint64_t base = static_cast<uint64_t>(t) << P.t_log2;
    Segment sg;
    segment_init(sg, P.cls, P.n_cls_all, seg, P.t_log2);
    segment_walk(sg, K, tile0 + t, P.t_log2, lane, [&](auto, const Fired& f) {
      for (int k = 0; k < kSlots; ++k) {
        if (!((f.v >> k) & 1u)) continue;
        const uint64_t j = base + f.shot[k];
        if (j >= n_shots) continue;
        uint32_t s = P.g_first[P.cls_groups[sg.goff + f.g[k]]];
        for (uint32_t pat = f.pat[k]; pat; pat >>= 1, ++s)
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
// Word (row k, 32-shot column c) of a measurement-major (tw32 == 0) or
// tiled (tw32 = T/32) record array.
__device__ __forceinline__ uint64_t rec_word(uint32_t k, uint64_t c, uint64_t ld32,
                                             uint32_t n_meas, uint32_t tw32) {
  if (tw32 == 0) return k * ld32 + c;
  return (c / tw32) * (static_cast<uint64_t>(n_meas) * tw32) + static_cast<uint64_t>(k) * tw32 +
         (c % tw32);
}

__global__ void k3_b8(const uint32_t* __restrict__ m32, uint64_t ld32, uint32_t n_meas,
                      uint64_t n_shots, uint32_t rec, uint8_t* __restrict__ out, bool staged,
                      uint32_t tw32) {
  extern __shared__ __align__(16) uint8_t stage[];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t n_words32 = (n_shots + 31) >> 5;
  const uint32_t kwords = (n_meas + 31) >> 5;
  const uint64_t shot0 = static_cast<uint64_t>(blockIdx.x) * nw * 32;
  const uint64_t col = (shot0 >> 5) + warp;
  const uint64_t my_shot = shot0 + warp * 32 + lane;
  for (uint32_t kw = 0; kw < kwords; ++kw) {
    const uint32_t k = kw * 32 + lane;
    uint32_t x = (k < n_meas && col < n_words32) ? m32[rec_word(k, col, ld32, n_meas, tw32)] : 0u;
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
                      uint64_t n_shots, uint8_t* __restrict__ out, uint32_t tw32) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const uint64_t n_words32 = (n_shots + 31) >> 5;
  const uint64_t col = static_cast<uint64_t>(blockIdx.x) * nw + warp;
  if (col >= n_words32) return;
  const uint64_t shot = col * 32 + lane;
  const uint64_t line = static_cast<uint64_t>(n_meas) + 1;
  const uint32_t kwords = (n_meas + 31) >> 5;
  for (uint32_t kw = 0; kw < kwords; ++kw) {
    const uint32_t k = kw * 32 + lane;
    uint32_t x = k < n_meas ? m32[rec_word(k, col, ld32, n_meas, tw32)] : 0u;
    x = transpose32(x);
    if (shot < n_shots) {
      uint8_t* dst = out + shot * line + kw * 32;
      const uint32_t lim = min(32u, n_meas - kw * 32);
      for (uint32_t b = 0; b < lim; ++b) dst[b] = ((x >> b) & 1u) ? '1' : '0';
    }
  }
  if (shot < n_shots) out[shot * line + n_meas] = '\n';
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

int check_launch() { return cudaGetLastError() == cudaSuccess ? 0 : -1; }

uint64_t host_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

template <class Kern>
int persistent_grid(Kern kernel, const LaunchCfg& L, size_t smem, uint32_t n_tiles,
                    uint32_t max_per_sm, int* grid, int threads = kFusedThreads) {
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -1;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
          cudaSuccess ||
      per_sm < 1)
    return -1;
  per_sm = std::min<int>(per_sm, static_cast<int>(max_per_sm));
  *grid = static_cast<int>(std::min<uint64_t>(n_tiles, static_cast<uint64_t>(per_sm) * L.num_sms));
  return 0;
}

template <bool kStaged, bool kRowStaged, int kLp, bool kPadPred = false, bool kU8 = false>
int launch_k1(const DevPlan& P, const LaunchCfg& L, const RoundKeys& K, uint64_t tile0,
              uint32_t n_tiles, uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t tstride,
              unsigned long long* cnt) {
  auto kern = k1_fused<kStaged, kRowStaged, kLp, kPadPred, kU8>;
  const size_t smem = fused_smem_bytes(P, P.t_log2, kStaged, kRowStaged);
  int grid = 0;
  const int threads = static_cast<int>(P.cta_threads);
  if (persistent_grid(kern, L, smem, n_tiles, P.cta_per_sm, &grid, threads)) return -1;
  const bool vec = (ld % 2 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  kern<<<grid, threads, smem, L.stream>>>(P, K, tile0, n_tiles, n_shots, out, ld, tstride, cnt,
                                          vec);
  return check_launch() ? -1 : 1;
}

}  // namespace

size_t fused_smem_bytes(const DevPlan& P, uint32_t t_log2, bool staged, bool row_staged) {
  const size_t tw = size_t{1} << (t_log2 - 5);
  size_t b = 2 * static_cast<size_t>(P.n_meas + 1) * tw * 4;       // tiles (+ spare row)
  b += align16(4ull * P.n_meas * (t_log2 >= 12 ? 32 : 1)) + 16;   // counts, dispensers
  if (row_staged) {
    b += align16(4ull * (P.n_meas + 1));
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
                        bool tiled) {
  const uint64_t T = 1ull << P.t_log2;
  const uint64_t tstride = tiled ? static_cast<uint64_t>(P.n_meas) * (T / 64) : T / 64;
  if (tiled) ld = T / 64;
  const uint32_t n_tiles = static_cast<uint32_t>((n_shots + T - 1) / T);
  const RoundKeys K = expand_keys(seed);
  auto* cnt = reinterpret_cast<unsigned long long*>(counts);
#define SP_K1(st, rs, lp, pp, u8) \
  launch_k1<st, rs, lp, pp, u8>(P, L, K, tile0, n_tiles, n_shots, out, ld, tstride, cnt)
#define SP_K1R(lp, pp, u8) \
  (P.row_staged ? SP_K1(false, true, lp, pp, u8) : SP_K1(false, false, lp, pp, u8))
#define SP_K1L(lp) \
  (P.pad_pred ? (P.u8 ? SP_K1R(lp, true, true) : SP_K1R(lp, true, false)) \
              : (P.u8 ? SP_K1R(lp, false, true) : SP_K1R(lp, false, false)))
  if (P.lp == 4) return SP_K1L(4);
  if (P.lp == 8) return SP_K1L(8);
  if (P.lp == 16) return SP_K1L(16);
  if (P.staged) return P.row_staged ? SP_K1(true, true, 0, false, false) : SP_K1(true, false, 0, false, false);
  return SP_K1R(0, false, false);
#undef SP_K1
#undef SP_K1R
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
    if (P.n_seg_all) {
      d_segments<<<grid, 256, 0, L.stream>>>(P, K, tile0, n_tiles, n_shots, S32, ld32);
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
                  uint64_t n_shots, int fmt, uint8_t* bytes, uint32_t tile_shots) {
  const uint32_t tw32 = tile_shots / 32;
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
                                                               n_shots, bytes, tw32);
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
        m32, 2 * ld, static_cast<uint32_t>(n_meas), n_shots, rec, bytes, staged, tw32);
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

int launch_debug_philox(const LaunchCfg& L, const uint32_t* ctr_key_dev, uint32_t* out_dev) {
  k_debug_philox<<<1, 1, 0, L.stream>>>(ctr_key_dev, out_dev);
  return check_launch() ? -1 : 1;
}

}  // namespace symphase
