// Device building blocks shared by the sampling kernels (sm_100a): Philox,
// geometric skips, the reference's keyed draw, the segment walk, named
// barriers and small shared-memory helpers. Included by kernels.cu and the
// fused-kernel variant units (k1_inst.cu).
#pragma once

#include "kernels.cuh"

#include <type_traits>

namespace symphase {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// Named barriers of the fused kernel (0 is __syncthreads).
constexpr uint32_t kMaxBuf = 4;  // shot-tile buffers of the fused kernel
constexpr uint32_t kBarDrain = 1;  // named barrier among the drain warps (0 is __syncthreads)

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

// Geometric skip floor(-ln(u) / -ln(1-p)) from a 24-bit random field f:
// u = (f + 1) * 2^-24 in [2^-24, 1] (so P(u <= x) is exact to 2^-24).
// Computed as lg2(u) * clg with clg = ln2 / ln(1-p) < 0. Near u = 1 the
// series of log2(1 - x) keeps full relative precision where lg2.approx would
// not. Clamped to 2^22 (segments are at most 2^22 trials, so a clamped skip
// still lands past the segment end, and 256 of them cannot overflow u32).
__device__ __forceinline__ uint32_t geo_skip(uint32_t f, float clg) {
  constexpr float kL = 1.4426950408889634f;  // 1 / ln 2
  const float u = static_cast<float>(f + 1u) * 0x1.0p-24f;
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
// lockstep. Every lane draws kBlocks Philox blocks per step, each giving four
// 24-bit skip fields — plus, for DEPOLARIZE, one word whose four base-n
// digits pick the non-identity Pauli of each firing (n = 3 for DEPOLARIZE1
// -> X, Z, Y; n = 15 for DEPOLARIZE2): the joint channel pmf of fill_group
// (sampler.cpp:24-42). Geometric gaps floor(Exp/-ln(1-p)) + 1 are laid
// end to end in lane order with a warp prefix sum, so one step yields up to
// 32 x kSlots firing positions with no divergence. Streams are keyed by
// (segment, global tile), independent of which warp, CTA or GPU runs them.
struct Segment {
  uint32_t g0, s0;  // first trial = (class position g0, shot s0 in the tile)
  uint32_t len, seg, goff, dist, pbase, npat;
  uint32_t lp;      // list entries the class needs (ClassInfo::lp), or of the current run
  uint32_t bnd;     // next length run in len_bnd (0xFFFFFFFF: none)
  uint32_t nbp;     // first class position of that run (0xFFFFFFFF: none)
  float clg;
};

// Philox blocks each lane draws per walk step (independent counters, so the
// two ten-round chains interleave), and the firings one step can yield.
constexpr int kBlocks = kWalkBlocks;
constexpr int kSlots = 4 * kBlocks;

// Firings of one walk step on one lane (slot k valid iff v & (1<<k)).
struct Fired {
  uint32_t v;
  uint32_t g[kSlots], shot[kSlots], pat[kSlots];  // class position, shot in tile, pattern
  uint32_t glast;  // class position of the step's last trial (warp-uniform)
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
  sg.lp = ci.lp;
  sg.clg = ci.clg;
  sg.bnd = ci.bnd;
  sg.nbp = 0xFFFFFFFFu;
}

// Length runs of a sorted class: the run holding class position g0 sets
// sg.lp, and sg.nbp is where the next run starts.
__device__ __forceinline__ void segment_runs(Segment& sg, const uint32_t* len_bnd) {
  if (sg.bnd == 0xFFFFFFFFu) return;
  uint32_t e = len_bnd[sg.bnd];
  sg.lp = e & 31u;
  for (;;) {
    const uint32_t n = len_bnd[sg.bnd + 1];
    if ((n >> 5) > sg.g0) {
      sg.nbp = n >> 5;
      ++sg.bnd;
      return;
    }
    ++sg.bnd;
    sg.lp = n & 31u;
  }
}
// Advance the runs to class position g (non-decreasing along a walk).
__device__ __forceinline__ void segment_runs_to(Segment& sg, const uint32_t* len_bnd, uint32_t g) {
  while (g >= sg.nbp) {
    const uint32_t e = len_bnd[sg.bnd];
    sg.lp = e & 31u;
    const uint32_t n = len_bnd[++sg.bnd];
    sg.nbp = n >> 5;
  }
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
  // floor(d / n) = (d * magic) >> 19, exact for d < n^4 (n = 3, 15)
  const uint32_t magic = n == 3 ? 174763u : 34953u;
  const uint32_t tmask = (1u << t_log2) - 1u;
  uint32_t pos = 0;  // trials consumed (warp-uniform), < len <= 2^22
  uint32_t incl[kSlots];
  uint32_t acc = 0;
  // Gaps of one step's firings from its Philox blocks (inclusive sums).
  auto skips = [&]() {
    acc = 0;
#pragma unroll
    for (int b = 0; b < kBlocks; ++b) {
      // Four 24-bit skip fields per block: the top bits of each word
      // (Bernoulli), or words x, y, z cut into four (DEPOLARIZE, whose
      // word w draws the four patterns).
      uint32_t fld[4];
      if (bern) {
        fld[0] = r[b].x >> 8; fld[1] = r[b].y >> 8; fld[2] = r[b].z >> 8; fld[3] = r[b].w >> 8;
      } else {
        fld[0] = r[b].x >> 8;
        fld[1] = __funnelshift_r(r[b].y, r[b].x, 16) & 0xFFFFFFu;
        fld[2] = __funnelshift_r(r[b].z, r[b].y, 24) & 0xFFFFFFu;
        fld[3] = r[b].z & 0xFFFFFFu;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc += geo_skip(fld[k], sg.clg) + 1u;  // gap to the next firing
        incl[4 * b + k] = acc;
      }
    }
  };
  skips();
  for (uint32_t draw = 0;; ++draw) {
    // warp total (REDUX, off the scan's dependency chain) and inclusive scan
    // of the lanes' gap sums (the shuffle's own in-range predicate guards
    // each add)
    const uint32_t total = __reduce_add_sync(kFull, acc);
    uint32_t scan = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
          "shfl.sync.up.b32 t|p, %0, %1, 0, 0xffffffff;\n\t"
          "@p add.u32 %0, %0, t;\n\t}"
          : "+r"(scan)
          : "r"(o));
    }
    // trial index (relative to the segment) of this lane's firings, minus 1
    const uint32_t base = pos + scan - acc - 1;
    const uint32_t sbase = sg.s0 + base;
    Fired f;
    f.v = 0;
#pragma unroll
    for (int b = 0; b < kBlocks; ++b) {
      // four base-n digits (n^4 <= 50625) from word w: the patterns of the
      // block's four firings, uniform over the n non-identity Paulis
      uint32_t digits = bern ? 0u : __umulhi(r[b].w, n * n * n * n);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int sl = 4 * b + k;
        f.pat[sl] = 1u;
        if (!bern) {
          const uint32_t q = (digits * magic) >> 19;
          f.pat[sl] = 1u + digits - q * n;
          digits = q;
        }
        const uint32_t t = sbase + incl[sl];  // < 2^12 + 2^31: no overflow
        f.g[sl] = sg.g0 + (t >> t_log2);
        f.shot[sl] = t & tmask;
        f.v |= (base + incl[sl] < sg.len ? 1u : 0u) << sl;
      }
    }
    f.glast = sg.g0 + ((sg.s0 + min(pos + total, sg.len) - 1) >> t_log2);
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
      skips();  // the next step's gaps, independent of this step's XORs
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
// Shared-memory mbarriers (sm_90+): arrive counts down, waiters spin on a
// phase parity without arriving, so waiting threads are not coupled.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(a)
               : "memory");
}
// One bounded try of the phase-parity wait (the hardware may suspend the
// warp for a while before returning false).
__device__ __forceinline__ bool mbar_try(uint32_t a, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for the phase with exponential back-off sleeps (32 ns doubling up to
// max_ns): a waiting warp issues a handful of instructions per wait instead
// of polling.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, uint32_t max_ns = 256) {
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
  uint32_t ns = 32;
  while (!mbar_try(a, parity)) {
    __nanosleep(ns);
    ns = min(2 * ns, max_ns);
  }
}


// Bulk (TMA) copies shared -> global for the drain: the async proxy reads the
// tile, so threads that wrote it (generic proxy) fence first; completion is
// tracked per issuing thread with bulk groups.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_and_wait_read() {
  asm volatile(
      "cp.async.bulk.commit_group;\n\t"
      "cp.async.bulk.wait_group.read 0;" ::: "memory");
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

}  // namespace
}  // namespace symphase
