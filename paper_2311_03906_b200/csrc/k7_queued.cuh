// K7, the queued form of the fused Philox sampler: the same slices, streams
// and records as K1 (k1_fused.cuh) bit for bit, with the generator's two
// halves — drawing firing positions and applying their flip lists — split
// over different warps that talk through shared-memory rings.
//
// K1's generator warps stall on the L2 latency of each step's flip-list loads
// (ncu: long-scoreboard stalls lead, 25 % occupancy at 113 registers). Here
//   * walker warps only draw: Philox block -> four geometric gaps -> warp
//     scan -> one u32 per firing, (flip-list index << t_log2) | shot, pushed
//     as one 16-byte shared store per lane into the warp's ring (a batch =
//     one walk step = up to 128 firings, plus a header word: valid count and
//     the longest list of the step's length run);
//   * apply warps wait for a free tile buffer, make the tile's fair-coin
//     words, then pop batches, fetch the four flip lists of their lane through
//     the texture pipe and XOR them into the tile with shared atomics. Their
//     state is tiny, so many of them are resident and the list latency hides
//     behind other warps;
//   * drain warps are K1's (k1_drain.inc), in two teams on alternate tiles.
// Walkers never touch a tile, so they run ahead of the apply warps by the ring
// depth, across tile boundaries. All roles fit 64 registers, so a CTA runs
// 1,024 threads (50 % occupancy). The launch autotune (abi.cpp) times K7
// against K1 per launch kind and keeps the faster (K7).
// Only for plans whose live classes are all one-list Bernoulli (mechanism)
// classes with exact flip lists of at most four u32 words; other plans run K1.
#pragma once

#include "device_common.cuh"

namespace symphase {
namespace {

constexpr uint32_t kQBatch = 128;            // entries per ring slot (one walk step)
constexpr uint32_t kQEnd = 0xFFFFFFFFu;      // header of a tile-end batch

// Shared-memory bytes of the rings: per walker warp `depth` slots of kQBatch
// entries, a header word and a full/empty mbarrier pair per slot.
constexpr uint32_t kQSlotBytes = kQBatch * 4 + 16;  // entries, then the header word (16-byte aligned)
__host__ __device__ constexpr size_t k7_ring_bytes(uint32_t n_walk, uint32_t depth) {
  return static_cast<size_t>(n_walk) * depth * (kQSlotBytes + 16);
}

template <int kThreads, bool kRowStaged, int kLp, int kEB>
__global__ void __launch_bounds__(kThreads, 1)
k7_queued(const DevPlan P, const RoundKeys K, uint64_t tile0, uint32_t n_tiles, uint64_t n_shots,
          uint64_t* __restrict__ out, uint64_t ld, uint64_t tile_stride,
          unsigned long long* __restrict__ counts, bool vec, uint32_t bulk,
          unsigned long long* __restrict__ det_counts) {
  constexpr bool kStaged = false;
#include "k1_prologue.inc"
  // rings: slots [walker][slot] of 128 entries + a header word, then the
  // slots' full / empty mbarriers
  const uint32_t n_gen = P.q_walk, n_app = P.q_apply, dlog = P.q_depth_log2, depth = 1u << dlog;
  p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t{15});
  uint8_t* ring = p;
  p += static_cast<size_t>(n_gen) * depth * kQSlotBytes;
  uint64_t* ring_full = reinterpret_cast<uint64_t*>(p);
  uint64_t* ring_empty = ring_full + n_gen * depth;
  p += static_cast<size_t>(n_gen) * depth * 16;
  {
    uint4* t4 = reinterpret_cast<uint4*>(tiles);
    for (uint32_t i = threadIdx.x; i < (n_buf * tile_words) / 4; i += blockDim.x)
      t4[i] = make_uint4(0, 0, 0, 0);
    if (with_counts)
      for (uint32_t i = threadIdx.x; i < P.n_meas * cnt_lanes; i += blockDim.x) cnt[i] = 0;
    if (with_dets)
      for (uint32_t i = threadIdx.x; i < (P.n_det + 1) * cnt_lanes; i += blockDim.x) det_cnt[i] = 0;
    if (threadIdx.x < kMaxBuf) {
      segctr[threadIdx.x] = 0;
      // a tile is complete when every apply thread (coin words, flip lists) is done with it
      mbar_init(mbar_full + threadIdx.x, n_app * 32);
      mbar_init(mbar_empty + threadIdx.x, tma_zero ? 1u : (blockDim.x - (n_gen + n_app) * 32) / P.drain_teams);
    }
    for (uint32_t i = threadIdx.x; i < n_gen * depth; i += blockDim.x) {
      mbar_init(ring_full + i, 1);   // the walker's elected lane
      mbar_init(ring_empty + i, 1);  // the apply warp's elected lane
    }
  }
  __syncthreads();

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t drain_first = (n_gen + n_app) * 32;  // first drain thread
  const uint32_t n_my =
      n_tiles > blockIdx.x ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;
  const uint32_t per = n_app / n_gen;  // apply warps per walker (batches dealt round robin)
  const uint32_t dmask = depth - 1;    // depth is a power of two

  if (warp < n_gen) {
    // ---------------- walkers ----------------
    // Walkers never touch a tile: they run ahead of the apply warps by up to
    // the ring depth, across tile boundaries. Slice s of the CTA's i-th tile
    // is walked by walker (s + i) mod n_gen (the slices are the streams, so
    // who walks them does not change the records).
    const uint32_t ring_s =
        static_cast<uint32_t>(__cvta_generic_to_shared(ring + warp * depth * kQSlotBytes));
    uint64_t* my_full = ring_full + warp * depth;
    uint64_t* my_empty = ring_empty + warp * depth;
    const uint32_t segd_s = static_cast<uint32_t>(__cvta_generic_to_shared(SEGD));
    uint32_t bno = 0;  // batches pushed so far (all tiles)
    // claim the slot of batch bno (wait until its previous batch was read)
    auto claim = [&]() {
      const uint32_t slot = bno & dmask;
      if (bno >= depth) mbar_wait(my_empty + slot, ((bno >> dlog) - 1) & 1, 32);
      return slot;
    };
    auto publish = [&](uint32_t slot, uint32_t hdr) {
      __syncwarp();
      if (lane == 0) {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(ring_s + slot * kQSlotBytes + kQBatch * 4), "r"(hdr)
                     : "memory");
        mbar_arrive(my_full + slot);
      }
      ++bno;
    };
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint64_t gtile = tile0 + blockIdx.x + static_cast<uint64_t>(i) * gridDim.x;
      uint32_t seg = (warp + n_gen - i % n_gen) % n_gen;
      Segment sg;
      auto fetch = [&](Segment& sn) {
        if (seg >= P.n_seg_live || (P.debug_mode & 2u)) return false;
        // the slice descriptors are staged in shared memory (launch_k7 requires it)
        uint4 a, b2;
        uint32_t clg;
        const uint32_t sa = segd_s + seg * static_cast<uint32_t>(sizeof(SegDesc));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "r"(sa));
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(b2.x), "=r"(b2.y), "=r"(b2.z), "=r"(b2.w) : "r"(sa + 16));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(clg) : "r"(sa + 32));
        sn.g0 = a.x;
        sn.s0 = a.y;
        sn.len = a.z;
        sn.seg = seg;
        sn.pbase = b2.x;
        sn.lp = b2.y >> 16;
        sn.bnd = b2.z;
        sn.nbp = b2.w;
        sn.clg = __uint_as_float(clg);
        seg += n_gen;
        return true;
      };
      bool have = fetch(sg);
      uint4 r = make_uint4(0, 0, 0, 0);
      if (have) r = segment_philox(sg, K, gtile, 0, 0, lane);
      while (have) {
        // One slice, the walk of segment_walk_t<true> (device_common.cuh) with
        // the same counters, gaps and positions; a firing at trial t of the
        // slice has list index pbase + g0 + ((s0 + t) >> t_log2) and shot
        // (s0 + t) & (T - 1), i.e. the entry is ebase + t.
        const uint32_t ebase = ((sg.pbase + sg.g0) << P.t_log2) + sg.s0;
        uint32_t pos = 0;
        for (uint32_t draw = 0;; ++draw) {
          const uint32_t i0 = geo_skip(r.x >> 8, sg.clg) + 1u;
          const uint32_t i1 = i0 + geo_skip(r.y >> 8, sg.clg) + 1u;
          const uint32_t i2 = i1 + geo_skip(r.z >> 8, sg.clg) + 1u;
          const uint32_t acc = i2 + geo_skip(r.w >> 8, sg.clg) + 1u;
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
          const uint32_t base = pos + scan - acc - 1;  // trial of this lane's firings, minus the gaps
          const uint32_t t0 = base + i0, t1 = base + i1, t2 = base + i2, t3 = base + acc;
          const uint32_t endpos = min(pos + total, sg.len);
          const uint32_t glast = sg.g0 + ((sg.s0 + endpos - 1) >> P.t_log2);
          pos += total;
          const bool more = pos < sg.len;
          // valid firings are a prefix in (lane, slot) order
          uint32_t n_valid = kQBatch;
          if (!more)
            n_valid = __reduce_add_sync(kFull, (t0 < sg.len ? 1u : 0u) + (t1 < sg.len ? 1u : 0u) +
                                                   (t2 < sg.len ? 1u : 0u) + (t3 < sg.len ? 1u : 0u));
          if (glast >= sg.nbp) segment_runs_to(sg, LENB, glast);
          const uint32_t lpu = sg.lp == 0 ? static_cast<uint32_t>(kLp) : sg.lp;
          Segment sn;
          bool have_next = false;
          if (more) {
            r = segment_philox(sg, K, gtile, draw + 1, 0, lane);
          } else {
            have_next = fetch(sn);
            if (have_next) r = segment_philox(sn, K, gtile, 0, 0, lane);
          }
          if (n_valid && !(P.debug_mode & 1u)) {
            const uint32_t slot = claim();
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(
                             ring_s + slot * kQSlotBytes + (lane << 4)),
                         "r"(ebase + t0), "r"(ebase + t1), "r"(ebase + t2), "r"(ebase + t3)
                         : "memory");
            publish(slot, n_valid | (lpu << 8));
          }
          if (!more) {
            if (have_next) sg = sn;
            have = have_next;
            break;
          }
        }
      }
      // tile end: one end batch to each of this walker's apply warps
      for (uint32_t c = 0; c < per; ++c) {
        const uint32_t slot = claim();
        publish(slot, kQEnd);
      }
    }
  } else if (warp < n_gen + n_app) {
    // ---------------- apply warps ----------------
    const uint32_t aw = warp - n_gen;
    const uint32_t src = aw / per, sub = aw - src * per;
    const uint32_t ring_s =
        static_cast<uint32_t>(__cvta_generic_to_shared(ring + src * depth * kQSlotBytes));
    uint64_t* my_full = ring_full + src * depth;
    uint64_t* my_empty = ring_empty + src * depth;
    constexpr int kWords = kLp * kEB / 4;  // u32 words per list (<= 4)
    static_assert(kWords >= 1 && kWords <= 4, "K7 keeps a lane's four lists in registers");
    const uint32_t tmask = (1u << P.t_log2) - 1u;
    const uint32_t row_b = tw * 4u;
    const uint32_t coin_tid = threadIdx.x - n_gen * 32, coin_stride = n_app * 32;
    uint32_t cb = sub;  // this warp's next batch of its walker
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint32_t b = i % n_buf;
      const uint64_t gtile = tile0 + blockIdx.x + static_cast<uint64_t>(i) * gridDim.x;
      const long long ta0 = clock64();
      if (i >= n_buf) mbar_wait(mbar_empty + b, ((i / n_buf) - 1) & 1, P.wait_ns);
      if (P.timers && lane == 0)  // [0] apply warps waiting for an empty tile buffer
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 0, clock64() - ta0);
      const uint32_t tile_s =
          static_cast<uint32_t>(__cvta_generic_to_shared(tiles + b * tile_words));
#include "k1_coins.inc"
      for (;;) {
        const uint32_t slot = cb & dmask;
        mbar_wait(my_full + slot, (cb >> dlog) & 1, 32);
        uint32_t hdr;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(hdr) : "r"(ring_s + slot * kQSlotBytes + kQBatch * 4)
                     : "memory");
        uint4 e;  // (an end batch's entries are stale and unused)
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w)
                     : "r"(ring_s + slot * kQSlotBytes + (lane << 4))
                     : "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(my_empty + slot);  // the slot can be refilled
        cb += per;
        if (hdr == kQEnd) break;
        const uint32_t n_valid = hdr & 0xFFu, lpu = hdr >> 8;
        const uint32_t ent[4] = {e.x, e.y, e.z, e.w};
        uint32_t lst[4][kWords];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const bool ok = 4 * lane + k < n_valid;
          const uint32_t li = ok ? ent[k] >> P.t_log2 : P.plist_dummy;
          // texture pipe: keeps these scattered loads off the LSU data pipe
          if constexpr (kWords == 1) {
            lst[k][0] = tex1Dfetch<unsigned int>(P.plist_tex, static_cast<int>(li));
          } else if constexpr (kWords == 2) {
            const uint2 v = tex1Dfetch<uint2>(P.plist_tex, static_cast<int>(li));
            lst[k][0] = v.x;
            lst[k][1] = v.y;
          } else {
            const uint4 v = tex1Dfetch<uint4>(P.plist_tex, static_cast<int>(li));
            lst[k][0] = v.x;
            lst[k][1] = v.y;
            lst[k][2] = v.z;
            lst[k][3] = v.w;
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t shot = ent[k] & tmask;
          const uint32_t wb = tile_s + ((shot >> 5) << 2);
          // an invalid slot XORs zero (its list is the all-padding one)
          const uint32_t bit = (4 * lane + k < n_valid ? 1u : 0u) << (shot & 31);
#pragma unroll
          for (int en = 0; en < kLp; ++en) {
            // the run's lists end by entry lpu (warp-uniform), checked per pair
            if (en >= 2 && (en & 1) == 0 && lpu <= static_cast<uint32_t>(en)) break;
            uint32_t a;
            if constexpr (kEB == 1) {
              const uint32_t row = __byte_perm(lst[k][en >> 2], 0u, 0x4440u | (en & 3));
              a = wb + row * row_b;
            } else if constexpr (kEB == 2) {
              const uint32_t w = lst[k][en >> 1];
              a = wb + ((en & 1) ? (w >> 16) : (w & 0xFFFFu));
            } else {
              a = wb + lst[k][en];
            }
            asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(a), "r"(bit) : "memory");
          }
        }
      }
      // tile end: this warp's XORs are done
      if (bulk) fence_proxy_async_smem();
      mbar_arrive(mbar_full + b);
      if (P.timers && lane == 0)  // [1] apply warps: whole tile, wait included
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 1, clock64() - ta0);
    }
  } else {
    // ---------------- drain warps ----------------
#include "k1_drain.inc"
  }
#include "k1_epilogue.inc"
}

}  // namespace

namespace k7 {
// Returns 1 when launched, 0 when the plan does not fit this variant (the
// caller runs K1), < 0 on a CUDA error.
template <int kThreads, bool kRowStaged, int kLp, int kEB>
int launch_k7(const DevPlan& P, const LaunchCfg& L, const RoundKeys& K, uint64_t tile0,
              uint32_t n_tiles, uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t tstride,
              unsigned long long* cnt, unsigned long long* det_cnt) {
  auto kern = k7_queued<kThreads, kRowStaged, kLp, kEB>;
  size_t smem = fused_smem_bytes(P, P.t_log2, false, kRowStaged, P.n_buf) + 16 +
                k7_ring_bytes(P.q_walk, 1u << P.q_depth_log2);
  if (smem > L.smem_optin) return 0;
  DevPlan Q = P;
  Q.drain_teams = (kThreads / 32 - P.q_walk - P.q_apply) % P.q_drain_teams == 0 && P.n_buf >= 2
                      ? P.q_drain_teams : 1;
  const size_t cls_bytes = align16(sizeof(ClassInfo) * P.n_cls_live);
  Q.cls_staged = smem + cls_bytes <= L.smem_optin;
  if (Q.cls_staged) smem += cls_bytes;
  const size_t seg_bytes = align16(sizeof(SegDesc) * P.n_seg_live) + align16(4ull * P.n_len_bnd);
  Q.seg_staged = P.seg_desc != nullptr && P.n_seg_live > 0 && smem + seg_bytes <= L.smem_optin;
  if (!Q.seg_staged || !P.plist_tex) return 0;  // the walkers read the slices from shared memory
  smem += seg_bytes;
  int grid = 0;
  if (persistent_grid(kern, L, smem, n_tiles, 1, &grid, kThreads)) return -1;
  const bool vec = (ld % 2 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const uint32_t bulk = !P.bulk_store || !vec ? 0u
                        : (ld * 2 == P.tw && tstride == static_cast<uint64_t>(P.n_meas) * ld) ? 1u
                        : P.bulk_store == 2 && P.tw * 4 >= 128 ? 2u : 0u;
  kern<<<grid, kThreads, smem, L.stream>>>(Q, K, tile0, n_tiles, n_shots, out, ld, tstride, cnt,
                                           vec, bulk, det_cnt);
  return check_launch() ? -1 : 1;
}
}  // namespace k7
}  // namespace symphase
