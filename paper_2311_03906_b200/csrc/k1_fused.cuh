// K1, the fused warp-specialised Philox sampler, as a template over its
// launch shape. Instantiated per (flip-list length, entry width) in separate
// units (k1_inst.cu, built once per variant) so the variants compile in
// parallel; kernels.cu dispatches to them through launch_k1.
#pragma once

#include "device_common.cuh"

namespace symphase {
namespace {

// ---- K1: fused, warp-specialised Philox sampler ---------------------------
//
// The planner rewrites M_sym = L·D (abi.cpp, chain transform): each row k has
// at most one earlier parent row p(k) and D row k = row k XOR row p(k), which
// for syndrome-extraction circuits is the detector-like difference of
// consecutive rounds — far fewer symbols per column. The kernel samples in
// D space and rebuilds M rows along parent paths (out[k] = d[k] ^ out[p(k)]).
//
// Per CTA (one per SM, 16 warps): n_buf shared-memory accumulation tiles
// [n_meas][T/32] u32 plus a spare region. Generator warps make each tile's
// fair-coin words and XOR them into the coins' D columns, then walk the
// tile's sampling slices (warp-cooperative geometric skips) and XOR each
// firing's flip list into the tile with shared atomics. Drain warps, once a
// tile is complete, rebuild rows along the heavy paths of the parent forest
// (or in one flat pass when there are no parents), stream the records to
// HBM with 16-byte stores, count, and clear the tile for reuse. mbarriers
// full[b] / empty[b] hand the buffers back and forth; each side waits
// without arriving, so generator warps never wait for one another. Row,
// coin and (table-walk variant) event tables are staged in shared memory
// when they fit.
template <bool kStaged, bool kRowStaged, int kLp, bool kPadPred, int kEB>
__global__ void __launch_bounds__(kFusedThreads, 1)
k1_fused(const DevPlan P, const RoundKeys K, uint64_t tile0, uint32_t n_tiles, uint64_t n_shots,
         uint64_t* __restrict__ out, uint64_t ld, uint64_t tile_stride,
         unsigned long long* __restrict__ counts, bool vec, uint32_t bulk,
         unsigned long long* __restrict__ det_counts) {
#include "k1_prologue.inc"
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
      mbar_init(mbar_full + threadIdx.x, P.gen_warps * 32);
      // TMA drain: one elected arrival + the zero-fill copy's bytes
      mbar_init(mbar_empty + threadIdx.x, tma_zero ? 1u : (blockDim.x - P.gen_warps * 32) / P.drain_teams);
    }
  }
  __syncthreads();

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_gen = P.gen_warps;
  const uint32_t drain_first = n_gen * 32;  // first drain thread
  const uint32_t coin_tid = threadIdx.x, coin_stride = n_gen * 32;  // the generators make the coin words
  const uint32_t n_my =
      n_tiles > blockIdx.x ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0u;

  if (warp < n_gen) {
    // ---------------- event generators ----------------
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint32_t b = i % n_buf;
      const uint64_t gtile = tile0 + blockIdx.x + static_cast<uint64_t>(i) * gridDim.x;
      long long tw0 = clock64();
      if (i >= n_buf) mbar_wait(mbar_empty + b, ((i / n_buf) - 1) & 1, P.wait_ns);
      long long tw1 = clock64();
      uint32_t* tile = tiles + b * tile_words;
      const uint32_t tile_s = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
#include "k1_coins.inc"
      const uint32_t spare = P.n_meas * tw;
      uint32_t seg = 0;
      Segment sg;
      // Exact flip list of (class position, pattern): kLp entries of kEB
      // bytes padded with spare-region entries — u8 row indices when the
      // tile has < 256 rows, u16 tile byte offsets when the tile is under
      // 64 KB, else u32 byte offsets — so the table is as small as possible
      // (L1/L2-resident) and a flip costs at most one extract, one add and
      // one shared XOR. Lists are loaded before the next Philox blocks are
      // computed (pre) where registers allow, so the L1/L2 latency hides
      // under that arithmetic; the rest are issued at the start of emit.
      // Invalid slots load the all-padding list.
      constexpr int kWords = kLp > 0 ? kLp * kEB / 4 : 1;  // u32 words per list
      constexpr int kPre = kWords * kSlots <= 32 ? kSlots : (kWords <= 8 && !kPadPred) ? 4 : 0;
      const uint32_t spare_b = spare * 4u;  // u16/u32 entries >= spare_b are padding
      const uint32_t row_b = tw * 4u;
      uint32_t lst[kSlots][kWords];
      auto load_lists = [&](auto, const Fired& f, int k0, int k1) {
#pragma unroll
        for (int k = 0; k < kSlots; ++k) {
          if (k < k0 || k >= k1) continue;
          const uint32_t li =
              ((f.v >> k) & 1u) ? sg.pbase + f.g[k] * sg.npat + f.pat[k] - 1 : P.plist_dummy;
          const uint32_t* src = reinterpret_cast<const uint32_t*>(PLIST) + static_cast<size_t>(li) * kWords;
          if (P.plist_tex) {  // texture pipe: keeps these scattered loads off the LSU data pipe
            if constexpr (kWords == 1) {
              lst[k][0] = tex1Dfetch<unsigned int>(P.plist_tex, static_cast<int>(li));
            } else if constexpr (kWords == 2) {
              const uint2 v = tex1Dfetch<uint2>(P.plist_tex, static_cast<int>(li));
              lst[k][0] = v.x;
              lst[k][1] = v.y;
            } else {
#pragma unroll
              for (int h = 0; h < kWords / 4; ++h) {
                const uint4 v = tex1Dfetch<uint4>(P.plist_tex, static_cast<int>(li * (kWords / 4) + h));
                lst[k][4 * h] = v.x;
                lst[k][4 * h + 1] = v.y;
                lst[k][4 * h + 2] = v.z;
                lst[k][4 * h + 3] = v.w;
              }
            }
            continue;
          }
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
        if (P.timers) {  // profiling counters: [4] walk steps, [5] firings
          const uint32_t nv = __reduce_add_sync(kFull, __popc(f.v));
          if (lane == 0) {
            atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 4, 1ull);
            atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 5,
                      static_cast<unsigned long long>(nv));
          }
        }
        if (P.debug_mode & 1u) {
          if (f.v == 0xFFFFFFFFu) tile[0] = f.g[0] ^ f.shot[1] ^ f.pat[2];  // keep the walk alive
          return;
        }
        if constexpr (kLp > 0) {
          // length runs: the step's longest list is at its last trial
          // (warp-uniform; a run boundary is crossed rarely)
          if (f.glast >= sg.nbp) segment_runs_to(sg, LENB, f.glast);
          const uint32_t lpu = sg.lp == 0 ? static_cast<uint32_t>(kLp) : sg.lp;
          if constexpr (kPre > 0 && kPre < kSlots) load_lists(bern_tag, f, kPre, kSlots);
#pragma unroll
          for (int half = 0; half < kSlots; half += 4) {
            if constexpr (kPre == 0) load_lists(bern_tag, f, half, half + 4);
#pragma unroll
            for (int k = half; k < half + 4; ++k) {
              const uint32_t wb = tile_s + ((f.shot[k] >> 5) << 2);
              const uint32_t bit = ((f.v >> k) & 1u) << (f.shot[k] & 31);
#pragma unroll
              for (int e = 0; e < kLp; ++e) {
                // the class's (or length run's) lists end by entry lpu
                // (warp-uniform): skip the padding
                // (checked per pair of entries: an odd length runs one
                // padding entry, which XORs the spare region)
                if (e >= 2 && (e & 1) == 0 && lpu <= static_cast<uint32_t>(e)) break;
                uint32_t a;
                bool real;
                if constexpr (kEB == 1) {
                  const uint32_t row = __byte_perm(lst[k][e >> 2], 0u, 0x4440u | (e & 3));
                  a = wb + row * row_b;
                  real = row != P.n_meas;
                } else if constexpr (kEB == 2) {
                  const uint32_t w = lst[k][e >> 1];
                  const uint32_t x = (e & 1) ? (w >> 16) : (w & 0xFFFFu);
                  a = wb + x;
                  real = x < spare_b;
                } else {
                  a = wb + lst[k][e];
                  real = lst[k][e] < spare_b;
                }
                // kPadPred (many firings per shot): skip padding so the ATOMS
                // pipe only carries real flips; else padding XORs the spare
                // row (never read).
                if constexpr (kPadPred) {
                  // predicated in PTX: an asm statement under a C++ branch
                  // would compile to a divergent branch per entry
                  asm volatile(
                      "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t"
                      "@p red.shared.xor.b32 [%0], %1;\n\t}" ::"r"(a),
                      "r"(bit), "r"(real ? 1u : 0u)
                      : "memory");
                } else {
                  asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(a), "r"(bit) : "memory");
                }
              }
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < kSlots; ++k) {
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
        if (P.seg_staged) {
          const SegDesc& e = SEGD[seg];
          sn.g0 = e.g0;
          sn.s0 = e.s0;
          sn.len = e.len;
          sn.seg = seg;
          sn.goff = e.goff;
          sn.pbase = e.pbase;
          sn.npat = e.meta & 0xFFu;
          sn.dist = (e.meta >> 8) & 0xFFu;
          sn.lp = e.meta >> 16;
          sn.bnd = e.bnd;
          sn.nbp = e.nbp;
          sn.clg = e.clg;
        } else {
          segment_init(sn, CLS, P.n_cls_live, seg, P.t_log2);
          segment_runs(sn, LENB);
        }
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
      // the drain's TMA copy (async proxy) reads what these XORs wrote
      if (bulk) fence_proxy_async_smem();
      mbar_arrive(mbar_full + b);
    }
  } else {
    // ---------------- drain warps ----------------
#include "k1_drain.inc"
  }
#include "k1_epilogue.inc"
}

}  // namespace

namespace k1 {
template <bool kStaged, bool kRowStaged, int kLp, bool kPadPred, int kEB>
int launch_k1(const DevPlan& P, const LaunchCfg& L, const RoundKeys& K, uint64_t tile0,
              uint32_t n_tiles, uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t tstride,
              unsigned long long* cnt, unsigned long long* det_cnt) {
  auto kern = k1_fused<kStaged, kRowStaged, kLp, kPadPred, kEB>;
  size_t smem = fused_smem_bytes(P, P.t_log2, kStaged, kRowStaged, P.n_buf);
  DevPlan Q = P;
  // drain teams need whole warps each
  if ((P.cta_threads / 32 - P.gen_warps) % P.drain_teams != 0) Q.drain_teams = 1;
  const size_t cls_bytes = align16(sizeof(ClassInfo) * P.n_cls_live);
  Q.cls_staged = !kStaged && smem + cls_bytes <= L.smem_optin;
  if (Q.cls_staged) smem += cls_bytes;
  const size_t seg_bytes = align16(sizeof(SegDesc) * P.n_seg_live) + align16(4ull * P.n_len_bnd);
  Q.seg_staged = P.seg_stage_ok && P.seg_desc != nullptr && P.n_seg_live > 0 &&
                 smem + seg_bytes <= L.smem_optin;
  if (Q.seg_staged) smem += seg_bytes;
  int grid = 0;
  const int threads = static_cast<int>(P.cta_threads);
  if (persistent_grid(kern, L, smem, n_tiles, P.cta_per_sm, &grid, threads)) return -1;
  const bool vec = (ld % 2 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  // TMA bulk stores of finished tiles: 1 = the whole tile is one contiguous
  // block (tiled layout), 2 = one copy per row segment (measurement-major,
  // worth it from 128-byte segments up), 0 = per-thread 16-byte stores.
  // (per-row copies measured slower than the 16-byte stores at cfg2: 145
  // rows x 512 bytes per tile; SP_BULK=2 forces them)
  const uint32_t bulk = !P.bulk_store || !vec ? 0u
                        : (ld * 2 == P.tw && tstride == static_cast<uint64_t>(P.n_meas) * ld) ? 1u
                        : P.bulk_store == 2 && P.tw * 4 >= 128 ? 2u : 0u;
  kern<<<grid, threads, smem, L.stream>>>(Q, K, tile0, n_tiles, n_shots, out, ld, tstride, cnt,
                                          vec, bulk, det_cnt);
  return check_launch() ? -1 : 1;
}

}  // namespace k1
}  // namespace symphase
