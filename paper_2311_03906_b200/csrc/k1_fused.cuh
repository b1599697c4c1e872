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
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t tw = P.tw, tw4_log2 = P.t_log2 - 7, tw4 = 1u << tw4_log2;
  // Tile rows, then a spare region (never read) that absorbs the XORs of
  // padded flip-list entries, spread over 32 banks.
  const uint32_t tile_words = P.n_meas * tw + spare_words(tw);
  const bool with_counts = counts != nullptr;
  // tiled-layout TMA drain: the stored tile is cleared by a bulk copy of zeros
  const bool tma_zero = bulk == 1 && P.zero_src != nullptr;
  uint32_t* tiles = reinterpret_cast<uint32_t*>(smem);
  // n_buf tile buffers (1..4): with 2+ the generators fill tiles ahead while
  // the drains empty tile i; 1 when two do not fit (very many rows)
  const uint32_t n_buf = P.n_buf;
  uint8_t* p = reinterpret_cast<uint8_t*>(tiles + n_buf * tile_words);
  // Flip counts: per (row, lane) partials when a warp walks one path per
  // 128-shot column group (T = 4096: no cross-lane reduction per row),
  // else one counter per row.
  const uint32_t cnt_lanes = count_lanes(P.t_log2, P.n_buf);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(p);
  p += align16(4ull * P.n_meas * cnt_lanes);
  // Detector flip counts (sp_sample_ex): one u32 per detector.
  const bool with_dets = det_counts != nullptr && P.n_det > 0;
  uint32_t* det_cnt = reinterpret_cast<uint32_t*>(p);  // [n_det + 1 spare][cnt_lanes]
  p += align16(4ull * (P.n_det + (P.n_det ? 1 : 0)) * cnt_lanes);
  const uint32_t det_s = static_cast<uint32_t>(__cvta_generic_to_shared(det_cnt));
  uint32_t* segctr = reinterpret_cast<uint32_t*>(p);  // per-buffer segment dispensers
  p += 16;
  // Tile hand-off: full[b] completes when every generator thread finished
  // its work on the tile in buffer b, empty[b] when every drain thread has
  // emptied it. Each side waits on the other's phase without arriving, so a
  // generator warp that runs out of slices moves on to the next tile
  // without waiting for the other generators.
  uint64_t* mbar_full = reinterpret_cast<uint64_t*>(p);
  uint64_t* mbar_empty = mbar_full + kMaxBuf;
  p += 16 * kMaxBuf;

  const ClassInfo* CLS = P.cls;
  const uint4* DESC = P.desc;
  const uint16_t* COLROW = P.colrow;
  const uint4* PLIST = P.plist;
  const uint32_t* PROWS = P.path_rows;
  const uint32_t* PPTR = P.path_ptr;
  const int32_t* PPAR = P.path_par;
  const uint16_t* KEEP = P.keep_rows;
  const uint32_t* CPTR = P.coin_ptr;
  const uint16_t* CROWS = P.coin_rows;
  const uint32_t* CSYM = P.dense_sym;
  if (kRowStaged) {
    uint32_t* s_prows = reinterpret_cast<uint32_t*>(p);
    p += align16(4ull * (P.n_meas + 4));
    uint32_t* s_pptr = reinterpret_cast<uint32_t*>(p);
    p += align16(4ull * (P.n_paths + 1));
    int32_t* s_ppar = reinterpret_cast<int32_t*>(p);
    p += align16(4ull * P.n_paths);
    uint16_t* s_keep = reinterpret_cast<uint16_t*>(p);
    p += align16(2ull * P.n_keep);
    for (uint32_t i = threadIdx.x; i < P.n_meas + 4; i += blockDim.x) s_prows[i] = P.path_rows[i];
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
    p += align16(2ull * P.n_colrow);  // (what is staged after the tables starts here)
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
  if (!kStaged && P.cls_staged) {  // class table (a few hundred bytes): searched at every slice
    ClassInfo* s_cls = reinterpret_cast<ClassInfo*>(p);
    p += align16(sizeof(ClassInfo) * P.n_cls_live);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(P.cls);
    uint32_t* dst = reinterpret_cast<uint32_t*>(s_cls);
    for (uint32_t i = threadIdx.x; i < P.n_cls_live * (sizeof(ClassInfo) / 4); i += blockDim.x)
      dst[i] = src[i];
    CLS = s_cls;
  }
  // Slice descriptors and length runs (set at launch when they fit): the
  // slice dispenser then resolves a slice with three shared loads.
  const SegDesc* SEGD = P.seg_desc;
  const uint32_t* LENB = P.len_bnd;
  if (P.seg_staged) {
    SegDesc* s_seg = reinterpret_cast<SegDesc*>(p);
    p += align16(sizeof(SegDesc) * P.n_seg_live);
    uint32_t* s_lenb = reinterpret_cast<uint32_t*>(p);
    p += align16(4ull * P.n_len_bnd);
    const uint4* src = reinterpret_cast<const uint4*>(P.seg_desc);
    uint4* dst = reinterpret_cast<uint4*>(s_seg);
    for (uint32_t i = threadIdx.x; i < P.n_seg_live * (sizeof(SegDesc) / 16); i += blockDim.x)
      dst[i] = src[i];
    for (uint32_t i = threadIdx.x; i < P.n_len_bnd; i += blockDim.x) s_lenb[i] = P.len_bnd[i];
    SEGD = s_seg;
    LENB = s_lenb;
  }
  if (P.coins_staged) {  // coin columns and symbols: small, read every tile
    uint32_t* s_cptr = reinterpret_cast<uint32_t*>(p);
    p += align16(4ull * (P.n_dense_live + 2));
    uint32_t* s_csym = reinterpret_cast<uint32_t*>(p);
    p += align16(4ull * P.n_dense_live);
    uint16_t* s_crows = reinterpret_cast<uint16_t*>(p);
    p += align16(2ull * P.n_coin_rows);
    for (uint32_t i = threadIdx.x; i < P.n_dense_live + 2; i += blockDim.x) s_cptr[i] = P.coin_ptr[i];
    for (uint32_t i = threadIdx.x; i < P.n_dense_live; i += blockDim.x) s_csym[i] = P.dense_sym[i];
    for (uint32_t i = threadIdx.x; i < P.n_coin_rows; i += blockDim.x) s_crows[i] = P.coin_rows[i];
    CPTR = s_cptr;
    CSYM = s_csym;
    CROWS = s_crows;
  }
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
      mbar_init(mbar_empty + threadIdx.x, tma_zero ? 1u : blockDim.x - P.gen_warps * 32);
    }
  }
  __syncthreads();

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n_gen = P.gen_warps;
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
      // Fair-coin words of this tile (dense symbols), keyed by (symbol,
      // 128-shot quad), XORed word-wise into the D rows of the symbol's
      // column; the last slot is the constant term (all ones). Two tasks per
      // iteration, so two Philox chains interleave.
      {
        const uint32_t n_tasks = (P.debug_mode & 4u) ? 0u : (P.n_dense_live + 1) << tw4_log2;
        auto coin_word = [&](uint32_t slot, uint32_t q) {
          if (slot >= P.n_dense_live) return make_uint4(kFull, kFull, kFull, kFull);
          const uint64_t gq = (gtile << tw4_log2) + q;
          return philox10(make_uint4(CSYM[slot], static_cast<uint32_t>(gq),
                                     (static_cast<uint32_t>(gq >> 32) & 0xFFFFFFu) | (kDomCoin << 24),
                                     0u),
                          K);
        };
        auto coin_xor = [&](uint32_t slot, uint32_t q, uint4 c) {
          for (uint32_t e = CPTR[slot]; e < CPTR[slot + 1]; ++e) {
            const uint32_t a = tile_s + ((static_cast<uint32_t>(CROWS[e]) + 4 * q) << 2);
            asm volatile(
                "red.shared.xor.b32 [%0], %1;\n\t"
                "red.shared.xor.b32 [%0+4], %2;\n\t"
                "red.shared.xor.b32 [%0+8], %3;\n\t"
                "red.shared.xor.b32 [%0+12], %4;" ::"r"(a),
                "r"(c.x), "r"(c.y), "r"(c.z), "r"(c.w)
                : "memory");
          }
        };
        const uint32_t stride = n_gen * 32;
        uint32_t j = threadIdx.x;
        for (; j + stride < n_tasks; j += 2 * stride) {
          const uint32_t j2 = j + stride;
          const uint4 c0 = coin_word(j >> tw4_log2, j & (tw4 - 1));
          const uint4 c1 = coin_word(j2 >> tw4_log2, j2 & (tw4 - 1));
          coin_xor(j >> tw4_log2, j & (tw4 - 1), c0);
          coin_xor(j2 >> tw4_log2, j2 & (tw4 - 1), c1);
        }
        if (j < n_tasks) coin_xor(j >> tw4_log2, j & (tw4 - 1), coin_word(j >> tw4_log2, j & (tw4 - 1)));
      }
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
    const uint32_t ct = threadIdx.x - n_gen * 32, nct = blockDim.x - n_gen * 32;
    const uint32_t cnt_s = static_cast<uint32_t>(__cvta_generic_to_shared(cnt));
    // row stride in bytes for the fast path's 32x32->64 address multiply
    const uint32_t ldb = ld < (1ull << 29) ? static_cast<uint32_t>(ld * 8) : 0u;
    for (uint32_t i = 0; i < n_my; ++i) {
      const uint32_t b = i % n_buf;
      const uint64_t t_local = blockIdx.x + static_cast<uint64_t>(i) * gridDim.x;
      long long td0 = clock64();
      mbar_wait(mbar_full + b, (i / n_buf) & 1, P.wait_ns);
      long long td1 = clock64();

      uint4* t4 = reinterpret_cast<uint4*>(tiles + b * tile_words);
      const uint32_t t4_s = static_cast<uint32_t>(__cvta_generic_to_shared(t4));
      const uint64_t first = t_local << P.t_log2;
      const uint64_t valid = min(static_cast<uint64_t>(1) << P.t_log2, n_shots - first);
      const uint32_t vq = static_cast<uint32_t>((valid + 127) >> 7);
      const uint32_t rem = static_cast<uint32_t>(valid & 127);
      const bool fast = vec && ldb != 0 && (valid == (static_cast<uint64_t>(1) << P.t_log2));
      uint64_t* const tbase = out + t_local * tile_stride;  // this tile's records
      // Row k's 128-shot column q is final: store 16 bytes to HBM (masked in a
      // partial tile), optionally count its ones.
      if ((bulk || (with_dets && P.flat_rows)) && !(P.debug_mode & 8u)) {
        // In-place drain: rows are rebuilt in place (every final row value
        // stays in the tile), detectors are counted from the finished rows,
        // then the tile leaves for HBM — as TMA bulk copies (one for the
        // whole tile in the tiled layout, one per row segment in the
        // measurement-major one) or 16-byte stores — and is cleared.
        const bool full = valid == (static_cast<uint64_t>(1) << P.t_log2);
        if (!full) {  // a partial tile: shots past the end become zero
          for (uint32_t j = ct; j < (P.n_meas << tw4_log2); j += nct) {
            const uint32_t q = j & (tw4 - 1);
            if (q >= vq) {
              t4[j] = make_uint4(0, 0, 0, 0);
            } else if (q == vq - 1 && rem) {
              uint4 v = t4[j];
              v.x &= rem >= 32 ? kFull : (1u << rem) - 1;
              v.y &= rem >= 64 ? kFull : rem > 32 ? (1u << (rem - 32)) - 1 : 0u;
              v.z &= rem >= 96 ? kFull : rem > 64 ? (1u << (rem - 64)) - 1 : 0u;
              v.w &= rem > 96 ? (1u << (rem - 96)) - 1 : 0u;
              t4[j] = v;
            }
          }
          named_sync(kBarDrain, nct);
        }
        auto count_item = [&](auto wp_tag, uint32_t k, uint4 v) {
          constexpr bool kWarpPath = decltype(wp_tag)::value;  // a warp per row (T = 4096)
          uint32_t pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
          if constexpr (kWarpPath) {
            if (cnt_lanes == 32) {
              asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnt_s + ((k * 32 + lane) << 2)),
                           "r"(pc)
                           : "memory");
            } else {
              pc = __reduce_add_sync(kFull, pc);
              if (lane == 0) atomicAdd(&cnt[k], pc);
            }
          } else {  // branch-free: one shared add per row item
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnt_s + (k << 2)), "r"(pc) : "memory");
          }
        };
        // detector {k, parent(k)} (or {k} for a root row): the row's D value;
        // rows without a detector add into the spare slot n_det (branch-free)
        auto count_det = [&](auto wp_tag, uint32_t e, uint4 d) {
          constexpr bool kWarpPath = decltype(wp_tag)::value;  // the warp holds one row
          const uint32_t slot = min(((e >> 16) & 0x7FFFu) - 1u, P.n_det);
          uint32_t pc = __popc(d.x) + __popc(d.y) + __popc(d.z) + __popc(d.w);
          if constexpr (kWarpPath) {
            if (cnt_lanes == 32) {  // per-lane partials
              asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(det_s + ((slot * 32 + lane) << 2)),
                           "r"(pc)
                           : "memory");
            } else {
              pc = __reduce_add_sync(kFull, pc);
              if (lane == 0) atomicAdd(&det_cnt[slot], pc);
            }
          } else {
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(det_s + (slot << 2)), "r"(pc) : "memory");
          }
        };
        // measurement-major records without TMA: each finished 16-byte item
        // is stored as the rebuild produces it (valid words only)
        const bool direct = bulk == 0 || (bulk == 2 && !full);
        auto store_item = [&](uint32_t k, uint32_t q, uint4 v) {
          if (q >= vq) return;
          const uint64_t w0 = (static_cast<uint64_t>(v.y) << 32) | v.x;
          const uint64_t w1 = (static_cast<uint64_t>(v.w) << 32) | v.z;
          if (fast) {
            *reinterpret_cast<ulonglong2*>(reinterpret_cast<uint8_t*>(tbase + 2 * q) +
                                           static_cast<uint64_t>(k) * ldb) = make_ulonglong2(w0, w1);
            return;
          }
          uint64_t* o = tbase + static_cast<uint64_t>(k) * ld + 2 * q;
          const bool two = q < vq - 1 || rem == 0 || rem > 64;
          if (vec && two) {
            *reinterpret_cast<ulonglong2*>(o) = make_ulonglong2(w0, w1);
          } else {
            o[0] = w0;
            if (two) o[1] = w1;
          }
        };
        // (counting modes are compile-time tags: no per-row flag checks)
        auto rebuild = [&](auto wp_tag, auto cnt_tag, auto det_tag, auto dir_tag) {
          constexpr bool kCnt = decltype(cnt_tag)::value, kDet = decltype(det_tag)::value;
          constexpr bool direct = decltype(dir_tag)::value;
          if (P.flat_rows) {  // no parents: the tile already holds the records
            if (kCnt || direct)
              for (uint32_t j = ct; j < (P.n_meas << tw4_log2); j += nct) {
                const uint4 v = t4[j];
                if constexpr (kCnt) count_item(wp_tag, j >> tw4_log2, v);
                if constexpr (direct) store_item(j >> tw4_log2, j & (tw4 - 1), v);
              }
            return;
          }
          for (uint32_t rd = 0; rd < P.n_rounds; ++rd) {
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
              // four rows per group: the group's entries and tile words are
              // loaded together (path_rows is padded by four entries), then
              // the parent chain runs through them
              auto row = [&](uint32_t e, uint4 c) {
                const uint32_t k = e & 0xFFFFu;
                prev = xor4(c, prev);
                t4[(k << tw4_log2) + q] = prev;
                if constexpr (kCnt) count_item(wp_tag, k, prev);
                if constexpr (kDet) count_det(wp_tag, e, c);
                if constexpr (direct) store_item(k, q, prev);
              };
              for (; x + 4 <= xe; x += 4) {  // whole groups: no per-row checks
                const uint32_t e0 = PROWS[x], e1 = PROWS[x + 1], e2 = PROWS[x + 2], e3 = PROWS[x + 3];
                const uint4 c0 = t4[((e0 & 0xFFFFu) << tw4_log2) + q];
                const uint4 c1 = t4[((e1 & 0xFFFFu) << tw4_log2) + q];
                const uint4 c2 = t4[((e2 & 0xFFFFu) << tw4_log2) + q];
                const uint4 c3 = t4[((e3 & 0xFFFFu) << tw4_log2) + q];
                row(e0, c0);
                row(e1, c1);
                row(e2, c2);
                row(e3, c3);
              }
              for (; x < xe; ++x) {
                const uint32_t e0 = PROWS[x];
                row(e0, t4[((e0 & 0xFFFFu) << tw4_log2) + q]);
              }
            }
            if (rd + 1 < P.n_rounds) named_sync(kBarDrain, nct);
          }
        };
        auto rebuild_dir = [&](auto wp_tag, auto dir_tag) {
          if (with_counts) {
            if (with_dets) rebuild(wp_tag, std::true_type{}, std::true_type{}, dir_tag);
            else rebuild(wp_tag, std::true_type{}, std::false_type{}, dir_tag);
          } else {
            if (with_dets) rebuild(wp_tag, std::false_type{}, std::true_type{}, dir_tag);
            else rebuild(wp_tag, std::false_type{}, std::false_type{}, dir_tag);
          }
        };
        auto rebuild_wp = [&](auto wp_tag) {
          if (direct) rebuild_dir(wp_tag, std::true_type{});
          else rebuild_dir(wp_tag, std::false_type{});
        };
        if (tw4 >= 32) rebuild_wp(std::true_type{});
        else rebuild_wp(std::false_type{});
        // other detectors: XOR of their measurements' finished rows (read
        // while the copy engine reads the same tile)
        auto general_dets = [&]() {
          for (uint32_t j = ct; j < (P.n_gdet << tw4_log2); j += nct) {
            const uint32_t gd = j >> tw4_log2, q = j & (tw4 - 1);
            uint4 v = make_uint4(0, 0, 0, 0);
            for (uint32_t m = P.gdet_ptr[gd]; m < P.gdet_ptr[gd + 1]; ++m)
              v = xor4(v, t4[(static_cast<uint32_t>(P.gdet_rows[m]) << tw4_log2) + q]);
            uint32_t pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            if (tw4 >= 32) {  // the warp holds one detector: one add
              if (cnt_lanes == 32) {  // per-lane partials
                atomicAdd(&det_cnt[P.gdet_id[gd] * 32 + lane], pc);
              } else {
                pc = __reduce_add_sync(kFull, pc);
                if (lane == 0 && pc) atomicAdd(&det_cnt[P.gdet_id[gd]], pc);
              }
            } else if (pc) {
              atomicAdd(&det_cnt[P.gdet_id[gd]], pc);
            }
          }
        };
        if (bulk) fence_proxy_async_smem();
        named_sync(kBarDrain, nct);
        const uint32_t row_bytes = tw * 4u;
        bool issued = false;
        if (bulk == 1) {  // the tiled layout allocates whole tiles
          if (ct == 0) {
            bulk_store(tbase, t4_s, P.n_meas * row_bytes);
            issued = true;
          }
        } else if (bulk == 2 && full) {
          for (uint32_t k = ct; k < P.n_meas; k += nct) {
            bulk_store(tbase + static_cast<uint64_t>(k) * ld, t4_s + k * row_bytes, row_bytes);
            issued = true;
          }
        }
        if (with_dets && P.n_gdet) general_dets();
        if (tma_zero) {
          // every thread is done reading the tile; the elected thread waits
          // until the copy engine has read it and then refills it with zeros
          // by TMA, completing `empty` — the others move on to the next tile
          if (issued) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          named_sync(kBarDrain, nct);
          if (ct == 0) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            segctr[b] = 0;
            if (i + n_buf < n_my) {
              const uint32_t bytes = P.n_meas * row_bytes;
              const uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(mbar_empty + b));
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                           : "memory");
              asm volatile(
                  "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(t4_s),
                  "l"(P.zero_src), "r"(bytes), "r"(bar)
                  : "memory");
            }
          }
        } else {
          if (issued) bulk_commit_and_wait_read();
          named_sync(kBarDrain, nct);  // every row has left the tile
          for (uint32_t j = ct; j < (P.n_meas << tw4_log2); j += nct) t4[j] = make_uint4(0, 0, 0, 0);
          if (ct == 0) segctr[b] = 0;
          if (i + n_buf < n_my) mbar_arrive(mbar_empty + b);
        }
        if (P.timers && lane == 0) {
          atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 2, td1 - td0);
          atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 3, clock64() - td1);
        }
        continue;
      }
      // Legacy drain (16-byte stores while the rows are rebuilt, rows
      // cleared as soon as no later row reads them); the counting modes
      // are compile-time tags, so no per-row flag checks.
      auto legacy = [&](auto cnt_tag, auto det_tag) {
        constexpr bool kCntL = decltype(cnt_tag)::value, kDetL = decltype(det_tag)::value;
        auto store_row = [&](auto fast_tag, auto wp_tag, uint32_t k, uint32_t q, uint4 v) {
          constexpr bool kFast = decltype(fast_tag)::value;  // full tile, aligned, ldb < 2^32
          constexpr bool kWarpPath = decltype(wp_tag)::value;  // a warp per row (T = 4096)
          uint64_t* obase = tbase + 2 * q;
          uint32_t pc = 0;
          if constexpr (kFast) {
            *reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(obase) +
                                      static_cast<uint64_t>(k) * ldb) = v;
            if constexpr (kCntL) pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
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
            if constexpr (kCntL) pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
          }
          if constexpr (kCntL) {
            if constexpr (kWarpPath) {
              if (cnt_lanes == 32) {  // per-lane partials, no reduction here
                asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnt_s + ((k * 32 + lane) << 2)),
                             "r"(pc)
                             : "memory");
              } else {  // the warp holds this row: one add per row
                pc = __reduce_add_sync(kFull, pc);
                if (lane == 0) atomicAdd(&cnt[k], pc);
              }
            } else {
              if (pc) atomicAdd(&cnt[k], pc);
            }
          }
        };
        if (P.flat_rows && !(P.debug_mode & 8u)) {
          // No parents (every row its own path, nothing kept): one pass over
          // the tile in row order, clearing as it goes.
          auto flat = [&](auto fast_tag, auto wp_tag) {
            for (uint32_t j = ct; j < (P.n_meas << tw4_log2); j += nct) {
              const uint4 v = t4[j];
              t4[j] = make_uint4(0, 0, 0, 0);
              store_row(fast_tag, wp_tag, j >> tw4_log2, j & (tw4 - 1), v);
            }
          };
          if (tw4 >= 32) {
            if (fast) flat(std::true_type{}, std::true_type{});
            else flat(std::false_type{}, std::true_type{});
          } else {
            if (fast) flat(std::true_type{}, std::false_type{});
            else flat(std::false_type{}, std::false_type{});
          }
        }
        // Rows along parent paths (heavy-path decomposition of the L forest):
        // one thread walks a path top-down for one 128-shot column, carrying
        // the running row value; a path's head waits only for its parent's
        // path, which ran in an earlier round.
        for (uint32_t rd = 0; rd < ((P.debug_mode & 8u) || P.flat_rows ? 0u : P.n_rounds); ++rd) {
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
            // One row of the path: row = tile word ^ parent row; keep or clear
            // the tile word, then store it (and count it).
            auto row_step = [&](auto fast_tag, auto wp_tag, uint32_t e, uint4 c) {
              const uint32_t k = e & 0xFFFFu;
              const uint4 v = xor4(c, prev);
              if constexpr (kDetL) {  // detector {k, parent(k)} or {k}: the row's D value
                // (rows without a detector add into the spare slot n_det)
                const uint32_t slot = min(((e >> 16) & 0x7FFFu) - 1u, P.n_det);
                uint4 dv = c;
                if (!decltype(fast_tag)::value) {  // a partial tile: valid shots only
                  if (q >= vq) dv = make_uint4(0, 0, 0, 0);
                  else if (q == vq - 1 && rem) {
                    dv.x &= rem >= 32 ? kFull : (1u << rem) - 1;
                    dv.y &= rem >= 64 ? kFull : rem > 32 ? (1u << (rem - 32)) - 1 : 0u;
                    dv.z &= rem >= 96 ? kFull : rem > 64 ? (1u << (rem - 64)) - 1 : 0u;
                    dv.w &= rem > 96 ? (1u << (rem - 96)) - 1 : 0u;
                  }
                }
                uint32_t pc = __popc(dv.x) + __popc(dv.y) + __popc(dv.z) + __popc(dv.w);
                if constexpr (decltype(wp_tag)::value) {
                  if (cnt_lanes == 32) {  // per-lane partials
                    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(det_s + ((slot * 32 + lane) << 2)),
                                 "r"(pc)
                                 : "memory");
                  } else {
                    pc = __reduce_add_sync(kFull, pc);
                    if (lane == 0) atomicAdd(&det_cnt[slot], pc);
                  }
                } else {
                  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(det_s + (slot << 2)), "r"(pc) : "memory");
                }
              }
              // Rows with light children keep their final value for a later
              // round; all others are cleared for tile i+2 right away.
              sts_or_zero(t4_s + (((k << tw4_log2) + q) << 4), v, e >> 31);
              prev = v;
              store_row(fast_tag, wp_tag, k, q, v);
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
        if (kDetL && P.n_gdet && !P.flat_rows) {
          // other detectors: their measurement rows are kept (planner) until
          // the tile ends; XOR them and count
          named_sync(kBarDrain, nct);
          for (uint32_t j = ct; j < (P.n_gdet << tw4_log2); j += nct) {
            const uint32_t gd = j >> tw4_log2, q = j & (tw4 - 1);
            uint4 v = make_uint4(0, 0, 0, 0);
            for (uint32_t m = P.gdet_ptr[gd]; m < P.gdet_ptr[gd + 1]; ++m)
              v = xor4(v, t4[(static_cast<uint32_t>(P.gdet_rows[m]) << tw4_log2) + q]);
            if (q >= vq) v = make_uint4(0, 0, 0, 0);
            else if (q == vq - 1 && rem) {
              v.x &= rem >= 32 ? kFull : (1u << rem) - 1;
              v.y &= rem >= 64 ? kFull : rem > 32 ? (1u << (rem - 32)) - 1 : 0u;
              v.z &= rem >= 96 ? kFull : rem > 64 ? (1u << (rem - 64)) - 1 : 0u;
              v.w &= rem > 96 ? (1u << (rem - 96)) - 1 : 0u;
            }
            uint32_t pc = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
            if (tw4 >= 32) {
              if (cnt_lanes == 32) {  // per-lane partials
                atomicAdd(&det_cnt[P.gdet_id[gd] * 32 + lane], pc);
              } else {
                pc = __reduce_add_sync(kFull, pc);
                if (lane == 0 && pc) atomicAdd(&det_cnt[P.gdet_id[gd]], pc);
              }
            } else if (pc) {
              atomicAdd(&det_cnt[P.gdet_id[gd]], pc);
            }
          }
        }
        if (P.n_keep) {
          named_sync(kBarDrain, nct);  // all light children have read their parents
          for (uint32_t j = ct; j < (P.n_keep << tw4_log2); j += nct)
            t4[(static_cast<uint32_t>(KEEP[j >> tw4_log2]) << tw4_log2) + (j & (tw4 - 1))] =
                make_uint4(0, 0, 0, 0);
        }
      };
      if (with_counts) {
        if (with_dets) legacy(std::true_type{}, std::true_type{});
        else legacy(std::true_type{}, std::false_type{});
      } else {
        if (with_dets) legacy(std::false_type{}, std::true_type{});
        else legacy(std::false_type{}, std::false_type{});
      }
      if (ct == 0) segctr[b] = 0;  // all generators are past tile i (full[b] completed)
      if (P.timers && lane == 0) {  // drain: [2] waiting FULL, [3] working
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 2, td1 - td0);
        atomicAdd(reinterpret_cast<unsigned long long*>(P.timers) + 3, clock64() - td1);
      }
      if (i + n_buf < n_my) mbar_arrive(mbar_empty + b);
    }
  }
  if (with_dets) {
    __syncthreads();
    if (cnt_lanes == 32) {  // per-lane partials: one warp per detector
      for (uint32_t k = threadIdx.x >> 5; k < P.n_det; k += blockDim.x >> 5) {
        const uint32_t c = __reduce_add_sync(kFull, det_cnt[k * 32 + lane]);
        if (lane == 0 && c) atomicAdd(&det_counts[k], static_cast<unsigned long long>(c));
      }
    } else {
      for (uint32_t i = threadIdx.x; i < P.n_det; i += blockDim.x)
        if (det_cnt[i]) atomicAdd(&det_counts[i], static_cast<unsigned long long>(det_cnt[i]));
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

}  // namespace

namespace k1 {
template <bool kStaged, bool kRowStaged, int kLp, bool kPadPred, int kEB>
int launch_k1(const DevPlan& P, const LaunchCfg& L, const RoundKeys& K, uint64_t tile0,
              uint32_t n_tiles, uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t tstride,
              unsigned long long* cnt, unsigned long long* det_cnt) {
  auto kern = k1_fused<kStaged, kRowStaged, kLp, kPadPred, kEB>;
  size_t smem = fused_smem_bytes(P, P.t_log2, kStaged, kRowStaged, P.n_buf);
  DevPlan Q = P;
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
