// K5 — column sampler for dense M_sym (sm_100a).
//
// When faults flip many measurements each (cfg5 at density 0.5: ~5,000 rows
// per fault symbol, 10-1,000 firings per shot), one shared atomic per flipped
// bit (K1) is hopeless and drawing S for the explicit product (K2) does
// n_meas x n_sym / 8 table lookups per 64 shots whatever the fault rate. K5
// instead keeps each shot's record in shared memory, shot-major (n_meas bits
// = ncw u32 words per shot), and XORs the dense M_sym column of every fired
// symbol into it with the whole warp: 16-byte loads of the column (L2), one
// 16-byte shared read-modify-write per lane and 4 words. Work is
// firings x ncw words — proportional to the fault rate, not to n_sym.
//
// Streams: one geometric-skip walk per (class, global shot) over the class's
// groups, the same warp-cooperative walk as K1 (device_common.cuh), keyed by
// (class | 2^31, global shot), so the records do not depend on the launch
// shape, and the draw mode (sp_draw_assignments) sets exactly the symbol bits
// the sampler XORs: records == M_sym . S(draw) bit for bit.
//
// Per CTA (512 threads, persistent over shot tiles of T = 32..128 shots):
// records initialised to the constant row (s0, p >= 1), warp w walks shots
// w, w + 16, ... (a warp owns its shots, so the column XORs need no atomics),
// then each warp turns 32 x 32 blocks of records into measurement-major words
// (warp bit transpose) and stores a row's T/32 words together, with per-row
// popcounts into shared counters.
#include "device_common.cuh"

#include <algorithm>

namespace symphase {
namespace {

constexpr int kK5Threads = 512;
constexpr int kK5Warps = kK5Threads / 32;
#ifndef K5_G
#define K5_G 8
#endif
#ifndef K5_UNR
#define K5_UNR 1
#endif
constexpr uint32_t kK5G = K5_G;
constexpr int kK5Unroll = K5_UNR;     // columns XORed per record pass (their loads in flight together)
// per-warp list of one step's fired symbols (32 lanes x 4 slots), padded to
// whole column groups with the zero column n_sym
constexpr uint32_t kK5Scratch = 128 + kK5G;

__device__ __forceinline__ uint32_t transpose32_k5(uint32_t x, uint32_t lane) {
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

template <bool kDraw>
__global__ void __launch_bounds__(kK5Threads, 1)
k5_columns(const K5Plan P, const RoundKeys K, uint64_t shot_begin, uint64_t n_shots,
           uint64_t* __restrict__ out, uint64_t ld, unsigned long long* __restrict__ counts,
           uint32_t* __restrict__ S32, uint64_t ld32) {
  extern __shared__ __align__(16) uint8_t smem[];
  const uint32_t T = 1u << P.t_log2, ncw = P.ncw;
  uint32_t* rec = reinterpret_cast<uint32_t*>(smem);  // [T][ncw]
  uint32_t* cnt = rec + (kDraw ? 0u : T * ncw);       // [n_meas]
  uint32_t* scratch = cnt + (kDraw ? 0u : P.n_meas) + (threadIdx.x >> 5) * kK5Scratch;  // this warp's list
  const bool with_counts = !kDraw && counts != nullptr;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (with_counts)
    for (uint32_t i = threadIdx.x; i < P.n_meas; i += blockDim.x) cnt[i] = 0;
  const uint64_t n_tiles = (n_shots + T - 1) >> P.t_log2;
  const uint32_t nw = (P.n_meas + 31) / 32;  // row words of a record
  const uint32_t n_cls = kDraw ? P.n_cls : P.n_cls_live;
  for (uint64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const uint64_t j0 = tile << P.t_log2;  // first shot of the tile (relative)
    const uint32_t valid = static_cast<uint32_t>(n_shots - j0 < T ? n_shots - j0 : T);
    if (!kDraw) {
      const uint4* c4 = reinterpret_cast<const uint4*>(P.row_const);
      uint4* r4 = reinterpret_cast<uint4*>(rec);
      const uint32_t q = ncw / 4;
      for (uint32_t i = threadIdx.x; i < T * q; i += blockDim.x) r4[i] = __ldg(c4 + i % q);
      __syncthreads();
    }
    // Symbol chunks (chunk-major over the warp's shots): every warp of every
    // CTA walks the same slice of the model's columns at about the same
    // time, so that slice stays L2-resident; a class's walk restarts at each
    // chunk (its own stream), which the draw mode follows too.
    for (uint32_t ch = 0; ch < P.n_chunks; ++ch)
    for (uint32_t s = warp; s < valid; s += kK5Warps) {
      const uint64_t gs = shot_begin + j0 + s;  // global shot: the stream key
      uint4* r4 = reinterpret_cast<uint4*>(rec + s * ncw);
      for (uint32_t c = 0; c < n_cls; ++c) {
        const ClassInfo ci = P.cls[c];
        const uint32_t g_lo = static_cast<uint32_t>(ci.trials * ch / P.n_chunks);
        const uint32_t g_hi = static_cast<uint32_t>(ci.trials * (ch + 1) / P.n_chunks);
        if (g_lo == g_hi) continue;
        Segment sg;
        sg.g0 = g_lo;
        sg.s0 = 0;
        sg.len = g_hi - g_lo;
        sg.seg = 0x80000000u | (ch << 16) | c;
        sg.goff = ci.goff;
        sg.dist = ci.dist;
        sg.pbase = 0;
        sg.npat = ci.npat;
        sg.lp = 0;
        sg.clg = ci.clg;
        // XOR the compacted symbols scratch[0 .. total) into the record
        // kK5G columns at a time: each lane owns 16-byte chunks of the
        // record, the group's column loads are in flight together, and the
        // record is read and written once per group.
        auto xor_list = [&](uint32_t total) {
          // pad the list to whole groups with the zero column: every group
          // issues kK5G loads, branch-free; offsets are u32 (uint4 units)
          const uint32_t padded = (total + kK5G - 1) / kK5G * kK5G;
          if (lane < padded - total) scratch[total + lane] = P.n_sym;
          __syncwarp();
          const uint32_t q = ncw / 4;
          const uint4* base = reinterpret_cast<const uint4*>(P.cols);
          for (uint32_t i0 = 0; i0 < padded; i0 += kK5G) {
            uint32_t off[kK5G];
#pragma unroll
            for (uint32_t t = 0; t < kK5G; ++t) off[t] = scratch[i0 + t] * q + lane;
#pragma unroll kK5Unroll
            for (uint32_t w4 = lane; w4 < q; w4 += 32) {
              uint4 acc = __ldg(base + off[0]);
#pragma unroll
              for (uint32_t t = 1; t < kK5G; ++t) {
                const uint4 c = __ldg(base + off[t]);
                acc.x ^= c.x; acc.y ^= c.y; acc.z ^= c.z; acc.w ^= c.w;
              }
#pragma unroll
              for (uint32_t t = 0; t < kK5G; ++t) off[t] += 32;
              uint4 r = r4[w4];
              r.x ^= acc.x; r.y ^= acc.y; r.z ^= acc.z; r.w ^= acc.w;
              r4[w4] = r;
            }
          }
        };
        auto warp_excl = [&](uint32_t mine, uint32_t& total) {  // exclusive prefix + total
          uint32_t incl = mine;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += y;
          }
          total = __shfl_sync(kFull, incl, 31);
          return incl - mine;
        };
        segment_walk(sg, K, gs, 0u, lane, [&](auto tag, const Fired& f) {
          constexpr bool kBern = decltype(tag)::value;
          if (kDraw) {  // the symbol bits this firing sets, straight into S
            const uint64_t j = j0 + s;
#pragma unroll
            for (int k = 0; k < kSlots; ++k) {
              if (!((f.v >> k) & 1u)) continue;
              uint32_t sym = __ldg(P.cls_sym + sg.goff + f.g[k]);
              for (uint32_t pp = f.pat[k]; pp; pp >>= 1, ++sym)
                if (pp & 1u) atomicOr(&S32[sym * ld32 + (j >> 5)], 1u << (j & 31));
            }
            return;
          }
          if constexpr (kBern) {
            // one symbol per firing: the whole step (<= 128) in one list
            if (!__any_sync(kFull, f.v != 0)) return;
            uint32_t total;
            uint32_t at = warp_excl(__popc(f.v), total);
#pragma unroll
            for (int k = 0; k < kSlots; ++k)
              if ((f.v >> k) & 1u) scratch[at++] = __ldg(P.cls_sym + sg.goff + f.g[k]);
            __syncwarp();
            xor_list(total);
            __syncwarp();  // the list is reused by the next step
          } else {
            // DEPOLARIZE: one symbol per pattern bit, a slot at a time (<= 128)
#pragma unroll
            for (int k = 0; k < kSlots; ++k) {
              const bool on = (f.v >> k) & 1u;
              const uint32_t pat = on ? f.pat[k] : 0u;
              if (!__any_sync(kFull, pat != 0)) continue;
              uint32_t total;
              uint32_t at = warp_excl(__popc(pat), total);
              uint32_t sym = on ? __ldg(P.cls_sym + sg.goff + f.g[k]) : 0u;
              for (uint32_t pp = pat; pp; pp >>= 1, ++sym)
                if (pp & 1u) scratch[at++] = sym;
              __syncwarp();
              xor_list(total);
              __syncwarp();
            }
          }
        });
      }
    }
    if (kDraw) continue;
    __syncthreads();
    // Records -> measurement-major words: warp takes row word rw (32 rows),
    // transposes the tile's T/32 blocks of 32 shots, and lane b stores row
    // 32 rw + b's T/32 words together.
    const uint32_t nb = T / 32;
    uint32_t* o32 = reinterpret_cast<uint32_t*>(out);
    const uint64_t ld32o = 2 * ld;
    const uint64_t wbase = j0 >> 5;                 // first u32 word of the tile
    const uint32_t valid_words = (valid + 31) / 32;  // u32 words inside the shot range
    for (uint32_t rw = warp; rw < nw; rw += kK5Warps) {
      uint32_t wv[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (uint32_t sb = 0; sb < 4; ++sb) {
        if (sb >= nb) break;
        const uint32_t s = sb * 32 + lane;
        const uint32_t x = s < valid ? rec[s * ncw + rw] : 0u;
        wv[sb] = transpose32_k5(x, lane);
      }
      const uint32_t k = rw * 32 + lane;
      if (k < P.n_meas) {
        uint32_t* o = o32 + static_cast<uint64_t>(k) * ld32o + wbase;
        if (nb == 4 && valid_words == 4 && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
          *reinterpret_cast<uint4*>(o) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
        } else {
#pragma unroll
          for (uint32_t sb = 0; sb < 4; ++sb)
            if (sb < valid_words) o[sb] = wv[sb];
          // the shot range ends inside a u64 word: its other half is padding (0)
          if (valid < T && ((wbase + valid_words) & 1)) o[valid_words] = 0u;
        }
        if (with_counts) {
          uint32_t pc = 0;
#pragma unroll
          for (uint32_t sb = 0; sb < 4; ++sb) pc += __popc(wv[sb]);
          if (pc) atomicAdd(&cnt[k], pc);
        }
      }
    }
    __syncthreads();
  }
  if (with_counts) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < P.n_meas; i += blockDim.x)
      if (cnt[i]) atomicAdd(&counts[i], static_cast<unsigned long long>(cnt[i]));
  }
}

}  // namespace

size_t k5_smem_bytes(uint32_t ncw, uint32_t t_log2, uint32_t n_meas) {
  return (static_cast<size_t>(ncw) << t_log2) * 4 + static_cast<size_t>(n_meas) * 4 +
         static_cast<size_t>(kK5Warps) * kK5Scratch * 4;
}

int launch_k5(const K5Plan& P, const LaunchCfg& L, uint64_t seed, uint64_t shot_begin,
              uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t* counts) {
  if (n_shots == 0 || P.n_meas == 0) return 0;
  const size_t smem = k5_smem_bytes(P.ncw, P.t_log2, P.n_meas);
  if (cudaFuncSetAttribute(k5_columns<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem)) != cudaSuccess)
    return -1;
  const uint64_t n_tiles = (n_shots + (1ull << P.t_log2) - 1) >> P.t_log2;
  const int grid = static_cast<int>(std::min<uint64_t>(n_tiles, L.num_sms));
  k5_columns<false><<<grid, kK5Threads, smem, L.stream>>>(
      P, expand_keys(seed), shot_begin, n_shots, out, ld,
      reinterpret_cast<unsigned long long*>(counts), nullptr, 0);
  return check_launch() ? -1 : 1;
}

int launch_k5_draw(const K5Plan& P, const LaunchCfg& L, uint64_t seed, uint64_t shot_begin,
                   uint64_t n_shots, uint64_t* S, uint64_t ldS) {
  if (n_shots == 0 || P.n_cls == 0) return 0;
  const uint64_t n_tiles = (n_shots + (1ull << P.t_log2) - 1) >> P.t_log2;
  const int grid = static_cast<int>(std::min<uint64_t>(n_tiles, 4ull * L.num_sms));
  k5_columns<true><<<grid, kK5Threads, 0, L.stream>>>(P, expand_keys(seed), shot_begin, n_shots,
                                                       nullptr, 0, nullptr,
                                                       reinterpret_cast<uint32_t*>(S), 2 * ldS);
  return check_launch() ? -1 : 1;
}

}  // namespace symphase
