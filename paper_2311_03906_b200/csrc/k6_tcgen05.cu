// K6 — the dense explicit-S product (bit_matrix.cpp:287-312, gf2_multiply)
// on the 5th-generation tensor cores: out = M_sym . S over GF(2) as an
// integer GEMM, tcgen05.mma kind::i8 with int32 accumulators in TMEM, and
// the parity (count & 1) of each accumulator as the record bit.
//
// Operands (u8, 0/1):
//   A = M_sym bytes, prepared once per model (k6_prep_a) in the K-major
//       no-swizzle core-matrix layout, one contiguous 16 KB block per
//       (128-row m-tile, 128-symbol k-stage): a stage is ONE bulk TMA copy
//       (cp.async.bulk, completion on the stage's mbarrier).
//   B = S bits of a 128-shot n-tile, expanded to bytes in shared memory by
//       eight expander warps in the MN-major (shots contiguous) core-matrix
//       layout: 16 shot bits -> 16 bytes, no bit transpose.
// Per CTA: four 128 x 128 output tiles (kTcMT m-tiles share every expanded
// B stage, so the expansion cost per MMA is a quarter of a one-tile CTA's),
// 2 pipeline stages (4 x 16 KB A + 16 KB B each), 4 x 128 TMEM columns.
// Warp 0 lane 0 issues the A copies, warp 1 lane 0 the MMAs (4 m-tiles x 4
// K-steps of 32 per stage), warps 4-11 expand B and then run the epilogue
// (tcgen05.ld of 32 columns per thread, parity, pack to words, store).
// tcgen05.commit arrives on the stage's `empty` barrier when the MMAs that
// read it are done.
// cfg5 shape (10^4 x 10^5, density 0.5, 2^20 shots): 892 ms vs 1020 ms for
// Four-Russians (profiles/k6_timing_r02.txt); 1 tile/CTA was 2.87 s.
//
// A prototype next to the Four-Russians kernel (k2_m4rm): selected with
// sp_set_product(SP_PRODUCT_TENSOR); results are bit-identical (integer
// counts are exact: <= n_sym < 2^31).
#include "kernels.cuh"

#include <algorithm>

#include "device_common.cuh"

namespace symphase {
namespace {

constexpr uint32_t kTcM = 128, kTcN = 128, kTcBK = 128, kTcStages = 2;
constexpr uint32_t kTcMT = 4;                 // m-tiles per CTA: four accumulators share each B stage
constexpr uint32_t kTcNG = kTcN / 16;         // 16-shot groups of an n-tile (B core matrices along N)
constexpr uint32_t kTcLboB = kTcNG * 128;     // B: bytes between k-groups
constexpr uint32_t kTcAStage = kTcM * kTcBK;  // bytes of one m-tile's A per stage
constexpr uint32_t kTcBStage = kTcN * kTcBK;
constexpr uint32_t kTcThreads = 384;   // warps 0-3: TMA / MMA / TMEM / spare; 4-11: B expanders + epilogue
constexpr uint32_t kTcExp = 256;        // expander threads
constexpr uint32_t kTcPk = kTcBK * kTcN / 8;  // packed S bytes per stage
constexpr uint32_t kTcPkChunks = kTcPk / 16;   // 16-byte cp.async chunks of a stage
constexpr uint32_t kTcPkSlots = 4, kTcPkAhead = 3;
constexpr uint32_t kBarExp = 2;         // named barrier of the expander warps
constexpr size_t kTcSmem = kTcStages * (kTcMT * kTcAStage + kTcBStage) + kTcPkSlots * kTcPk +
                           8 * (3 * kTcStages + 1) + 16 + 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 16 bits -> 16 bytes of 0/1, as a uint4 (bit i -> byte i).
__device__ __forceinline__ uint4 spread16(uint32_t bits) {
  auto nib = [](uint32_t n) { return (n * 0x00204081u) & 0x01010101u; };
  return make_uint4(nib(bits & 0xFu), nib((bits >> 4) & 0xFu), nib((bits >> 8) & 0xFu),
                    nib((bits >> 12) & 0xFu));
}

// tcgen05 shared-memory matrix descriptor, no swizzle (version 1 = sm_100).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

// Instruction descriptor: D s32, A u8 K-major, B u8 MN-major, M = kTcM, N = kTcN.
constexpr uint32_t kTcIdesc = (2u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (1u << 16) |
                              ((kTcN >> 3) << 17) | ((kTcM >> 4) << 24);

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_spin(uint32_t bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}

// A: M_sym bits (dense row-major words, [n_meas][ldm]) -> u8 core-matrix
// tiles At[mt][ks][chunk c (8)][row group g (16)][row r (8)][16 bytes], i.e.
// byte (row mt*128 + g*8 + r, symbol ks*128 + c*16 + j).
__global__ void k6_prep_a(const uint64_t* __restrict__ dense, uint64_t ldm, uint32_t n_meas,
                          uint32_t n_sym, uint32_t k_stages, uint64_t units, uint4* __restrict__ At) {
  for (uint64_t u = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; u < units;
       u += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r = u & 7u, g = (u >> 3) & 15u, c = (u >> 7) & 7u;
    const uint64_t blk = u >> 10;  // (mt, ks)
    const uint32_t ks = static_cast<uint32_t>(blk % k_stages);
    const uint32_t mt = static_cast<uint32_t>(blk / k_stages);
    const uint32_t row = mt * kTcM + g * 8 + r;
    const uint32_t k0 = ks * kTcBK + c * 16;
    uint32_t bits = 0;
    if (row < n_meas && k0 < n_sym) {
      bits = static_cast<uint32_t>(dense[static_cast<uint64_t>(row) * ldm + (k0 >> 6)] >> (k0 & 63)) & 0xFFFFu;
      if (n_sym - k0 < 16) bits &= (1u << (n_sym - k0)) - 1u;
    }
    At[u] = spread16(bits);
  }
}

__global__ void __launch_bounds__(kTcThreads, 1)
k6_tc_product(const uint8_t* __restrict__ At, uint32_t k_stages, const uint64_t* __restrict__ S,
              uint64_t ldS, uint32_t n_sym, uint64_t n_shots, uint32_t n_meas,
              uint64_t* __restrict__ out, uint64_t ld) {
  extern __shared__ __align__(1024) uint8_t smem_k6[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_k6) + 1023) & ~uintptr_t{1023});
  uint8_t* sA = base;
  uint8_t* sB = base + kTcStages * kTcMT * kTcAStage;
  uint8_t* sP = sB + kTcStages * kTcBStage;  // packed S ring (cp.async)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + kTcPkSlots * kTcPk);
  uint64_t* full_a = bars;
  uint64_t* full_b = bars + kTcStages;
  uint64_t* empty = bars + 2 * kTcStages;
  uint64_t* done = bars + 3 * kTcStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * kTcStages + 1);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t nt = blockIdx.x, mt = blockIdx.y * kTcMT;  // first of the CTA's m-tiles

  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kTcStages; ++s) {
      mbar_init(full_a + s, 1);
      mbar_init(full_b + s, kTcExp);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {  // TMEM: 128 lanes x kTcN int32 columns per accumulator tile
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kTcN * kTcMT)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---- A producer: one bulk copy per stage ----
    if (lane == 0) {
      const uint8_t* src = At + static_cast<uint64_t>(mt) * k_stages * kTcAStage;
      for (uint32_t ks = 0; ks < k_stages; ++ks) {
        const uint32_t s = ks % kTcStages;
        if (ks >= kTcStages) mbar_wait_spin(smem_u32(empty + s), ((ks / kTcStages) - 1) & 1);
        mbar_expect_tx(smem_u32(full_a + s), kTcMT * kTcAStage);
        for (uint32_t a = 0; a < kTcMT; ++a)  // the next m-tile's blocks follow k_stages blocks later
          bulk_load(smem_u32(sA + (s * kTcMT + a) * kTcAStage),
                    src + (static_cast<uint64_t>(a) * k_stages + ks) * kTcAStage, kTcAStage,
                    smem_u32(full_a + s));
      }
    }
  } else if (warp == 1) {
    // ---- MMA issuer ----
    if (lane == 0) {
      for (uint32_t ks = 0; ks < k_stages; ++ks) {
        const uint32_t s = ks % kTcStages, ph = (ks / kTcStages) & 1;
        mbar_wait_spin(smem_u32(full_a + s), ph);
        mbar_wait_spin(smem_u32(full_b + s), ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a0 = smem_u32(sA + s * kTcMT * kTcAStage), b0 = smem_u32(sB + s * kTcBStage);
#pragma unroll
        for (uint32_t kk = 0; kk < kTcBK / 32; ++kk) {
          // K = 32 per MMA: A chunks 2kk, 2kk+1 (LBO 2048 between chunks, SBO
          // 128 between row groups); B k-groups 4kk..4kk+3 (LBO kTcLboB
          // between k-groups, SBO 128 between 16-shot groups)
          const uint64_t db = umma_desc(b0 + kk * 4 * kTcLboB, kTcLboB, 128);
          const uint32_t acc = (ks | kk) != 0;
#pragma unroll
          for (uint32_t a = 0; a < kTcMT; ++a) {  // accumulator a: columns a * kTcN ..
            const uint64_t da = umma_desc(a0 + a * kTcAStage + kk * 2 * 2048, 2048, 128);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + a * kTcN),
                "l"(da), "l"(db), "r"(kTcIdesc), "r"(acc)
                : "memory");
          }
        }
        // the stage's smem may be refilled once these MMAs have read it
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(empty + s))
                     : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(done))
                   : "memory");
    }
  } else if (warp >= 4) {
    // ---- B expanders: S bits -> MN-major u8 core matrices ----
    // The packed S slice of stage ks (128 symbols x kTcN shots, one 16-byte
    // chunk per thread) is fetched kTcPkAhead stages ahead with cp.async
    // into a ring; then unit (k-group kg, shot group ng, k-row kr) = 16
    // bytes at ((kg * kTcNG + ng) * 8 + kr) * 16 is spread from 16 bits.
    const uint32_t et = threadIdx.x - 128;
    const uint64_t n0 = static_cast<uint64_t>(nt) * kTcN;
    const uint32_t n_words = static_cast<uint32_t>((n_shots + 63) >> 6);
    constexpr uint32_t kCpr = kTcN / 128;  // 16-byte chunks per symbol row of a stage
    auto fetch = [&](uint32_t ks) {  // chunk et: symbol row et / kCpr, 128 shots (et % kCpr)
      if (ks < k_stages && et < kTcPkChunks) {
        const uint32_t k = ks * kTcBK + et / kCpr;
        const uint32_t w = static_cast<uint32_t>(n0 >> 6) + (et % kCpr) * 2;  // first of 2 words
        const uint32_t dst = smem_u32(sP + (ks % kTcPkSlots) * kTcPk + et * 16);
        // two 8-byte copies (rows of S are only 8-byte aligned); rows past
        // n_sym and words past the record are zero-filled
        const uint64_t* row = S + static_cast<uint64_t>(k < n_sym ? k : 0) * ldS;
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
          const bool ok = k < n_sym && w + h < n_words;
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + 8 * h),
                       "l"(row + (ok ? w + h : 0)), "r"(ok ? 8u : 0u)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (uint32_t a = 0; a < kTcPkAhead; ++a) fetch(a);
    for (uint32_t ks = 0; ks < k_stages; ++ks) {
      const uint32_t s = ks % kTcStages;
      fetch(ks + kTcPkAhead);
      asm volatile("cp.async.wait_group %0;" ::"n"(kTcPkAhead) : "memory");
      named_sync(kBarExp, kTcExp);  // every chunk of stage ks has landed
      if (ks >= kTcStages) mbar_wait_spin(smem_u32(empty + s), ((ks / kTcStages) - 1) & 1);
      uint4* dst = reinterpret_cast<uint4*>(sB + s * kTcBStage);
      const uint16_t* pk = reinterpret_cast<const uint16_t*>(sP + (ks % kTcPkSlots) * kTcPk);
#pragma unroll 4
      for (uint32_t i = 0; i < (kTcBK * kTcN / 16) / kTcExp; ++i) {
        const uint32_t u = et + kTcExp * i;  // unit index in [0, kTcBK * kTcN / 16)
        const uint32_t ng = u % kTcNG, kr = (u / kTcNG) & 7u, kg = u / (kTcNG * 8);
        uint32_t bits = pk[(kg * 8 + kr) * kTcNG + ng];
        const uint64_t shot = n0 + ng * 16;
        if (shot >= n_shots) bits = 0;
        else if (n_shots - shot < 16) bits &= (1u << (n_shots - shot)) - 1u;
        dst[(kg * kTcNG + ng) * 8 + kr] = spread16(bits);  // (a 256-entry smem LUT was slower)
      }
      fence_proxy_async_smem();  // the tensor core reads the stage through the async proxy
      mbar_arrive(full_b + s);
    }
    // ---- epilogue: accumulator parity -> record words ----
    mbar_wait_spin(smem_u32(done), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t q = warp & 3;               // TMEM lane quarter of this warp
    uint32_t* out32 = reinterpret_cast<uint32_t*>(out);
    for (uint32_t acc = (warp - 4) >> 2; acc < kTcMT; acc += 2)  // two warps per lane quarter
    for (uint32_t c = 0; c < kTcN / 32; ++c) {
      const uint32_t row = (mt + acc) * kTcM + q * 32 + lane;
      uint32_t v[32];
      const uint32_t taddr = tmem + ((q * 32) << 16) + acc * kTcN + c * 32;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
          "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
          "%30, %31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
            "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]),
            "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]),
            "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      uint32_t w = 0;
#pragma unroll
      for (int j = 0; j < 32; ++j) w |= (v[j] & 1u) << j;
      const uint64_t shot = n0 + c * 32;
      // whole u64 words within ceil(n_shots / 64) (bits past n_shots are 0)
      if (row < n_meas && ((shot >> 6) << 6) < n_shots)
        out32[static_cast<uint64_t>(row) * ld * 2 + (shot >> 5)] = w;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTcN * kTcMT)
                 : "memory");
}

}  // namespace

uint64_t tc_a_bytes(uint32_t n_meas, uint32_t n_sym) {
  // m-tiles rounded up to the CTA's kTcMT (the extra ones are zero rows)
  const uint64_t mt = (n_meas + kTcM * kTcMT - 1) / (kTcM * kTcMT) * kTcMT;
  const uint64_t ks = (std::max<uint32_t>(n_sym, 1) + kTcBK - 1) / kTcBK;
  return mt * ks * kTcAStage;
}

int launch_tc_prep(const LaunchCfg& L, const uint64_t* dense, uint64_t ldm, uint32_t n_meas,
                   uint32_t n_sym, uint8_t* At) {
  const uint32_t ks = (std::max<uint32_t>(n_sym, 1) + kTcBK - 1) / kTcBK;
  const uint64_t units = tc_a_bytes(n_meas, n_sym) / 16;
  if (units == 0) return 0;
  k6_prep_a<<<L.num_sms * 8, 256, 0, L.stream>>>(dense, ldm, n_meas, n_sym, ks, units,
                                                 reinterpret_cast<uint4*>(At));
  return check_launch() ? -1 : 1;
}

int launch_tc_product(const LaunchCfg& L, const uint8_t* At, uint32_t n_meas, uint32_t n_sym,
                      const uint64_t* S, uint64_t ldS, uint64_t n_shots, uint64_t* out, uint64_t ld) {
  if (n_meas == 0 || n_shots == 0) return 0;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(k6_tc_product, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kTcSmem)) != cudaSuccess)
      return -1;
    attr = true;
  }
  const uint32_t ks = (std::max<uint32_t>(n_sym, 1) + kTcBK - 1) / kTcBK;
  const uint64_t n_tiles = (n_shots + kTcN - 1) / kTcN;
  const uint64_t m_ctas = (n_meas + kTcM * kTcMT - 1) / (kTcM * kTcMT);
  if (n_tiles > 0x7FFFFFFFull || m_ctas > 65535) return -1;
  dim3 grid(static_cast<unsigned>(n_tiles), static_cast<unsigned>(m_ctas));
  k6_tc_product<<<grid, kTcThreads, kTcSmem, L.stream>>>(At, ks, S, ldS, n_sym, n_shots, n_meas, out, ld);
  return check_launch() ? -1 : 1;
}

}  // namespace symphase
