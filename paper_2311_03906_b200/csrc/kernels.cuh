// Device-side plan and kernel launchers for the sampling hot path (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace symphase {

// Random-stream domains (top byte of Philox counter word 3).
#ifndef SP_KBLOCKS
#define SP_KBLOCKS 1
#endif
// Philox blocks each lane draws per walk step (4 skip fields each).
constexpr int kWalkBlocks = SP_KBLOCKS;
constexpr uint32_t kDomChain = 1u;  // geometric-skip event chains
constexpr uint32_t kDomCoin = 2u;   // bit-sliced fair-coin words
constexpr uint32_t kDomThin = 3u;   // pattern choice of thinned groups (draw kernel)

// One class = all sparse channels sharing (distribution, p). Its trial space
// for one shot tile is the flattened (group, shot) grid, group-major, cut into
// n_seg segments of L trials (the last one shorter), one warp walk each.
struct ClassInfo {
  uint64_t L = 0;        // trials per segment (<= 2^22)
  uint64_t trials = 0;   // groups * T
  uint32_t seg_off = 0;  // first segment id of the class
  uint32_t n_seg = 0;
  uint32_t goff = 0;    // first class position (index into desc / cls_groups)
  float clg = 0.f;      // ln 2 / ln(1 - p) (<= 0): log2(u) -> geometric skip
  uint32_t dist = 0;    // 1 Bernoulli, 3 DEPOLARIZE1, 4 DEPOLARIZE2
  uint32_t pbase = 0;   // first flip list of the class (lists in plist)
  uint32_t npat = 1;    // non-identity patterns per group: 1, 3 or 15
  uint32_t lp = 0;      // longest flip list of the class (2/4/8/16; 0 = longer)
  // Bernoulli classes hold their groups sorted by flip-list length; len_bnd
  // [bnd ..] lists (first class position << 5 | length) of each length run,
  // ending with a sentinel, so a walk knows the longest list of its step.
  uint32_t bnd = 0xFFFFFFFFu;  // none: every list runs lp entries
};

// One sampling slice of a tile, resolved on the host (the fused kernel's
// slice dispenser reads it from shared memory instead of searching the class
// table): first trial (class position g0, shot s0), length, the class's
// fields, and the flip-list length run holding g0 (lp, next run bnd/nbp).
struct SegDesc {
  uint32_t g0 = 0, s0 = 0, len = 0, goff = 0;
  uint32_t pbase = 0, meta = 0;  // meta = npat | dist << 8 | lp << 16
  uint32_t bnd = 0xFFFFFFFFu, nbp = 0xFFFFFFFFu;
  float clg = 0.f;
  uint32_t pad[3] = {0, 0, 0};
};

// Everything a kernel needs about the loaded model, all device pointers.
// Built once per model by abi.cpp (build_plan).
struct DevPlan {
  uint32_t n_meas = 0, n_sym = 0, n_groups = 0;
  uint32_t t_log2 = 0, tw = 0;  // shot tile T = 1 << t_log2; tw = T/32 u32 words

  // M_sym, CSR over measurements (expression lists) and CSR over symbols.
  const uint64_t* row_ptr = nullptr;
  const uint32_t* sym_idx = nullptr;
  const uint64_t* col_ptr = nullptr;   // [n_sym+1]
  const uint32_t* col_rows = nullptr;  // [nnz]
  // dense row-major M_sym words [n_meas][ldm] (only when requested)
  const uint64_t* dense = nullptr;
  uint64_t ldm = 0;
  // the same bits group-major for the Four-Russians product: byte g of row k
  // (symbols 8g .. 8g+7) at dense_gm[g * gm_ld + k], gm_ld = n_meas padded to 16
  const uint8_t* dense_gm = nullptr;
  uint64_t gm_ld = 0;
  // CSR product work list (K2): the rows cut into segments of <= ~1024
  // symbols, so one very long row (the final measurements of a scrambled
  // circuit can hold 10^5 symbols) is spread over many warps. Segment s
  // covers sym_idx[k2_seg_ptr[s] .. k2_seg_ptr[s+1]) of row k2_seg_row[s] &
  // 0x7FFFFFFF; bit 31 marks a row cut in several segments, whose partial
  // XORs are combined with atomics into a zeroed row (k2_split_rows).
  uint32_t n_k2_seg = 0, n_k2_split = 0;
  const uint64_t* k2_seg_ptr = nullptr;
  const uint32_t* k2_seg_row = nullptr;
  const uint32_t* k2_split_rows = nullptr;

  // Group table (symbols.hpp:36-42).
  const uint32_t* g_first = nullptr;
  const uint32_t* g_arity = nullptr;
  const uint8_t* g_dist = nullptr;
  const double* g_param = nullptr;

  // Constant rows in compat mode (s0 only): bit k = measurement k XORs 1.
  const uint32_t* row_const_compat = nullptr;
  // Symbols whose assignment row is identically one in Philox mode (s0 and
  // Bernoulli(p>=1)); in compat mode only s0 (== ones_syms[0]).
  uint32_t n_ones = 0;
  const uint32_t* ones_syms = nullptr;

  // Dense (bit-sliced) symbols: fair coins and Bernoulli(1/2). Live slots
  // first. The fused kernel XORs each live slot's coin words into the D rows
  // of its column coin_rows[coin_ptr[slot] .. coin_ptr[slot+1]) (entries =
  // row * tw); slot n_dense_live stands for the constant term (all ones).
  uint32_t n_dense_live = 0, n_dense_all = 0;
  const uint32_t* dense_sym = nullptr;  // slot -> symbol id
  const uint32_t* coin_ptr = nullptr;   // [n_dense_live + 2]
  const uint16_t* coin_rows = nullptr;
  uint32_t n_coin_rows = 0;
  uint32_t coins_staged = 0;  // coin tables copied into shared memory

  // Sparse channels (see ClassInfo). Live classes first.
  uint32_t n_cls_live = 0, n_cls_all = 0;
  uint32_t n_seg_live = 0, n_seg_all = 0;
  const ClassInfo* cls = nullptr;
  const uint32_t* cls_groups = nullptr;  // class position -> group id
  // Thinned groups (abi.cpp): pseudo group j >= n_groups fires for source
  // group thin_src[j] (UINT32_MAX: a merged bucket, not a symbol of S); per
  // group g_masks = non-null pattern mask | null pattern mask << 16. The
  // null classes (after live and dead) are walked by the draw kernel's
  // second pass.
  uint32_t n_cls_null = 0, n_seg_null = 0;
  const uint32_t* thin_src = nullptr;
  // Mechanism pseudo variables (abi.cpp): pseudo j >= n_groups with
  // mech_pat[j - n_groups] != 0 is one Pauli pattern of source group
  // thin_src[j - n_groups], drawn as an independent Bernoulli mechanism.
  const uint32_t* mech_pat = nullptr;
  const uint32_t* g_masks = nullptr;
  // Fused-kernel event tables in D space (M_sym = L·D, see abi.cpp), class-
  // position order: desc = {colrow base, len0 | len1 << 16, len2 | len3 << 16,
  // group id}; colrow entries = D row * tw (u16: n_meas * tw < 65536).
  uint32_t n_desc_live = 0;
  const uint4* desc = nullptr;
  const uint16_t* colrow = nullptr;
  uint64_t n_colrow = 0;
  // Exact per-(group, pattern) flip lists in D space: lp entries padded
  // with spare-region entries (lp = 4, 8 or 16; 0 = lists too long, use the
  // desc/colrow loops). Entries are u8 row indices when n_meas < 256, u16
  // tile byte offsets (row * tw * 4) when the tile is under 64 KB, else u32.
  // List of (class position g, pattern pi) = plist[(pbase + g*npat + pi-1)].
  uint32_t lp = 0;
  uint32_t pad_pred = 0;  // skip padding entries (many firings per shot) vs XOR the spare row
  uint32_t plist_dummy = 0;  // index of an all-padding list (invalid slots load it)
  uint32_t entry_bytes = 4;  // 1: u8 row indices, 2: u16 / 4: u32 tile byte offsets
  const uint4* plist = nullptr;
  // the same lists as a linear texture (texel = a list of 4 / 8 bytes, or a
  // 16-byte piece of a longer one); 0 = none, load through plist
  cudaTextureObject_t plist_tex = 0;
  const uint32_t* len_bnd = nullptr;  // length runs of the sorted Bernoulli classes (ClassInfo::bnd)
  uint32_t n_len_bnd = 0;
  const SegDesc* seg_desc = nullptr;  // [n_seg_live]
  uint32_t seg_staged = 0;            // seg_desc and len_bnd copied to shared memory (set at launch)
  uint32_t seg_stage_ok = 1;          // SP_SEG_STAGE=0 keeps them in global memory
  // Zeros (n_meas * tw u32, device): the TMA drain clears a stored tile with a
  // bulk copy from here, completing on the tile's `empty` barrier (SP_TMA_ZERO=0: threads clear it)
  const uint32_t* zero_src = nullptr;
  // Row reconstruction out[k] = d[k] ^ out[parent[k]] along the paths of a
  // heavy-path decomposition of the parent forest: path p lists rows
  // path_rows[path_ptr[p] .. path_ptr[p+1]) top-down; path_par[p] is the head's
  // parent (or -1), which lies on a path of an earlier round (round_ptr).
  // Entry = row | keep << 31 (keep: row has light children, so its final
  // value stays in the tile until the tile ends); path_rows has one padding
  // entry at the end so the walk can always prefetch x + 1. keep_rows lists
  // the rows to clear at the end.
  const uint32_t* path_rows = nullptr;
  const uint32_t* path_ptr = nullptr;
  const int32_t* path_par = nullptr;
  const uint16_t* keep_rows = nullptr;
  const uint32_t* round_ptr = nullptr;  // [n_rounds + 1] over paths
  uint32_t n_paths = 0, n_rounds = 1, n_keep = 0;
  uint32_t flat_rows = 0;  // no parents at all: the drain is one pass in row order
  // Detector counts (sp_sample_ex): a detector equal to {k, parent(k)} (or
  // {k} for a root row) is counted from row k's D value while the drain
  // rebuilds the row (its index + 1 in bits 16..30 of k's path_rows entry);
  // the others ("general") XOR their measurements' finished rows.
  uint32_t n_det = 0, n_gdet = 0;
  const uint32_t* gdet_ptr = nullptr;   // [n_gdet + 1]
  const uint16_t* gdet_rows = nullptr;  // measurement rows
  const uint32_t* gdet_id = nullptr;    // detector index

  // Fused-kernel launch shape (chosen by the planner).
  uint32_t staged = 0;       // event tables copied into shared memory
  uint32_t row_staged = 0;   // row tables copied into shared memory
  uint32_t gen_warps = 12;   // event-generator warps; the rest drain tiles
  uint32_t cta_per_sm = 1;
  uint32_t cta_threads = 512;
  uint32_t n_buf = 2;        // shot-tile buffers in shared memory (1 or 2)
  uint32_t drain_teams = 1;  // drain warps split into teams that take alternate tiles (1 or 2)
  // K7 (k7_queued.cuh), the queued form of the fused sampler: walker warps
  // push firings into shared-memory rings, apply warps XOR their flip lists
  // (same streams and records as K1). q_sel[kind] says whether K7 serves a
  // launch kind (kind = 2 * tiled + counts detectors), with q_shape[kind]
  // walker (= apply) warps: the launch autotune times K7 against the tuned K1
  // per kind. q_apply is a multiple of q_walk; a ring holds 2^q_depth_log2 batches.
  uint32_t queued_ok = 0;  // the plan is eligible for K7
  uint32_t q_sel[4] = {0, 0, 0, 0};
  uint32_t q_shape[4] = {8, 8, 8, 8};
  uint32_t q_fixed_shape = 0;  // SP_Q_WALK / SP_Q_APPLY given: q_walk / q_apply as set
  uint32_t q_walk = 8, q_apply = 8, q_depth_log2 = 2, q_threads = 1024;  // the launch's shape (set from q_shape)
  uint32_t q_drain_teams = 2;  // K7 has warps to spare for two drain teams
  // Drain stores finished tiles with TMA bulk copies (rows rebuilt in place,
  // then one copy per tile in the tiled layout or one per row segment of
  // >= 128 bytes in the measurement-major layout) instead of per-thread
  // 16-byte stores (SP_BULK=0 turns it off).
  uint32_t bulk_store = 1;
  // Class table copied into shared memory (set at launch when it fits): the
  // segment dispenser's class search then reads shared memory, not L2.
  uint32_t cls_staged = 0;
  // Profiling switches (SP_DEBUG_MODE): bit 0 skips the firing XORs, bit 1
  // skips the segment walks, bit 2 skips the coin words, bit 3 skips the row
  // rebuild. Results are wrong when set.
  uint32_t debug_mode = 0;
  uint32_t wait_ns = 256;  // longest back-off sleep of an mbarrier wait (ns)
  // Optional per-role cycle counters (SP_PHASE_TIMERS=1): gen wait/work,
  // drain wait/work, summed over warps and tiles (u64[4], device).
  long long* timers = nullptr;

  // Compat mode: group ids (>= 1) with at least one live symbol.
  uint32_t n_live_groups = 0;
  const uint32_t* live_groups = nullptr;
};

// K5 column sampler (k5_columns.cu) for dense M_sym: shot-major records in
// shared memory, each fired symbol's dense column XORed in by a warp.
struct K5Plan {
  uint32_t n_meas = 0, n_sym = 0;
  uint32_t ncw = 0;        // u32 words per record / column (n_meas bits, padded to 4 words)
  uint32_t t_log2 = 7;     // shots per CTA tile (32..128; not part of the streams)
  uint32_t n_cls = 0, n_cls_live = 0;  // classes: live first (sampled), then dead (drawn only)
  const ClassInfo* cls = nullptr;      // per class: trials = its groups, goff, dist, clg, npat
  const uint32_t* cls_groups = nullptr;
  const uint32_t* cls_sym = nullptr;    // class position -> first symbol of its group
  const uint32_t* cols = nullptr;       // [n_sym][ncw] dense M_sym columns
  const uint32_t* row_const = nullptr;  // [ncw] rows that are one in every shot
  uint32_t n_chunks = 1;  // symbol chunks walked in turn (columns of a chunk stay L2-resident)
};

// Philox4x32-10 round keys for one seed (host-expanded, read from the
// kernel-parameter bank).
struct RoundKeys {
  uint32_t k[20];
};
RoundKeys expand_keys(uint64_t seed);

struct LaunchCfg {
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
};

// 16 warps per CTA, one CTA per SM (a 32-warp variant with 64 registers per
// thread measured slower on both cfg2 and cfg3).
#ifndef SP_FUSED_THREADS
#define SP_FUSED_THREADS 512
#endif
constexpr int kFusedThreads = SP_FUSED_THREADS;

// Words of the fused kernel's spare tile region (after the n_meas rows):
// padded flip-list entries point into it, spread over 32 banks (u32 lists:
// offset n_meas*tw + r, r < 32, plus the firing's word < tw).
__host__ __device__ constexpr uint32_t spare_words(uint32_t tw) { return ((tw + 32) + 3) & ~3u; }

constexpr uint32_t kMaxBufHost = 4;  // tile buffers of the fused kernel (device: kMaxBuf)

// Per-row flip-count slots of the fused kernel: 32 per-lane partials when a
// warp walks one path per 4096-shot tile (no per-row reduction), unless
// three or more tile buffers leave no room for them.
__host__ __device__ constexpr uint32_t count_lanes(uint32_t t_log2, uint32_t n_buf) {
  return t_log2 >= 12 && n_buf <= 2 ? 32u : 1u;
}

// Shared-memory bytes of the fused kernel for a plan shape.
size_t fused_smem_bytes(const DevPlan& P, uint32_t t_log2, bool staged, bool row_staged,
                        uint32_t n_buf = 2);

// K1 fused sampler (Philox). Returns number of launches issued, <0 on error.
int launch_fused_sample(const DevPlan& P, const LaunchCfg& L, uint64_t seed, uint64_t tile0,
                        uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t* counts,
                        bool tiled = false, uint64_t* det_counts = nullptr);
// K4 fused sampler, compat RNG (bit-exact keyed_draw / fill_group).
int launch_fused_sample_compat(const DevPlan& P, const LaunchCfg& L, uint64_t seed,
                               uint64_t tile0, uint64_t n_shots, uint64_t* out, uint64_t ld,
                               uint64_t* counts);
// draw_assignments on device (same streams as the fused kernels).
// segments = false: S rows of sparse channels are left zero (K5 draws them).
int launch_draw(const DevPlan& P, const LaunchCfg& L, bool compat, uint64_t seed, uint64_t tile0,
                uint64_t n_shots, uint64_t* S, uint64_t ldS, bool segments = true);
// K2 explicit-S product: sparse (CSR rows) or dense (row-major words).
int launch_product(const DevPlan& P, const LaunchCfg& L, bool dense, const uint64_t* S,
                   uint64_t ldS, uint64_t n_shots, uint64_t* out, uint64_t ld);
// K5 column sampler (dense M_sym).
size_t k5_smem_bytes(uint32_t ncw, uint32_t t_log2, uint32_t n_meas);
int launch_k5(const K5Plan& P, const LaunchCfg& L, uint64_t seed, uint64_t shot_begin,
              uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t* counts);
// draw_assignments for the K5 streams (S must be zeroed, ones/coins filled).
int launch_k5_draw(const K5Plan& P, const LaunchCfg& L, uint64_t seed, uint64_t shot_begin,
                   uint64_t n_shots, uint64_t* S, uint64_t ldS);
// K6 — the dense explicit-S product on the tensor cores (k6_tcgen05.cu):
// A = M_sym bytes in the core-matrix tile layout (tc_a_bytes, built once per
// model from the dense words by launch_tc_prep), then the GEMM + parity.
uint64_t tc_a_bytes(uint32_t n_meas, uint32_t n_sym);
int launch_tc_prep(const LaunchCfg& L, const uint64_t* dense, uint64_t ldm, uint32_t n_meas,
                   uint32_t n_sym, uint8_t* At);
int launch_tc_product(const LaunchCfg& L, const uint8_t* At, uint32_t n_meas, uint32_t n_sym,
                      const uint64_t* S, uint64_t ldS, uint64_t n_shots, uint64_t* out, uint64_t ld);
// K3 encode (fmt 0 = '01', 1 = 'b8').
// tile_shots == 0: measurement-major input; else tiled blocks of tile_shots.
int launch_encode(const LaunchCfg& L, const uint64_t* m, uint64_t ld, uint64_t n_meas,
                  uint64_t n_shots, int fmt, uint8_t* bytes, uint32_t tile_shots = 0);
// Tiled records -> measurement-major.
int launch_untile(const LaunchCfg& L, const uint64_t* in, uint64_t n_meas, uint32_t tile_shots,
                  uint64_t n_shots, uint64_t* out, uint64_t ld);
// counts[k] += popcount of row k of measurement-major records (n_shots bits).
int launch_row_counts(const LaunchCfg& L, const uint64_t* m, uint64_t ld, uint64_t n_meas,
                      uint64_t n_shots, uint64_t* counts);
// Known-answer hook for the Philox4x32-10 implementation.
int launch_debug_philox(const LaunchCfg& L, const uint32_t* ctr_key_dev, uint32_t* out_dev);

}  // namespace symphase
