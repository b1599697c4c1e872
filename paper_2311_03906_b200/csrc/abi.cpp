// C-ABI implementation (include/symphase_b200.h): context, plan building,
// device buffers, launches. Host C++ over the CUDA runtime; no torch types.
#include "../../include/symphase_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <map>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "frontend.hpp"
#include "plan_stages.hpp"

extern char** environ;
#include "kernels.cuh"

using namespace symphase;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Owned device buffer.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { reset(); }
  void reset() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* upload(const std::vector<T>& v, cudaStream_t s) {
    // reuse the allocation when it is large enough (stream-ordered copy; no
    // cudaFree, which would synchronise the device)
    const size_t need = std::max<size_t>(v.size() * sizeof(T), 16);
    if (!p || bytes < need) {
      reset();
      bytes = need;
      ck(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    if (!v.empty()) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s),
                       "cudaMemcpyAsync H2D");
    return static_cast<T*>(p);
  }
  void* ensure(size_t b) {
    if (bytes >= b && p) return p;
    reset();
    ck(cudaMalloc(&p, b), "cudaMalloc");
    bytes = b;
    return p;
  }
};

// Host-side sampling plan derived from M_sym + the group table.
struct HostPlan {
  uint64_t n_meas = 0, n_sym = 0, n_groups = 0, nnz = 0;
  std::vector<uint64_t> row_ptr;
  std::vector<uint32_t> sym_idx;
  uint64_t max_sym_plus1 = 0;
  std::vector<sp_group> groups;
  std::vector<uint64_t> dense_words;  // only if dense product requested / loaded
  uint64_t ldm = 0;
  // detectors registered by sp_set_detectors (CSR over measurement indices)
  std::vector<uint64_t> det_ptr{0};
  std::vector<uint32_t> det_meas;
};

}  // namespace

struct sp_model {
  Model m;
};

struct sp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  sp_rng rng = SP_RNG_PHILOX;
  sp_product product = SP_PRODUCT_AUTO;
  LaunchCfg L;
  bool have_msym = false, have_groups = false, plan_ready = false, fused_ok = false;
  bool plan_built = false;  // dp/hp-derived buffers describe the model with plan_fp
  bool unfused = false;     // sp_sample draws S and runs the explicit-S product (faster here)
  bool k5_ok = false;       // sp_sample / sp_draw_assignments use the K5 column sampler
  K5Plan k5;
  DBuf b_k5_cls, b_k5_groups, b_k5_sym, b_k5_cols, b_k5_rc;
  uint64_t plan_fp = 0;
  std::string fused_why;
  HostPlan hp;
  DevPlan dp;
  // plan buffers
  DBuf b_row_ptr, b_sym_idx, b_col_ptr, b_col_rows, b_dense, b_dense_gm, b_first, b_arity, b_dist, b_param,
      b_row_const_compat, b_ones, b_dense_sym, b_coin_ptr, b_coin_rows, b_cls, b_cls_groups, b_thin_src, b_mech_pat, b_len_bnd, b_seg_desc, b_zero, b_g_masks,
      b_desc, b_colrow, b_live_groups, b_path_rows, b_path_ptr, b_path_par, b_round_ptr, b_plist, b_keep_rows, b_timers,
      b_gdet_ptr, b_gdet_rows, b_gdet_id;
  uint64_t dnnz = 0;  // nnz of D (chain transform), for reports
  // K2's own copy of the rows (independent of the group table)
  bool prod_ready = false;
  DevPlan pp;
  DBuf p_row_ptr, p_sym_idx, p_dense, p_dense_gm, p_seg_ptr, p_seg_row, p_split_rows;
  DBuf p_tc_a;          // K6: M_sym bytes in the tensor-core tile layout
  bool tc_ready = false;
  // sp_sample_to_host: double-buffered records/bytes, a copy stream and the
  // events that hand each buffer between the compute and copy streams
  DBuf s_out[2], s_bytes[2];
  DBuf s_S;  // sp_sample without an on-chip tile: the drawn assignments of one chunk
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  uint64_t launches = 0;
  // texture view of the flip lists (the fused samplers fetch them through the
  // texture pipe, which leaves the LSU data pipe to the tile's shared atomics)
  cudaTextureObject_t plist_tex = 0;
  ~sp_ctx() {
    if (plist_tex) cudaDestroyTextureObject(plist_tex);
    for (int b = 0; b < 2; ++b) {
      if (ev_ready[b]) cudaEventDestroy(ev_ready[b]);
      if (ev_free[b]) cudaEventDestroy(ev_free[b]);
    }
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }
};

namespace {

int set_device(sp_ctx* c) {
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(SP_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return SP_OK;
}

long env_long(const char* name, long dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::strtol(v, nullptr, 10) : dflt;
}

// Content fingerprint of the loaded model and of the SP_* planner switches.
uint64_t model_fingerprint(const HostPlan& h) {
  uint64_t fp = 0xcbf29ce484222325ull;
  auto mix = [&](const void* data, size_t n) {  // FNV-1a over 64-bit words
    const uint8_t* b = static_cast<const uint8_t*>(data);
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
      uint64_t w;
      std::memcpy(&w, b + i, 8);
      fp = (fp ^ w) * 0x100000001b3ull;
    }
    for (; i < n; ++i) fp = (fp ^ b[i]) * 0x100000001b3ull;
  };
  const uint64_t dims[4] = {h.n_meas, h.n_sym, h.groups.size(), h.ldm};
  mix(dims, sizeof dims);
  mix(h.row_ptr.data(), h.row_ptr.size() * 8);
  mix(h.sym_idx.data(), h.sym_idx.size() * 4);
  mix(h.dense_words.data(), h.dense_words.size() * 8);
  mix(h.groups.data(), h.groups.size() * sizeof(sp_group));
  mix(h.det_ptr.data(), h.det_ptr.size() * 8);
  mix(h.det_meas.data(), h.det_meas.size() * 4);
  for (char** e = environ; e && *e; ++e)
    if (std::strncmp(*e, "SP_", 3) == 0) mix(*e, std::strlen(*e));
  return fp;
}

// SP_PLAN_TIMING=1: per-phase host times of build_plan on stderr.
struct PlanTimer {
  bool on = std::getenv("SP_PLAN_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[plan] %-22s %8.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// K2 variant: the Four-Russians dense product costs the same at any density
// (n_meas x words x n_sym / 8 table lookups); the CSR walk costs nnz x words.
// Measured on B200 at cfg5's shape the two cross at density ~0.15.
constexpr double kDenseProductDensity = 0.15;
bool dense_product(const sp_ctx* c) {
  if (c->product == SP_PRODUCT_DENSE || c->product == SP_PRODUCT_TENSOR) return true;
  if (c->product != SP_PRODUCT_AUTO) return false;
  const double cells = static_cast<double>(c->hp.n_meas) * static_cast<double>(c->hp.n_sym);
  return cells > 0 && static_cast<double>(c->hp.nnz) > kDenseProductDensity * cells;
}
// K6 (tcgen05 int8 GEMM) vs K2 (Four-Russians) for a dense product: K6 wins
// at every measured shape with >= 4096 symbols and loses at 1000 symbols
// (profiles/k6_shapes_r02.txt); its u8 operand copy of M_sym is capped.
constexpr uint64_t kTensorMinSym = 4096;
constexpr uint64_t kTensorMaxABytes = 16ull << 30;
bool tensor_product(const sp_ctx* c) {
  if (c->product == SP_PRODUCT_TENSOR) return true;
  return c->product == SP_PRODUCT_AUTO && dense_product(c) && c->hp.n_sym >= kTensorMinSym &&
         tc_a_bytes(static_cast<uint32_t>(c->hp.n_meas), static_cast<uint32_t>(c->hp.n_sym)) <=
             kTensorMaxABytes;
}
// Dense row-major M_sym words from the CSR rows (first use only).
void ensure_dense_words(HostPlan& h) {
  if (!h.dense_words.empty()) return;
  h.ldm = std::max<uint64_t>((h.n_sym + 63) / 64, 1);
  h.dense_words.assign(h.n_meas * h.ldm, 0);
  for (uint64_t k = 0; k < h.n_meas; ++k)
    for (uint64_t i = h.row_ptr[k]; i < h.row_ptr[k + 1]; ++i)
      h.dense_words[k * h.ldm + h.sym_idx[i] / 64] |= uint64_t{1} << (h.sym_idx[i] % 64);
}

// The explicit-S product of plan d (whose dense words are M_sym's): K6 when
// tensor_product() picks it (the u8 operand layout is built on first use and
// kept until the model changes), else K2. Returns launch_* codes.
int run_product(sp_ctx* c, const DevPlan& d, const uint64_t* S, uint64_t ldS, uint64_t n_shots,
                uint64_t* out, uint64_t ld) {
  if (!tensor_product(c) || !d.dense) return launch_product(d, c->L, dense_product(c), S, ldS, n_shots, out, ld);
  int prep = 0;
  if (!c->tc_ready) {
    auto* at = static_cast<uint8_t*>(c->p_tc_a.ensure(tc_a_bytes(d.n_meas, d.n_sym)));
    prep = launch_tc_prep(c->L, d.dense, d.ldm, d.n_meas, d.n_sym, at);
    if (prep < 0) return prep;
    c->tc_ready = true;
  }
  const int r = launch_tc_product(c->L, static_cast<const uint8_t*>(c->p_tc_a.p), d.n_meas, d.n_sym, S,
                                  ldS, n_shots, out, ld);
  return r < 0 ? r : r + prep;
}

// K5 column sampler plan (k5_columns.cu): for models the fused kernel does
// not serve (too many flips per shot) whose firings x record words per shot
// are far below the explicit product's work. Classes are built from the raw
// group table (live first, then dead ones, which only the draw walks).
void build_k5(sp_ctx* c, const std::vector<uint64_t>& col_ptr, const std::vector<uint32_t>& col_rows,
              const std::vector<uint32_t>& ones, double events_per_shot, double flips_per_shot,
              uint64_t n_dense_live) {
  c->k5_ok = false;
  const HostPlan& h = c->hp;
  const long mode = env_long("SP_K5", -1);  // -1 auto, 0 never, 1 whenever eligible
  if (mode == 0 || n_dense_live > 0 || h.n_meas == 0) return;
  const uint64_t n_meas = h.n_meas, n_sym = h.n_sym, G = h.groups.size();
  const uint32_t ncw = static_cast<uint32_t>(((n_meas + 31) / 32 + 3) & ~uint64_t{3});
  int lg = -1;
  for (int t = 7; t >= 5 && lg < 0; --t)
    if (k5_smem_bytes(ncw, t, static_cast<uint32_t>(n_meas)) <= c->L.smem_optin) lg = t;
  if (lg < 0) return;
  // work per shot: firings x record words (K5) vs the explicit product's
  // word operations per shot (CSR walk or Four-Russians lookups)
  // (u32 words per shot: K5 XORs ncw words per firing; the CSR walk XORs nnz
  // u64 words and the Four-Russians product n_meas * n_sym / 8 per 64 shots)
  const double k5_work = events_per_shot * ncw;
  const double k2_work = std::min(static_cast<double>(h.nnz),
                                  static_cast<double>(n_meas) * ((n_sym + 7) / 8)) / 32.0;
  if (mode < 0 && !(k5_work < 0.25 * k2_work)) return;
  // vs the fused kernel, which pays per flipped bit: with exact flip lists
  // (<= 16 entries) a flip costs about 0.35 K5 words (cfg3); on the
  // table-walk path (long lists) about 6 (cfg5: K5 wins at 100 rows per
  // column, K1 at 10, for 316-word records)
  if (mode < 0 && c->fused_ok && !(k5_work < (c->dp.lp ? 0.35 : 6.0) * flips_per_shot)) return;
  if (static_cast<double>(n_sym) * ncw * 4 > 8e9) return;  // columns must fit comfortably
  struct KC { uint8_t dist; double p; std::vector<uint32_t> groups; };
  std::vector<KC> live, dead;
  std::map<std::pair<uint8_t, uint64_t>, size_t> lk, dk;
  for (uint64_t g = 1; g < G; ++g) {
    const sp_group& gr = h.groups[g];
    const double p = gr.param;
    const bool sparse = (gr.dist == SP_DIST_BERNOULLI && p > 0.0 && p < 1.0 && p != 0.5) ||
                        ((gr.dist == SP_DIST_DEPOLARIZE1 || gr.dist == SP_DIST_DEPOLARIZE2) && p > 0.0);
    if (!sparse) continue;
    bool is_live = false;
    for (uint32_t b = 0; b < gr.arity; ++b)
      is_live |= col_ptr[gr.first_symbol + b + 1] > col_ptr[gr.first_symbol + b];
    uint64_t pbits;
    std::memcpy(&pbits, &p, 8);
    auto& km = is_live ? lk : dk;
    auto& v = is_live ? live : dead;
    auto key = std::make_pair(gr.dist, pbits);
    auto it = km.find(key);
    // a walk covers <= 2^22 trials (the skip clamp): split larger classes
    if (it == km.end() || v[it->second].groups.size() >= (1u << 22)) {
      it = km.insert_or_assign(key, v.size()).first;
      v.push_back(KC{gr.dist, std::min(p, 1.0), {}});
    }
    v[it->second].groups.push_back(static_cast<uint32_t>(g));
  }
  std::vector<ClassInfo> cls;
  std::vector<uint32_t> cg;
  for (auto* v : {&live, &dead})
    for (const KC& k : *v) {
      ClassInfo ci{};
      ci.dist = k.dist;
      ci.clg = static_cast<float>(0.69314718055994531 / std::log1p(-k.p));
      ci.goff = static_cast<uint32_t>(cg.size());
      ci.trials = k.groups.size();
      ci.npat = k.dist == SP_DIST_DEPOLARIZE2 ? 15 : k.dist == SP_DIST_DEPOLARIZE1 ? 3 : 1;
      cls.push_back(ci);
      cg.insert(cg.end(), k.groups.begin(), k.groups.end());
    }
  // dense columns (plus an all-zero column n_sym that pads K5's column
  // groups), and the rows that are one in every shot (s0, p >= 1)
  std::vector<uint32_t> cols(static_cast<size_t>(n_sym + 1) * ncw, 0), rc(ncw, 0);
  for (uint64_t sidx = 0; sidx < n_sym; ++sidx)
    for (uint64_t i = col_ptr[sidx]; i < col_ptr[sidx + 1]; ++i)
      cols[sidx * ncw + col_rows[i] / 32] ^= 1u << (col_rows[i] % 32);
  for (uint32_t sidx : ones)
    for (uint32_t w = 0; w < ncw; ++w) rc[w] ^= cols[static_cast<size_t>(sidx) * ncw + w];
  K5Plan& P = c->k5;
  cudaStream_t s = c->stream;
  P = K5Plan{};
  P.n_meas = static_cast<uint32_t>(n_meas);
  P.n_sym = static_cast<uint32_t>(n_sym);
  P.ncw = ncw;
  P.t_log2 = static_cast<uint32_t>(lg);
  P.n_cls = static_cast<uint32_t>(cls.size());
  P.n_cls_live = static_cast<uint32_t>(live.size());
  if (cls.empty()) cls.push_back(ClassInfo{});
  if (cg.empty()) cg.push_back(0);
  P.cls = c->b_k5_cls.upload(cls, s);
  P.cls_groups = c->b_k5_groups.upload(cg, s);
  std::vector<uint32_t> csym(cg.size());
  for (size_t i = 0; i < cg.size(); ++i) csym[i] = h.groups[cg[i]].first_symbol;
  P.cls_sym = c->b_k5_sym.upload(csym, s);
  P.cols = c->b_k5_cols.upload(cols, s);
  P.row_const = c->b_k5_rc.upload(rc, s);
  {  // ~32 MB of columns per chunk (a quarter of the L2) when the columns
     // outgrow the L2 and a shot fires tens to hundreds of times (measured at
     // cfg5 density 0.5: p = 1e-3 27 -> 18 ms with 4 chunks; p = 1e-4 and
     // 1e-2 are faster unchunked: too few firings per chunk walk, resp. not
     // bound by column misses)
    const double col_bytes = static_cast<double>(n_sym) * ncw * 4;
    long dflt = std::max<long>(1, static_cast<long>(std::ceil(col_bytes / (32.0 * (1 << 20)))));
    if (events_per_shot < 30.0 || events_per_shot > 300.0) dflt = 1;
    P.n_chunks = static_cast<uint32_t>(std::min<long>(std::max<long>(env_long("SP_K5_CHUNKS", dflt), 1), 32767));
  }
  ck(cudaStreamSynchronize(s), "K5 plan upload");
  c->k5_ok = true;
}

// Group-major bytes of the dense words (k2_m4rm): byte g of row k at
// [g * ld + k], ld = n_meas rounded up to 16.
std::vector<uint8_t> group_major_bytes(const HostPlan& h, uint64_t* ld) {
  const uint64_t n_g = (h.n_sym + 7) / 8;
  *ld = (h.n_meas + 15) & ~uint64_t{15};
  std::vector<uint8_t> gm(std::max<uint64_t>(n_g * *ld, 1), 0);
  for (uint64_t k = 0; k < h.n_meas; ++k)
    for (uint64_t g = 0; g < n_g; ++g)
      gm[g * *ld + k] = static_cast<uint8_t>(h.dense_words[k * h.ldm + g / 8] >> (8 * (g % 8)));
  return gm;
}

void build_plan(sp_ctx* c) {
  PlanTimer ptm;
  c->unfused = env_long("SP_UNFUSED", -1) > 0;
  HostPlan& h = c->hp;
  DevPlan& d = c->dp;
  cudaStream_t s = c->stream;
  const uint64_t n_meas = h.n_meas, n_sym = h.n_sym, G = h.groups.size();
  if (dense_product(c)) ensure_dense_words(h);  // the unfused path's product

  // Symbol -> group map; the registry tiles [0, n_sym) with its groups.
  std::vector<uint32_t> sym_group(n_sym, UINT32_MAX);
  for (uint64_t g = 0; g < G; ++g) {
    const sp_group& gr = h.groups[g];
    for (uint32_t b = 0; b < gr.arity; ++b) {
      uint64_t sidx = uint64_t{gr.first_symbol} + b;
      if (sidx >= n_sym || sym_group[sidx] != UINT32_MAX)
        throw std::invalid_argument("group table does not tile the symbol range");
      sym_group[sidx] = static_cast<uint32_t>(g);
    }
  }
  for (uint64_t sidx = 0; sidx < n_sym; ++sidx)
    if (sym_group[sidx] == UINT32_MAX) throw std::invalid_argument("symbol without a group");

  // CSR over symbols (CSR-of-variables).
  std::vector<uint64_t> col_ptr(n_sym + 1, 0);
  for (uint32_t sidx : h.sym_idx) col_ptr[sidx + 1]++;
  for (uint64_t i = 0; i < n_sym; ++i) col_ptr[i + 1] += col_ptr[i];
  std::vector<uint32_t> col_rows(h.nnz);
  {
    std::vector<uint64_t> fillp(col_ptr.begin(), col_ptr.end() - 1);
    for (uint64_t k = 0; k < n_meas; ++k)
      for (uint64_t i = h.row_ptr[k]; i < h.row_ptr[k + 1]; ++i)
        col_rows[fillp[h.sym_idx[i]]++] = static_cast<uint32_t>(k);
  }
  auto col_len = [&](uint64_t sidx) { return col_ptr[sidx + 1] - col_ptr[sidx]; };
  ptm.mark("groups+csc");

  // D = L^-1 M (chain transform); skipped when M is dense enough that the
  // parent search (sum of squared column lengths) would be expensive.
  double sq = 0;
  for (uint64_t sidx = 0; sidx < n_sym; ++sidx) sq += static_cast<double>(col_len(sidx)) * col_len(sidx);
  plan::ChainXf X = plan::chain_transform(n_meas, h.row_ptr, h.sym_idx, col_ptr, col_rows,
                              sq < 2e9 && env_long("SP_NO_CHAIN", 0) == 0);
  // A transform that saves < 5 % of the nonzeros is not worth the drain's
  // parent walks: without any parent the drain is a flat pass.
  if (static_cast<double>(X.si.size()) > 0.95 * static_cast<double>(h.nnz))
    X = plan::chain_transform(n_meas, h.row_ptr, h.sym_idx, col_ptr, col_rows, false);
  c->dnnz = X.si.size();
  ptm.mark("chain transform");
  std::vector<uint64_t> dcol_ptr(n_sym + 1, 0);
  for (uint32_t sidx : X.si) dcol_ptr[sidx + 1]++;
  for (uint64_t i = 0; i < n_sym; ++i) dcol_ptr[i + 1] += dcol_ptr[i];
  std::vector<uint32_t> dcol_rows(X.si.size());
  {
    std::vector<uint64_t> fillp(dcol_ptr.begin(), dcol_ptr.end() - 1);
    for (uint64_t k = 0; k < n_meas; ++k)
      for (uint64_t i = X.rp[k]; i < X.rp[k + 1]; ++i) dcol_rows[fillp[X.si[i]]++] = static_cast<uint32_t>(k);
  }
  auto dcol_len = [&](uint64_t sidx) { return dcol_ptr[sidx + 1] - dcol_ptr[sidx]; };

  const size_t cw = (n_meas + 31) / 32 + 1;
  std::vector<uint32_t> row_const(cw, 0), row_const_compat(cw, 0);  // D rows / M rows
  auto xor_rows = [&](std::vector<uint32_t>& mask, uint64_t sidx) {
    for (uint64_t i = dcol_ptr[sidx]; i < dcol_ptr[sidx + 1]; ++i)
      mask[dcol_rows[i] >> 5] ^= 1u << (dcol_rows[i] & 31);
  };
  std::vector<uint32_t> ones{0};
  xor_rows(row_const, 0);
  for (uint64_t i = col_ptr[0]; i < col_ptr[1]; ++i)
    row_const_compat[col_rows[i] >> 5] ^= 1u << (col_rows[i] & 31);

  // Classify groups: dense (coins, Bernoulli(1/2)), constant-folded
  // (Bernoulli(p>=1)), never (p == 0), or a sparse class keyed by (dist, p).
  std::vector<uint32_t> dense_live, dense_dead;
  struct Cls {
    uint8_t dist;
    double p;
    uint32_t lpc;  // flip-list length class (live): every pattern's D list has <= lpc rows
    std::vector<uint32_t> groups;
    bool runs = false;  // one-list groups sorted by list length (length runs, ClassInfo::bnd)
  };
  std::vector<Cls> live_cls, dead_cls, null_cls;
  std::map<std::tuple<uint8_t, uint64_t, uint32_t>, size_t> live_key, dead_key, null_key;
  // Longest flip list over a group's patterns (symmetric differences of the
  // D columns of the pattern's symbols), rounded up to 2, 4, 8, 16 (0: longer).
  std::vector<uint32_t> mrg_a, mrg_b;
  const bool split_lists = env_long("SP_LIST_CLASSES", 1) != 0;
  const bool len_runs = env_long("SP_LEN_RUNS", 1) != 0;
  auto list_class = [&](const sp_group& gr) -> uint32_t {
    const uint32_t npat = (1u << gr.arity) - 1;
    size_t mx = 0;
    for (uint32_t pat = 1; pat <= npat; ++pat) {
      mrg_a.clear();
      for (uint32_t b = 0; b < gr.arity; ++b) {
        if (!((pat >> b) & 1u)) continue;
        const uint64_t sidx = gr.first_symbol + b;
        mrg_b.clear();
        std::set_symmetric_difference(mrg_a.begin(), mrg_a.end(), dcol_rows.begin() + dcol_ptr[sidx],
                                      dcol_rows.begin() + dcol_ptr[sidx + 1], std::back_inserter(mrg_b));
        mrg_a.swap(mrg_b);
      }
      mx = std::max(mx, mrg_a.size());
    }
    return mx <= 2 ? 2u : mx <= 4 ? 4u : mx <= 8 ? 8u : mx <= 16 ? 16u : 0u;
  };
  // Channel merging (exact). A sparse group whose non-empty flip lists are
  // all one list L acts as Bernoulli(p_eff) on L (p_eff = p * #patterns with
  // list L / #patterns). Independent such groups on the same L merge into one
  // Bernoulli with the piling-up rate q = (1 - prod(1 - 2 p_eff)) / 2 — the
  // same distribution of records with far fewer firings when many channels
  // hit the same rows (cfg4: 72,723 groups, 73 firings per shot, on one row).
  // The merged variable is a pseudo symbol (id >= n_sym) with D column L; the
  // merged-away groups are still drawn by sp_draw_assignments (as dead
  // classes), so S stays complete, but K1 records of a merged model are not
  // M_sym . S of that S. Buckets of >= SP_MERGE_MIN (64) groups are merged.
  //
  // Thinning (exact, keeps K1 == M_sym . S of its own draw). A single-list
  // group that is not merged becomes its own pseudo variable: Bernoulli(p_eff)
  // on L, so the patterns that flip nothing cost no firings. The draw kernel
  // maps a firing of that pseudo group back to one of the group's non-null
  // patterns (uniform, keyed hash) and draws the null patterns in a second
  // pass: Bernoulli(p_null / (1 - p_eff)) over the trials where the group did
  // not fire (a null event on a trial that fired is dropped), so every
  // pattern keeps probability p / #patterns and S stays exact.
  const long merge_min = env_long("SP_MERGE_MIN", 64);
  const bool thin = env_long("SP_THIN", 1) != 0;
  std::vector<uint8_t> merged(G, 0), thinned(G, 0);
  std::vector<sp_group> pseudo;        // group id G + j
  std::vector<uint32_t> thin_src;      // pseudo j -> thinned source group (UINT32_MAX: a merged bucket)
  std::vector<uint32_t> g_masks(G, 0);  // thinned group: non-null pattern mask | null mask << 16
  std::vector<double> null_p(G, 0.0);   // thinned group: rate of its null events given no firing
  {
    std::map<std::vector<uint32_t>, std::pair<std::vector<uint32_t>, double>> buckets;
    std::map<uint32_t, std::pair<double, uint32_t>> singles;  // g -> (p_eff, non-null mask)
    std::vector<uint32_t> la, lb, one;
    for (uint64_t g = 1; g < G && (merge_min > 0 || thin); ++g) {
      const sp_group& gr = h.groups[g];
      const double p = gr.param;
      const bool sparse = (gr.dist == SP_DIST_BERNOULLI && p > 0.0 && p < 1.0 && p != 0.5) ||
                          ((gr.dist == SP_DIST_DEPOLARIZE1 || gr.dist == SP_DIST_DEPOLARIZE2) && p > 0.0);
      if (!sparse) continue;
      bool live = false;
      for (uint32_t b = 0; b < gr.arity; ++b) live |= col_len(gr.first_symbol + b) > 0;
      if (!live) continue;
      const uint32_t npat = (1u << gr.arity) - 1;
      uint32_t k = 0, nonnull = 0;
      bool single = true;
      one.clear();
      for (uint32_t pat = 1; pat <= npat && single; ++pat) {
        la.clear();
        for (uint32_t b = 0; b < gr.arity; ++b) {
          if (!((pat >> b) & 1u)) continue;
          const uint64_t sidx = gr.first_symbol + b;
          lb.clear();
          std::set_symmetric_difference(la.begin(), la.end(), dcol_rows.begin() + dcol_ptr[sidx],
                                        dcol_rows.begin() + dcol_ptr[sidx + 1], std::back_inserter(lb));
          la.swap(lb);
        }
        if (la.empty()) continue;
        if (k == 0) one = la;
        else if (la != one) single = false;
        nonnull |= 1u << (pat - 1);
        ++k;
      }
      if (!single || k == 0) continue;
      const double p_eff = std::min(p, 1.0) * k / npat;
      auto& bk = buckets[one];
      if (bk.first.empty()) bk.second = 1.0;
      bk.first.push_back(static_cast<uint32_t>(g));
      bk.second *= 1.0 - 2.0 * p_eff;
      // (p_eff = 1/2 would make the pseudo variable a fair coin: not thinned)
      if (k < npat && p_eff < 0.5) singles.emplace(static_cast<uint32_t>(g), std::make_pair(p_eff, nonnull));
    }
    for (auto& [rows, bk] : buckets) {
      if (merge_min <= 0 || static_cast<long>(bk.first.size()) < merge_min) {
        if (!thin) continue;
        for (uint32_t g : bk.first) {  // thin each of the bucket's groups on its own
          auto it = singles.find(g);
          if (it == singles.end()) continue;
          const sp_group& gr = h.groups[g];
          const uint32_t npat = (1u << gr.arity) - 1;
          const double p_eff = it->second.first;
          const uint32_t nonnull = it->second.second;
          const uint64_t sym = dcol_ptr.size() - 1;
          for (uint32_t r : rows) dcol_rows.push_back(r);
          dcol_ptr.push_back(dcol_rows.size());
          sp_group pg{};
          pg.dist = SP_DIST_BERNOULLI;
          pg.param = p_eff;
          pg.first_symbol = static_cast<uint32_t>(sym);
          pg.arity = 1;
          pseudo.push_back(pg);
          thin_src.push_back(g);
          const uint32_t nullm = ((1u << npat) - 1) & ~nonnull;
          g_masks[g] = nonnull | (nullm << 16);
          null_p[g] = (gr.param * __builtin_popcount(nullm) / npat) / (1.0 - p_eff);
          thinned[g] = 1;
          merged[g] = 1;
        }
        continue;
      }
      const uint64_t sym = dcol_ptr.size() - 1;  // next pseudo symbol id
      for (uint32_t r : rows) dcol_rows.push_back(r);
      dcol_ptr.push_back(dcol_rows.size());
      sp_group pg{};
      pg.dist = SP_DIST_BERNOULLI;
      pg.param = 0.5 * (1.0 - bk.second);
      pg.first_symbol = static_cast<uint32_t>(sym);
      pg.arity = 1;
      pseudo.push_back(pg);
      thin_src.push_back(UINT32_MAX);
      for (uint32_t g : bk.first) merged[g] = 1;
    }
  }
  // Mechanism decomposition (exact). DEPOLARIZE1(p) is the composition of
  // three independent Pauli channels X, Y, Z each firing with q1 =
  // (1 - sqrt(1 - 4p/3)) / 2, and DEPOLARIZE2(p) of fifteen independent ones
  // (one per non-identity two-qubit Pauli) with q2 = (1 - (1 - 16p/15)^(1/8))
  // / 2: the XOR of the fired patterns' symplectic vectors is uniform over the
  // non-zero vectors with total rate p (Fourier over GF(2)^n: each non-trivial
  // character sees the factor (1 - 2q) from exactly half of the patterns). So
  // every remaining multi-list DEPOLARIZE group becomes one Bernoulli(q)
  // pseudo variable per pattern, whose D column is that pattern's flip list:
  // no pattern digits (four skips per Philox block), and classes of one exact
  // list length (no padded XORs). Patterns that flip nothing become dead
  // pseudo variables, walked only by the draw kernel, which XORs each firing's
  // pattern into the source group's symbols (mech_pat) — so S is exactly
  // DEPOLARIZE-distributed and K1 == M_sym . S(draw) still holds bit for bit.
  // Valid while q < 1/2 (p < 3/4, resp. 15/16); SP_MECH=0 turns it off.
  std::vector<uint32_t> mech_pat;      // pseudo j -> pattern of its source group (0: not a mechanism)
  std::vector<uint8_t> mech(G, 0);
  if (env_long("SP_MECH", 1) != 0) {
    std::vector<uint32_t> la, lb;
    for (uint64_t g = 1; g < G; ++g) {
      const sp_group& gr = h.groups[g];
      const double p = gr.param;
      if (merged[g] || !(p > 0.0)) continue;
      const double q = plan::mechanism_rate(gr.dist, p);
      if (!(q > 0.0 && q < 0.5)) continue;
      bool live = false;
      for (uint32_t b = 0; b < gr.arity; ++b) live |= col_len(gr.first_symbol + b) > 0;
      if (!live) continue;  // a dead group keeps its plain dead class
      const uint32_t npat = (1u << gr.arity) - 1;
      for (uint32_t pat = 1; pat <= npat; ++pat) {
        la.clear();
        for (uint32_t b = 0; b < gr.arity; ++b) {
          if (!((pat >> b) & 1u)) continue;
          const uint64_t sidx = gr.first_symbol + b;
          lb.clear();
          std::set_symmetric_difference(la.begin(), la.end(), dcol_rows.begin() + dcol_ptr[sidx],
                                        dcol_rows.begin() + dcol_ptr[sidx + 1], std::back_inserter(lb));
          la.swap(lb);
        }
        const uint64_t sym = dcol_ptr.size() - 1;
        dcol_rows.insert(dcol_rows.end(), la.begin(), la.end());
        dcol_ptr.push_back(dcol_rows.size());
        sp_group pg{};
        pg.dist = SP_DIST_BERNOULLI;
        pg.param = q;
        pg.first_symbol = static_cast<uint32_t>(sym);
        pg.arity = 1;
        pseudo.push_back(pg);
        thin_src.push_back(static_cast<uint32_t>(g));
        mech_pat.resize(pseudo.size(), 0);
        mech_pat.back() = pat;
      }
      mech[g] = 1;
    }
  }
  mech_pat.resize(pseudo.size(), 0);
  const bool merged_any =
      std::any_of(thin_src.begin(), thin_src.end(), [](uint32_t v) { return v == UINT32_MAX; });
  auto grp = [&](uint64_t g) -> const sp_group& { return g < G ? h.groups[g] : pseudo[g - G]; };

  std::vector<uint32_t> live_groups;
  double events_per_shot = 0, flips_per_shot = 0;
  for (uint64_t g = 1; g < G + pseudo.size(); ++g) {
    const sp_group& gr = grp(g);
    const bool is_pseudo = g >= G;
    bool live = false;
    uint64_t flips = 0;
    for (uint32_t b = 0; b < gr.arity; ++b) {
      // (a pseudo variable is live when its flip list is not empty)
      live |= is_pseudo ? dcol_len(gr.first_symbol + b) > 0 : col_len(gr.first_symbol + b) > 0;
      flips += dcol_len(gr.first_symbol + b);
    }
    if (live && !is_pseudo) live_groups.push_back(static_cast<uint32_t>(g));  // compat (M space)
    if (!is_pseudo && mech[g]) continue;  // sampled and drawn through its mechanisms
    if (!is_pseudo && thinned[g]) {
      // fires through its pseudo variable; the draw kernel's second pass
      // draws its null patterns (Bernoulli null_p over the trials it did not fire)
      uint64_t pbits;
      std::memcpy(&pbits, &null_p[g], 8);
      auto key = std::make_tuple(static_cast<uint8_t>(SP_DIST_BERNOULLI), pbits, 0u);
      auto it = null_key.find(key);
      if (it == null_key.end()) {
        it = null_key.emplace(key, null_cls.size()).first;
        null_cls.push_back(Cls{SP_DIST_BERNOULLI, std::min(null_p[g], 1.0), 0u, {}});
      }
      null_cls[it->second].groups.push_back(static_cast<uint32_t>(g));
      continue;
    }
    if (!is_pseudo && merged[g]) live = false;  // sampled through its merged variable
    const double p = gr.param;
    switch (gr.dist) {
      case SP_DIST_CONSTANT:
        throw std::invalid_argument("constant group other than group 0");
      case SP_DIST_COIN:
        (live ? dense_live : dense_dead).push_back(gr.first_symbol);
        continue;
      case SP_DIST_BERNOULLI:
        if (p == 0.5) {
          (live ? dense_live : dense_dead).push_back(gr.first_symbol);
          continue;
        }
        if (p >= 1.0) {
          ones.push_back(gr.first_symbol);
          xor_rows(row_const, gr.first_symbol);
          continue;
        }
        break;
      case SP_DIST_DEPOLARIZE1:
      case SP_DIST_DEPOLARIZE2:
        break;
      default:
        throw std::invalid_argument("unknown group distribution");
    }
    if (!(p > 0.0)) continue;  // never fires (p == 0, or NaN)
    if (live) {
      events_per_shot += std::min(p, 1.0);
      flips_per_shot += std::min(p, 1.0) * flips / gr.arity * (gr.arity == 1 ? 1.0 : gr.arity == 2 ? 4.0 / 3 : 32.0 / 15);
    }
    uint64_t pbits;
    std::memcpy(&pbits, &p, 8);
    // Live classes are split by flip-list length, so a slice's warp only
    // runs as many list entries as its class needs.
    // One-list (Bernoulli) groups of one p form one class whatever their
    // list lengths: they are sorted by length below and the kernel bounds
    // each step by the longest list of its run (SP_LEN_RUNS=0: split).
    const bool runs = live && len_runs && gr.arity == 1;
    const uint32_t lpc = runs ? 99u : live && split_lists ? list_class(gr) : 0u;
    auto key = std::make_tuple(gr.dist, pbits, lpc);
    auto& keymap = live ? live_key : dead_key;
    auto& cls = live ? live_cls : dead_cls;
    auto it = keymap.find(key);
    if (it == keymap.end()) {
      it = keymap.emplace(key, cls.size()).first;
      cls.push_back(Cls{gr.dist, std::min(p, 1.0), lpc, {}});
    }
    cls[it->second].groups.push_back(static_cast<uint32_t>(g));
  }
  {
    // Merge length classes holding < 5 % of their (dist, p) family's trials
    // into the next longer class (or the longest one into its neighbour),
    // so no class is too small to fill its slices. lpc 0 (lists > 16) is
    // the longest.
    auto rank = [](uint32_t l) { return l == 0 ? 98u : l; };  // 99: a length-run family
    std::stable_sort(live_cls.begin(), live_cls.end(), [&](const Cls& a, const Cls& b) {
      if (a.dist != b.dist) return a.dist < b.dist;
      if (a.p != b.p) return a.p < b.p;
      return rank(a.lpc) < rank(b.lpc);
    });
    std::vector<Cls> merged;
    for (size_t i = 0; i < live_cls.size();) {
      size_t j = i;
      uint64_t fam = 0;
      while (j < live_cls.size() && live_cls[j].dist == live_cls[i].dist && live_cls[j].p == live_cls[i].p)
        fam += live_cls[j++].groups.size();
      std::vector<Cls> f(std::make_move_iterator(live_cls.begin() + i),
                         std::make_move_iterator(live_cls.begin() + j));
      for (size_t k = 0; k + 1 < f.size();) {  // small ones flow upward
        if (f[k].groups.size() * 20 < fam) {
          f[k + 1].groups.insert(f[k + 1].groups.end(), f[k].groups.begin(), f[k].groups.end());
          f.erase(f.begin() + k);
        } else {
          ++k;
        }
      }
      if (f.size() > 1 && f.back().groups.size() * 20 < fam) {  // a small longest class
        Cls& prev = f[f.size() - 2];
        prev.groups.insert(prev.groups.end(), f.back().groups.begin(), f.back().groups.end());
        prev.lpc = f.back().lpc;
        f.pop_back();
      }
      for (Cls& c : f) {
        std::sort(c.groups.begin(), c.groups.end());
        if (c.lpc == 99u) {  // length runs: groups by (list length, id)
          std::stable_sort(c.groups.begin(), c.groups.end(), [&](uint32_t a, uint32_t b) {
            return dcol_len(grp(a).first_symbol) < dcol_len(grp(b).first_symbol);
          });
          const uint64_t mx = dcol_len(grp(c.groups.back()).first_symbol);
          c.lpc = mx <= 16 ? static_cast<uint32_t>(std::max<uint64_t>(mx, 1)) : 0u;
          c.runs = mx <= 16;
        }
        merged.push_back(std::move(c));
      }
      i = j;
    }
    live_cls.swap(merged);
  }

  // Dense slots (live first). The fused kernel XORs each live slot's coin
  // words into its D column; the extra slot n_dense_live is the constant
  // term (all-ones words into the rows of row_const).
  const uint64_t n_dense_live = dense_live.size();
  std::vector<uint32_t> dense_sym = dense_live;
  dense_sym.insert(dense_sym.end(), dense_dead.begin(), dense_dead.end());
  std::vector<uint32_t> coin_ptr{0};
  std::vector<uint32_t> coin_rows_k;  // D rows; scaled by tw once T is known
  for (uint32_t sym : dense_live) {
    for (uint64_t i = dcol_ptr[sym]; i < dcol_ptr[sym + 1]; ++i) coin_rows_k.push_back(dcol_rows[i]);
    coin_ptr.push_back(static_cast<uint32_t>(coin_rows_k.size()));
  }
  for (uint64_t k = 0; k < n_meas; ++k)
    if ((row_const[k >> 5] >> (k & 31)) & 1u) coin_rows_k.push_back(static_cast<uint32_t>(k));
  coin_ptr.push_back(static_cast<uint32_t>(coin_rows_k.size()));
  uint64_t live_positions = 0, live_colrow = 0;
  for (const Cls& cl : live_cls)
    for (uint32_t g : cl.groups) {
      ++live_positions;
      for (uint32_t b = 0; b < grp(g).arity; ++b) live_colrow += dcol_len(grp(g).first_symbol + b);
    }

  ptm.mark("classify");
  // ---- launch shape: tile T, table staging, generator/drain warp split ----
  d = DevPlan{};
  d.n_meas = static_cast<uint32_t>(n_meas);
  d.n_sym = static_cast<uint32_t>(n_sym);
  d.n_groups = static_cast<uint32_t>(G);
  d.n_dense_live = static_cast<uint32_t>(n_dense_live);
  d.n_dense_all = static_cast<uint32_t>(dense_sym.size());
  d.n_cls_live = static_cast<uint32_t>(live_cls.size());
  d.n_desc_live = static_cast<uint32_t>(live_positions);
  d.n_colrow = live_colrow;
  d.n_paths = static_cast<uint32_t>(n_meas);  // upper bounds for the smem estimate
  d.n_keep = static_cast<uint32_t>(n_meas);
  const size_t optin = c->L.smem_optin;
  int lg = -1;
  bool staged = false, row_staged = false;
  const long force_lg = env_long("SP_TLOG2", 0), force_st = env_long("SP_STAGED", -1),
             force_rs = env_long("SP_ROWSTAGED", -1);
  // The shot tile T is part of the random-stream structure (streams are
  // keyed by global tile), so it depends only on the model and the device's
  // shared memory: the largest T whose tiles fit double-buffered with no
  // tables staged — else single-buffered (very many rows). Staging then
  // takes what is left: row tables, then (T >= 512) the event tables of the
  // table-walk variant.
  uint32_t n_buf = 2;
  const long force_nb = std::min<long>(env_long("SP_NBUF", 0), 4);
  for (uint32_t nb = force_nb > 0 ? force_nb : 2; nb >= 1 && lg < 0; --nb) {
    if (force_nb > 0 && nb != static_cast<uint32_t>(force_nb)) break;
    for (int t = 12; t >= 7 && lg < 0; --t) {
      if (force_lg && t != force_lg) continue;
      if (static_cast<uint64_t>(n_meas + 1) * (1u << (t - 5)) >= 65536) continue;  // u16 row offsets
      if (fused_smem_bytes(d, t, false, false, nb) <= optin) {
        lg = t;
        n_buf = nb;
      }
    }
  }
  if (lg >= 0) {
    row_staged = force_rs >= 0 ? force_rs != 0 : fused_smem_bytes(d, lg, false, true, n_buf) <= optin;
    staged = force_st >= 0 ? force_st != 0
                           : lg >= 9 && fused_smem_bytes(d, lg, true, row_staged, n_buf) <= optin;
    if (fused_smem_bytes(d, lg, staged, row_staged, n_buf) > optin) lg = -1;  // forced staging does not fit
  }
  c->fused_ok = lg >= 0;
  if (lg < 0) {
    c->fused_why = "M_sym has too many measurement rows for an on-chip shot tile; use "
                   "sp_draw_assignments + sp_sample_given_S";
    lg = 7;
  }
  // Very many bit flips per shot (dense M_sym with frequent faults): one
  // shared atomic per flip cannot compete with drawing S and running the
  // explicit-S product (measured: cfg5 density 0.01, p = 1e-2 is 1e5 flips
  // per shot, fused 401 ms vs 87 ms), so the fused plan is not built at all.
  if (c->fused_ok && flips_per_shot > static_cast<double>(env_long("SP_FUSED_MAX_FLIPS", 50000))) {
    c->fused_ok = false;
    c->fused_why = "too many flips per shot for the fused sampler; sp_sample draws S and runs the "
                   "explicit-S product";
  }
  const uint64_t T = 1ull << lg;
  d.t_log2 = static_cast<uint32_t>(lg);
  d.tw = static_cast<uint32_t>(T / 32);
  d.staged = staged;
  d.row_staged = row_staged;
  d.n_buf = n_buf;
  {
    const size_t smem = fused_smem_bytes(d, d.t_log2, staged, row_staged, n_buf);
    d.cta_per_sm = static_cast<uint32_t>(std::max<long>(
        1, std::min<long>(env_long("SP_CTAS", 2), static_cast<long>((228 * 1024) / (smem + 1024)))));
    const double ev = events_per_shot * T, flips = flips_per_shot * T;
    // Generator warps also make the coin words and XOR them into their D
    // columns; drain warps only rebuild and store rows (~20 instructions per
    // 128-shot row word).
    const double gen = ev * 60.0 + flips * 4.0 + n_dense_live * (T / 128.0) * 60.0 +
                       coin_rows_k.size() * (T / 32.0) * 3.0;
    const double items = static_cast<double>(n_meas) * (T / 128);
    const double drain = items * 20.0;
    d.cta_threads = static_cast<uint32_t>(env_long("SP_CTA_THREADS", kFusedThreads));
    const long n_warps = d.cta_threads / 32;
    // measured on B200: the drain's latency chains want ~15% more warps than
    // its instruction share (cfg2 and cfg3 both peak at 10 of 16)
    long gw = std::lround(n_warps * 0.85 * gen / std::max(gen + drain, 1.0));
    gw = std::min<long>(gw, n_warps - std::max<long>(1, n_warps / 4));
    gw = env_long("SP_GEN_WARPS", gw);
    d.gen_warps = static_cast<uint32_t>(std::min<long>(std::max<long>(gw, 1), n_warps - 1));
  }

  // Segments: each class's flattened (group, shot) space of a tile is cut
  // into slices (<= 2^22 trials, >= 32), one warp walk each. A walk over a
  // slice holding N firings takes floor(N / S) + 1 steps of S slots (S =
  // 32 lanes x 4 skips per Philox block), so the slice count per class
  // minimises expected steps + a fixed per-slice cost (init, first Philox
  // latency), subject to enough slices per tile to keep every generator warp
  // busy with two tiles in flight. SP_SEG_EVENTS=E forces ~E firings/slice.
  const double ev_tile = events_per_shot * T;
  auto exp_steps = [](double lam, double S) {  // E[floor(N/S)] + 1, N ~ Poisson(lam)
    double e = 1.0;
    const double sd = std::sqrt(std::max(lam, 1e-9));
    for (int j = 1;; ++j) {
      const double tail = 0.5 * std::erfc((j * S - 0.5 - lam) / (sd * std::sqrt(2.0)));
      e += tail;
      if (j * S > lam && tail < 1e-7) break;
    }
    return e;
  };
  const double seg_cost = env_long("SP_SEG_COST_PCT", 35) / 100.0;
  const long seg_fe = env_long("SP_SEG_EVENTS", 0);
  std::vector<double> seg_lam(live_cls.size()), seg_S(live_cls.size());
  std::vector<uint64_t> seg_nmin(live_cls.size()), seg_nmax(live_cls.size());
  // Slice counts of the live classes (in live_cls order). The slices are the
  // random streams (keyed by slice id and global tile), so they depend only
  // on the model and the tile size — never on the launch shape — and a seed
  // gives the same records on any GPU count and any tuned warp split.
  auto plan_segments = [&](uint32_t min_slices) {
    std::vector<uint64_t> nseg(live_cls.size(), 1);
    auto cost = [&](size_t c, uint64_t n) {
      return n * (exp_steps(seg_lam[c] / n, seg_S[c]) + seg_cost);
    };
    uint64_t total = 0;
    for (size_t c = 0; c < live_cls.size(); ++c) {
      const uint64_t trials = live_cls[c].groups.size() * T;
      seg_lam[c] = trials * live_cls[c].p;
      seg_S[c] = 32.0 * 4 * kWalkBlocks;
      seg_nmin[c] = std::max<uint64_t>(1, (trials + 4194303) / 4194304);
      seg_nmax[c] = std::max<uint64_t>(seg_nmin[c], trials / 32);
      uint64_t best = seg_nmin[c];
      if (seg_fe > 0) {
        best = static_cast<uint64_t>(std::ceil(seg_lam[c] / seg_fe));
      } else {
        double bc = cost(c, best);
        const uint64_t hi =
            std::min<uint64_t>(seg_nmax[c], static_cast<uint64_t>(2 * seg_lam[c] / seg_S[c]) + 2);
        for (uint64_t n = seg_nmin[c] + 1; n <= hi; ++n) {
          const double cn = cost(c, n);
          if (cn < bc) { bc = cn; best = n; }
        }
      }
      nseg[c] = std::min(std::max(best, seg_nmin[c]), seg_nmax[c]);
      total += nseg[c];
    }
    const uint64_t min_total = seg_fe > 0 ? 0 : min_slices;
    while (total < min_total) {  // split where it costs the fewest extra steps
      size_t arg = live_cls.size();
      double dmin = 0;
      for (size_t c = 0; c < live_cls.size(); ++c) {
        if (nseg[c] >= seg_nmax[c]) continue;
        const double dc = cost(c, nseg[c] + 1) - cost(c, nseg[c]);
        if (arg == live_cls.size() || dc < dmin) { dmin = dc; arg = c; }
      }
      if (arg == live_cls.size()) break;
      ++nseg[arg];
      ++total;
    }
    return nseg;
  };
  // at least 16 slices per tile: every generator warp takes one or two per
  // tile (measured best for cfg2 and cfg3 among 8..32)
  std::vector<uint64_t> live_nseg = plan_segments(static_cast<uint32_t>(env_long("SP_SEG_MIN", 16)));
  {
    // Longest slices first: warps take slices in id order, so a warp that
    // finishes early picks up a short one. (The order is fixed here; the
    // launch autotune below only changes slice counts.)
    std::vector<size_t> ord(live_cls.size());
    std::vector<double> steps(live_cls.size());
    for (size_t c = 0; c < ord.size(); ++c) {
      ord[c] = c;
      steps[c] = exp_steps(seg_lam[c] / live_nseg[c], seg_S[c]);
    }
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return steps[a] > steps[b]; });
    std::vector<Cls> cls2;
    std::vector<uint64_t> nseg2;
    for (size_t c : ord) {
      cls2.push_back(std::move(live_cls[c]));
      nseg2.push_back(live_nseg[c]);
    }
    live_cls.swap(cls2);
    live_nseg.swap(nseg2);
  }
  // Dead classes are only walked by the standalone draw kernel.
  const double E = std::min(std::max(ev_tile / d.gen_warps, 32.0), 2048.0);
  std::vector<ClassInfo> cls_info;
  std::vector<uint32_t> cls_groups;
  std::vector<uint32_t> len_bnd;
  std::vector<uint4> desc;
  std::vector<uint16_t> colrow16;
  // Exact flip lists per (group, pattern): XOR of the D columns of the
  // pattern's set symbols, as row * tw offsets.
  // flat: list i = pl_rows[pl_off[i] .. pl_off[i+1])
  std::vector<uint32_t> pl_off{0};
  std::vector<uint16_t> pl_rows;
  std::vector<uint16_t> scratch;
  size_t max_plist = 0;
  const bool fused_tables = c->fused_ok;
  auto add_classes = [&](const std::vector<Cls>& cls, bool live) {
    for (size_t c = 0; c < cls.size(); ++c) {
      const Cls& cl = cls[c];
      ClassInfo ci{};
      ci.dist = cl.dist;
      // p == 1 -> -0: every trial fires
      ci.clg = static_cast<float>(0.69314718055994531 / std::log1p(-cl.p));
      ci.goff = static_cast<uint32_t>(cls_groups.size());
      ci.trials = cl.groups.size() * T;
      ci.npat = cl.dist == SP_DIST_DEPOLARIZE2 ? 15 : cl.dist == SP_DIST_DEPOLARIZE1 ? 3 : 1;
      ci.lp = cl.lpc;  // the kernel runs min(lp, plan lp) list entries for this class
      ci.pbase = static_cast<uint32_t>(pl_off.size() - 1);
      if (live && cl.runs) {  // (first position << 5 | length) per run, then a sentinel
        ci.bnd = static_cast<uint32_t>(len_bnd.size());
        uint64_t prev = UINT64_MAX;
        for (size_t i = 0; i < cl.groups.size(); ++i) {
          const uint64_t len = std::max<uint64_t>(dcol_len(grp(cl.groups[i]).first_symbol), 1);
          if (len != prev) len_bnd.push_back(static_cast<uint32_t>(i << 5) | static_cast<uint32_t>(len));
          prev = len;
        }
        len_bnd.push_back(0xFFFFFFFFu);
      }
      cls_info.push_back(ci);
      for (uint32_t g : cl.groups) {
        cls_groups.push_back(g);
        if (!live || !fused_tables) continue;  // event tables serve the fused kernel only
        const sp_group& gr = grp(g);
        for (uint32_t pat = 1; pat <= ci.npat; ++pat) {
          // symmetric difference of the D columns of the pattern's symbols,
          // merged in place at the end of pl_rows (sorted, as row * tw)
          const size_t start = pl_rows.size();
          for (uint32_t b = 0; b < gr.arity; ++b) {
            if (!((pat >> b) & 1u)) continue;
            const uint64_t sidx = gr.first_symbol + b;
            scratch.assign(pl_rows.begin() + start, pl_rows.end());
            pl_rows.resize(start);
            size_t i = 0;
            uint64_t j = dcol_ptr[sidx];
            while (i < scratch.size() || j < dcol_ptr[sidx + 1]) {
              const uint32_t a = i < scratch.size() ? scratch[i] : UINT32_MAX;
              const uint32_t c2 = j < dcol_ptr[sidx + 1] ? dcol_rows[j] * d.tw : UINT32_MAX;
              if (a < c2) { pl_rows.push_back(static_cast<uint16_t>(a)); ++i; }
              else if (c2 < a) { pl_rows.push_back(static_cast<uint16_t>(c2)); ++j; }
              else { ++i; ++j; }
            }
          }
          max_plist = std::max<size_t>(max_plist, pl_rows.size() - start);
          pl_off.push_back(static_cast<uint32_t>(pl_rows.size()));
        }
        uint32_t lens[4] = {0, 0, 0, 0};
        const uint32_t base = static_cast<uint32_t>(colrow16.size());
        for (uint32_t b = 0; b < gr.arity; ++b) {
          const uint64_t sidx = gr.first_symbol + b;
          lens[b] = static_cast<uint32_t>(dcol_len(sidx));
          if (lens[b] > 0xFFFF) throw std::invalid_argument("M_sym column longer than 65535");
          for (uint64_t i = dcol_ptr[sidx]; i < dcol_ptr[sidx + 1]; ++i)
            colrow16.push_back(static_cast<uint16_t>(dcol_rows[i] * d.tw));
        }
        desc.push_back(make_uint4(base, lens[0] | (lens[1] << 16), lens[2] | (lens[3] << 16), g));
      }
    }
  };
  ptm.mark("segment plan");
  add_classes(live_cls, true);
  add_classes(dead_cls, false);
  const size_t n_cls_ld = cls_info.size();  // live + dead; null classes follow
  add_classes(null_cls, false);
  ptm.mark("flip lists");
  // Segment table: live classes get the planned slice counts, dead ones
  // (walked only by the standalone draw kernel) ~E firings per slice.
  auto apply_segments = [&](const std::vector<uint64_t>& nseg_live) {
    uint64_t n_chains = 0;
    for (size_t c = 0; c < cls_info.size(); ++c) {
      ClassInfo& ci = cls_info[c];
      uint64_t n_seg = 0;
      if (c < live_cls.size()) {
        n_seg = nseg_live[c];
      } else {
        const double pc = c < n_cls_ld ? dead_cls[c - live_cls.size()].p : null_cls[c - n_cls_ld].p;
        double len = std::ceil(E / pc);
        len = std::min(std::max(len, 32.0), 4194304.0);  // kernel skips clamp at 2^22
        n_seg = std::max<uint64_t>((ci.trials + static_cast<uint64_t>(len) - 1) /
                                       static_cast<uint64_t>(len), 1);
      }
      ci.L = (ci.trials + n_seg - 1) / n_seg;
      ci.n_seg = static_cast<uint32_t>(n_seg);
      ci.seg_off = static_cast<uint32_t>(n_chains);
      n_chains += n_seg;
      if (c + 1 == live_cls.size()) d.n_seg_live = static_cast<uint32_t>(n_chains);
      if (c + 1 == n_cls_ld) d.n_seg_all = static_cast<uint32_t>(n_chains);
    }
    if (live_cls.empty()) d.n_seg_live = 0;
    if (n_cls_ld == 0) d.n_seg_all = 0;
    if (n_chains >= (1ull << 32)) throw std::invalid_argument("too many sampling chains");
    d.n_seg_null = static_cast<uint32_t>(n_chains) - d.n_seg_all;
    d.cls = c->b_cls.upload(cls_info, s);
    // the live slices resolved on the host (the kernel's dispenser reads
    // them instead of searching the classes and length runs)
    std::vector<SegDesc> sd;
    const uint64_t T_ = uint64_t{1} << d.t_log2;
    for (size_t cc = 0; cc < live_cls.size(); ++cc) {
      const ClassInfo& ci = cls_info[cc];
      for (uint32_t i = 0; i < ci.n_seg; ++i) {
        SegDesc e{};
        const uint64_t first = static_cast<uint64_t>(i) * ci.L;
        e.g0 = static_cast<uint32_t>(first / T_);
        e.s0 = static_cast<uint32_t>(first % T_);
        e.len = static_cast<uint32_t>(std::min(first + ci.L, ci.trials) - first);
        e.goff = ci.goff;
        e.pbase = ci.pbase;
        e.clg = ci.clg;
        uint32_t lp = ci.lp;
        if (ci.bnd != 0xFFFFFFFFu) {  // the length run holding g0, and where the next starts
          uint32_t b = ci.bnd;
          lp = len_bnd[b] & 31u;
          while ((len_bnd[b + 1] >> 5) <= e.g0) lp = len_bnd[++b] & 31u;
          e.bnd = b + 1;
          e.nbp = len_bnd[b + 1] >> 5;
        }
        e.meta = ci.npat | (ci.dist << 8) | (lp << 16);
        sd.push_back(e);
      }
    }
    if (sd.empty()) sd.push_back(SegDesc{});
    d.seg_desc = c->b_seg_desc.upload(sd, s);
  };

  std::vector<uint32_t> g_first(G), g_arity(G);
  std::vector<uint8_t> g_dist(G);
  std::vector<double> g_param(G);
  for (uint64_t g = 0; g < G; ++g) {
    g_first[g] = h.groups[g].first_symbol;
    g_arity[g] = h.groups[g].arity;
    g_dist[g] = h.groups[g].dist;
    g_param[g] = h.groups[g].param;
  }

  d.row_ptr = c->b_row_ptr.upload(h.row_ptr, s);
  d.sym_idx = c->b_sym_idx.upload(h.sym_idx, s);
  d.col_ptr = c->b_col_ptr.upload(col_ptr, s);
  d.col_rows = c->b_col_rows.upload(col_rows, s);
  if (!h.dense_words.empty()) {
    d.dense = c->b_dense.upload(h.dense_words, s);
    d.ldm = h.ldm;
    const std::vector<uint8_t> gm = group_major_bytes(h, &d.gm_ld);
    d.dense_gm = c->b_dense_gm.upload(gm, s);
    ck(cudaStreamSynchronize(s), "dense upload");
  }
  d.g_first = c->b_first.upload(g_first, s);
  d.g_arity = c->b_arity.upload(g_arity, s);
  d.g_dist = c->b_dist.upload(g_dist, s);
  d.g_param = c->b_param.upload(g_param, s);
  d.row_const_compat = c->b_row_const_compat.upload(row_const_compat, s);
  d.n_ones = static_cast<uint32_t>(ones.size());
  d.ones_syms = c->b_ones.upload(ones, s);
  d.dense_sym = c->b_dense_sym.upload(dense_sym, s);
  {
    std::vector<uint16_t> coin_rows(coin_rows_k.size() + 1, 0);
    for (size_t i = 0; i < coin_rows_k.size(); ++i)
      coin_rows[i] = static_cast<uint16_t>(coin_rows_k[i] * d.tw);
    d.coin_ptr = c->b_coin_ptr.upload(coin_ptr, s);
    d.coin_rows = c->b_coin_rows.upload(coin_rows, s);
    d.n_coin_rows = static_cast<uint32_t>(coin_rows_k.size());
    if (c->fused_ok && env_long("SP_COINS_SMEM", 1) != 0) {
      DevPlan t = d;
      t.coins_staged = 1;
      if (fused_smem_bytes(t, t.t_log2, t.staged, t.row_staged, t.n_buf) <= optin) d.coins_staged = 1;
    }
  }
  d.n_cls_all = static_cast<uint32_t>(n_cls_ld);
  d.n_cls_null = static_cast<uint32_t>(cls_info.size() - n_cls_ld);
  apply_segments(live_nseg);
  if (thin_src.empty()) thin_src.push_back(UINT32_MAX);  // never read; keeps the buffer non-null
  d.thin_src = c->b_thin_src.upload(thin_src, s);
  if (len_bnd.empty()) len_bnd.push_back(0xFFFFFFFFu);
  d.len_bnd = c->b_len_bnd.upload(len_bnd, s);
  d.n_len_bnd = static_cast<uint32_t>(len_bnd.size());
  if (mech_pat.empty()) mech_pat.push_back(0);
  d.mech_pat = c->b_mech_pat.upload(mech_pat, s);
  d.g_masks = c->b_g_masks.upload(g_masks, s);
  d.cls_groups = c->b_cls_groups.upload(cls_groups, s);
  d.desc = c->b_desc.upload(desc, s);
  d.colrow = c->b_colrow.upload(colrow16, s);
  {
    const long force_lp = env_long("SP_LP", -1);
    d.lp = max_plist <= 4 ? 4 : max_plist <= 8 ? 8 : max_plist <= 16 ? 16 : 0;
    if (force_lp >= 0) d.lp = static_cast<uint32_t>(force_lp);
    if (d.lp && d.lp < max_plist) d.lp = 0;
    // Unconditional padded XORs cost ATOMS throughput (~12 lanes/clk/SM on
    // B200); they only pay off when firings per shot are few.
    d.pad_pred = events_per_shot * d.lp > 32.0;
    if (const long fp = env_long("SP_PAD_PRED", -1); fp >= 0) d.pad_pred = fp != 0;
    if (d.lp) {
      // Entries: u8 row indices when the tile has <= 256 rows (a list is
      // 4-16 bytes, so the table stays in L1), else byte offsets into the
      // tile (row * tw * 4: a flip is one add + one shared XOR). Padding =
      // the spare tile row (row n_meas), absorbed and never read; one extra
      // all-padding list (index n_lists) stands in for invalid slots.
      const size_t n_lists = pl_off.size() - 1;
      d.plist_dummy = static_cast<uint32_t>(n_lists);
      const uint64_t tile_bytes = (n_meas * d.tw + spare_words(d.tw)) * 4;
      d.entry_bytes = n_meas < 256 ? 1 : tile_bytes <= 65536 ? 2 : 4;
      if (const long fe = env_long("SP_ENTRY_BYTES", 0); fe == 2 || fe == 4) d.entry_bytes = fe;
      if (d.entry_bytes == 2 && tile_bytes > 65536) d.entry_bytes = 4;
      // padding: spare-region offsets varied per list and entry, so the
      // padding XORs of a warp spread over the banks (u8: the spare row)
      const size_t n_ent = (n_lists + 1) * d.lp;
      std::vector<uint8_t> bytes(((n_ent * d.entry_bytes) + 15) & ~size_t{15}, 0);
      for (size_t i = 0; i <= n_lists; ++i) {
        const size_t len = i < n_lists ? pl_off[i + 1] - pl_off[i] : 0;
        for (size_t j = 0; j < d.lp; ++j) {
          uint32_t v;
          if (j < len) {
            const uint32_t r = pl_rows[pl_off[i] + j];
            v = d.entry_bytes == 1 ? r / d.tw : 4u * r;
          } else {
            v = d.entry_bytes == 1 ? static_cast<uint32_t>(n_meas)
                                   : 4u * static_cast<uint32_t>(n_meas * d.tw + ((i * 7 + j * 13) & 31));
          }
          std::memcpy(bytes.data() + (i * d.lp + j) * d.entry_bytes, &v, d.entry_bytes);  // little-endian
        }
      }
      std::vector<uint4> packed(bytes.size() / 16);
      std::memcpy(packed.data(), bytes.data(), bytes.size());
      d.plist = c->b_plist.upload(packed, s);
      // texel = one list (4, 8 bytes) or a 16-byte piece of it
      if (c->plist_tex) {
        cudaDestroyTextureObject(c->plist_tex);
        c->plist_tex = 0;
      }
      d.plist_tex = 0;
      if (env_long("SP_LIST_TEX", 1) != 0) {
        const uint32_t lb = d.lp * d.entry_bytes;  // bytes per list
        const uint32_t tb = lb >= 16 ? 16 : lb;    // bytes per texel
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypeLinear;
        rd.res.linear.devPtr = const_cast<uint4*>(d.plist);
        rd.res.linear.sizeInBytes = packed.size() * 16;
        rd.res.linear.desc = cudaCreateChannelDesc(32, tb >= 8 ? 32 : 0, tb >= 16 ? 32 : 0,
                                                   tb >= 16 ? 32 : 0, cudaChannelFormatKindUnsigned);
        cudaTextureDesc td{};
        td.readMode = cudaReadModeElementType;
        cudaDeviceProp prop{};
        int dev = 0;
        cudaGetDevice(&dev);
        int max_lin = 0;
        cudaDeviceGetAttribute(&max_lin, cudaDevAttrMaxTexture1DLinearWidth, dev);
        if (tb >= 4 && packed.size() * 16 / tb <= static_cast<size_t>(max_lin) &&
            cudaCreateTextureObject(&c->plist_tex, &rd, &td, nullptr) == cudaSuccess)
          d.plist_tex = c->plist_tex;
        else
          cudaGetLastError();
        (void)prop;
      }
    }
  }
  {
    // K7 (k7_queued.cuh) serves plans whose live classes are all one-list
    // Bernoulli (mechanism) classes with exact flip lists of at most four
    // words: a firing is then one u32, (list index << t_log2) | shot.
    // SP_QUEUED=0 keeps K1; SP_Q_WALK / SP_Q_APPLY / SP_Q_DEPTH / SP_Q_THREADS set the shape.
    bool ok = c->fused_ok && d.lp != 0 && d.lp * d.entry_bytes <= 16 && !live_cls.empty();
    for (const Cls& cl : live_cls) ok = ok && cl.dist == SP_DIST_BERNOULLI;
    ok = ok && ((static_cast<uint64_t>(pl_off.size()) + 1) << d.t_log2) < (1ull << 32);
    d.q_threads = env_long("SP_Q_THREADS", 1024) == 768 ? 768 : 1024;
    const long warps = d.q_threads / 32;
    long qw = std::max<long>(1, env_long("SP_Q_WALK", 8));
    long qa = std::max<long>(1, env_long("SP_Q_APPLY", qw));
    qa = std::max<long>(qw, qa / qw * qw);
    if (qw + qa >= warps) ok = false;
    const long qd = std::min<long>(std::max<long>(env_long("SP_Q_DEPTH", 4), 2), 64);
    uint32_t qdl = 1;
    while ((1l << qdl) < qd) ++qdl;
    d.q_walk = static_cast<uint32_t>(qw);
    d.q_apply = static_cast<uint32_t>(qa);
    d.q_depth_log2 = qdl;
    d.q_drain_teams = env_long("SP_Q_TEAMS", 2) == 1 ? 1u : 2u;
    // SP_QUEUED: 1 = K7 whenever eligible, 0 = never, unset = the launch
    // autotune times it against K1 and keeps the faster
    d.queued_ok = ok && d.plist_tex != 0 && env_long("SP_QUEUED", -1) != 0;
    d.q_fixed_shape = std::getenv("SP_Q_WALK") != nullptr || std::getenv("SP_Q_APPLY") != nullptr;
    for (int kd = 0; kd < 4; ++kd) {
      d.q_sel[kd] = d.queued_ok && env_long("SP_QUEUED", -1) == 1;
      d.q_shape[kd] = d.q_walk;
    }
  }
  ptm.mark("uploads");
  {
    const plan::DrainPlan dp = plan::plan_drain(X.parent, h.det_ptr, h.det_meas);
    d.n_det = dp.n_det;
    d.n_gdet = static_cast<uint32_t>(dp.gdet_id.size());
    d.gdet_ptr = c->b_gdet_ptr.upload(dp.gdet_ptr, s);
    d.gdet_rows = c->b_gdet_rows.upload(dp.gdet_rows.empty() ? std::vector<uint16_t>{0} : dp.gdet_rows, s);
    d.gdet_id = c->b_gdet_id.upload(dp.gdet_id.empty() ? std::vector<uint32_t>{0} : dp.gdet_id, s);
    const auto& path_rows = dp.path_rows;
    const auto& path_ptr = dp.path_ptr;
    const auto& path_par = dp.path_par;
    const auto& keep_rows = dp.keep_rows;
    const auto& round_ptr = dp.round_ptr;
    d.n_paths = dp.n_paths;
    d.n_rounds = dp.n_rounds;
    d.n_keep = static_cast<uint32_t>(keep_rows.size());
    d.flat_rows = dp.flat;
    d.path_rows = c->b_path_rows.upload(path_rows, s);
    d.path_ptr = c->b_path_ptr.upload(path_ptr, s);
    d.path_par = c->b_path_par.upload(path_par, s);
    d.keep_rows = c->b_keep_rows.upload(keep_rows, s);
    d.round_ptr = c->b_round_ptr.upload(round_ptr, s);
  }
  d.n_live_groups = static_cast<uint32_t>(live_groups.size());
  d.live_groups = c->b_live_groups.upload(live_groups, s);
  d.debug_mode = static_cast<uint32_t>(env_long("SP_DEBUG_MODE", 0));
  d.wait_ns = static_cast<uint32_t>(std::max<long>(32, env_long("SP_WAIT_NS", 256)));
  d.bulk_store = static_cast<uint32_t>(env_long("SP_BULK", 1));
  d.drain_teams = env_long("SP_DRAIN_TEAMS", 1) == 2 && d.n_buf >= 2 ? 2u : 1u;
  d.seg_stage_ok = static_cast<uint32_t>(env_long("SP_SEG_STAGE", 1));
  if (env_long("SP_TMA_ZERO", 1) != 0) {
    const size_t zb = static_cast<size_t>(n_meas) * d.tw * 4;
    d.zero_src = static_cast<const uint32_t*>(c->b_zero.ensure(std::max<size_t>(zb, 16)));
    ck(cudaMemsetAsync(const_cast<uint32_t*>(d.zero_src), 0, std::max<size_t>(zb, 16), s), "zero tile");
  }
  if (env_long("SP_PHASE_TIMERS", 0)) {
    std::vector<long long> z(8, 0);
    d.timers = c->b_timers.upload(z, s);
  }
  ck(cudaStreamSynchronize(s), "plan upload");

  ptm.mark("paths");
  // Launch autotune: the generator/drain warp split and the padded-XOR mode
  // (launch parameters only: results do not depend on them) are measured,
  // not modelled — a few short
  // launches of the fused kernel over ~16 tiles per CTA: first the padding
  // mode at the model's split, then the splits around it. SP_GEN_WARPS /
  // SP_PAD_PRED fix a choice; SP_AUTOTUNE=0 keeps the model's.
  const bool fix_gw = env_long("SP_GEN_WARPS", 0) != 0;
  const bool fix_pp = env_long("SP_PAD_PRED", -1) >= 0 || d.lp == 0;
  // Tuned shapes are cached per (model, device, plan shape) fingerprint, so
  // re-loading the same model does not re-measure.
  const uint64_t fp =
      ((model_fingerprint(h) ^ (static_cast<uint64_t>(c->L.num_sms) << 32 | d.t_log2)) *
       0x100000001b3ull) ^
      (d.lp | static_cast<uint64_t>(d.entry_bytes) << 8 | static_cast<uint64_t>(d.cta_threads) << 16 |
       static_cast<uint64_t>(d.n_det != 0) << 32);  // detector counting shifts the tuned split
  static std::mutex tune_mu;
  // fp -> (gen_warps, pad_pred | unfused << 1 | K7 per launch kind << 4..7 | its 12 + 12 shape << 8..11)
  static std::map<uint64_t, std::pair<uint32_t, uint32_t>> tune_cache;
  bool cached = false;
  if (!fix_gw || !fix_pp) {
    std::lock_guard<std::mutex> lk(tune_mu);
    auto it = tune_cache.find(fp);
    if (it != tune_cache.end()) {
      if (!fix_gw) d.gen_warps = it->second.first;
      if (!fix_pp) d.pad_pred = it->second.second & 1u;
      c->unfused = (it->second.second & 2u) != 0;
      if (d.queued_ok && env_long("SP_QUEUED", -1) < 0) {
        const uint32_t v = it->second.second;
        for (int kd = 0; kd < 4; ++kd) {
          d.q_sel[kd] = (v >> (4 + kd)) & 1u;
          d.q_shape[kd] = ((v >> (8 + kd)) & 1u) ? 12u : 8u;
        }
      }
      cached = true;
    }
  }
  if (!cached && c->fused_ok && !live_cls.empty() && n_meas > 0 && !(fix_gw && fix_pp) &&
      env_long("SP_AUTOTUNE", 1) != 0) {
    const long n_warps = d.cta_threads / 32;
    // >= 16 tiles per CTA and >= 2^20 shots (short launches time noisily),
    // with the calibration records kept under ~512 MB
    const uint64_t T_ = 1ull << d.t_log2;
    const uint64_t per_cta = static_cast<uint64_t>(c->L.num_sms) * d.cta_per_sm;
    uint64_t cal_tiles = std::max<uint64_t>(16 * per_cta, ((1ull << 20) + T_ - 1) / T_);
    cal_tiles = std::min(cal_tiles, std::max<uint64_t>(per_cta, (512ull << 23) / (n_meas * T_)));
    const uint64_t cal_shots = cal_tiles * T_;
    const uint64_t ldw = cal_shots / 64;
    uint64_t* buf = nullptr;
    uint64_t* dcnt = nullptr;  // registered detectors: tune with their counting on
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ck(cudaMalloc(reinterpret_cast<void**>(&buf), n_meas * ldw * 8), "cudaMalloc (autotune)");
    if (d.n_det) ck(cudaMalloc(reinterpret_cast<void**>(&dcnt), d.n_det * 8ull), "cudaMalloc (autotune)");
    ck(cudaEventCreate(&e0), "cudaEventCreate");
    ck(cudaEventCreate(&e1), "cudaEventCreate");
    bool cal_tiled = true;
    auto launch_once = [&](uint64_t seed) {
      ck(cudaEventRecord(e0, s), "cudaEventRecord");
      // tiled layout: contiguous stores, so the kernel's own balance decides
      if (launch_fused_sample(d, c->L, seed, 0, cal_shots, buf, ldw, nullptr, cal_tiled, dcnt) < 0)
        throw CudaError("autotune launch failed");
      ck(cudaEventRecord(e1, s), "cudaEventRecord");
      ck(cudaEventSynchronize(e1), "cudaEventSynchronize");
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
      return ms;
    };
    auto time_launch = [&]() {
      float t = launch_once(0x5EED);
      for (int rep = 1; rep < 3; ++rep) t = std::min(t, launch_once(0x5EEDull + rep));
      return t;  // min of 3
    };
    try {
      // Warm up until the clocks settle (an idle GPU starts slow, which
      // would bias whichever candidate runs first): >= 20 ms of launches or
      // two consecutive timings within 2 %.
      {
        float prev = launch_once(1), spent = prev;
        for (int k = 0; k < 64 && spent < 20.f; ++k) {
          const float t = launch_once(2 + k);
          spent += t;
          if (spent >= 5.f && std::fabs(t - prev) < 0.02f * prev) break;
          prev = t;
        }
      }
      // (padded-XOR mode, generator warps) jointly; candidates timed round
      // robin, so drift hits all of them alike, and the min of 3 kept.
      if (!fix_gw || !fix_pp) {
        const uint32_t gw0 = d.gen_warps, pp0 = d.pad_pred;
        std::vector<std::pair<uint32_t, uint32_t>> cand;
        for (long dg : {0L, -1L, 1L, -2L, 2L}) {
          const long g = static_cast<long>(gw0) + dg;
          if (fix_gw && dg != 0) continue;
          // the model's own pick is always a candidate (a model with very
          // few firings may want a single generator warp)
          if (dg != 0 && (g < std::min<long>(n_warps / 2, gw0) || g > n_warps - 2 || g < 1)) continue;
          for (uint32_t pp : {pp0, pp0 ^ 1u}) {
            if (fix_pp && pp != pp0) continue;
            cand.emplace_back(static_cast<uint32_t>(g), pp);
          }
        }
        std::vector<float> best(cand.size(), 1e30f);
        for (int rep = 0; rep < 3; ++rep)
          for (size_t i = 0; i < cand.size(); ++i) {
            d.gen_warps = cand[i].first;
            d.pad_pred = cand[i].second;
            best[i] = std::min(best[i], launch_once(0x5EEDull + 7 * rep + i));
          }
        size_t bi = 0;  // cand[0] is the model's pick: others must beat it by 1 %
        for (size_t i = 1; i < cand.size(); ++i)
          if (best[i] < best[bi] * (bi == 0 ? 0.99f : 1.f)) bi = i;
        d.gen_warps = cand[bi].first;
        d.pad_pred = cand[bi].second;
      }
      // K7 (queued) against the tuned K1: same records, so the faster one
      // serves the launches. Two shapes: 8 + 8 warps and 12 + 12 (the rest
      // drain). Decided per launch kind — tiled or measurement-major records,
      // with or without detector counts (the drain's work and share differ).
      if (d.queued_ok && env_long("SP_QUEUED", -1) < 0) {
        std::vector<uint32_t> shapes{d.q_fixed_shape ? d.q_walk : 8u};
        if (!d.q_fixed_shape) shapes.push_back(12u);
        uint64_t* const dcnt_reg = dcnt;
        for (uint32_t kd = 0; kd < 4; ++kd) {
          if ((kd & 1u) && !dcnt_reg) {  // no detectors registered: as without counts
            d.q_sel[kd] = d.q_sel[kd - 1];
            d.q_shape[kd] = d.q_shape[kd - 1];
            continue;
          }
          dcnt = (kd & 1u) ? dcnt_reg : nullptr;
          cal_tiled = (kd & 2u) != 0;
          // candidates timed round robin (drift hits all alike), min kept;
          // 4 to 16 rounds: short launches time noisily
          std::vector<float> best(shapes.size() + 1, 1e30f);
          d.q_sel[kd] = 0;
          const float t0 = launch_once(0x5EED);
          const int reps = static_cast<int>(std::min(16.f, std::max(4.f, std::ceil(3.f / std::max(t0, 1e-3f)))));
          for (int rep = 0; rep < reps; ++rep)
            for (size_t i = 0; i <= shapes.size(); ++i) {
              d.q_sel[kd] = i > 0;
              if (i > 0) d.q_shape[kd] = shapes[i - 1];
              best[i] = std::min(best[i], launch_once(0x5EEDull + 11 * rep + i));
            }
          int bi = -1;
          float t_best = best[0] * 0.98f;  // K7 must win by 2 %
          for (size_t i = 0; i < shapes.size(); ++i)
            if (best[i + 1] < t_best) { t_best = best[i + 1]; bi = static_cast<int>(i); }
          d.q_sel[kd] = bi >= 0;
          d.q_shape[kd] = shapes[std::max(bi, 0)];
        }
        dcnt = dcnt_reg;
        cal_tiled = true;
      }
      // Fused vs unfused (device draw of S + explicit-S product): the same
      // bits for an unmerged model (K1 == M_sym . S of its own draw), so the
      // faster one serves sp_sample. Unfused wins when firings x list
      // lengths per shot are very large (cfg5 density 0.01, p = 1e-2).
      if (!merged_any && env_long("SP_UNFUSED", -1) < 0) {
        const float t_fused = time_launch() / static_cast<float>(cal_shots);
        const uint64_t n_u = std::min<uint64_t>(
            cal_shots, std::max<uint64_t>(1, (256ull << 20) / (n_sym / 8 + 1) / (1ull << d.t_log2)) << d.t_log2);
        const uint64_t ldS = n_u / 64;
        uint64_t* S = nullptr;
        ck(cudaMalloc(reinterpret_cast<void**>(&S), n_sym * ldS * 8), "cudaMalloc (autotune S)");
        float tu = 0.f;
        for (int rep = 0; rep < 3; ++rep) {
          ck(cudaEventRecord(e0, s), "cudaEventRecord");
          const int r1 = launch_draw(d, c->L, false, 0x5EEDull + rep, 0, n_u, S, ldS);
          const int r2 = run_product(c, d, S, ldS, n_u, buf, ldS);
          ck(cudaEventRecord(e1, s), "cudaEventRecord");
          ck(cudaEventSynchronize(e1), "cudaEventSynchronize");
          if (r1 < 0 || r2 < 0) {
            cudaFree(S);
            throw CudaError("autotune unfused launch failed");
          }
          float ms = 0.f;
          ck(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
          if (rep > 0) tu = rep == 1 ? ms : std::min(tu, ms);
        }
        cudaFree(S);
        c->unfused = tu / static_cast<float>(n_u) < 0.8f * t_fused;
      }
    } catch (...) {
      cudaFree(buf);
      if (dcnt) cudaFree(dcnt);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      throw;
    }
    cudaFree(buf);
    if (dcnt) cudaFree(dcnt);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (d.timers) d.timers = c->b_timers.upload(std::vector<long long>(8, 0), s);
    ck(cudaStreamSynchronize(s), "plan upload");
    std::lock_guard<std::mutex> lk(tune_mu);
    uint32_t qbits = 0;
    for (int kd = 0; kd < 4; ++kd)
      qbits |= (d.q_sel[kd] ? 1u << (4 + kd) : 0u) | (d.q_shape[kd] == 12 ? 1u << (8 + kd) : 0u);
    tune_cache[fp] = {d.gen_warps, d.pad_pred | (c->unfused ? 2u : 0u) | qbits};
  }
  ptm.mark("autotune");
  build_k5(c, col_ptr, col_rows, ones, events_per_shot, flips_per_shot, n_dense_live);
  ptm.mark("k5");
  c->plan_ready = true;
}

// Re-upload the raw model arrays of an unchanged model; the derived plan
// (chain transform, flip lists, paths, tuned launch shape) stays.
void refresh_model_uploads(sp_ctx* c) {
  HostPlan& h = c->hp;
  DevPlan& d = c->dp;
  cudaStream_t s = c->stream;
  d.row_ptr = c->b_row_ptr.upload(h.row_ptr, s);
  d.sym_idx = c->b_sym_idx.upload(h.sym_idx, s);
  const uint64_t G = h.groups.size();
  std::vector<uint32_t> g_first(G), g_arity(G);
  std::vector<uint8_t> g_dist(G);
  std::vector<double> g_param(G);
  for (uint64_t g = 0; g < G; ++g) {
    g_first[g] = h.groups[g].first_symbol;
    g_arity[g] = h.groups[g].arity;
    g_dist[g] = h.groups[g].dist;
    g_param[g] = h.groups[g].param;
  }
  d.g_first = c->b_first.upload(g_first, s);
  d.g_arity = c->b_arity.upload(g_arity, s);
  d.g_dist = c->b_dist.upload(g_dist, s);
  d.g_param = c->b_param.upload(g_param, s);
}

int ensure_plan(sp_ctx* c) {
  if (!c->have_msym || !c->have_groups)
    return fail(SP_ERR_NOT_LOADED, "load M_sym and the group table first");
  if (c->plan_ready) return SP_OK;
  try {
    uint64_t total = 0;
    for (const sp_group& g : c->hp.groups) total += g.arity;
    if (total != c->hp.n_sym)
      return fail(SP_ERR_INVALID_ARGUMENT, "group arities do not add up to n_sym");
    // Re-loading the model this plan was built from (same content, same
    // planner switches) keeps the plan: only the raw arrays are uploaded.
    const uint64_t fp = model_fingerprint(c->hp);
    if (c->plan_built && fp == c->plan_fp) {
      refresh_model_uploads(c);
      c->plan_ready = true;
      return SP_OK;
    }
    c->plan_built = false;
    build_plan(c);
    c->plan_fp = fp;
    c->plan_built = true;
  } catch (const std::invalid_argument& e) {
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());
  } catch (const CudaError& e) {
    return fail(SP_ERR_CUDA, e.what());
  } catch (const std::bad_alloc&) {
    return fail(SP_ERR_INVALID_ARGUMENT, "host allocation failed while building the plan");
  }
  return SP_OK;
}

int launched(sp_ctx* c, int r, const char* what) {
  if (r < 0) {
    cudaError_t e = cudaGetLastError();
    return fail(SP_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  c->launches += static_cast<uint64_t>(r);
  return SP_OK;
}

}  // namespace

extern "C" {

const char* sp_last_error(void) { return g_err.c_str(); }
int sp_abi_version(void) { return SP_ABI_VERSION; }

int sp_model_from_text(const char* text, sp_model** out) {
  if (!text || !out) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  try {
    auto m = new sp_model;
    try {
      m->m = run_initialization(parse_circuit(text));
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
    return SP_OK;
  } catch (const ParseError& e) {
    return fail(SP_ERR_PARSE, e.what());
  } catch (const std::logic_error& e) {
    return fail(SP_ERR_LOGIC, e.what());
  } catch (const std::exception& e) {
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());
  }
}

int sp_parse_circuit(const char* text, uint64_t cap_instr, uint8_t* kinds, double* params,
                     uint64_t* lines, uint64_t* tgt_ptr, uint64_t cap_targets, uint32_t* targets,
                     uint64_t* n_instr_out, uint64_t* n_targets_out) {
  if (!text || !n_instr_out || !n_targets_out) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  try {
    const std::vector<Instr> prog = parse_circuit(text);
    uint64_t nt = 0;
    for (const Instr& in : prog) nt += in.targets.size();
    *n_instr_out = prog.size();
    *n_targets_out = nt;
    if (!kinds) return SP_OK;  // sizes only
    if (cap_instr < prog.size() || cap_targets < nt || !params || !lines || !tgt_ptr || (nt && !targets))
      return fail(SP_ERR_INVALID_ARGUMENT, "output buffers too small");
    uint64_t t = 0;
    tgt_ptr[0] = 0;
    for (size_t i = 0; i < prog.size(); ++i) {
      kinds[i] = static_cast<uint8_t>(prog[i].op);
      params[i] = prog[i].p;
      lines[i] = prog[i].line;
      for (uint32_t q : prog[i].targets) targets[t++] = q;
      tgt_ptr[i + 1] = t;
    }
    return SP_OK;
  } catch (const ParseError& e) {
    return fail(SP_ERR_PARSE, e.what());
  } catch (const std::exception& e) {
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());
  }
}

int sp_model_from_program(uint64_t n_instr, const uint8_t* kinds, const double* params,
                          const uint64_t* tgt_ptr, const uint32_t* targets, sp_model** out) {
  if (!out || (n_instr && (!kinds || !params || !tgt_ptr)))
    return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  try {
    std::vector<Instr> prog(n_instr);
    for (uint64_t i = 0; i < n_instr; ++i) {
      if (kinds[i] > static_cast<uint8_t>(Op::Tick))
        return fail(SP_ERR_INVALID_ARGUMENT, "unknown instruction kind");
      Instr& in = prog[i];
      in.op = static_cast<Op>(kinds[i]);
      in.p = params[i];
      if (tgt_ptr[i + 1] < tgt_ptr[i] || (tgt_ptr[i + 1] > tgt_ptr[i] && !targets))
        return fail(SP_ERR_INVALID_ARGUMENT, "bad target offsets");
      in.targets.assign(targets + tgt_ptr[i], targets + tgt_ptr[i + 1]);
      // the shape rules parse_circuit enforces (circuit.cpp:79-168)
      const bool noise = in.op == Op::XErr || in.op == Op::YErr || in.op == Op::ZErr ||
                         in.op == Op::Dep1 || in.op == Op::Dep2;
      const bool pairs = in.op == Op::CX || in.op == Op::Dep2;
      if (noise && (in.p < 0.0 || in.p > 1.0))
        return fail(SP_ERR_INVALID_ARGUMENT, "probability out of [0,1]");
      if ((in.op == Op::Tick) != in.targets.empty())
        return fail(SP_ERR_INVALID_ARGUMENT, in.op == Op::Tick ? "TICK takes no targets" : "missing targets");
      if (pairs) {
        if (in.targets.size() & 1) return fail(SP_ERR_INVALID_ARGUMENT, "odd number of pair targets");
        for (size_t k = 0; k < in.targets.size(); k += 2)
          if (in.targets[k] == in.targets[k + 1])
            return fail(SP_ERR_INVALID_ARGUMENT, "pair targets the same qubit twice");
      }
    }
    auto m = std::make_unique<sp_model>();
    m->m = run_initialization(prog);
    *out = m.release();
    return SP_OK;
  } catch (const std::logic_error& e) {
    return fail(SP_ERR_LOGIC, e.what());
  } catch (const std::exception& e) {
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());
  }
}

void sp_model_destroy(sp_model* m) { delete m; }

int sp_model_dims(const sp_model* m, uint64_t* n_qubits, uint64_t* n_meas, uint64_t* n_sym,
                  uint64_t* n_groups, uint64_t* nnz) {
  if (!m) return fail(SP_ERR_INVALID_ARGUMENT, "null model");
  if (n_qubits) *n_qubits = m->m.n_qubits;
  if (n_meas) *n_meas = m->m.n_meas();
  if (n_sym) *n_sym = m->m.n_sym;
  if (n_groups) *n_groups = m->m.groups.size();
  if (nnz) *nnz = m->m.sym_idx.size();
  return SP_OK;
}

int sp_model_export(const sp_model* m, uint64_t* row_ptr, uint32_t* sym_idx, sp_group* groups) {
  if (!m) return fail(SP_ERR_INVALID_ARGUMENT, "null model");
  if (row_ptr) std::memcpy(row_ptr, m->m.row_ptr.data(), m->m.row_ptr.size() * 8);
  if (sym_idx && !m->m.sym_idx.empty())
    std::memcpy(sym_idx, m->m.sym_idx.data(), m->m.sym_idx.size() * 4);
  if (groups) {
    for (size_t g = 0; g < m->m.groups.size(); ++g) {
      sp_group o{};
      o.dist = m->m.groups[g].dist;
      o.param = m->m.groups[g].param;
      o.first_symbol = m->m.groups[g].first;
      o.arity = m->m.groups[g].arity;
      groups[g] = o;
    }
  }
  return SP_OK;
}

int sp_detector_rows(uint64_t n_meas, const uint64_t* row_ptr, const uint32_t* sym_idx,
                     uint64_t n_det, const uint64_t* det_ptr, const uint32_t* det_meas,
                     uint64_t* out_row_ptr, uint32_t* out_sym_idx, uint64_t cap,
                     uint64_t* nnz_out) {
  if (!row_ptr || (n_det && (!det_ptr || (det_ptr[n_det] && !det_meas))) || !out_row_ptr || !nnz_out)
    return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  try {
    std::vector<uint32_t> acc, tmp;
    uint64_t nnz = 0;
    out_row_ptr[0] = 0;
    for (uint64_t k = 0; k < n_det; ++k) {
      acc.clear();
      for (uint64_t i = det_ptr[k]; i < det_ptr[k + 1]; ++i) {
        const uint64_t m = det_meas[i];
        if (m >= n_meas) return fail(SP_ERR_OUT_OF_RANGE, "detector measurement id out of range");
        tmp.clear();
        std::set_symmetric_difference(acc.begin(), acc.end(), sym_idx + row_ptr[m],
                                      sym_idx + row_ptr[m + 1], std::back_inserter(tmp));
        acc.swap(tmp);
      }
      if (out_sym_idx) {
        if (nnz + acc.size() > cap) return fail(SP_ERR_INVALID_ARGUMENT, "out_sym_idx too small");
        std::copy(acc.begin(), acc.end(), out_sym_idx + nnz);
      }
      nnz += acc.size();
      out_row_ptr[k + 1] = nnz;
    }
    *nnz_out = nnz;
  } catch (const std::bad_alloc&) {
    return fail(SP_ERR_INVALID_ARGUMENT, "host allocation failed");
  }
  return SP_OK;
}

int sp_ctx_create(int device, sp_ctx** out) {
  if (!out) return fail(SP_ERR_INVALID_ARGUMENT, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(SP_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(SP_ERR_INVALID_ARGUMENT, "device index out of range");
  auto c = new sp_ctx;
  c->device = device;
  if (int r = set_device(c)) {
    delete c;
    return r;
  }
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    delete c;
    return fail(SP_ERR_UNSUPPORTED, "this library is built for sm_100a (B200)");
  }
  c->L.num_sms = prop.multiProcessorCount;
  c->L.smem_optin = prop.sharedMemPerBlockOptin;
  *out = c;
  return SP_OK;
}

void sp_ctx_destroy(sp_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  delete ctx;
}

int sp_set_stream(sp_ctx* ctx, void* stream) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  ctx->stream = static_cast<cudaStream_t>(stream);
  ctx->L.stream = ctx->stream;
  return SP_OK;
}

int sp_set_rng(sp_ctx* ctx, sp_rng rng) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (rng != SP_RNG_PHILOX && rng != SP_RNG_COMPAT_SPLITMIX)
    return fail(SP_ERR_INVALID_ARGUMENT, "unknown rng");
  ctx->rng = rng;
  return SP_OK;
}

int sp_set_product(sp_ctx* ctx, sp_product v) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (v != SP_PRODUCT_AUTO && v != SP_PRODUCT_SPARSE && v != SP_PRODUCT_DENSE && v != SP_PRODUCT_TENSOR)
    return fail(SP_ERR_INVALID_ARGUMENT, "unknown product variant");
  ctx->product = v;
  if (dense_product(ctx) && ctx->hp.dense_words.empty() && ctx->have_msym) {
    // Build the dense words from the CSR rows on first request.
    ensure_dense_words(ctx->hp);
    ctx->plan_ready = false;
    ctx->prod_ready = false;
    ctx->tc_ready = false;
  }
  return SP_OK;
}

int sp_load_msym_csr(sp_ctx* ctx, uint64_t n_meas, uint64_t n_sym, const uint64_t* row_ptr,
                     const uint32_t* sym_idx) {
  if (!ctx || !row_ptr) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (n_meas >= (1ull << 31) || n_sym >= (1ull << 32) - 1)
    return fail(SP_ERR_UNSUPPORTED, "M_sym dimensions exceed 32-bit indexing");
  HostPlan& h = ctx->hp;
  h.n_meas = n_meas;
  h.n_sym = n_sym;
  h.row_ptr.assign(row_ptr, row_ptr + n_meas + 1);
  if (h.row_ptr[0] != 0) return fail(SP_ERR_INVALID_ARGUMENT, "row_ptr[0] must be 0");
  h.nnz = h.row_ptr[n_meas];
  h.sym_idx.assign(sym_idx, sym_idx + h.nnz);
  h.max_sym_plus1 = 0;
  for (uint64_t k = 0; k < n_meas; ++k) {
    if (h.row_ptr[k + 1] < h.row_ptr[k]) return fail(SP_ERR_INVALID_ARGUMENT, "row_ptr not monotone");
    for (uint64_t i = h.row_ptr[k]; i < h.row_ptr[k + 1]; ++i) {
      if (i > h.row_ptr[k] && h.sym_idx[i] <= h.sym_idx[i - 1])
        return fail(SP_ERR_INVALID_ARGUMENT, "expression symbols must be strictly increasing");
      h.max_sym_plus1 = std::max<uint64_t>(h.max_sym_plus1, uint64_t{h.sym_idx[i]} + 1);
    }
  }
  h.dense_words.clear();
  h.ldm = 0;
  ctx->have_msym = true;
  ctx->plan_ready = false;
  ctx->prod_ready = false;
  ctx->tc_ready = false;
  if (ctx->product == SP_PRODUCT_DENSE) sp_set_product(ctx, SP_PRODUCT_DENSE);
  return SP_OK;
}

int sp_load_msym_dense(sp_ctx* ctx, uint64_t n_meas, uint64_t n_sym, const uint64_t* words,
                       uint64_t ld_words) {
  if (!ctx || (!words && n_meas)) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (ld_words < (n_sym + 63) / 64) return fail(SP_ERR_INVALID_ARGUMENT, "ld_words too small");
  std::vector<uint64_t> rp{0};
  std::vector<uint32_t> si;
  for (uint64_t k = 0; k < n_meas; ++k) {
    for (uint64_t w = 0; w < (n_sym + 63) / 64; ++w) {
      uint64_t x = words[k * ld_words + w];
      if (w == (n_sym - 1) / 64 && n_sym % 64) x &= (uint64_t{1} << (n_sym % 64)) - 1;
      while (x) {
        si.push_back(static_cast<uint32_t>(w * 64 + __builtin_ctzll(x)));
        x &= x - 1;
      }
    }
    rp.push_back(si.size());
  }
  int r = sp_load_msym_csr(ctx, n_meas, n_sym, rp.data(), si.data());
  if (r) return r;
  HostPlan& h = ctx->hp;
  h.ldm = std::max<uint64_t>((n_sym + 63) / 64, 1);
  h.dense_words.assign(n_meas * h.ldm, 0);
  for (uint64_t k = 0; k < n_meas; ++k)
    for (uint64_t w = 0; w < (n_sym + 63) / 64; ++w) h.dense_words[k * h.ldm + w] = words[k * ld_words + w];
  if (n_sym % 64)
    for (uint64_t k = 0; k < n_meas; ++k)
      h.dense_words[k * h.ldm + (n_sym - 1) / 64] &= (uint64_t{1} << (n_sym % 64)) - 1;
  ctx->prod_ready = false;
  ctx->tc_ready = false;
  return SP_OK;
}

int sp_load_groups(sp_ctx* ctx, uint64_t n_groups, const sp_group* groups) {
  if (!ctx || !groups || n_groups == 0) return fail(SP_ERR_INVALID_ARGUMENT, "need >= 1 group");
  const sp_group& g0 = groups[0];
  if (g0.dist != SP_DIST_CONSTANT || g0.first_symbol != 0 || g0.arity != 1)
    return fail(SP_ERR_INVALID_ARGUMENT, "group 0 must be the constant symbol s0");
  for (uint64_t g = 1; g < n_groups; ++g) {
    const sp_group& x = groups[g];
    uint32_t want = x.dist == SP_DIST_DEPOLARIZE1 ? 2 : x.dist == SP_DIST_DEPOLARIZE2 ? 4 : 1;
    if (x.dist > SP_DIST_DEPOLARIZE2 || x.arity != want)
      return fail(SP_ERR_INVALID_ARGUMENT, "group arity does not match its distribution");
  }
  ctx->hp.groups.assign(groups, groups + n_groups);
  ctx->hp.n_groups = n_groups;
  ctx->have_groups = true;
  ctx->plan_ready = false;
  return SP_OK;
}

int sp_load_model(sp_ctx* ctx, const sp_model* m) {
  if (!ctx || !m) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  int r = sp_load_msym_csr(ctx, m->m.n_meas(), m->m.n_sym, m->m.row_ptr.data(), m->m.sym_idx.data());
  if (r) return r;
  std::vector<sp_group> g(m->m.groups.size());
  sp_model_export(m, nullptr, nullptr, g.data());
  return sp_load_groups(ctx, g.size(), g.data());
}

int sp_shot_tile(sp_ctx* ctx, uint64_t* tile) {
  if (!ctx || !tile) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  *tile = 1ull << ctx->dp.t_log2;
  return SP_OK;
}

int sp_sample(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots, uint64_t* d_out,
              uint64_t ld, uint64_t* d_counts) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (n_shots == 0) return fail(SP_ERR_INVALID_ARGUMENT, "need at least one shot");  // sampler.cpp:50
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  const uint64_t T = 1ull << ctx->dp.t_log2;
  if (shot_begin % T) return fail(SP_ERR_INVALID_ARGUMENT, "shot_begin must be a multiple of the shot tile");
  if (ctx->hp.n_meas == 0) return SP_OK;
  if (!d_out || ld < (n_shots + 63) / 64) return fail(SP_ERR_INVALID_ARGUMENT, "output too small");
  if (ctx->k5_ok && ctx->rng == SP_RNG_PHILOX) {  // column sampler (dense M_sym)
    const int r = launch_k5(ctx->k5, ctx->L, seed, shot_begin, n_shots, d_out, ld, d_counts);
    return launched(ctx, r, "K5 column sampler launch");
  }
  if (!ctx->fused_ok || (ctx->unfused && ctx->rng == SP_RNG_PHILOX)) {
    // Too many rows for an on-chip shot tile, or measured faster: the same
    // streams through the unfused path, draw S (device) then the explicit-S
    // product, in shot chunks that keep S under ~2 GB. Same records as the
    // fused kernel.
    const uint64_t per_shot = std::max<uint64_t>(ctx->hp.n_sym, 1) / 8 + 1;
    uint64_t chunk = std::max<uint64_t>((2ull << 30) / per_shot / T, 1) * T;
    chunk = std::min(chunk, (n_shots + T - 1) / T * T);
    const uint64_t ldS = chunk / 64;
    try {
      uint64_t* d_S = static_cast<uint64_t*>(ctx->s_S.ensure(ctx->hp.n_sym * ldS * 8));
      for (uint64_t done = 0; done < n_shots; done += chunk) {
        const uint64_t n = std::min(chunk, n_shots - done);
        if (int r = sp_draw_assignments(ctx, seed, shot_begin + done, n, d_S, ldS)) return r;
        if (int r = sp_sample_given_S(ctx, d_S, ctx->hp.n_sym, ldS, n, d_out + done / 64, ld))
          return r;
        if (d_counts) {
          const int r = launch_row_counts(ctx->L, d_out + done / 64, ld, ctx->hp.n_meas, n, d_counts);
          if (int e = launched(ctx, r, "row counts launch")) return e;
        }
      }
    } catch (const CudaError& e) {
      return fail(SP_ERR_CUDA, e.what());
    }
    return SP_OK;
  }
  const uint64_t tile0 = shot_begin / T;
  int r = ctx->rng == SP_RNG_PHILOX
              ? launch_fused_sample(ctx->dp, ctx->L, seed, tile0, n_shots, d_out, ld, d_counts)
              : launch_fused_sample_compat(ctx->dp, ctx->L, seed, tile0, n_shots, d_out, ld, d_counts);
  return launched(ctx, r, "fused sampler launch");
}

int sp_set_detectors(sp_ctx* ctx, uint64_t n_det, const uint64_t* det_ptr, const uint32_t* det_meas) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (n_det && (!det_ptr || det_ptr[0] != 0 || (det_ptr[n_det] && !det_meas)))
    return fail(SP_ERR_INVALID_ARGUMENT, "detector CSR: det_ptr[0] must be 0 and det_meas non-null");
  if (n_det > 0xFFFFFFFFull) return fail(SP_ERR_INVALID_ARGUMENT, "too many detectors");
  for (uint64_t j = 0; j < n_det; ++j)
    if (det_ptr[j + 1] < det_ptr[j]) return fail(SP_ERR_INVALID_ARGUMENT, "det_ptr must not decrease");
  if (ctx->have_msym)
    for (uint64_t i = 0; i < (n_det ? det_ptr[n_det] : 0); ++i)
      if (det_meas[i] >= ctx->hp.n_meas)
        return fail(SP_ERR_OUT_OF_RANGE, "detector refers to a measurement out of range");
  ctx->hp.det_ptr.assign(det_ptr ? det_ptr : nullptr, det_ptr ? det_ptr + n_det + 1 : nullptr);
  if (ctx->hp.det_ptr.empty()) ctx->hp.det_ptr.push_back(0);
  ctx->hp.det_meas.assign(det_meas, det_meas + (n_det ? det_ptr[n_det] : 0));
  ctx->plan_ready = false;
  return SP_OK;
}

int sp_sample_ex(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots, uint64_t* d_out,
                 uint64_t ld, uint64_t* d_counts, uint64_t* d_det_counts) {
  if (!d_det_counts)
    return ld ? sp_sample(ctx, seed, shot_begin, n_shots, d_out, ld, d_counts)
              : sp_sample_tiled(ctx, seed, shot_begin, n_shots, d_out, d_counts);
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (n_shots == 0) return fail(SP_ERR_INVALID_ARGUMENT, "need at least one shot");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  if (ctx->hp.det_ptr.size() < 2) return fail(SP_ERR_NOT_LOADED, "no detectors registered (sp_set_detectors)");
  if (!ctx->fused_ok || ctx->k5_ok || ctx->unfused || ctx->rng != SP_RNG_PHILOX)
    return fail(SP_ERR_UNSUPPORTED, "detector counts are produced by the fused Philox sampler only");
  const uint64_t T = 1ull << ctx->dp.t_log2;
  if (shot_begin % T) return fail(SP_ERR_INVALID_ARGUMENT, "shot_begin must be a multiple of the shot tile");
  if (!d_out || (ld && ld < (n_shots + 63) / 64)) return fail(SP_ERR_INVALID_ARGUMENT, "output too small");
  const int r = launch_fused_sample(ctx->dp, ctx->L, seed, shot_begin / T, n_shots, d_out, ld,
                                    d_counts, ld == 0, d_det_counts);
  return launched(ctx, r, "fused sampler launch");
}

uint64_t sp_tiled_words(sp_ctx* ctx, uint64_t n_shots) {
  if (!ctx || set_device(ctx) || ensure_plan(ctx)) return 0;
  const uint64_t T = 1ull << ctx->dp.t_log2;
  return (n_shots + T - 1) / T * ctx->hp.n_meas * (T / 64);
}

int sp_sample_tiled(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
                    uint64_t* d_out, uint64_t* d_counts) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (n_shots == 0) return fail(SP_ERR_INVALID_ARGUMENT, "need at least one shot");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  if (!ctx->fused_ok) return fail(SP_ERR_UNSUPPORTED, ctx->fused_why);
  if (ctx->k5_ok)
    return fail(SP_ERR_UNSUPPORTED, "this model is sampled by the column sampler (measurement-major "
                                    "records only); use sp_sample");
  if (ctx->rng != SP_RNG_PHILOX)
    return fail(SP_ERR_UNSUPPORTED, "tiled output is produced by the Philox sampler only");
  const uint64_t T = 1ull << ctx->dp.t_log2;
  if (shot_begin % T) return fail(SP_ERR_INVALID_ARGUMENT, "shot_begin must be a multiple of the shot tile");
  if (ctx->hp.n_meas == 0) return SP_OK;
  if (!d_out) return fail(SP_ERR_INVALID_ARGUMENT, "null output");
  int r = launch_fused_sample(ctx->dp, ctx->L, seed, shot_begin / T, n_shots, d_out, 0, d_counts,
                              true);
  return launched(ctx, r, "fused sampler launch");
}

int sp_untile(sp_ctx* ctx, const uint64_t* d_tiled, uint64_t n_shots, uint64_t* d_out,
              uint64_t ld) {
  if (!ctx || !d_tiled || !d_out) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  if (ld < (n_shots + 63) / 64) return fail(SP_ERR_INVALID_ARGUMENT, "ld too small");
  int r = launch_untile(ctx->L, d_tiled, ctx->hp.n_meas, 1u << ctx->dp.t_log2, n_shots, d_out, ld);
  return launched(ctx, r, "untile launch");
}

int sp_encode_tiled(sp_ctx* ctx, const uint64_t* d_tiled, uint64_t n_shots, sp_format fmt,
                    uint8_t* d_bytes) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (fmt != SP_FMT_01 && fmt != SP_FMT_B8) return fail(SP_ERR_INVALID_ARGUMENT, "unknown format");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  int r = launch_encode(ctx->L, d_tiled, 0, ctx->hp.n_meas, n_shots, fmt, d_bytes,
                        1u << ctx->dp.t_log2);
  return launched(ctx, r, "encode launch");
}

int sp_draw_assignments(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
                        uint64_t* d_S, uint64_t ldS) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (n_shots == 0) return fail(SP_ERR_INVALID_ARGUMENT, "need at least one shot");  // sampler.cpp:50
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  const uint64_t T = 1ull << ctx->dp.t_log2;
  if (shot_begin % T) return fail(SP_ERR_INVALID_ARGUMENT, "shot_begin must be a multiple of the shot tile");
  if (!d_S || ldS < (n_shots + 63) / 64) return fail(SP_ERR_INVALID_ARGUMENT, "output too small");
  const bool k5 = ctx->k5_ok && ctx->rng == SP_RNG_PHILOX;
  int r = launch_draw(ctx->dp, ctx->L, ctx->rng == SP_RNG_COMPAT_SPLITMIX, seed, shot_begin / T,
                      n_shots, d_S, ldS, !k5);
  if (int e = launched(ctx, r, "draw launch")) return e;
  if (k5) {  // the K5 streams: exactly the symbols the column sampler fires
    r = launch_k5_draw(ctx->k5, ctx->L, seed, shot_begin, n_shots, d_S, ldS);
    return launched(ctx, r, "K5 draw launch");
  }
  return SP_OK;
}

int sp_sample_given_S(sp_ctx* ctx, const uint64_t* d_S, uint64_t n_sym_S, uint64_t ldS,
                      uint64_t n_shots, uint64_t* d_out, uint64_t ld) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (!ctx->have_msym) return fail(SP_ERR_NOT_LOADED, "load M_sym first");
  if (ctx->hp.max_sym_plus1 > n_sym_S)
    return fail(SP_ERR_OUT_OF_RANGE, "symbol id out of range");  // sampler.cpp:63-67
  if (int r = set_device(ctx)) return r;
  if (n_shots == 0 || ctx->hp.n_meas == 0) return SP_OK;
  if (!d_S || ldS < (n_shots + 63) / 64 || !d_out || ld < (n_shots + 63) / 64)
    return fail(SP_ERR_INVALID_ARGUMENT, "buffer too small");
  // K2 only needs the row lists (and dense words): it has its own device
  // copy, independent of the group table and of the fused sampler's plan.
  const bool dense = dense_product(ctx);
  if (dense && ctx->hp.dense_words.empty()) {
    ensure_dense_words(ctx->hp);
    ctx->prod_ready = false;
    ctx->tc_ready = false;
  }
  if (!ctx->prod_ready) {
    try {
      ctx->pp = DevPlan{};
      ctx->pp.n_meas = static_cast<uint32_t>(ctx->hp.n_meas);
      ctx->pp.n_sym = static_cast<uint32_t>(ctx->hp.n_sym);
      ctx->pp.row_ptr = ctx->p_row_ptr.upload(ctx->hp.row_ptr, ctx->stream);
      ctx->pp.sym_idx = ctx->p_sym_idx.upload(ctx->hp.sym_idx, ctx->stream);
      {
        // segment work list: rows cut into pieces of <= kSegLen symbols
        const uint64_t kSegLen = static_cast<uint64_t>(env_long("SP_K2_SEG", 1024));
        std::vector<uint64_t> sp{0};
        std::vector<uint32_t> sr, split;
        for (uint64_t k = 0; k < ctx->hp.n_meas; ++k) {
          const uint64_t b = ctx->hp.row_ptr[k], e = ctx->hp.row_ptr[k + 1];
          const uint64_t pieces = e - b > kSegLen ? (e - b + kSegLen - 1) / kSegLen : 1;
          if (pieces > 1) split.push_back(static_cast<uint32_t>(k));
          for (uint64_t q = 0; q < pieces; ++q) {
            sp.push_back(pieces > 1 ? std::min(e, b + (q + 1) * kSegLen) : e);
            sr.push_back(static_cast<uint32_t>(k) | (pieces > 1 ? 0x80000000u : 0u));
          }
        }
        if (!split.empty()) {  // only worth a work list when some row is cut
          ctx->pp.k2_seg_ptr = ctx->p_seg_ptr.upload(sp, ctx->stream);
          ctx->pp.k2_seg_row = ctx->p_seg_row.upload(sr, ctx->stream);
          ctx->pp.k2_split_rows = ctx->p_split_rows.upload(split, ctx->stream);
          ctx->pp.n_k2_seg = static_cast<uint32_t>(sr.size());
          ctx->pp.n_k2_split = static_cast<uint32_t>(split.size());
          ck(cudaStreamSynchronize(ctx->stream), "segment upload");
        }
      }
      if (!ctx->hp.dense_words.empty()) {
        ctx->pp.dense = ctx->p_dense.upload(ctx->hp.dense_words, ctx->stream);
        ctx->pp.ldm = ctx->hp.ldm;
        const std::vector<uint8_t> gm = group_major_bytes(ctx->hp, &ctx->pp.gm_ld);
        ctx->pp.dense_gm = ctx->p_dense_gm.upload(gm, ctx->stream);
        ck(cudaStreamSynchronize(ctx->stream), "dense upload");
      }
      ctx->prod_ready = true;
      ctx->tc_ready = false;
    } catch (const CudaError& e) {
      return fail(SP_ERR_CUDA, e.what());
    }
  }
  if (dense && !ctx->pp.dense) return fail(SP_ERR_NOT_LOADED, "dense M_sym words not built");
  try {
    return launched(ctx, run_product(ctx, ctx->pp, d_S, ldS, n_shots, d_out, ld), "product launch");
  } catch (const CudaError& e) {
    return fail(SP_ERR_CUDA, e.what());
  }
}

uint64_t sp_encoded_size(uint64_t n_meas, uint64_t n_shots, sp_format fmt) {
  return fmt == SP_FMT_01 ? n_shots * (n_meas + 1) : n_shots * ((n_meas + 7) / 8);
}

int sp_encode(sp_ctx* ctx, const uint64_t* d_m, uint64_t ld, uint64_t n_meas, uint64_t n_shots,
              sp_format fmt, uint8_t* d_bytes) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (fmt != SP_FMT_01 && fmt != SP_FMT_B8) return fail(SP_ERR_INVALID_ARGUMENT, "unknown format");
  if (int r = set_device(ctx)) return r;
  if (n_meas && n_shots && ld < (n_shots + 63) / 64) return fail(SP_ERR_INVALID_ARGUMENT, "ld too small");
  int r = launch_encode(ctx->L, d_m, ld, n_meas, n_shots, fmt, d_bytes);
  return launched(ctx, r, "encode launch");
}

int sp_sample_to_host(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
                      sp_format fmt, uint8_t* h_out, uint64_t cap, uint64_t* written) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (n_shots == 0) return fail(SP_ERR_INVALID_ARGUMENT, "need at least one shot");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  const uint64_t n_meas = ctx->hp.n_meas;
  const uint64_t need = sp_encoded_size(n_meas, n_shots, fmt);
  if (cap < need || (!h_out && need)) return fail(SP_ERR_INVALID_ARGUMENT, "host buffer too small");
  const uint64_t T = 1ull << ctx->dp.t_log2;
  if (shot_begin % T) return fail(SP_ERR_INVALID_ARGUMENT, "shot_begin must be a multiple of the shot tile");
  // Chunks of ~32 MB of encoded records (a multiple of the shot tile), two
  // buffers deep: chunk i+1 is sampled and encoded on the compute stream
  // while chunk i is copied to the host on the copy stream.
  const uint64_t per_shot = std::max<uint64_t>(sp_encoded_size(n_meas, 1, fmt), 1);
  uint64_t chunk = std::max<uint64_t>((32ull << 20) / per_shot / T, 1) * T;
  chunk = std::min(chunk, (n_shots + T - 1) / T * T);
  const uint64_t ld = chunk / 64;
  try {
    if (!ctx->copy_stream) {
      ck(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
      for (int b = 0; b < 2; ++b) {
        ck(cudaEventCreateWithFlags(&ctx->ev_ready[b], cudaEventDisableTiming), "cudaEventCreate");
        ck(cudaEventCreateWithFlags(&ctx->ev_free[b], cudaEventDisableTiming), "cudaEventCreate");
      }
    }
    uint64_t* d_m[2];
    uint8_t* d_b[2];
    for (int b = 0; b < 2; ++b) {
      d_m[b] = static_cast<uint64_t*>(ctx->s_out[b].ensure(std::max<uint64_t>(n_meas * ld * 8, 16)));
      d_b[b] = static_cast<uint8_t*>(ctx->s_bytes[b].ensure(std::max<uint64_t>(chunk * per_shot, 16)));
    }
    uint64_t off = 0;
    uint64_t i = 0;
    for (uint64_t done = 0; done < n_shots; done += chunk, ++i) {
      const int b = static_cast<int>(i & 1);
      const uint64_t n = std::min(chunk, n_shots - done);
      if (i >= 2) ck(cudaStreamWaitEvent(ctx->stream, ctx->ev_free[b], 0), "cudaStreamWaitEvent");
      int r = SP_OK;
      if (ctx->rng == SP_RNG_PHILOX && n_meas && ctx->fused_ok && !ctx->unfused && !ctx->k5_ok) {
        // tiled records: coalesced stores for any row count
        if ((r = sp_sample_tiled(ctx, seed, shot_begin + done, n, d_m[b], nullptr))) return r;
        if ((r = sp_encode_tiled(ctx, d_m[b], n, fmt, d_b[b]))) return r;
      } else {
        if (n_meas && (r = sp_sample(ctx, seed, shot_begin + done, n, d_m[b], ld, nullptr))) return r;
        if ((r = sp_encode(ctx, d_m[b], ld, n_meas, n, fmt, d_b[b]))) return r;
      }
      const uint64_t nb = sp_encoded_size(n_meas, n, fmt);
      ck(cudaEventRecord(ctx->ev_ready[b], ctx->stream), "cudaEventRecord");
      ck(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev_ready[b], 0), "cudaStreamWaitEvent");
      if (nb) ck(cudaMemcpyAsync(h_out + off, d_b[b], nb, cudaMemcpyDeviceToHost, ctx->copy_stream), "D2H");
      ck(cudaEventRecord(ctx->ev_free[b], ctx->copy_stream), "cudaEventRecord");
      off += nb;
    }
    // the compute stream must not run ahead of the copies into host memory
    ck(cudaStreamWaitEvent(ctx->stream, ctx->ev_free[(i - 1) & 1], 0), "cudaStreamWaitEvent");
    ck(cudaStreamSynchronize(ctx->copy_stream), "sync");
    ck(cudaStreamSynchronize(ctx->stream), "sync");
    if (written) *written = off;
  } catch (const CudaError& e) {
    return fail(SP_ERR_CUDA, e.what());
  }
  return SP_OK;
}

uint64_t sp_launch_count(const sp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int sp_synchronize(sp_ctx* ctx) {
  if (!ctx) return fail(SP_ERR_INVALID_ARGUMENT, "null ctx");
  if (int r = set_device(ctx)) return r;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return fail(SP_ERR_CUDA, std::string("sync: ") + cudaGetErrorString(e));
  return SP_OK;
}

// Launch shape and table sizes of the fused sampler's plan (for reports):
// {T, gen_warps, cta_threads, staged, row_staged, lp, pad_pred, n_paths,
//  n_rounds, n_keep, n_seg_live, n_cls_live, n_dense_live, nnz(D), smem bytes,
//  sampler (for tiled launches): 0 draw + product, 1 K1, 2 K5, 3 K7, 4 K7 for launches counting
//  detectors and K1 for the others, 5 the reverse (gen_warps / cta_threads are K7's walkers / threads when it serves the
//  launches of the registered mode)}
int sp_plan_info(sp_ctx* ctx, uint64_t* out16) {
  if (!ctx || !out16) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  const DevPlan& d = ctx->dp;
  // K7 serves tiled launches: 3 = all of them, 4 = only those counting
  // detectors (sp_sample_ex), 5 = only the others; 1 = K1 serves all
  // (sp_sampler_kernel answers for any launch kind)
  const bool fz = ctx->fused_ok && !ctx->k5_ok && d.queued_ok;
  const bool k7p = fz && d.q_sel[2], k7d = fz && d.q_sel[3];
  const bool k7 = d.n_det ? k7d : k7p;
  const uint32_t k7w = d.q_fixed_shape ? d.q_walk : d.q_shape[d.n_det ? 3 : 2];
  const uint64_t sampler = ctx->k5_ok ? 2u : !ctx->fused_ok ? 0u : k7p && k7d ? 3u : k7d ? 4u : k7p ? 5u : 1u;
  const uint64_t v[16] = {1ull << d.t_log2, k7 ? k7w : d.gen_warps, k7 ? d.q_threads : d.cta_threads, d.staged, d.row_staged,
                          d.lp, d.pad_pred, d.n_paths, d.n_rounds, d.n_keep, d.n_seg_live,
                          d.n_cls_live, d.n_dense_live, ctx->dnnz,
                          fused_smem_bytes(d, d.t_log2, d.staged, d.row_staged, d.n_buf),
                          sampler};
  std::memcpy(out16, v, sizeof(v));
  return SP_OK;
}

// Which sampler serves one kind of sp_sample / sp_sample_tiled / sp_sample_ex
// launch: 0 draw + product, 1 K1, 2 K5, 3 K7.
int sp_sampler_kernel(sp_ctx* ctx, int tiled, int with_detector_counts, uint32_t* out) {
  if (!ctx || !out) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = set_device(ctx)) return r;
  if (int r = ensure_plan(ctx)) return r;
  const DevPlan& d = ctx->dp;
  const uint32_t kind = (tiled ? 2u : 0u) | (with_detector_counts ? 1u : 0u);
  *out = ctx->k5_ok ? 2u : !ctx->fused_ok || ctx->unfused ? 0u : d.queued_ok && d.q_sel[kind] ? 3u : 1u;
  return SP_OK;
}

// Test/profiling hook: copies (and clears) the fused kernel's per-role cycle
// counters when the plan was built with SP_PHASE_TIMERS=1: out[0..3] cycles
// (generators waiting / working, drains waiting / working), out[4] walk steps,
// out[5] firings, out[6..7] reserved.
int sp_debug_timers(sp_ctx* ctx, long long* out4) {  // 8 values
  if (!ctx || !out4) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (!ctx->dp.timers) return fail(SP_ERR_NOT_LOADED, "timers not enabled (SP_PHASE_TIMERS=1)");
  if (cudaMemcpy(out4, ctx->dp.timers, 64, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemset(ctx->dp.timers, 0, 64) != cudaSuccess)
    return fail(SP_ERR_CUDA, "timer copy failed");
  return SP_OK;
}

int sp_debug_philox(sp_ctx* ctx, const uint32_t* ctr_key, uint32_t* out) {
  if (!ctx || !ctr_key || !out) return fail(SP_ERR_INVALID_ARGUMENT, "null argument");
  if (int r = set_device(ctx)) return r;
  try {
    DBuf in, o;
    uint32_t* din = static_cast<uint32_t*>(in.ensure(6 * 4));
    uint32_t* dout = static_cast<uint32_t*>(o.ensure(4 * 4));
    ck(cudaMemcpy(din, ctr_key, 6 * 4, cudaMemcpyHostToDevice), "H2D");
    int r = launch_debug_philox(ctx->L, din, dout);
    if (int e = launched(ctx, r, "philox launch")) return e;
    ck(cudaMemcpy(out, dout, 4 * 4, cudaMemcpyDeviceToHost), "D2H");
  } catch (const CudaError& e) {
    return fail(SP_ERR_CUDA, e.what());
  }
  return SP_OK;
}

}  // extern "C"
