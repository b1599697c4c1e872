// Device-side plan and kernel launchers for the sampling hot path (sm_100a).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace symphase {

// Random-stream domains (top byte of Philox counter word 3).
constexpr uint32_t kDomChain = 1u;  // geometric-skip event chains
constexpr uint32_t kDomCoin = 2u;   // bit-sliced fair-coin words

// Everything a kernel needs about the loaded model, all device pointers.
// Built once per sp_load_* by plan.cpp.
struct DevPlan {
  uint32_t n_meas = 0, n_sym = 0, n_groups = 0;
  uint32_t t_log2 = 0, tw = 0;  // shot tile T = 1 << t_log2; tw = T/32 u32 words

  // M_sym, CSR over measurements (expression lists) and CSR over symbols.
  const uint64_t* row_ptr = nullptr;
  const uint32_t* sym_idx = nullptr;
  const uint64_t* col_ptr = nullptr;   // [n_sym+1]
  const uint32_t* col_rows = nullptr;  // [nnz]
  // dense row-major M_sym words [n_meas][ldm] (only when loaded / built)
  const uint64_t* dense = nullptr;
  uint64_t ldm = 0;

  // Group table (symbols.hpp:36-42).
  const uint32_t* g_first = nullptr;
  const uint32_t* g_arity = nullptr;
  const uint8_t* g_dist = nullptr;
  const double* g_param = nullptr;

  // Constant rows: bit k set when measurement k XORs a constant 1
  // (s0, plus Bernoulli(p>=1) symbols in Philox mode).
  const uint32_t* row_const = nullptr;         // Philox mode
  const uint32_t* row_const_compat = nullptr;  // s0 only (compat mode)
  // Symbols whose assignment row is identically one in Philox mode (s0 and
  // Bernoulli(p>=1)); in compat mode only s0 (== ones_syms[0]).
  uint32_t n_ones = 0;
  const uint32_t* ones_syms = nullptr;

  // Dense (bit-sliced) symbols: fair coins and Bernoulli(1/2).
  uint32_t n_dense_live = 0, n_dense_all = 0;  // live slots come first
  const uint32_t* dense_sym = nullptr;         // slot -> symbol id
  const uint32_t* drow_ptr = nullptr;          // [n_meas+1] -> drow_slot
  const uint32_t* drow_slot = nullptr;

  // Sparse channels: classes of groups sharing (distribution, p), each
  // sampled as one Bernoulli process over its flattened (group, shot) trial
  // space of a tile, cut into chains of roughly equal expected event count.
  uint32_t n_chains_live = 0, n_chains_all = 0;  // live chains come first
  const uint32_t* ch_class = nullptr;
  const uint64_t* ch_lo = nullptr;
  const uint64_t* ch_hi = nullptr;
  const uint8_t* cls_dist = nullptr;
  const float* cls_inv = nullptr;   // 1 / -ln(1 - p)
  const uint64_t* cls_goff = nullptr;
  const uint32_t* cls_groups = nullptr;

  // Compat mode: group ids (>= 1) with at least one live symbol, and all.
  uint32_t n_live_groups = 0;
  const uint32_t* live_groups = nullptr;
};

struct LaunchCfg {
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
};

// Shared-memory bytes the fused kernel needs per CTA for tile width tw.
size_t fused_smem_bytes(uint32_t n_meas, uint32_t n_dense, uint32_t tw, bool counts);

// K1 fused sampler (Philox). Returns number of launches issued, <0 on error.
int launch_fused_sample(const DevPlan& P, const LaunchCfg& L, uint64_t seed, uint64_t tile0,
                        uint64_t n_shots, uint64_t* out, uint64_t ld, uint64_t* counts);
// K4 fused sampler, compat RNG (bit-exact keyed_draw / fill_group).
int launch_fused_sample_compat(const DevPlan& P, const LaunchCfg& L, uint64_t seed,
                               uint64_t tile0, uint64_t n_shots, uint64_t* out, uint64_t ld,
                               uint64_t* counts);
// draw_assignments on device (same streams as the fused kernels).
int launch_draw(const DevPlan& P, const LaunchCfg& L, bool compat, uint64_t seed, uint64_t tile0,
                uint64_t n_shots, uint64_t* S, uint64_t ldS);
// K2 explicit-S product: sparse (CSR rows) or dense (row-major words).
int launch_product(const DevPlan& P, const LaunchCfg& L, bool dense, const uint64_t* S,
                   uint64_t ldS, uint64_t n_shots, uint64_t* out, uint64_t ld);
// K3 encode (fmt 0 = '01', 1 = 'b8').
int launch_encode(const LaunchCfg& L, const uint64_t* m, uint64_t ld, uint64_t n_meas,
                  uint64_t n_shots, int fmt, uint8_t* bytes);
// Known-answer hook for the Philox4x32-10 implementation.
int launch_debug_philox(const LaunchCfg& L, const uint32_t* ctr_key_dev, uint32_t* out_dev);

}  // namespace symphase
