// Host-side stages of the sampling planner (abi.cpp build_plan) that need no
// device: the chain transform M = L·D, the drain plan (heavy paths of the
// parent forest + detector classification) and the mechanism rates of the
// exact DEPOLARIZE decomposition. Unit-tested on the CPU by
// tests/cpp/test_plan_stages.cpp (tests/test_plan_cpu.py).
#pragma once

#include <cstdint>
#include <vector>

namespace symphase::plan {

// M_sym = L·D "chain" transform. Row k gets at most one parent p(k) < k —
// the earlier row sharing the most symbols with it — whenever
// |row_k XOR row_p| < |row_k|; D row k is that symmetric difference (else
// row k itself). Then out[k] = (D·S)[k] ^ out[p(k)] exactly over GF(2). For
// repeated syndrome extraction this turns cumulative measurement rows into
// detector-like round differences, so fault columns of D are several times
// shorter than those of M (fewer bit flips per firing).
struct ChainXf {
  std::vector<int32_t> parent;
  std::vector<uint64_t> rp;   // D rows, CSR over measurements
  std::vector<uint32_t> si;
  std::vector<uint32_t> depth;
  uint32_t n_levels = 1;
};
ChainXf chain_transform(uint64_t n_meas, const std::vector<uint64_t>& row_ptr,
                        const std::vector<uint32_t>& sym_idx, const std::vector<uint64_t>& col_ptr,
                        const std::vector<uint32_t>& col_rows, bool enable);

// How the fused kernel's drain rebuilds rows (out[k] = d[k] ^ out[p(k)]) and
// counts detectors. Paths of a heavy-path decomposition of the parent
// forest, in rounds (a path's head has its parent on a path of an earlier
// round); path_rows entries = row | (row detector index + 1) << 16 | keep
// << 31, padded by 4 entries for the walk's prefetch. keep: the row's final
// value stays in the tile until the tile ends (a light child or a general
// detector reads it). A detector equal to {k, p(k)} (or {k} for a root row)
// is a row detector of row k; the others are general (their rows XORed).
struct DrainPlan {
  std::vector<uint32_t> path_rows, path_ptr{0}, round_ptr;
  std::vector<int32_t> path_par;
  std::vector<uint16_t> keep_rows;
  uint32_t n_paths = 0, n_rounds = 1;
  bool flat = false;  // no parents and nothing kept: a flat pass in row order
  uint32_t n_det = 0;
  std::vector<uint32_t> gdet_ptr{0}, gdet_id;
  std::vector<uint16_t> gdet_rows;
};
DrainPlan plan_drain(const std::vector<int32_t>& parent, const std::vector<uint64_t>& det_ptr,
                     const std::vector<uint32_t>& det_meas);

// Rate q of each independent Pauli mechanism in the exact decomposition of
// DEPOLARIZE1(p) (3 mechanisms) / DEPOLARIZE2(p) (15 mechanisms): the XOR of
// the fired patterns is uniform over the non-identity patterns with total
// rate p. Returns -1 when the channel is not decomposable (other
// distributions, p >= 3/4 resp. 15/16) or q would not be in (0, 1/2).
double mechanism_rate(uint8_t dist, double p);

}  // namespace symphase::plan
