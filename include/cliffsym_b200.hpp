// cliffsym_b200.hpp — header-only C++ shim that re-exposes the reference's
// sampler API (cliffsym, proj/core/include/cliffsym/{sampler,symbols,
// circuit,tableau}.hpp) on top of the C ABI in symphase_b200.h.
//
// A maintainer switches a cliffsym caller over by including this header and
// using namespace cliffsym_b200 instead of cliffsym.
// Semantics kept from the reference:
//   * draw_assignments(registry, n, seed) is bit-identical to the reference
//     (device keyed_draw/fill_group, sampler.hpp:14-28, sampler.cpp:11-59);
//   * sample(expressions, batch) / gf2_multiply_sparse are exact GF(2)
//     products (sampler.cpp:61-112, bit_matrix.cpp:314-328);
//   * encode_shots produces the same '01' / 'b8' bytes (sampler.cpp:118-140);
//   * errors are the same exception types: std::invalid_argument (n_smp == 0),
//     std::out_of_range (symbol id >= batch rows), ParseError, std::logic_error.
// Bit matrices here are plain row-major u64 words (rows x ceil(cols/64)),
// not 512x512 tiles; get_bit/set_bit/same_bits behave like TiledBitMatrix's.
// sample_shots() is the fused B200 path (draw + product in one kernel).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include <cuda_runtime.h>

#include "symphase_b200.h"

namespace cliffsym_b200 {

// circuit.hpp:42-47: "line N: ..." plus the line number.
struct ParseError : std::runtime_error {
  explicit ParseError(const std::string& what)
      : std::runtime_error(what), line(std::strtoull(what.c_str() + (what.rfind("line ", 0) == 0 ? 5 : what.size()), nullptr, 10)) {}
  ParseError(size_t l, const std::string& what)
      : std::runtime_error("line " + std::to_string(l) + ": " + what), line(l) {}
  size_t line;
};

inline void throw_status(int code) {
  if (code == SP_OK) return;
  std::string msg = sp_last_error();
  switch (code) {
    case SP_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SP_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case SP_ERR_PARSE: throw ParseError(msg);
    case SP_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

// BitVec (bitvec.hpp:14-112) subset: packed LSB-first bits.
class BitVec {
 public:
  BitVec() = default;
  explicit BitVec(size_t n) : n_(n), w_((n + 63) / 64, 0) {}
  size_t size() const { return n_; }
  bool get(size_t i) const {
    if (i >= n_) throw std::out_of_range("BitVec index");
    return (w_[i >> 6] >> (i & 63)) & 1;
  }
  void set(size_t i, bool v) {
    if (i >= n_) throw std::out_of_range("BitVec index");
    uint64_t m = uint64_t{1} << (i & 63);
    w_[i >> 6] = v ? (w_[i >> 6] | m) : (w_[i >> 6] & ~m);
  }
  uint8_t get_byte(size_t b) const {
    size_t wi = b >> 3;
    return wi < w_.size() ? static_cast<uint8_t>(w_[wi] >> ((b & 7) * 8)) : 0;
  }
  std::span<const uint64_t> words() const { return w_; }
  bool operator==(const BitVec&) const = default;

 private:
  size_t n_ = 0;
  std::vector<uint64_t> w_;
};

// TiledBitMatrix (bit_matrix.hpp:67-125) behaviour over bit-sliced rows
// (TiledBitMatrix below is an alias, so reference code compiles unchanged).
class BitMatrix {
 public:
  BitMatrix() = default;
  BitMatrix(size_t rows, size_t cols)
      : rows_(rows), cols_(cols), ld_(std::max<size_t>((cols + 63) / 64, 1)), w_(rows * ld_, 0) {}
  size_t rows() const { return rows_; }
  size_t cols() const { return cols_; }
  size_t ld() const { return ld_; }
  bool get_bit(size_t r, size_t c) const {
    check(r, c);
    return (w_[r * ld_ + c / 64] >> (c % 64)) & 1;
  }
  void set_bit(size_t r, size_t c, bool v) {
    check(r, c);
    uint64_t m = uint64_t{1} << (c % 64);
    uint64_t& x = w_[r * ld_ + c / 64];
    x = v ? (x | m) : (x & ~m);
  }
  void flip_bit(size_t r, size_t c) {
    check(r, c);
    w_[r * ld_ + c / 64] ^= uint64_t{1} << (c % 64);
  }
  bool same_bits(const BitMatrix& o) const {
    return rows_ == o.rows_ && cols_ == o.cols_ && w_ == o.w_;
  }
  BitVec column_bits(size_t c) const {
    BitVec out(rows_);
    for (size_t r = 0; r < rows_; ++r)
      if (get_bit(r, c)) out.set(r, true);
    return out;
  }
  std::string to_text() const {
    std::string s;
    for (size_t r = 0; r < rows_; ++r) {
      for (size_t c = 0; c < cols_; ++c) s.push_back(get_bit(r, c) ? '1' : '0');
      s.push_back('\n');
    }
    return s;
  }
  uint64_t* data() { return w_.data(); }
  const uint64_t* data() const { return w_.data(); }
  size_t bytes() const { return w_.size() * 8; }

 private:
  void check(size_t r, size_t c) const {
    if (r >= rows_ || c >= cols_) throw std::out_of_range("BitMatrix index");
  }
  size_t rows_ = 0, cols_ = 0, ld_ = 1;
  std::vector<uint64_t> w_;
};

using TiledBitMatrix = BitMatrix;

// symbols.hpp:19-100
enum class GroupDistribution : uint8_t {
  kConstantOne = SP_DIST_CONSTANT,
  kBernoulli = SP_DIST_BERNOULLI,
  kFairCoin = SP_DIST_COIN,
  kDepolarize1 = SP_DIST_DEPOLARIZE1,
  kDepolarize2 = SP_DIST_DEPOLARIZE2,
};

struct SymbolGroup {
  GroupDistribution distribution = GroupDistribution::kConstantOne;
  double param = 0.0;
  uint32_t first_symbol = 0;
  uint32_t arity = 1;
};

class SymbolRegistry {
 public:
  SymbolRegistry() { groups_.push_back(SymbolGroup{}); }
  size_t size() const { return size_; }
  size_t group_count() const { return groups_.size(); }
  const SymbolGroup& group(uint32_t gid) const { return groups_.at(gid); }
  std::span<const SymbolGroup> groups() const { return groups_; }
  uint32_t add_fault_group(GroupDistribution dist, double param, uint32_t arity, size_t = 0) {
    uint32_t first = static_cast<uint32_t>(size_);
    groups_.push_back(SymbolGroup{dist, param, first, arity});
    size_ += arity;
    return first;
  }
  uint32_t add_measurement_symbol(size_t = 0) {
    uint32_t id = static_cast<uint32_t>(size_);
    groups_.push_back(SymbolGroup{GroupDistribution::kFairCoin, 0.5, id, 1});
    size_ += 1;
    return id;
  }
  std::vector<sp_group> to_abi() const {
    std::vector<sp_group> g(groups_.size());
    for (size_t i = 0; i < g.size(); ++i) {
      g[i] = sp_group{};
      g[i].dist = static_cast<uint8_t>(groups_[i].distribution);
      g[i].param = groups_[i].param;
      g[i].first_symbol = groups_[i].first_symbol;
      g[i].arity = groups_[i].arity;
    }
    return g;
  }

 private:
  size_t size_ = 1;
  std::vector<SymbolGroup> groups_;
};

struct MeasurementExpression {
  std::vector<uint32_t> symbols;  // strictly increasing
  bool evaluate(const BitVec& assignment) const {
    bool v = false;
    for (uint32_t s : symbols) v ^= assignment.get(s);
    return v;
  }
  bool operator==(const MeasurementExpression&) const = default;
};

// circuit.hpp:13-40 (same kind order as the C ABI's program arrays).
enum class InstrKind : uint8_t {
  kH, kS, kSDag, kX, kY, kZ, kCX, kM, kR, kXError, kYError, kZError, kDepolarize1, kDepolarize2, kTick
};

struct Instruction {
  InstrKind kind = InstrKind::kTick;
  std::vector<uint32_t> targets;
  double param = 0.0;  // probability, noise kinds only
  size_t line = 0;     // 1-based source line, 0 when synthesized
};

struct CircuitSummary {  // circuit.hpp:67-79 (the fields the sampler path reads)
  size_t n_qubits = 0;
  size_t n_measurements = 0;
};

struct InitResult {
  size_t n_qubits = 0;
  CircuitSummary summary;
  SymbolRegistry registry;
  std::vector<MeasurementExpression> expressions;
};

// parse_circuit (circuit.hpp:55) through the library's parser.
inline std::vector<Instruction> parse_circuit(std::string_view text) {
  std::string t(text);
  uint64_t n = 0, nt = 0;
  throw_status(sp_parse_circuit(t.c_str(), 0, nullptr, nullptr, nullptr, nullptr, 0, nullptr, &n, &nt));
  std::vector<uint8_t> kinds(n + 1);
  std::vector<double> params(n + 1);
  std::vector<uint64_t> lines(n + 1), ptr(n + 1);
  std::vector<uint32_t> tg(nt + 1);
  throw_status(sp_parse_circuit(t.c_str(), n, kinds.data(), params.data(), lines.data(), ptr.data(),
                                nt, tg.data(), &n, &nt));
  std::vector<Instruction> prog(n);
  for (uint64_t i = 0; i < n; ++i) {
    prog[i].kind = static_cast<InstrKind>(kinds[i]);
    prog[i].param = params[i];
    prog[i].line = lines[i];
    prog[i].targets.assign(tg.begin() + ptr[i], tg.begin() + ptr[i + 1]);
  }
  return prog;
}

namespace detail {
inline InitResult init_from_model(sp_model* m) {
  std::unique_ptr<sp_model, void (*)(sp_model*)> guard(m, sp_model_destroy);
  uint64_t nq, nm, ns, ng, nnz;
  throw_status(sp_model_dims(m, &nq, &nm, &ns, &ng, &nnz));
  std::vector<uint64_t> rp(nm + 1);
  std::vector<uint32_t> si(std::max<uint64_t>(nnz, 1));
  std::vector<sp_group> g(ng);
  throw_status(sp_model_export(m, rp.data(), si.data(), g.data()));
  InitResult r;
  r.n_qubits = nq;
  r.summary.n_qubits = nq;
  r.summary.n_measurements = nm;
  for (uint64_t i = 1; i < ng; ++i) {
    auto d = static_cast<GroupDistribution>(g[i].dist);
    if (d == GroupDistribution::kFairCoin)
      r.registry.add_measurement_symbol();
    else
      r.registry.add_fault_group(d, g[i].param, g[i].arity);
  }
  r.expressions.resize(nm);
  for (uint64_t k = 0; k < nm; ++k) r.expressions[k].symbols.assign(si.begin() + rp[k], si.begin() + rp[k + 1]);
  return r;
}
}  // namespace detail

// run_initialization (tableau.hpp:101) on a parsed or synthesized program.
inline InitResult run_initialization(const std::vector<Instruction>& prog) {
  std::vector<uint8_t> kinds(prog.size() + 1);
  std::vector<double> params(prog.size() + 1);
  std::vector<uint64_t> ptr{0};
  std::vector<uint32_t> tg;
  for (size_t i = 0; i < prog.size(); ++i) {
    kinds[i] = static_cast<uint8_t>(prog[i].kind);
    params[i] = prog[i].param;
    tg.insert(tg.end(), prog[i].targets.begin(), prog[i].targets.end());
    ptr.push_back(tg.size());
  }
  if (tg.empty()) tg.push_back(0);
  sp_model* m = nullptr;
  throw_status(sp_model_from_program(prog.size(), kinds.data(), params.data(), ptr.data(), tg.data(), &m));
  return detail::init_from_model(m);
}

// parse_circuit + run_initialization in one call.
inline InitResult run_initialization_text(std::string_view text) {
  std::string t(text);
  sp_model* m = nullptr;
  throw_status(sp_model_from_text(t.c_str(), &m));
  return detail::init_from_model(m);
}

// sampler.hpp:30-46
struct SymbolAssignmentBatch {
  BitMatrix data;  // (n_s + 1) x n_smp
  size_t n_symbols() const { return data.rows(); }
  size_t n_shots() const { return data.cols(); }
};

struct SampleMatrix {
  BitMatrix data;  // n_m x n_smp
  std::vector<uint32_t> measurement_order;
  size_t n_measurements() const { return data.rows(); }
  size_t n_shots() const { return data.cols(); }
};

enum class ShotFormat : uint8_t { k01 = SP_FMT_01, kB8 = SP_FMT_B8 };

namespace detail {

// Grow-only device buffer, reused across calls (no cudaMalloc per call).
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  void* ensure(size_t bytes) {
    bytes = std::max<size_t>(bytes, 16);
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      cuda_check(cudaMalloc(&p, bytes));
      n = bytes;
    }
    return p;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

// Device contexts per host thread (the ABI's threading rule), one per role,
// so one call never replaces the model another role's context holds (a
// draw_assignments between two sample_shots calls keeps the loaded model).
enum Role { kDraw = 0, kProduct = 1, kFused = 2, kEncode = 3, kRoles = 4 };
struct Slot {
  sp_ctx* c = nullptr;
  DevBuf a, b;
};
inline Slot& slot(Role r) {
  struct Holder {
    Slot s[kRoles];
    Holder() {
      for (Slot& x : s) throw_status(sp_ctx_create(0, &x.c));
    }
    ~Holder() {
      for (Slot& x : s) sp_ctx_destroy(x.c);
    }
  };
  thread_local Holder h;
  return h.s[r];
}
inline sp_ctx* ctx(Role r = kProduct) { return slot(r).c; }

inline void load_rows(sp_ctx* c, std::span<const std::vector<uint32_t>> rows, uint64_t n_sym) {
  std::vector<uint64_t> rp{0};
  std::vector<uint32_t> si;
  for (const auto& r : rows) {
    si.insert(si.end(), r.begin(), r.end());
    rp.push_back(si.size());
  }
  if (si.empty()) si.push_back(0);
  throw_status(sp_load_msym_csr(c, rows.size(), n_sym, rp.data(), si.data()));
}

inline std::vector<std::vector<uint32_t>> rows_of(const std::vector<MeasurementExpression>& e) {
  std::vector<std::vector<uint32_t>> r(e.size());
  for (size_t i = 0; i < e.size(); ++i) r[i] = e[i].symbols;
  return r;
}

inline void sorted_unique_check(const std::vector<std::vector<uint32_t>>& rows) {
  for (const auto& r : rows)
    for (size_t i = 1; i < r.size(); ++i)
      if (r[i] <= r[i - 1]) throw std::invalid_argument("expression symbols must be strictly increasing");
}

}  // namespace detail

// draw_assignments (sampler.hpp:51-52): bit-identical to the reference.
inline SymbolAssignmentBatch draw_assignments(const SymbolRegistry& registry, size_t n_smp,
                                              uint64_t seed) {
  if (n_smp == 0) throw std::invalid_argument("need at least one shot");
  detail::Slot& sl = detail::slot(detail::kDraw);
  sp_ctx* c = sl.c;
  std::vector<std::vector<uint32_t>> none;
  detail::load_rows(c, none, registry.size());
  auto g = registry.to_abi();
  throw_status(sp_load_groups(c, g.size(), g.data()));
  throw_status(sp_set_rng(c, SP_RNG_COMPAT_SPLITMIX));
  SymbolAssignmentBatch b{BitMatrix(registry.size(), n_smp)};
  void* d = sl.a.ensure(b.data.bytes());
  throw_status(sp_draw_assignments(c, seed, 0, n_smp, static_cast<uint64_t*>(d), b.data.ld()));
  cuda_check(cudaMemcpy(b.data.data(), d, b.data.bytes(), cudaMemcpyDeviceToHost));
  return b;
}

// gf2_multiply_sparse (bit_matrix.hpp:133-134).
inline BitMatrix gf2_multiply_sparse(std::span<const std::vector<uint32_t>> a_rows,
                                     const BitMatrix& b) {
  detail::Slot& sl = detail::slot(detail::kProduct);
  sp_ctx* c = sl.c;
  std::vector<std::vector<uint32_t>> rows(a_rows.begin(), a_rows.end());
  for (auto& r : rows) std::sort(r.begin(), r.end());
  detail::sorted_unique_check(rows);
  throw_status(sp_set_product(c, SP_PRODUCT_AUTO));
  detail::load_rows(c, rows, b.rows());
  BitMatrix out(rows.size(), b.cols());
  if (rows.empty() || b.cols() == 0) {
    for (const auto& r : rows)
      for (uint32_t s : r)
        if (s >= b.rows()) throw std::out_of_range("sparse row index");
    return out;
  }
  void* dS = sl.a.ensure(b.bytes());
  void* dO = sl.b.ensure(out.bytes());
  cuda_check(cudaMemcpy(dS, b.data(), b.bytes(), cudaMemcpyHostToDevice));
  throw_status(sp_sample_given_S(c, static_cast<const uint64_t*>(dS), b.rows(), b.ld(), b.cols(),
                                 static_cast<uint64_t*>(dO), out.ld()));
  cuda_check(cudaMemcpy(out.data(), dO, out.bytes(), cudaMemcpyDeviceToHost));
  return out;
}

// gf2_multiply (bit_matrix.hpp:129): dense a [m x k] times b [k x n] — the
// device's dense explicit-S product (Four-Russians tables).
inline BitMatrix gf2_multiply(const BitMatrix& a, const BitMatrix& b) {
  if (a.cols() != b.rows()) throw std::invalid_argument("gf2_multiply: inner dimensions differ");
  BitMatrix out(a.rows(), b.cols());
  if (a.rows() == 0 || b.cols() == 0) return out;
  detail::Slot& sl = detail::slot(detail::kProduct);
  sp_ctx* c = sl.c;
  throw_status(sp_load_msym_dense(c, a.rows(), std::max<size_t>(a.cols(), 1), a.data(), a.ld()));
  throw_status(sp_set_product(c, SP_PRODUCT_DENSE));
  void* dS = sl.a.ensure(b.bytes());
  void* dO = sl.b.ensure(out.bytes());
  cuda_check(cudaMemcpy(dS, b.data(), b.bytes(), cudaMemcpyHostToDevice));
  throw_status(sp_sample_given_S(c, static_cast<const uint64_t*>(dS), std::max<size_t>(b.rows(), 1),
                                 b.ld(), b.cols(), static_cast<uint64_t*>(dO), out.ld()));
  cuda_check(cudaMemcpy(out.data(), dO, out.bytes(), cudaMemcpyDeviceToHost));
  return out;
}

// sample(expressions, batch, threads) (sampler.hpp:57-58). `threads` only
// changed scheduling in the reference; the device path ignores it.
inline SampleMatrix sample(const std::vector<MeasurementExpression>& expressions,
                           const SymbolAssignmentBatch& batch, unsigned threads = 1) {
  (void)threads;
  for (const auto& e : expressions)
    for (uint32_t s : e.symbols)
      if (s >= batch.n_symbols()) throw std::out_of_range("symbol id out of range");
  auto rows = detail::rows_of(expressions);
  SampleMatrix m;
  m.data = gf2_multiply_sparse(rows, batch.data);
  m.measurement_order.resize(expressions.size());
  for (size_t i = 0; i < expressions.size(); ++i) m.measurement_order[i] = static_cast<uint32_t>(i);
  return m;
}

// The fused B200 path: draw + product in one kernel (Philox streams by
// default; SP_RNG_COMPAT_SPLITMIX reproduces draw_assignments + sample).
inline SampleMatrix sample_shots(const InitResult& init, size_t n_smp, uint64_t seed,
                                 sp_rng rng = SP_RNG_PHILOX) {
  if (n_smp == 0) throw std::invalid_argument("need at least one shot");
  detail::Slot& sl = detail::slot(detail::kFused);
  sp_ctx* c = sl.c;
  auto rows = detail::rows_of(init.expressions);
  detail::load_rows(c, rows, init.registry.size());
  auto g = init.registry.to_abi();
  throw_status(sp_load_groups(c, g.size(), g.data()));
  throw_status(sp_set_rng(c, rng));
  SampleMatrix m;
  m.data = BitMatrix(init.expressions.size(), n_smp);
  m.measurement_order.resize(init.expressions.size());
  for (size_t i = 0; i < m.measurement_order.size(); ++i) m.measurement_order[i] = static_cast<uint32_t>(i);
  if (init.expressions.empty()) return m;
  void* d = sl.a.ensure(m.data.bytes());
  throw_status(sp_sample(c, seed, 0, n_smp, static_cast<uint64_t*>(d), m.data.ld(), nullptr));
  cuda_check(cudaMemcpy(m.data.data(), d, m.data.bytes(), cudaMemcpyDeviceToHost));
  return m;
}

// encode_shots (sampler.hpp:65).
inline std::string encode_shots(const SampleMatrix& m, ShotFormat format) {
  const uint64_t n_m = m.n_measurements(), n = m.n_shots();
  const uint64_t size = sp_encoded_size(n_m, n, static_cast<sp_format>(format));
  std::string out(size, '\0');
  if (size == 0) return out;
  detail::Slot& sl = detail::slot(detail::kEncode);
  void* dm = sl.a.ensure(m.data.bytes());
  void* db = sl.b.ensure(size);
  cuda_check(cudaMemcpy(dm, m.data.data(), m.data.bytes(), cudaMemcpyHostToDevice));
  throw_status(sp_encode(sl.c, static_cast<const uint64_t*>(dm), m.data.ld(), n_m, n,
                         static_cast<sp_format>(format), static_cast<uint8_t*>(db)));
  cuda_check(cudaMemcpy(out.data(), db, size, cudaMemcpyDeviceToHost));
  return out;
}

// shot_bits (sampler.hpp:68).
inline BitVec shot_bits(const SampleMatrix& m, size_t shot) { return m.data.column_bits(shot); }

}  // namespace cliffsym_b200
