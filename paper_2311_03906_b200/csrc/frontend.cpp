// Host front end — see frontend.hpp for scope. Accepts the language of the
// reference's parse_circuit (circuit.cpp:79-168) with its own table-driven
// scanner and validator; independent implementations of summarize
// (circuit.cpp:188-226), decompose_noise (circuit.cpp:228-281) and the
// one-pass symbolic tableau (tableau.cpp:17-198, 318-382).
#include "frontend.hpp"
#include "frontend_dev.hpp"

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <optional>

namespace symphase {

namespace {

// Instruction vocabulary: spelling (upper case) -> opcode and the shape
// rules the parser checks (a probability argument for noise channels,
// target pairs for two-qubit instructions, no targets for TICK).
struct OpSpec {
  const char* name;
  Op op;
  bool noise, pairs;
};
constexpr OpSpec kOps[] = {
    {"H", Op::H, false, false},         {"S", Op::S, false, false},
    {"S_DAG", Op::SDag, false, false},  {"X", Op::X, false, false},
    {"Y", Op::Y, false, false},         {"Z", Op::Z, false, false},
    {"CX", Op::CX, false, true},        {"CNOT", Op::CX, false, true},
    {"M", Op::M, false, false},         {"MZ", Op::M, false, false},
    {"R", Op::R, false, false},         {"X_ERROR", Op::XErr, true, false},
    {"Y_ERROR", Op::YErr, true, false}, {"Z_ERROR", Op::ZErr, true, false},
    {"DEPOLARIZE1", Op::Dep1, true, false}, {"DEPOLARIZE2", Op::Dep2, true, true},
    {"TICK", Op::Tick, false, false}};
// Stim-format instructions the flat circuit model does not cover.
constexpr const char* kUnsupported[] = {"REPEAT", "DETECTOR", "OBSERVABLE_INCLUDE",
                                        "QUBIT_COORDS", "SHIFT_COORDS"};

const OpSpec* find_op(std::string_view name) {
  std::string up(name);
  std::transform(up.begin(), up.end(), up.begin(),
                 [](unsigned char c) { return static_cast<char>(std::toupper(c)); });
  for (const OpSpec& o : kOps)
    if (up == o.name) return &o;
  return nullptr;
}

// The characters operator>> skips on a C-locale stream.
constexpr bool blank(char c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// Splits circuit text into lines of whitespace-separated words, with '#'
// comments removed; calls emit(line number, words) for each non-empty line.
template <class Emit>
void scan_lines(std::string_view text, Emit&& emit) {
  std::vector<std::string_view> words;
  size_t number = 1, i = 0;
  bool in_comment = false;
  const size_t n = text.size();
  while (i <= n) {
    if (i == n || text[i] == '\n') {  // end of a line
      if (!words.empty()) emit(number, words);
      words.clear();
      in_comment = false;
      ++number;
      ++i;
      continue;
    }
    if (in_comment || blank(text[i])) {
      ++i;
      continue;
    }
    if (text[i] == '#') {
      in_comment = true;
      ++i;
      continue;
    }
    const size_t b = i;
    while (i < n && !blank(text[i]) && text[i] != '#') ++i;
    words.push_back(text.substr(b, i - b));
  }
}

template <class T>
bool parse_number(std::string_view w, T& out) {
  const auto r = std::from_chars(w.data(), w.data() + w.size(), out);
  return r.ec == std::errc{} && r.ptr == w.data() + w.size();
}

// One instruction from its words: NAME[(p)] target target ...
Instr make_instr(size_t line, const std::vector<std::string_view>& words) {
  std::string_view head = words.front();
  std::optional<double> arg;
  if (const size_t lp = head.find('('); lp != std::string_view::npos) {
    if (head.back() != ')') throw ParseError(line, "malformed parameter");
    const std::string_view inner = head.substr(lp + 1, head.size() - lp - 2);
    double v = 0;
    if (!parse_number(inner, v)) throw ParseError(line, "bad probability '" + std::string(inner) + "'");
    arg = v;
    head = head.substr(0, lp);
  }
  const OpSpec* spec = find_op(head);
  if (!spec) {
    for (const char* u : kUnsupported)
      if (head == u)
        throw ParseError(line, "unsupported instruction '" + std::string(head) +
                                   "' (flat gate/noise/measure circuits only)");
    throw ParseError(line, "unknown instruction '" + std::string(head) + "'");
  }
  Instr in;
  in.op = spec->op;
  in.line = line;
  in.targets.reserve(words.size() - 1);
  for (size_t k = 1; k < words.size(); ++k) {
    uint32_t q = 0;
    if (!parse_number(words[k], q)) throw ParseError(line, "bad target '" + std::string(words[k]) + "'");
    in.targets.push_back(q);
  }
  // shape rules
  if (spec->noise && !arg) throw ParseError(line, "noise instruction needs a probability");
  if (!spec->noise && arg) throw ParseError(line, "unexpected parameter on non-noise instruction");
  if (arg) {
    if (*arg < 0.0 || *arg > 1.0) throw ParseError(line, "probability out of [0,1]");
    in.p = *arg;
  }
  const bool tick = spec->op == Op::Tick;
  if (tick && !in.targets.empty()) throw ParseError(line, "TICK takes no targets");
  if (!tick && in.targets.empty()) throw ParseError(line, "missing targets");
  if (spec->pairs) {
    if (in.targets.size() & 1)
      throw ParseError(line, "odd number of targets for a two-qubit instruction");
    for (size_t k = 0; k + 1 < in.targets.size(); k += 2)
      if (in.targets[k] == in.targets[k + 1]) throw ParseError(line, "pair targets the same qubit twice");
  }
  return in;
}

}  // namespace

// Accepts the reference's circuit language (circuit.cpp:79-168): the same
// instruction set, the same rejections and line numbers, its own scanner.
std::vector<Instr> parse_circuit(std::string_view text) {
  std::vector<Instr> prog;
  scan_lines(text, [&](size_t line, const std::vector<std::string_view>& words) {
    prog.push_back(make_instr(line, words));
  });
  return prog;
}

namespace {

// The pass's inner loops, compiled for AVX-512 and AVX2 as well as the
// baseline (picked at load time by the CPU): the word XOR of phase rows and
// the x/z part of a rowsum (i-exponent of the product, then the XOR).
#define SP_CLONES __attribute__((target_clones("avx512f", "avx2", "default")))
SP_CLONES void xor_words(uint64_t* __restrict__ d, const uint64_t* __restrict__ s, size_t n) {
  for (size_t k = 0; k < n; ++k) d[k] ^= s[k];
}
// i-exponent of (x1,z1) * (x2,z2) (single_qubit_phase_exponent, pauli.cpp:7-12,
// summed over qubits) mod 4; then (x2,z2) ^= (x1,z1) when xor_in.
SP_CLONES int product_exponent(const uint64_t* __restrict__ x1, const uint64_t* __restrict__ z1,
                               uint64_t* __restrict__ x2, uint64_t* __restrict__ z2, size_t n,
                               bool xor_in) {
  int64_t plus = 0, minus = 0;
  for (size_t k = 0; k < n; ++k) {
    const uint64_t a = x1[k], b = z1[k], c = x2[k], d = z2[k];
    const uint64_t p = (a & ~b & ~c & d) | (a & b & c & ~d) | (~a & b & c & d);
    const uint64_t q = (a & ~b & c & d) | (a & b & ~c & d) | (~a & b & c & ~d);
    plus += __builtin_popcountll(p);
    minus += __builtin_popcountll(q);
    if (xor_in) {
      x2[k] = c ^ a;
      z2[k] = d ^ b;
    }
  }
  return static_cast<int>((((plus - minus) % 4) + 4) % 4);
}

// Stabilizer tableau with symbolic phases on the stabilizer half only.
// Rows [0, n) destabilizers, [n, 2n) stabilizers; x/z row-major packed.
class SymTableau {
 public:
  // dev: keep the phase matrix in device memory (frontend_dev.cu); row XORs
  // of measurements run as kernels, single-bit flips are queued.
  // may_move: start on the host and move the phase matrix to the device
  // once the row XORs are heavy (see note_op).
  SymTableau(size_t n, size_t capacity, bool dev, bool may_move = false)
      : may_move_(may_move && !dev), n_(n), wq_((n + 63) / 64), ws_((capacity + 63) / 64),
        rw_((2 * n + 63) / 64), xc_(n * ((2 * n + 63) / 64), 0), zc_(n * ((2 * n + 63) / 64), 0),
        x_(2 * n * wq_, 0), z_(2 * n * wq_, 0), ph_(dev ? 0 : n * ws_, 0), hi_(n, 0) {
    for (size_t i = 0; i < n; ++i) {
      x_[i * wq_ + i / 64] |= bit(i);              // destabilizer X_i
      z_[(n + i) * wq_ + i / 64] |= bit(i);        // stabilizer Z_i
    }
    if (dev) dev_ = phase_dev_create(n, ws_);
  }
  ~SymTableau() { phase_dev_destroy(dev_); }
  SymTableau(const SymTableau&) = delete;
  SymTableau& operator=(const SymTableau&) = delete;

  // Gates and symbol-conditioned Paulis work on a qubit-major copy of x/z
  // (column q = one bit per row, 2n bits): every update is O(n/64) words,
  // and the phase flips go to the rows of a bit mask. Measurements use the
  // row-major form; the two are converted (64 x 64 block transposes) when
  // the instruction kind switches.
  // H, S, S_DAG, CX: tableau.cpp:38-78 (phase term into the constant symbol).
  void h(uint32_t a) {
    to_cols();
    uint64_t* xa = &xc_[a * rw_]; uint64_t* za = &zc_[a * rw_];
    flip_rows(0, [&](size_t w) { return xa[w] & za[w]; });
    for (size_t w = 0; w < rw_; ++w) std::swap(xa[w], za[w]);
  }
  void s(uint32_t a) {
    to_cols();
    uint64_t* xa = &xc_[a * rw_]; uint64_t* za = &zc_[a * rw_];
    flip_rows(0, [&](size_t w) { return xa[w] & za[w]; });
    for (size_t w = 0; w < rw_; ++w) za[w] ^= xa[w];
  }
  void s_dag(uint32_t a) {
    to_cols();
    uint64_t* xa = &xc_[a * rw_]; uint64_t* za = &zc_[a * rw_];
    flip_rows(0, [&](size_t w) { return xa[w] & ~za[w]; });
    for (size_t w = 0; w < rw_; ++w) za[w] ^= xa[w];
  }
  void cx(uint32_t a, uint32_t b) {
    to_cols();
    uint64_t* xa = &xc_[a * rw_]; uint64_t* za = &zc_[a * rw_];
    uint64_t* xb = &xc_[b * rw_]; uint64_t* zb = &zc_[b * rw_];
    flip_rows(0, [&](size_t w) { return xa[w] & zb[w] & ~(xb[w] ^ za[w]); });
    for (size_t w = 0; w < rw_; ++w) { xb[w] ^= xa[w]; za[w] ^= zb[w]; }
  }

  // One gate instruction while the row-major form is current: applied in
  // place instead of converting to the qubit-major form (a conversion is
  // 2 x rw x wq 64 x 64 transposes; in the paper's Fig. 3 families every
  // layer would otherwise convert twice: gates, then measurements).
  // H/S/S_DAG on distinct qubits: one sweep over the rows with a qubit mask
  // (the gates act on different qubits, so each row's constant-phase flips
  // add up: their parity is flipped in). CX on distinct qubits: per pair
  // over the rows, when that is cheaper than the conversion.
  // Returns false when the instruction should go the qubit-major way.
  bool layer_in_rows(Op op, const std::vector<uint32_t>& q) {
    if (cols_ || q.empty()) return false;
    // Work in the row-major form since the last conversion stays below one
    // conversion's (ops: ~1,500 per 64 x 64 block, ~8 per swept row word,
    // ~12 per row per CX), so a run of small instructions cannot cost more
    // than converting would have.
    const double conv = 2.0 * rw_ * wq_ * 1500.0;
    const double cost = op == Op::CX ? static_cast<double>(q.size() / 2) * 2.0 * n_ * 12.0
                                     : 2.0 * n_ * wq_ * 8.0;
    if (row_work_ + cost > conv) return false;
    row_work_ += cost;
    mask_.assign(wq_, 0);
    for (uint32_t a : q) {
      if (mask_[a / 64] & bit(a)) return false;  // a repeated qubit: apply gate by gate
      mask_[a / 64] |= bit(a);
    }
    const uint64_t* mk = mask_.data();
    if (op == Op::CX) {
      for (size_t i = 0; i + 1 < q.size(); i += 2) {
        const uint32_t a = q[i], b = q[i + 1];
        const size_t wa = a / 64, wb = b / 64;
        const uint64_t ma = bit(a), mb = bit(b);
        for (size_t r = 0; r < 2 * n_; ++r) {
          uint64_t* x = &x_[r * wq_]; uint64_t* z = &z_[r * wq_];
          const bool xa = x[wa] & ma, za = z[wa] & ma, xb = x[wb] & mb, zb = z[wb] & mb;
          if (r >= n_ && xa && zb && !(xb ^ za)) flip_phase(r - n_, 0);
          if (xa) x[wb] ^= mb;
          if (zb) z[wa] ^= ma;
        }
      }
      return true;
    }
    for (size_t r = 0; r < 2 * n_; ++r) {
      uint64_t* x = &x_[r * wq_]; uint64_t* z = &z_[r * wq_];
      int par = 0;
      for (size_t k = 0; k < wq_; ++k) {
        const uint64_t xv = x[k], zv = z[k], m = mk[k];
        if (op == Op::H) {
          par += __builtin_popcountll(xv & zv & m);
          x[k] = (xv & ~m) | (zv & m);
          z[k] = (zv & ~m) | (xv & m);
        } else {
          par += __builtin_popcountll((op == Op::S ? xv & zv : xv & ~zv) & m);
          z[k] = zv ^ (xv & m);
        }
      }
      if (r >= n_ && (par & 1)) flip_phase(r - n_, 0);
    }
    return true;
  }

  // Symbol-conditioned Paulis (tableau.cpp:80-100): XOR symbol s into the
  // phase of every stabilizer row the Pauli anticommutes with.
  // Works in whichever layout is current (a reset's conditional X follows
  // its measurement, so no conversion).
  void pauli(uint32_t a, bool px, bool pz, uint32_t sym) {
    if (!cols_) {
      const size_t w = a / 64; const uint64_t m = bit(a);
      for (size_t i = 0; i < n_; ++i) {
        size_t r = n_ + i;
        bool xa = x_[r * wq_ + w] & m, za = z_[r * wq_ + w] & m;
        if ((px && za) ^ (pz && xa)) flip_phase(i, sym);
      }
      return;
    }
    const uint64_t* xa = &xc_[a * rw_]; const uint64_t* za = &zc_[a * rw_];
    const uint64_t mx = px ? ~0ull : 0ull, mz = pz ? ~0ull : 0ull;
    flip_rows(sym, [&](size_t w) { return (mx & za[w]) ^ (mz & xa[w]); });
  }

  // A reset's X conditioned on every symbol of its measurement's outcome
  // (tableau.cpp:355-362 applies one conditional X per symbol): the rows it
  // anticommutes with are the same for all symbols, so find them once and
  // flip the whole expression into each (same XORs, reordered).
  void pauli_x_all(uint32_t a, const std::vector<uint32_t>& syms) {
    if (syms.empty()) return;
    if (syms.size() == 1) return pauli(a, true, false, syms[0]);
    rows_.clear();
    if (!cols_) {
      const size_t w = a / 64; const uint64_t m = bit(a);
      for (size_t i = 0; i < n_; ++i)
        if (z_[(n_ + i) * wq_ + w] & m) rows_.push_back(static_cast<uint32_t>(i));
    } else {
      const uint64_t* za = &zc_[a * rw_];
      for_rows([&](size_t w) { return za[w]; }, [&](size_t i) { rows_.push_back(static_cast<uint32_t>(i)); });
    }
    const uint32_t top = *std::max_element(syms.begin(), syms.end()) / 64 + 1;
    for (uint32_t i : rows_) {
      if (dev_) {
        for (uint32_t s : syms) flips_.push_back(static_cast<uint64_t>(i) << 32 | s);
      } else {
        uint64_t* p = &ph_[i * ws_];
        for (uint32_t s : syms) p[s / 64] ^= bit(s);
      }
      hi_[i] = std::max(hi_[i], top);
    }
  }

  // Z-basis measurement (tableau.cpp:146-198). Returns sorted symbol ids.
  std::vector<uint32_t> measure(uint32_t a, uint64_t& n_sym, std::vector<Group>& groups) {
    to_rows();
    if (may_move_ && heavy_ >= kHeavyOps) move_to_device();
    const size_t w = a / 64; const uint64_t m = bit(a);
    size_t pivot = 2 * n_;
    for (size_t r = n_; r < 2 * n_; ++r)
      if (x_[r * wq_ + w] & m) { pivot = r; break; }

    if (pivot < 2 * n_) {
      targets_.clear();
      size_t n_stab = 0;
      for (size_t r = 0; r < 2 * n_; ++r) {
        if (r == pivot || r + n_ == pivot) continue;
        if (x_[r * wq_ + w] & m) {
          rowsum(r, pivot);
          n_stab += r >= n_;
        }
      }
      if (!dev_) note_op(n_stab * hi_[pivot - n_]);
      if (dev_ && !targets_.empty()) {  // the phase XORs rowsum deferred, in one launch
        flush_flips();
        phase_dev_xor_rows(dev_, static_cast<uint32_t>(pivot - n_), targets_.data(), targets_.size(),
                           hi_[pivot - n_]);
      }
      std::memcpy(&x_[(pivot - n_) * wq_], &x_[pivot * wq_], wq_ * 8);
      std::memcpy(&z_[(pivot - n_) * wq_], &z_[pivot * wq_], wq_ * 8);
      std::memset(&x_[pivot * wq_], 0, wq_ * 8);
      std::memset(&z_[pivot * wq_], 0, wq_ * 8);
      z_[pivot * wq_ + w] |= m;
      size_t i = pivot - n_;
      if (dev_) {
        flush_flips();
        phase_dev_clear_row(dev_, static_cast<uint32_t>(i), hi_[i]);
      } else {
        std::memset(&ph_[i * ws_], 0, hi_[i] * 8);
      }
      hi_[i] = 0;
      uint32_t sym = static_cast<uint32_t>(n_sym++);  // add_measurement_symbol, symbols.hpp:73-81
      groups.push_back(Group{kCoin, 0.5, sym, 1});
      if (sym / 64 >= ws_) throw std::logic_error("symbol capacity exhausted (pre-pass undercount)");
      flip_phase(i, sym);
      return {sym};
    }

    // Determined: product of the stabilizers selected by destabilizers that
    // anticommute with Z_a is +/-Z_a; its symbolic phase is the outcome.
    std::vector<uint64_t> sx(wq_, 0), sz(wq_, 0);
    std::vector<uint64_t> sp(dev_ ? 0 : ws_, 0);
    size_t shi = 0;
    uint64_t const_flip = 0;
    targets_.clear();
    for (size_t i = 0; i < n_; ++i) {
      if (!(x_[i * wq_ + w] & m)) continue;
      const uint64_t* x1 = &x_[(n_ + i) * wq_];
      const uint64_t* z1 = &z_[(n_ + i) * wq_];
      int res = product_exponent(x1, z1, sx.data(), sz.data(), wq_, true);
      if (res & 1) throw std::logic_error("non-hermitian generator product: tableau corrupt");
      if (dev_) {
        targets_.push_back(static_cast<uint32_t>(i));
      } else {
        const uint64_t* p1 = &ph_[i * ws_];
        xor_words(sp.data(), p1, hi_[i]);
      }
      shi = std::max<size_t>(shi, hi_[i]);
      if (res == 2) const_flip ^= 1;
    }
    const uint64_t* spp = sp.data();
    if (!dev_) {
      size_t words = 0;
      for (size_t i = 0; i < n_; ++i)
        if (x_[i * wq_ + w] & m) words += hi_[i];
      note_op(words);
    }
    if (dev_) {
      flush_flips();
      spp = phase_dev_reduce(dev_, targets_.data(), targets_.size(),
                             static_cast<uint32_t>(std::max<size_t>(shi, 1)));
    }
    bool ok = true;
    for (size_t k = 0; k < wq_; ++k) {
      if (sx[k] != 0) ok = false;
      if (sz[k] != (k == w ? m : 0)) ok = false;
    }
    if (!ok) throw std::logic_error("determined measurement did not reduce to Z_a");
    std::vector<uint32_t> e;
    for (size_t k = 0; k < std::max<size_t>(shi, 1); ++k) {
      uint64_t v = spp[k] ^ (k == 0 ? const_flip : 0);
      while (v) {
        e.push_back(static_cast<uint32_t>(k * 64 + __builtin_ctzll(v)));
        v &= v - 1;
      }
    }
    return e;
  }

 private:
  static uint64_t bit(size_t i) { return uint64_t{1} << (i & 63); }

  // flip_phase(row - n, sym) for every stabilizer row whose bit is set in
  // the column-form mask fn(word).
  template <class F>
  void flip_rows(uint32_t sym, F&& fn) {
    for_rows(fn, [&](size_t i) { flip_phase(i, sym); });
  }
  // visit(row - n) for every stabilizer row whose bit is set in fn(word)
  template <class F, class V>
  void for_rows(F&& fn, V&& visit) {
    for (size_t w = n_ / 64; w < rw_; ++w) {
      uint64_t v = fn(w);
      const size_t r0 = w * 64;
      if (r0 < n_) v &= ~0ull << (n_ - r0);  // destabilizer rows carry no phase
      if (r0 + 64 > 2 * n_) v &= (2 * n_ - r0 >= 64) ? ~0ull : ((1ull << (2 * n_ - r0)) - 1);
      while (v) {
        const size_t r = r0 + static_cast<size_t>(__builtin_ctzll(v));
        v &= v - 1;
        visit(r - n_);
      }
    }
  }

  // 64 x 64 bit transpose in place: bit j of word i <-> bit i of word j.
  static void transpose64(uint64_t* a) {
    uint64_t m = 0x00000000FFFFFFFFull;
    for (int j = 32; j != 0; j >>= 1, m ^= m << j) {
      for (int k = 0; k < 64; k = ((k | j) + 1) & ~j) {
        const uint64_t t = ((a[k] >> j) ^ a[k | j]) & m;
        a[k] ^= t << j;
        a[k | j] ^= t;
      }
    }
  }
  // Row-major x_/z_ [2n][wq_] <-> qubit-major xc_/zc_ [n][rw_].
  void to_cols() {
    if (cols_) return;
    convert(true);
    cols_ = true;
  }
  void to_rows() {
    if (!cols_) return;
    convert(false);
    cols_ = false;
    row_work_ = 0;
  }
  void convert(bool to_c) {
    uint64_t blk[64];
    for (int pass = 0; pass < 2; ++pass) {
      std::vector<uint64_t>& rm = pass ? z_ : x_;
      std::vector<uint64_t>& cm = pass ? zc_ : xc_;
      for (size_t R = 0; R < rw_; ++R) {      // 64-row block
        for (size_t Q = 0; Q < wq_; ++Q) {    // 64-qubit block
          if (to_c) {
            for (size_t i = 0; i < 64; ++i) {
              const size_t r = R * 64 + i;
              blk[i] = r < 2 * n_ ? rm[r * wq_ + Q] : 0;
            }
            transpose64(blk);
            for (size_t j = 0; j < 64 && Q * 64 + j < n_; ++j) cm[(Q * 64 + j) * rw_ + R] = blk[j];
          } else {
            for (size_t j = 0; j < 64; ++j) {
              const size_t q = Q * 64 + j;
              blk[j] = q < n_ ? cm[q * rw_ + R] : 0;
            }
            transpose64(blk);
            for (size_t i = 0; i < 64 && R * 64 + i < 2 * n_; ++i) rm[(R * 64 + i) * wq_ + Q] = blk[i];
          }
        }
      }
    }
  }

  // Host or device phase matrix: a device row operation costs a launch (and,
  // for a determined outcome, a round trip: ~15-50 us), a host one about
  // 0.25 ns per 64-bit word XORed. Start on the host (small circuits, surface
  // codes: few rows per operation) and move the matrix to the device after
  // kHeavyOps consecutive measurements each XORing more than kHeavyWords
  // (wide random circuits: hundreds of rows x thousands of words).
  static constexpr size_t kHeavyWords = size_t{1} << 17;
  static constexpr int kHeavyOps = 4;
  void note_op(size_t words) { heavy_ = words > kHeavyWords ? heavy_ + 1 : 0; }
  void move_to_device() {
    may_move_ = false;
    try {
      dev_ = phase_dev_create(n_, ws_);
      phase_dev_upload(dev_, ph_.data());
    } catch (const std::runtime_error&) {  // no device memory: stay on the host
      phase_dev_destroy(dev_);
      dev_ = nullptr;
      return;
    }
    std::vector<uint64_t>().swap(ph_);
  }

  void flip_phase(size_t i, uint32_t sym) {
    if (dev_) {
      flips_.push_back(static_cast<uint64_t>(i) << 32 | sym);
    } else {
      ph_[i * ws_ + sym / 64] ^= bit(sym);
    }
    hi_[i] = std::max<uint32_t>(hi_[i], sym / 64 + 1);
  }
  // queued single-bit flips, applied before the next device row operation
  void flush_flips() {
    if (!flips_.empty()) phase_dev_flips(dev_, flips_.data(), flips_.size());
    flips_.clear();
  }

  // dst := src * dst (rowsum_rows, tableau.cpp:113-144). Destabilizer phases
  // are not tracked (they never reach an outcome), so only stabilizer targets
  // pay for the phase.
  void rowsum(size_t dst, size_t src) {
    uint64_t* xd = &x_[dst * wq_]; uint64_t* zd = &z_[dst * wq_];
    const uint64_t* xs = &x_[src * wq_]; const uint64_t* zs = &z_[src * wq_];
    if (dst < n_) {
      for (size_t k = 0; k < wq_; ++k) { xd[k] ^= xs[k]; zd[k] ^= zs[k]; }
      return;
    }
    {
      int res = product_exponent(xs, zs, xd, zd, wq_, true);
      if (res & 1) throw std::logic_error("non-hermitian generator product: tableau corrupt");
      size_t di = dst - n_, si = src - n_;
      if (dev_) {
        targets_.push_back(static_cast<uint32_t>(di));  // XORed by the caller in one launch
      } else {
        uint64_t* pd = &ph_[di * ws_]; const uint64_t* ps = &ph_[si * ws_];
        xor_words(pd, ps, hi_[si]);
      }
      hi_[di] = std::max(hi_[di], hi_[si]);
      if (res == 2) flip_phase(di, 0);
    }
  }

  bool may_move_ = false;
  int heavy_ = 0;          // consecutive heavy host row operations
  size_t n_, wq_, ws_;
  size_t rw_ = 0;          // words per qubit column (2n rows)
  bool cols_ = false;      // the qubit-major copy is current (row-major stale)
  std::vector<uint64_t> xc_, zc_;
  std::vector<uint64_t> x_, z_, ph_;
  std::vector<uint32_t> hi_;
  PhaseDev* dev_ = nullptr;
  std::vector<uint64_t> flips_;    // queued (row << 32 | symbol) flips (dev_)
  std::vector<uint32_t> targets_;  // rows of the current device row operation
  std::vector<uint32_t> rows_;     // scratch (pauli_x_all)
  std::vector<uint64_t> mask_;     // scratch (layer_in_rows)
  double row_work_ = 0;            // layer_in_rows work since the last to_rows
};

}  // namespace

Model run_initialization(const std::vector<Instr>& prog) {
  Model M;
  M.groups.push_back(Group{});  // group 0: the constant symbol (symbols.hpp:49-52)
  // summarize (circuit.cpp:188-226): qubit count and symbol capacity.
  size_t n = 0, cap = 1;
  for (const auto& in : prog) {
    for (uint32_t t : in.targets) n = std::max<size_t>(n, size_t{t} + 1);
    switch (in.op) {
      case Op::M: case Op::R: cap += in.targets.size(); break;
      case Op::XErr: case Op::YErr: case Op::ZErr: cap += in.targets.size(); break;
      case Op::Dep1: cap += 2 * in.targets.size(); break;
      case Op::Dep2: cap += 2 * in.targets.size(); break;
      default: break;
    }
  }
  M.n_qubits = n;
  if (n == 0) return M;

  // Phase matrix: on the host, moved to the device when its row operations
  // turn heavy (SymTableau::note_op), or from the start when it is very large
  // (n x capacity bits >= 2^30, 128 MB) — if a GPU is present.
  // SP_FRONTEND_DEV=0 keeps it on the host, =1 puts it on the device.
  const char* env = std::getenv("SP_FRONTEND_DEV");
  const double bits = static_cast<double>(n) * static_cast<double>(cap);
  bool dev = env ? std::atoi(env) != 0 : bits >= static_cast<double>(1ull << 30);
  // (a smaller matrix never has a row operation heavy enough to move)
  const bool gpu = (dev || bits >= static_cast<double>(1ull << 24)) && phase_dev_available();
  if (dev && !gpu) dev = false;
  const bool may_move = !env && gpu;
  std::unique_ptr<SymTableau> tp;
  try {
    tp = std::make_unique<SymTableau>(n, cap, dev, may_move);
  } catch (const std::runtime_error&) {  // no device memory for the phase matrix
    if (!dev) throw;
    tp = std::make_unique<SymTableau>(n, cap, false);
  }
  SymTableau& t = *tp;
  uint64_t& n_sym = M.n_sym;
  auto add_fault = [&](uint8_t dist, double p, uint32_t arity) {
    uint32_t first = static_cast<uint32_t>(n_sym);
    M.groups.push_back(Group{dist, p, first, arity});
    n_sym += arity;
    return first;
  };
  auto push_row = [&](const std::vector<uint32_t>& e) {
    M.sym_idx.insert(M.sym_idx.end(), e.begin(), e.end());
    M.row_ptr.push_back(M.sym_idx.size());
  };
  for (const auto& in : prog) {
    const auto& q = in.targets;
    switch (in.op) {
      case Op::H: if (!t.layer_in_rows(in.op, q)) for (uint32_t a : q) t.h(a); break;
      case Op::S: if (!t.layer_in_rows(in.op, q)) for (uint32_t a : q) t.s(a); break;
      case Op::SDag: if (!t.layer_in_rows(in.op, q)) for (uint32_t a : q) t.s_dag(a); break;
      case Op::X: for (uint32_t a : q) t.pauli(a, true, false, 0); break;
      case Op::Y: for (uint32_t a : q) t.pauli(a, true, true, 0); break;
      case Op::Z: for (uint32_t a : q) t.pauli(a, false, true, 0); break;
      case Op::CX:
        if (!t.layer_in_rows(in.op, q))
          for (size_t i = 0; i + 1 < q.size(); i += 2) t.cx(q[i], q[i + 1]);
        break;
      case Op::M: for (uint32_t a : q) push_row(t.measure(a, n_sym, M.groups)); break;
      case Op::R:
        // Reset = measure + X conditioned on the outcome (tableau.cpp:355-362).
        for (uint32_t a : q) {
          t.pauli_x_all(a, t.measure(a, n_sym, M.groups));
        }
        break;
      // decompose_noise (circuit.cpp:228-281): one group per channel target.
      case Op::XErr: for (uint32_t a : q) t.pauli(a, true, false, add_fault(kBernoulli, in.p, 1)); break;
      case Op::ZErr: for (uint32_t a : q) t.pauli(a, false, true, add_fault(kBernoulli, in.p, 1)); break;
      case Op::YErr: for (uint32_t a : q) t.pauli(a, true, true, add_fault(kBernoulli, in.p, 1)); break;
      case Op::Dep1:
        for (uint32_t a : q) {
          uint32_t s = add_fault(kDep1, in.p, 2);
          t.pauli(a, true, false, s);
          t.pauli(a, false, true, s + 1);
        }
        break;
      case Op::Dep2:
        for (size_t i = 0; i + 1 < q.size(); i += 2) {
          uint32_t s = add_fault(kDep2, in.p, 4);
          t.pauli(q[i], true, false, s);
          t.pauli(q[i], false, true, s + 1);
          t.pauli(q[i + 1], true, false, s + 2);
          t.pauli(q[i + 1], false, true, s + 3);
        }
        break;
      case Op::Tick: break;
    }
  }
  return M;
}

}  // namespace symphase
