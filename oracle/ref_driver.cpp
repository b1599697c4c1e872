// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" driver over the *unmodified* reference library (cliffsym
// core, compiled from /root/reference/proj/core/src by oracle/Makefile into
// oracle/_ref/). Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference leg may load it.
//
// Every entry point calls the reference's own public API:
//   parse_circuit            circuit.hpp:55
//   run_initialization       tableau.hpp:101 (tableau.cpp:318-382)
//   draw_assignments         sampler.hpp:51-52 (sampler.cpp:48-59)
//   sample                   sampler.hpp:57-58 (sampler.cpp:61-112)
//   encode_shots             sampler.hpp:65   (sampler.cpp:118-140)
//   gf2_multiply_sparse      bit_matrix.hpp:133-134
// Bit-sliced buffers use this repo's device layout: u64 words, row-major,
// bit j%64 of word j/64 of row r = element (r, j).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "cliffsym/bit_matrix.hpp"
#include "cliffsym/circuit.hpp"
#include "cliffsym/sampler.hpp"
#include "cliffsym/symbols.hpp"
#include "cliffsym/tableau.hpp"

using namespace cliffsym;

struct ref_ctx {
  InitResult init;
};

namespace {

void set_err(char* err, size_t errlen, const char* what) {
  if (err && errlen) {
    std::strncpy(err, what, errlen - 1);
    err[errlen - 1] = 0;
  }
}

TiledBitMatrix from_sliced(uint64_t rows, uint64_t cols, const uint64_t* w, uint64_t ld) {
  TiledBitMatrix m(rows, cols);
  for (uint64_t r = 0; r < rows; ++r) {
    const uint64_t* row = w + r * ld;
    for (uint64_t c0 = 0; c0 < cols; c0 += 64) {
      uint64_t x = row[c0 / 64];
      if (cols - c0 < 64) x &= (uint64_t{1} << (cols - c0)) - 1;
      while (x) {
        unsigned b = static_cast<unsigned>(__builtin_ctzll(x));
        x &= x - 1;
        m.set_bit(r, c0 + b, true);
      }
    }
  }
  return m;
}

void to_sliced(const TiledBitMatrix& m, uint64_t* w, uint64_t ld) {
  for (uint64_t r = 0; r < m.rows(); ++r) std::memset(w + r * ld, 0, ld * sizeof(uint64_t));
  // Column access is the cheap direction for column-major tiles.
  TiledBitMatrix c = m;
  c.ensure_order(TileOrder::kColumnMajor);
  for (uint64_t j = 0; j < c.cols(); ++j) {
    BitVec col = c.column_bits(j);
    for (uint64_t wi = 0; wi < col.words().size(); ++wi) {
      uint64_t x = col.word(wi);
      while (x) {
        unsigned b = static_cast<unsigned>(__builtin_ctzll(x));
        x &= x - 1;
        uint64_t r = wi * 64 + b;
        w[r * ld + j / 64] |= uint64_t{1} << (j % 64);
      }
    }
  }
}

}  // namespace

extern "C" {

// 0 ok; 1 parse / runtime error; 2 std::logic_error (cliffsym.cpp:346-355 mapping)
int ref_init(const char* text, ref_ctx** out, char* err, size_t errlen) {
  try {
    auto ctx = new ref_ctx;
    ctx->init = run_initialization(parse_circuit(text));
    *out = ctx;
    return 0;
  } catch (const ParseError& e) {
    set_err(err, errlen, e.what());
    return 1;
  } catch (const std::logic_error& e) {
    set_err(err, errlen, e.what());
    return 2;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 1;
  }
}

// An InitResult from explicit expressions + a group table (cfg5's random
// M_sym has no circuit): the reference's own SymbolRegistry and
// MeasurementExpression, so draw_assignments / sample run unchanged on it.
int ref_init_model(uint64_t n_meas, const uint64_t* row_ptr, const uint32_t* sym_idx,
                   uint64_t n_groups, const uint8_t* dist, const double* param,
                   const uint32_t* arity, ref_ctx** out) {
  try {
    auto ctx = new ref_ctx;
    for (uint64_t g = 1; g < n_groups; ++g) {
      const auto d = static_cast<GroupDistribution>(dist[g]);
      if (d == GroupDistribution::kFairCoin) ctx->init.registry.add_measurement_symbol(0);
      else ctx->init.registry.add_fault_group(d, param[g], arity[g], 0);
    }
    ctx->init.expressions.resize(n_meas);
    for (uint64_t k = 0; k < n_meas; ++k)
      ctx->init.expressions[k].symbols.assign(sym_idx + row_ptr[k], sym_idx + row_ptr[k + 1]);
    *out = ctx;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

void ref_free(ref_ctx* c) { delete c; }

void ref_dims(const ref_ctx* c, uint64_t* n_meas, uint64_t* n_sym, uint64_t* n_groups,
              uint64_t* nnz, uint64_t* n_qubits) {
  *n_meas = c->init.expressions.size();
  *n_sym = c->init.registry.size();
  *n_groups = c->init.registry.group_count();
  uint64_t z = 0;
  for (const auto& e : c->init.expressions) z += e.symbols.size();
  *nnz = z;
  *n_qubits = c->init.summary.n_qubits;
}

void ref_export_rows(const ref_ctx* c, uint64_t* row_ptr, uint32_t* sym_idx) {
  uint64_t p = 0;
  row_ptr[0] = 0;
  for (size_t k = 0; k < c->init.expressions.size(); ++k) {
    for (uint32_t s : c->init.expressions[k].symbols) sym_idx[p++] = s;
    row_ptr[k + 1] = p;
  }
}

void ref_export_groups(const ref_ctx* c, uint8_t* dist, double* param, uint32_t* first,
                       uint32_t* arity) {
  auto gs = c->init.registry.groups();
  for (size_t g = 0; g < gs.size(); ++g) {
    dist[g] = static_cast<uint8_t>(gs[g].distribution);
    param[g] = gs[g].param;
    first[g] = gs[g].first_symbol;
    arity[g] = gs[g].arity;
  }
}

// sample() on a supplied batch. 0 ok, -1 std::out_of_range, -2 other.
int ref_sample_given(uint64_t n_meas, const uint64_t* row_ptr, const uint32_t* sym_idx,
                     uint64_t n_sym, uint64_t n_shots, const uint64_t* S, uint64_t ldS,
                     uint64_t* out, uint64_t ld, unsigned threads) {
  try {
    std::vector<MeasurementExpression> exprs(n_meas);
    for (uint64_t k = 0; k < n_meas; ++k) {
      exprs[k].symbols.assign(sym_idx + row_ptr[k], sym_idx + row_ptr[k + 1]);
    }
    SymbolAssignmentBatch batch{from_sliced(n_sym, n_shots, S, ldS)};
    SampleMatrix m = sample(exprs, batch, threads);
    to_sliced(m.data, out, ld);
    return 0;
  } catch (const std::out_of_range&) {
    return -1;
  } catch (const std::exception&) {
    return -2;
  }
}

// gf2_multiply_sparse (bit_matrix.cpp:314-328) on a supplied batch.
int ref_gf2_multiply_sparse(uint64_t n_rows, const uint64_t* row_ptr, const uint32_t* idx,
                            uint64_t b_rows, uint64_t b_cols, const uint64_t* B,
                            uint64_t ldB, uint64_t* out, uint64_t ld) {
  try {
    std::vector<std::vector<uint32_t>> rows(n_rows);
    for (uint64_t k = 0; k < n_rows; ++k) rows[k].assign(idx + row_ptr[k], idx + row_ptr[k + 1]);
    TiledBitMatrix b = from_sliced(b_rows, b_cols, B, ldB);
    TiledBitMatrix r = gf2_multiply_sparse(rows, b);
    to_sliced(r, out, ld);
    return 0;
  } catch (const std::out_of_range&) {
    return -1;
  } catch (const std::exception&) {
    return -2;
  }
}

// draw_assignments(registry, n, seed) exported bit-sliced [n_sym][ldS].
int ref_draw(const ref_ctx* c, uint64_t n_shots, uint64_t seed, uint64_t* S, uint64_t ldS) {
  try {
    SymbolAssignmentBatch b = draw_assignments(c->init.registry, n_shots, seed);
    to_sliced(b.data, S, ldS);
    return 0;
  } catch (const std::invalid_argument&) {
    return -2;
  } catch (const std::exception&) {
    return -3;
  }
}

// The cmd_sample timed region (cliffsym.cpp:108-113): draw + sample + encode.
// fmt 0 = '01', 1 = 'b8'. Returns bytes written, or -needed if cap too small.
int64_t ref_sample_encode(const ref_ctx* c, uint64_t n_shots, uint64_t seed, int fmt,
                          unsigned threads, uint8_t* out, uint64_t cap) {
  try {
    SymbolAssignmentBatch b = draw_assignments(c->init.registry, n_shots, seed);
    SampleMatrix m = sample(c->init.expressions, b, threads);
    std::string s = encode_shots(m, fmt == 1 ? ShotFormat::kB8 : ShotFormat::k01);
    if (s.size() > cap) return -static_cast<int64_t>(s.size());
    std::memcpy(out, s.data(), s.size());
    return static_cast<int64_t>(s.size());
  } catch (const std::exception&) {
    return INT64_MIN;
  }
}

// encode_shots on a supplied measurement-major matrix [n_meas][ld].
int64_t ref_encode(uint64_t n_meas, uint64_t n_shots, const uint64_t* m, uint64_t ld, int fmt,
                   uint8_t* out, uint64_t cap) {
  SampleMatrix sm;
  sm.data = from_sliced(n_meas, n_shots, m, ld);
  sm.measurement_order.resize(n_meas);
  for (uint64_t i = 0; i < n_meas; ++i) sm.measurement_order[i] = static_cast<uint32_t>(i);
  std::string s = encode_shots(sm, fmt == 1 ? ShotFormat::kB8 : ShotFormat::k01);
  if (s.size() > cap) return -static_cast<int64_t>(s.size());
  std::memcpy(out, s.data(), s.size());
  return static_cast<int64_t>(s.size());
}

// CPU-baseline timing of the reference path on this host.
//   mode 0 ("as shipped", cmd_sample): one draw_assignments(n) + sample(threads)
//          + encode_shots(b8) call.
//   mode 1 ("API parallelised over shot chunks"): `threads` workers, each
//          running draw_assignments(chunk, seed + c) + sample(.., 1) +
//          encode_shots(b8) over its share of chunks.
// Returns wall seconds (steady_clock), or -1 on error.
double ref_time(const ref_ctx* c, uint64_t total_shots, uint64_t chunk, unsigned threads,
                uint64_t seed, int mode) {
  using Clock = std::chrono::steady_clock;
  try {
    auto t0 = Clock::now();
    if (mode == 0) {
      SymbolAssignmentBatch b = draw_assignments(c->init.registry, total_shots, seed);
      SampleMatrix m = sample(c->init.expressions, b, threads);
      std::string s = encode_shots(m, ShotFormat::kB8);
      if (s.empty() && total_shots) return -1;
    } else {
      uint64_t n_chunks = (total_shots + chunk - 1) / chunk;
      std::vector<std::thread> ws;
      for (unsigned w = 0; w < threads; ++w) {
        ws.emplace_back([&, w] {
          for (uint64_t ci = w; ci < n_chunks; ci += threads) {
            uint64_t n = std::min(chunk, total_shots - ci * chunk);
            SymbolAssignmentBatch b = draw_assignments(c->init.registry, n, seed + ci);
            SampleMatrix m = sample(c->init.expressions, b, 1);
            std::string s = encode_shots(m, ShotFormat::kB8);
            (void)s;
          }
        });
      }
      for (auto& t : ws) t.join();
    }
    return std::chrono::duration<double>(Clock::now() - t0).count();
  } catch (const std::exception&) {
    return -1.0;
  }
}

}  // extern "C"
