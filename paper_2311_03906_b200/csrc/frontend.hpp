// Host front end: circuit text -> one symbolic forward pass -> M_sym + channel table.
//
// This is the *producer* at the drop-in boundary: it turns the
// reference circuit format into exactly the reference's InitResult content —
// the measurement expressions (rows of M_sym) and the symbol-group registry —
// so the device sampler sees the same symbol numbering as the reference
// (symbols.hpp:47-86, circuit.cpp:228-281, tableau.cpp:318-382).
//
// It is an independent implementation, not a port: x/z bits live in row-major
// packed words, only stabilizer rows carry symbolic phases (destabilizer
// phases never reach an outcome), and phase XORs stop at the highest symbol
// allocated so far. Expressions are nevertheless identical to the reference's:
// each outcome is a unique affine-linear function of the symbols, so any
// correct elimination order yields the same sorted symbol list (pinned by
// tests/test_frontend_cpu.py against oracle/_ref on random circuits).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace symphase {

// InstrKind, circuit.hpp:13-29 (same order).
enum class Op : uint8_t { H, S, SDag, X, Y, Z, CX, M, R, XErr, YErr, ZErr, Dep1, Dep2, Tick };

struct Instr {
  Op op = Op::Tick;
  std::vector<uint32_t> targets;
  double p = 0.0;
  size_t line = 0;
};

// ParseError, circuit.hpp:42-47: message "line N: ...".
struct ParseError : std::runtime_error {
  ParseError(size_t line, const std::string& what)
      : std::runtime_error("line " + std::to_string(line) + ": " + what), line(line) {}
  size_t line;
};

// GroupDistribution numbering, symbols.hpp:19-25.
enum Dist : uint8_t { kConst = 0, kBernoulli = 1, kCoin = 2, kDep1 = 3, kDep2 = 4 };

struct Group {
  uint8_t dist = kConst;
  double param = 0.0;
  uint32_t first = 0;
  uint32_t arity = 1;
};

// The hot path's input contract (InitResult.expressions + registry).
struct Model {
  uint64_t n_qubits = 0;
  uint64_t n_sym = 1;                // registry.size(): s0 + faults + coins
  std::vector<Group> groups;         // group 0 = constant
  std::vector<uint64_t> row_ptr{0};  // CSR over measurements
  std::vector<uint32_t> sym_idx;     // strictly increasing per row
  uint64_t n_meas() const { return row_ptr.size() - 1; }
};

// parse_circuit semantics (circuit.cpp:79-168).
std::vector<Instr> parse_circuit(std::string_view text);

// run_initialization semantics (tableau.cpp:318-382). Throws std::logic_error
// on an internal invariant failure, like the reference.
Model run_initialization(const std::vector<Instr>& prog);

}  // namespace symphase
