// The reference's sampler unit tests (proj/tests/test_sampler.cpp) re-hosted
// on the cliffsym_b200 C++ shim, i.e. run against the B200 library through
// include/cliffsym_b200.hpp. Case names and tolerances follow the reference
// file; each case cites its line range. Minimal harness: prints one line per
// failed check and exits non-zero on any failure.
#include <cmath>
#include <cstdio>
#include <random>

#include "cliffsym_b200.hpp"

using namespace cliffsym_b200;

static int g_fail = 0, g_checks = 0;
#define CHECK(x)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(x)) {                                                               \
      ++g_fail;                                                               \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);                \
    }                                                                         \
  } while (0)

static InitResult init_from(const char* text) { return run_initialization_text(text); }

static void check_within_4sigma(size_t hits, size_t shots, double p) {
  double sigma = std::sqrt(p * (1.0 - p) / static_cast<double>(shots));
  double phat = static_cast<double>(hits) / static_cast<double>(shots);
  CHECK(std::abs(phat - p) <= 4.0 * sigma + 1e-12);
}

int main() {
  {  // constant row is all ones (test_sampler.cpp:30-34)
    auto init = init_from("H 0\nM 0\n");
    auto batch = draw_assignments(init.registry, 300, 5);
    for (size_t j = 0; j < 300; ++j) CHECK(batch.data.get_bit(0, j));
  }
  {  // noiseless deterministic circuit (36-46)
    auto init = init_from("X 0\nM 0\nM 0\n");
    CHECK(init.registry.size() == 1);
    auto batch = draw_assignments(init.registry, 64, 1);
    CHECK(batch.n_symbols() == 1);
    auto m = sample(init.expressions, batch);
    for (size_t j = 0; j < 64; ++j) {
      CHECK(m.data.get_bit(0, j));
      CHECK(m.data.get_bit(1, j));
    }
  }
  {  // degenerate fault probabilities (48-60)
    auto init = init_from("X_ERROR(1) 0\nX_ERROR(0) 1\nM 0 1\n");
    auto batch = draw_assignments(init.registry, 500, 99);
    for (size_t j = 0; j < 500; ++j) {
      CHECK(batch.data.get_bit(1, j));
      CHECK(!batch.data.get_bit(2, j));
    }
    auto m = sample(init.expressions, batch);
    for (size_t j = 0; j < 500; ++j) {
      CHECK(m.data.get_bit(0, j));
      CHECK(!m.data.get_bit(1, j));
    }
    auto f = sample_shots(init, 500, 99);  // fused Philox path
    for (size_t j = 0; j < 500; ++j) {
      CHECK(f.data.get_bit(0, j));
      CHECK(!f.data.get_bit(1, j));
    }
  }
  {  // identical seeds reproduce the batch (62-69)
    auto init = init_from("DEPOLARIZE1(0.2) 0\nH 0\nM 0\nX_ERROR(0.4) 0\nM 0\n");
    auto a = draw_assignments(init.registry, 1000, 42);
    auto b = draw_assignments(init.registry, 1000, 42);
    CHECK(a.data.same_bits(b.data));
    auto c = draw_assignments(init.registry, 1000, 43);
    CHECK(!a.data.same_bits(c.data));
  }
  {  // sparse == dense == per-shot evaluation, threaded == single (71-112)
    std::mt19937_64 rng(11);
    for (int trial = 0; trial < 10; ++trial) {
      size_t n_sym = 1 + rng() % 60, n_m = 1 + rng() % 40, n_smp = 1 + rng() % 700;
      BitMatrix batch_bits(n_sym, n_smp);
      for (size_t r = 0; r < n_sym; ++r)
        for (size_t c = 0; c < n_smp; ++c) batch_bits.set_bit(r, c, rng() & 1);
      SymbolAssignmentBatch batch{batch_bits};
      std::vector<MeasurementExpression> exprs(n_m);
      BitMatrix dense(n_m, n_sym);
      for (size_t k = 0; k < n_m; ++k)
        for (uint32_t s = 0; s < n_sym; ++s)
          if (rng() % 4 == 0) {
            exprs[k].symbols.push_back(s);
            dense.set_bit(k, s, true);
          }
      SampleMatrix fast = sample(exprs, batch);
      // dense multiply by definition
      BitMatrix expect(n_m, n_smp);
      for (size_t k = 0; k < n_m; ++k)
        for (size_t t = 0; t < n_sym; ++t)
          if (dense.get_bit(k, t))
            for (size_t j = 0; j < n_smp; ++j)
              if (batch.data.get_bit(t, j)) expect.flip_bit(k, j);
      CHECK(fast.data.same_bits(expect));
      for (size_t j = 0; j < n_smp; ++j) {
        BitVec assign(n_sym);
        for (size_t s = 0; s < n_sym; ++s) assign.set(s, batch.data.get_bit(s, j));
        for (size_t k = 0; k < n_m; ++k) CHECK(fast.data.get_bit(k, j) == exprs[k].evaluate(assign));
      }
      SampleMatrix threaded = sample(exprs, batch, 4);
      CHECK(threaded.data.same_bits(fast.data));
    }
  }
  {  // out-of-range symbol throws std::out_of_range (114-118)
    SymbolAssignmentBatch batch{BitMatrix(3, 8)};
    std::vector<MeasurementExpression> exprs{MeasurementExpression{{5}}};
    bool threw = false;
    try {
      sample(exprs, batch);
    } catch (const std::out_of_range&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // encode_shots formats (120-147)
    SampleMatrix m;
    m.data = BitMatrix(3, 1);
    m.data.set_bit(0, 0, true);
    m.data.set_bit(2, 0, true);
    m.measurement_order = {0, 1, 2};
    CHECK(encode_shots(m, ShotFormat::k01) == "101\n");
    std::string b8 = encode_shots(m, ShotFormat::kB8);
    CHECK(b8.size() == 1 && static_cast<uint8_t>(b8[0]) == 0x05);
    SampleMatrix nine;
    nine.data = BitMatrix(9, 1);
    for (size_t k = 0; k < 9; ++k) nine.data.set_bit(k, 0, true);
    std::string bytes = encode_shots(nine, ShotFormat::kB8);
    CHECK(bytes.size() == 2 && static_cast<uint8_t>(bytes[0]) == 0xFF &&
          static_cast<uint8_t>(bytes[1]) == 0x01);
    SampleMatrix none;
    none.data = BitMatrix(0, 0);
    CHECK(encode_shots(none, ShotFormat::k01).empty());
    CHECK(encode_shots(none, ShotFormat::kB8).empty());
  }
  {  // n_smp == 0 -> std::invalid_argument (sampler.cpp:50)
    auto init = init_from("H 0\nM 0\n");
    bool threw = false;
    try {
      draw_assignments(init.registry, 0, 1);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
  }
  {  // parse errors surface as ParseError (circuit.cpp:79-168)
    bool threw = false;
    try {
      init_from("H 0\nFROB 1\n");
    } catch (const ParseError&) {
      threw = true;
    }
    CHECK(threw);
  }
  // Statistical cases (149-203) on both the reference-compatible draw and the
  // fused Philox sampler.
  for (int fused = 0; fused < 2; ++fused) {
    {  // bernoulli marginals (149-161)
      const size_t shots = 100000;
      auto init = init_from("X_ERROR(0.1) 0\nX_ERROR(0.5) 1\nM 0 1\n");
      SampleMatrix m = fused ? sample_shots(init, shots, 1234)
                             : sample(init.expressions, draw_assignments(init.registry, shots, 1234));
      size_t h0 = 0, h1 = 0;
      for (size_t j = 0; j < shots; ++j) {
        h0 += m.data.get_bit(0, j);
        h1 += m.data.get_bit(1, j);
      }
      check_within_4sigma(h0, shots, 0.1);
      check_within_4sigma(h1, shots, 0.5);
    }
    {  // measurement coins are fair (180-187)
      const size_t shots = 100000;
      auto init = init_from("H 0\nM 0\n");
      SampleMatrix m = fused ? sample_shots(init, shots, 31337)
                             : sample(init.expressions, draw_assignments(init.registry, shots, 31337));
      size_t hits = 0;
      for (size_t j = 0; j < shots; ++j) hits += m.data.get_bit(0, j);
      check_within_4sigma(hits, shots, 0.5);
    }
    {  // xor convolution (189-203)
      const size_t shots = 200000;
      auto init = init_from("X_ERROR(0.05) 0\nX_ERROR(0.2) 0\nX_ERROR(0.45) 0\nM 0\n");
      CHECK(init.expressions.size() == 1);
      CHECK((init.expressions[0].symbols == std::vector<uint32_t>{1, 2, 3}));
      SampleMatrix m = fused ? sample_shots(init, shots, 2024)
                             : sample(init.expressions, draw_assignments(init.registry, shots, 2024));
      size_t hits = 0;
      for (size_t j = 0; j < shots; ++j) hits += m.data.get_bit(0, j);
      check_within_4sigma(hits, shots, 0.5 * (1.0 - (1 - 0.1) * (1 - 0.4) * (1 - 0.9)));
    }
  }
  {  // depolarize pattern frequencies (163-178), reference-compatible draw
    const size_t shots = 100000;
    const double p = 0.3;
    auto init = init_from("DEPOLARIZE1(0.3) 0\n");
    auto batch = draw_assignments(init.registry, shots, 777);
    size_t counts[4] = {0, 0, 0, 0};
    for (size_t j = 0; j < shots; ++j)
      counts[batch.data.get_bit(1, j) | (batch.data.get_bit(2, j) << 1)]++;
    check_within_4sigma(counts[0], shots, 1.0 - p);
    check_within_4sigma(counts[1], shots, p / 3.0);
    check_within_4sigma(counts[2], shots, p / 3.0);
    check_within_4sigma(counts[3], shots, p / 3.0);
  }
  {  // a draw_assignments call between two fused samples keeps the fused
     // context's model: both samples of the same seed are identical
    auto init = init_from("X_ERROR(0.3) 0\nDEPOLARIZE1(0.2) 1\nM 0 1\n");
    auto other = init_from("H 0\nM 0\n");
    auto a = sample_shots(init, 5000, 7);
    auto batch = draw_assignments(other.registry, 100, 1);
    CHECK(batch.n_symbols() == other.registry.size());
    auto b = sample_shots(init, 5000, 7);
    CHECK(a.data.same_bits(b.data));
    // parse_circuit + run_initialization(program) == run_initialization_text
    auto prog = parse_circuit("X_ERROR(0.3) 0\nDEPOLARIZE1(0.2) 1\nM 0 1\n");
    CHECK(prog.size() == 3 && prog[1].kind == InstrKind::kDepolarize1 && prog[2].targets.size() == 2);
    CHECK(run_initialization(prog).expressions == init.expressions);
    bool threw = false;
    try {
      parse_circuit("H 0\nFROB 1\n");
    } catch (const ParseError& e) {
      threw = e.line == 2;
    }
    CHECK(threw);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
