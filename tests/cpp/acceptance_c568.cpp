// The reference acceptance criteria 5, 6 and 8 (proj/tests/acceptance.cpp:
// 268-361 and 437-533: noise marginals through the full pipeline, sparse vs
// dense vs per-shot products, sampling cost independent of circuit length),
// their source text taken unchanged from the reference file by
// oracle/Makefile (acceptance_c568.inc), compiled against the B200 library
// through the C++ shim. Prints one line per criterion; exits non-zero if any
// fails. (The other criteria exercise the reference's CLI, state-vector
// oracle and circuit generators, which are out of scope.)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "cliffsym/bit_matrix.hpp"
#include "cliffsym/sampler.hpp"
#include "cliffsym/tableau.hpp"
#include "test_support.hpp"

using namespace cliffsym;
using Clock = std::chrono::steady_clock;

namespace {

struct Failure {
  std::string what;
};

void require(bool ok, const std::string& what) {
  if (!ok) throw Failure{what};
}

#include "acceptance_c568.inc"

}  // namespace

int main() {
  int failed = 0;
  auto run = [&](const char* name, auto&& fn) {
    try {
      fn();
      std::printf("[PASS] %s\n", name);
    } catch (const Failure& f) {
      ++failed;
      std::printf("[FAIL] %s: %s\n", name, f.what.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("[FAIL] %s: exception %s\n", name, e.what());
    }
  };
  run("criterion 5 (noise marginals)", [] { criterion_5(); });
  run("criterion 6 (sparse == dense == per-shot)", [] { criterion_6(); });
  std::string detail;
  run("criterion 8 (sampling independent of gate count)", [&] { criterion_8(detail); });
  std::printf("criterion 8: %s\n", detail.c_str());
  return failed ? 1 : 0;
}
