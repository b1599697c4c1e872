// Compatibility header: reference code that includes "cliffsym/sampler.hpp"
// compiles unchanged against the B200 library through the C++ shim.
#pragma once
#include "cliffsym_b200.hpp"
namespace cliffsym {
using namespace cliffsym_b200;
}  // namespace cliffsym
