// Device phase store of the symbolic pass (frontend_dev.cu).
#pragma once

#include <cstddef>
#include <cstdint>

namespace symphase {

struct PhaseDev;
bool phase_dev_available();
// n_rows phase rows of ws u64 words each, zeroed.
PhaseDev* phase_dev_create(size_t n_rows, uint64_t ws);
void phase_dev_destroy(PhaseDev* p);
// XOR single bits: entry = row << 32 | symbol.
void phase_dev_flips(PhaseDev* p, const uint64_t* flips, size_t n);
// ph[t] ^= ph[src] over words [0, words) for each target row.
void phase_dev_xor_rows(PhaseDev* p, uint32_t src, const uint32_t* targets, size_t n_t,
                        uint32_t words);
// Copy host phase rows [0, n_rows) x ws words (row-major) into the store
// (the host pass moving its phase matrix to the device mid-circuit).
void phase_dev_upload(PhaseDev* p, const uint64_t* host);
void phase_dev_clear_row(PhaseDev* p, uint32_t row, uint32_t words);
// XOR of the given rows over words [0, words), returned in a host buffer
// (valid until the next call).
const uint64_t* phase_dev_reduce(PhaseDev* p, const uint32_t* rows, size_t n_r, uint32_t words);

}  // namespace symphase
