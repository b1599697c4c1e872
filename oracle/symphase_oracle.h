/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the sampling hot path.
 *
 * A plain-C restatement of the reference's sampler (cliffsym, /root/reference
 * proj/core). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it; the product library never links it.
 *
 * Pinned against (a) the reference library itself, built by oracle/Makefile
 * into oracle/_ref/ and driven through oracle/ref_driver.cpp, and (b) the
 * reference test suite's golden vectors (tests/golden/, test_sampler.cpp:
 * 30-147). See tests/test_oracle_cpu.py.
 *
 * Layout ("bit-sliced"): u64 words, row-major, bit j%64 of word j/64 of row r
 * is element (r, j). Rows of S are symbols, rows of the result are
 * measurements, columns are shots — the logical orientation of the
 * reference's SymbolAssignmentBatch / SampleMatrix (sampler.hpp:32-46).
 */
#ifndef SYMPHASE_ORACLE_H
#define SYMPHASE_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* GroupDistribution numbering (symbols.hpp:19-25). */
enum { ORC_CONST = 0, ORC_BERNOULLI = 1, ORC_COIN = 2, ORC_DEP1 = 3, ORC_DEP2 = 4 };

uint64_t orc_mix64(uint64_t x);                                     /* sampler.hpp:14-19 */
uint64_t orc_keyed_draw(uint64_t seed, uint64_t group, uint64_t shot); /* sampler.hpp:24-26 */
double orc_unit_double(uint64_t u);                                 /* sampler.hpp:28 */
/* Symbol bits of one group from one draw (fill_group, sampler.cpp:11-44):
 * bit b of the result is the value of symbol first_symbol + b. */
unsigned orc_group_bits(int dist, double param, uint64_t u);

/* draw_assignments (sampler.cpp:48-59). S is [n_sym][ldS]. Returns 0, or -2
 * for n_shots == 0 (std::invalid_argument at sampler.cpp:50). */
int orc_draw_assignments(uint64_t n_groups, const uint8_t* dist, const double* param,
                         const uint32_t* first, const uint32_t* arity, uint64_t n_sym,
                         uint64_t n_shots, uint64_t seed, uint64_t* S, uint64_t ldS);

/* Same draws for global shots [shot_begin, shot_begin + n_shots): keyed_draw
 * is keyed by the shot index (sampler.hpp:21-26), so any shot range can be
 * drawn independently — the multi-GPU sharding invariant. */
int orc_draw_assignments_range(uint64_t n_groups, const uint8_t* dist, const double* param,
                               const uint32_t* first, const uint32_t* arity, uint64_t n_sym,
                               uint64_t shot_begin, uint64_t n_shots, uint64_t seed, uint64_t* S,
                               uint64_t ldS);

/* sample(expressions, batch) / gf2_multiply_sparse (sampler.cpp:61-112,
 * bit_matrix.cpp:314-328): row k of out = XOR of S rows listed in row k.
 * Returns 0, or -1 when a symbol id >= n_sym (std::out_of_range,
 * sampler.cpp:63-67). */
int orc_sample_sparse(uint64_t n_meas, const uint64_t* row_ptr, const uint32_t* sym_idx,
                      uint64_t n_sym, uint64_t n_shots, const uint64_t* S, uint64_t ldS,
                      uint64_t* out, uint64_t ld);

/* encode_shots (sampler.cpp:118-140). fmt 0 = '01', 1 = 'b8'. Returns the
 * number of bytes written (n_shots*(n_meas+1) or n_shots*ceil(n_meas/8)). */
uint64_t orc_encode(uint64_t n_meas, uint64_t n_shots, const uint64_t* m, uint64_t ld,
                    int fmt, uint8_t* out);

#ifdef __cplusplus
}
#endif
#endif
