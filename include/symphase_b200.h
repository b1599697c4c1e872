/*
 * symphase_b200.h — C ABI of the B200-native SymPhase sampling hot path.
 *
 * Drop-in boundary for the reference's sampler operator API (cliffsym,
 * proj/core/include/cliffsym/sampler.hpp). The reference has no C ABI of its
 * own; each entry point below names the reference call it replaces.
 *
 * Conventions
 *   - Return SP_OK (0) or a negative sp_status; sp_last_error() returns a
 *     thread-local message for the last failure on the calling thread.
 *   - Exception mapping of the reference (sampler.cpp:50, 63-67;
 *     bit_matrix.cpp:288, 322): std::invalid_argument -> SP_ERR_INVALID_ARGUMENT,
 *     std::out_of_range -> SP_ERR_OUT_OF_RANGE, ParseError -> SP_ERR_PARSE,
 *     std::logic_error -> SP_ERR_LOGIC.
 *   - One host thread per context, one context per device. Device work is
 *     asynchronous on the context's stream (sp_set_stream); pointers named
 *     d_* are device pointers, h_* host pointers. The caller owns every
 *     buffer it passes in.
 *   - Bit-sliced layout ("measurement-major" for results, "symbol-major" for
 *     assignments): u64 words, row-major with leading dimension ld (in
 *     words); bit j%64 of word j/64 of row r is element (r, j). Rows are
 *     measurements (or symbols), columns are shots. This is the logical
 *     orientation of the reference's SampleMatrix / SymbolAssignmentBatch
 *     (sampler.hpp:32-46) with the BitVec bit order (bitvec.hpp:21-23).
 *     Padding bits past n_shots are written as zero.
 */
#ifndef SYMPHASE_B200_H
#define SYMPHASE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SP_ABI_VERSION 1

typedef enum {
  SP_OK = 0,
  SP_ERR_INVALID_ARGUMENT = -1, /* std::invalid_argument */
  SP_ERR_OUT_OF_RANGE = -2,     /* std::out_of_range */
  SP_ERR_PARSE = -3,            /* cliffsym::ParseError (circuit.hpp:42-47) */
  SP_ERR_LOGIC = -4,            /* std::logic_error */
  SP_ERR_CUDA = -5,             /* CUDA runtime failure */
  SP_ERR_NOT_LOADED = -6,       /* M_sym / channel table not loaded yet */
  SP_ERR_UNSUPPORTED = -7       /* shape outside what a kernel handles */
} sp_status;

/* GroupDistribution, symbols.hpp:19-25 (same numbering). */
enum {
  SP_DIST_CONSTANT = 0,
  SP_DIST_BERNOULLI = 1,
  SP_DIST_COIN = 2,
  SP_DIST_DEPOLARIZE1 = 3,
  SP_DIST_DEPOLARIZE2 = 4
};

/* SymbolGroup, symbols.hpp:36-42 (instruction_index dropped). */
typedef struct {
  uint8_t dist;
  uint8_t reserved[7];
  double param;
  uint32_t first_symbol;
  uint32_t arity;
} sp_group;

typedef enum {
  SP_RNG_PHILOX = 0,          /* counter-based Philox4x32-10 + geometric skip (default) */
  SP_RNG_COMPAT_SPLITMIX = 1  /* bit-exact keyed_draw/fill_group (sampler.hpp:14-28, sampler.cpp:11-44) */
} sp_rng;

typedef enum { SP_FMT_01 = 0, SP_FMT_B8 = 1 } sp_format; /* ShotFormat, sampler.hpp:60-63 */

typedef enum {
  SP_PRODUCT_AUTO = 0,   /* DENSE when nnz(M_sym) > 0.15 n_meas n_sym (measured crossover), else SPARSE */
  SP_PRODUCT_SPARSE = 1, /* CSR over measurements (expression lists) */
  SP_PRODUCT_DENSE = 2,  /* dense row-major M_sym words, Four-Russians tables */
  SP_PRODUCT_TENSOR = 3  /* dense M_sym as an integer GEMM on the tensor cores (tcgen05.mma
                            kind::i8, int32 counts in TMEM, parity of each count) */
} sp_product;

typedef struct sp_ctx sp_ctx;
typedef struct sp_model sp_model;

const char* sp_last_error(void);
int sp_abi_version(void);

/* ---- host front end: parse_circuit (circuit.hpp:55) + run_initialization
 *      (tableau.hpp:101). Produces InitResult.expressions (CSR rows of M_sym,
 *      sorted symbol ids) and InitResult.registry (the group table). ------- */
int sp_model_from_text(const char* text, sp_model** out);
void sp_model_destroy(sp_model* m);
int sp_model_dims(const sp_model* m, uint64_t* n_qubits, uint64_t* n_meas, uint64_t* n_sym,
                  uint64_t* n_groups, uint64_t* nnz);
/* row_ptr[n_meas+1], sym_idx[nnz], groups[n_groups]; any may be NULL. */
int sp_model_export(const sp_model* m, uint64_t* row_ptr, uint32_t* sym_idx, sp_group* groups);

/* parse_circuit (circuit.hpp:55, circuit.cpp:79-168) as flat arrays: kind
 * (InstrKind order, circuit.hpp:13-29), parameter, 1-based source line and
 * the targets of instruction i in targets[tgt_ptr[i] .. tgt_ptr[i+1]).
 * Two-pass: with kinds == NULL only *n_instr_out / *n_targets_out are set.
 * SP_ERR_PARSE with the reference's "line N: ..." message on bad input. */
int sp_parse_circuit(const char* text, uint64_t cap_instr, uint8_t* kinds, double* params,
                     uint64_t* lines, uint64_t* tgt_ptr, uint64_t cap_targets,
                     uint32_t* targets, uint64_t* n_instr_out, uint64_t* n_targets_out);
/* run_initialization(const std::vector<Instruction>&) (tableau.hpp:101) on a
 * structured program in the same flat form; the instruction shapes are
 * checked like parse_circuit's (SP_ERR_INVALID_ARGUMENT). */
int sp_model_from_program(uint64_t n_instr, const uint8_t* kinds, const double* params,
                          const uint64_t* tgt_ptr, const uint32_t* targets, sp_model** out);

/* Detector layer (not in the reference: its parser has no DETECTOR,
 * circuit.cpp:117-121). A detector is the XOR of a set of measurements;
 * detector k = measurements det_meas[det_ptr[k] .. det_ptr[k+1]). Its symbolic
 * row is the GF(2) sum of those M_sym rows (sorted symmetric difference), so
 * D_sym = A * M_sym. Loading D_sym rows (with the same group table) into a
 * context samples detector records and per-detector counts with the same
 * kernels; for a supplied S, D_sym * S == A * (M_sym * S) bit for bit.
 * Two-pass: call with out_sym_idx == NULL to get *nnz_out, then again with a
 * buffer of that many entries. Measurement ids must be < n_meas
 * (SP_ERR_OUT_OF_RANGE otherwise). */
int sp_detector_rows(uint64_t n_meas, const uint64_t* row_ptr, const uint32_t* sym_idx,
                     uint64_t n_det, const uint64_t* det_ptr, const uint32_t* det_meas,
                     uint64_t* out_row_ptr, uint32_t* out_sym_idx, uint64_t cap,
                     uint64_t* nnz_out);

/* ---- device context ---------------------------------------------------- */
int sp_ctx_create(int device, sp_ctx** out);
void sp_ctx_destroy(sp_ctx* ctx);
int sp_set_stream(sp_ctx* ctx, void* cuda_stream); /* cudaStream_t; NULL = legacy default */
int sp_set_rng(sp_ctx* ctx, sp_rng rng);
int sp_set_product(sp_ctx* ctx, sp_product variant);

/* M_sym as the reference's expression list: row k = sorted symbol ids of
 * measurement k (MeasurementExpression, symbols.hpp:90-100). Host pointers.
 * The library derives CSR-of-variables (per-symbol measurement lists), the
 * dense row-major words and the per-channel sampling plan on the device. */
int sp_load_msym_csr(sp_ctx* ctx, uint64_t n_meas, uint64_t n_sym, const uint64_t* h_row_ptr,
                     const uint32_t* h_sym_idx);
/* M_sym as dense row-major words [n_meas][ld_words] (bit s of row k = 1 iff
 * symbol s appears in measurement k). Host pointer. */
int sp_load_msym_dense(sp_ctx* ctx, uint64_t n_meas, uint64_t n_sym, const uint64_t* h_words,
                       uint64_t ld_words);
/* SymbolRegistry groups (symbols.hpp:47-86). Host pointer; group 0 must be
 * the constant group. */
int sp_load_groups(sp_ctx* ctx, uint64_t n_groups, const sp_group* h_groups);
int sp_load_model(sp_ctx* ctx, const sp_model* m); /* = csr + groups */

/* Plan. The first call that needs the model builds the sampling plan on the
 * host and uploads it: the chain transform M = L*D, per-(group, pattern) flip
 * lists, the sampling slices, and the heavy-path drain order. The first plan
 * for a model also measures the fused kernel's generator/drain warp split and
 * padded-XOR mode with a few short launches, cached per model fingerprint.
 * Re-loading a model with identical content keeps the plan and only
 * re-uploads the raw arrays.
 *
 * Results never depend on that tuning. Random streams are keyed by
 * (seed, sampling slice, global T-shot tile), and the slices and T depend
 * only on the model and the device's shared memory. The SP_* environment
 * switches in DESIGN.md change speed, not bits, except SP_TLOG2, SP_SEG_MIN,
 * SP_SEG_EVENTS and SP_LIST_CLASSES, which redefine the slices. */

/* Shot-tile size T of the fused sampler for the loaded model. Random streams
 * are keyed by (seed, global T-shot tile), so any split of a shot range into
 * calls whose shot_begin is a multiple of T — one GPU or many — yields the
 * same bits. */
int sp_shot_tile(sp_ctx* ctx, uint64_t* tile);

/* K1 — fused sampler: draw_assignments + sample (sampler.cpp:48-112) in one
 * kernel. d_out: measurement-major [n_meas][ld], ld >= ceil(n_shots/64).
 * Column j of d_out is global shot shot_begin + j; shot_begin % T == 0.
 * d_counts (nullable): u64 [n_meas], += number of shots with outcome 1. */
int sp_sample(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
              uint64_t* d_out, uint64_t ld, uint64_t* d_counts);

/* K1 with tiled records (the layout the fused kernel produces natively,
 * cf. the reference's 512x512-bit TiledBitMatrix, bit_matrix.hpp:13-31):
 * d_out holds ceil(n_shots/T) blocks; block b is [n_meas][T/64] u64 words
 * for shots shot_begin + b*T .. + T (bits past n_shots are 0). Every store
 * of the kernel is then contiguous, whatever n_meas is. Philox RNG only.
 * sp_tiled_words gives the size in u64 words. */
uint64_t sp_tiled_words(sp_ctx* ctx, uint64_t n_shots);
int sp_sample_tiled(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
                    uint64_t* d_out, uint64_t* d_counts);
/* Detector counts in the sampling launch (not in the reference: its parser
 * has no DETECTOR, circuit.cpp:117-121; the multi-GPU reduction of
 * BASELINE configs[2] needs per-detector flip counts). sp_set_detectors
 * registers detectors as sets of measurement indices (CSR, host pointers;
 * a measurement listed twice cancels); sp_sample_ex then samples the
 * records exactly like sp_sample (ld > 0, measurement-major) or
 * sp_sample_tiled (ld == 0) and, when d_det_counts is not NULL, adds to
 * d_det_counts[k] (u64, device) the number of shots in which detector k is
 * 1 — counted by the fused kernel's drain from the finished rows, with no
 * pass over the records. Fused Philox sampler only (SP_ERR_UNSUPPORTED
 * otherwise); SP_ERR_NOT_LOADED without registered detectors. */
int sp_set_detectors(sp_ctx* ctx, uint64_t n_det, const uint64_t* det_ptr,
                     const uint32_t* det_meas);
int sp_sample_ex(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
                 uint64_t* d_out, uint64_t ld, uint64_t* d_counts, uint64_t* d_det_counts);
/* Tiled records -> measurement-major [n_meas][ld]. */
int sp_untile(sp_ctx* ctx, const uint64_t* d_tiled, uint64_t n_shots, uint64_t* d_out,
              uint64_t ld);
/* encode_shots straight from tiled records. */
int sp_encode_tiled(sp_ctx* ctx, const uint64_t* d_tiled, uint64_t n_shots, sp_format fmt,
                    uint8_t* d_bytes);

/* draw_assignments (sampler.hpp:51-52) on the device: the exact assignment
 * matrix S the fused sampler uses for these shots (row 0 = constant = all
 * ones), so sp_sample == M_sym . S bit for bit — also for thinned channels
 * (a channel whose non-null patterns all flip one list fires as one
 * Bernoulli variable; its firings map back to a uniform non-null pattern and
 * its null patterns come from a second pass, so S keeps the channel's pmf).
 * The exception is a model where the planner merged many channels with one
 * common flip list into a single variable (SP_MERGE_MIN): there S is an
 * independent draw of every original symbol, correct in distribution.
 * d_S: [n_sym][ldS]. With
 * SP_RNG_COMPAT_SPLITMIX it is bit-identical to the reference's
 * draw_assignments(registry, n, seed) when shot_begin=0. */
int sp_draw_assignments(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
                        uint64_t* d_S, uint64_t ldS);

/* K2 — sample(expressions, batch) / gf2_multiply_sparse on a supplied
 * batch (sampler.cpp:61-112, bit_matrix.cpp:314-328). d_S: [n_sym_S][ldS].
 * SP_ERR_OUT_OF_RANGE if an expression names a symbol >= n_sym_S
 * (sampler.cpp:63-67). */
int sp_sample_given_S(sp_ctx* ctx, const uint64_t* d_S, uint64_t n_sym_S, uint64_t ldS,
                      uint64_t n_shots, uint64_t* d_out, uint64_t ld);

/* K3 — encode_shots (sampler.cpp:118-140) on the device. Writes
 * sp_encoded_size() bytes to d_bytes. */
uint64_t sp_encoded_size(uint64_t n_meas, uint64_t n_shots, sp_format fmt);
int sp_encode(sp_ctx* ctx, const uint64_t* d_m, uint64_t ld, uint64_t n_meas, uint64_t n_shots,
              sp_format fmt, uint8_t* d_bytes);

/* The cmd_sample timed region (cliffsym.cpp:108-113) with a HOST output:
 * fused sample + device encode + device->host copy into h_out (pinned or
 * pageable), synchronous. cap = capacity of h_out in bytes. */
int sp_sample_to_host(sp_ctx* ctx, uint64_t seed, uint64_t shot_begin, uint64_t n_shots,
                      sp_format fmt, uint8_t* h_out, uint64_t cap, uint64_t* written);

/* Test hook: one Philox4x32-10 block on the device. ctr_key = {c0,c1,c2,c3,k0,k1}. */
int sp_debug_philox(sp_ctx* ctx, const uint32_t* ctr_key, uint32_t* out);

/* Launch shape and table sizes of the loaded model's fused-sampler plan:
 * {T, gen_warps, cta_threads, staged, row_staged, lp, pad_pred, n_paths,
 *  n_rounds, n_keep, n_segments, n_classes, n_dense, nnz(D), smem_bytes, sampler}
 * with sampler (of tiled launches) 1 = fused K1, 3 = its queued form K7 (same
 * records; gen_warps / cta_threads are then K7's walker warps / threads), 4 = K7 for launches that
 * count detectors and K1 for the others, 5 = the reverse (the launch autotune
 * decides per mode), 2 = K5 column sampler (dense M_sym), 0 = draw S +
 * explicit product. */
int sp_plan_info(sp_ctx* ctx, uint64_t* out16);
/* Which sampler serves one kind of launch (records tiled or measurement-major,
 * with or without per-detector counts): 0 draw S + explicit product, 1 fused
 * K1, 2 K5 column sampler, 3 K7 (the queued form of K1, same records). The
 * launch autotune decides K1 vs K7 per kind on the first load of a model. */
int sp_sampler_kernel(sp_ctx* ctx, int tiled, int with_detector_counts, uint32_t* out);

/* Profiling hook: per-role cycle counters of the fused kernel (gen wait,
 * gen work, drain wait, drain work), then walk steps, firings and two
 * reserved slots, enabled by SP_PHASE_TIMERS=1 at plan build; copied out
 * (8 values) and cleared. */
int sp_debug_timers(sp_ctx* ctx, long long* out8);

/* Number of kernel launches this context has issued so far. */
uint64_t sp_launch_count(const sp_ctx* ctx);
int sp_synchronize(sp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SYMPHASE_B200_H */
