/*
 * ssjoin_b200.h -- C ABI of the B200-native candidate-verification engine
 * (verification phase of exact set-similarity self-joins, Bellas & Gounaris,
 * arXiv 1812.09141).
 *
 * The reference has no FFI: its seam is the C++ class
 *   ssjoin::VerificationEngine      (proj/include/ssjoin/verify.hpp:241-351)
 * called once per sealed chunk by the join driver's dispatcher thread
 *   ssjoin::run_join, role H1       (proj/include/ssjoin/pipeline.hpp:215-258, call at :228).
 * Every entry point below replaces one piece of that surface; the citation is on each.
 * Plain pointers and sizes only. All functions return SSJ_OK (0) or an ssj_status code,
 * with a thread-local message available from ssj_last_error(). There is no CPU fallback:
 * every verification entry point runs the sm_100a kernels or fails.
 *
 * Threading: an engine is used by one host thread at a time (the reference calls
 * verify_chunk only from H1, pipeline.hpp:228). Each entry point selects the engine's
 * device itself, so an engine created on thread H0 may be driven from thread H1.
 */
#ifndef SSJOIN_B200_H
#define SSJOIN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSJ_ABI_VERSION 1

typedef enum {
    SSJ_OK = 0,
    SSJ_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
    SSJ_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range: set index >= n (collection.hpp:87) */
    SSJ_ERR_CUDA = 3,             /* CUDA runtime / launch failure */
    SSJ_ERR_RUNTIME = 4,          /* std::runtime_error class */
    SSJ_ERR_NO_DEVICE = 5         /* no CUDA device: the engine refuses to run */
} ssj_status;

/* similarity.hpp:11 SimilarityFunction */
typedef enum { SSJ_JACCARD = 0, SSJ_COSINE = 1, SSJ_DICE = 2, SSJ_OVERLAP = 3 } ssj_function;

/* verify.hpp:18 StrategyKind */
typedef enum { SSJ_STRATEGY_A = 0, SSJ_STRATEGY_B = 1, SSJ_STRATEGY_C = 2, SSJ_STRATEGY_AUTO = 3 } ssj_strategy_kind;

/* verify.hpp:31 OutputMode */
typedef enum { SSJ_MODE_COUNT = 0, SSJ_MODE_PAIRS = 1 } ssj_mode;

/* similarity.hpp:67-82 SimilarityPredicate {function, Threshold{num, den}, overlap_threshold} */
typedef struct {
    int32_t function; /* ssj_function */
    uint32_t reserved;
    uint64_t num;
    uint64_t den;
    uint64_t overlap_threshold;
} ssj_predicate;

/* verify.hpp:21-29 Strategy {kind, group_size (power of two)} */
typedef struct {
    int32_t kind; /* ssj_strategy_kind */
    uint32_t group_size;
} ssj_strategy;

/* verify.hpp:183-195 VerifyStats (accumulated, like the reference's atomics) */
typedef struct {
    uint64_t pairs_verified;
    uint64_t early_exit_prunes;
    uint64_t comparison_budget_violations;
} ssj_stats;

typedef struct ssj_engine ssj_engine;

/* ---- version / errors ------------------------------------------------------------- */
int ssj_abi_version(void);
const char* ssj_last_error(void);
/* Number of visible CUDA devices (0 when none). */
int ssj_device_count(void);

/* ---- similarity arithmetic (host side; similarity.hpp) ------------------------------ */
/* Threshold::parse (similarity.hpp:30-56): "0.8", ".85", "1", "4/5" -> reduced num/den. */
int ssj_threshold_parse(const char* text, uint64_t* num, uint64_t* den);
/* SimilarityPredicate::validate (similarity.hpp:74-81). */
int ssj_predicate_validate(const ssj_predicate* pred);
/* Strategy::validate (verify.hpp:25-28). */
int ssj_strategy_validate(const ssj_strategy* strategy);
/* equivalent_overlap (similarity.hpp:108-123), exact u128 arithmetic. */
uint64_t ssj_equivalent_overlap(const ssj_predicate* pred, uint64_t size_r, uint64_t size_s);

/* ---- engine ------------------------------------------------------------------------ */
/*
 * VerificationEngine(collection, pred, mode, strategy)   (verify.hpp:243-245)
 * The collection is the reference's CSR (collection.hpp:76-94): tokens[offsets[n_sets]],
 * offsets[n_sets + 1], sets sorted with strictly increasing tokens. It is re-laid out
 * once into the device's 32-byte-aligned padded CSR and uploaded; unlike the reference
 * (which keeps a reference, verify.hpp:347) the host arrays may be freed after return.
 * `strategy` is validated (verify.hpp:25-28); Auto is resolved here (verify.hpp:245).
 */
int ssj_engine_create(ssj_engine** out, int device, const uint32_t* tokens,
                      const uint32_t* offsets, uint32_t n_sets, const ssj_predicate* pred,
                      int32_t mode, const ssj_strategy* strategy);

/* Same, but the collection is already in this device's memory in the engine's padded
 * layout (produced by another engine: see ssj_engine_device_collection), e.g. after an
 * NCCL broadcast over NVLink. The engine does not take ownership. */
int ssj_engine_create_from_device(ssj_engine** out, int device, const uint32_t* d_tokens,
                                  uint64_t n_padded_tokens, const uint32_t* d_sets /*2*n*/,
                                  uint32_t n_sets, uint64_t n_tokens_total,
                                  const ssj_predicate* pred, int32_t mode,
                                  const ssj_strategy* strategy);

/* The engine's device-resident collection: padded token array and the {pos, size} set
 * descriptors (uint32 pairs). Pointers stay valid until ssj_engine_destroy. */
int ssj_engine_device_collection(const ssj_engine* e, const uint32_t** d_tokens,
                                 uint64_t* n_padded_tokens, const uint32_t** d_sets);

void ssj_engine_destroy(ssj_engine* e);

/* VerificationEngine::strategy() (verify.hpp:255): the resolved strategy (never Auto). */
int ssj_engine_strategy(const ssj_engine* e, ssj_strategy* resolved);
int ssj_engine_device(const ssj_engine* e);

/* ---- the hot call ------------------------------------------------------------------ */
/*
 * VerificationEngine::verify_chunk(chunk, pool, stats)   (verify.hpp:257-275)
 * C[nC] candidate set indices, C_O[nCO] = (probe, cumulative end) pairs (chunk.hpp:20-48),
 * both HOST memory (pinned memory from ssj_host_alloc is copied without staging).
 *   flags_out : host, nC bytes, slot order = C order, 0/1; required in Pairs mode,
 *               ignored (may be NULL) in Count mode (verify.hpp:258-264).
 *   count_out : number of qualifying candidates (= sum of flags).
 *   stats     : nullable; accumulated like VerifyStats::record (verify.hpp:188-194),
 *               recorded for strategies A and B only, as in the reference (C records
 *               nothing, verify.hpp:303-345).
 * Errors: SSJ_ERR_OUT_OF_RANGE if any probe/candidate >= n_sets (collection.hpp:87),
 * SSJ_ERR_INVALID_ARGUMENT on a malformed C_O (end offsets decreasing or > nC).
 * The engine does not retain C / C_O / flags after return (pipeline.hpp:238 ownership).
 */
int ssj_verify_chunk(ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                     uint64_t nCO, uint8_t* flags_out, uint64_t* count_out, ssj_stats* stats);

/* Asynchronous pair of ssj_verify_chunk for double buffering (at most 2 in flight; the
 * host buffers must stay untouched until the matching wait returns). Tickets complete
 * in submission order. */
int ssj_submit_chunk(ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                     uint64_t nCO, uint8_t* flags_out, uint64_t* ticket);
int ssj_wait_chunk(ssj_engine* e, uint64_t ticket, uint64_t* count_out, ssj_stats* stats);

/*
 * Result compaction for a chunk (pairs with overlaps): verifies like ssj_verify_chunk and
 * returns the qualifying slots in ascending slot order with their TRUE overlaps |r ∩ s|
 * (oracle.hpp:48-62 semantics; the merge is completed for qualifying pairs).
 * slots_out / overlaps_out: host arrays of capacity cap; *n_out = number of results
 * (if > cap only cap are written and SSJ_ERR_RUNTIME is returned).
 */
int ssj_verify_chunk_results(ssj_engine* e, const uint32_t* C, uint64_t nC,
                             const uint32_t* C_O, uint64_t nCO, uint32_t* slots_out,
                             uint32_t* overlaps_out, uint64_t cap, uint64_t* n_out);

/*
 * Device-resident variant (kernel-only path; the chunk is already in HBM):
 * d_C, d_C_O, d_flags (nullable) are device pointers; d_result is a device array of
 * SSJ_RESULT_WORDS uint64 that the call zeroes and fills asynchronously on `stream`
 * (a cudaStream_t, NULL = the engine's compute stream):
 *   [0] count  [1] error bits  [2..4] stats (pairs_verified, prunes, violations)
 * No host synchronisation; read d_result after the stream completes.
 */
#define SSJ_RESULT_WORDS 8
#define SSJ_RESULT_COUNT 0
#define SSJ_RESULT_ERROR 1
#define SSJ_RESULT_STATS 2
int ssj_verify_chunk_device(ssj_engine* e, const uint32_t* d_C, uint64_t nC,
                            const uint32_t* d_C_O, uint64_t nCO, uint8_t* d_flags,
                            uint64_t* d_result, void* stream);

/* Number of kernels ssj_verify_chunk_device launches for a chunk of this shape
 * (for launch accounting in benchmarks). */
int ssj_launches_per_chunk(const ssj_engine* e, uint64_t nC, uint64_t nCO);

/*
 * Instrumentation: algorithmic bytes of a device-resident chunk under the reference's
 * early-exit loop: sum over pairs of 4 + 8 + 1 + 4*min(j_exit+1, |s|)
 * plus over slices 8 + 8 + 4*|r|. Runs a replay kernel; result written to *d_bytes
 * (device u64) on `stream`.
 */
int ssj_chunk_algorithmic_bytes_device(ssj_engine* e, const uint32_t* d_C, uint64_t nC,
                                       const uint32_t* d_C_O, uint64_t nCO,
                                       uint64_t* d_bytes, void* stream);

/* ---- pinned host buffers (ChunkBuilder storage; double-buffered by the driver) ------- */
void* ssj_host_alloc(size_t bytes);
void ssj_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* SSJOIN_B200_H */
