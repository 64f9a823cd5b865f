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
 * `strategy` is validated (verify.hpp:25-28); Auto is resolved here (verify.hpp:245, see
 * ssj_engine_strategy / ssj_engine_kernel_strategy).
 */
int ssj_engine_create(ssj_engine** out, int device, const uint32_t* tokens,
                      const uint32_t* offsets, uint32_t n_sets, const ssj_predicate* pred,
                      int32_t mode, const ssj_strategy* strategy);

/* The engine's padded layout: set i's tokens start at token 8 * pos8[i] (32-byte aligned),
 * each set padded to a multiple of 8 tokens with 0xFFFFFFFF, and SSJ_TOKEN_TAIL_PAD
 * 0xFFFFFFFF tokens after the last set (the kernels read whole steps past a set's end). */
#define SSJ_TOKEN_TAIL_PAD 512

/* Same, but the collection is already in this device's memory in the engine's padded
 * layout (produced by another engine: see ssj_engine_device_collection), e.g. after an
 * NCCL broadcast over NVLink. The engine does not take ownership. n_padded_tokens must
 * cover the last set plus SSJ_TOKEN_TAIL_PAD (checked). */
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

/* ---- one engine over several GPUs (the engine run_join builds,
 *      pipeline.hpp:156, and hands every chunk, :228) --------------------------------------
 * devices[0..n_devices): CUDA ordinals (a device may repeat: several engines on one GPU).
 * The padded collection is uploaded ONCE (devices[0]) and fanned out device to device over
 * NVLink / NVSwitch with peer copies in a doubling tree (round k: the 2^k devices holding it
 * copy to the next 2^k). The result is an ordinary ssj_engine*: ssj_verify_chunk, submit/wait,
 * _results and _pairs cut each chunk into n_devices contiguous probe-slice ranges of equal
 * work -- per slice 4|r| + k (13 + 4|r|), SURVEY §8(d)'s bytes with |s| <= |r| -- verify them
 * concurrently (one engine per device, its own streams) and return flags in C order (each
 * device writes its range of the caller's buffer), counts and stats summed; ssj_gpu_join
 * runs probe shard g on device g. Device-pointer entry points (ssj_verify_chunk_device,
 * ssj_chunk_algorithmic_bytes_device) need a one-device engine (SSJ_ERR_INVALID_ARGUMENT). */
int ssj_engine_create_multi(ssj_engine** out, const int32_t* devices, uint32_t n_devices,
                            const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                            const ssj_predicate* pred, int32_t mode, const ssj_strategy* strategy);
/* The engine's devices (1 for a one-device engine) and the collection fan-out time. */
int ssj_engine_devices(const ssj_engine* e, int32_t* devices, uint32_t cap, uint32_t* n_devices,
                       double* fanout_ms);
/* The split a multi-device engine applies to a chunk (host only; no GPU needed):
 * ranges[4 g .. 4 g + 3] = {first slice, end slice, first slot, end slot} of part g.
 * set_sizes: |set| per set (the probes' sizes weigh the slices). SSJ_ERR_INVALID_ARGUMENT on a
 * malformed C_O (end offsets decreasing or beyond nC), like verification. */
int ssj_chunk_split(const uint32_t* set_sizes, uint32_t n_sets, uint32_t parts,
                    const uint32_t* C_O, uint64_t nCO, uint64_t nC, uint64_t* ranges);

/* VerificationEngine::strategy() (verify.hpp:255): the resolved strategy (never Auto),
 * resolved exactly as the reference resolves it (verify.hpp:249-253: Auto -> B when the
 * average set size is <= 10, else C with group >= 128); VerifyStats follow it (C records
 * none). */
int ssj_engine_strategy(const ssj_engine* e, ssj_strategy* resolved);
/* The kernel family that runs: the requested A / B / C, and for Auto strategy A's kernels
 * (load-balanced thread-per-pair + warp-per-long-pair; 3.5-90x faster than B / C on the
 * B200). Flags and counts do not depend on it. */
int ssj_engine_kernel_strategy(const ssj_engine* e, ssj_strategy* exec);
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
 * H2 on the GPU (decode_pairs, pipeline.hpp:79-92, and write_pairs order, report.hpp:39-42):
 * verifies the chunk and returns the qualifying pairs as original input ids
 * (r_id, s_id) with r_id > s_id, two uint32 per pair, plus their true overlaps (nullable).
 * sorted != 0 sorts them on the device (radix sort on r_id << 32 | s_id); sorted == 0 returns
 * them in decode_pairs order (slot = C order, pipeline.hpp:79-92). Original ids come
 * from ssj_engine_set_original_ids (identity if never set). Only the qualifying pairs cross
 * PCIe (no per-candidate flags). stats: nullable, as in ssj_verify_chunk.
 */
int ssj_engine_set_original_ids(ssj_engine* e, const uint32_t* original_id /* n_sets; NULL = identity */);
int ssj_verify_chunk_pairs(ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                           uint64_t nCO, uint32_t* pairs_out, uint32_t* overlaps_out,
                           uint64_t cap, uint64_t* n_out, int sorted, ssj_stats* stats);

/*
 * Device-resident variant (kernel-only path; the chunk is already in HBM):
 * d_C, d_C_O, d_flags (nullable) are device pointers; d_result is a device array of
 * SSJ_RESULT_WORDS uint64 that the call zeroes and fills asynchronously on `stream`
 * (a cudaStream_t; NULL = the legacy default stream, as in the CUDA runtime):
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

/* Kernel timing on the launching stream (benchmark instrumentation): when enabled,
 * ssj_verify_chunk_device brackets its whole verification (result resets, prep/bitmap
 * kernels and the strategy's kernels) with CUDA events recorded on the caller's stream; ssj_engine_kernel_time synchronises on them and returns the summed
 * kernel milliseconds and launch count since the last call (then resets). */
int ssj_engine_set_profiling(ssj_engine* e, int enabled);
int ssj_engine_kernel_time(ssj_engine* e, double* total_ms, uint64_t* launches);

/* Copy the engine's device collection into caller-owned device buffers of the same device
 * (d_tokens: n_padded_tokens u32, d_sets: 2*n_sets u32) on `stream`, e.g. to hand it to an
 * NCCL broadcast. NULL stream = the legacy default stream. */
int ssj_engine_export_collection(const ssj_engine* e, uint32_t* d_tokens, uint32_t* d_sets,
                                 void* stream);

/* Number of kernels ssj_verify_chunk_device launches for a chunk of this shape
 * (for launch accounting in benchmarks). */
int ssj_launches_per_chunk(const ssj_engine* e, uint64_t nC, uint64_t nCO);

/*
 * Instrumentation: algorithmic bytes of a device-resident chunk under the reference's
 * early-exit loop: sum over pairs of 4 + 8 + 1 + 4*min(j_exit+1, |s|)
 * plus over slices 8 + 8 + 4*|r|. Runs a replay kernel; result written to *d_bytes
 * (device u64) on `stream` (NULL = the legacy default stream).
 */
int ssj_chunk_algorithmic_bytes_device(ssj_engine* e, const uint32_t* d_C, uint64_t nC,
                                       const uint32_t* d_C_O, uint64_t nCO,
                                       uint64_t* d_bytes, void* stream);

/* ---- candidate generation (role H0; joiners.hpp:47-183) ------------------------------ */
/* pipeline.hpp:25 Algorithm */
typedef enum { SSJ_ALG_ALLPAIRS = 0, SSJ_ALG_PPJOIN = 1, SSJ_ALG_GROUPJOIN = 2 } ssj_algorithm;

typedef struct ssj_candidates ssj_candidates;
/*
 * The candidate stream of probes [probe_begin, probe_end) as one unbounded chunk (C, C_O),
 * identical batch for batch to the reference generators (allpairs_generate
 * joiners.hpp:47-71, ppjoin_generate :75-102, groupjoin_generate :111-183). threads > 1
 * runs AllPairs / PPJoin on that many host threads (0 = all); threads == 1 and GroupJoin
 * follow the reference's sequential control flow. GroupJoin's intra-group pairs
 * (:175-179) are returned separately as (a, b) host pairs.
 */
int ssj_generate_candidates(const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                            const ssj_predicate* pred, int32_t algorithm, uint32_t probe_begin,
                            uint32_t probe_end, uint32_t threads, ssj_candidates** out);
/* Several probe windows (windows[2k], windows[2k+1]) = [lo, hi) concatenated in the given
 * order into one chunk, sharing one static index (AllPairs / PPJoin). */
int ssj_generate_candidates_windows(const uint32_t* tokens, const uint32_t* offsets,
                                    uint32_t n_sets, const ssj_predicate* pred, int32_t algorithm,
                                    const uint32_t* windows, uint32_t n_windows, uint32_t threads,
                                    ssj_candidates** out);
int ssj_candidates_sizes(const ssj_candidates* c, uint64_t* nC, uint64_t* nCO, uint64_t* n_host);
int ssj_candidates_copy(const ssj_candidates* c, uint32_t* C, uint32_t* C_O, uint32_t* host_pairs);
void ssj_candidates_free(ssj_candidates* c);

/* ---- collections: synthetic benchmark data + precoded preprocessing ------------------- */
typedef struct ssj_collection ssj_collection;
typedef struct {
    uint64_t seed;
    uint32_t n_sets;
    uint32_t min_size, max_size;
    int32_t zipf_sizes;
    double size_skew;
    uint32_t universe;
    int32_t zipf_tokens;
    double token_skew;
    double duplicate_fraction; /* chance a record is a near-copy of an earlier one */
    uint32_t max_edits;        /* tokens replaced in a near-copy: uniform in [0, max_edits] */
    int32_t distinct_tokens;   /* 1: draw `size` distinct tokens (post-dedup size == size) */
    uint32_t threads;          /* 0 = all host threads; output does not depend on it */
} ssj_synth_config;
/* Synthetic records (oracle.hpp:71-125 knobs + near-duplicates), then preprocess_precoded
 * ordering (collection.hpp:134-168). */
int ssj_synth_collection(const ssj_synth_config* cfg, ssj_collection** out);
/* preprocess_precoded (collection.hpp:134-168) of records rec_tokens[rec_offsets[i]..[i+1]). */
int ssj_preprocess_precoded(const uint32_t* rec_tokens, const uint64_t* rec_offsets,
                            uint64_t n_records, ssj_collection** out);
int ssj_collection_sizes(const ssj_collection* c, uint64_t* n_sets, uint64_t* n_tokens,
                         uint64_t* dropped_empty);
int ssj_collection_copy(const ssj_collection* c, uint32_t* tokens, uint32_t* offsets,
                        uint32_t* original_id);
void ssj_collection_free(ssj_collection* c);

/* ---- the join driver (pipeline.hpp:150-361, run_join) ------------------------------------ */
/* PipelineConfig::chunk_observer (pipeline.hpp:42-43): called on the dispatcher thread
 * for every verified chunk; flags is NULL in Count mode. */
typedef void (*ssj_chunk_observer)(void* user, const uint32_t* C, uint64_t nC,
                                   const uint32_t* C_O, uint64_t nCO, const uint8_t* flags,
                                   uint64_t count);

/* PipelineConfig (pipeline.hpp:36-51) + device knobs. */
typedef struct {
    int32_t algorithm;        /* default SSJ_ALG_PPJOIN */
    int32_t mode;             /* default SSJ_MODE_COUNT */
    uint64_t chunk_budget;    /* M_c bytes, default 64 MiB; UINT64_MAX = one chunk */
    ssj_strategy strategy;    /* default {Auto, 32} */
    uint32_t workers;         /* validated >= 1 like the reference; the grid replaces the pool */
    int32_t device;           /* CUDA device of the verification engine */
    uint32_t filter_threads;  /* H0 generation threads; 1 = the reference's sequential loop;
                                 SSJ_FILTER_ON_GPU = generation on the engine's device
                                 (AllPairs / PPJoin: the whole join runs as ssj_gpu_join) */
    uint32_t reserved;
    ssj_chunk_observer observer;
    void* observer_user;
    const int32_t* devices;   /* nullable: verification on these GPUs (ssj_engine_create_multi);
                                 `device` is used when NULL */
    uint32_t n_devices;
    uint32_t max_inflight;    /* chunks the dispatcher keeps on the GPU at once: 1 (default) is
                                 the reference's rendezvous (<= 2 chunks live, pipeline.hpp:
                                 105-141); 2 submits chunk k+1 before waiting for chunk k
                                 (<= 3 live) */
} ssj_join_config;

/* JoinReport (pipeline.hpp:63-75) + PhaseTimings (:53-58) + ours. */
typedef struct {
    uint64_t count;
    uint64_t chunk_count;
    uint64_t candidate_count;
    uint64_t host_verified_pairs;
    uint64_t max_live_candidate_bytes;
    uint64_t pairs_verified;
    uint64_t early_exit_prunes;
    uint64_t comparison_budget_violations;
    uint64_t n_pairs;
    ssj_strategy resolved_strategy;
    double filtering_ms;
    double serialization_ms;  /* includes hand-off back-pressure, as in the reference */
    double verification_ms;   /* dispatcher busy time in verify_chunk */
    double join_ms;
    double handoff_wait_ms;   /* ours: the part of serialization_ms spent blocked in put() */
    double setup_ms;          /* ours: engine creation incl. the one-time collection upload
                                 (before join_ms starts, like pipeline.hpp:314) */
} ssj_join_report;

#define SSJ_FILTER_ON_GPU 0xFFFFFFFFu

typedef struct ssj_join_result ssj_join_result;
/* Fills the reference's PipelineConfig defaults. */
void ssj_join_config_init(ssj_join_config* cfg);
/* run_join(collection, pred, config): H0 = caller thread (generation + serialization into
 * pinned chunk buffers), H1 = dispatcher (ssj_verify_chunk on the GPU), H2 = pair decoding.
 * original_id may be NULL (identity). */
int ssj_run_join(const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                 const uint32_t* original_id, const ssj_predicate* pred,
                 const ssj_join_config* cfg, ssj_join_result** out);
int ssj_join_result_report(const ssj_join_result* r, ssj_join_report* report);
/* Result pairs (r_id, s_id), r_id > s_id, original ids, unsorted (like JoinReport::pairs). */
int ssj_join_result_pairs(const ssj_join_result* r, uint32_t* pairs /* 2 * n_pairs */);
void ssj_join_result_free(ssj_join_result* r);

/* ---- candidate generation + join on the GPU ------------------- */
/*
 * AllPairs / PPJoin candidates of probes [probe_begin, probe_end) generated on the engine's
 * device from its resident collection (static index over all index prefixes, built once per
 * engine): the same stream as ssj_generate_candidates / the reference generators
 * (joiners.hpp:47-102), returned in host buffers. *nC_out / *nCO_out receive the sizes;
 * SSJ_ERR_RUNTIME when a capacity is too small (sizes still reported). The collection must be
 * in the reference's preprocessed order (sizes non-decreasing, collection.hpp:115-119),
 * else SSJ_ERR_INVALID_ARGUMENT. GroupJoin (whole collection only): its phase-1 stream
 * (groupjoin_generate's sink batches, joiners.hpp:160-171).
 */
int ssj_gpu_generate_candidates(ssj_engine* e, int32_t algorithm, uint32_t probe_begin,
                                uint32_t probe_end, uint32_t* C_out, uint64_t C_cap,
                                uint64_t* nC_out, uint32_t* C_O_out, uint64_t C_O_cap,
                                uint64_t* nCO_out);

typedef struct {
    uint64_t count;            /* qualifying pairs */
    uint64_t candidate_count;  /* candidates generated and verified */
    uint64_t intra_group_pairs; /* GroupJoin phase-2 pairs (the reference's host-verified pairs) */
    uint64_t chunk_count;      /* device-resident chunks */
    double index_ms;           /* one-time static index build (0 when cached) */
    double filtering_ms;       /* candidate generation (bounds + generate + compact) */
    double verification_ms;    /* verification kernels + pair decoding */
    double join_ms;            /* wall time of the call */
} ssj_gpu_join_report;

/*
 * Self-join run entirely on the engine's device: candidate generation (AllPairs / PPJoin /
 * GroupJoin) in probe (group) blocks of at most max_chunk_candidates candidate upper bound
 * (0 = 256M), each block verified in place by the strategy-A kernels; GroupJoin's
 * intra-group pairs (phase 2) are generated and verified on the device too. Pairs mode (pairs_out != NULL): qualifying pairs as
 * (max(orig), min(orig)) original ids (ssj_engine_set_original_ids; identity by default)
 * sorted like write_pairs (report.hpp:39-42); *n_pairs = their number (SSJ_ERR_RUNTIME when
 * pairs_cap is smaller). Count mode: pairs_out == NULL.
 */
int ssj_gpu_join(ssj_engine* e, int32_t algorithm, uint64_t max_chunk_candidates,
                 uint32_t* pairs_out, uint64_t pairs_cap, uint64_t* n_pairs,
                 ssj_gpu_join_report* report);
/* Shard `shard` of `n_shards` of the same join (multi-GPU: one engine per device, no
 * exchange step): the probes are cut into n_shards contiguous ranges of equal candidate
 * upper bound; the shards' pairs are disjoint and their union is ssj_gpu_join's.
 * GroupJoin runs as one shard. */
int ssj_gpu_join_shard(ssj_engine* e, int32_t algorithm, uint32_t shard, uint32_t n_shards,
                       uint64_t max_chunk_candidates, uint32_t* pairs_out, uint64_t pairs_cap,
                       uint64_t* n_pairs, ssj_gpu_join_report* report);

/* ---- diagnostics -------------------------------------------------------------------- */
/* Streaming read bandwidth (GB/s) of a `bytes` device buffer read `reps` times with 16-byte
 * loads: with bytes < L2 (126 MB) it measures L2-resident reads, with bytes >> L2 HBM reads.
 * Used by bench.py for the roofline denominators of L2-resident working sets. */
int ssj_measure_read_bandwidth(int device, uint64_t bytes, uint32_t reps, double* gbs);

/* ---- pinned host buffers (ChunkBuilder storage; double-buffered by the driver) ------- */
void* ssj_host_alloc(size_t bytes);
void ssj_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif /* SSJOIN_B200_H */
