// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim that compiles the UNMODIFIED reference headers
// (/root/reference/proj/include/ssjoin/*.hpp, read-only, never copied) into
// oracle/_ref/libssjref.so (recipe: oracle/Makefile, target `ref`). It is used to
//   * generate the golden vectors under tests/golden/ (tests/golden/make_golden.py),
//   * cross-check the C restatement (oracle/ssj_oracle.c) in tests when present,
//   * time the reference CPU verification as bench.py's cpu_baseline / --impl reference.
// Nothing in the product (paper_1812_09141_b200/) links or loads this library.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "ssjoin/chunk.hpp"
#include "ssjoin/collection.hpp"
#include "ssjoin/joiners.hpp"
#include "ssjoin/oracle.hpp"
#include "ssjoin/pipeline.hpp"
#include "ssjoin/similarity.hpp"
#include "ssjoin/verify.hpp"
#include "ssjoin/worker_pool.hpp"

using namespace ssjoin;

namespace {

thread_local std::string g_err;

SimilarityPredicate make_pred(int fn, std::uint64_t num, std::uint64_t den, std::uint64_t ovt) {
    SimilarityPredicate p;
    p.function = static_cast<SimilarityFunction>(fn);
    p.threshold = {num, den};
    p.overlap_threshold = ovt;
    return p;
}

struct RefChunks {
    std::vector<CandidateChunk> chunks;
    std::vector<std::vector<std::uint8_t>> flags;
    std::vector<std::uint64_t> counts;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- collections -------------------------------------------------------------------
struct ref_coll {
    Collection c;
};

// oracle.hpp:83-125 synth_collection, then Dictionary::build + preprocess
// (collection.hpp:27-52, :99-131): the reference's own test-fixture path (helpers.hpp:25-29).
ref_coll* ref_synth(std::uint64_t seed, std::uint64_t sets, std::uint32_t min_size,
                    std::uint32_t max_size, int zipf_sizes, double size_skew,
                    std::uint32_t universe, int zipf_tokens, double token_skew,
                    double duplicate_fraction) {
    try {
        SynthConfig cfg;
        cfg.sets = sets;
        cfg.min_size = min_size;
        cfg.max_size = max_size;
        cfg.zipf_sizes = zipf_sizes != 0;
        cfg.size_skew = size_skew;
        cfg.universe = universe;
        cfg.zipf_tokens = zipf_tokens != 0;
        cfg.token_skew = token_skew;
        cfg.duplicate_fraction = duplicate_fraction;
        auto records = synth_collection(seed, cfg);
        auto dict = Dictionary::build(records);
        auto* h = new ref_coll;
        h->c = preprocess(records, dict);
        return h;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// Verbatim collection (helpers.hpp:15-23 from_sets semantics when original_id is null).
ref_coll* ref_coll_from_csr(const std::uint32_t* tokens, const std::uint32_t* offsets,
                            std::uint32_t n_sets, const std::uint32_t* original_id) {
    auto* h = new ref_coll;
    h->c.tokens.assign(tokens, tokens + offsets[n_sets]);
    h->c.offsets.assign(offsets, offsets + n_sets + 1);
    h->c.original_id.resize(n_sets);
    for (std::uint32_t i = 0; i < n_sets; ++i)
        h->c.original_id[i] = original_id ? original_id[i] : i;
    return h;
}

void ref_coll_sizes(const ref_coll* h, std::uint64_t* n_sets, std::uint64_t* n_tokens) {
    *n_sets = h->c.size();
    *n_tokens = h->c.tokens.size();
}

void ref_coll_copy(const ref_coll* h, std::uint32_t* tokens, std::uint32_t* offsets,
                   std::uint32_t* original_id) {
    std::memcpy(tokens, h->c.tokens.data(), h->c.tokens.size() * 4);
    std::memcpy(offsets, h->c.offsets.data(), h->c.offsets.size() * 4);
    std::memcpy(original_id, h->c.original_id.data(), h->c.original_id.size() * 4);
}

void ref_coll_free(ref_coll* h) { delete h; }

// ---- similarity / merge primitives ---------------------------------------------------
std::uint64_t ref_equivalent_overlap(int fn, std::uint64_t num, std::uint64_t den,
                                     std::uint64_t ovt, std::uint64_t r, std::uint64_t s) {
    return equivalent_overlap(make_pred(fn, num, den, ovt), r, s);
}

int ref_meets_threshold(int fn, std::uint64_t num, std::uint64_t den, std::uint64_t ovt,
                        std::uint64_t o, std::uint64_t r, std::uint64_t s) {
    return meets_threshold(make_pred(fn, num, den, ovt), o, r, s) ? 1 : 0;
}

int ref_threshold_parse(const char* text, std::uint64_t* num, std::uint64_t* den) {
    try {
        auto t = Threshold::parse(text);
        *num = t.num;
        *den = t.den;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

void ref_verify_pair_count(const std::uint32_t* r, std::uint64_t m, const std::uint32_t* s,
                           std::uint64_t n, std::uint64_t required, std::uint64_t* overlap,
                           int* met, std::uint32_t* comparisons) {
    auto res = verify_pair_count({r, m}, {s, n}, required);
    *overlap = res.overlap;
    *met = res.met ? 1 : 0;
    *comparisons = res.comparisons;
}

void ref_intersect_path_partitions(const std::uint32_t* r, std::uint64_t m,
                                   const std::uint32_t* s, std::uint64_t n,
                                   std::uint32_t workers, std::uint32_t* out /*3*workers*/,
                                   std::uint64_t* counts /*workers*/) {
    auto parts = intersect_path_partitions({r, m}, {s, n}, workers);
    for (std::uint32_t k = 0; k < workers; ++k) {
        out[3 * k] = parts[k].start_r;
        out[3 * k + 1] = parts[k].start_s;
        out[3 * k + 2] = parts[k].hops;
        counts[k] = partition_count({r, m}, {s, n}, parts[k]);
    }
}

// ---- worker pool + verification engine (the CPU baseline) ------------------------------
struct ref_pool {
    std::unique_ptr<WorkerPool> pool;
};

ref_pool* ref_pool_create(unsigned workers) {
    auto* p = new ref_pool;
    p->pool = std::make_unique<WorkerPool>(workers ? workers : std::thread::hardware_concurrency());
    return p;
}

unsigned ref_pool_workers(const ref_pool* p) { return p->pool->workers(); }
void ref_pool_free(ref_pool* p) { delete p; }
unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// VerificationEngine(coll, pred, mode, {kind, group}).verify_chunk(chunk, pool, &stats)
// (verify.hpp:241-275). flags may be null (Count mode). stats: 3 x u64 or null.
int ref_verify_chunk(const ref_coll* h, ref_pool* pool, int fn, std::uint64_t num,
                     std::uint64_t den, std::uint64_t ovt, int kind, std::uint32_t group,
                     int pairs_mode, const std::uint32_t* C, std::uint64_t nC,
                     const std::uint32_t* C_O, std::uint64_t nCO, std::uint8_t* flags,
                     std::uint64_t* count, std::uint64_t* stats, int* resolved_kind,
                     std::uint32_t* resolved_group) {
    try {
        CandidateChunk chunk;
        chunk.C.assign(C, C + nC);
        chunk.C_O.assign(C_O, C_O + nCO);
        Strategy st{static_cast<StrategyKind>(kind), group};
        VerificationEngine engine(h->c, make_pred(fn, num, den, ovt),
                                  pairs_mode ? OutputMode::Pairs : OutputMode::Count, st);
        if (resolved_kind) *resolved_kind = static_cast<int>(engine.strategy().kind);
        if (resolved_group) *resolved_group = engine.strategy().group_size;
        VerifyStats vs;
        auto out = engine.verify_chunk(chunk, *pool->pool, &vs);
        *count = out.count;
        if (flags && pairs_mode) std::memcpy(flags, out.flags.data(), out.flags.size());
        if (stats) {
            stats[0] = vs.pairs_verified.load();
            stats[1] = vs.early_exit_prunes.load();
            stats[2] = vs.comparison_budget_violations.load();
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Timed variant for the CPU baseline: the chunk is decoded into a CandidateChunk once
// (outside the timing), then verify_chunk is called `reps` times; returns best seconds.
// flags (nullable, Pairs mode): the flags of the last run, copied after its timing.
double ref_time_verify_chunk(const ref_coll* h, ref_pool* pool, int fn, std::uint64_t num,
                             std::uint64_t den, std::uint64_t ovt, int kind,
                             std::uint32_t group, int pairs_mode, const std::uint32_t* C,
                             std::uint64_t nC, const std::uint32_t* C_O, std::uint64_t nCO,
                             int reps, std::uint64_t* count, std::uint8_t* flags) {
    try {
        CandidateChunk chunk;
        chunk.C.assign(C, C + nC);
        chunk.C_O.assign(C_O, C_O + nCO);
        VerificationEngine engine(h->c, make_pred(fn, num, den, ovt),
                                  pairs_mode ? OutputMode::Pairs : OutputMode::Count,
                                  {static_cast<StrategyKind>(kind), group});
        double best = -1;
        for (int i = 0; i < reps; ++i) {
            auto t0 = std::chrono::steady_clock::now();
            auto out = engine.verify_chunk(chunk, *pool->pool);
            double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            *count = out.count;
            if (best < 0 || sec < best) best = sec;
            if (flags && pairs_mode && i + 1 == reps)  // the last run's flags (outside the timing)
                std::memcpy(flags, out.flags.data(), out.flags.size());
        }
        return best;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ---- the reference join (pipeline.hpp:150-361) -------------------------------------------
struct ref_join {
    JoinReport report;
    RefChunks chunks;  // recorded through PipelineConfig::chunk_observer (pipeline.hpp:43)
};

// algorithm: 0 AllPairs, 1 PPJoin, 2 GroupJoin. record_chunks: keep every verified chunk.
ref_join* ref_run_join(const ref_coll* h, int fn, std::uint64_t num, std::uint64_t den,
                       std::uint64_t ovt, int algorithm, std::uint64_t budget, int kind,
                       std::uint32_t group, int pairs_mode, unsigned workers,
                       int record_chunks) {
    try {
        auto* j = new ref_join;
        PipelineConfig cfg;
        cfg.algorithm = static_cast<Algorithm>(algorithm);
        cfg.chunk_budget = budget;
        cfg.strategy = {static_cast<StrategyKind>(kind), group};
        cfg.mode = pairs_mode ? OutputMode::Pairs : OutputMode::Count;
        cfg.workers = workers;
        if (record_chunks) {
            cfg.chunk_observer = [j](const CandidateChunk& c, const VerificationOutput& o) {
                j->chunks.chunks.push_back(c);
                j->chunks.flags.push_back(o.flags);
                j->chunks.counts.push_back(o.count);
            };
        }
        j->report = run_join(h->c, make_pred(fn, num, den, ovt), cfg);
        return j;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// report fields: count, chunk_count, candidate_count, host_verified_pairs,
// max_live_candidate_bytes, pairs_verified, early_exit_prunes,
// comparison_budget_violations, n_pairs, resolved kind, resolved group
void ref_join_report(const ref_join* j, std::uint64_t* out /*11*/, double* timings /*4*/) {
    const auto& r = j->report;
    out[0] = r.count;
    out[1] = r.chunk_count;
    out[2] = r.candidate_count;
    out[3] = r.host_verified_pairs;
    out[4] = r.max_live_candidate_bytes;
    out[5] = r.pairs_verified;
    out[6] = r.early_exit_prunes;
    out[7] = r.comparison_budget_violations;
    out[8] = r.pairs.size();
    out[9] = static_cast<std::uint64_t>(r.resolved_strategy.kind);
    out[10] = r.resolved_strategy.group_size;
    timings[0] = r.timings.filtering_ms;
    timings[1] = r.timings.serialization_ms;
    timings[2] = r.timings.verification_ms;
    timings[3] = r.timings.join_ms;
}

// pairs sorted ascending (report.hpp:39-42 write_pairs order), 2 x u32 each
void ref_join_pairs(const ref_join* j, std::uint32_t* out) {
    auto pairs = j->report.pairs;
    std::sort(pairs.begin(), pairs.end());
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        out[2 * i] = pairs[i].first;
        out[2 * i + 1] = pairs[i].second;
    }
}

// pairs in JoinReport::pairs order (H2 decode order, pipeline.hpp:79-92 / :189-211)
void ref_join_pairs_unsorted(const ref_join* j, std::uint32_t* out) {
    const auto& pairs = j->report.pairs;
    for (std::size_t i = 0; i < pairs.size(); ++i) {
        out[2 * i] = pairs[i].first;
        out[2 * i + 1] = pairs[i].second;
    }
}

std::uint64_t ref_join_chunk_count(const ref_join* j) { return j->chunks.chunks.size(); }

void ref_join_chunk_sizes(const ref_join* j, std::uint64_t i, std::uint64_t* nC,
                          std::uint64_t* nCO, std::uint64_t* count) {
    *nC = j->chunks.chunks[i].C.size();
    *nCO = j->chunks.chunks[i].C_O.size();
    *count = j->chunks.counts[i];
}

void ref_join_chunk_copy(const ref_join* j, std::uint64_t i, std::uint32_t* C,
                         std::uint32_t* C_O, std::uint8_t* flags) {
    const auto& c = j->chunks.chunks[i];
    std::memcpy(C, c.C.data(), c.C.size() * 4);
    std::memcpy(C_O, c.C_O.data(), c.C_O.size() * 4);
    const auto& f = j->chunks.flags[i];
    if (flags && !f.empty()) std::memcpy(flags, f.data(), f.size());
}

void ref_join_free(ref_join* j) { delete j; }

// ---- brute-force oracle (oracle.hpp:36-67) ---------------------------------------------
// Returns total count; fills up to cap (r, s, overlap) triples. -1 on guard violation.
std::int64_t ref_brute_force(const ref_coll* h, int fn, std::uint64_t num, std::uint64_t den,
                             std::uint64_t ovt, std::uint32_t* out, std::uint64_t cap) {
    try {
        auto res = brute_force_join(h->c, make_pred(fn, num, den, ovt));
        for (std::size_t i = 0; i < res.pairs.size() && i < cap; ++i) {
            out[3 * i] = res.pairs[i].r;
            out[3 * i + 1] = res.pairs[i].s;
            out[3 * i + 2] = static_cast<std::uint32_t>(res.pairs[i].overlap);
        }
        return static_cast<std::int64_t>(res.pairs.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ---- candidate generators (joiners.hpp:47-183), one batch per probe ------------------
// Emits the candidate stream as one unbounded chunk (ChunkBuilder default budget) into
// caller-provided growable buffers via a two-pass protocol: pass cap=0 to learn sizes.
struct ref_cands {
    CandidateChunk chunk;
    std::vector<std::uint32_t> host_pairs;  // GroupJoin phase-2 (probe, candidate) pairs
};

ref_cands* ref_generate(const ref_coll* h, int fn, std::uint64_t num, std::uint64_t den,
                        std::uint64_t ovt, int algorithm) {
    try {
        auto* out = new ref_cands;
        ChunkBuilder builder;
        auto pred = make_pred(fn, num, den, ovt);
        auto sink = [&](const CandidateBatch& b) { builder.append(b.probe, b.candidates); };
        switch (algorithm) {
            case 0: allpairs_generate(h->c, pred, sink); break;
            case 1: ppjoin_generate(h->c, pred, sink); break;
            default:
                groupjoin_generate(h->c, pred, sink, [&](SetIndex a, SetIndex b) {
                    out->host_pairs.push_back(a);
                    out->host_pairs.push_back(b);
                });
        }
        if (!builder.empty()) out->chunk = builder.seal();
        return out;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_cands_sizes(const ref_cands* c, std::uint64_t* nC, std::uint64_t* nCO,
                     std::uint64_t* nHost) {
    *nC = c->chunk.C.size();
    *nCO = c->chunk.C_O.size();
    *nHost = c->host_pairs.size() / 2;
}

void ref_cands_copy(const ref_cands* c, std::uint32_t* C, std::uint32_t* C_O,
                    std::uint32_t* host_pairs) {
    std::memcpy(C, c->chunk.C.data(), c->chunk.C.size() * 4);
    std::memcpy(C_O, c->chunk.C_O.data(), c->chunk.C_O.size() * 4);
    if (host_pairs) std::memcpy(host_pairs, c->host_pairs.data(), c->host_pairs.size() * 4);
}

void ref_cands_free(ref_cands* c) { delete c; }

}  // extern "C"
