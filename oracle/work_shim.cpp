// work_shim.cpp -- TEST / BENCHMARK INFRASTRUCTURE ONLY.
//
// Lets bench.py's `--impl reference` arm build the benchmark workload without loading the
// product library (libssjoin_b200.so): the deterministic synthetic collection
// (paper_1812_09141_b200/csrc/synth.cpp) and the candidate batch of the GPU arm
// (candidates.cpp, parallel AllPairs / PPJoin over probe windows -- the same stream as the
// reference's allpairs_generate / ppjoin_generate, joiners.hpp:47-102) are compiled into
// oracle/_ref/libssjref.so next to the reference shim, with hidden visibility. The
// predicate arithmetic they call (ssj_equivalent_overlap, ssj_predicate_validate) is bound
// here to the reference's own similarity.hpp (equivalent_overlap :108-123, validate :74-81),
// so the workload is produced with the reference's arithmetic. No CUDA, no GPU code.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "ssjoin/similarity.hpp"

#include "../include/ssjoin_b200.h"
#include "../paper_1812_09141_b200/csrc/host_common.hpp"

namespace {
thread_local std::string g_werr;

ssjoin::SimilarityPredicate to_ref(const ssj_predicate& p) {
    ssjoin::SimilarityPredicate q;
    q.function = static_cast<ssjoin::SimilarityFunction>(p.function);
    q.threshold = {p.num, p.den};
    q.overlap_threshold = p.overlap_threshold;
    return q;
}
}  // namespace

namespace ssjh {
int set_error(int code, const std::string& msg) {
    g_werr = msg;
    return code;
}
}  // namespace ssjh

#define EXPORT __attribute__((visibility("default")))

extern "C" {

uint64_t ssj_equivalent_overlap(const ssj_predicate* p, uint64_t r, uint64_t s) {
    return ssjoin::equivalent_overlap(to_ref(*p), r, s);
}

int ssj_predicate_validate(const ssj_predicate* p) {
    if (!p) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null predicate");
    try {
        to_ref(*p).validate();
    } catch (const std::exception& e) {
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, e.what());
    }
    return SSJ_OK;
}

EXPORT const char* ref_work_last_error() { return g_werr.c_str(); }

// ssj_synth_collection (synth.cpp) -> sizes, then copy; returns an opaque handle.
EXPORT void* ref_work_synth(const ssj_synth_config* cfg, uint64_t* n_sets, uint64_t* n_tokens) {
    ssj_collection* c = nullptr;
    if (ssj_synth_collection(cfg, &c)) return nullptr;
    ssj_collection_sizes(c, n_sets, n_tokens, nullptr);
    return c;
}

EXPORT void ref_work_synth_copy(void* h, uint32_t* tokens, uint32_t* offsets,
                                uint32_t* original_id) {
    auto* c = static_cast<ssj_collection*>(h);
    ssj_collection_copy(c, tokens, offsets, original_id);
    ssj_collection_free(c);
}

// ssj_generate_candidates_windows (candidates.cpp): one chunk over the probe windows.
EXPORT void* ref_work_generate_windows(const uint32_t* tokens, const uint32_t* offsets,
                                       uint32_t n_sets, const ssj_predicate* pred,
                                       int32_t algorithm, const uint32_t* windows,
                                       uint32_t n_windows, uint32_t threads, uint64_t* nC,
                                       uint64_t* nCO) {
    ssj_candidates* c = nullptr;
    if (ssj_generate_candidates_windows(tokens, offsets, n_sets, pred, algorithm, windows,
                                        n_windows, threads, &c))
        return nullptr;
    ssj_candidates_sizes(c, nC, nCO, nullptr);
    return c;
}

EXPORT void ref_work_candidates_copy(void* h, uint32_t* C, uint32_t* C_O) {
    auto* c = static_cast<ssj_candidates*>(h);
    ssj_candidates_copy(c, C, C_O, nullptr);
    ssj_candidates_free(c);
}

}  // extern "C"
