// gpu_filter.cuh -- AllPairs / PPJoin candidate generation on the GPU.
//
// The reference generates candidates on one host thread with an incremental inverted index
// (joiners.hpp:47-102): probe i looks up the postings of its probe-prefix tokens among the
// index-prefixes of sets 0..i-1 (appended in set order), keeps sets passing the length filter,
// and deduplicates with epoch marks (first occurrence wins, joiners.hpp:28-41, :62-66).
//
// On the device the index is static (all sets' index prefixes, postings set-ascending, built
// once by a stable radix sort), so every probe is independent:
//   * postings of token t usable by probe i are one contiguous range: sets >= S_min (the
//     collection is size-ascending, so the length filter is a lower bound on the set id) and
//     < i (the incremental index holds sets 0..i-1 only) -- two binary searches;
//   * s is emitted at its first prefix position p: s is a duplicate at p iff one of its
//     index-prefix tokens u < r[p] also belongs to r -- checked against r's sorted tokens;
//   * PPJoin applies the positional filter at that first match (joiners.hpp:92-95).
// The emitted stream -- probe order, prefix-position order, posting order -- is identical to
// the reference's batch for batch (tests compare it with the reference's golden streams).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ssj_device.cuh"
#include "verify_kernels.cuh"

namespace ssjb {

// Device-resident static index over a collection's index prefixes.
struct FilterIndex {
    uint32_t* head = nullptr;   // [universe + 1] posting offsets per token
    uint2* post = nullptr;      // {set, position in the set} per posting, set-ascending per token
    uint64_t n_post = 0;
    uint32_t universe = 0;
    uint32_t n_sets = 0;
    int algorithm = 0;          // SSJ_ALG_ALLPAIRS / SSJ_ALG_PPJOIN
    PredDev pred{};
    const uint32_t* tokens = nullptr;  // padded CSR (engine-owned)
    const uint2* sets = nullptr;       // {pos8, size} (engine-owned)
    const uint4* heads = nullptr;      // packed head records (engine-owned, nullable)
    unsigned long long* work = nullptr;  // generate_kernel's probe counter (dynamic schedule)
};

// Build the index (synchronous on `st`). Returns cudaSuccess or the first error.
cudaError_t filter_index_build(FilterIndex* ix, const uint32_t* d_tokens, const uint2* d_sets,
                               uint32_t n_sets, const PredDev& pred, int algorithm,
                               cudaStream_t st);
void filter_index_free(FilterIndex* ix);

// Upper bound on probe i's candidates (sum of its posting ranges) for probes [a, b):
// d_bound[k] = bound of probe a + k.
cudaError_t filter_bounds(const FilterIndex& ix, uint32_t a, uint32_t b,
                          unsigned long long* d_bound, cudaStream_t st);

// Candidates of probes [a, b) written at d_C + (d_base[k] - base0) (d_base: exclusive scan
// of the bounds); d_count[k] receives the number emitted for probe a + k, d_flag[k] = count > 0.
cudaError_t filter_generate(const FilterIndex& ix, uint32_t a, uint32_t b,
                            const unsigned long long* d_base, unsigned long long base0,
                            uint32_t* d_C, unsigned long long* d_count, uint32_t* d_flag,
                            cudaStream_t st);

// Compact [a, b)'s per-probe candidates into the chunk format (chunk.hpp:20-28): C contiguous,
// C_O = (probe, cumulative end) for non-empty probes only (joiners.hpp:70). d_out_base =
// exclusive scan of d_count, d_slot = exclusive scan of d_flag.
cudaError_t filter_compact(uint32_t a, uint32_t b, const unsigned long long* d_base,
                           unsigned long long base0, const uint32_t* d_C,
                           const unsigned long long* d_count,
                           const unsigned long long* d_out_base, const uint32_t* d_slot,
                           uint32_t* d_outC, uint32_t* d_outCO, cudaStream_t st);

}  // namespace ssjb

namespace ssjb {

// ---- GroupJoin (joiners.hpp:111-183) ---------------------------------------------------------
// Groups: maximal runs of consecutive sets with equal size, equal probe-prefix length and
// equal probe prefix (the collection order puts them next to each other). The reference
// filters the groups' representatives like PPJoin and expands matched group pairs to member
// pairs (phase 1); pairs inside a group (phase 2) are verified separately.
struct GroupIndex {
    uint32_t n_groups = 0;
    uint32_t* first = nullptr;   // [n_groups] first member (the representative)
    uint32_t* count = nullptr;   // [n_groups] members
    uint2* fc = nullptr;         // [n_groups] {first, count}: one gather per matched group
    uint2* rep = nullptr;        // [n_groups] the representative's {pos8, size}
    uint4* rep_heads = nullptr;  // [2 n_groups] the representative's head record (nullable)
    FilterIndex ix;              // PPJoin index over the representatives
};

cudaError_t group_index_build(GroupIndex* gi, const uint32_t* d_tokens, const uint2* d_sets,
                              const uint4* d_heads, uint32_t n_sets, const PredDev& pred,
                              cudaStream_t st);
void group_index_free(GroupIndex* gi);

// Phase-1 sizes of groups [a, b) from their matched lists (d_M at d_base[k] - base0, d_mcnt[k]
// groups each): d_per[k] = candidates per member (sum of the matched groups' sizes),
// d_cand[k] = members * per (0 when nothing matched), d_nbat[k] = batches (members or 0).
cudaError_t group_sizes(const GroupIndex& gi, uint32_t a, uint32_t b,
                        const unsigned long long* d_base, unsigned long long base0,
                        const uint32_t* d_M, const unsigned long long* d_mcnt,
                        unsigned long long* d_per, unsigned long long* d_cand, uint32_t* d_nbat,
                        cudaStream_t st);

// Phase-1 stream of groups [a, b): every member of group g is a probe whose candidates are
// the members of g's matched groups in matched order (joiners.hpp:160-170). d_coff / d_soff:
// exclusive scans of d_cand / d_nbat.
cudaError_t group_expand(const GroupIndex& gi, uint32_t a, uint32_t b,
                         const unsigned long long* d_base, unsigned long long base0,
                         const uint32_t* d_M, const unsigned long long* d_mcnt,
                         const unsigned long long* d_per, const unsigned long long* d_coff,
                         const uint32_t* d_soff, uint32_t* d_C, uint32_t* d_CO, cudaStream_t st);

// Phase-2 chunk of groups [a, b) (joiners.hpp:175-179): probe first+i (i >= 1) with candidates
// first..first+i-1. d_coff / d_soff: exclusive scans of c(c-1)/2 and c-1 per group.
cudaError_t group_intra(const GroupIndex& gi, uint32_t a, uint32_t b,
                        const unsigned long long* d_coff, const uint32_t* d_soff,
                        uint32_t* d_C, uint32_t* d_CO, cudaStream_t st);
// per group of [a, b): d_icand[k] = c(c-1)/2, d_islc[k] = c - 1 (c = members)
cudaError_t group_intra_sizes(const GroupIndex& gi, uint32_t a, uint32_t b,
                              unsigned long long* d_icand, uint32_t* d_islc, cudaStream_t st);

}  // namespace ssjb
