// host_join.hpp -- internal declarations of the host-side join pieces.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <vector>

#include "host_common.hpp"

namespace ssjh {

struct CandidateStream {
    std::vector<uint32_t> C;
    std::vector<uint32_t> C_O;  // (probe, end) per non-empty batch, one unbounded chunk
};

struct StaticIndex;

// Parallel AllPairs / PPJoin: a static index over the index-prefixes of the first
// `index_sets` sets, then any probe window [lo, hi) with hi <= index_sets.
class ParallelGenerator {
public:
    ParallelGenerator(const CollView& c, const ssj_predicate& p, int algorithm,
                      uint32_t index_sets, unsigned threads);
    ~ParallelGenerator();
    int generate(uint32_t probe_begin, uint32_t probe_end, CandidateStream* out);

private:
    CollView c_;
    ssj_predicate p_;
    bool positional_;
    uint32_t universe_ = 0;
    unsigned threads_ = 1;
    std::unique_ptr<StaticIndex> idx_;
};

// Parallel AllPairs / PPJoin over probes [probe_begin, probe_end): identical stream to the
// reference's sequential generator restricted to those probes.
int generate_candidates(const CollView& c, const ssj_predicate& p, int algorithm,
                        uint32_t probe_begin, uint32_t probe_end, unsigned threads,
                        CandidateStream* out);

// The reference's sequential generators (joiners.hpp:47-183) with its exact control flow:
// sink(probe, candidates, k) per non-empty batch; host_verifier(a, b) for GroupJoin's
// intra-group pairs.
int generate_sequential(const CollView& c, const ssj_predicate& p, int algorithm,
                        const std::function<void(uint32_t, const uint32_t*, size_t)>& sink,
                        const std::function<void(uint32_t, uint32_t)>& host_verifier);

}  // namespace ssjh
