// gpu_verification_engine.hpp -- drop-in C++ replacement for ssjoin::VerificationEngine
// (proj/include/ssjoin/verify.hpp:241-351) running on a B200 through the C ABI
// (include/ssjoin_b200.h, libssjoin_b200.so).
//
// Include AFTER the reference's "ssjoin/verify.hpp": this header uses the reference's own
// types (Collection, SimilarityPredicate, OutputMode, Strategy, CandidateChunk, WorkerPool,
// VerifyStats, VerificationOutput) so that swapping the engine is a one-line change in
// run_join (pipeline.hpp:156):
//
//     VerificationEngine engine(collection, pred, config.mode, config.strategy);
//  -> GpuVerificationEngine engine(collection, pred, config.mode, config.strategy);
//
// Semantics kept: same constructor and verify_chunk signature; Auto resolved at
// construction (verify.hpp:245) and reported by strategy(); flags only in Pairs mode, slot
// order = C order, byte-identical to the reference; count; VerifyStats recorded for
// strategies A/B only; std::invalid_argument / std::out_of_range / std::runtime_error as the
// reference would throw. verify_chunk is const and may be called from several threads at
// once, like the reference's: calls are serialised on an internal mutex (the engine's chunk
// slots and scratch are per engine). Difference: the collection is copied to the GPU at
// construction (the reference keeps a reference); there is no CPU fallback.
//
// Multi-GPU: the constructor taking a device list builds one engine over several GPUs
// (ssj_engine_create_multi: one host upload, NVLink peer fan-out of the collection); each
// chunk is split by probe-slice ranges across them and the flags come back in C order.
#pragma once

#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ssjoin_b200.h"

namespace ssjoin {

namespace gpu_detail {
inline void check(int rc) {
    if (rc == SSJ_OK) return;
    const std::string msg = ssj_last_error();
    if (rc == SSJ_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    if (rc == SSJ_ERR_OUT_OF_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error("ssjoin_b200: " + msg);
}

inline ssj_predicate to_c(const SimilarityPredicate& p) {
    ssj_predicate c{};
    c.function = static_cast<int32_t>(p.function);
    c.num = p.threshold.num;
    c.den = p.threshold.den;
    c.overlap_threshold = p.overlap_threshold;
    return c;
}
}  // namespace gpu_detail

class GpuVerificationEngine {
public:
    GpuVerificationEngine(const Collection& collection, SimilarityPredicate pred, OutputMode mode,
                          Strategy strategy, int device = 0)
        : mode_(mode) {
        const ssj_predicate p = gpu_detail::to_c(pred);
        const ssj_strategy s{static_cast<int32_t>(strategy.kind), strategy.group_size};
        const uint32_t* tokens = collection.tokens.empty() ? nullptr : collection.tokens.data();
        gpu_detail::check(ssj_engine_create(&engine_, device, tokens, collection.offsets.data(),
                                            static_cast<uint32_t>(collection.size()), &p,
                                            mode == OutputMode::Pairs ? SSJ_MODE_PAIRS
                                                                      : SSJ_MODE_COUNT,
                                            &s));
        resolve();
    }

    // One engine over several GPUs (probe-slice sharding of every chunk).
    GpuVerificationEngine(const Collection& collection, SimilarityPredicate pred, OutputMode mode,
                          Strategy strategy, const std::vector<int>& devices)
        : mode_(mode) {
        const ssj_predicate p = gpu_detail::to_c(pred);
        const ssj_strategy s{static_cast<int32_t>(strategy.kind), strategy.group_size};
        const uint32_t* tokens = collection.tokens.empty() ? nullptr : collection.tokens.data();
        gpu_detail::check(ssj_engine_create_multi(
            &engine_, devices.data(), static_cast<uint32_t>(devices.size()), tokens,
            collection.offsets.data(), static_cast<uint32_t>(collection.size()), &p,
            mode == OutputMode::Pairs ? SSJ_MODE_PAIRS : SSJ_MODE_COUNT, &s));
        resolve();
    }

    GpuVerificationEngine(const GpuVerificationEngine&) = delete;
    GpuVerificationEngine& operator=(const GpuVerificationEngine&) = delete;
    ~GpuVerificationEngine() { ssj_engine_destroy(engine_); }

    Strategy strategy() const { return strategy_; }

    // verify.hpp:257-275. The WorkerPool is accepted for signature parity: the GPU grid
    // replaces it.
    VerificationOutput verify_chunk(const CandidateChunk& chunk, WorkerPool& /*pool*/,
                                    VerifyStats* stats = nullptr) const {
        VerificationOutput out;
        if (mode_ == OutputMode::Pairs) out.flags.assign(chunk.candidate_count(), 0);
        ssj_stats st{};
        uint64_t count = 0;
        std::lock_guard<std::mutex> lock(mu_);
        gpu_detail::check(ssj_verify_chunk(engine_, chunk.C.data(), chunk.C.size(),
                                           chunk.C_O.data(), chunk.C_O.size(),
                                           out.flags.empty() ? nullptr : out.flags.data(),
                                           &count, &st));
        out.count = count;
        if (stats) {
            stats->pairs_verified.fetch_add(st.pairs_verified, std::memory_order_relaxed);
            stats->early_exit_prunes.fetch_add(st.early_exit_prunes, std::memory_order_relaxed);
            stats->comparison_budget_violations.fetch_add(st.comparison_budget_violations,
                                                          std::memory_order_relaxed);
        }
        return out;
    }

    ssj_engine* native_handle() const { return engine_; }

private:
    void resolve() {
        ssj_strategy r{};
        gpu_detail::check(ssj_engine_strategy(engine_, &r));
        strategy_ = {static_cast<StrategyKind>(r.kind), r.group_size};
    }

    mutable std::mutex mu_;
    ssj_engine* engine_ = nullptr;
    OutputMode mode_;
    Strategy strategy_;
};

}  // namespace ssjoin
