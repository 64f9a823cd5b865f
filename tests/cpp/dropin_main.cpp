// dropin_main.cpp -- the drop-in check, compiled against the UNMODIFIED reference headers
// (read-only, /root/reference/proj/include) and our C++ wrapper + C ABI:
// GpuVerificationEngine must return exactly what ssjoin::VerificationEngine returns on the
// reference's own candidate chunks, and decode_pairs (pipeline.hpp:79-92) over its flags
// must give the brute-force oracle's pairs (oracle.hpp:36-67).
// Built by `make -C oracle dropin` into oracle/_ref/dropin_test; run by
// tests/test_gpu_dropin.py on a GPU box. Exit code 0 = all checks passed.
#include <algorithm>
#include <cstdio>
#include <vector>

#include "ssjoin/chunk.hpp"
#include "ssjoin/joiners.hpp"
#include "ssjoin/oracle.hpp"
#include "ssjoin/pipeline.hpp"
#include "ssjoin/verify.hpp"
#include "ssjoin_b200/gpu_verification_engine.hpp"

using namespace ssjoin;

static int failures = 0;
#define EXPECT(cond, ...)                        \
    do {                                         \
        if (!(cond)) {                           \
            ++failures;                          \
            std::printf("FAIL: " __VA_ARGS__);   \
            std::printf("\n");                   \
        }                                        \
    } while (0)

int main() {
    WorkerPool pool(4);
    int checks = 0;
    for (std::uint64_t seed : {41ull, 42ull, 43ull, 101ull, 777ull}) {
        SynthConfig cfg;
        cfg.sets = seed == 777 ? 2000 : 400;
        cfg.min_size = 1;
        cfg.max_size = seed == 43 ? 120 : 40;
        cfg.universe = seed == 777 ? 400 : 200;
        cfg.zipf_tokens = seed == 777;
        cfg.duplicate_fraction = 0.2;
        auto records = synth_collection(seed, cfg);
        auto dict = Dictionary::build(records);
        auto c = preprocess(records, dict);
        for (auto [num, den] : {std::pair<std::uint64_t, std::uint64_t>{1, 2}, {7, 10}, {9, 10}}) {
            SimilarityPredicate pred;
            pred.threshold = {num, den};
            ChunkBuilder builder;
            ppjoin_generate(c, pred, [&](const CandidateBatch& b) { builder.append(b.probe, b.candidates); });
            if (builder.empty()) builder.append(0, {});
            auto chunk = builder.seal();
            auto truth = brute_force_join(c, pred);
            for (auto kind : {StrategyKind::A, StrategyKind::B, StrategyKind::C, StrategyKind::Auto}) {
                for (std::uint32_t group : {1u, 32u, 128u}) {
                    VerificationEngine ref(c, pred, OutputMode::Pairs, {kind, group});
                    GpuVerificationEngine gpu(c, pred, OutputMode::Pairs, {kind, group});
                    VerifyStats rs, gs;
                    auto ro = ref.verify_chunk(chunk, pool, &rs);
                    auto go = gpu.verify_chunk(chunk, pool, &gs);
                    ++checks;
                    EXPECT(go.flags == ro.flags, "flags seed=%llu t=%llu/%llu kind=%d B=%u",
                           (unsigned long long)seed, (unsigned long long)num,
                           (unsigned long long)den, (int)kind, group);
                    EXPECT(go.count == ro.count && go.count == truth.count(), "count");
                    // resolved exactly like the reference (verify.hpp:249-253), Auto included
                    EXPECT(gpu.strategy().kind == ref.strategy().kind &&
                               gpu.strategy().group_size == ref.strategy().group_size,
                           "resolved strategy kind=%d B=%u", (int)kind, group);
                    // stats equal for every strategy (C, and Auto resolved to C, record none)
                    EXPECT(gs.pairs_verified.load() == rs.pairs_verified.load() &&
                               gs.early_exit_prunes.load() == rs.early_exit_prunes.load() &&
                               gs.comparison_budget_violations.load() ==
                                   rs.comparison_budget_violations.load(),
                           "stats kind=%d B=%u", (int)kind, group);
                    auto got = decode_pairs(chunk, go.flags, c.original_id);
                    std::sort(got.begin(), got.end());
                    std::vector<ResultPair> want;
                    for (const auto& p : truth.pairs) {
                        auto a = c.original_id[p.r], b = c.original_id[p.s];
                        want.emplace_back(std::max(a, b), std::min(a, b));
                    }
                    std::sort(want.begin(), want.end());
                    EXPECT(got == want, "pairs");
                }
            }
            // Count mode: no flags, same count (test_verify.cpp:198-203)
            GpuVerificationEngine counter(c, pred, OutputMode::Count, {StrategyKind::B, 8});
            auto co = counter.verify_chunk(chunk, pool);
            EXPECT(co.flags.empty() && co.count == truth.count(), "count mode");
        }
    }
    // Error behaviour: out-of-range set index throws std::out_of_range (collection.hpp:87)
    {
        Collection c;
        c.tokens = {1, 2, 3};
        c.offsets = {0, 3};
        c.original_id = {0};
        SimilarityPredicate pred;
        pred.threshold = {1, 2};
        GpuVerificationEngine gpu(c, pred, OutputMode::Pairs, {StrategyKind::A, 1});
        CandidateChunk bad;
        bad.C = {5};
        bad.C_O = {0, 1};
        bool threw = false;
        try {
            gpu.verify_chunk(bad, pool);
        } catch (const std::out_of_range&) {
            threw = true;
        }
        EXPECT(threw, "out_of_range");
    }
    std::printf("%s: %d engine comparisons, %d failures\n", failures ? "DROPIN FAILED" : "DROPIN OK",
                checks, failures);
    return failures ? 1 : 0;
}
