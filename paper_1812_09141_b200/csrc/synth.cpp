// synth.cpp -- deterministic synthetic collections for the benchmark configurations
// (real datasets are unavailable offline) and the precoded preprocessing path.
//
// The reference's fixture generator (oracle.hpp:71-125, SynthConfig) draws sizes and
// tokens from std:: distributions and copies whole records as exact duplicates. This
// generator keeps its knobs (uniform / Zipf sizes, uniform / Zipf tokens, duplicate
// fraction) and adds what SURVEY.md §7 (hard part 8) asks for: near-duplicates (a copy of
// an earlier record with a few tokens replaced) and distinct-token draws, so that post-dedup
// set sizes hit the target averages. Tokens are emitted frequency-coded (rank r of a Zipf
// draw becomes code universe-1-r, i.e. rare tokens sort first, as Dictionary::build does,
// collection.hpp:27-52), then go through preprocess_precoded (collection.hpp:134-168).
// Randomness: splitmix64-seeded xoshiro256**, one stream per record, so the output is
// independent of the thread count.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>
#include <thread>
#include <vector>

#include "host_common.hpp"

namespace {

inline uint64_t splitmix64(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

struct Rng {
    uint64_t s[4];
    explicit Rng(uint64_t seed) {
        for (auto& v : s) v = splitmix64(seed);
    }
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    uint64_t next() {
        const uint64_t result = rotl(s[1] * 5, 7) * 9;
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return result;
    }
    double uniform() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
    uint64_t below(uint64_t n) { return n ? (uint64_t)(((unsigned __int128)next() * n) >> 64) : 0; }
};

struct Zipf {
    std::vector<double> cdf;
    void init(uint32_t n, double skew) {
        cdf.resize(n);
        double acc = 0;
        for (uint32_t k = 0; k < n; ++k) {
            acc += 1.0 / std::pow(k + 1.0, skew);
            cdf[k] = acc;
        }
    }
    uint32_t sample(Rng& r) const {
        const double u = r.uniform() * cdf.back();
        return (uint32_t)(std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin());
    }
};

}  // namespace

struct ssj_collection {
    std::vector<uint32_t> tokens;
    std::vector<uint32_t> offsets{0};
    std::vector<uint32_t> original_id;
    uint64_t dropped = 0;
};

namespace {

// collection.hpp:134-168: per-record sort + dedup, drop empties, order by (size, lex, line).
ssj_collection* preprocess(std::vector<std::vector<uint32_t>>& recs, unsigned threads) {
    const size_t n = recs.size();
    {
        std::atomic<size_t> next{0};
        auto work = [&]() {
            for (;;) {
                const size_t b = next.fetch_add(4096);
                if (b >= n) break;
                for (size_t i = b; i < std::min(n, b + 4096); ++i) {
                    auto& v = recs[i];
                    std::sort(v.begin(), v.end());
                    v.erase(std::unique(v.begin(), v.end()), v.end());
                }
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < threads; ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
    }
    auto* c = new ssj_collection;
    std::vector<uint32_t> order;
    order.reserve(n);
    for (size_t i = 0; i < n; ++i) {
        if (recs[i].empty()) ++c->dropped;
        else order.push_back((uint32_t)i);
    }
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        const auto& x = recs[a];
        const auto& y = recs[b];
        if (x.size() != y.size()) return x.size() < y.size();
        if (x != y) return std::lexicographical_compare(x.begin(), x.end(), y.begin(), y.end());
        return a < b;
    });
    size_t total = 0;
    for (uint32_t i : order) total += recs[i].size();
    c->tokens.reserve(total);
    c->offsets.reserve(order.size() + 1);
    c->original_id.reserve(order.size());
    for (uint32_t i : order) {
        c->tokens.insert(c->tokens.end(), recs[i].begin(), recs[i].end());
        c->offsets.push_back((uint32_t)c->tokens.size());
        c->original_id.push_back(i);
    }
    return c;
}

}  // namespace

extern "C" {

int ssj_synth_collection(const ssj_synth_config* cfg, ssj_collection** out) {
    if (!cfg || !out) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    if (cfg->universe == 0 || cfg->min_size > cfg->max_size)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "bad synth config");
    const uint32_t n = cfg->n_sets;
    unsigned threads = cfg->threads ? cfg->threads : std::max(1u, std::thread::hardware_concurrency());
    Zipf size_z, tok_z;
    if (cfg->zipf_sizes) size_z.init(cfg->max_size - cfg->min_size + 1, cfg->size_skew);
    if (cfg->zipf_tokens) tok_z.init(cfg->universe, cfg->token_skew);
    auto draw_token = [&](Rng& r) -> uint32_t {
        if (cfg->zipf_tokens) return cfg->universe - 1 - tok_z.sample(r);  // rare first
        return (uint32_t)r.below(cfg->universe);
    };

    // Pass 1 (sequential, cheap): which records are near-copies, and of what.
    std::vector<int64_t> src(n, -1);
    {
        Rng r(cfg->seed ^ 0xD1B54A32D192ED03ull);
        for (uint32_t i = 1; i < n; ++i)
            if (cfg->duplicate_fraction > 0 && r.uniform() < cfg->duplicate_fraction)
                src[i] = (int64_t)r.below(i);
    }
    // Pass 2 (parallel): fresh records.
    std::vector<std::vector<uint32_t>> recs(n);
    {
        std::atomic<uint32_t> next{0};
        auto work = [&]() {
            std::vector<uint32_t> tmp;
            for (;;) {
                const uint32_t b = next.fetch_add(1024);
                if (b >= n) break;
                for (uint32_t i = b; i < std::min<uint32_t>(n, b + 1024); ++i) {
                    if (src[i] >= 0) continue;
                    Rng r(cfg->seed * 0x9E3779B97F4A7C15ull + i + 1);
                    const uint32_t size = cfg->zipf_sizes
                                              ? cfg->min_size + size_z.sample(r)
                                              : cfg->min_size + (uint32_t)r.below(cfg->max_size - cfg->min_size + 1);
                    auto& v = recs[i];
                    v.clear();
                    if (!cfg->distinct_tokens) {
                        for (uint32_t t = 0; t < size; ++t) v.push_back(draw_token(r));
                        continue;
                    }
                    const uint32_t want = std::min(size, cfg->universe);
                    for (int round = 0; round < 64 && v.size() < want; ++round) {
                        const size_t need = want - v.size();
                        for (size_t t = 0; t < need + need / 4 + 1; ++t) v.push_back(draw_token(r));
                        std::sort(v.begin(), v.end());
                        v.erase(std::unique(v.begin(), v.end()), v.end());
                        if (v.size() > want) {
                            // drop random extras to land exactly on `want`
                            while (v.size() > want) v.erase(v.begin() + (ptrdiff_t)r.below(v.size()));
                        }
                    }
                }
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 1; t < threads; ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
    }
    // Pass 3 (sequential, in order): near-copies of earlier records with edits.
    for (uint32_t i = 0; i < n; ++i) {
        if (src[i] < 0) continue;
        Rng r(cfg->seed * 0x2545F4914F6CDD1Dull + i + 7);
        recs[i] = recs[(size_t)src[i]];
        const uint32_t edits = cfg->max_edits ? (uint32_t)r.below(cfg->max_edits + 1) : 0;
        for (uint32_t e = 0; e < edits && !recs[i].empty(); ++e)
            recs[i][r.below(recs[i].size())] = draw_token(r);
    }
    *out = preprocess(recs, threads);
    return SSJ_OK;
}

int ssj_preprocess_precoded(const uint32_t* rec_tokens, const uint64_t* rec_offsets,
                            uint64_t n_records, ssj_collection** out) {
    if (!out || (n_records && !rec_offsets)) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    if (n_records > 0xFFFFFFFFull) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "too many records");
    std::vector<std::vector<uint32_t>> recs(n_records);
    for (uint64_t i = 0; i < n_records; ++i)
        recs[i].assign(rec_tokens + rec_offsets[i], rec_tokens + rec_offsets[i + 1]);
    *out = preprocess(recs, std::max(1u, std::thread::hardware_concurrency()));
    return SSJ_OK;
}

int ssj_collection_sizes(const ssj_collection* c, uint64_t* n_sets, uint64_t* n_tokens,
                         uint64_t* dropped) {
    if (!c) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null collection");
    if (n_sets) *n_sets = c->original_id.size();
    if (n_tokens) *n_tokens = c->tokens.size();
    if (dropped) *dropped = c->dropped;
    return SSJ_OK;
}

int ssj_collection_copy(const ssj_collection* c, uint32_t* tokens, uint32_t* offsets,
                        uint32_t* original_id) {
    if (!c) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null collection");
    if (tokens && !c->tokens.empty()) std::memcpy(tokens, c->tokens.data(), c->tokens.size() * 4);
    if (offsets) std::memcpy(offsets, c->offsets.data(), c->offsets.size() * 4);
    if (original_id && !c->original_id.empty())
        std::memcpy(original_id, c->original_id.data(), c->original_id.size() * 4);
    return SSJ_OK;
}

void ssj_collection_free(ssj_collection* c) { delete c; }

}  // extern "C"
