// candidates.cpp -- the CPU candidate generators that feed the verification engine
// (role H0 of the reference's join driver). Candidate streams are identical, batch for
// batch and candidate for candidate, to the reference's sequential generators
// (joiners.hpp:47-183), which the tests pin against golden streams the reference produced.
//
// B200-side addition: AllPairs and PPJoin can run on many host threads. For a probe i the
// reference consults an incremental index holding the index-prefixes of sets 0..i-1,
// appended in set order (joiners.hpp:62-68). A static index over all sets, whose posting
// lists are therefore sorted by set id, read only up to the first posting with set >= i,
// yields the same postings in the same order -- so probes are independent and the
// per-probe batches can be produced in parallel and concatenated in probe order.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <thread>
#include <vector>

#include "host_common.hpp"
#include "host_join.hpp"

namespace ssjh {

typedef unsigned __int128 u128;

static uint64_t ceil_div(u128 a, u128 b) { return (uint64_t)((a + b - 1) / b); }

uint64_t size_lower_bound(const ssj_predicate& p, uint64_t r) {
    // similarity.hpp:135-164 (min only); a zero lower bound is raised to 1 (:162)
    const uint64_t num = p.num, den = p.den;
    uint64_t lo = 0;
    switch (p.function) {
        case SSJ_JACCARD: lo = ceil_div((u128)num * r, den); break;
        case SSJ_COSINE: lo = ceil_div((u128)num * num * r, (u128)den * den); break;
        case SSJ_DICE: lo = ceil_div((u128)num * r, 2 * den - num); break;
        default: lo = p.overlap_threshold; break;
    }
    return lo == 0 ? 1 : lo;
}

PrefixLengths prefix_lengths(const ssj_predicate& p, uint32_t size) {
    // filters.hpp:148-159
    auto clamp = [size](uint64_t len) -> uint32_t {
        if (len < 1) return 1;
        return (uint32_t)std::min<uint64_t>(len, size);
    };
    PrefixLengths out;
    const uint64_t minsize = size_lower_bound(p, size);
    out.probe = clamp(minsize >= size ? 1 : size - minsize + 1);
    const uint64_t self = ssj_equivalent_overlap(&p, size, size);
    out.index = clamp(self >= size ? 1 : size - self + 1);
    return out;
}

bool positional_keep(const ssj_predicate& p, uint32_t size_r, uint32_t size_s, uint32_t pos_r,
                     uint32_t pos_s) {
    // filters.hpp:174-181 with current_overlap = 1 (joiners.hpp:94, :121)
    const uint64_t required = ssj_equivalent_overlap(&p, size_r, size_s);
    const uint64_t rest = std::min<uint64_t>(size_r - pos_r - 1, size_s - pos_s - 1);
    return 1 + rest >= required;
}

namespace {

// joiners.hpp:21-24 (size_t there): max token + 1, in 64 bits (token 0xFFFFFFFF is legal
// and gives 2^32). The generators index per-token lists by it, so a universe beyond
// kMaxUniverse is refused with std::invalid_argument (the reference would attempt a
// 2^32-entry allocation and fail with bad_alloc).
constexpr uint64_t kMaxUniverse = 1ull << 31;

uint32_t token_universe(const CollView& c) {
    const uint64_t T = c.n ? c.offsets[c.n] : 0;
    uint64_t universe = 0;
    for (uint64_t k = c.offsets[0]; k < T; ++k) universe = std::max<uint64_t>(universe, (uint64_t)c.tokens[k] + 1);
    if (universe > kMaxUniverse)
        throw std::invalid_argument("token values >= 2^31: too large a universe for the inverted index");
    return (uint32_t)universe;
}

}  // namespace

// Static inverted index: token -> postings (set, position), sets ascending.
struct StaticIndex {
    std::vector<uint64_t> head;  // universe + 1
    std::vector<uint32_t> set, pos;

    void build(const CollView& c, const ssj_predicate& p, uint32_t universe, uint32_t n_sets) {
        head.assign((size_t)universe + 1, 0);
        std::vector<uint32_t> ilen(n_sets);
        for (uint32_t i = 0; i < n_sets; ++i) {
            ilen[i] = c.size(i) ? prefix_lengths(p, c.size(i)).index : 0;
            const uint32_t* r = c.set(i);
            for (uint32_t q = 0; q < ilen[i] && q < c.size(i); ++q) ++head[r[q] + 1];
        }
        for (uint32_t t = 0; t < universe; ++t) head[t + 1] += head[t];
        set.resize(head[universe]);
        pos.resize(head[universe]);
        std::vector<uint64_t> fill(head.begin(), head.end() - 1);
        for (uint32_t i = 0; i < n_sets; ++i) {
            const uint32_t* r = c.set(i);
            for (uint32_t q = 0; q < ilen[i] && q < c.size(i); ++q) {
                const uint64_t k = fill[r[q]]++;
                set[k] = i;
                pos[k] = q;
            }
        }
    }
};

namespace {

struct Marks {
    std::vector<uint32_t> stamp;
    uint32_t epoch = 0;
    explicit Marks(size_t n) : stamp(n, 0) {}
    void next() {
        if (++epoch == 0) {  // wrapped: reset
            std::fill(stamp.begin(), stamp.end(), 0);
            epoch = 1;
        }
    }
    bool mark(uint32_t i) {
        if (stamp[i] == epoch) return false;
        stamp[i] = epoch;
        return true;
    }
};

// Candidates of probe i (joiners.hpp:58-69 AllPairs, :86-101 PPJoin).
void probe_candidates(const CollView& c, const ssj_predicate& p, const StaticIndex& idx,
                      uint32_t universe, bool positional, uint32_t i, Marks& seen,
                      std::vector<uint32_t>& out) {
    const uint32_t size_r = c.size(i);
    if (size_r == 0) return;
    const uint32_t* r = c.set(i);
    const PrefixLengths lens = prefix_lengths(p, size_r);
    const uint64_t minsize = size_lower_bound(p, size_r);
    seen.next();
    for (uint32_t q = 0; q < lens.probe; ++q) {
        const uint32_t t = r[q];
        if (t >= universe) continue;
        for (uint64_t k = idx.head[t]; k < idx.head[t + 1]; ++k) {
            const uint32_t s = idx.set[k];
            if (s >= i) break;  // postings are set-ascending: the rest were added after probe i
            const uint32_t size_s = c.size(s);
            if (size_s < minsize) continue;
            if (!positional) {
                if (seen.mark(s)) out.push_back(s);
            } else {
                if (!seen.mark(s)) continue;
                if (positional_keep(p, size_r, size_s, q, idx.pos[k])) out.push_back(s);
            }
        }
    }
}

}  // namespace

ParallelGenerator::ParallelGenerator(const CollView& c, const ssj_predicate& p, int algorithm,
                                     uint32_t index_sets, unsigned threads)
    : c_(c), p_(p), positional_(algorithm == SSJ_ALG_PPJOIN) {
    universe_ = token_universe(c);
    idx_ = std::make_unique<StaticIndex>();
    idx_->build(c, p, universe_, std::min(index_sets, c.n));
    threads_ = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
}

ParallelGenerator::~ParallelGenerator() = default;

int ParallelGenerator::generate(uint32_t probe_begin, uint32_t probe_end, CandidateStream* out) {
    probe_end = std::min(probe_end, c_.n);
    out->C.clear();
    out->C_O.clear();
    if (probe_begin >= probe_end) return SSJ_OK;
    const uint32_t span = probe_end - probe_begin;
    const uint32_t block = 256;
    const uint32_t n_blocks = (span + block - 1) / block;
    std::vector<std::vector<uint32_t>> bC(n_blocks), bCO(n_blocks);
    std::atomic<uint32_t> next{0};
    auto worker = [&]() {
        Marks seen(c_.n);
        std::vector<uint32_t> cands;
        for (;;) {
            const uint32_t b = next.fetch_add(1);
            if (b >= n_blocks) break;
            const uint32_t lo = probe_begin + b * block;
            const uint32_t hi = std::min(probe_end, lo + block);
            auto& C = bC[b];
            auto& CO = bCO[b];
            for (uint32_t i = lo; i < hi; ++i) {
                cands.clear();
                probe_candidates(c_, p_, *idx_, universe_, positional_, i, seen, cands);
                if (cands.empty()) continue;  // joiners.hpp:70: empty batches are not sunk
                C.insert(C.end(), cands.begin(), cands.end());
                CO.push_back(i);
                CO.push_back((uint32_t)C.size());  // block-local end, rebased below
            }
        }
    };
    const unsigned nt = std::min<unsigned>(threads_, n_blocks);
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    size_t totC = 0, totCO = 0;
    for (uint32_t b = 0; b < n_blocks; ++b) {
        totC += bC[b].size();
        totCO += bCO[b].size();
    }
    if (totC > 0xFFFFFFFFull)
        return set_error(SSJ_ERR_INVALID_ARGUMENT, "candidate stream exceeds u32 offsets");
    out->C.resize(totC);
    out->C_O.resize(totCO);
    uint64_t cbase = 0, cobase = 0;
    for (uint32_t b = 0; b < n_blocks; ++b) {
        if (!bC[b].empty()) std::memcpy(out->C.data() + cbase, bC[b].data(), bC[b].size() * 4);
        for (size_t k = 0; k < bCO[b].size(); k += 2) {
            out->C_O[cobase + k] = bCO[b][k];
            out->C_O[cobase + k + 1] = (uint32_t)(cbase + bCO[b][k + 1]);
        }
        cbase += bC[b].size();
        cobase += bCO[b].size();
        std::vector<uint32_t>().swap(bC[b]);
    }
    return SSJ_OK;
}

int generate_candidates(const CollView& c, const ssj_predicate& p, int algorithm,
                        uint32_t probe_begin, uint32_t probe_end, unsigned threads,
                        CandidateStream* out) {
    if (algorithm != SSJ_ALG_ALLPAIRS && algorithm != SSJ_ALG_PPJOIN)
        return set_error(SSJ_ERR_INVALID_ARGUMENT, "parallel generation supports allpairs/ppjoin");
    ParallelGenerator gen(c, p, algorithm, std::min(probe_end, c.n), threads);
    return gen.generate(probe_begin, probe_end, out);
}

// Sequential generators with the reference's exact control flow, used by the join driver.
int generate_sequential(const CollView& c, const ssj_predicate& p, int algorithm,
                        const std::function<void(uint32_t, const uint32_t*, size_t)>& sink,
                        const std::function<void(uint32_t, uint32_t)>& host_verifier) {
    const uint32_t n = c.n;
    const uint32_t universe = token_universe(c);
    if (algorithm == SSJ_ALG_ALLPAIRS || algorithm == SSJ_ALG_PPJOIN) {
        // joiners.hpp:47-102: incremental index, probe before insert
        std::vector<std::vector<std::pair<uint32_t, uint32_t>>> lists(universe);
        Marks seen(n);
        std::vector<uint32_t> cands;
        const bool positional = algorithm == SSJ_ALG_PPJOIN;
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t size_r = c.size(i);
            const uint32_t* r = c.set(i);
            const PrefixLengths lens = prefix_lengths(p, size_r);
            const uint64_t minsize = size_lower_bound(p, size_r);
            seen.next();
            cands.clear();
            for (uint32_t q = 0; q < lens.probe && q < size_r; ++q) {
                for (const auto& post : lists[r[q]]) {
                    const uint32_t size_s = c.size(post.first);
                    if (size_s < minsize) continue;
                    if (!positional) {
                        if (seen.mark(post.first)) cands.push_back(post.first);
                    } else {
                        if (!seen.mark(post.first)) continue;
                        if (positional_keep(p, size_r, size_s, q, post.second))
                            cands.push_back(post.first);
                    }
                }
            }
            if (!cands.empty()) sink(i, cands.data(), cands.size());
            for (uint32_t q = 0; q < lens.index && q < size_r; ++q)
                lists[r[q]].push_back({i, q});
        }
        return SSJ_OK;
    }
    if (algorithm != SSJ_ALG_GROUPJOIN)
        return set_error(SSJ_ERR_INVALID_ARGUMENT, "unknown algorithm");
    // joiners.hpp:111-183 GroupJoin: groups of equal size and equal probe prefix
    struct Group {
        uint32_t first, count;
    };
    std::vector<Group> groups;
    {
        uint32_t prev_size = 0, prev_len = 0;
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t size = c.size(i);
            const uint32_t plen = prefix_lengths(p, size).probe;
            bool same = false;
            if (!groups.empty() && size == prev_size && plen == prev_len) {
                const uint32_t* rep = c.set(groups.back().first);
                same = std::equal(c.set(i), c.set(i) + std::min(plen, size), rep);
            }
            if (same) {
                ++groups.back().count;
            } else {
                groups.push_back({i, 1});
                prev_size = size;
                prev_len = plen;
            }
        }
    }
    std::vector<std::vector<std::pair<uint32_t, uint32_t>>> lists(universe);
    Marks seen(groups.size());
    std::vector<uint32_t> matched, cands;
    for (uint32_t g = 0; g < groups.size(); ++g) {
        const uint32_t* rep = c.set(groups[g].first);
        const uint32_t size_r = c.size(groups[g].first);
        const PrefixLengths lens = prefix_lengths(p, size_r);
        const uint64_t minsize = size_lower_bound(p, size_r);
        seen.next();
        matched.clear();
        for (uint32_t q = 0; q < lens.probe && q < size_r; ++q) {
            for (const auto& post : lists[rep[q]]) {
                const uint32_t h = post.first;
                const uint32_t size_s = c.size(groups[h].first);
                if (size_s < minsize) continue;
                if (!seen.mark(h)) continue;
                if (positional_keep(p, size_r, size_s, q, post.second)) matched.push_back(h);
            }
        }
        if (!matched.empty()) {
            for (uint32_t m = 0; m < groups[g].count; ++m) {
                cands.clear();
                for (uint32_t h : matched)
                    for (uint32_t k = 0; k < groups[h].count; ++k) cands.push_back(groups[h].first + k);
                sink(groups[g].first + m, cands.data(), cands.size());
            }
        }
        for (uint32_t a = 1; a < groups[g].count; ++a)
            for (uint32_t b = 0; b < a; ++b) host_verifier(groups[g].first + a, groups[g].first + b);
        for (uint32_t q = 0; q < lens.index && q < size_r; ++q) lists[rep[q]].push_back({g, q});
    }
    return SSJ_OK;
}

}  // namespace ssjh

// ---- C ABI ------------------------------------------------------------------------------
struct ssj_candidates {
    ssjh::CandidateStream s;
    std::vector<uint32_t> host_pairs;
};

extern "C" {

int ssj_generate_candidates(const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                            const ssj_predicate* pred, int32_t algorithm, uint32_t probe_begin,
                            uint32_t probe_end, uint32_t threads, ssj_candidates** out) {
    if (!out || !offsets || !pred) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    int rc = ssj_predicate_validate(pred);
    if (rc) return rc;
    ssjh::CollView c{tokens, offsets, n_sets};
    auto* h = new ssj_candidates;
    try {
        if (algorithm == SSJ_ALG_GROUPJOIN || threads == 1) {
            // sequential reference control flow (GroupJoin is sequential by nature)
            probe_end = std::min(probe_end, n_sets);
            rc = ssjh::generate_sequential(
                c, *pred, algorithm,
                [&](uint32_t probe, const uint32_t* cand, size_t k) {
                    if (probe < probe_begin || probe >= probe_end) return;
                    h->s.C.insert(h->s.C.end(), cand, cand + k);
                    h->s.C_O.push_back(probe);
                    h->s.C_O.push_back((uint32_t)h->s.C.size());
                },
                [&](uint32_t a, uint32_t b) {
                    h->host_pairs.push_back(a);
                    h->host_pairs.push_back(b);
                });
        } else {
            rc = ssjh::generate_candidates(c, *pred, algorithm, probe_begin, probe_end, threads,
                                           &h->s);
        }
    } catch (const std::invalid_argument& e) {
        rc = ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        rc = ssjh::set_error(SSJ_ERR_RUNTIME, e.what());
    }
    if (rc) {
        delete h;
        return rc;
    }
    *out = h;
    return SSJ_OK;
}

int ssj_generate_candidates_windows(const uint32_t* tokens, const uint32_t* offsets,
                                    uint32_t n_sets, const ssj_predicate* pred, int32_t algorithm,
                                    const uint32_t* windows, uint32_t n_windows, uint32_t threads,
                                    ssj_candidates** out) {
    if (!out || !offsets || !pred || (n_windows && !windows))
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    int rc = ssj_predicate_validate(pred);
    if (rc) return rc;
    if (algorithm != SSJ_ALG_ALLPAIRS && algorithm != SSJ_ALG_PPJOIN)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "windows: allpairs/ppjoin only");
    uint32_t hi_max = 0;
    for (uint32_t w = 0; w < n_windows; ++w) hi_max = std::max(hi_max, std::min(windows[2 * w + 1], n_sets));
    ssjh::CollView c{tokens, offsets, n_sets};
    auto* h = new ssj_candidates;
    try {
        ssjh::ParallelGenerator gen(c, *pred, algorithm, hi_max, threads);
        ssjh::CandidateStream part;
        for (uint32_t w = 0; w < n_windows; ++w) {
            if ((rc = gen.generate(windows[2 * w], std::min(windows[2 * w + 1], n_sets), &part))) break;
            const uint64_t base = h->s.C.size();
            if (base + part.C.size() > 0xFFFFFFFFull) {
                rc = ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "candidate stream exceeds u32 offsets");
                break;
            }
            h->s.C.insert(h->s.C.end(), part.C.begin(), part.C.end());
            for (size_t k = 0; k < part.C_O.size(); k += 2) {
                h->s.C_O.push_back(part.C_O[k]);
                h->s.C_O.push_back((uint32_t)(base + part.C_O[k + 1]));
            }
        }
    } catch (const std::invalid_argument& e) {
        rc = ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        rc = ssjh::set_error(SSJ_ERR_RUNTIME, e.what());
    }
    if (rc) {
        delete h;
        return rc;
    }
    *out = h;
    return SSJ_OK;
}

int ssj_candidates_sizes(const ssj_candidates* h, uint64_t* nC, uint64_t* nCO, uint64_t* n_host) {
    if (!h) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null candidates");
    if (nC) *nC = h->s.C.size();
    if (nCO) *nCO = h->s.C_O.size();
    if (n_host) *n_host = h->host_pairs.size() / 2;
    return SSJ_OK;
}

int ssj_candidates_copy(const ssj_candidates* h, uint32_t* C, uint32_t* C_O, uint32_t* host_pairs) {
    if (!h) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null candidates");
    if (C && !h->s.C.empty()) std::memcpy(C, h->s.C.data(), h->s.C.size() * 4);
    if (C_O && !h->s.C_O.empty()) std::memcpy(C_O, h->s.C_O.data(), h->s.C_O.size() * 4);
    if (host_pairs && !h->host_pairs.empty())
        std::memcpy(host_pairs, h->host_pairs.data(), h->host_pairs.size() * 4);
    return SSJ_OK;
}

void ssj_candidates_free(ssj_candidates* h) { delete h; }

}  // extern "C"
