// pipeline.cpp -- run_join (pipeline.hpp:150-361) with the verification engine on a B200.
//
// Roles and hand-offs are the reference's (the paper's co-process scheme):
//   H0 (caller thread)  candidate generation + serialization into budgeted chunks; the
//                       chunk storage is pinned host memory (ssj_host_alloc), so the
//                       engine's copy stream DMAs it without staging;
//   H1 (dispatcher)     ssj_verify_chunk on the GPU (H2D of C/C_O in pieces overlapped with
//                       the kernels and the D2H of the flags);
//   H2 (post-process)   flags -> (max, min) original-id pairs (pipeline.hpp:79-92).
// A rendezvous hand-off keeps at most two chunks live, exactly like ChunkHandoff
// (pipeline.hpp:105-141), and the sink splits batches at the budget like
// pipeline.hpp:276-297. GroupJoin's intra-group pairs (joiners.hpp:175-179), which the
// reference verifies on H0 with the CPU merge (pipeline.hpp:299-312), are batched into
// chunks and verified on the GPU by a second engine sharing the device collection.
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "host_common.hpp"
#include "host_join.hpp"

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct SsjError : std::runtime_error {
    int code;
    SsjError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void ck(int rc) {
    if (rc) throw SsjError(rc, ssj_last_error());
}

// Growable pinned array: chunk storage the copy engine reads directly.
template <typename T>
struct PinnedVec {
    T* p = nullptr;
    size_t n = 0, cap = 0;
    PinnedVec() = default;
    PinnedVec(const PinnedVec&) = delete;
    ~PinnedVec() { ssj_host_free(p); }
    void reserve(size_t want) {
        if (want <= cap) return;
        size_t nc = std::max<size_t>({want, cap * 2, 4096});
        T* q = static_cast<T*>(ssj_host_alloc(nc * sizeof(T)));
        if (!q) throw std::bad_alloc();
        if (n) std::memcpy(q, p, n * sizeof(T));
        ssj_host_free(p);
        p = q;
        cap = nc;
    }
    void append(const T* a, size_t k) {
        if (!k) return;
        reserve(n + k);
        std::memcpy(p + n, a, k * sizeof(T));
        n += k;
    }
    void push_back(T v) {
        reserve(n + 1);
        p[n++] = v;
    }
};

// chunk.hpp:20-28 CandidateChunk in pinned memory, plus its flags.
struct Chunk {
    PinnedVec<uint32_t> C, CO;
    PinnedVec<uint8_t> flags;
    PinnedVec<uint32_t> pairs;  // pairs decoded on the GPU (pairs mode without observer);
                                // capacity reused across chunks, never zero-filled
    bool decoded = false;
    uint64_t ticket = 0;        // dispatcher: the engine ticket while in flight
    uint64_t byte_size() const { return 4ull * (C.n + CO.n); }  // chunk.hpp:25-27
    void clear() {
        C.n = CO.n = 0;
        pairs.n = 0;
        decoded = false;
    }
};

class ChunkPool {
public:
    explicit ChunkPool(size_t n) {
        for (size_t i = 0; i < n; ++i) {
            all_.push_back(std::make_unique<Chunk>());
            free_.push_back(all_.back().get());
        }
    }
    Chunk* acquire() {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return !free_.empty(); });
        Chunk* c = free_.back();
        free_.pop_back();
        c->clear();
        return c;
    }
    void release(Chunk* c) {
        std::lock_guard<std::mutex> lk(m_);
        free_.push_back(c);
        cv_.notify_all();
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    std::vector<std::unique_ptr<Chunk>> all_;
    std::vector<Chunk*> free_;
};

// pipeline.hpp:105-141 ChunkHandoff: rendezvous of one sealed chunk.
class Handoff {
public:
    // Blocks until the consumer took the chunk. Returns false when the hand-off was closed
    // (consumer failed): the chunk is dropped and stays with the producer.
    bool put(Chunk* c) {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return !slot_ || closed_; });
        if (closed_) return false;
        slot_ = c;
        cv_.notify_all();
        cv_.wait(lk, [&] { return slot_ != c || closed_; });
        if (slot_ == c) {  // closed before it was taken
            slot_ = nullptr;
            return false;
        }
        return true;
    }
    Chunk* take() {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return slot_ || closed_; });
        Chunk* c = slot_;
        slot_ = nullptr;
        cv_.notify_all();
        return c;
    }
    void close() {
        std::lock_guard<std::mutex> lk(m_);
        closed_ = true;
        cv_.notify_all();
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    Chunk* slot_ = nullptr;
    bool closed_ = false;
};

struct EngineHolder {
    ssj_engine* e = nullptr;
    ~EngineHolder() { ssj_engine_destroy(e); }
};

}  // namespace

struct ssj_join_result {
    ssj_join_report report{};
    std::vector<uint32_t> pairs;  // 2 per pair
};

extern "C" {

void ssj_join_config_init(ssj_join_config* cfg) {
    // pipeline.hpp:36-51 defaults
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->algorithm = SSJ_ALG_PPJOIN;
    cfg->mode = SSJ_MODE_COUNT;
    cfg->chunk_budget = 64ull << 20;
    cfg->strategy.kind = SSJ_STRATEGY_AUTO;
    cfg->strategy.group_size = 32;
    cfg->workers = 1;
    cfg->device = 0;
    cfg->filter_threads = 1;
}

int ssj_run_join(const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                 const uint32_t* original_id, const ssj_predicate* pred,
                 const ssj_join_config* cfg, ssj_join_result** out) {
    if (!out || !pred || !cfg || !offsets)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    // PipelineConfig::validate (pipeline.hpp:45-50), then pred.validate() (:153)
    if (cfg->chunk_budget < 12)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "chunk budget below one batch record");
    if (cfg->workers < 1) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "workers must be >= 1");
    int rc = ssj_strategy_validate(&cfg->strategy);
    if (rc) return rc;
    if ((rc = ssj_predicate_validate(pred))) return rc;
    if (cfg->algorithm < SSJ_ALG_ALLPAIRS || cfg->algorithm > SSJ_ALG_GROUPJOIN)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "unknown algorithm");
    if (cfg->mode != SSJ_MODE_COUNT && cfg->mode != SSJ_MODE_PAIRS)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "bad output mode");
    if (cfg->max_inflight > 2)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "max_inflight must be 0, 1 or 2");
    if (cfg->devices && !cfg->n_devices)
        return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "empty device list");

    const bool pairs_mode = cfg->mode == SSJ_MODE_PAIRS;
    const uint64_t budget = cfg->chunk_budget;
    ssjh::CollView coll{tokens, offsets, n_sets};
    std::vector<uint32_t> identity;
    if (!original_id) {
        identity.resize(n_sets);
        for (uint32_t i = 0; i < n_sets; ++i) identity[i] = i;
        original_id = identity.data();
    }

    auto result = std::make_unique<ssj_join_result>();
    ssj_join_report& report = result->report;
    const auto setup_start = Clock::now();
    EngineHolder engine, host_engine;
    // pipeline.hpp:156: the engine -- one GPU, or one engine over several (probe-slice split
    // of every chunk, ssj_engine_create_multi)
    if ((rc = cfg->devices ? ssj_engine_create_multi(&engine.e, cfg->devices, cfg->n_devices, tokens,
                                                     offsets, n_sets, pred, cfg->mode,
                                                     &cfg->strategy)
                           : ssj_engine_create(&engine.e, cfg->device, tokens, offsets, n_sets, pred,
                                               cfg->mode, &cfg->strategy)))
        return rc;
    const int engine_device = ssj_engine_device(engine.e);
    ssj_engine_strategy(engine.e, &report.resolved_strategy);
    if (pairs_mode && (rc = ssj_engine_set_original_ids(engine.e, original_id))) return rc;
    report.setup_ms = ms_since(setup_start);

    if (cfg->filter_threads == SSJ_FILTER_ON_GPU) {
        // H0 on the device: candidates are generated, verified and decoded there
        if (cfg->observer)
            return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT,
                                   "chunk_observer needs host chunks (GPU filtering keeps them on "
                                   "the device)");
        const auto join_start = Clock::now();
        const uint64_t max_chunk = budget == UINT64_MAX ? 0 : std::max<uint64_t>(budget / 4, 1);
        ssj_gpu_join_report gr{};
        uint64_t n = 0;
        std::vector<uint32_t> pairs;
        if (pairs_mode) {
            // a generous first capacity; rerun only when the result is larger
            const uint64_t cap0 = std::max<uint64_t>(1u << 20, n_sets);
            pairs.resize(2 * cap0);
            rc = ssj_gpu_join(engine.e, cfg->algorithm, max_chunk, pairs.data(), cap0, &n, &gr);
            if (rc && n > cap0) {
                pairs.resize(2 * n);
                rc = ssj_gpu_join(engine.e, cfg->algorithm, max_chunk, pairs.data(), n, &n, &gr);
            }
            if (rc) return rc;
            pairs.resize(2 * n);
        } else if ((rc = ssj_gpu_join(engine.e, cfg->algorithm, max_chunk, nullptr, 0, &n, &gr))) {
            return rc;
        }
        report.count = gr.count;
        report.candidate_count = gr.candidate_count;
        report.host_verified_pairs = gr.intra_group_pairs;
        report.chunk_count = gr.chunk_count;
        report.filtering_ms = gr.index_ms + gr.filtering_ms;
        report.verification_ms = gr.verification_ms;
        result->pairs = std::move(pairs);
        report.n_pairs = result->pairs.size() / 2;
        report.join_ms = ms_since(join_start);
        *out = result.release();
        return SSJ_OK;
    }

    // chunks in flight on the dispatcher (1: the reference's rendezvous, at most 2 live)
    const uint32_t inflight = std::max<uint32_t>(cfg->max_inflight, 1);
    ChunkPool pool(2 + inflight);
    Handoff to_dispatcher;
    std::mutex h2_mutex;
    std::condition_variable h2_cv;
    Chunk* h2_slot = nullptr;
    bool h2_closed = false, h2_busy = false;

    std::vector<uint32_t> engine_pairs;
    uint64_t engine_count = 0, verified_chunks = 0, verified_candidates = 0;
    double verification_ms = 0;
    ssj_stats stats{};       // H1's chunks (written by the dispatcher thread only)
    ssj_stats host_stats{};  // GroupJoin phase 2 (written by H0 only); summed after the joins

    std::mutex fail_mutex;
    int fail_code = 0;
    std::string fail_msg;
    auto capture = [&](int code, const std::string& msg) {
        std::lock_guard<std::mutex> lk(fail_mutex);
        if (!fail_code) {
            fail_code = code;
            fail_msg = msg;
        }
    };

    std::mutex live_mutex;
    uint64_t sealed_live = 0, max_live = 0;
    auto observe_live = [&](uint64_t open_bytes) {
        std::lock_guard<std::mutex> lk(live_mutex);
        max_live = std::max(max_live, sealed_live + open_bytes);
    };

    // ---- H2: flags -> pairs (pipeline.hpp:189-211, decode_pairs :79-92) -------------------
    std::thread h2([&] {
        try {
            for (;;) {
                std::unique_lock<std::mutex> lk(h2_mutex);
                h2_cv.wait(lk, [&] { return h2_slot || h2_closed; });
                if (!h2_slot) return;
                Chunk* ch = h2_slot;
                h2_slot = nullptr;
                lk.unlock();
                uint64_t prev = 0;
                if (ch->decoded)
                    engine_pairs.insert(engine_pairs.end(), ch->pairs.p, ch->pairs.p + ch->pairs.n);
                for (size_t e = 0; !ch->decoded && e + 1 < ch->CO.n; e += 2) {
                    const uint32_t pid = original_id[ch->CO.p[e]];
                    const uint64_t end = ch->CO.p[e + 1];
                    for (uint64_t s = prev; s < end; ++s) {
                        if (!ch->flags.p[s]) continue;
                        const uint32_t cid = original_id[ch->C.p[s]];
                        engine_pairs.push_back(std::max(pid, cid));
                        engine_pairs.push_back(std::min(pid, cid));
                    }
                    prev = end;
                }
                {
                    std::lock_guard<std::mutex> live(live_mutex);
                    sealed_live -= ch->byte_size();
                }
                pool.release(ch);
                lk.lock();
                h2_busy = false;
                h2_cv.notify_all();
            }
        } catch (const std::exception& e) {
            capture(SSJ_ERR_RUNTIME, e.what());
        }
    });

    // ---- H1: dispatch sealed chunks to the GPU engine (pipeline.hpp:215-258) ---------------
    // With max_inflight = 2 the dispatcher submits chunk k+1 before it waits for chunk k, so
    // the engine's copy and compute streams always have the next chunk queued.
    std::thread h1([&] {
        std::vector<Chunk*> queue;  // submitted, not yet finished (oldest first)
        auto to_h2_or_free = [&](Chunk* ch) {
            if (pairs_mode) {
                std::unique_lock<std::mutex> lk(h2_mutex);
                h2_cv.wait(lk, [&] { return !h2_busy; });
                h2_busy = true;
                h2_slot = ch;
                h2_cv.notify_all();
            } else {
                {
                    std::lock_guard<std::mutex> live(live_mutex);
                    sealed_live -= ch->byte_size();
                }
                pool.release(ch);
            }
        };
        auto finish = [&](Chunk* ch, uint64_t count) {
            ++verified_chunks;
            verified_candidates += ch->C.n;
            if (cfg->observer)
                cfg->observer(cfg->observer_user, ch->C.p, ch->C.n, ch->CO.p, ch->CO.n,
                              pairs_mode ? ch->flags.p : nullptr, count);
            engine_count += count;
            to_h2_or_free(ch);
        };
        auto wait_oldest = [&]() {
            Chunk* ch = queue.front();
            queue.erase(queue.begin());
            uint64_t count = 0;
            const auto t0 = Clock::now();
            ck(ssj_wait_chunk(engine.e, ch->ticket, &count, &stats));
            verification_ms += ms_since(t0);
            finish(ch, count);
        };
        try {
            for (;;) {
                if (pairs_mode && inflight == 1) {
                    std::unique_lock<std::mutex> lk(h2_mutex);
                    h2_cv.wait(lk, [&] { return !h2_busy; });
                }
                Chunk* ch = to_dispatcher.take();
                if (!ch) break;
                const auto t0 = Clock::now();
                if (pairs_mode && !cfg->observer) {
                    // H2 on the GPU: only the qualifying pairs (original ids) cross PCIe, in
                    // decode_pairs order (synchronous: one chunk at a time)
                    while (!queue.empty()) wait_oldest();
                    uint64_t count = 0;
                    ch->pairs.reserve(2 * (ch->C.n + 1));
                    ck(ssj_verify_chunk_pairs(engine.e, ch->C.p, ch->C.n, ch->CO.p, ch->CO.n,
                                              ch->pairs.p, nullptr, ch->C.n + 1, &count, 0,
                                              &stats));
                    ch->pairs.n = 2 * count;
                    ch->decoded = true;
                    verification_ms += ms_since(t0);
                    finish(ch, count);
                    continue;
                }
                if (pairs_mode) ch->flags.reserve(ch->C.n + 1);
                ck(ssj_submit_chunk(engine.e, ch->C.p, ch->C.n, ch->CO.p, ch->CO.n,
                                    pairs_mode ? ch->flags.p : nullptr, &ch->ticket));
                verification_ms += ms_since(t0);
                queue.push_back(ch);
                if (queue.size() >= inflight) wait_oldest();
            }
            while (!queue.empty()) wait_oldest();
            std::unique_lock<std::mutex> lk(h2_mutex);
            h2_cv.wait(lk, [&] { return !h2_busy && !h2_slot; });
            h2_closed = true;
            h2_cv.notify_all();
        } catch (const SsjError& e) {
            capture(e.code, e.what());
        } catch (const std::exception& e) {
            capture(SSJ_ERR_RUNTIME, e.what());
        }
        if (fail_code) {
            for (Chunk* ch : queue) {  // drain what is still on the GPU (errors already captured)
                uint64_t c = 0;
                ssj_wait_chunk(engine.e, ch->ticket, &c, nullptr);
            }
            to_dispatcher.close();
            std::lock_guard<std::mutex> lk(h2_mutex);
            h2_closed = true;
            h2_cv.notify_all();
        }
    });

    // ---- H0: generation + serialization on the calling thread -----------------------------
    const auto join_start = Clock::now();  // pipeline.hpp:314: after engine and thread setup
    std::vector<uint32_t> host_pairs;
    uint64_t host_count = 0;
    double serialization_ms = 0, handoff_wait_ms = 0, generation_ms = 0;
    Chunk* open = pool.acquire();

    auto hand_off = [&]() {  // pipeline.hpp:266-274
        Chunk* sealed = open;
        {
            std::lock_guard<std::mutex> lk(live_mutex);
            sealed_live += sealed->byte_size();
            max_live = std::max(max_live, sealed_live);
        }
        const auto tw = Clock::now();
        const bool taken = to_dispatcher.put(sealed);
        handoff_wait_ms += ms_since(tw);
        if (!taken) {  // consumer failed: drop the chunk, surface its error after the joins
            {
                std::lock_guard<std::mutex> lk(live_mutex);
                sealed_live -= sealed->byte_size();
            }
            sealed->clear();
            open = sealed;
            throw SsjError(SSJ_ERR_RUNTIME, "dispatcher stopped");
        }
        open = pool.acquire();
    };
    auto capacity = [&]() -> uint64_t {  // chunk.hpp:64-68
        const uint64_t used = open->byte_size();
        if (used + 8 > budget) return 0;
        return (budget - used - 8) / 4;
    };
    auto entry_fits = [&]() { return open->byte_size() + 8 <= budget; };

    auto sink = [&](uint32_t probe, const uint32_t* cands, size_t k) {  // pipeline.hpp:276-297
        const auto t0 = Clock::now();
        size_t done = 0;
        bool appended = false;
        while (done < k || !appended) {
            const uint64_t cap = capacity();
            const size_t take = (size_t)std::min<uint64_t>(cap, k - done);
            if ((take == 0 && done < k) || (done == k && !entry_fits())) {
                if (open->CO.n == 0) throw SsjError(SSJ_ERR_RUNTIME, "chunk budget below one batch record");
                hand_off();
                continue;
            }
            open->C.append(cands + done, take);
            open->CO.push_back(probe);
            open->CO.push_back((uint32_t)open->C.n);
            done += take;
            appended = true;
            if (done == k) break;
        }
        observe_live(open->byte_size());
        serialization_ms += ms_since(t0);
    };

    // GroupJoin phase 2 (joiners.hpp:175-179): batched into chunks for a second engine.
    Chunk host_chunk;
    auto flush_host = [&]() {
        if (host_chunk.CO.n == 0) return;
        if (!host_engine.e) {
            const uint32_t* dt = nullptr;
            const uint32_t* ds = nullptr;
            uint64_t np = 0;
            ck(ssj_engine_device_collection(engine.e, &dt, &np, &ds));
            ssj_strategy a{SSJ_STRATEGY_A, 1};  // host_verify always records stats (:304)
            ck(ssj_engine_create_from_device(&host_engine.e, engine_device, dt, np, ds, n_sets,
                                             n_sets ? (uint64_t)offsets[n_sets] - offsets[0] : 0,
                                             pred, SSJ_MODE_PAIRS, &a));
        }
        host_chunk.flags.reserve(host_chunk.C.n + 1);
        uint64_t cnt = 0;
        ck(ssj_verify_chunk(host_engine.e, host_chunk.C.p, host_chunk.C.n, host_chunk.CO.p,
                            host_chunk.CO.n, host_chunk.flags.p, &cnt, &host_stats));
        host_count += cnt;
        if (pairs_mode) {
            uint64_t prev = 0;
            for (size_t e = 0; e + 1 < host_chunk.CO.n; e += 2) {
                const uint32_t a = original_id[host_chunk.CO.p[e]];
                const uint64_t end = host_chunk.CO.p[e + 1];
                for (uint64_t s = prev; s < end; ++s) {
                    if (!host_chunk.flags.p[s]) continue;
                    const uint32_t b = original_id[host_chunk.C.p[s]];
                    host_pairs.push_back(std::max(a, b));
                    host_pairs.push_back(std::min(a, b));
                }
                prev = end;
            }
        }
        host_chunk.clear();
    };
    auto host_verify = [&](uint32_t a, uint32_t b) {
        // consecutive (a, b) with equal a form one slice
        if (host_chunk.CO.n && host_chunk.CO.p[host_chunk.CO.n - 2] == a &&
            host_chunk.CO.p[host_chunk.CO.n - 1] == host_chunk.C.n) {
            host_chunk.C.push_back(b);
            host_chunk.CO.p[host_chunk.CO.n - 1] = (uint32_t)host_chunk.C.n;
        } else {
            host_chunk.C.push_back(b);
            host_chunk.CO.push_back(a);
            host_chunk.CO.push_back((uint32_t)host_chunk.C.n);
        }
        if (host_chunk.C.n >= (4u << 20)) flush_host();
    };

    try {
        const auto gen_start = Clock::now();
        if (cfg->filter_threads != 1 && cfg->algorithm != SSJ_ALG_GROUPJOIN && n_sets) {
            ssjh::ParallelGenerator gen(coll, *pred, cfg->algorithm, n_sets, cfg->filter_threads);
            ssjh::CandidateStream stream;
            const uint32_t window = 32768;
            for (uint32_t lo = 0; lo < n_sets && !fail_code; lo += window) {
                ck(gen.generate(lo, std::min<uint64_t>((uint64_t)lo + window, n_sets), &stream));
                uint64_t prev = 0;
                for (size_t e = 0; e + 1 < stream.C_O.size(); e += 2) {
                    const uint64_t end = stream.C_O[e + 1];
                    sink(stream.C_O[e], stream.C.data() + prev, end - prev);
                    prev = end;
                }
            }
        } else {
            ck(ssjh::generate_sequential(coll, *pred, cfg->algorithm, sink, host_verify));
        }
        flush_host();
        if (open->CO.n) {
            const auto t0 = Clock::now();
            hand_off();
            serialization_ms += ms_since(t0);
        }
        generation_ms = ms_since(gen_start);
    } catch (const SsjError& e) {
        if (std::string(e.what()) != "dispatcher stopped") capture(e.code, e.what());
    } catch (const std::bad_alloc&) {
        capture(SSJ_ERR_RUNTIME, "pinned host allocation failed");
    } catch (const std::invalid_argument& e) {
        capture(SSJ_ERR_INVALID_ARGUMENT, e.what());
    } catch (const std::exception& e) {
        capture(SSJ_ERR_RUNTIME, e.what());
    }
    to_dispatcher.close();
    h1.join();
    h2.join();
    if (fail_code) return ssjh::set_error(fail_code, fail_msg);

    report.count = engine_count + host_count;
    if (pairs_mode) {
        result->pairs = std::move(engine_pairs);
        result->pairs.insert(result->pairs.end(), host_pairs.begin(), host_pairs.end());
    }
    report.n_pairs = result->pairs.size() / 2;
    report.chunk_count = verified_chunks;
    report.candidate_count = verified_candidates;
    report.host_verified_pairs = host_count;
    report.max_live_candidate_bytes = max_live;
    report.pairs_verified = stats.pairs_verified + host_stats.pairs_verified;
    report.early_exit_prunes = stats.early_exit_prunes + host_stats.early_exit_prunes;
    report.comparison_budget_violations =
        stats.comparison_budget_violations + host_stats.comparison_budget_violations;
    report.serialization_ms = serialization_ms;
    report.filtering_ms = std::max(0.0, generation_ms - serialization_ms);
    report.verification_ms = verification_ms;
    report.handoff_wait_ms = handoff_wait_ms;
    report.join_ms = ms_since(join_start);
    *out = result.release();
    return SSJ_OK;
}

int ssj_join_result_report(const ssj_join_result* r, ssj_join_report* report) {
    if (!r || !report) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    *report = r->report;
    return SSJ_OK;
}

int ssj_join_result_pairs(const ssj_join_result* r, uint32_t* pairs) {
    if (!r) return ssjh::set_error(SSJ_ERR_INVALID_ARGUMENT, "null result");
    if (pairs && !r->pairs.empty()) std::memcpy(pairs, r->pairs.data(), r->pairs.size() * 4);
    return SSJ_OK;
}

void ssj_join_result_free(ssj_join_result* r) { delete r; }

}  // extern "C"
