// multi_device.cpp -- one verification engine over several B200s.
//
// The reference builds one VerificationEngine (pipeline.hpp:156) and its dispatcher hands it
// every chunk (:228). Here that engine may span G GPUs:
//   * construction: the padded collection is built and uploaded once (devices[0]) and fanned
//     out device to device with peer copies over NVLink/NVSwitch in a doubling tree (round k:
//     the 2^k devices holding it copy to the next 2^k), so no GPU sends more than log2(G)
//     copies and the host link carries it once;
//   * a chunk is cut into G contiguous probe-slice ranges of equal work -- per slice
//     4|r| + k (13 + 4|r|), the SURVEY §8(d) bytes with |s| bounded by |r| (every candidate of
//     a probe is at most as long as the probe, chunk.hpp:20-28 / collection order) -- a slice
//     is never split, so each device stages its own probes; every device verifies its range
//     asynchronously (its own streams) and writes its flags straight into the caller's buffer
//     at the range's slot offset, so the flags come back in C order with no gather step;
//     counts and stats are summed on the host. There is no collective on the data path;
//   * the all-GPU join runs probe shard g of G on device g (ssj_gpu_join_shard).
#include "multi_device.hpp"

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "host_common.hpp"

namespace ssjm {

namespace {

struct Part {
    uint32_t sub = 0;
    uint64_t c_lo = 0, n = 0;
    std::vector<uint32_t> co;  // the range's C_O, end offsets rebased to c_lo
    uint64_t ticket = 0;
    bool submitted = false;
};

struct Pending {
    bool busy = false;
    uint64_t ticket = 0;
    std::vector<Part> parts;
};

int fail(int code, const std::string& msg) { return ssjh::set_error(code, msg); }

// Per-thread error text of a worker thread, re-raised on the calling thread.
struct WorkerResult {
    int rc = SSJ_OK;
    std::string msg;
    void capture(int r) {
        rc = r;
        if (r) msg = ssj_last_error();
    }
};

int first_error(const std::vector<WorkerResult>& w) {
    for (const auto& r : w)
        if (r.rc) return fail(r.rc, r.msg);
    return SSJ_OK;
}

}  // namespace

struct Group {
    std::vector<int32_t> devices;
    std::vector<ssj_engine*> subs;
    std::vector<std::pair<int, void*>> owned;  // (device, buffer) of the fanned-out copies
    std::vector<uint32_t> sizes;               // |set| per set (host), for the balance
    Pending pend[2];
    uint64_t next_ticket = 0;
    double fanout_ms = 0;
};

ssj_engine* first(const Group& g) { return g.subs.front(); }
uint32_t size(const Group& g) { return (uint32_t)g.subs.size(); }

int split_chunk(const std::vector<uint32_t>& set_sizes, uint32_t parts, const uint32_t* C_O,
                uint64_t nCO, uint64_t nC, std::vector<Range>* out) {
    const uint64_t p = nCO / 2;
    std::vector<double> pre(p + 1, 0.0);
    uint64_t prev = 0;
    for (uint64_t i = 0; i < p; ++i) {
        const uint32_t probe = C_O[2 * i];
        const uint64_t end = C_O[2 * i + 1];
        if (end < prev || end > nC)  // decode (chunk.hpp:36-48) would misread it
            return fail(SSJ_ERR_INVALID_ARGUMENT,
                        "malformed C_O: end offsets decreasing or beyond C");
        const double r = probe < set_sizes.size() ? (double)set_sizes[probe] : 0.0;
        pre[i + 1] = pre[i] + 4.0 * r + (double)(end - prev) * (13.0 + 4.0 * r);
        prev = end;
    }
    out->assign(parts, Range{});
    uint64_t a = 0;
    for (uint32_t g = 0; g < parts; ++g) {
        uint64_t b = p;
        if (g + 1 < parts) {
            const double target = pre[p] * (double)(g + 1) / (double)parts;
            b = (uint64_t)(std::lower_bound(pre.begin() + a, pre.end(), target) - pre.begin());
            b = std::min(std::max(b, a), p);
            if (b > a && pre[b] - target > target - pre[b - 1]) --b;  // the nearer cut
        }
        Range& r = (*out)[g];
        r.slice_begin = a;
        r.slice_end = b;
        r.c_lo = a ? C_O[2 * a - 1] : 0;
        r.c_hi = g + 1 == parts ? nC : (b ? C_O[2 * b - 1] : 0);  // trailing slots: the last
        a = b;
    }
    return SSJ_OK;
}

int create_group(Group** out, const int32_t* devices, uint32_t n_devices, const uint32_t* tokens,
                 const uint32_t* offsets, uint32_t n_sets, const ssj_predicate* pred, int32_t mode,
                 const ssj_strategy* strategy) {
    *out = nullptr;
    auto g = std::make_unique<Group>();
    g->devices.assign(devices, devices + n_devices);
    g->sizes.resize(n_sets);
    for (uint32_t i = 0; i < n_sets; ++i) g->sizes[i] = offsets[i + 1] - offsets[i];
    auto cleanup = [&](int rc) {
        destroy_group(g.release());
        return rc;
    };
    ssj_engine* e0 = nullptr;
    int rc = ssj_engine_create(&e0, devices[0], tokens, offsets, n_sets, pred, mode, strategy);
    if (rc) return cleanup(rc);
    g->subs.push_back(e0);
    const uint32_t* d_tok0 = nullptr;
    const uint32_t* d_sets0 = nullptr;
    uint64_t n_padded = 0;
    if ((rc = ssj_engine_device_collection(e0, &d_tok0, &n_padded, &d_sets0))) return cleanup(rc);
    const size_t tok_bytes = n_padded * sizeof(uint32_t);
    const size_t set_bytes = (size_t)std::max<uint32_t>(n_sets, 1) * 2 * sizeof(uint32_t);
    const uint64_t n_tokens = n_sets ? (uint64_t)offsets[n_sets] - offsets[0] : 0;

    // doubling-tree fan-out: holders[i] = (tokens, sets) on devices[i]
    std::vector<std::pair<const void*, const void*>> holders(n_devices, {nullptr, nullptr});
    holders[0] = {d_tok0, d_sets0};
    const auto t0 = std::chrono::steady_clock::now();
    for (uint32_t have = 1; have < n_devices; have *= 2) {
        const uint32_t hi = std::min(n_devices, 2 * have);
        std::vector<std::pair<int, cudaStream_t>> streams;
        int err = SSJ_OK;
        for (uint32_t i = have; i < hi && !err; ++i) {
            const uint32_t src = i - have;
            const int dst_dev = devices[i], src_dev = devices[src];
            if (cudaSetDevice(dst_dev) != cudaSuccess) {
                err = fail(SSJ_ERR_CUDA, "cudaSetDevice failed (fan-out)");
                break;
            }
            int can = 0;
            if (dst_dev != src_dev && cudaDeviceCanAccessPeer(&can, dst_dev, src_dev) == cudaSuccess &&
                can) {
                if (cudaDeviceEnablePeerAccess(src_dev, 0) != cudaSuccess) cudaGetLastError();
            }
            void* dt = nullptr;
            void* dsets = nullptr;
            if (cudaMalloc(&dt, tok_bytes) != cudaSuccess || cudaMalloc(&dsets, set_bytes) != cudaSuccess) {
                cudaGetLastError();
                if (dt) g->owned.push_back({dst_dev, dt});
                err = fail(SSJ_ERR_CUDA, "cudaMalloc of a collection copy failed");
                break;
            }
            g->owned.push_back({dst_dev, dt});
            g->owned.push_back({dst_dev, dsets});
            cudaStream_t st = nullptr;
            if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
                err = fail(SSJ_ERR_CUDA, "cudaStreamCreate failed (fan-out)");
                break;
            }
            streams.push_back({dst_dev, st});
            if (cudaMemcpyPeerAsync(dt, dst_dev, holders[src].first, src_dev, tok_bytes, st) !=
                    cudaSuccess ||
                cudaMemcpyPeerAsync(dsets, dst_dev, holders[src].second, src_dev, set_bytes, st) !=
                    cudaSuccess) {
                err = fail(SSJ_ERR_CUDA, "peer copy of the collection failed");
                break;
            }
            holders[i] = {dt, dsets};
        }
        for (auto& ds : streams) {  // a round's copies run concurrently; wait for all of them
            cudaSetDevice(ds.first);
            if (cudaStreamSynchronize(ds.second) != cudaSuccess && !err)
                err = fail(SSJ_ERR_CUDA, "peer copy of the collection failed");
            cudaStreamDestroy(ds.second);
        }
        if (err) return cleanup(err);
    }
    g->fanout_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (uint32_t i = 1; i < n_devices; ++i) {
        ssj_engine* e = nullptr;
        rc = ssj_engine_create_from_device(
            &e, devices[i], static_cast<const uint32_t*>(holders[i].first), n_padded,
            static_cast<const uint32_t*>(holders[i].second), n_sets, n_tokens, pred, mode, strategy);
        if (rc) return cleanup(rc);
        g->subs.push_back(e);
    }
    *out = g.release();
    return SSJ_OK;
}

void destroy_group(Group* g) {
    if (!g) return;
    for (int t = 0; t < 2; ++t)  // drain chunks still in flight
        if (g->pend[t].busy) wait(*g, g->pend[t].ticket, nullptr, nullptr);
    for (ssj_engine* e : g->subs) ssj_engine_destroy(e);
    for (auto& ob : g->owned) {
        cudaSetDevice(ob.first);
        cudaFree(ob.second);
    }
    delete g;
}

int devices(const Group& g, int32_t* out, uint32_t cap, uint32_t* n, double* fanout_ms) {
    if (n) *n = (uint32_t)g.devices.size();
    if (out)
        for (uint32_t i = 0; i < cap && i < g.devices.size(); ++i) out[i] = g.devices[i];
    if (fanout_ms) *fanout_ms = g.fanout_ms;
    return SSJ_OK;
}

namespace {

int make_parts(const Group& g, const uint32_t* C_O, uint64_t nCO, uint64_t nC,
               std::vector<Part>* parts) {
    std::vector<Range> rg;
    int rc = split_chunk(g.sizes, size(g), C_O, nCO, nC, &rg);
    if (rc) return rc;
    parts->clear();
    for (uint32_t s = 0; s < rg.size(); ++s) {
        Part pt;
        pt.sub = s;
        pt.c_lo = rg[s].c_lo;
        pt.n = rg[s].c_hi - rg[s].c_lo;
        pt.co.reserve(2 * (rg[s].slice_end - rg[s].slice_begin));
        for (uint64_t i = rg[s].slice_begin; i < rg[s].slice_end; ++i) {
            pt.co.push_back(C_O[2 * i]);
            pt.co.push_back((uint32_t)(C_O[2 * i + 1] - pt.c_lo));
        }
        if (pt.n || !pt.co.empty()) parts->push_back(std::move(pt));
    }
    return SSJ_OK;
}

}  // namespace

int wait(Group& g, uint64_t ticket, uint64_t* count_out, ssj_stats* stats) {
    Pending& pd = g.pend[ticket & 1];
    if (!pd.busy || pd.ticket != ticket) return fail(SSJ_ERR_INVALID_ARGUMENT, "unknown ticket");
    int rc = SSJ_OK;
    std::string msg;
    uint64_t total = 0;
    ssj_stats sum{};
    for (Part& pt : pd.parts) {
        if (!pt.submitted) continue;
        uint64_t c = 0;
        ssj_stats st{};
        const int r = ssj_wait_chunk(g.subs[pt.sub], pt.ticket, &c, &st);
        if (r && !rc) {
            rc = r;
            msg = ssj_last_error();
        }
        total += c;
        sum.pairs_verified += st.pairs_verified;
        sum.early_exit_prunes += st.early_exit_prunes;
        sum.comparison_budget_violations += st.comparison_budget_violations;
    }
    pd.busy = false;
    pd.parts.clear();
    if (rc) return fail(rc, msg);
    if (count_out) *count_out = total;
    if (stats) {
        stats->pairs_verified += sum.pairs_verified;
        stats->early_exit_prunes += sum.early_exit_prunes;
        stats->comparison_budget_violations += sum.comparison_budget_violations;
    }
    return SSJ_OK;
}

int submit(Group& g, const uint32_t* C, uint64_t nC, const uint32_t* C_O, uint64_t nCO,
           uint8_t* flags_out, uint64_t* ticket) {
    const uint64_t t = g.next_ticket;
    Pending& pd = g.pend[t & 1];
    if (pd.busy) return fail(SSJ_ERR_RUNTIME, "two chunks already in flight: wait first");
    int rc = make_parts(g, C_O, nCO, nC, &pd.parts);
    if (rc) return rc;
    pd.busy = true;
    pd.ticket = t;
    for (Part& pt : pd.parts) {
        rc = ssj_submit_chunk(g.subs[pt.sub], C ? C + pt.c_lo : nullptr, pt.n,
                              pt.co.empty() ? nullptr : pt.co.data(), pt.co.size(),
                              flags_out ? flags_out + pt.c_lo : nullptr, &pt.ticket);
        if (rc) break;
        pt.submitted = true;
    }
    if (rc) {
        const std::string msg = ssj_last_error();
        wait(g, t, nullptr, nullptr);  // drain the parts already submitted
        return fail(rc, msg);
    }
    g.next_ticket = t + 1;
    *ticket = t;
    return SSJ_OK;
}

int verify_results(Group& g, const uint32_t* C, uint64_t nC, const uint32_t* C_O, uint64_t nCO,
                   uint32_t* slots_out, uint32_t* overlaps_out, uint64_t cap, uint64_t* n_out) {
    std::vector<Part> parts;
    int rc = make_parts(g, C_O, nCO, nC, &parts);
    if (rc) return rc;
    std::vector<std::vector<uint32_t>> sl(parts.size()), ov(parts.size());
    std::vector<uint64_t> cnt(parts.size(), 0);
    std::vector<WorkerResult> res(parts.size());
    std::vector<std::thread> th;
    for (size_t k = 0; k < parts.size(); ++k)
        th.emplace_back([&, k] {
            const Part& pt = parts[k];
            sl[k].resize(pt.n + 1);
            ov[k].resize(pt.n + 1);
            res[k].capture(ssj_verify_chunk_results(
                g.subs[pt.sub], C ? C + pt.c_lo : nullptr, pt.n,
                pt.co.empty() ? nullptr : pt.co.data(), pt.co.size(), sl[k].data(), ov[k].data(),
                pt.n + 1, &cnt[k]));
        });
    for (auto& t : th) t.join();
    if ((rc = first_error(res))) return rc;
    uint64_t n = 0;
    for (size_t k = 0; k < parts.size(); ++k)  // ranges ascend: slot order is kept
        for (uint64_t i = 0; i < cnt[k]; ++i, ++n)
            if (n < cap) {
                slots_out[n] = (uint32_t)(sl[k][i] + parts[k].c_lo);
                overlaps_out[n] = ov[k][i];
            }
    *n_out = n;
    if (n > cap) return fail(SSJ_ERR_RUNTIME, "result capacity exceeded");
    return SSJ_OK;
}

int verify_pairs(Group& g, const uint32_t* C, uint64_t nC, const uint32_t* C_O, uint64_t nCO,
                 uint32_t* pairs_out, uint32_t* overlaps_out, uint64_t cap, uint64_t* n_out,
                 int sorted, ssj_stats* stats) {
    std::vector<Part> parts;
    int rc = make_parts(g, C_O, nCO, nC, &parts);
    if (rc) return rc;
    const size_t P = parts.size();
    std::vector<std::unique_ptr<uint32_t[]>> pr(P), ov(P);  // not zero-filled
    std::vector<uint64_t> cnt(P, 0);
    std::vector<ssj_stats> st(P, ssj_stats{});
    std::vector<WorkerResult> res(P);
    std::vector<std::thread> th;
    for (size_t k = 0; k < P; ++k)
        th.emplace_back([&, k] {
            const Part& pt = parts[k];
            pr[k].reset(new uint32_t[2 * (pt.n + 1)]);
            ov[k].reset(new uint32_t[pt.n + 1]);
            res[k].capture(ssj_verify_chunk_pairs(
                g.subs[pt.sub], C ? C + pt.c_lo : nullptr, pt.n,
                pt.co.empty() ? nullptr : pt.co.data(), pt.co.size(), pr[k].get(), ov[k].get(),
                pt.n + 1, &cnt[k], sorted, &st[k]));
        });
    for (auto& t : th) t.join();
    if ((rc = first_error(res))) return rc;
    uint64_t n = 0;
    for (size_t k = 0; k < P; ++k) n += cnt[k];
    *n_out = n;
    if (stats)
        for (size_t k = 0; k < P; ++k) {
            stats->pairs_verified += st[k].pairs_verified;
            stats->early_exit_prunes += st[k].early_exit_prunes;
            stats->comparison_budget_violations += st[k].comparison_budget_violations;
        }
    // slot order: the ranges ascend, so concatenation keeps it; write_pairs order: a merge
    std::vector<std::pair<unsigned long long, uint32_t>> all;
    all.reserve(n);
    for (size_t k = 0; k < P; ++k)
        for (uint64_t i = 0; i < cnt[k]; ++i)
            all.push_back({((unsigned long long)pr[k][2 * i] << 32) | pr[k][2 * i + 1], ov[k][i]});
    if (sorted) std::stable_sort(all.begin(), all.end(), [](const auto& a, const auto& b) {
        return a.first < b.first;
    });
    const uint64_t w = std::min<uint64_t>(n, cap);
    for (uint64_t i = 0; i < w; ++i) {
        pairs_out[2 * i] = (uint32_t)(all[i].first >> 32);
        pairs_out[2 * i + 1] = (uint32_t)all[i].first;
        if (overlaps_out) overlaps_out[i] = all[i].second;
    }
    if (n > cap) return fail(SSJ_ERR_RUNTIME, "result capacity exceeded");
    return SSJ_OK;
}

int set_original_ids(Group& g, const uint32_t* original_id) {
    for (ssj_engine* e : g.subs) {
        const int rc = ssj_engine_set_original_ids(e, original_id);
        if (rc) return rc;
    }
    return SSJ_OK;
}

int gpu_join_shard(Group& g, int32_t algorithm, uint32_t shard, uint32_t n_shards,
                   uint64_t max_chunk_candidates, uint32_t* pairs_out, uint64_t pairs_cap,
                   uint64_t* n_pairs, ssj_gpu_join_report* report) {
    if (n_shards == 0 || shard >= n_shards) return fail(SSJ_ERR_INVALID_ARGUMENT, "bad shard");
    const auto t0 = std::chrono::steady_clock::now();
    // GroupJoin's groups are one sequential stream: it runs on the first device
    const uint32_t G = algorithm == SSJ_ALG_GROUPJOIN ? 1u : size(g);
    const bool want = pairs_out != nullptr;
    std::vector<std::vector<uint32_t>> pr(G);
    std::vector<uint64_t> np(G, 0);
    std::vector<ssj_gpu_join_report> rep(G, ssj_gpu_join_report{});
    std::vector<WorkerResult> res(G);
    std::vector<std::thread> th;
    for (uint32_t k = 0; k < G; ++k)
        th.emplace_back([&, k] {
            if (want) pr[k].resize(2 * std::max<uint64_t>(pairs_cap, 1));
            res[k].capture(ssj_gpu_join_shard(g.subs[k], algorithm, shard * G + k, n_shards * G,
                                              max_chunk_candidates, want ? pr[k].data() : nullptr,
                                              want ? pairs_cap : 0, &np[k], &rep[k]));
        });
    for (auto& t : th) t.join();
    int rc = first_error(res);
    if (rc) return rc;
    ssj_gpu_join_report r{};
    uint64_t total = 0;
    for (uint32_t k = 0; k < G; ++k) {
        r.count += rep[k].count;
        r.candidate_count += rep[k].candidate_count;
        r.intra_group_pairs += rep[k].intra_group_pairs;
        r.chunk_count += rep[k].chunk_count;
        r.index_ms = std::max(r.index_ms, rep[k].index_ms);  // devices work concurrently
        r.filtering_ms = std::max(r.filtering_ms, rep[k].filtering_ms);
        r.verification_ms = std::max(r.verification_ms, rep[k].verification_ms);
        total += np[k];
    }
    if (want) {
        // the shards' pair sets are disjoint; each is sorted: merge into write_pairs order
        std::vector<unsigned long long> keys;
        keys.reserve(total);
        for (uint32_t k = 0; k < G; ++k)
            for (uint64_t i = 0; i < np[k]; ++i)
                keys.push_back(((unsigned long long)pr[k][2 * i] << 32) | pr[k][2 * i + 1]);
        std::sort(keys.begin(), keys.end());
        const uint64_t w = std::min<uint64_t>(total, pairs_cap);
        for (uint64_t i = 0; i < w; ++i) {
            pairs_out[2 * i] = (uint32_t)(keys[i] >> 32);
            pairs_out[2 * i + 1] = (uint32_t)keys[i];
        }
    }
    if (n_pairs) *n_pairs = want ? total : 0;
    r.join_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (report) *report = r;
    if (want && total > pairs_cap) return fail(SSJ_ERR_RUNTIME, "pair capacity exceeded");
    return SSJ_OK;
}

int set_profiling(Group& g, int enabled) {
    for (ssj_engine* e : g.subs) {
        const int rc = ssj_engine_set_profiling(e, enabled);
        if (rc) return rc;
    }
    return SSJ_OK;
}

int kernel_time(Group& g, double* total_ms, uint64_t* launches) {
    double mx = 0;
    uint64_t n = 0;
    for (ssj_engine* e : g.subs) {
        double ms = 0;
        uint64_t l = 0;
        const int rc = ssj_engine_kernel_time(e, &ms, &l);
        if (rc) return rc;
        mx = std::max(mx, ms);  // the devices verify concurrently
        n += l;
    }
    if (total_ms) *total_ms = mx;
    if (launches) *launches = n;
    return SSJ_OK;
}

}  // namespace ssjm
