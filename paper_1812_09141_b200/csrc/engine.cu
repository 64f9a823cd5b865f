// engine.cu -- the C ABI (include/ssjoin_b200.h) over the sm_100a verification kernels.
//
// One ssj_engine = one VerificationEngine (verify.hpp:241-351) bound to one GPU:
//   * the Collection (collection.hpp:76-94) is re-laid out into a 32-byte-aligned padded
//     CSR plus {pos8, size} descriptors and uploaded once;
//   * each chunk (chunk.hpp:20-28) crosses PCIe in pieces on a copy stream while the
//     compute stream verifies the pieces already resident and a second copy stream returns
//     their flags (the paper's co-process scheme inside one chunk);
//   * two chunk slots allow ssj_submit_chunk / ssj_wait_chunk double buffering.
// No CPU verification path exists here: without a device every entry point fails.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "../../include/ssjoin_b200.h"
#include "host_common.hpp"
#include "gpu_filter.cuh"
#include "verify_kernels.cuh"
#include "multi_device.hpp"

using ssjb::KParams;
using ssjb::PredDev;

namespace {

thread_local std::string g_err;

int fail(int code, std::string msg) {
    g_err = std::move(msg);
    return code;
}

#define SSJ_CK(x)                                                                       \
    do {                                                                                \
        cudaError_t _e = (x);                                                           \
        if (_e != cudaSuccess)                                                          \
            return fail(SSJ_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(_e)); \
    } while (0)

typedef unsigned __int128 u128;

uint64_t host_ceil_div(u128 a, u128 b) { return (uint64_t)((a + b - 1) / b); }

// Restores the caller's current device on scope exit (torch and other users keep theirs).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceScope() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

constexpr int kEventsPerSlot = 96;
constexpr uint64_t kPieceMinSlots = 1ull << 22;  // 4M candidates = 16 MB of C per piece
constexpr int kMaxPieces = 32;
using ssjb::kCounters;  // per piece: deferred long slices, runs, short tiles, long-pass
                              // work, short-tile work

template <typename T>
int ensure_device(T** ptr, size_t* cap, size_t need) {
    if (need <= *cap && *ptr) return SSJ_OK;
    if (*ptr) cudaFree(*ptr);
    *ptr = nullptr;
    *cap = 0;
    size_t alloc = std::max<size_t>(need, 1);
    alloc = alloc + alloc / 4;  // grow with headroom
    SSJ_CK(cudaMalloc(reinterpret_cast<void**>(ptr), alloc * sizeof(T)));
    *cap = alloc;
    return SSJ_OK;
}

template <typename T>
int ensure_pinned(T** ptr, size_t* cap, size_t need) {
    if (need <= *cap && *ptr) return SSJ_OK;
    if (*ptr) cudaFreeHost(*ptr);
    *ptr = nullptr;
    *cap = 0;
    size_t alloc = std::max<size_t>(need, 1);
    alloc = alloc + alloc / 4;
    SSJ_CK(cudaHostAlloc(reinterpret_cast<void**>(ptr), alloc * sizeof(T), cudaHostAllocDefault));
    *cap = alloc;
    return SSJ_OK;
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

struct ChunkSlot {
    uint32_t* dC = nullptr;
    size_t capC = 0;
    uint32_t* dCO = nullptr;
    size_t capCO = 0;
    uint8_t* dflags = nullptr;
    size_t capF = 0;
    uint32_t* dtile = nullptr;
    size_t capT = 0;
    ssjb::SliceDesc* dslices = nullptr;
    size_t capS = 0;
    uint32_t* dbits = nullptr;
    size_t capB = 0;
    uint32_t* drank = nullptr;
    size_t capR = 0;
    uint32_t* ddefer = nullptr;          // long-pair slots (strategy A)
    size_t capDf = 0;
    unsigned long long* ddefer_n = nullptr;  // kCounters counters per piece
    size_t capCtr = 0;
    uint32_t* dbmlist = nullptr;         // slices with a probe bitmap (strategy A)
    size_t capBL = 0;
    ssjb::RunDesc* druns = nullptr;      // runs of long slices (strategy A)
    size_t capRu = 0;
    uint32_t* dshort = nullptr;          // short tiles (strategy A)
    size_t capSh = 0;
    unsigned long long* dacc = nullptr;
    unsigned long long* hacc = nullptr;  // pinned mirror of dacc
    uint8_t* hflags = nullptr;           // pinned staging for pageable flag buffers
    size_t capHF = 0;
    cudaEvent_t ev[kEventsPerSlot] = {};
    cudaEvent_t done = nullptr;
    bool busy = false;
    uint64_t ticket = 0;
    uint8_t* user_flags = nullptr;
    bool flags_staged = false;
    uint64_t nC = 0;
};

}  // namespace

namespace ssjh {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace ssjh

// Device scratch of the GPU join (cached on the engine across calls).
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
    int alloc(size_t bytes) {
        cudaFree(p);
        p = nullptr;
        if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess)
            return ssjh::set_error(SSJ_ERR_CUDA, "cudaMalloc failed (GPU join)");
        return SSJ_OK;
    }
};

// Per-join scratch: per-probe bounds (scanned), block buffers.
struct GenState {
    DevBuf bound, base, G, count, flag, obase, slot, C, CO, tmp;
    DevBuf per, cand, coff, iflag, islot;  // GroupJoin expansion / intra-group chunk
    DevBuf acc, keys, sorted;              // join result words; pair keys (pairs mode)
    size_t keys_cap = 0, sorted_cap = 0;
    size_t gj_cap = 0, gjC_cap = 0, gjCO_cap = 0, cand_cap = 0, coff_cap = 0, iflag_cap = 0,
           islot_cap = 0;
    size_t tmp_bytes = 0, G_cap = 0, C_cap = 0, blk_cap = 0;
    std::vector<unsigned long long> hbase;  // exclusive scan of the bounds, n + 1 entries
};


struct ssj_engine {
    int device = 0;
    ssj_predicate hpred{};
    PredDev pred{};
    int32_t mode = SSJ_MODE_COUNT;
    ssj_strategy strategy{};  // resolved as the reference resolves it (reported, stats rule)
    ssj_strategy exec{};      // the kernel family that runs (Auto: strategy A's kernels)
    uint32_t n_sets = 0;
    uint64_t n_tokens = 0;      // unpadded token count (Collection::tokens.size())
    uint64_t n_padded = 0;      // padded device tokens
    uint32_t* d_tokens = nullptr;
    uint2* d_sets = nullptr;
    bool owns_collection = true;
    uint32_t* d_req_tab = nullptr;  // Jaccard/Dice required overlap by |r|+|s|
    uint4* d_heads = nullptr;       // packed set heads (null: tokens too large to pack)
    uint32_t long_words = 0;            // long pass: bitmap words a probe range can need (0: cap)
    uint32_t max_set_size = 0xFFFFFFFFu;  // largest |s| (unknown: all ones); no set longer
                                          // than kLongPair -> no long pairs, no long pass
    unsigned long long heads_tex = 0;   // linear uint4 textures over d_heads / d_tokens for
    unsigned long long tokens_tex = 0;  // the run kernel's gathers (0: not created)
    ssjb::FilterIndex* fidx = nullptr;  // GPU candidate generation index (built on first use)
    GenState* gen = nullptr;            // its bounds and block buffers
    ssjb::GroupIndex* gidx = nullptr;   // GroupJoin groups + representative index (first use)
    GenState* gen_g = nullptr;          // GroupJoin: bounds over groups and block buffers
    uint32_t req_tab_n = 0;
    cudaStream_t s_comp = nullptr, s_h2d = nullptr, s_d2h = nullptr;
    // strategy A: warp_tile_kernel runs on s_aux beside run_kernel (forked and joined with
    // two events), so the two passes' tails overlap
    cudaStream_t s_aux = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    ChunkSlot slot[2];
    uint64_t next_ticket = 0;
    // pageable-input staging
    uint32_t* bounce[2] = {nullptr, nullptr};
    size_t bounce_cap[2] = {0, 0};
    cudaEvent_t bounce_ev[2] = {nullptr, nullptr};
    // device-API scratch
    uint32_t* dev_tile = nullptr;
    size_t dev_tile_cap = 0;
    ssjb::SliceDesc* dev_slices = nullptr;
    size_t dev_slices_cap = 0;
    uint32_t* dev_bits = nullptr;
    size_t dev_bits_cap = 0;
    uint32_t* dev_rank = nullptr;
    size_t dev_rank_cap = 0;
    uint32_t* dev_defer = nullptr;
    size_t dev_defer_cap = 0;
    unsigned long long* dev_defer_n = nullptr;  // kCounters
    size_t dev_defer_n_cap = 0;
    uint32_t* dev_bmlist = nullptr;
    size_t dev_bmlist_cap = 0;
    ssjb::RunDesc* dev_runs = nullptr;
    size_t dev_runs_cap = 0;
    uint32_t* dev_short = nullptr;
    size_t dev_short_cap = 0;
    // results mode
    uint32_t* d_res_slots = nullptr;
    uint32_t* d_res_ov = nullptr;
    size_t res_cap = 0;
    size_t res_cap2 = 0;
    unsigned long long* d_res_n = nullptr;
    // GPU pair decoding (ssj_verify_chunk_pairs)
    uint32_t* d_oid = nullptr;
    unsigned long long* d_keys = nullptr;
    size_t keys_cap = 0;
    unsigned long long* d_keys_alt = nullptr;
    size_t keys_alt_cap = 0;
    uint32_t* d_ov_alt = nullptr;
    size_t ov_alt_cap = 0;
    uint32_t* d_slot_alt = nullptr;  // result slots sorted into C order
    size_t slot_alt_cap = 0;
    void* d_sort_tmp = nullptr;
    size_t sort_tmp_cap = 0;
    // multi-device engine (ssj_engine_create_multi): the per-device engines; every entry
    // point dispatches to multi_device.cpp when set
    ssjm::Group* group = nullptr;
    // kernel timing (ssj_engine_set_profiling)
    bool profiling = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;
};

namespace {

// verify.hpp:249-253: Auto resolves to B (average set size <= 10, collection.hpp:91-93) or
// to C with group >= 128; strategy() and JoinReport::resolved_strategy report exactly that,
// and the stats follow it (C records none, verify.hpp:303-345). Those are worker-pool
// policies: on the B200 one kernel family covers both regimes -- strategy A's load-balanced
// kernels (thread per short pair, warp per long pair, the cooperative scheme of C) -- so Auto
// EXECUTES the A kernels whatever it reports. Flags and counts are identical for every
// strategy; an explicit A, B or C runs that strategy's own kernels.
void resolve_strategy(ssj_engine& e, ssj_strategy s) {
    if (s.kind != SSJ_STRATEGY_AUTO) {
        e.strategy = e.exec = s;
        return;
    }
    const uint64_t avg = e.n_sets ? e.n_tokens / e.n_sets : 0;
    e.strategy = avg <= 10 ? ssj_strategy{SSJ_STRATEGY_B, s.group_size}
                           : ssj_strategy{SSJ_STRATEGY_C, std::max<uint32_t>(s.group_size, 128)};
    e.exec = {SSJ_STRATEGY_A, s.group_size};
}

int make_pred_dev(const ssj_predicate& p, PredDev* out) {
    PredDev d{};
    d.fn = p.function;
    d.num = p.num;
    d.den = p.den;
    d.ovt = p.overlap_threshold;
    if (p.function == SSJ_JACCARD) {
        d.A = p.num;
        d.B = p.den + p.num;  // u64 like similarity.hpp:114
    } else if (p.function == SSJ_DICE) {
        d.A = p.num;
        d.B = 2 * p.den;  // u64 like similarity.hpp:118
    }
    if ((p.function == SSJ_JACCARD || p.function == SSJ_DICE) && d.B == 0)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "threshold denominator overflows");
    d.wide = (d.A >= (1ull << 30) || d.B >= (1ull << 32)) ? 1 : 0;
    if ((p.function == SSJ_JACCARD || p.function == SSJ_DICE) && !d.wide) {
        d.A32 = (uint32_t)d.A;
        d.B32 = (uint32_t)d.B;
        d.Binv = 0xFFFFFFFFu / d.B32;
    }
    *out = d;
    return SSJ_OK;
}

KParams base_params(const ssj_engine& e) {
    KParams p{};
    p.tokens = e.d_tokens;
    p.sets = e.d_sets;
    p.n_sets = e.n_sets;
    p.pred = e.pred;
    p.req_tab = e.d_req_tab;
    p.req_tab_n = e.req_tab_n;
    // packed heads go to the kernels together with their texture (run_kernel gathers them
    // through it); without one the kernels read descriptors and the CSR
    p.heads = e.heads_tex ? e.d_heads : nullptr;
    p.heads_tex = e.heads_tex;
    p.long_words = e.long_words;
    p.tokens_tex = e.tokens_tex;
    return p;
}

// A linear texture of uint4 texels over `bytes` of device memory, or 0 when the buffer is
// wider than the device's 1D linear texture limit (the kernels then gather with LDG).
unsigned long long make_linear_tex(const void* ptr, size_t bytes) {
    int dev = 0, max_w = 0;
    if (!ptr || !bytes || cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_w, cudaDevAttrMaxTexture1DLinearWidth, dev) != cudaSuccess)
        return 0;
    if (bytes / sizeof(uint4) > (size_t)max_w || bytes / sizeof(uint4) > 0x7FFFFFFFull) return 0;
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = const_cast<void*>(ptr);
    rd.res.linear.desc = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
    rd.res.linear.sizeInBytes = bytes;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t = 0;
    if (cudaCreateTextureObject(&t, &rd, &td, nullptr) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return (unsigned long long)t;
}

// Packed set heads (verify_kernels.cuh) for the run kernel; left null when some token is
// too large for the packing (the kernels then read descriptors and the CSR instead).
int build_heads(ssj_engine& e) {
    if (!e.n_sets) return SSJ_OK;
    unsigned* d_max = nullptr;
    SSJ_CK(cudaMalloc(&e.d_heads, (size_t)e.n_sets * 2 * sizeof(uint4)));
    SSJ_CK(cudaMalloc(&d_max, sizeof(unsigned)));
    SSJ_CK(cudaMemset(d_max, 0, sizeof(unsigned)));
    SSJ_CK(ssjb::launch_build_heads(e.d_tokens, e.d_sets, e.n_sets, e.d_heads, d_max, 0));
    unsigned mx = 0;
    SSJ_CK(cudaMemcpy(&mx, d_max, sizeof(unsigned), cudaMemcpyDeviceToHost));
    cudaFree(d_max);
    // the widest probe range (tokens <= mx) bounds the long pass's shared bitmap: bits and
    // ranks of (mx >> 5) + 1 words plus the guard word, rounded to 16 bytes
    if (mx < 0xFFFFFFE0u) {
        const uint64_t w = (((uint64_t)(mx >> 5) + 2) + 3) & ~3ull;
        e.long_words = (uint32_t)std::min<uint64_t>(w, ssjb::kMaxBitmapWords);
    }
    if (mx >= ssjb::kHeadTokenLimit) {
        cudaFree(e.d_heads);
        e.d_heads = nullptr;
    }
    e.heads_tex = make_linear_tex(e.d_heads, (size_t)e.n_sets * 2 * sizeof(uint4));
    e.tokens_tex = make_linear_tex(e.d_tokens, (size_t)e.n_padded * sizeof(uint32_t));
    return SSJ_OK;
}

// Cosine (similarity.hpp:93-102): the reference searches k with u128 products k^2 den^2 and
// num^2 r s. They are exact while num * max_size + den < 2^64 (then k <= num sqrt(r s) / den
// + 1 and every product is < 2^128); beyond that the reference's own arithmetic wraps, so
// such a threshold is refused instead of being reproduced. Inside the range the device's
// double-precision start value est - 2 is below the answer (est < 2^32, relative error
// < 2^-50), so its upward search ends on the reference's k exactly.
int check_cosine_range(const ssj_predicate& p, uint32_t max_size) {
    if (p.function != SSJ_COSINE) return SSJ_OK;
    if ((u128)p.num * max_size + p.den >= ((u128)1 << 64))
        return fail(SSJ_ERR_INVALID_ARGUMENT,
                    "Cosine threshold num * max set size overflows the reference's u128 "
                    "arithmetic (similarity.hpp:93-102)");
    return SSJ_OK;
}

// Jaccard and Dice: equivalent_overlap depends on |r| + |s| only (similarity.hpp:113-118),
// so the kernels read it from a table built here with the exact u128 formula.
int build_req_table(ssj_engine& e, uint32_t max_size) {
    if (e.hpred.function != SSJ_JACCARD && e.hpred.function != SSJ_DICE) return SSJ_OK;
    const uint64_t n = 2ull * max_size + 1;
    if (n > (1ull << 22)) return SSJ_OK;  // formula path for huge sets
    std::vector<uint32_t> tab(n);
    for (uint64_t sum = 0; sum < n; ++sum) {
        const uint64_t req = ssj_equivalent_overlap(&e.hpred, sum, 0);
        if (req > 0xFFFFFFFFull) return SSJ_OK;
        tab[sum] = (uint32_t)req;
    }
    SSJ_CK(cudaMalloc(&e.d_req_tab, n * sizeof(uint32_t)));
    SSJ_CK(cudaMemcpy(e.d_req_tab, tab.data(), n * sizeof(uint32_t), cudaMemcpyHostToDevice));
    e.req_tab_n = (uint32_t)n;
    return SSJ_OK;
}

// Upload helper: host -> device on stream st. Pinned memory goes straight to the DMA
// engine; pageable memory is staged through the engine's two pinned bounce buffers.
int upload(ssj_engine& e, void* dst, const void* src, size_t bytes, cudaStream_t st, bool pinned,
           int* bounce_turn) {
    if (bytes == 0) return SSJ_OK;
    if (pinned) {
        SSJ_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return SSJ_OK;
    }
    const size_t piece = 8u << 20;
    size_t done = 0;
    while (done < bytes) {
        const size_t n = std::min(piece, bytes - done);
        const int b = (*bounce_turn)++ & 1;
        SSJ_CK(cudaEventSynchronize(e.bounce_ev[b]));
        int rc = ensure_pinned(&e.bounce[b], &e.bounce_cap[b], piece / 4);
        if (rc) return rc;
        std::memcpy(e.bounce[b], static_cast<const char*>(src) + done, n);
        SSJ_CK(cudaMemcpyAsync(static_cast<char*>(dst) + done, e.bounce[b], n,
                               cudaMemcpyHostToDevice, st));
        SSJ_CK(cudaEventRecord(e.bounce_ev[b], st));
        done += n;
    }
    return SSJ_OK;
}

// Bitmap words reserved per chunk for strategy A's probe bitmaps (overflow falls back to
// the merge path, so this only bounds memory, never correctness).
uint64_t bitmap_words_for(uint64_t nC) { return std::max<uint64_t>(4ull << 20, nC / 8); }

int ensure_tile_scratch(ssjb::SliceDesc** slices, size_t* capS, uint32_t** bits, size_t* capB,
                        uint32_t** rank, size_t* capR, uint32_t** list, size_t* capL,
                        uint32_t n_slices, uint64_t nC) {
    int rc;
    if ((rc = ensure_device(slices, capS, std::max<size_t>(n_slices, 1)))) return rc;
    if ((rc = ensure_device(list, capL, std::max<size_t>(n_slices, 1)))) return rc;
    const uint64_t words = bitmap_words_for(nC);
    if ((rc = ensure_device(bits, capB, words))) return rc;
    if ((rc = ensure_device(rank, capR, words))) return rc;
    return SSJ_OK;
}

// want_stats = false: the caller reports no VerifyStats (the all-GPU join), so the kernels
// skip their per-pair stats accumulation. fork: warp_tile_kernel beside run_kernel on the
// engine's aux stream (device-resident chunks; the host path's pieces already overlap their
// copies with the kernels, and measured slower with the fork: cfg2 e2e 12.6 vs 13.3 G/s)
cudaError_t launch_strategy(const ssj_engine& e, const KParams& p, int out, uint32_t tile_begin,
                            uint32_t tile_end, cudaStream_t st, bool want_stats = true,
                            bool fork = true) {
    const bool stats = want_stats && e.strategy.kind != SSJ_STRATEGY_C;
    switch (e.exec.kind) {
        case SSJ_STRATEGY_B: return ssjb::launch_block(p, out, stats, e.exec.group_size, st);
        case SSJ_STRATEGY_C: return ssjb::launch_path(p, out, e.exec.group_size, st);
        default: {
            cudaError_t err = ssjb::launch_tiles(p, out, stats, tile_begin, tile_end, st,
                                                 SSJB_TILES_FORK && fork ? e.s_aux : nullptr, e.ev_fork,
                                                 e.ev_join);
            if (err != cudaSuccess) return err;
            // no set longer than kLongPair: no pair is deferred, nothing for the long pass
            if (e.max_set_size <= ssjb::kLongPair) return cudaSuccess;
            return ssjb::launch_long(p, out, stats, tile_begin, tile_end, st);
        }
    }
}

int check_chunk_args(const ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                     uint64_t nCO) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (nC && !C) return fail(SSJ_ERR_INVALID_ARGUMENT, "null C with nC > 0");
    if (nCO >= 2 && !C_O) return fail(SSJ_ERR_INVALID_ARGUMENT, "null C_O with nCO > 0");
    if (nCO / 2 > 0xFFFFFFFFull) return fail(SSJ_ERR_INVALID_ARGUMENT, "too many slices");
    if (nC > 0xFFFFFFFFull)  // C_O end offsets are u32 (chunk.hpp:20-28)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "chunk too large: C_O offsets are 32-bit");
    return SSJ_OK;
}

int decode_error(unsigned long long bits) {
    if (bits & ssjb::kErrOutOfRange) return fail(SSJ_ERR_OUT_OF_RANGE, "set index out of range");
    if (bits & ssjb::kErrBadOffsets)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "malformed C_O: end offsets decreasing or beyond C");
    return SSJ_OK;
}

// Enqueue one chunk (host buffers) on slot s. out = kOutFlags / kOutCount / kOutResults.
int enqueue_chunk(ssj_engine& e, ChunkSlot& s, const uint32_t* C, uint64_t nC,
                  const uint32_t* C_O, uint64_t nCO, uint8_t* flags_out, int out) {
    const uint32_t n_slices = (uint32_t)(nCO / 2);
    const uint32_t n_tiles = (uint32_t)((nC + ssjb::kTile - 1) / ssjb::kTile);
    int rc;
    if ((rc = ensure_device(&s.dC, &s.capC, nC))) return rc;
    if ((rc = ensure_device(&s.dCO, &s.capCO, (size_t)n_slices * 2))) return rc;
    if ((rc = ensure_device(&s.dtile, &s.capT, (size_t)n_tiles + 1))) return rc;
    if (out == ssjb::kOutFlags && (rc = ensure_device(&s.dflags, &s.capF, nC))) return rc;
    const bool tiles = e.exec.kind == SSJ_STRATEGY_A;
    if (tiles && (rc = ensure_tile_scratch(&s.dslices, &s.capS, &s.dbits, &s.capB, &s.drank,
                                           &s.capR, &s.dbmlist, &s.capBL, n_slices, nC)))
        return rc;
    if (tiles && (rc = ensure_device(&s.ddefer, &s.capDf, std::max<size_t>(nC, 1)))) return rc;
    if (tiles && (rc = ensure_device(&s.druns, &s.capRu, 2 * (size_t)n_tiles + 2))) return rc;
    if (tiles && (rc = ensure_device(&s.dshort, &s.capSh, (size_t)n_tiles + 1))) return rc;
    if (out == ssjb::kOutResults) {
        if ((rc = ensure_device(&e.d_res_slots, &e.res_cap, nC))) return rc;
        if ((rc = ensure_device(&e.d_res_ov, &e.res_cap2, nC))) return rc;
    }

    s.user_flags = nullptr;
    s.flags_staged = false;
    s.nC = nC;
    const bool flags_pinned = out == ssjb::kOutFlags && is_pinned(flags_out);
    if (out == ssjb::kOutFlags) {
        s.user_flags = flags_out;
        if (!flags_pinned) {
            if ((rc = ensure_pinned(&s.hflags, &s.capHF, nC))) return rc;
            s.flags_staged = true;
        }
    }
    const bool c_pinned = nC == 0 || is_pinned(C);
    const bool co_pinned = n_slices == 0 || is_pinned(C_O);

    KParams p = base_params(e);
    p.C = s.dC;
    p.nC = nC;
    p.C_O = s.dCO;
    p.n_slices = n_slices;
    p.tile_first = s.dtile;
    p.n_tiles = n_tiles;
    p.flags = s.dflags;
    p.res_slots = e.d_res_slots;
    p.res_ov = e.d_res_ov;
    p.res_n = e.d_res_n;
    p.res_cap = nC;
    p.acc = s.dacc;
    if (tiles) {
        p.slices = s.dslices;
        p.bm_bits = s.dbits;
        p.bm_rank = s.drank;
        p.bm_list = s.dbmlist;
        p.bm_cap = bitmap_words_for(nC);
    }

    // Pieces of the slot range: H2D(piece q+1) overlaps verify(piece q) overlaps D2H(q-1).
    // Strategies B and C map CTAs to slices, so they take the chunk as one piece.
    uint64_t piece = nC;
    if (e.exec.kind == SSJ_STRATEGY_A) {
        piece = std::max<uint64_t>(kPieceMinSlots, (nC + kMaxPieces - 1) / kMaxPieces);
        piece = (piece + ssjb::kRun - 1) / ssjb::kRun * ssjb::kRun;  // runs never straddle pieces
    }
    if (piece == 0) piece = 1;
    // per-piece counters of the work lists prep builds, then (one piece) the look-back words
    // of its ordered run list
    const size_t lb_words = 1 + ((size_t)n_slices + 255) / 256;
    const size_t ctr_words = (size_t)kCounters * kMaxPieces + lb_words;
    if (tiles) {
        if ((rc = ensure_device(&s.ddefer_n, &s.capCtr, ctr_words))) return rc;
        p.seg_slots = piece;
        p.runs_all = s.druns;
        p.short_all = s.dshort;
        p.ctr_all = s.ddefer_n;
        p.lb_status = s.ddefer_n + (size_t)kCounters * kMaxPieces;
    }

    int ev = 0;
    int turn = 0;
    SSJ_CK(cudaMemsetAsync(s.dacc, 0, SSJ_RESULT_WORDS * sizeof(unsigned long long), e.s_comp));
    // strategies B and C walk the slices only: slots past the last C_O end keep flag 0
    // (strategy A's tiles write those flags themselves)
    if (!tiles && out == ssjb::kOutFlags && nC)
        SSJ_CK(cudaMemsetAsync(s.dflags, 0, nC, e.s_comp));
    if (tiles)
        SSJ_CK(cudaMemsetAsync(s.ddefer_n, 0, ctr_words * sizeof(unsigned long long), e.s_comp));
    if (out == ssjb::kOutResults)
        SSJ_CK(cudaMemsetAsync(e.d_res_n, 0, sizeof(unsigned long long), e.s_comp));
    if ((rc = upload(e, s.dCO, C_O, (size_t)n_slices * 2 * sizeof(uint32_t), e.s_comp, co_pinned,
                     &turn)))
        return rc;
    SSJ_CK(ssjb::launch_prep(p, e.s_comp));

    for (uint64_t lo = 0; lo < nC || (lo == 0 && nC == 0); lo += piece) {
        const uint64_t hi = std::min(nC, lo + piece);
        if (hi > lo) {
            if ((rc = upload(e, s.dC + lo, C + lo, (hi - lo) * sizeof(uint32_t), e.s_h2d, c_pinned,
                             &turn)))
                return rc;
            SSJ_CK(cudaEventRecord(s.ev[ev], e.s_h2d));
            SSJ_CK(cudaStreamWaitEvent(e.s_comp, s.ev[ev], 0));
            ++ev;
        }
        const uint32_t t0 = (uint32_t)(lo / ssjb::kTile);
        const uint32_t t1 = (uint32_t)((hi + ssjb::kTile - 1) / ssjb::kTile);
        if (tiles) {  // this piece's long pairs: their own segment and counter
            const int pc = (int)(lo / piece);
            p.defer = s.ddefer + lo;
            p.defer_n = s.ddefer_n + kCounters * pc;
            p.seg_tag = (uint32_t)pc + 1;
            p.defer_cap = hi - lo;
            p.runs = s.druns + 2 * (size_t)t0;
            p.runs_n = s.ddefer_n + kCounters * pc + 1;
            p.runs_cap = 2 * (uint64_t)(t1 - t0);
            p.short_tiles = s.dshort + t0;
            p.short_n = s.ddefer_n + kCounters * pc + 2;
            p.short_cap = t1 - t0;
        }
        SSJ_CK(launch_strategy(e, p, out, t0, t1, e.s_comp, true, false));
        if (out == ssjb::kOutFlags && hi > lo) {
            SSJ_CK(cudaEventRecord(s.ev[ev], e.s_comp));
            SSJ_CK(cudaStreamWaitEvent(e.s_d2h, s.ev[ev], 0));
            ++ev;
            uint8_t* dst = (s.flags_staged ? s.hflags : flags_out) + lo;
            SSJ_CK(cudaMemcpyAsync(dst, s.dflags + lo, hi - lo, cudaMemcpyDeviceToHost, e.s_d2h));
        }
        if (ev + 2 >= kEventsPerSlot) return fail(SSJ_ERR_RUNTIME, "too many pieces");
        if (nC == 0) break;
    }
    SSJ_CK(cudaEventRecord(s.ev[ev], e.s_comp));
    SSJ_CK(cudaStreamWaitEvent(e.s_d2h, s.ev[ev], 0));
    SSJ_CK(cudaMemcpyAsync(s.hacc, s.dacc, SSJ_RESULT_WORDS * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, e.s_d2h));
    SSJ_CK(cudaEventRecord(s.done, e.s_d2h));
    return SSJ_OK;
}

int finish_chunk(ssj_engine& e, ChunkSlot& s, uint64_t* count_out, ssj_stats* stats) {
    SSJ_CK(cudaEventSynchronize(s.done));
    s.busy = false;
    int rc = decode_error(s.hacc[SSJ_RESULT_ERROR]);
    if (rc) return rc;
    if (s.flags_staged && s.user_flags) std::memcpy(s.user_flags, s.hflags, s.nC);
    if (count_out) *count_out = s.hacc[SSJ_RESULT_COUNT];
    if (stats && e.strategy.kind != SSJ_STRATEGY_C) {
        stats->pairs_verified += s.hacc[SSJ_RESULT_STATS + 0];
        stats->early_exit_prunes += s.hacc[SSJ_RESULT_STATS + 1];
        stats->comparison_budget_violations += s.hacc[SSJ_RESULT_STATS + 2];
    }
    return SSJ_OK;
}

void destroy_slot(ChunkSlot& s) {
    cudaFree(s.dC);
    cudaFree(s.dCO);
    cudaFree(s.dflags);
    cudaFree(s.dtile);
    cudaFree(s.dslices);
    cudaFree(s.dbits);
    cudaFree(s.drank);
    cudaFree(s.ddefer);
    cudaFree(s.ddefer_n);
    cudaFree(s.druns);
    cudaFree(s.dbmlist);
    cudaFree(s.dshort);
    cudaFree(s.dacc);
    cudaFreeHost(s.hacc);
    cudaFreeHost(s.hflags);
    for (auto& ev : s.ev)
        if (ev) cudaEventDestroy(ev);
    if (s.done) cudaEventDestroy(s.done);
}

int init_engine_runtime(ssj_engine& e) {
    SSJ_CK(cudaStreamCreateWithFlags(&e.s_comp, cudaStreamNonBlocking));
    SSJ_CK(cudaStreamCreateWithFlags(&e.s_h2d, cudaStreamNonBlocking));
    SSJ_CK(cudaStreamCreateWithFlags(&e.s_d2h, cudaStreamNonBlocking));
    SSJ_CK(cudaStreamCreateWithFlags(&e.s_aux, cudaStreamNonBlocking));
    SSJ_CK(cudaEventCreateWithFlags(&e.ev_fork, cudaEventDisableTiming));
    SSJ_CK(cudaEventCreateWithFlags(&e.ev_join, cudaEventDisableTiming));
    for (auto& s : e.slot) {
        for (auto& ev : s.ev) SSJ_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        SSJ_CK(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
        SSJ_CK(cudaMalloc(&s.dacc, SSJ_RESULT_WORDS * sizeof(unsigned long long)));
        SSJ_CK(cudaHostAlloc(&s.hacc, SSJ_RESULT_WORDS * sizeof(unsigned long long),
                             cudaHostAllocDefault));
    }
    for (auto& ev : e.bounce_ev) SSJ_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SSJ_CK(cudaMalloc(&e.d_res_n, sizeof(unsigned long long)));
    return SSJ_OK;
}

int validate_engine_args(const ssj_predicate* pred, int32_t mode, const ssj_strategy* strategy) {
    if (!pred || !strategy) return fail(SSJ_ERR_INVALID_ARGUMENT, "null predicate or strategy");
    int rc = ssj_predicate_validate(pred);
    if (rc) return rc;
    if ((rc = ssj_strategy_validate(strategy))) return rc;
    if (mode != SSJ_MODE_COUNT && mode != SSJ_MODE_PAIRS)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "bad output mode");
    return SSJ_OK;
}

int check_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(SSJ_ERR_NO_DEVICE,
                    "no CUDA device: the B200 verification engine has no CPU fallback");
    }
    if (device < 0 || device >= n) return fail(SSJ_ERR_INVALID_ARGUMENT, "bad device ordinal");
    return SSJ_OK;
}

}  // namespace

extern "C" {

int ssj_abi_version(void) { return SSJ_ABI_VERSION; }
const char* ssj_last_error(void) { return g_err.c_str(); }

int ssj_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int ssj_threshold_parse(const char* text, uint64_t* num_out, uint64_t* den_out) {
    // similarity.hpp:30-56 (Threshold::parse) and :58-62 (reduce).
    if (!text || !num_out || !den_out) return fail(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    const std::string t(text);
    if (t.empty()) return fail(SSJ_ERR_INVALID_ARGUMENT, "empty threshold");
    auto digits = [](const std::string& d, uint64_t* v) {
        // std::stoull: optional leading whitespace/sign are not produced by this grammar;
        // requires at least one leading digit and ignores trailing characters.
        size_t k = 0;
        uint64_t x = 0;
        while (k < d.size() && d[k] >= '0' && d[k] <= '9') x = x * 10 + (uint64_t)(d[k++] - '0');
        if (k == 0) return false;
        *v = x;
        return true;
    };
    uint64_t num = 0, den = 1;
    const size_t slash = t.find('/');
    if (slash != std::string::npos) {
        if (!digits(t.substr(0, slash), &num) || !digits(t.substr(slash + 1), &den))
            return fail(SSJ_ERR_INVALID_ARGUMENT, "bad threshold: " + t);
    } else {
        const size_t dot = t.find('.');
        std::string ip = t.substr(0, dot);
        if (ip.empty()) ip = "0";
        if (!digits(ip, &num)) return fail(SSJ_ERR_INVALID_ARGUMENT, "bad threshold: " + t);
        if (dot != std::string::npos) {
            for (size_t i = dot + 1; i < t.size(); ++i) {
                const char c = t[i];
                if (c < '0' || c > '9') return fail(SSJ_ERR_INVALID_ARGUMENT, "bad threshold: " + t);
                num = num * 10 + (uint64_t)(c - '0');
                den *= 10;
            }
        }
    }
    if (den == 0) return fail(SSJ_ERR_INVALID_ARGUMENT, "bad threshold: " + t);
    uint64_t a = num, b = den;
    while (b) {
        const uint64_t r = a % b;
        a = b;
        b = r;
    }
    if (a > 1) {
        num /= a;
        den /= a;
    }
    *num_out = num;
    *den_out = den;
    return SSJ_OK;
}

int ssj_predicate_validate(const ssj_predicate* p) {
    // similarity.hpp:74-81
    if (!p) return fail(SSJ_ERR_INVALID_ARGUMENT, "null predicate");
    if (p->function < SSJ_JACCARD || p->function > SSJ_OVERLAP)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "unknown similarity function");
    if (p->function != SSJ_OVERLAP) {
        if (p->num == 0 || p->num > p->den)
            return fail(SSJ_ERR_INVALID_ARGUMENT, "normalized threshold must be in (0,1]");
    } else if (p->overlap_threshold < 1) {
        return fail(SSJ_ERR_INVALID_ARGUMENT, "overlap threshold must be >= 1");
    }
    return SSJ_OK;
}

int ssj_strategy_validate(const ssj_strategy* s) {
    // verify.hpp:25-28
    if (!s) return fail(SSJ_ERR_INVALID_ARGUMENT, "null strategy");
    if (s->kind < SSJ_STRATEGY_A || s->kind > SSJ_STRATEGY_AUTO)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "unknown strategy kind");
    if (s->group_size < 1 || (s->group_size & (s->group_size - 1)) != 0)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "group size must be a power of two");
    return SSJ_OK;
}

uint64_t ssj_equivalent_overlap(const ssj_predicate* p, uint64_t r, uint64_t s) {
    // similarity.hpp:108-123 (host copy of the device formula in ssj_device.cuh)
    const uint64_t num = p->num, den = p->den;
    switch (p->function) {
        case SSJ_JACCARD: return host_ceil_div((u128)num * (r + s), den + num);
        case SSJ_DICE: return host_ceil_div((u128)num * (r + s), 2 * den);
        case SSJ_OVERLAP: return p->overlap_threshold;
        case SSJ_COSINE: {
            u128 rhs = (u128)num * num * r * s;
            if (rhs == 0) return 0;
            long double est = (long double)num / den * sqrtl((long double)r * (long double)s);
            uint64_t k = est > 2.0L ? (uint64_t)est - 2 : 0;
            while ((u128)k * k * den * den < rhs) ++k;
            return k;
        }
    }
    return 0;
}

int ssj_engine_create(ssj_engine** out, int device, const uint32_t* tokens, const uint32_t* offsets,
                      uint32_t n_sets, const ssj_predicate* pred, int32_t mode,
                      const ssj_strategy* strategy) {
    if (!out) return fail(SSJ_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    int rc = validate_engine_args(pred, mode, strategy);
    if (rc) return rc;
    if (!offsets) return fail(SSJ_ERR_INVALID_ARGUMENT, "null offsets");
    if (n_sets && offsets[n_sets] && !tokens) return fail(SSJ_ERR_INVALID_ARGUMENT, "null tokens");
    for (uint32_t i = 0; i < n_sets; ++i)
        if (offsets[i + 1] < offsets[i])
            return fail(SSJ_ERR_INVALID_ARGUMENT, "offsets must be non-decreasing");
    if ((rc = check_device(device))) return rc;
    DeviceScope ds(device);

    auto* e = new ssj_engine;
    e->device = device;
    e->hpred = *pred;
    e->mode = mode;
    e->n_sets = n_sets;
    e->n_tokens = n_sets ? (uint64_t)offsets[n_sets] - offsets[0] : 0;
    if ((rc = make_pred_dev(*pred, &e->pred))) {
        delete e;
        return rc;
    }
    resolve_strategy(*e, *strategy);

    // Padded CSR: every set starts on a 32-byte boundary; SSJ_TOKEN_TAIL_PAD sentinel tokens
    // at the end so that the kernels' speculative reads past a set's end (32-byte head reads,
    // the long pass's next-step prefetch) stay in bounds.
    std::vector<uint2> sets(n_sets ? n_sets : 1);
    uint64_t pos = 0;
    for (uint32_t i = 0; i < n_sets; ++i) {
        const uint32_t sz = offsets[i + 1] - offsets[i];
        sets[i] = make_uint2((uint32_t)(pos / 8), sz);
        pos += (uint64_t)(sz + 7u) & ~7ull;
    }
    if (pos / 8 >= 0xFFFFFFFFull) {
        delete e;
        return fail(SSJ_ERR_INVALID_ARGUMENT, "collection too large for u32 set positions");
    }
    e->n_padded = pos + SSJ_TOKEN_TAIL_PAD;
    std::vector<uint32_t> padded(e->n_padded, 0xFFFFFFFFu);
    for (uint32_t i = 0; i < n_sets; ++i) {
        const uint32_t sz = offsets[i + 1] - offsets[i];
        if (sz) std::memcpy(&padded[(size_t)sets[i].x * 8], tokens + offsets[i], sz * sizeof(uint32_t));
    }
    auto cleanup = [&](int code) {
        ssj_engine_destroy(e);
        return code;
    };
    if ((rc = init_engine_runtime(*e))) return cleanup(rc);
    if (cudaMalloc(&e->d_tokens, e->n_padded * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&e->d_sets, sets.size() * sizeof(uint2)) != cudaSuccess)
        return cleanup(fail(SSJ_ERR_CUDA, "cudaMalloc of the collection failed"));
    if (cudaMemcpy(e->d_tokens, padded.data(), e->n_padded * sizeof(uint32_t),
                   cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(e->d_sets, sets.data(), sets.size() * sizeof(uint2), cudaMemcpyHostToDevice) !=
            cudaSuccess)
        return cleanup(fail(SSJ_ERR_CUDA, "collection upload failed"));
    uint32_t max_size = 0;
    for (uint32_t i = 0; i < n_sets; ++i) max_size = std::max(max_size, offsets[i + 1] - offsets[i]);
    e->max_set_size = max_size;
    if ((rc = check_cosine_range(*pred, max_size))) return cleanup(rc);
    if ((rc = build_req_table(*e, max_size))) return cleanup(rc);
    if ((rc = build_heads(*e))) return cleanup(rc);
    *out = e;
    return SSJ_OK;
}

int ssj_engine_create_from_device(ssj_engine** out, int device, const uint32_t* d_tokens,
                                  uint64_t n_padded_tokens, const uint32_t* d_sets, uint32_t n_sets,
                                  uint64_t n_tokens_total, const ssj_predicate* pred, int32_t mode,
                                  const ssj_strategy* strategy) {
    if (!out) return fail(SSJ_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    int rc = validate_engine_args(pred, mode, strategy);
    if (rc) return rc;
    if (!d_tokens || !d_sets) return fail(SSJ_ERR_INVALID_ARGUMENT, "null device collection");
    if ((rc = check_device(device))) return rc;
    DeviceScope ds(device);
    auto* e = new ssj_engine;
    e->device = device;
    e->hpred = *pred;
    e->mode = mode;
    e->n_sets = n_sets;
    e->n_tokens = n_tokens_total;
    e->n_padded = n_padded_tokens;
    e->owns_collection = false;
    e->d_tokens = const_cast<uint32_t*>(d_tokens);
    e->d_sets = reinterpret_cast<uint2*>(const_cast<uint32_t*>(d_sets));
    if (n_sets) {  // the last set (largest position) must be followed by the tail pad
        uint2 last{};
        if (cudaMemcpy(&last, e->d_sets + (n_sets - 1), sizeof(uint2), cudaMemcpyDeviceToHost) !=
                cudaSuccess ||
            (uint64_t)last.x * 8 + (((uint64_t)last.y + 7) & ~7ull) + SSJ_TOKEN_TAIL_PAD >
                n_padded_tokens) {
            delete e;
            return fail(SSJ_ERR_INVALID_ARGUMENT,
                        "device collection is not in the engine's padded layout (tail pad)");
        }
    }
    if ((rc = make_pred_dev(*pred, &e->pred))) {
        delete e;
        return rc;
    }
    resolve_strategy(*e, *strategy);
    if ((rc = init_engine_runtime(*e))) {
        ssj_engine_destroy(e);
        return rc;
    }
    if (n_sets && e->hpred.function != SSJ_OVERLAP) {
        std::vector<uint2> sets(n_sets);
        if (cudaMemcpy(sets.data(), d_sets, n_sets * sizeof(uint2), cudaMemcpyDeviceToHost) !=
            cudaSuccess) {
            ssj_engine_destroy(e);
            return fail(SSJ_ERR_CUDA, "reading set descriptors failed");
        }
        uint32_t max_size = 0;
        for (const auto& sd : sets) max_size = std::max(max_size, sd.y);
        e->max_set_size = max_size;
        if ((rc = check_cosine_range(*pred, max_size)) || (rc = build_req_table(*e, max_size))) {
            ssj_engine_destroy(e);
            return rc;
        }
    }
    if ((rc = build_heads(*e))) {
        ssj_engine_destroy(e);
        return rc;
    }
    *out = e;
    return SSJ_OK;
}

int ssj_engine_create_multi(ssj_engine** out, const int32_t* devices, uint32_t n_devices,
                            const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                            const ssj_predicate* pred, int32_t mode, const ssj_strategy* strategy) {
    if (!out) return fail(SSJ_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    if (!devices || n_devices == 0) return fail(SSJ_ERR_INVALID_ARGUMENT, "empty device list");
    int rc = validate_engine_args(pred, mode, strategy);
    if (rc) return rc;
    if (!offsets) return fail(SSJ_ERR_INVALID_ARGUMENT, "null offsets");
    for (uint32_t i = 0; i < n_devices; ++i)
        if ((rc = check_device(devices[i]))) return rc;
    DeviceScope ds(devices[0]);
    ssjm::Group* g = nullptr;
    if ((rc = ssjm::create_group(&g, devices, n_devices, tokens, offsets, n_sets, pred, mode,
                                 strategy)))
        return rc;
    auto* e = new ssj_engine;
    ssj_engine* e0 = ssjm::first(*g);
    e->group = g;
    e->device = devices[0];
    e->hpred = *pred;
    e->pred = e0->pred;
    e->mode = mode;
    e->strategy = e0->strategy;
    e->exec = e0->exec;
    e->n_sets = n_sets;
    e->n_tokens = e0->n_tokens;
    e->n_padded = e0->n_padded;
    e->max_set_size = e0->max_set_size;
    e->owns_collection = false;
    *out = e;
    return SSJ_OK;
}

int ssj_engine_devices(const ssj_engine* e, int32_t* devices, uint32_t cap, uint32_t* n_devices,
                       double* fanout_ms) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (e->group) return ssjm::devices(*e->group, devices, cap, n_devices, fanout_ms);
    if (n_devices) *n_devices = 1;
    if (devices && cap) devices[0] = e->device;
    if (fanout_ms) *fanout_ms = 0;
    return SSJ_OK;
}

int ssj_chunk_split(const uint32_t* set_sizes, uint32_t n_sets, uint32_t parts, const uint32_t* C_O,
                    uint64_t nCO, uint64_t nC, uint64_t* ranges) {
    if (!parts || !ranges || (n_sets && !set_sizes) || (nCO >= 2 && !C_O))
        return fail(SSJ_ERR_INVALID_ARGUMENT, "null argument or zero parts");
    std::vector<uint32_t> sizes(set_sizes, set_sizes + n_sets);
    std::vector<ssjm::Range> rg;
    int rc = ssjm::split_chunk(sizes, parts, C_O, nCO, nC, &rg);
    if (rc) return rc;
    for (uint32_t g = 0; g < parts; ++g) {
        ranges[4 * g] = rg[g].slice_begin;
        ranges[4 * g + 1] = rg[g].slice_end;
        ranges[4 * g + 2] = rg[g].c_lo;
        ranges[4 * g + 3] = rg[g].c_hi;
    }
    return SSJ_OK;
}

int ssj_engine_device_collection(const ssj_engine* e, const uint32_t** d_tokens,
                                 uint64_t* n_padded_tokens, const uint32_t** d_sets) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (e->group)  // the first device's copy
        return ssj_engine_device_collection(ssjm::first(*e->group), d_tokens, n_padded_tokens, d_sets);
    if (d_tokens) *d_tokens = e->d_tokens;
    if (n_padded_tokens) *n_padded_tokens = e->n_padded;
    if (d_sets) *d_sets = reinterpret_cast<const uint32_t*>(e->d_sets);
    return SSJ_OK;
}

void ssj_engine_destroy(ssj_engine* e) {
    if (!e) return;
    if (e->group) {
        ssjm::destroy_group(e->group);
        delete e;
        return;
    }
    DeviceScope ds(e->device);
    if (e->s_comp) cudaStreamSynchronize(e->s_comp);
    if (e->s_h2d) cudaStreamSynchronize(e->s_h2d);
    if (e->s_d2h) cudaStreamSynchronize(e->s_d2h);
    for (auto& s : e->slot) destroy_slot(s);
    for (int b = 0; b < 2; ++b) {
        cudaFreeHost(e->bounce[b]);
        if (e->bounce_ev[b]) cudaEventDestroy(e->bounce_ev[b]);
    }
    if (e->owns_collection) {
        cudaFree(e->d_tokens);
        cudaFree(e->d_sets);
    }
    cudaFree(e->dev_tile);
    cudaFree(e->dev_slices);
    cudaFree(e->dev_bits);
    cudaFree(e->dev_rank);
    cudaFree(e->dev_defer);
    cudaFree(e->dev_defer_n);
    cudaFree(e->dev_runs);
    cudaFree(e->dev_bmlist);
    cudaFree(e->dev_short);
    cudaFree(e->d_req_tab);
    if (e->heads_tex) cudaDestroyTextureObject((cudaTextureObject_t)e->heads_tex);
    if (e->tokens_tex) cudaDestroyTextureObject((cudaTextureObject_t)e->tokens_tex);
    cudaFree(e->d_heads);
    if (e->fidx) {
        ssjb::filter_index_free(e->fidx);
        delete e->fidx;
    }
    delete e->gen;
    if (e->gidx) {
        ssjb::group_index_free(e->gidx);
        delete e->gidx;
    }
    delete e->gen_g;
    cudaFree(e->d_res_slots);
    cudaFree(e->d_res_ov);
    cudaFree(e->d_res_n);
    cudaFree(e->d_oid);
    cudaFree(e->d_keys);
    cudaFree(e->d_keys_alt);
    cudaFree(e->d_ov_alt);
    cudaFree(e->d_slot_alt);
    cudaFree(e->d_sort_tmp);
    for (auto& pe : e->prof_events) {
        cudaEventDestroy(pe.first);
        cudaEventDestroy(pe.second);
    }
    if (e->s_comp) cudaStreamDestroy(e->s_comp);
    if (e->s_h2d) cudaStreamDestroy(e->s_h2d);
    if (e->s_d2h) cudaStreamDestroy(e->s_d2h);
    if (e->s_aux) cudaStreamDestroy(e->s_aux);
    if (e->ev_fork) cudaEventDestroy(e->ev_fork);
    if (e->ev_join) cudaEventDestroy(e->ev_join);
    delete e;
}

int ssj_engine_strategy(const ssj_engine* e, ssj_strategy* resolved) {
    if (!e || !resolved) return fail(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    *resolved = e->strategy;
    return SSJ_OK;
}

int ssj_engine_kernel_strategy(const ssj_engine* e, ssj_strategy* exec) {
    if (!e || !exec) return fail(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    *exec = e->exec;
    return SSJ_OK;
}

int ssj_engine_device(const ssj_engine* e) { return e ? e->device : -1; }

int ssj_submit_chunk(ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                     uint64_t nCO, uint8_t* flags_out, uint64_t* ticket) {
    int rc = check_chunk_args(e, C, nC, C_O, nCO);
    if (rc) return rc;
    if (!ticket) return fail(SSJ_ERR_INVALID_ARGUMENT, "null ticket");
    if (e->group) return ssjm::submit(*e->group, C, nC, C_O, nCO, flags_out, ticket);
    DeviceScope ds(e->device);
    const uint64_t t = e->next_ticket;
    ChunkSlot& s = e->slot[t & 1];
    if (s.busy) return fail(SSJ_ERR_RUNTIME, "two chunks already in flight: wait first");
    const int out = (e->mode == SSJ_MODE_PAIRS && flags_out) ? ssjb::kOutFlags : ssjb::kOutCount;
    if ((rc = enqueue_chunk(*e, s, C, nC, C_O, nCO, flags_out, out))) {
        // drain whatever was enqueued so the slot is reusable
        cudaStreamSynchronize(e->s_comp);
        cudaStreamSynchronize(e->s_h2d);
        cudaStreamSynchronize(e->s_d2h);
        return rc;
    }
    s.busy = true;
    s.ticket = t;
    e->next_ticket = t + 1;
    *ticket = t;
    return SSJ_OK;
}

int ssj_wait_chunk(ssj_engine* e, uint64_t ticket, uint64_t* count_out, ssj_stats* stats) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (e->group) return ssjm::wait(*e->group, ticket, count_out, stats);
    DeviceScope ds(e->device);
    ChunkSlot& s = e->slot[ticket & 1];
    if (!s.busy || s.ticket != ticket) return fail(SSJ_ERR_INVALID_ARGUMENT, "unknown ticket");
    return finish_chunk(*e, s, count_out, stats);
}

int ssj_verify_chunk(ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                     uint64_t nCO, uint8_t* flags_out, uint64_t* count_out, ssj_stats* stats) {
    uint64_t t = 0;
    int rc = ssj_submit_chunk(e, C, nC, C_O, nCO, flags_out, &t);
    if (rc) return rc;
    return ssj_wait_chunk(e, t, count_out, stats);
}

int ssj_verify_chunk_results(ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                             uint64_t nCO, uint32_t* slots_out, uint32_t* overlaps_out,
                             uint64_t cap, uint64_t* n_out) {
    int rc = check_chunk_args(e, C, nC, C_O, nCO);
    if (rc) return rc;
    if (!n_out || (cap && (!slots_out || !overlaps_out)))
        return fail(SSJ_ERR_INVALID_ARGUMENT, "null output");
    if (e->group)
        return ssjm::verify_results(*e->group, C, nC, C_O, nCO, slots_out, overlaps_out, cap, n_out);
    DeviceScope ds(e->device);
    ChunkSlot& s = e->slot[e->next_ticket & 1];
    if (s.busy) return fail(SSJ_ERR_RUNTIME, "a chunk is in flight on this slot: wait first");
    if ((rc = enqueue_chunk(*e, s, C, nC, C_O, nCO, nullptr, ssjb::kOutResults))) {
        cudaDeviceSynchronize();
        return rc;
    }
    SSJ_CK(cudaEventSynchronize(s.done));
    if ((rc = decode_error(s.hacc[SSJ_RESULT_ERROR]))) return rc;
    unsigned long long n = 0;
    SSJ_CK(cudaMemcpy(&n, e->d_res_n, sizeof(n), cudaMemcpyDeviceToHost));
    *n_out = n;
    std::vector<uint32_t> sl(n), ov(n);
    if (n) {
        SSJ_CK(cudaMemcpy(sl.data(), e->d_res_slots, n * 4, cudaMemcpyDeviceToHost));
        SSJ_CK(cudaMemcpy(ov.data(), e->d_res_ov, n * 4, cudaMemcpyDeviceToHost));
    }
    // Ascending slot order (the warp-aggregated appends are unordered).
    std::vector<uint64_t> key(n);
    for (uint64_t i = 0; i < n; ++i) key[i] = ((uint64_t)sl[i] << 32) | ov[i];
    std::sort(key.begin(), key.end());
    const uint64_t w = std::min<uint64_t>(n, cap);
    for (uint64_t i = 0; i < w; ++i) {
        slots_out[i] = (uint32_t)(key[i] >> 32);
        overlaps_out[i] = (uint32_t)key[i];
    }
    if (n > cap) return fail(SSJ_ERR_RUNTIME, "result capacity exceeded");
    return SSJ_OK;
}

int ssj_engine_set_original_ids(ssj_engine* e, const uint32_t* original_id) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (e->group) return ssjm::set_original_ids(*e->group, original_id);
    DeviceScope ds(e->device);
    if (!e->d_oid) SSJ_CK(cudaMalloc(&e->d_oid, (size_t)std::max<uint32_t>(e->n_sets, 1) * 4));
    if (original_id) {
        SSJ_CK(cudaMemcpy(e->d_oid, original_id, (size_t)e->n_sets * 4, cudaMemcpyHostToDevice));
    } else {
        std::vector<uint32_t> id(e->n_sets);
        for (uint32_t i = 0; i < e->n_sets; ++i) id[i] = i;
        SSJ_CK(cudaMemcpy(e->d_oid, id.data(), (size_t)e->n_sets * 4, cudaMemcpyHostToDevice));
    }
    return SSJ_OK;
}

int ssj_verify_chunk_pairs(ssj_engine* e, const uint32_t* C, uint64_t nC, const uint32_t* C_O,
                           uint64_t nCO, uint32_t* pairs_out, uint32_t* overlaps_out,
                           uint64_t cap, uint64_t* n_out, int sorted, ssj_stats* stats) {
    int rc = check_chunk_args(e, C, nC, C_O, nCO);
    if (rc) return rc;
    if (!n_out || (cap && !pairs_out)) return fail(SSJ_ERR_INVALID_ARGUMENT, "null output");
    if (e->group)
        return ssjm::verify_pairs(*e->group, C, nC, C_O, nCO, pairs_out, overlaps_out, cap, n_out,
                                  sorted, stats);
    DeviceScope ds(e->device);
    if (!e->d_oid && (rc = ssj_engine_set_original_ids(e, nullptr))) return rc;
    ChunkSlot& s = e->slot[e->next_ticket & 1];
    if (s.busy) return fail(SSJ_ERR_RUNTIME, "a chunk is in flight on this slot: wait first");
    if ((rc = enqueue_chunk(*e, s, C, nC, C_O, nCO, nullptr, ssjb::kOutResults))) {
        cudaDeviceSynchronize();
        return rc;
    }
    if ((rc = finish_chunk(*e, s, nullptr, stats))) return rc;
    unsigned long long n = 0;
    SSJ_CK(cudaMemcpy(&n, e->d_res_n, sizeof(n), cudaMemcpyDeviceToHost));
    *n_out = n;
    if (n) {
        if ((rc = ensure_device(&e->d_keys, &e->keys_cap, n))) return rc;
        auto grow_tmp = [&](size_t need) -> int {
            if (need <= e->sort_tmp_cap) return SSJ_OK;
            cudaFree(e->d_sort_tmp);
            e->d_sort_tmp = nullptr;
            e->sort_tmp_cap = 0;
            SSJ_CK(cudaMalloc(&e->d_sort_tmp, need));
            e->sort_tmp_cap = need;
            return SSJ_OK;
        };
        KParams p = base_params(*e);
        p.C = s.dC;
        p.nC = nC;
        p.C_O = s.dCO;
        p.n_slices = (uint32_t)(nCO / 2);
        p.res_slots = e->d_res_slots;
        uint32_t* ovs = e->d_res_ov;
        if (!sorted) {
            // decode_pairs order (pipeline.hpp:79-92: slices, then slots): the warp-aggregated
            // appends are unordered, so the qualifying slots are radix-sorted first
            if ((rc = ensure_device(&e->d_slot_alt, &e->slot_alt_cap, n))) return rc;
            if ((rc = ensure_device(&e->d_ov_alt, &e->ov_alt_cap, n))) return rc;
            int bits = 1;
            while (bits < 32 && (1ull << bits) < nC) ++bits;
            size_t tmp = 0;
            SSJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, e->d_res_slots, e->d_slot_alt,
                                                   e->d_res_ov, e->d_ov_alt, (int)n, 0, bits,
                                                   e->s_comp));
            if ((rc = grow_tmp(tmp))) return rc;
            SSJ_CK(cub::DeviceRadixSort::SortPairs(e->d_sort_tmp, tmp, e->d_res_slots,
                                                   e->d_slot_alt, e->d_res_ov, e->d_ov_alt,
                                                   (int)n, 0, bits, e->s_comp));
            p.res_slots = e->d_slot_alt;
            ovs = e->d_ov_alt;
        }
        SSJ_CK(ssjb::launch_pairs(p, e->d_oid, n, e->d_keys, e->s_comp));
        unsigned long long* keys = e->d_keys;
        if (sorted) {  // write_pairs order (report.hpp:39-42) by a device radix sort
            if ((rc = ensure_device(&e->d_keys_alt, &e->keys_alt_cap, n))) return rc;
            if ((rc = ensure_device(&e->d_ov_alt, &e->ov_alt_cap, n))) return rc;
            size_t tmp = 0;
            SSJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, e->d_keys, e->d_keys_alt,
                                                   e->d_res_ov, e->d_ov_alt, (int)n, 0, 64,
                                                   e->s_comp));
            if ((rc = grow_tmp(tmp))) return rc;
            SSJ_CK(cub::DeviceRadixSort::SortPairs(e->d_sort_tmp, tmp, e->d_keys, e->d_keys_alt,
                                                   e->d_res_ov, e->d_ov_alt, (int)n, 0, 64,
                                                   e->s_comp));
            keys = e->d_keys_alt;
            ovs = e->d_ov_alt;
        }
        SSJ_CK(cudaStreamSynchronize(e->s_comp));
        const uint64_t w = std::min<uint64_t>(n, cap);
        std::vector<unsigned long long> hk(w);
        if (w) {
            SSJ_CK(cudaMemcpy(hk.data(), keys, w * 8, cudaMemcpyDeviceToHost));
            if (overlaps_out) SSJ_CK(cudaMemcpy(overlaps_out, ovs, w * 4, cudaMemcpyDeviceToHost));
        }
        for (uint64_t i = 0; i < w; ++i) {
            pairs_out[2 * i] = (uint32_t)(hk[i] >> 32);
            pairs_out[2 * i + 1] = (uint32_t)hk[i];
        }
    }
    if (n > cap) return fail(SSJ_ERR_RUNTIME, "result capacity exceeded");
    return SSJ_OK;
}

namespace {

// Verification of a device-resident chunk on stream st (no synchronisation). out = kOutFlags
// (d_flags), kOutCount or kOutResults (qualifying slots/overlaps appended to the engine's
// result buffers; e->d_res_n is zeroed here). d_acc: SSJ_RESULT_WORDS words.
int verify_device(ssj_engine* e, const uint32_t* d_C, uint64_t nC, const uint32_t* d_C_O,
                  uint64_t nCO, int out, uint8_t* d_flags, unsigned long long* d_acc,
                  cudaStream_t st, bool stats = true) {
    int rc;
    const uint32_t n_slices = (uint32_t)(nCO / 2);
    const uint32_t n_tiles = (uint32_t)((nC + ssjb::kTile - 1) / ssjb::kTile);
    if ((rc = ensure_device(&e->dev_tile, &e->dev_tile_cap, (size_t)n_tiles + 1))) return rc;
    const bool tiles = e->exec.kind == SSJ_STRATEGY_A;
    if (tiles && (rc = ensure_tile_scratch(&e->dev_slices, &e->dev_slices_cap, &e->dev_bits,
                                           &e->dev_bits_cap, &e->dev_rank, &e->dev_rank_cap,
                                           &e->dev_bmlist, &e->dev_bmlist_cap,
                                           n_slices, nC)))
        return rc;
    if (tiles && (rc = ensure_device(&e->dev_defer, &e->dev_defer_cap, std::max<size_t>(nC, 1))))
        return rc;
    const size_t ctr_words = tiles ? (size_t)kCounters + 1 + ((size_t)n_slices + 255) / 256 : 0;
    if (tiles && (rc = ensure_device(&e->dev_defer_n, &e->dev_defer_n_cap, ctr_words))) return rc;
    if (tiles && (rc = ensure_device(&e->dev_runs, &e->dev_runs_cap, 2 * (size_t)n_tiles + 2)))
        return rc;
    if (tiles && (rc = ensure_device(&e->dev_short, &e->dev_short_cap, (size_t)n_tiles + 1)))
        return rc;
    if (out == ssjb::kOutResults) {
        if ((rc = ensure_device(&e->d_res_slots, &e->res_cap, std::max<uint64_t>(nC, 1)))) return rc;
        if ((rc = ensure_device(&e->d_res_ov, &e->res_cap2, std::max<uint64_t>(nC, 1)))) return rc;
        if (!e->d_res_n) SSJ_CK(cudaMalloc(&e->d_res_n, sizeof(unsigned long long)));
        SSJ_CK(cudaMemsetAsync(e->d_res_n, 0, sizeof(unsigned long long), st));
    }
    KParams p = base_params(*e);
    p.C = d_C;
    p.nC = nC;
    p.C_O = d_C_O;
    p.n_slices = n_slices;
    p.tile_first = e->dev_tile;
    p.n_tiles = n_tiles;
    p.flags = d_flags;
    p.acc = d_acc;
    if (out == ssjb::kOutResults) {
        p.res_slots = e->d_res_slots;
        p.res_ov = e->d_res_ov;
        p.res_n = e->d_res_n;
        p.res_cap = nC;
    }
    if (tiles) {
        p.slices = e->dev_slices;
        p.bm_bits = e->dev_bits;
        p.bm_rank = e->dev_rank;
        p.bm_list = e->dev_bmlist;
        p.bm_cap = bitmap_words_for(nC);
        p.defer = e->dev_defer;
        p.defer_n = e->dev_defer_n;
        p.seg_tag = 1;
        p.defer_cap = nC;
        p.runs = e->dev_runs;
        p.runs_n = e->dev_defer_n + 1;
        p.runs_cap = 2 * (uint64_t)n_tiles;
        p.short_tiles = e->dev_short;
        p.short_n = e->dev_defer_n + 2;
        p.short_cap = n_tiles;
        p.seg_slots = std::max<uint64_t>(nC, 1);  // one segment
        p.runs_all = e->dev_runs;
        p.short_all = e->dev_short;
        p.ctr_all = e->dev_defer_n;
        p.lb_status = e->dev_defer_n + kCounters;
    }
    // profiling brackets the whole verification of the chunk: result/counter resets, prep
    // (validation, slice descriptors, probe bitmaps) and the strategy's kernels
    cudaEvent_t k0 = nullptr, k1 = nullptr;
    if (e->profiling) {
        if (e->prof_used == e->prof_events.size()) {
            cudaEvent_t a, b;
            SSJ_CK(cudaEventCreate(&a));
            SSJ_CK(cudaEventCreate(&b));
            e->prof_events.push_back({a, b});
        }
        k0 = e->prof_events[e->prof_used].first;
        k1 = e->prof_events[e->prof_used].second;
        ++e->prof_used;
        SSJ_CK(cudaEventRecord(k0, st));
    }
    SSJ_CK(cudaMemsetAsync(d_acc, 0, SSJ_RESULT_WORDS * sizeof(uint64_t), st));
    if (!tiles && out == ssjb::kOutFlags && nC) SSJ_CK(cudaMemsetAsync(d_flags, 0, nC, st));
    if (tiles) SSJ_CK(cudaMemsetAsync(e->dev_defer_n, 0, ctr_words * sizeof(unsigned long long), st));
    SSJ_CK(ssjb::launch_prep(p, st));
    SSJ_CK(launch_strategy(*e, p, out, 0, n_tiles, st, stats));
    if (k1) SSJ_CK(cudaEventRecord(k1, st));
    return SSJ_OK;
}

}  // namespace

int ssj_verify_chunk_device(ssj_engine* e, const uint32_t* d_C, uint64_t nC, const uint32_t* d_C_O,
                            uint64_t nCO, uint8_t* d_flags, uint64_t* d_result, void* stream) {
    int rc = check_chunk_args(e, d_C, nC, d_C_O, nCO);
    if (rc) return rc;
    if (!d_result) return fail(SSJ_ERR_INVALID_ARGUMENT, "null d_result");
    if (e->group)
        return fail(SSJ_ERR_INVALID_ARGUMENT,
                    "device-resident chunks live on one GPU: use a one-device engine");
    DeviceScope ds(e->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    const int out = (e->mode == SSJ_MODE_PAIRS && d_flags) ? ssjb::kOutFlags : ssjb::kOutCount;
    return verify_device(e, d_C, nC, d_C_O, nCO, out, d_flags,
                         reinterpret_cast<unsigned long long*>(d_result), st);
}

// ---- candidate generation + join on the GPU -------------------------------------------------
}  // extern "C"

namespace {

typedef unsigned __int128 u128_host;

int ensure_filter_index(ssj_engine* e, int algorithm, double* build_ms) {
    if (algorithm != SSJ_ALG_ALLPAIRS && algorithm != SSJ_ALG_PPJOIN)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "GPU generation supports allpairs and ppjoin");
    if (build_ms) *build_ms = 0;
    if (!e->fidx) {
        auto t0 = std::chrono::steady_clock::now();
        // the static index relies on the reference's collection order (collection.hpp:115-119:
        // sizes non-decreasing), like the incremental index's length filter does
        if (e->n_sets) {
            std::vector<uint2> sd(e->n_sets);
            SSJ_CK(cudaMemcpy(sd.data(), e->d_sets, (size_t)e->n_sets * sizeof(uint2),
                              cudaMemcpyDeviceToHost));
            for (uint32_t i = 1; i < e->n_sets; ++i)
                if (sd[i].y < sd[i - 1].y)
                    return fail(SSJ_ERR_INVALID_ARGUMENT,
                                "GPU generation needs the collection in preprocessed (size, "
                                "lexicographic) order");
        }
        e->fidx = new ssjb::FilterIndex;
        cudaError_t err = ssjb::filter_index_build(e->fidx, e->d_tokens, e->d_sets, e->n_sets,
                                                   e->pred, algorithm, e->s_comp);
        if (err != cudaSuccess) {
            delete e->fidx;
            e->fidx = nullptr;
            if (err == cudaErrorInvalidValue)
                return fail(SSJ_ERR_INVALID_ARGUMENT,
                            "GPU index build: token values or index size beyond 2^31");
            return fail(SSJ_ERR_CUDA, std::string("GPU index build: ") + cudaGetErrorString(err));
        }
        if (build_ms)
            *build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    e->fidx->algorithm = algorithm;  // one index serves both (postings carry positions)
    e->fidx->heads = e->d_heads;
    return SSJ_OK;
}

template <typename F>
int cub_run(GenState& g, F&& f, cudaStream_t st) {
    size_t need = 0;
    SSJ_CK(f((void*)nullptr, need));
    if (need > g.tmp_bytes) {
        int rc;
        if ((rc = g.tmp.alloc(need))) return rc;
        g.tmp_bytes = need;
    }
    SSJ_CK(f(g.tmp.p, need));
    (void)st;
    return SSJ_OK;
}

int ensure_group_index(ssj_engine* e, double* build_ms) {
    if (build_ms) *build_ms = 0;
    if (e->gidx) return SSJ_OK;
    int rc;
    if ((rc = ensure_filter_index(e, SSJ_ALG_PPJOIN, nullptr))) return rc;  // also checks the order
    auto t0 = std::chrono::steady_clock::now();
    e->gidx = new ssjb::GroupIndex;
    cudaError_t err = ssjb::group_index_build(e->gidx, e->d_tokens, e->d_sets, e->d_heads, e->n_sets,
                                              e->pred, e->s_comp);
    if (err != cudaSuccess) {
        delete e->gidx;
        e->gidx = nullptr;
        return fail(SSJ_ERR_CUDA, std::string("GroupJoin index build: ") + cudaGetErrorString(err));
    }
    if (build_ms)
        *build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return SSJ_OK;
}

int gen_bounds_ix(ssj_engine* e, const ssjb::FilterIndex& ix, uint32_t n, GenState& g);

// Bounds of all probes and their exclusive scan (device + host copy).
int gen_bounds(ssj_engine* e, GenState& g) {
    return gen_bounds_ix(e, *e->fidx, e->n_sets, g);
}

int gen_bounds_ix(ssj_engine* e, const ssjb::FilterIndex& ix, uint32_t n, GenState& g) {
    cudaStream_t st = e->s_comp;
    int rc;
    if ((rc = g.bound.alloc((size_t)n * 8 + 8)) || (rc = g.base.alloc(((size_t)n + 1) * 8)))
        return rc;
    SSJ_CK(ssjb::filter_bounds(ix, 0, n, g.bound.as<unsigned long long>(), st));
    SSJ_CK(cudaMemsetAsync(g.base.p, 0, 8, st));
    if (n) {
        auto* in = g.bound.as<unsigned long long>();
        auto* out = g.base.as<unsigned long long>() + 1;
        if ((rc = cub_run(g, [&](void* t, size_t& b) {
                 return cub::DeviceScan::InclusiveSum(t, b, in, out, (int)n, st);
             }, st)))
            return rc;
    }
    g.hbase.resize((size_t)n + 1);
    SSJ_CK(cudaMemcpyAsync(g.hbase.data(), g.base.p, ((size_t)n + 1) * 8, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaStreamSynchronize(st));
    return SSJ_OK;
}

// Candidates of probes [a, b) as a compacted device chunk in g.C / g.CO.
int gen_block_ix(ssj_engine* e, const ssjb::FilterIndex& ix, GenState& g, uint32_t a, uint32_t b,
                 uint64_t* nC, uint64_t* nCO, bool compact);
int gen_block(ssj_engine* e, GenState& g, uint32_t a, uint32_t b, uint64_t* nC, uint64_t* nCO) {
    return gen_block_ix(e, *e->fidx, g, a, b, nC, nCO, true);
}

int gen_block_ix(ssj_engine* e, const ssjb::FilterIndex& ix, GenState& g, uint32_t a, uint32_t b,
                 uint64_t* nC, uint64_t* nCO, bool compact) {
    cudaStream_t st = e->s_comp;
    const uint32_t np = b - a;
    const unsigned long long base0 = g.hbase[a];
    const uint64_t ub = g.hbase[b] - base0;
    int rc;
    if (ub > g.G_cap) {
        if ((rc = g.G.alloc(ub * 4))) return rc;
        g.G_cap = ub;
    }
    if (ub > g.C_cap) {
        if ((rc = g.C.alloc(ub * 4))) return rc;
        g.C_cap = ub;
    }
    if (np > g.blk_cap) {
        if ((rc = g.count.alloc((size_t)np * 8)) || (rc = g.flag.alloc((size_t)np * 4)) ||
            (rc = g.obase.alloc((size_t)np * 8)) || (rc = g.slot.alloc((size_t)np * 4)) ||
            (rc = g.CO.alloc((size_t)np * 8)))
            return rc;
        g.blk_cap = np;
        g.gjCO_cap = 2ull * np;
    }
    const auto* base = g.base.as<unsigned long long>() + a;
    SSJ_CK(ssjb::filter_generate(ix, a, b, base, base0, g.G.as<uint32_t>(),
                                 g.count.as<unsigned long long>(), g.flag.as<uint32_t>(), st));
    if (!compact) {  // GroupJoin: the matched lists stay in g.G / g.count (expanded later)
        *nC = *nCO = 0;
        return SSJ_OK;
    }
    auto* cnt = g.count.as<unsigned long long>();
    auto* ob = g.obase.as<unsigned long long>();
    auto* fl = g.flag.as<uint32_t>();
    auto* sl = g.slot.as<uint32_t>();
    if ((rc = cub_run(g, [&](void* t, size_t& bb) {
             return cub::DeviceScan::ExclusiveSum(t, bb, cnt, ob, (int)np, st);
         }, st)))
        return rc;
    if ((rc = cub_run(g, [&](void* t, size_t& bb) {
             return cub::DeviceScan::ExclusiveSum(t, bb, fl, sl, (int)np, st);
         }, st)))
        return rc;
    unsigned long long last_ob = 0, last_cnt = 0;
    uint32_t last_sl = 0, last_fl = 0;
    SSJ_CK(cudaMemcpyAsync(&last_ob, ob + np - 1, 8, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&last_cnt, cnt + np - 1, 8, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&last_sl, sl + np - 1, 4, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&last_fl, fl + np - 1, 4, cudaMemcpyDeviceToHost, st));
    SSJ_CK(ssjb::filter_compact(a, b, base, base0, g.G.as<uint32_t>(), cnt, ob, sl,
                                g.C.as<uint32_t>(), g.CO.as<uint32_t>(), st));
    SSJ_CK(cudaStreamSynchronize(st));
    *nC = last_ob + last_cnt;
    *nCO = 2ull * (last_sl + last_fl);
    if (*nC > 0xFFFFFFFFull) return fail(SSJ_ERR_INVALID_ARGUMENT, "probe block exceeds u32 offsets");
    return SSJ_OK;
}

template <typename T>
int ensure_buf(DevBuf& b, size_t& cap, uint64_t need) {
    if (need <= cap && b.p) return SSJ_OK;
    const uint64_t n = std::max<uint64_t>(need, cap + cap / 2);
    int rc;
    if ((rc = b.alloc(n * sizeof(T)))) return rc;
    cap = n;
    return SSJ_OK;
}

// GroupJoin phase 1 of groups [a, b) (joiners.hpp:144-171): matched groups of every group
// (PPJoin over the representatives), expanded to member batches -> g.C / g.CO.
int gj_phase1(ssj_engine* e, GenState& g, uint32_t a, uint32_t b, uint64_t* nC, uint64_t* nCO) {
    const ssjb::GroupIndex& gi = *e->gidx;
    cudaStream_t st = e->s_comp;
    int rc;
    uint64_t unused = 0;
    if ((rc = gen_block_ix(e, gi.ix, g, a, b, &unused, &unused, false))) return rc;
    const uint32_t np = b - a;
    if ((rc = ensure_buf<unsigned long long>(g.per, g.gj_cap, np)) ||
        (rc = ensure_buf<unsigned long long>(g.cand, g.cand_cap, np)) ||
        (rc = ensure_buf<unsigned long long>(g.coff, g.coff_cap, np)))
        return rc;
    const auto* base = g.base.as<unsigned long long>() + a;
    const unsigned long long base0 = g.hbase[a];
    auto* per = g.per.as<unsigned long long>();
    auto* cand = g.cand.as<unsigned long long>();
    auto* coff = g.coff.as<unsigned long long>();
    auto* nbat = g.flag.as<uint32_t>();
    auto* soff = g.slot.as<uint32_t>();
    SSJ_CK(ssjb::group_sizes(gi, a, b, base, base0, g.G.as<uint32_t>(),
                             g.count.as<unsigned long long>(), per, cand, nbat, st));
    if ((rc = cub_run(g, [&](void* t, size_t& bb) {
             return cub::DeviceScan::ExclusiveSum(t, bb, cand, coff, (int)np, st);
         }, st)))
        return rc;
    if ((rc = cub_run(g, [&](void* t, size_t& bb) {
             return cub::DeviceScan::ExclusiveSum(t, bb, nbat, soff, (int)np, st);
         }, st)))
        return rc;
    unsigned long long lc = 0, lo = 0;
    uint32_t ls = 0, lb = 0;
    SSJ_CK(cudaMemcpyAsync(&lo, coff + np - 1, 8, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&lc, cand + np - 1, 8, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&ls, soff + np - 1, 4, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&lb, nbat + np - 1, 4, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaStreamSynchronize(st));
    *nC = lo + lc;
    *nCO = 2ull * (ls + lb);
    if (*nC > 0xFFFFFFFFull) return fail(SSJ_ERR_INVALID_ARGUMENT, "group block exceeds u32 offsets");
    if ((rc = ensure_buf<uint32_t>(g.C, g.C_cap, *nC)) ||
        (rc = ensure_buf<uint32_t>(g.CO, g.gjCO_cap, *nCO)))
        return rc;
    SSJ_CK(ssjb::group_expand(gi, a, b, base, base0, g.G.as<uint32_t>(),
                              g.count.as<unsigned long long>(), per, coff, soff,
                              g.C.as<uint32_t>(), g.CO.as<uint32_t>(), st));
    SSJ_CK(cudaStreamSynchronize(st));
    return SSJ_OK;
}

// GroupJoin phase 2 of groups [a, b) (joiners.hpp:175-179): the pairs inside every group as a
// chunk (probe first + i, candidates first .. first + i - 1) -> g.C / g.CO.
int gj_phase2(ssj_engine* e, GenState& g, uint32_t a, uint32_t b, uint64_t* nC, uint64_t* nCO) {
    const ssjb::GroupIndex& gi = *e->gidx;
    cudaStream_t st = e->s_comp;
    int rc;
    const uint32_t np = b - a;
    // scratch cached across calls (no cudaMalloc / cudaFree inside a warm join)
    if ((rc = ensure_buf<unsigned long long>(g.cand, g.cand_cap, np)) ||
        (rc = ensure_buf<unsigned long long>(g.coff, g.coff_cap, np)) ||
        (rc = ensure_buf<uint32_t>(g.iflag, g.iflag_cap, np)) ||
        (rc = ensure_buf<uint32_t>(g.islot, g.islot_cap, np)))
        return rc;
    auto* cand = g.cand.as<unsigned long long>();
    auto* coff = g.coff.as<unsigned long long>();
    auto* islc = g.iflag.as<uint32_t>();
    auto* soff = g.islot.as<uint32_t>();
    SSJ_CK(ssjb::group_intra_sizes(gi, a, b, cand, islc, st));
    if ((rc = cub_run(g, [&](void* t, size_t& bb) {
             return cub::DeviceScan::ExclusiveSum(t, bb, cand, coff, (int)np, st);
         }, st)))
        return rc;
    if ((rc = cub_run(g, [&](void* t, size_t& bb) {
             return cub::DeviceScan::ExclusiveSum(t, bb, islc, soff, (int)np, st);
         }, st)))
        return rc;
    unsigned long long lc = 0, lo = 0;
    uint32_t ls = 0, lb = 0;
    SSJ_CK(cudaMemcpyAsync(&lo, coff + np - 1, 8, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&lc, cand + np - 1, 8, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&ls, soff + np - 1, 4, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaMemcpyAsync(&lb, islc + np - 1, 4, cudaMemcpyDeviceToHost, st));
    SSJ_CK(cudaStreamSynchronize(st));
    *nC = lo + lc;
    *nCO = 2ull * (ls + lb);
    if (*nC > 0xFFFFFFFFull) return fail(SSJ_ERR_INVALID_ARGUMENT, "intra-group pairs exceed u32 offsets");
    if ((rc = ensure_buf<uint32_t>(g.C, g.C_cap, *nC)) ||
        (rc = ensure_buf<uint32_t>(g.CO, g.gjCO_cap, *nCO)))
        return rc;
    SSJ_CK(ssjb::group_intra(gi, a, b, coff, soff, g.C.as<uint32_t>(), g.CO.as<uint32_t>(), st));
    SSJ_CK(cudaStreamSynchronize(st));
    return SSJ_OK;
}

}  // namespace

extern "C" {

int ssj_gpu_generate_candidates(ssj_engine* e, int32_t algorithm, uint32_t probe_begin,
                                uint32_t probe_end, uint32_t* C_out, uint64_t C_cap,
                                uint64_t* nC_out, uint32_t* C_O_out, uint64_t C_O_cap,
                                uint64_t* nCO_out) {
    if (!e || !nC_out || !nCO_out) return fail(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    if (e->group)  // the stream does not depend on the device: the first one generates it
        return ssj_gpu_generate_candidates(ssjm::first(*e->group), algorithm, probe_begin,
                                           probe_end, C_out, C_cap, nC_out, C_O_out, C_O_cap,
                                           nCO_out);
    DeviceScope ds(e->device);
    int rc;
    probe_end = std::min(probe_end, e->n_sets);
    *nC_out = *nCO_out = 0;
    uint64_t nC = 0, nCO = 0;
    GenState* gp = nullptr;
    if (algorithm == SSJ_ALG_GROUPJOIN) {
        // phase 1 over all groups (the stream is per group; windows do not apply)
        if (probe_begin != 0 || probe_end != e->n_sets)
            return fail(SSJ_ERR_INVALID_ARGUMENT, "GroupJoin generation covers the whole collection");
        if ((rc = ensure_group_index(e, nullptr))) return rc;
        if (!e->gen_g) e->gen_g = new GenState;
        gp = e->gen_g;
        const uint32_t G = e->gidx->n_groups;
        if (!G) return SSJ_OK;
        if (gp->hbase.empty() && (rc = gen_bounds_ix(e, e->gidx->ix, G, *gp))) return rc;
        if ((rc = gj_phase1(e, *gp, 0, G, &nC, &nCO))) return rc;
    } else {
        if ((rc = ensure_filter_index(e, algorithm, nullptr))) return rc;
        if (probe_begin >= probe_end) return SSJ_OK;
        if (!e->gen) e->gen = new GenState;
        gp = e->gen;
        if (gp->hbase.empty() && (rc = gen_bounds(e, *gp))) return rc;
        if ((rc = gen_block(e, *gp, probe_begin, probe_end, &nC, &nCO))) return rc;
    }
    GenState& g = *gp;
    *nC_out = nC;
    *nCO_out = nCO;
    if (nC > C_cap || nCO > C_O_cap) return fail(SSJ_ERR_RUNTIME, "output capacity too small");
    if (nC) SSJ_CK(cudaMemcpy(C_out, g.C.p, nC * 4, cudaMemcpyDeviceToHost));
    if (nCO) SSJ_CK(cudaMemcpy(C_O_out, g.CO.p, nCO * 4, cudaMemcpyDeviceToHost));
    return SSJ_OK;
}

int ssj_gpu_join(ssj_engine* e, int32_t algorithm, uint64_t max_chunk_candidates,
                 uint32_t* pairs_out, uint64_t pairs_cap, uint64_t* n_pairs,
                 ssj_gpu_join_report* report) {
    return ssj_gpu_join_shard(e, algorithm, 0, 1, max_chunk_candidates, pairs_out, pairs_cap,
                              n_pairs, report);
}

int ssj_gpu_join_shard(ssj_engine* e, int32_t algorithm, uint32_t shard, uint32_t n_shards,
                       uint64_t max_chunk_candidates, uint32_t* pairs_out, uint64_t pairs_cap,
                       uint64_t* n_pairs, ssj_gpu_join_report* report) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (n_shards == 0 || shard >= n_shards) return fail(SSJ_ERR_INVALID_ARGUMENT, "bad shard");
    if (pairs_out && !n_pairs) return fail(SSJ_ERR_INVALID_ARGUMENT, "null n_pairs");
    if (e->group)
        return ssjm::gpu_join_shard(*e->group, algorithm, shard, n_shards, max_chunk_candidates,
                                    pairs_out, pairs_cap, n_pairs, report);
    DeviceScope ds(e->device);
    const auto t_start = std::chrono::steady_clock::now();
    ssj_gpu_join_report rep{};
    int rc;
    const bool groupjoin = algorithm == SSJ_ALG_GROUPJOIN;
    if (groupjoin && n_shards != 1)
        return fail(SSJ_ERR_INVALID_ARGUMENT, "GroupJoin on the GPU runs as one shard");
    if ((rc = groupjoin ? ensure_group_index(e, &rep.index_ms)
                        : ensure_filter_index(e, algorithm, &rep.index_ms)))
        return rc;
    const bool want_pairs = pairs_out != nullptr;
    if (want_pairs && !e->d_oid && (rc = ssj_engine_set_original_ids(e, nullptr))) return rc;
    cudaStream_t st = e->s_comp;
    cudaEvent_t ev[4];
    for (auto& x : ev) SSJ_CK(cudaEventCreate(&x));
    struct EvGuard {
        cudaEvent_t* ev;
        ~EvGuard() {
            for (int i = 0; i < 4; ++i) cudaEventDestroy(ev[i]);
        }
    } evg{ev};
    const uint64_t cap = max_chunk_candidates ? max_chunk_candidates : (256ull << 20);
    GenState*& gslot = groupjoin ? e->gen_g : e->gen;
    if (!gslot) gslot = new GenState;
    GenState& g = *gslot;
    // units: probes (AllPairs / PPJoin) or groups (GroupJoin), filtered through `ix`
    const ssjb::FilterIndex& ix = groupjoin ? e->gidx->ix : *e->fidx;
    const uint32_t n_units = groupjoin ? e->gidx->n_groups : e->n_sets;
    SSJ_CK(cudaEventRecord(ev[0], st));
    if (g.hbase.empty() && (rc = gen_bounds_ix(e, ix, n_units, g))) return rc;  // cached
    SSJ_CK(cudaEventRecord(ev[1], st));
    SSJ_CK(cudaEventSynchronize(ev[1]));
    float ms = 0;
    SSJ_CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
    rep.filtering_ms += ms;
    // scratch cached on the engine: a warm join allocates nothing
    if (!g.acc.p && (rc = g.acc.alloc(SSJ_RESULT_WORDS * 8))) return rc;
    DevBuf& acc = g.acc;
    DevBuf& keys_all = g.keys;
    size_t& keys_cap = g.keys_cap;
    uint64_t keys_n = 0;
    // verification of one device-resident chunk (g.C / g.CO), results appended
    auto consume = [&](uint64_t nC, uint64_t nCO) -> int {
        if (!nC) return SSJ_OK;
        int r;
        const int out = want_pairs ? ssjb::kOutResults : ssjb::kOutCount;
        if ((r = verify_device(e, g.C.as<uint32_t>(), nC, g.CO.as<uint32_t>(), nCO, out, nullptr,
                               acc.as<unsigned long long>(), st, /*stats=*/false)))
            return r;
        unsigned long long words[SSJ_RESULT_WORDS];
        SSJ_CK(cudaMemcpyAsync(words, acc.p, sizeof(words), cudaMemcpyDeviceToHost, st));
        unsigned long long nres = 0;
        if (want_pairs) SSJ_CK(cudaMemcpyAsync(&nres, e->d_res_n, 8, cudaMemcpyDeviceToHost, st));
        SSJ_CK(cudaStreamSynchronize(st));
        if ((r = decode_error(words[SSJ_RESULT_ERROR]))) return r;
        rep.count += words[SSJ_RESULT_COUNT];
        if (want_pairs && nres) {
            if (keys_n + nres > keys_cap) {
                DevBuf grown;
                const uint64_t nc = std::max<uint64_t>(2 * keys_cap, keys_n + nres);
                if ((r = grown.alloc(nc * 8))) return r;
                if (keys_n)
                    SSJ_CK(cudaMemcpyAsync(grown.p, keys_all.p, keys_n * 8, cudaMemcpyDeviceToDevice, st));
                std::swap(grown.p, keys_all.p);
                keys_cap = nc;
            }
            KParams p = base_params(*e);
            p.C = g.C.as<uint32_t>();
            p.nC = nC;
            p.C_O = g.CO.as<uint32_t>();
            p.n_slices = (uint32_t)(nCO / 2);
            p.res_slots = e->d_res_slots;
            SSJ_CK(ssjb::launch_pairs(p, e->d_oid, nres, keys_all.as<unsigned long long>() + keys_n, st));
            keys_n += nres;
        }
        return SSJ_OK;
    };
    // this shard's units: equal shares of the total candidate upper bound
    const uint64_t total = g.hbase[n_units];
    auto cut = [&](uint32_t k) -> uint32_t {
        if (k == 0) return 0;
        if (k >= n_shards) return n_units;
        const unsigned long long target = (unsigned long long)((u128_host)total * k / n_shards);
        return (uint32_t)(std::lower_bound(g.hbase.begin(), g.hbase.end(), target) - g.hbase.begin());
    };
    const uint32_t p_begin = std::min(cut(shard), n_units);
    const uint32_t n = std::max(p_begin, std::min(cut(shard + 1), n_units));
    // GroupJoin phase 2: exclusive scan of the groups' intra pair counts c (c - 1) / 2, so its
    // blocks are cut by the same candidate budget as phase 1's (a group is never split)
    std::vector<unsigned long long> ibase;
    if (groupjoin && n > p_begin) {
        const uint32_t np = n - p_begin;
        if ((rc = ensure_buf<unsigned long long>(g.cand, g.cand_cap, np)) ||
            (rc = ensure_buf<unsigned long long>(g.coff, g.coff_cap, np)) ||
            (rc = ensure_buf<uint32_t>(g.iflag, g.iflag_cap, np)) ||
            (rc = ensure_buf<uint32_t>(g.islot, g.islot_cap, np)))
            return rc;
        auto* cand = g.cand.as<unsigned long long>();
        auto* coff = g.coff.as<unsigned long long>();
        SSJ_CK(ssjb::group_intra_sizes(*e->gidx, p_begin, n, cand, g.iflag.as<uint32_t>(), st));
        if ((rc = cub_run(g, [&](void* t, size_t& bb) {
                 return cub::DeviceScan::ExclusiveSum(t, bb, cand, coff, (int)np, st);
             }, st)))
            return rc;
        ibase.resize((size_t)np + 1);
        unsigned long long last = 0;
        SSJ_CK(cudaMemcpyAsync(ibase.data(), coff, (size_t)np * 8, cudaMemcpyDeviceToHost, st));
        SSJ_CK(cudaMemcpyAsync(&last, cand + np - 1, 8, cudaMemcpyDeviceToHost, st));
        SSJ_CK(cudaStreamSynchronize(st));
        ibase[np] = ibase[np - 1] + last;
    }
    for (int phase = 0; phase < (groupjoin ? 2 : 1); ++phase) {
        for (uint32_t a = p_begin; a < n;) {
            // the longest block whose candidate count (bound) fits the budget (>= 1 unit)
            uint32_t b;
            if (phase == 0) {
                b = (uint32_t)(std::upper_bound(g.hbase.begin() + a + 1, g.hbase.end(),
                                                g.hbase[a] + cap) - g.hbase.begin()) - 1;
            } else {
                const size_t k = a - p_begin;  // ibase[k] = intra pairs of groups [p_begin, a)
                b = p_begin + (uint32_t)(std::upper_bound(ibase.begin() + k + 1, ibase.end(),
                                                          ibase[k] + cap) - ibase.begin()) - 1;
            }
            if (b <= a) b = a + 1;
            b = std::min(b, n);
            uint64_t nC = 0, nCO = 0;
            SSJ_CK(cudaEventRecord(ev[0], st));
            if (!groupjoin) rc = gen_block(e, g, a, b, &nC, &nCO);
            else if (phase == 0) rc = gj_phase1(e, g, a, b, &nC, &nCO);
            else rc = gj_phase2(e, g, a, b, &nC, &nCO);
            if (rc) return rc;
            SSJ_CK(cudaEventRecord(ev[1], st));
            if ((rc = consume(nC, nCO))) return rc;
            SSJ_CK(cudaEventRecord(ev[2], st));
            SSJ_CK(cudaEventSynchronize(ev[2]));
            SSJ_CK(cudaEventElapsedTime(&ms, ev[0], ev[1]));
            rep.filtering_ms += ms;
            SSJ_CK(cudaEventElapsedTime(&ms, ev[1], ev[2]));
            rep.verification_ms += ms;
            if (phase == 0) rep.candidate_count += nC;
            else rep.intra_group_pairs += nC;  // GroupJoin phase 2 (joiners.hpp:175-179)
            rep.chunk_count += nC ? 1 : 0;
            a = b;
        }
    }
    if (want_pairs) {
        *n_pairs = keys_n;
        if (keys_n) {
            // write_pairs order (report.hpp:39-42): radix sort of the (r_id << 32 | s_id) keys
            DevBuf& sorted = g.sorted;
            if ((rc = ensure_buf<unsigned long long>(sorted, g.sorted_cap, keys_n))) return rc;
            auto* kin = keys_all.as<unsigned long long>();
            auto* kout = sorted.as<unsigned long long>();
            if ((rc = cub_run(g, [&](void* t, size_t& bb) {
                     return cub::DeviceRadixSort::SortKeys(t, bb, kin, kout, (int)keys_n, 0, 64, st);
                 }, st)))
                return rc;
            std::vector<unsigned long long> hk(std::min<uint64_t>(keys_n, pairs_cap));
            if (!hk.empty())
                SSJ_CK(cudaMemcpyAsync(hk.data(), kout, hk.size() * 8, cudaMemcpyDeviceToHost, st));
            SSJ_CK(cudaStreamSynchronize(st));
            for (size_t i = 0; i < hk.size(); ++i) {
                pairs_out[2 * i] = (uint32_t)(hk[i] >> 32);
                pairs_out[2 * i + 1] = (uint32_t)hk[i];
            }
        }
    } else if (n_pairs) {
        *n_pairs = 0;
    }
    rep.join_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    if (report) *report = rep;
    if (want_pairs && keys_n > pairs_cap) return fail(SSJ_ERR_RUNTIME, "pair capacity exceeded");
    return SSJ_OK;
}

int ssj_engine_set_profiling(ssj_engine* e, int enabled) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (e->group) return ssjm::set_profiling(*e->group, enabled);
    e->profiling = enabled != 0;
    e->prof_used = 0;
    return SSJ_OK;
}

int ssj_engine_kernel_time(ssj_engine* e, double* total_ms, uint64_t* launches) {
    if (!e) return fail(SSJ_ERR_INVALID_ARGUMENT, "null engine");
    if (e->group) return ssjm::kernel_time(*e->group, total_ms, launches);
    DeviceScope ds(e->device);
    double sum = 0;
    for (size_t i = 0; i < e->prof_used; ++i) {
        float ms = 0;
        SSJ_CK(cudaEventSynchronize(e->prof_events[i].second));
        SSJ_CK(cudaEventElapsedTime(&ms, e->prof_events[i].first, e->prof_events[i].second));
        sum += ms;
    }
    if (total_ms) *total_ms = sum;
    if (launches) *launches = e->prof_used;
    e->prof_used = 0;
    return SSJ_OK;
}

int ssj_engine_export_collection(const ssj_engine* e, uint32_t* d_tokens, uint32_t* d_sets,
                                 void* stream) {
    if (!e || !d_tokens || !d_sets) return fail(SSJ_ERR_INVALID_ARGUMENT, "null argument");
    if (e->group) return ssj_engine_export_collection(ssjm::first(*e->group), d_tokens, d_sets, stream);
    DeviceScope ds(e->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    SSJ_CK(cudaMemcpyAsync(d_tokens, e->d_tokens, e->n_padded * sizeof(uint32_t),
                           cudaMemcpyDeviceToDevice, st));
    SSJ_CK(cudaMemcpyAsync(d_sets, e->d_sets, (size_t)std::max<uint32_t>(e->n_sets, 1) * sizeof(uint2),
                           cudaMemcpyDeviceToDevice, st));
    return SSJ_OK;
}

int ssj_launches_per_chunk(const ssj_engine* e, uint64_t nC, uint64_t nCO) {
    // prep + one verification kernel (B, C); the memsets of the result block are not ours.
    // Strategy A: prep (validation, descriptors, tile index, run and short-tile lists), probe
    // bitmaps (when there are slices), run_kernel and warp_tile_kernel (when there are
    // slots), and the long-pair pass (when some set is longer than kLongPair).
    const int per = (e && e->exec.kind == SSJ_STRATEGY_A)
                        ? (nCO >= 2 ? 2 : 1) + (nC ? 2 : 0) +
                              (e->max_set_size > ssjb::kLongPair ? 1 : 0)
                        : 2;
    return e && e->group ? per * (int)ssjm::size(*e->group) : per;
}

int ssj_chunk_algorithmic_bytes_device(ssj_engine* e, const uint32_t* d_C, uint64_t nC,
                                       const uint32_t* d_C_O, uint64_t nCO, uint64_t* d_bytes,
                                       void* stream) {
    if (e && e->group)
        return fail(SSJ_ERR_INVALID_ARGUMENT,
                    "device-resident chunks live on one GPU: use a one-device engine");
    int rc = check_chunk_args(e, d_C, nC, d_C_O, nCO);
    if (rc) return rc;
    DeviceScope ds(e->device);
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
    KParams p = base_params(*e);
    p.C = d_C;
    p.nC = nC;
    p.C_O = d_C_O;
    p.n_slices = (uint32_t)(nCO / 2);
    SSJ_CK(cudaMemsetAsync(d_bytes, 0, sizeof(uint64_t), st));
    SSJ_CK(ssjb::launch_bytes(p, reinterpret_cast<unsigned long long*>(d_bytes), st));
    return SSJ_OK;
}

int ssj_measure_read_bandwidth(int device, uint64_t bytes, uint32_t reps, double* gbs) {
    int rc = check_device(device);
    if (rc) return rc;
    if (!gbs || bytes < 16 || !reps) return fail(SSJ_ERR_INVALID_ARGUMENT, "bad arguments");
    DeviceScope ds(device);
    void* buf = nullptr;
    unsigned* sink = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    auto cleanup = [&]() {
        cudaFree(buf);
        cudaFree(sink);
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    };
    if (cudaMalloc(&buf, bytes) != cudaSuccess || cudaMalloc(&sink, 4) != cudaSuccess ||
        cudaMemset(buf, 1, bytes) != cudaSuccess || cudaEventCreate(&a) != cudaSuccess ||
        cudaEventCreate(&b) != cudaSuccess) {
        cleanup();
        return fail(SSJ_ERR_CUDA, "bandwidth probe setup failed");
    }
    ssjb::launch_read_bw(buf, bytes, 2, sink, 0);  // warm-up (and L2 fill)
    cudaEventRecord(a, 0);
    ssjb::launch_read_bw(buf, bytes, reps, sink, 0);
    cudaEventRecord(b, 0);
    float ms = 0;
    const cudaError_t err = cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    cleanup();
    if (err != cudaSuccess) return fail(SSJ_ERR_CUDA, cudaGetErrorString(err));
    *gbs = (double)bytes * reps / (ms / 1e3) / 1e9;
    return SSJ_OK;
}

void* ssj_host_alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        g_err = "cudaHostAlloc failed";
        return nullptr;
    }
    return p;
}

void ssj_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
