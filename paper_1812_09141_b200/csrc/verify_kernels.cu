// verify_kernels.cu -- sm_100a candidate-verification kernels.
//
// The reference verifies a chunk on a CPU worker pool under one of three work
// assignments (verify.hpp:232-345, the paper's thread-allocation alternatives A/B/C,
// PAPER.md:605-644). Here each becomes a grid:
//   A  (= Auto) thread per pair, load-balanced independently of slice lengths:
//      prep_kernel       : thread per slice: validation, slice descriptor, tile index, the
//                          runs of long slices (>= kRunMinSlice) and the short-tile lists
//      bitmap_kernel     : global probe bitmaps of the slices that read one (warp-tile
//                          slices with >= kSliceBitmapMinCands candidates, run slices whose
//                          probe range exceeds the byte map)
//      run_kernel        : runs; candidate head records through the texture path, the probe
//                          as a byte map + bitmap + ranks in shared memory (built by one
//                          warp, published with mbarriers), first 8 tokens per thread and a
//                          per-warp continuation queue (the headline kernel)
//      warp_tile_kernel  : 64-slot warp tiles of short slices (shuffle slot -> slice search);
//                          on device-resident chunks it runs beside run_kernel on a second
//                          stream
//      long_slice_kernel : pairs longer than kLongPair, CTA per slice with the probe bitmap
//                          and rank in shared memory, 128 tokens per warp step
//   B  block_kernel : one CTA per probe slice (paper Alt B): the probe set is staged in
//                     shared memory and the CTA's threads stride over the slice's
//                     candidates, each running the sequential early-exit merge.
//   C  path_kernel  : one CTA per probe slice, groups of G lanes per candidate pair
//                     (paper Alt C / verify.hpp:303-345): the G lanes split the pair's
//                     merge path with the reference's diagonal partitions
//                     (verify.hpp:110-166) and reduce their counts with shuffles. Unlike
//                     the reference it walks the path in rounds of G*kHops hops and stops
//                     as soon as the verdict is decided.
// All three produce the reference's flags bit for bit (see ssj_device.cuh).
#include <atomic>

#include <cub/block/block_scan.cuh>

#include "verify_kernels.cuh"
#include "../../include/ssjoin_b200.h"

#ifndef SSJB_RUN_TEX
#define SSJB_RUN_TEX 1  // run_kernel gathers candidate heads through the texture path
#endif
#ifndef SSJB_CONT_TEX
#define SSJB_CONT_TEX 1  // run_kernel's continuation blocks read the CSR through the texture path
#endif
#ifndef SSJB_RUN_REQTAB
#define SSJB_RUN_REQTAB 1  // run_kernel reads the required overlap from the engine's table
#endif
#ifndef SSJB_RUN_OWN_BITMAP
#define SSJB_RUN_OWN_BITMAP 1  // run slices' probe bitmaps built by run_kernel
#endif
#ifndef SSJB_RUN_AHEAD
#define SSJB_RUN_AHEAD 1  // run_kernel: a warp free at a slice change builds the next map too
#endif
#ifndef SSJB_ORDERED_MIN_SLOTS
#define SSJB_ORDERED_MIN_SLOTS (1u << 24)  // device path: run list in slot order from 16M candidates
#endif
#ifndef SSJB_TILE_DESC_SHFL
#define SSJB_TILE_DESC_SHFL 1
#endif
#ifndef SSJB_TILE_DYN
#define SSJB_TILE_DYN 1  // warp_tile_kernel takes short tiles from a per-launch counter
#endif

namespace ssjb {

namespace {


__host__ __device__ __forceinline__ uint32_t bitmap_alloc_words(uint32_t nw) {
    return (nw + 4u) & ~3u;
}

__device__ __forceinline__ void acc_add(unsigned long long* acc, int word, unsigned v) {
    const unsigned w = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && w) atomicAdd(acc + word, (unsigned long long)w);
}

__device__ __forceinline__ void flag_error(unsigned long long* acc, unsigned long long bits) {
    atomicOr(acc + 1, bits);
}

// Warp-aggregated append of qualifying (slot, overlap) results: one atomicAdd per warp.
// Must be called by all 32 lanes of the warp.
__device__ __forceinline__ void warp_append(const KParams& p, bool met, uint64_t slot,
                                            uint32_t ov) {
    const unsigned mask = __ballot_sync(0xffffffffu, met);
    if (!mask) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(p.res_n, (unsigned long long)__popc(mask));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (met) {
        const unsigned long long idx = base + __popc(mask & ((1u << lane) - 1u));
        if (idx < p.res_cap) {
            p.res_slots[idx] = (uint32_t)slot;
            p.res_ov[idx] = ov;
        }
    }
}

// One candidate pair, thread-sequential (strategies A and B).
// r/m: probe tokens (shared or global); returns met, *ov = true overlap in results mode.
template <int kOut>
__device__ __forceinline__ bool verify_pair(const KParams& p, const uint32_t* r, uint32_t m,
                                            uint32_t cand, uint32_t* ov, uint32_t* n_out) {
    if (cand >= p.n_sets) {
        flag_error(p.acc, kErrOutOfRange);
        *n_out = 0;
        return false;
    }
    const uint2 sd = __ldg(p.sets + cand);
    const uint32_t n = sd.y;
    *n_out = n;
    const uint4* s4 = reinterpret_cast<const uint4*>(p.tokens + (size_t)sd.x * 8);
    // Speculative: every set position has >= 8 readable tokens (padding + tail sentinel).
    const uint4 w0 = __ldg(s4);
    const uint4 w1 = __ldg(s4 + 1);
    const uint64_t req = dev_required(p.pred, m, n);
    if (req == 0) {
        // verify.hpp:57: the loop exits before any comparison and met = (0 >= 0).
        if (kOut == kOutResults)
            *ov = full_overlap_seq(r, m, reinterpret_cast<const uint32_t*>(s4), n);
        return true;
    }
    if (req > (uint64_t)min(m, n)) return false;  // overlap <= min(m, n) < req
    return merge_thread<kOut == kOutResults>(r, m, s4, n, (uint32_t)req, w0, w1, ov);
}

// 8 consecutive tokens (32 bytes, 32-byte aligned) in one 256-bit load.
__device__ __forceinline__ void ld_tokens8(const uint32_t* __restrict__ s, uint32_t t[8]) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]),
                   "=r"(t[6]), "=r"(t[7])
                 : "l"(s));
}

// The same 8 tokens through the texture path (two uint4 texels of a linear texture over the
// array; texel = 4 tokens, so the 32-byte-aligned group at token offset 8k is texels 2k, 2k+1).
// Scattered 32-byte gathers through TLD do not compete with the kernels' shared-memory lookups
// for the LSU pipe the way LDG.256 does (tools/tex_microbench.cu: 8 byte-map lookups per row
// cost 29 % of the gather rate behind LDG.256, 2 % behind TLD).
__device__ __forceinline__ void tex_tokens8(unsigned long long tex, uint64_t group8, uint32_t t[8]) {
    const uint4 a = tex1Dfetch<uint4>(tex, (int)(2 * group8));
    const uint4 b = tex1Dfetch<uint4>(tex, (int)(2 * group8 + 1));
    t[0] = a.x; t[1] = a.y; t[2] = a.z; t[3] = a.w;
    t[4] = b.x; t[5] = b.y; t[6] = b.z; t[7] = b.w;
}

// A pair longer than kLongPair tokens is left to long_slice_kernel: the first pass marks its
// slice once per chunk segment (tag = segment index + 1 in the slice descriptor's spare word)
// and lists it; long_slice_kernel re-derives the slice's long pairs from C.
__device__ __forceinline__ void mark_long_slice(const KParams& p, uint32_t e) {
    unsigned* mk = reinterpret_cast<unsigned*>(p.slices + e) + 6;  // SliceDesc::pad0
    if (atomicMax(mk, p.seg_tag) < p.seg_tag) {
        const unsigned long long idx = atomicAdd(p.defer_n, 1ull);
        if (idx < p.defer_cap) p.defer[idx] = e;  // cap = segment slots >= marked slices
    }
}

// First slice e in [lo, hi) whose end offset (C_O[2e+1]) is > key.
__device__ __forceinline__ uint32_t upper_bound_ends(const uint32_t* __restrict__ C_O,
                                                     uint32_t lo, uint32_t hi, uint64_t key) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(C_O + 2 * (size_t)mid + 1) <= key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------------------------------
// Prep (thread per slice): validate C_O (chunk.hpp:36-48 decode assumptions) and -- for
// strategy A -- write the slice's descriptor (probe position/size; for slices with
// >= kSliceBitmapMinCands candidates a probe-bitmap allocation), its part of the tile index
// and its work lists:
//   * tile_first[t] (the slice holding slot t * kTile) is read only for short tiles and their
//     successors, so a short slice writes it for every tile starting inside it and a long
//     slice only for its first and last such tile (a short tile's first slot and its
//     successor's first slot lie in a short slice, or at a long slice's last / first tile);
//   * a long slice (>= kRunMinSlice candidates) emits its runs of <= kRun slots into every
//     segment it overlaps (runs never straddle segments);
//   * a tile is short when it holds a slot of a short slice or an uncovered slot; it is listed
//     by exactly one owner, without atomics on the tiles: the short slice holding its first
//     slot, else (the tile starts inside a long slice, which then ends in it) the first short
//     slice in it, else the uncovered tail. A short slice starting inside a tile owns that
//     tile iff the slice before it (the previous non-empty one) is long.
// Every list position comes from ONE atomic per warp (a scan over the lanes, keyed by the
// segment: slices are in slot order, so a warp's lanes with equal segment are contiguous).

// Warp-aggregated allocation: lane requests k items from counter(key); lanes with equal key
// are contiguous. All 32 lanes call it. Returns the lane's first position.
template <typename Ctr>
__device__ __forceinline__ unsigned long long warp_alloc(uint64_t key, uint32_t k, Ctr counter) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t incl = k;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
        const uint64_t kk = __shfl_up_sync(0xffffffffu, key, off);
        if (lane >= (uint32_t)off && kk == key) incl += v;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const uint32_t last = 31 - __clz(peers);
    unsigned long long base = 0;
    if (lane == last && incl) base = atomicAdd(counter(key), (unsigned long long)incl);
    base = __shfl_sync(0xffffffffu, base, last);
    return base + incl - k;
}

__device__ __forceinline__ unsigned long long* seg_counter(const KParams& p, uint64_t seg, int c) {
    return p.ctr_all + kCounters * seg + c;
}

// Tiles of segment `seg` (its lists' capacities: short tiles 1x, runs 2x).
__device__ __forceinline__ uint64_t seg_tiles(const KParams& p, uint64_t seg) {
    const uint64_t t0 = seg * p.seg_slots / kTile;  // segments start on tile boundaries
    const uint64_t t1 = ((seg + 1) * p.seg_slots + kTile - 1) / kTile;  // the last may be partial
    return min(t1, (uint64_t)p.n_tiles) - min(t0, (uint64_t)p.n_tiles);
}

__device__ __forceinline__ void write_runs(const KParams& p, uint32_t e, uint64_t seg,
                                           unsigned long long k, uint64_t lo, uint64_t hi) {
    RunDesc* runs = p.runs_all + 2 * (seg * p.seg_slots / kTile) + k;
    const uint64_t cap = 2 * seg_tiles(p, seg) + 2;  // only a malformed C_O could exceed it
    for (uint64_t i = 0; lo + i * kRun < hi && k + i < cap; ++i) {
        RunDesc d;
        d.slice = e;
        d.begin = (uint32_t)(lo + i * kRun);
        d.end = (uint32_t)min(lo + (i + 1) * kRun, hi);
        d.pad = 0;
        runs[i] = d;
    }
}

// Append tile t to its segment's short list (per-lane atomic: the rare paths).
__device__ __forceinline__ void list_short_tile(const KParams& p, uint64_t t) {
    const uint64_t seg = t * kTile / p.seg_slots;
    const unsigned long long k = atomicAdd(seg_counter(p, seg, 2), 1ull);
    if (k < seg_tiles(p, seg)) p.short_all[seg * p.seg_slots / kTile + k] = (uint32_t)t;
}

// Length of the last non-empty slice before slice `idx` whose slots end at `pos` (0 if none):
// walks back over zero-width slices.
__device__ __forceinline__ uint64_t prev_nonempty_len(const KParams& p, uint64_t idx, uint64_t pos) {
    while (idx > 0) {
        --idx;
        const uint64_t pb = idx ? min((uint64_t)p.C_O[2 * idx - 1], p.nC) : 0;
        if (pb < pos) return pos - pb;
        if (pb > pos) return 0;  // malformed C_O (reported by validation)
    }
    return 0;
}

// The slots past the last slice's end `last_end`: never verified (flag 0); their tiles are
// short. The tile holding last_end is the tail's unless a short slice overlaps it.
__device__ __forceinline__ void uncovered_tail(const KParams& p, uint64_t n_entries,
                                               uint64_t last_end) {
    if (last_end >= p.nC) return;
    for (uint64_t t = (last_end + kTile - 1) / kTile; t < p.n_tiles; ++t) {
        p.tile_first[t] = p.n_slices;
        list_short_tile(p, t);
    }
    if (last_end % kTile) {  // a short last slice already listed it
        const uint64_t len = prev_nonempty_len(p, n_entries, last_end);
        if (len == 0 || len >= kRunMinSlice) list_short_tile(p, last_end / kTile);
    }
}

constexpr uint32_t kPrepThreads = 256;
constexpr uint32_t kLbTicket = 0;  // lb_status[0]: CTA tickets; lb_status[1 + k]: CTA k's word
constexpr unsigned long long kLbAggregate = 1ull << 62, kLbPrefix = 2ull << 62;
constexpr unsigned long long kLbValue = (1ull << 62) - 1;

// One segment (the device path): the runs are listed in slot order, so that run_kernel's CTAs,
// which sweep the run list together, sweep the chunk in order. A run's position is the
// exclusive prefix of the runs of all earlier slices: a block scan plus a decoupled look-back
// over the CTAs (CTAs take their slice ranges in ticket order, so a CTA only waits for CTAs
// that already run). status[k]: flag (aggregate / inclusive prefix) | value, one 64-bit word.
__device__ __forceinline__ unsigned long long ordered_run_base(const KParams& p, uint32_t ticket,
                                                              uint32_t nrun, uint32_t* s_tmp) {
    using Scan = cub::BlockScan<uint32_t, kPrepThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ unsigned long long s_base;
    uint32_t excl = 0, total = 0;
    Scan(scan_tmp).ExclusiveSum(nrun, excl, total);
    unsigned long long* status = p.lb_status + 1;
    if (threadIdx.x < 32) {  // warp 0: publish, then look back 32 predecessors at a time
        const uint32_t lane = threadIdx.x;
        unsigned long long prefix = 0;
        if (lane == 0) atomicExch(status + ticket, (ticket ? kLbAggregate : kLbPrefix) | total);
        for (int64_t j = (int64_t)ticket - 1; j >= 0; j -= 32) {
            const int64_t jj = j - (int64_t)lane;  // lane 0 = the nearest predecessor
            unsigned long long v = kLbPrefix;     // before CTA 0: an inclusive prefix of 0
            if (jj >= 0) {
                do {
                    v = *(volatile unsigned long long*)(status + jj);
                } while (v == 0);
            }
            const unsigned pm = __ballot_sync(0xffffffffu, (v & kLbPrefix) != 0);
            const uint32_t upto = pm ? (uint32_t)(__ffs(pm) - 1) : 31u;  // nearest prefix, inclusive
            // run counts: every prefix is < 2^32 (a run covers >= 1 of < 2^32 slots)
            const uint32_t part = lane <= upto ? (uint32_t)(v & kLbValue) : 0u;
            prefix += __reduce_add_sync(0xffffffffu, part);
            if (pm) break;
        }
        if (lane == 0) {
            if (ticket) atomicExch(status + ticket, kLbPrefix | (prefix + total));
            if (total) atomicAdd(p.ctr_all + 1, (unsigned long long)total);  // the run count
            s_base = prefix;
        }
    }
    __syncthreads();
    (void)s_tmp;
    return s_base + excl;
}

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const KParams p) {
    // slices in ticket order (ordered run list) or by block index
    __shared__ uint32_t s_ticket;
    // (small chunks: the run list's order buys no L2 locality, skip the look-back)
    const bool ordered = p.ctr_all && p.lb_status && p.seg_slots >= p.nC &&
                         p.nC >= (uint64_t)SSJB_ORDERED_MIN_SLOTS;
    if (ordered) {
        if (threadIdx.x == 0) s_ticket = (uint32_t)atomicAdd(p.lb_status + kLbTicket, 1ull);
        __syncthreads();
    }
    const uint32_t cta = ordered ? s_ticket : blockIdx.x;
    const uint64_t idx = (uint64_t)cta * kPrepThreads + threadIdx.x;
    const bool live = idx < p.n_slices;
    uint32_t end = 0, begin = 0, probe = 0;
    if (live) {
        end = p.C_O[2 * idx + 1];
        begin = idx ? p.C_O[2 * idx - 1] : 0;
        probe = p.C_O[2 * idx];
        if (end < begin || (uint64_t)end > p.nC) flag_error(p.acc, kErrBadOffsets);
        if (end > begin && probe >= p.n_sets) flag_error(p.acc, kErrOutOfRange);
    }
    if (p.slices) {  // launch-uniform
        uint4 d0 = make_uint4(end, 0, 0, kNone);
        uint4 d1 = make_uint4(0, 0, 0, 0);
        uint32_t na = 0;  // bitmap words requested
        if (live && probe < p.n_sets) {
            const uint2 rd = p.sets[probe];
            d0.y = rd.x;
            d0.z = rd.y;
            // a probe bitmap pays off for long slices (long pairs build their own in shared
            // memory, long_slice_kernel)
            if (p.bm_cap && rd.y && end > begin && end - begin >= kSliceBitmapMinCands) {
                const uint32_t* r = p.tokens + (size_t)rd.x * 8;
                const uint32_t lo = r[0] & ~31u;
                const uint32_t hi = r[rd.y - 1];
                const uint32_t nw = ((hi - lo) >> 5) + 1;
                // the words plus at least one zero word (clamped lookups of tokens beyond the
                // range land there), rounded to 16 bytes for cp.async; no bitmap when the
                // probe holds token 0xFFFFFFFF (the padding value)
                if (nw <= kMaxBitmapWords && hi != 0xFFFFFFFFu) {
                    d1.x = lo;
                    d1.y = nw;
                    // run_kernel builds the bitmap of a run slice whose range fits its byte
                    // map itself (in shared memory): no global words for those
                    const bool own = SSJB_RUN_OWN_BITMAP && end - begin >= kRunMinSlice &&
                                     nw * 32u <= kRunMapRange;
                    if (!own) na = bitmap_alloc_words(nw);
                }
            }
        }
        const unsigned long long off =
            warp_alloc(0, na, [&](uint64_t) { return p.acc + kAccBitmapWords; });
        const bool got = na && off + na <= p.bm_cap;
        if (got) d0.w = (uint32_t)off;
        else if (na) d1 = make_uint4(0, 0, 0, 0);  // wanted global words, none left: merge path
        if (p.bm_list) {
            const unsigned long long li =
                warp_alloc(0, got ? 1u : 0u, [&](uint64_t) { return p.acc + kAccBitmapSlices; });
            if (got) p.bm_list[li] = (uint32_t)idx;
        }
        if (live) {
            uint4* dst = reinterpret_cast<uint4*>(p.slices + idx);
            dst[0] = d0;
            dst[1] = d1;
        }
    }
    if (!p.ctr_all) return;  // launch-uniform: strategies B and C need no work lists
    // strategy A work lists (clamped: a malformed C_O only reports)
    const uint64_t b = live ? min((uint64_t)begin, p.nC) : 0, e = live ? min((uint64_t)end, p.nC) : 0;
    const bool any = e > b;
    const bool is_long = any && e - b >= kRunMinSlice;
    const uint64_t t_lo = (b + kTile - 1) / kTile, t_hi = (e + kTile - 1) / kTile;  // tiles starting in it
    // short slice: the tiles it owns -- those starting in it, and the one it starts in when
    // the previous non-empty slice is long
    const bool own_first = any && !is_long && b % kTile && prev_nonempty_len(p, idx, b) >= kRunMinSlice;
    const uint64_t t0 = own_first ? b / kTile : t_lo;  // owned tiles [t0, t_hi)
    // the lane's key: its segment (slices are in slot order, so equal keys are contiguous);
    // idle lanes after the last slice share the largest key
    const uint64_t seg = live ? b / p.seg_slots : ~0ull;
    const uint64_t seg_end = (seg + 1) * p.seg_slots;
    // runs in the lane's first segment / short tiles in the key segment: warp-aggregated;
    // whatever lies in later segments: per lane
    const uint32_t nrun = is_long ? (uint32_t)((min(e, seg_end) - b + kRun - 1) / kRun) : 0u;
    const uint64_t t_key_end = any && !is_long ? min(t_hi, seg_end / kTile) : 0;
    const uint32_t nt = any && !is_long && t_key_end > t0 ? (uint32_t)(t_key_end - t0) : 0u;
    const unsigned long long rk =
        ordered ? ordered_run_base(p, cta, nrun, nullptr)
                : warp_alloc(seg, nrun, [&](uint64_t s) { return seg_counter(p, s, 1); });
    const unsigned long long sk = warp_alloc(seg, nt, [&](uint64_t s) { return seg_counter(p, s, 2); });
    if (!live) return;
    if (any) {
        if (is_long) {
            if (t_lo < t_hi) {
                p.tile_first[t_lo] = (uint32_t)idx;
                p.tile_first[t_hi - 1] = (uint32_t)idx;
            }
            write_runs(p, (uint32_t)idx, seg, rk, b, min(e, seg_end));
            for (uint64_t s2 = seg + 1; s2 * p.seg_slots < e; ++s2) {
                const uint64_t lo = s2 * p.seg_slots, hi = min(e, (s2 + 1) * p.seg_slots);
                const unsigned long long k = atomicAdd(
                    seg_counter(p, s2, 1), (unsigned long long)((hi - lo + kRun - 1) / kRun));
                write_runs(p, (uint32_t)idx, s2, k, lo, hi);
            }
        } else {
            for (uint64_t t = t_lo; t < t_hi; ++t) p.tile_first[t] = (uint32_t)idx;
            uint32_t* list = p.short_all + seg * p.seg_slots / kTile + sk;
            const uint64_t cap = seg_tiles(p, seg);
            for (uint32_t q = 0; q < nt && sk + q < cap; ++q) list[q] = (uint32_t)(t0 + q);
            for (uint64_t t = max(t0, t_key_end); t < t_hi; ++t) list_short_tile(p, t);
        }
    }
    if (idx + 1 == p.n_slices) uncovered_tail(p, p.n_slices, e > b ? e : b);
    if (idx == 0) p.tile_first[p.n_tiles] = p.n_slices;
}

// The empty chunk's tile index: every slot is uncovered.
__global__ void prep_empty_kernel(const KParams p) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.ctr_all) {
        p.tile_first[p.n_tiles] = 0;
        uncovered_tail(p, 0, 0);
    }
}

// Probe bitmaps (one warp per slice): bits of the probe's tokens relative to `lo`, then the
// number of probe tokens below every word (warp-wide exclusive scan).
__global__ void bitmap_kernel(const KParams p) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    // one warp per slice listed by prep_kernel
    const uint64_t n_list = *(volatile unsigned long long*)(p.acc + kAccBitmapSlices);
    for (uint64_t it = warp; it < n_list; it += n_warps) {
        const uint32_t e = __ldg(p.bm_list + it);
        const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(p.slices + e));
        const uint4 d1 = __ldg(reinterpret_cast<const uint4*>(p.slices + e) + 1);
        uint32_t* bits = p.bm_bits + d0.w;
        uint32_t* rank = p.bm_rank + d0.w;
        const uint32_t lo = d1.x, nw = d1.y;
        for (uint32_t w = lane; w < bitmap_alloc_words(nw); w += 32) bits[w] = 0;
        __syncwarp();
        const uint32_t* r = p.tokens + (size_t)d0.y * 8;
        for (uint32_t u = lane; u < d0.z; u += 32) {
            const uint32_t dd = __ldg(r + u) - lo;
            atomicOr(bits + (dd >> 5), 1u << (dd & 31));
        }
        __threadfence_block();
        __syncwarp();
        // ranks, 128 words per round: lane l takes words 4l..4l+3 in one 16-byte load (the
        // allocation is a multiple of 4 words and zero past nw), so a 1,300-word probe takes
        // 11 round trips to L2 instead of 41
        const uint32_t alloc = bitmap_alloc_words(nw);
        uint32_t carry = 0;
        for (uint32_t base = 0; base < nw; base += 128) {
            const uint32_t w = base + 4 * lane;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (w < alloc) v = __ldcg(reinterpret_cast<const uint4*>(bits + w));
            const uint32_t c0 = __popc(v.x), c1 = __popc(v.y), c2 = __popc(v.z), c3 = __popc(v.w);
            const uint32_t tot = c0 + c1 + c2 + c3;
            uint32_t incl = tot;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= (uint32_t)off) incl += u;
            }
            const uint32_t x = carry + incl - tot;
            if (w < nw) rank[w] = x;
            if (w + 1 < nw) rank[w + 1] = x + c0;
            if (w + 2 < nw) rank[w + 2] = x + c0 + c1;
            if (w + 3 < nw) rank[w + 3] = x + c0 + c1 + c2;
            carry += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

// ---------------------------------------------------------------------------------------
// Required overlap: table lookup by |r| + |s| for Jaccard / Dice (the value depends on the
// sum only; the table is filled on the host with the exact u128 formula), else the formula.
__device__ __forceinline__ uint64_t required_of(const KParams& p, uint32_t m, uint32_t n) {
    const uint32_t sum = m + n;
    if (p.req_tab && sum < p.req_tab_n) return __ldg(p.req_tab + sum);
    return dev_required(p.pred, m, n);
}

// Membership-bitmap verification of one pair: bits[k] holds probe tokens lo+32k..lo+32k+31,
// rank[k] the number of probe tokens below lo+32k (shared or global memory). The candidate
// is walked in blocks of 8 tokens (registers); after each block the merge position is known
// exactly -- j = candidate tokens consumed, i = #probe tokens <= the block's last token -- so
// the reference's bound (verify.hpp:58) is evaluated at (i, j): sound, and the verdict is
// bit-exact. The 8 lookups of a block are independent (no dependent load chain).
template <bool kFull>
__device__ __forceinline__ bool verify_bitmap(const uint32_t* __restrict__ bits,
                                              const uint32_t* __restrict__ rank, uint32_t lo,
                                              uint32_t nbits, uint32_t m,
                                              const uint4* __restrict__ s4, uint32_t n,
                                              uint32_t req, uint4 w0, uint4 w1,
                                              uint32_t* ov_out) {
    const uint32_t slack_r = m - req, slack_s = n - req;
    uint32_t ov = 0, j = 0;
    for (;;) {
        const uint32_t t[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        const uint32_t cnt = min(8u, n - j);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const uint32_t d = t[q] - lo;
            const bool in = (uint32_t)q < cnt && d < nbits;
            const uint32_t word = in ? bits[d >> 5] : 0u;
            ov += (word >> (d & 31)) & 1u;
        }
        j += cnt;
        if (j >= n) break;  // s exhausted: the verdict is ov >= req
        if (!kFull && ov >= req) break;
        if (ov < req) {
            const uint32_t tl = t[7];  // cnt == 8 here (s not exhausted)
            const uint32_t d = tl - lo;
            uint32_t i;
            if (tl < lo) {
                i = 0;
            } else if (d >= nbits) {
                i = m;
            } else {
                i = rank[d >> 5] + __popc(bits[d >> 5] & ((2u << (d & 31)) - 1u));
            }
            if (i - ov > slack_r || j - ov > slack_s) {
                if (kFull) *ov_out = 0;
                return false;
            }
        }
        w0 = __ldg(s4 + (j >> 2));
        w1 = __ldg(s4 + (j >> 2) + 1);
    }
    if (kFull) *ov_out = ov >= req ? ov : 0;
    return ov >= req;
}


// ---------------------------------------------------------------------------------------
// Strategy A, warp-tile form: every warp owns kTile = 32 * kItems consecutive slots and works
// alone -- no shared memory, no CTA barriers. Lane l owns slots slot0 + l*kItems + [0, kItems)
// (C ids in one vector load, flags in one vector store). The slices of the warp tile (first
// one from the prep kernel's index) are read one per lane; a slot's slice is found by a
// 5-step shuffle binary search over those ends. Slice descriptors, probe bitmaps and probe
// tokens are read through L1 (lanes of a tile share them). Long candidates are left to
// long_slice_kernel (their slice is marked).
// The tile's loads that do not depend on other loads: the lane's C ids and the tile's first
// and last slice (prefetched one tile ahead by warp_tile_kernel).
struct TilePre {
    uint32_t cand[SSJB_TILE_ITEMS];
    uint32_t e0, e1;
};

__device__ __forceinline__ void tile_prefetch(const KParams& p, uint32_t tile, TilePre& t) {
    constexpr int kItems = SSJB_TILE_ITEMS;
    const uint64_t slot0 = (uint64_t)tile * kTile;
    const uint64_t slot1 = min(slot0 + (uint64_t)kTile, p.nC);
    const uint64_t my0 = slot0 + (uint64_t)(threadIdx.x & 31) * kItems;
#pragma unroll
    for (int q = 0; q < kItems; ++q) t.cand[q] = my0 + q < slot1 ? __ldg(p.C + my0 + q) : 0u;
    t.e0 = slot0 < p.nC ? __ldg(p.tile_first + tile) : kNone;
    t.e1 = slot0 < p.nC ? __ldg(p.tile_first + tile + 1) : kNone;
}

template <int kOut, bool kStats, bool kPacked>
__device__ __forceinline__ void warp_tile(const KParams& p, const uint32_t tile, const TilePre& pre,
                                          unsigned& count, unsigned& prunes, unsigned& verified) {
    constexpr int kItems = SSJB_TILE_ITEMS;
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t slot0 = (uint64_t)tile * kTile;
    if (slot0 >= p.nC) return;
    const uint64_t slot1 = min(slot0 + (uint64_t)kTile, p.nC);
    const uint64_t my0 = slot0 + (uint64_t)lane * kItems;

    uint32_t cand[kItems];
#pragma unroll
    for (int q = 0; q < kItems; ++q) cand[q] = pre.cand[q];
    uint2 sd[kItems];
    uint32_t hr[kPacked ? kItems : 1][8];  // kPacked: the candidates' head records
    if (kPacked) {
        // one 256-bit load per candidate: first 8 tokens, CSR position and |s|
#pragma unroll
        for (int q = 0; q < kItems; ++q) {
            if (cand[q] < p.n_sets) {
                ld_tokens8(reinterpret_cast<const uint32_t*>(p.heads + 2 * (size_t)cand[q]), hr[q]);
            } else {
#pragma unroll
                for (int u = 0; u < 8; ++u) hr[q][u] = 0;
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < kItems; ++q)
            sd[q] = cand[q] < p.n_sets ? __ldg(p.sets + cand[q]) : make_uint2(0, 0);
    }

    const uint32_t e0 = pre.e0;
    uint32_t ns = 0;
    if (e0 < p.n_slices) {
        uint32_t e_hi = pre.e1;
        if (e_hi >= p.n_slices) e_hi = p.n_slices - 1;
        ns = e_hi - e0 + 1;
    }
    const bool small = ns <= 32;  // warp-uniform
    const uint32_t my_end = lane < ns ? __ldg(p.C_O + 2 * ((size_t)e0 + lane) + 1) : 0xFFFFFFFFu;
    const uint32_t beg0 = (e0 && e0 < p.n_slices) ? __ldg(p.C_O + 2 * (size_t)e0 - 1) : 0u;
    // small tiles: lane l also holds slice e0 + l's descriptor (loaded beside its end), and a
    // slot takes its slice's descriptor by shuffles -- no dependent load after the search
    uint4 my_d0 = make_uint4(0, 0, 0, kNone);
    if (SSJB_TILE_DESC_SHFL && small && lane < ns)
        my_d0 = __ldg(reinterpret_cast<const uint4*>(p.slices + e0 + lane));

    uint4 nw0, nw1;
    if (!kPacked) {
        const uint4* s4 = reinterpret_cast<const uint4*>(p.tokens + (size_t)sd[0].x * 8);
        nw0 = __ldg(s4);
        nw1 = __ldg(s4 + 1);
    }
    uint32_t flag_bits[(kItems + 3) / 4] = {};
    bool all_written = true;
#pragma unroll
    for (int q = 0; q < kItems; ++q) {
        const uint64_t slot = my0 + q;
        uint4 cw0, cw1;
        if (kPacked) {
            sd[q].x = __byte_perm(__byte_perm(hr[q][0], hr[q][1], 0x0073), __byte_perm(hr[q][2], hr[q][3], 0x0073), 0x5410);
            sd[q].y = __byte_perm(__byte_perm(hr[q][4], hr[q][5], 0x0073), __byte_perm(hr[q][6], hr[q][7], 0x0073), 0x5410);
            cw0 = make_uint4(hr[q][0] & kHeadTokenMask, hr[q][1] & kHeadTokenMask,
                             hr[q][2] & kHeadTokenMask, hr[q][3] & kHeadTokenMask);
            cw1 = make_uint4(hr[q][4] & kHeadTokenMask, hr[q][5] & kHeadTokenMask,
                             hr[q][6] & kHeadTokenMask, hr[q][7] & kHeadTokenMask);
        } else {
            cw0 = nw0;
            cw1 = nw1;
            if (q + 1 < kItems) {
                const uint4* s4n = reinterpret_cast<const uint4*>(p.tokens + (size_t)sd[q + 1].x * 8);
                nw0 = __ldg(s4n);
                nw1 = __ldg(s4n + 1);
            }
        }
        // slice of this slot: number of the tile's slice ends <= slot (all lanes shuffle)
        uint32_t li = 0;
        uint32_t s_end = 0, s_beg = 0;
        if (small) {
            const uint32_t key = (uint32_t)min(slot, (uint64_t)0xFFFFFFFEu);
#pragma unroll
            for (uint32_t step = 16; step > 0; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, my_end, li + step - 1);
                if (v <= key) li += step;
            }
            const uint32_t v = __shfl_sync(0xffffffffu, my_end, li & 31);
            if (li < 32 && v <= key) ++li;
            s_end = __shfl_sync(0xffffffffu, my_end, li & 31);
            const uint32_t pe = __shfl_sync(0xffffffffu, my_end, (li - 1) & 31);
            s_beg = li ? pe : beg0;
        }
        uint4 d0s = make_uint4(0, 0, 0, kNone);
        if (SSJB_TILE_DESC_SHFL && small) {
            d0s.x = __shfl_sync(0xffffffffu, my_d0.x, li & 31);
            d0s.y = __shfl_sync(0xffffffffu, my_d0.y, li & 31);
            d0s.z = __shfl_sync(0xffffffffu, my_d0.z, li & 31);
            d0s.w = __shfl_sync(0xffffffffu, my_d0.w, li & 31);
        }
        // a tile without slices lies past the last C_O end: never verified, flag 0
        bool met = false, written = ns == 0;
        uint32_t ov = 0;
        if (slot < slot1 && ns) {
            uint32_t e = e0 + li;
            if (!small) {
                // the slot's slice is among the tile's ns slices (tile_first[t + 1] bounds
                // them): a short search whose C_O loads hit the lines my_end just read
                e = upper_bound_ends(p.C_O, e0, min(e0 + ns, p.n_slices), slot);
                if (e < p.n_slices) {
                    s_end = __ldg(p.C_O + 2 * (size_t)e + 1);
                    s_beg = e ? __ldg(p.C_O + 2 * (size_t)e - 1) : 0u;
                }
            }
            // slots of slices with >= kRunMinSlice candidates belong to run_kernel
            const bool in_run = e < p.n_slices && (!small || li < ns) && s_end > s_beg &&
                                min((uint64_t)s_end, p.nC) - s_beg >= kRunMinSlice;
            if (in_run) {
                // flag written by run_kernel
            } else if (e < p.n_slices && (!small || li < ns)) {
                written = true;
                const uint4 d0 = (SSJB_TILE_DESC_SHFL && small)
                                     ? d0s
                                     : __ldg(reinterpret_cast<const uint4*>(p.slices + e));
                const uint32_t m = d0.z;
                const uint32_t* r = p.tokens + (size_t)d0.y * 8;
                if (cand[q] >= p.n_sets) {
                    flag_error(p.acc, kErrOutOfRange);
                } else {
                    const uint32_t n = sd[q].y;
                    const uint4* s4 = reinterpret_cast<const uint4*>(p.tokens + (size_t)sd[q].x * 8);
                    const uint64_t req = required_of(p, m, n);
                    bool deferred = false;
                    if (p.defer && n > kLongPair && req >= 1 && req <= (uint64_t)min(m, n)) {
                        mark_long_slice(p, e);
                        deferred = true;
                        written = false;  // long_slice_kernel writes it
                    }
                    if (deferred) {
                        // verdict, flag and stats come from long_slice_kernel
                    } else if (req == 0) {
                        met = true;  // verify.hpp:57: no comparison, met = (0 >= 0)
                        if (kOut == kOutResults)
                            ov = full_overlap_seq(r, m, reinterpret_cast<const uint32_t*>(s4), n);
                    } else if (req <= (uint64_t)min(m, n)) {
                        if (d0.w != kNone) {
                            const uint2 d1 = __ldg(reinterpret_cast<const uint2*>(p.slices + e) + 2);
                            met = verify_bitmap<kOut == kOutResults>(
                                p.bm_bits + d0.w, p.bm_rank + d0.w, d1.x, d1.y * 32, m, s4, n,
                                (uint32_t)req, cw0, cw1, &ov);
                        } else {
                            met = merge_thread<kOut == kOutResults>(r, m, s4, n, (uint32_t)req,
                                                                    cw0, cw1, &ov);
                        }
                    }
                    if (kStats && !deferred) {
                        ++verified;
                        prunes += (!met && (m + n) > 0);
                    }
                }
            } else {
                written = true;  // slot past the last slice: never verified, flag 0
            }
        }
        all_written = all_written && (written || slot >= slot1);
        count += met;
        flag_bits[q >> 2] |= (met ? 1u : 0u) << (8 * (q & 3));
        if (kOut == kOutFlags && !written && slot < slot1) flag_bits[q >> 2] |= 0x80u << (8 * (q & 3));
        if (kOut == kOutResults) warp_append(p, met, slot, ov);
    }
    if (kOut == kOutFlags) {
        if (all_written && kItems == 8 && my0 + kItems <= slot1 && (((uintptr_t)(p.flags + my0)) & 7) == 0) {
            *reinterpret_cast<uint2*>(p.flags + my0) = make_uint2(flag_bits[0], flag_bits[1 % ((kItems + 3) / 4)]);
        } else if (all_written && kItems == 4 && my0 + kItems <= slot1 && (((uintptr_t)(p.flags + my0)) & 3) == 0) {
            *reinterpret_cast<uint32_t*>(p.flags + my0) = flag_bits[0];
        } else if (all_written && kItems == 2 && my0 + kItems <= slot1 && (((uintptr_t)(p.flags + my0)) & 1) == 0) {
            *reinterpret_cast<uint16_t*>(p.flags + my0) = (uint16_t)flag_bits[0];
        } else {
#pragma unroll
            for (int q = 0; q < kItems; ++q) {
                const uint32_t f = (flag_bits[q >> 2] >> (8 * (q & 3))) & 0xFFu;
                if (my0 + q < slot1 && !(f & 0x80u)) p.flags[my0 + q] = f & 1u;
            }
        }
    }
}

// Strategy A, warp-tile form: every warp owns kTile = 32 * kItems consecutive slots and works
// alone -- no shared memory, no CTA barriers. Lane l owns slots slot0 + l*kItems + [0, kItems)
// (C ids in one vector load, flags in one vector store). The slices of the warp tile (first
// one from the prep kernel's index) are read one per lane; a slot's slice is found by a
// 5-step shuffle binary search over those ends. Slice descriptors, probe bitmaps and probe
// tokens are read through L1 (lanes of a tile share them). Long candidates are left to
// long_slice_kernel. Persistent over the segment's short-tile list; slots of slices with
// >= kRunMinSlice candidates are left to run_kernel.
template <int kOut, bool kStats, bool kPacked>
__global__ void __launch_bounds__(kThreadsA, kTileMinBlocks) warp_tile_kernel(const KParams p) {
    const uint64_t n = min((uint64_t)*p.short_n, p.short_cap);
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t n_warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned count = 0, prunes = 0, verified = 0;
    // software pipeline over the warp's tiles: the next tile's C ids and slice bounds are in
    // flight while this tile is verified, the tile after next's index one step earlier.
    // Tiles are taken dynamically from a per-launch counter (p.defer_n[4]): their cost varies
    // with the pair lengths, and a static stride leaves SMs idle in the launch's tail.
    const uint32_t lane = threadIdx.x & 31;
    // (only when warps get several tiles each: with ~2 per warp the atomics cost more than
    // the tail they remove)
    unsigned long long* const ctr =
        SSJB_TILE_DYN && p.defer_n && n >= 4 * n_warps ? p.defer_n + 4 : nullptr;
    uint64_t step_i = 0;
    auto next_index = [&]() -> uint64_t {  // warp-uniform
        if (!ctr) return gw + (step_i++) * n_warps;
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(ctr, 1ull);
        return __shfl_sync(0xffffffffu, t, 0);
    };
    uint64_t w = next_index();
    uint64_t wn = w < n ? next_index() : n;
    uint32_t tile = w < n ? __ldg(p.short_tiles + w) : 0u;
    uint32_t tile_n = wn < n ? __ldg(p.short_tiles + wn) : 0u;
    TilePre cur;
    if (w < n) tile_prefetch(p, tile, cur);
    while (w < n) {
        TilePre nxt;
        const bool more = wn < n;
        if (more) tile_prefetch(p, tile_n, nxt);
        const uint64_t wnn = more ? next_index() : n;
        const uint32_t tile_nn = wnn < n ? __ldg(p.short_tiles + wnn) : 0u;
        warp_tile<kOut, kStats, kPacked>(p, tile, cur, count, prunes, verified);
        if (more) cur = nxt;
        w = wn;
        wn = wnn;
        tile = tile_n;
        tile_n = tile_nn;
    }
    acc_add(p.acc, 0, count);
    if (kStats) {
        acc_add(p.acc, 2, verified);
        acc_add(p.acc, 3, prunes);
    }
}

// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}


// mbarrier helpers (shared::cta); try_wait has acquire, arrive release semantics (CTA scope).
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
                 "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "W%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra W%=;\n}\n" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
        "r"(parity) : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred P;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(b)), "r"(parity) : "memory");
    return ok != 0;
}

// One warp builds a probe's map in shared memory (byte map over [lo, lo + 32 nw) with entry
// 32 nw empty, then the bitmap words and the per-word ranks for the exact bound) and
// publishes it on `full`. Out of line: it runs once per slice change, and inlined its
// registers would weigh on the verification loop.
__device__ __noinline__ void build_probe_map(const KParams& p, uint8_t* mp, uint32_t rpos8,
                                             uint32_t rsize, uint32_t lo, uint32_t nw,
                                             uint32_t bofs, uint64_t* full) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t range = nw * 32u;
    const uint32_t* r = p.tokens + (size_t)rpos8 * 8;
    uint32_t* sb = reinterpret_cast<uint32_t*>(mp + kRunMapBytes);
    for (uint32_t u = lane; u * 16 <= range; u += 32)
        reinterpret_cast<uint4*>(mp)[u] = make_uint4(0, 0, 0, 0);
    if (SSJB_RUN_OWN_BITMAP) {
        for (uint32_t w = lane; w < nw; w += 32) sb[w] = 0;
        __syncwarp();
        for (uint32_t i = lane; i < rsize; i += 32) {
            const uint32_t d = __ldg(r + i) - lo;
            mp[d] = 1;
            atomicOr(sb + (d >> 5), 1u << (d & 31));
        }
        __syncwarp();
        // lane l: words [l*per, l*per + per) (per <= 8), exclusive warp scan of their counts
        const uint32_t per = (nw + 31) / 32;
        uint32_t tot = 0;
        for (uint32_t q = 0, w = lane * per; q < per && w < nw; ++q, ++w) tot += __popc(sb[w]);
        uint32_t incl = tot;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= (uint32_t)off) incl += v;
        }
        uint32_t x = incl - tot;
        for (uint32_t q = 0, w = lane * per; q < per && w < nw; ++q, ++w) {
            sb[kRunMapWords + w] = x;
            x += __popc(sb[w]);
        }
    } else {  // copied from the prep pass's global bitmap
        for (uint32_t w = lane; w < nw; w += 32) {
            sb[w] = __ldg(p.bm_bits + bofs + w);
            sb[kRunMapWords + w] = __ldg(p.bm_rank + bofs + w);
        }
        __syncwarp();
        for (uint32_t i = lane; i < rsize; i += 32) mp[__ldg(r + i) - lo] = 1;
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) mbar_arrive(full);
}

// Per-run uniform state (every thread holds the same values).
struct RunState {
    uint32_t begin, end;      // slots
    uint32_t slice;           // slice index (kNone: no run)
    uint32_t rpos8, rsize;    // probe
    uint32_t bofs, lo, nw;    // probe bitmap (bofs = kNone: none)
};

__device__ __forceinline__ void load_run(const KParams& p, uint64_t k, uint64_t nr, RunState& r) {
    if (k < nr) {
        const uint4 d = __ldg(reinterpret_cast<const uint4*>(p.runs) + k);
        r.slice = d.x;
        r.begin = d.y;
        r.end = d.z;
    } else {
        r.slice = kNone;
        r.begin = r.end = 0;
    }
}

__device__ __forceinline__ void load_slice(const KParams& p, RunState& r) {
    if (r.slice != kNone) {
        const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(p.slices + r.slice));
        const uint2 d1 = __ldg(reinterpret_cast<const uint2*>(p.slices + r.slice) + 2);
        r.rpos8 = d0.y;
        r.rsize = d0.z;
        r.bofs = d0.w;
        r.lo = d1.x;
        r.nw = d1.y;
    } else {
        r.rpos8 = r.rsize = 0;
        r.bofs = kNone;
        r.lo = r.nw = 0;
    }
}

// Membership of 8 tokens in the probe: tokens outside [lo, lo + R) -- including the padding
// past |s| -- are clamped onto entry R, which is always empty, so a block costs 8
// unconditional lookups.
//   kMap   : byte map in shared memory (map[d] = 1 iff lo + d is a probe token), R = range
//   !kMap  : membership bitmap in global memory (word R/32 is zero), read through L1
template <bool kMap>
__device__ __forceinline__ uint32_t count8(const uint8_t* __restrict__ map,
                                           const uint32_t* __restrict__ bits, uint32_t lo,
                                           uint32_t R, const uint32_t t[8]) {
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t d = min(t[q] - lo, R);
        if (kMap) c += map[d];
        else c += (__ldg(bits + (d >> 5)) >> (d & 31)) & 1u;
    }
    return c;
}

// Continue a pair after its first 8 tokens (j = 8, ov = matches so far), 8 tokens per step
// from the CSR (256-bit loads). After each step the merge position is exact (j = tokens of s
// consumed, i = probe tokens <= the step's last token, from the global bitmap's rank), so
// the reference's bound (verify.hpp:58) is evaluated there; verdicts are bit-exact (see
// ssj_device.cuh).
// Probe tokens <= t (the merge position i on the probe side once s's tokens up to t are
// consumed), from the probe bitmap's words and per-word ranks.
template <bool kMap>
__device__ __forceinline__ uint32_t probe_rank(const uint32_t* __restrict__ bits,
                                               const uint32_t* __restrict__ rank, uint32_t lo,
                                               uint32_t nbits, uint32_t m, uint32_t t) {
    const uint32_t d = t - lo;
    if (t < lo) return 0;
    if (d >= nbits) return m;
    const uint32_t w = kMap ? bits[d >> 5] : __ldg(bits + (d >> 5));
    const uint32_t rk = kMap ? rank[d >> 5] : __ldg(rank + (d >> 5));
    return rk + __popc(w & ((2u << (d & 31)) - 1u));
}

template <bool kFull, bool kMap>
__device__ __forceinline__ bool bm_continue(const uint8_t* __restrict__ map,
                                            const uint32_t* __restrict__ bits,
                                            const uint32_t* __restrict__ rank, uint32_t lo,
                                            uint32_t nbits, uint32_t m,
                                            const uint32_t* __restrict__ s, uint32_t n,
                                            uint32_t req, uint32_t ov, uint32_t* ov_out,
                                            unsigned long long ttex, uint32_t spos8) {
    const uint32_t slack_r = m - req, slack_s = n - req;
    uint32_t j = 8;
    for (;;) {
        uint32_t t[8];
        if (SSJB_CONT_TEX && ttex) tex_tokens8(ttex, (uint64_t)spos8 + (j >> 3), t);
        else ld_tokens8(s + j, t);
        ov += count8<kMap>(map, bits, lo, nbits, t);
        j += 8;
        if (j >= n) break;  // s exhausted (padding never matches): the verdict is ov >= req
        if (!kFull && ov >= req) break;
        if (ov < req) {
            const uint32_t i = probe_rank<kMap>(bits, rank, lo, nbits, m, t[7]);
            if (i - ov > slack_r || j - ov > slack_s) {
                if (kFull) *ov_out = 0;
                return false;
            }
        }
    }
    if (kFull) *ov_out = ov >= req ? ov : 0;
    return ov >= req;
}

// Required overlap of a run's pair: the engine's table by |r| + |s| (Jaccard / Dice; one
// L1-resident load: a run's candidates span a few table lines) or the exact 32-bit formula.
__device__ __forceinline__ uint32_t run_required(const KParams& p, uint32_t m, uint32_t n) {
    if (SSJB_RUN_REQTAB && p.req_tab) return __ldg(p.req_tab + m + n);  // m, n <= max set size
    return dev_required_fast(p.pred, m, n);
}

// Long pairs of a run are left to long_slice_kernel: one lane marks the run's slice (all 32
// lanes call it).
__device__ __forceinline__ bool warp_defer(const KParams& p, bool want, uint32_t slice) {
    const unsigned mask = __ballot_sync(0xffffffffu, want);
    if (mask && (threadIdx.x & 31) == (uint32_t)(__ffs(mask) - 1)) mark_long_slice(p, slice);
    return want;
}

// Verify one run whose probe has a bitmap, in two phases per warp:
//  1. every lane tests the first 8 tokens of each of its kRunItems candidates (staged in
//     shared memory at hd) against the probe; the pair is decided when |s| <= 8, when the
//     overlap already reaches `required` (not in results mode), or when the s-side bound
//     (verify.hpp:58) rejects it; otherwise (slot, s, |s|, required, overlap) goes to the
//     warp's queue (in the heads area, behind the items still to be read);
//  2. the queue is drained 32 entries per round with bm_continue (no divergence between
//     lanes whose pairs need one block and lanes whose pairs need several).
// pos8[q] / n[q]: the candidate's CSR position and size (pos8 = kNone: no candidate);
// kPacked: the staged heads are packed records (tokens in the low 24 bits).
template <int kOut, bool kStats, bool kMap, bool kPacked, bool kReg>
__device__ __forceinline__ void run_bitmap(const KParams& p, const RunState& R,
                                           const uint32_t* pos8, const uint32_t* nn,
                                           const uint8_t* __restrict__ map,
                                           const uint32_t* __restrict__ bits,
                                           const uint32_t* __restrict__ rank, uint4* hd,
                                           const uint32_t (&hr)[kRunItems][8],
                                           unsigned& count, unsigned& prunes,
                                           unsigned& verified) {
    constexpr bool kFull = kOut == kOutResults;
    constexpr uint32_t T = kRunThreads, I = kRunItems;
    const uint32_t lane = threadIdx.x & 31, tid = threadIdx.x;
    const uint32_t m = R.rsize, lo = R.lo, nbits = R.nw * 32u;
    uint32_t nq = 0;
    uint32_t rqv[I];  // every item's required overlap first: the table loads overlap
#pragma unroll
    for (uint32_t q = 0; q < I; ++q) rqv[q] = pos8[q] != kNone ? run_required(p, m, nn[q]) : 0u;
#pragma unroll
    for (uint32_t q = 0; q < I; ++q) {
        const uint32_t slot = R.begin + q * T + tid;
        const bool valid = pos8[q] != kNone;
        const uint32_t n = nn[q];
        const uint32_t rq = rqv[q];
        const bool inrange = valid && rq >= 1 && rq <= min(m, n);
        const bool deferred = warp_defer(p, inrange && n > kLongPair, R.slice);
        bool met = valid && rq == 0, decided = true;
        uint32_t ov = 0;
        if (inrange && !deferred) {
            uint32_t t8[8];
            if (kReg) {
#pragma unroll
                for (int u = 0; u < 8; ++u) t8[u] = hr[q][u];
            } else {
                const uint4 w0 = hd[(q * 32 + lane) * 2], w1 = hd[(q * 32 + lane) * 2 + 1];
                t8[0] = w0.x; t8[1] = w0.y; t8[2] = w0.z; t8[3] = w0.w;
                t8[4] = w1.x; t8[5] = w1.y; t8[6] = w1.z; t8[7] = w1.w;
            }
            if (kPacked) {
#pragma unroll
                for (int u = 0; u < 8; ++u) t8[u] &= kHeadTokenMask;
            }
            ov = count8<kMap>(map, bits, lo, nbits, t8);
            if (n <= 8) met = ov >= rq;
            else if (!kFull && ov >= rq) met = true;
            else if (ov < rq && 8u - ov > n - rq) met = false;
            else decided = false;
        } else if (kFull && met) {
            ov = full_overlap_seq(p.tokens + (size_t)R.rpos8 * 8, m,
                                  p.tokens + (size_t)pos8[q] * 8, n);
        }
        if (!kReg) __syncwarp();  // heads of item q read by every lane before the queue covers them
        const unsigned qmask = __ballot_sync(0xffffffffu, !decided);
        if (!decided)
            hd[nq + __popc(qmask & ((1u << lane) - 1u))] =
                make_uint4(slot, pos8[q], n, rq | (ov << 16));
        nq += __popc(qmask);
        if (valid && decided && !deferred) {
            if (kOut == kOutFlags) p.flags[slot] = met ? 1 : 0;
            if (kStats) {
                ++verified;
                prunes += (!met && (m + n) > 0);
            }
            count += met;
        }
        if (kFull) warp_append(p, valid && decided && !deferred && met, slot, ov);
    }
    __syncwarp();
    for (uint32_t base = 0; base < nq; base += 32) {
        const uint32_t e = base + lane;
        bool met = false;
        uint32_t ov = 0, slot = 0;
        if (e < nq) {
            const uint4 qe = hd[e];
            slot = qe.x;
            const uint32_t n = qe.z, rq = qe.w & 0xFFFFu;
            met = bm_continue<kFull, kMap>(map, bits, rank, lo, nbits, m,
                                           p.tokens + (size_t)qe.y * 8, n, rq, qe.w >> 16, &ov,
                                           p.tokens_tex, qe.y);
            if (kOut == kOutFlags) p.flags[slot] = met ? 1 : 0;
            if (kStats) {
                ++verified;
                prunes += (!met && (m + n) > 0);
            }
            count += met;
        }
        if (kFull) warp_append(p, met, slot, ov);
    }
    __syncwarp();  // queue read before the next heads land here
}

// A run whose probe has no bitmap: thread-sequential early-exit merge per candidate.
template <int kOut, bool kStats, bool kPacked, bool kReg>
__device__ __forceinline__ void run_merge(const KParams& p, const RunState& R,
                                          const uint32_t* pos8, const uint32_t* nn,
                                          const uint4* hd, unsigned& count, unsigned& prunes,
                                          unsigned& verified) {
    constexpr bool kFull = kOut == kOutResults;
    constexpr uint32_t T = kRunThreads, I = kRunItems;
    const uint32_t lane = threadIdx.x & 31, tid = threadIdx.x;
    const uint32_t m = R.rsize;
    const uint32_t* r = p.tokens + (size_t)R.rpos8 * 8;
#pragma unroll
    for (uint32_t q = 0; q < I; ++q) {
        const uint32_t slot = R.begin + q * T + tid;
        const bool valid = pos8[q] != kNone;
        const uint32_t n = nn[q];
        const uint32_t rq = valid ? run_required(p, m, n) : 0u;
        const bool inrange = valid && rq >= 1 && rq <= min(m, n);
        const bool deferred = warp_defer(p, inrange && n > kLongPair, R.slice);
        bool met = valid && rq == 0;
        uint32_t ov = 0;
        const uint32_t* s = p.tokens + (size_t)pos8[q] * 8;
        if (inrange && !deferred) {
            // the CSR (not the packed record) holds the exact tokens
            const uint4* s4 = reinterpret_cast<const uint4*>(s);
            const uint4 w0 = (kPacked || kReg) ? __ldg(s4) : hd[(q * 32 + lane) * 2];
            const uint4 w1 = (kPacked || kReg) ? __ldg(s4 + 1) : hd[(q * 32 + lane) * 2 + 1];
            met = merge_thread<kFull>(r, m, s4, n, rq, w0, w1, &ov);
        } else if (kFull && met) {
            ov = full_overlap_seq(r, m, s, n);
        }
        if (valid && !deferred) {
            if (kOut == kOutFlags) p.flags[slot] = met ? 1 : 0;
            if (kStats) {
                ++verified;
                prunes += (!met && (m + n) > 0);
            }
            count += met;
        }
        if (kFull) warp_append(p, valid && !deferred && met, slot, ov);
    }
    __syncwarp();
}

// run_kernel: persistent; CTA c of G verifies blocks c, c + G, c + 2G, ... of kRunBlock
// consecutive runs of the segment's list (the list follows slot order, and the runs of one
// slice are consecutive). All CTAs thus work on one moving window of the chunk -- the
// candidates of nearby probes share L2 -- and consecutive runs of a block usually share
// their slice.
//
// Thread t owns slots begin + q*kRunThreads + t (q < kRunItems) of every run. By default
// (kRunHeadBufs = 0, packed heads) the C ids are prefetched one run ahead and each
// candidate's 32-byte head record -- first 8 tokens, |s|, CSR position -- is gathered
// through the texture path straight into registers at the run's start (the variants with
// cp.async head buffers in shared memory remain for collections without packed heads).
// When a run starts a new slice whose probe spans <= kRunMapRange tokens, the probe's byte
// map, bitmap words and ranks are built in one of kMB shared buffers by ONE warp -- the
// first to get there -- and published with an mbarrier; the others wait for that
// publication only, never for each other (no CTA barrier). That warp also builds the next
// run's map ahead when its buffer is already free (kMB = 3 for short slices).
template <int kOut, bool kStats, bool kPacked, uint32_t kMB>
__global__ void __launch_bounds__(kRunThreads, kRunMinBlocks) run_kernel(const KParams p) {
    extern __shared__ __align__(16) uint32_t rsh[];
    constexpr uint32_t T = kRunThreads, I = kRunItems;
    // uint4 per warp head buffer; with register heads only the continuation queue (I*32)
    constexpr uint32_t HB = kRunHeadBufs == 0 ? I * 32 : I * 2 * 32;
    constexpr uint32_t NB = kRunHeadBufs;  // 0: heads in registers (LDG.256), queue-only buffer
    constexpr bool kReg = NB == 0;
    constexpr uint32_t NBS = kReg ? 1 : NB;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint4* const hbase = reinterpret_cast<uint4*>(rsh) + warp * (NBS * HB);  // [bufs][item][lane][half]
    // [2][kRunMapBuf]: probe byte map, then its bitmap words and ranks (for the exact bound)
    uint8_t* const s_map = reinterpret_cast<uint8_t*>(rsh + (T / 32) * NBS * HB * 4);
    const uint32_t nr = (uint32_t)min((uint64_t)*p.runs_n, p.runs_cap);
    // this CTA's runs: blocks blockIdx.x, blockIdx.x + G, ... of kRunBlock consecutive runs
    const uint32_t stride = (gridDim.x - 1) * kRunBlock;
    auto next_run = [&](uint32_t r) -> uint32_t {
        return ((r + 1) % kRunBlock) ? r + 1 : r + 1 + stride;
    };
    unsigned count = 0, prunes = 0, verified = 0;
    const uint32_t first = blockIdx.x * kRunBlock;
    if (first < nr) {
        auto map_ok = [](const RunState& r) {
            return (SSJB_RUN_OWN_BITMAP || r.bofs != kNone) && r.nw && r.nw * 32u <= kRunMapRange;
        };
        auto load_c = [&](const RunState& r, uint32_t* c) {
#pragma unroll
            for (uint32_t q = 0; q < I; ++q) {
                const uint32_t slot = r.begin + q * T + tid;
                c[q] = slot < r.end ? __ldg(p.C + slot) : kNone;  // checked when used
            }
        };
        // packed heads of the candidates c[] -> head buffer b (cp.async group per run);
        // returns the mask of items with a candidate
        auto issue_heads = [&](const uint32_t* c, uint32_t b) -> uint32_t {
            uint4* hd = hbase + b * HB;
            uint32_t vm = 0;
#pragma unroll
            for (uint32_t q = 0; q < I; ++q) {
                if (c[q] < p.n_sets) {
                    cp_async16(hd + (q * 32 + lane) * 2, p.heads + 2 * (size_t)c[q]);
                    cp_async16(hd + (q * 32 + lane) * 2 + 1, p.heads + 2 * (size_t)c[q] + 1);
                    vm |= 1u << q;
                } else if (c[q] != kNone) {
                    flag_error(p.acc, kErrOutOfRange);
                }
            }
            cp_async_commit();
            return vm;
        };
        auto load_d = [&](const uint32_t* c, uint2* d) {
#pragma unroll
            for (uint32_t q = 0; q < I; ++q) {
                d[q] = make_uint2(kNone, 0);
                if (c[q] < p.n_sets) d[q] = __ldg(p.sets + c[q]);
                else if (c[q] != kNone) flag_error(p.acc, kErrOutOfRange);
            }
        };

        uint32_t hr[I][8];  // kReg: first 8 tokens (packed records) of run k's candidates
        uint32_t run0 = first, run1 = next_run(first), run2 = next_run(run1);
        RunState R0, R1;
        load_run(p, run0, nr, R0);
        load_run(p, run1, nr, R1);
        load_slice(p, R0);
        uint32_t c[I];
        uint2 d0[I];  // !kPacked: set descriptors of run k (then k+1)
        load_c(R0, c);
        uint32_t vm0 = 0;  // kPacked: items of run k with a candidate
        if (kPacked) {
            if (NB == 2) vm0 = issue_heads(c, 0);
        } else {
            load_d(c, d0);
        }
        if (!kPacked || NB == 2) load_c(R1, c);
        uint32_t map_slice = kNone, mb = 0;  // slice whose map is in buffer mb
        // Probe maps without CTA barriers: every warp sees the same sequence of maps (k =
        // 0, 1, ...; map k in buffer k % NB). The first warp to reach map k claims its build
        // (s_claim), waits until every warp has left map k - NB (empty[k % NB]: one arrival
        // per warp), builds it alone and publishes it (full[k % NB]: one arrival). The other
        // warps only wait for the publication -- never for each other.
        __shared__ uint64_t s_full[kMB], s_empty[kMB];
        __shared__ uint32_t s_claim;
        uint32_t map_seq = 0;
        if (tid == 0) {
            for (uint32_t b = 0; b < kMB; ++b) {
                mbar_init(&s_full[b], 1);
                mbar_init(&s_empty[b], T / 32);
            }
            s_claim = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();

        for (uint32_t k = 0; run0 < nr; ++k) {
            const uint32_t hb = NB == 2 ? (k & 1u) : 0u;
            uint4* const hd = hbase + hb * HB;
            uint2 d1[I];
            uint32_t vm1 = 0;
            if (kReg) {
                // run k's heads straight into registers (one 256-bit load per candidate)
#pragma unroll
                for (uint32_t q = 0; q < I; ++q) {
                    if (kPacked && SSJB_RUN_TEX) {
                        // packed heads are only handed to the kernels with their texture
                        // (base_params), so no per-item pointer or texture checks here
                        const bool ok = c[q] < p.n_sets;
                        if (ok) tex_tokens8(p.heads_tex, c[q], hr[q]);
                        else if (c[q] != kNone) flag_error(p.acc, kErrOutOfRange);
                        vm1 |= (uint32_t)ok << q;
                        continue;
                    }
                    const uint32_t* src = nullptr;
                    if (kPacked) {
                        if (c[q] < p.n_sets) src = reinterpret_cast<const uint32_t*>(p.heads + 2 * (size_t)c[q]);
                        else if (c[q] != kNone) flag_error(p.acc, kErrOutOfRange);
                    } else if (d0[q].x != kNone) {
                        src = p.tokens + (size_t)d0[q].x * 8;
                    }
                    if (src) ld_tokens8(src, hr[q]);
                    if (kPacked) vm1 |= (src != nullptr) << q;
                }
                if (kPacked) vm0 = vm1;
                else load_d(c, d1);
            } else if (kPacked) {
                vm1 = issue_heads(c, NB == 2 ? hb ^ 1u : 0u);  // run k+1 (double buffer) or run k
                if (NB == 1) vm0 = vm1;
            } else {
                // heads of run k (cp.async) and descriptors of run k+1 (NB >= 1 here)
#pragma unroll
                for (uint32_t q = 0; q < I; ++q) {
                    if (d0[q].x != kNone) {
                        const uint4* src = reinterpret_cast<const uint4*>(p.tokens + (size_t)d0[q].x * 8);
                        cp_async16(hd + (q * 32 + lane) * 2, src);
                        cp_async16(hd + (q * 32 + lane) * 2 + 1, src + 1);
                    }
                }
                cp_async_commit();
                load_d(c, d1);
            }
            // prefetch: slice of run k+1, C ids of run k+2 (k+1 when single-buffered), run k+2
            load_slice(p, R1);
            RunState R2;
            load_run(p, run2, nr, R2);
            load_c((!kPacked || NB == 2) ? R2 : R1, c);

            // the probe's byte map (CTA-uniform condition)
            const bool use_map = map_ok(R0);
            if (use_map && R0.slice != map_slice) {
                map_slice = R0.slice;
                const uint32_t k = map_seq++;
                mb = k % kMB;
                __syncwarp();
                if (k > 0 && lane == 0) mbar_arrive(&s_empty[(k - 1) % kMB]);
                uint32_t won = 0;
                if (lane == 0)  // (a map built ahead is usually claimed already: no CAS)
                    won = *(volatile uint32_t*)&s_claim == k && atomicCAS(&s_claim, k, k + 1) == k;
                if (__shfl_sync(0xffffffffu, won, 0)) {
                    if (k >= kMB) mbar_wait(&s_empty[mb], ((k / kMB) - 1) & 1u);
                    build_probe_map(p, s_map + mb * kRunMapBuf, R0.rpos8, R0.rsize, R0.lo, R0.nw,
                                    R0.bofs, &s_full[mb]);
                }
                // build ahead: the next run opens a new mapped slice (map k + 1) and its buffer
                // is already free -- build it now instead of waiting for map k (a second map
                // ahead from run k+2, with a fourth buffer, measured slower: J 0.90 3.50 vs
                // 2.49 ms)
                auto try_ahead = [&](uint32_t kk, uint32_t rpos8, uint32_t rsize, uint32_t lo,
                                     uint32_t nw, uint32_t bofs) {
                    const uint32_t bb = kk % kMB;
                    uint32_t won1 = 0;
                    if (lane == 0 && *(volatile uint32_t*)&s_claim == kk &&
                        (kk < kMB || mbar_test(&s_empty[bb], ((kk / kMB) - 1) & 1u)))
                        won1 = atomicCAS(&s_claim, kk, kk + 1) == kk;
                    if (__shfl_sync(0xffffffffu, won1, 0))
                        build_probe_map(p, s_map + bb * kRunMapBuf, rpos8, rsize, lo, nw, bofs,
                                        &s_full[bb]);
                };
                if (SSJB_RUN_AHEAD) {
                    const bool new1 = R1.slice != R0.slice && map_ok(R1);
                    if (new1) try_ahead(k + 1, R1.rpos8, R1.rsize, R1.lo, R1.nw, R1.bofs);
                }
                mbar_wait(&s_full[mb], (k / kMB) & 1u);
            }

            uint32_t pos8[I], nn[I];
            if (kPacked) {
                if (!kReg) {
                    if (NB == 2) cp_async_wait<1>();  // run k's group (run k+1's may stay in flight)
                    else cp_async_wait<0>();
                    __syncwarp();
                }
#pragma unroll
                for (uint32_t q = 0; q < I; ++q) {
                    pos8[q] = kNone;
                    nn[q] = 0;
                    if (vm0 >> q & 1u) {
                        uint4 w0, w1;
                        if (kReg) {
                            w0 = make_uint4(hr[q][0], hr[q][1], hr[q][2], hr[q][3]);
                            w1 = make_uint4(hr[q][4], hr[q][5], hr[q][6], hr[q][7]);
                        } else {
                            w0 = hd[(q * 32 + lane) * 2];
                            w1 = hd[(q * 32 + lane) * 2 + 1];
                        }
                        pos8[q] = __byte_perm(__byte_perm(w0.x, w0.y, 0x0073), __byte_perm(w0.z, w0.w, 0x0073), 0x5410);
                        nn[q] = __byte_perm(__byte_perm(w1.x, w1.y, 0x0073), __byte_perm(w1.z, w1.w, 0x0073), 0x5410);
                    }
                }
            } else {
                if (!kReg) cp_async_wait<0>();
                __syncwarp();
#pragma unroll
                for (uint32_t q = 0; q < I; ++q) {
                    pos8[q] = d0[q].x;
                    nn[q] = d0[q].y;
                }
            }
            if (use_map) {
                const uint8_t* mp = s_map + mb * kRunMapBuf;
                const uint32_t* sb = reinterpret_cast<const uint32_t*>(mp + kRunMapBytes);
                run_bitmap<kOut, kStats, true, kPacked, kReg>(p, R0, pos8, nn, mp, sb,
                                                              sb + kRunMapWords, hd, hr, count,
                                                              prunes, verified);
            } else if (R0.bofs != kNone) {
                run_bitmap<kOut, kStats, false, kPacked, kReg>(p, R0, pos8, nn, nullptr,
                                                               p.bm_bits + R0.bofs,
                                                               p.bm_rank + R0.bofs, hd, hr,
                                                               count, prunes, verified);
            } else {
                run_merge<kOut, kStats, kPacked, kReg>(p, R0, pos8, nn, hd, count, prunes, verified);
            }

            R0 = R1;
            R1 = R2;
            run0 = run1;
            run1 = run2;
            run2 = next_run(run2);
            vm0 = vm1;
            if (!kPacked) {
#pragma unroll
                for (uint32_t q = 0; q < I; ++q) d0[q] = d1[q];
            }
        }
    }
    acc_add(p.acc, 0, count);
    if (kStats) {
        acc_add(p.acc, 2, verified);
        acc_add(p.acc, 3, prunes);
    }
}

// ---------------------------------------------------------------------------------------
// Strategy B: one CTA per probe slice, threads stride over the slice's candidates.
template <int kOut, bool kStats>
__global__ void block_kernel(const KParams p, const uint32_t rcap) {
    extern __shared__ __align__(16) uint32_t dsh[];
    unsigned count = 0, prunes = 0, verified = 0;
    for (uint32_t e = blockIdx.x; e < p.n_slices; e += gridDim.x) {
        const uint32_t begin = e ? __ldg(p.C_O + 2 * (size_t)e - 1) : 0;
        const uint32_t end = __ldg(p.C_O + 2 * (size_t)e + 1);
        if (end <= begin || (uint64_t)end > p.nC) continue;  // block-uniform
        const uint32_t probe = __ldg(p.C_O + 2 * (size_t)e);
        const uint2 rd = probe < p.n_sets ? __ldg(p.sets + probe) : make_uint2(0, 0);
        const uint32_t m = rd.y;
        const uint32_t padded = (m + 7u) & ~7u;
        const bool staged = padded <= rcap;
        __syncthreads();  // previous slice's readers are done with dsh
        if (staged) {
            const uint4* src = reinterpret_cast<const uint4*>(p.tokens + (size_t)rd.x * 8);
            uint4* dst = reinterpret_cast<uint4*>(dsh);
            for (uint32_t u = threadIdx.x; u < padded / 4; u += blockDim.x) dst[u] = __ldg(src + u);
        }
        __syncthreads();
        const uint32_t* r = staged ? dsh : p.tokens + (size_t)rd.x * 8;
        for (uint64_t base = begin; base < end; base += blockDim.x) {
            const uint64_t slot = base + threadIdx.x;
            bool met = false;
            uint32_t ov = 0;
            if (slot < end) {
                uint32_t n = 0;
                met = verify_pair<kOut>(p, r, m, __ldg(p.C + slot), &ov, &n);
                if (kStats) {
                    ++verified;
                    prunes += (!met && (m + n) > 0);
                }
                if (kOut == kOutFlags) p.flags[slot] = met ? 1 : 0;
            }
            count += met;
            if (kOut == kOutResults) warp_append(p, met, slot, ov);
        }
    }
    acc_add(p.acc, 0, count);
    if (kStats) {
        acc_add(p.acc, 2, verified);
        acc_add(p.acc, 3, prunes);
    }
}

// ---------------------------------------------------------------------------------------
// Strategy C: G lanes per pair over merge-path partitions, round-level early exit.
constexpr uint32_t kHops = 16;

// One pair walked by a group of G lanes (group-uniform control flow; gmask = the group's
// lanes). Each round the lanes take consecutive segments of kHops merge-path hops starting
// at the reference's diagonal split (verify.hpp:86-103) and count matches at their r-side
// hop (verify.hpp:157-163); counts are shuffle-reduced. After each round the merge position
// (iD, jD) at the round's last diagonal is exact, so the reference's bound
// overlap + min(m - iD, n - jD) < required (verify.hpp:58) is evaluated there. With kFull
// the path is walked to the end for qualifying pairs (ov = |r ∩ s|).
template <int G, bool kFull>
__device__ __forceinline__ bool path_pair(const uint32_t* r, uint32_t m, const uint32_t* s,
                                          uint32_t n, uint64_t req, uint32_t lane,
                                          unsigned gmask, uint32_t* ov_out) {
    if (req > (uint64_t)min(m, n)) {
        *ov_out = 0;
        return false;
    }
    if (req == 0 && !kFull) return true;
    const uint32_t total = m + n;
    uint32_t D = 0, ov = 0;
    while (D < total) {
        const uint32_t d = D + lane * kHops;
        uint32_t cnt = 0, ie = m, je = n;
        if (d < total) {
            uint32_t i = dev_merge_path_split(r, m, s, n, d);
            uint32_t j = d - i;
            const uint32_t hops = min(kHops, total - d);
            for (uint32_t h = 0; h < hops && (i < m || j < n); ++h) {
                if (j >= n || (i < m && r[i] <= s[j])) {
                    if (j < n && r[i] == s[j]) ++cnt;
                    ++i;
                } else {
                    ++j;
                }
            }
            ie = i;
            je = j;
        }
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) cnt += __shfl_xor_sync(gmask, cnt, off, G);
        ov += cnt;
        const uint32_t Dn = min(D + G * kHops, total);
        const uint32_t lb = (Dn - D - 1) / kHops;  // last lane with work
        const uint32_t iD = __shfl_sync(gmask, ie, lb, G);
        const uint32_t jD = __shfl_sync(gmask, je, lb, G);
        D = Dn;
        if (!kFull && ov >= req) {
            *ov_out = ov;
            return true;
        }
        if (ov < req && (uint64_t)ov + min(m - iD, n - jD) < req) {
            *ov_out = 0;
            return false;
        }
    }
    *ov_out = ov;  // full path walked: ov = |r ∩ s|
    return ov >= req;
}

template <int G, int kOut>
__global__ void path_kernel(const KParams p, const uint32_t rcap) {
    extern __shared__ __align__(16) uint32_t dsh[];
    const uint32_t lane = threadIdx.x % G;
    const uint32_t group = threadIdx.x / G;
    const uint32_t ngroups = blockDim.x / G;
    const unsigned gmask =
        G == 32 ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) / G * G));
    unsigned count = 0;
    for (uint32_t e = blockIdx.x; e < p.n_slices; e += gridDim.x) {
        const uint32_t begin = e ? __ldg(p.C_O + 2 * (size_t)e - 1) : 0;
        const uint32_t end = __ldg(p.C_O + 2 * (size_t)e + 1);
        if (end <= begin || (uint64_t)end > p.nC) continue;
        const uint32_t probe = __ldg(p.C_O + 2 * (size_t)e);
        const uint2 rd = probe < p.n_sets ? __ldg(p.sets + probe) : make_uint2(0, 0);
        const uint32_t m = rd.y;
        const uint32_t padded = (m + 7u) & ~7u;
        const bool staged = padded <= rcap;
        __syncthreads();
        if (staged) {
            const uint4* src = reinterpret_cast<const uint4*>(p.tokens + (size_t)rd.x * 8);
            uint4* dst = reinterpret_cast<uint4*>(dsh);
            for (uint32_t u = threadIdx.x; u < padded / 4; u += blockDim.x) dst[u] = __ldg(src + u);
        }
        __syncthreads();
        const uint32_t* r = staged ? dsh : p.tokens + (size_t)rd.x * 8;
        for (uint64_t base = begin; base < end; base += ngroups) {
            const uint64_t slot = base + group;
            bool met = false;
            uint32_t ov = 0;
            if (slot < end) {  // group-uniform
                const uint32_t cand = __ldg(p.C + slot);
                if (cand >= p.n_sets) {
                    if (lane == 0) flag_error(p.acc, kErrOutOfRange);
                } else {
                    const uint2 sd = __ldg(p.sets + cand);
                    met = path_pair<G, kOut == kOutResults>(
                        r, m, p.tokens + (size_t)sd.x * 8, sd.y, required_of(p, m, sd.y), lane,
                        gmask, &ov);
                }
                if (kOut == kOutFlags && lane == 0) p.flags[slot] = met ? 1 : 0;
            }
            const bool leader_met = met && lane == 0;
            count += leader_met;
            if (kOut == kOutResults) warp_append(p, leader_met, slot, ov);
        }
    }
    acc_add(p.acc, 0, count);
}

// ---------------------------------------------------------------------------------------
// Long pairs (candidate longer than kLongPair tokens), slice-parallel: CTA per slice marked
// by the first pass in this chunk segment. The CTA builds the probe's membership bitmap and
// per-word rank in shared memory (zero-fill, atomicOr scatter of the probe's tokens, block
// scan), then its warps sweep the slice's slots of the segment 32 at a time; every long
// candidate is verified by the whole warp: 32 candidate tokens per step (one coalesced 128 B
// load), membership lookups, popc(ballot), and the reference's bound (verify.hpp:58) at the
// exact merge position after the step's last token (rank lookup). Probes spanning more than
// kMaxBitmapWords words walk the merge path (path_pair) instead.
#ifndef SSJB_LONG_THREADS
#define SSJB_LONG_THREADS 512
#endif
constexpr uint32_t kLongThreads = SSJB_LONG_THREADS;
#ifndef SSJB_LONG_FIRST
#define SSJB_LONG_FIRST 128  // tokens of a long pair's first step (32 or 32 * kLongPerLane)
#endif
#ifndef SSJB_LONG_PER_LANE
#define SSJB_LONG_PER_LANE 4
#endif
constexpr uint32_t kLongPerLane = SSJB_LONG_PER_LANE;  // candidate tokens per lane per step
#ifndef SSJB_LONG_V2
#define SSJB_LONG_V2 1
#endif
#ifndef SSJB_LONG_DYN_SLICES
#define SSJB_LONG_DYN_SLICES 1
#endif

// Next-step token loads of the long pass. ptxas sinks plain (.nc) loads below the step's exit
// branches, next to their first use; a strong load keeps its place ahead of the lookups.
#ifndef SSJB_LONG_LD
#define SSJB_LONG_LD 2
#endif
__device__ __forceinline__ uint32_t ldg_nc_v(const uint32_t* p) {
    uint32_t v;
#if SSJB_LONG_LD == 0
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
#elif SSJB_LONG_LD == 1
    asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
#else
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
#endif
    return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
constexpr size_t kLongSmemBytes = (size_t)(2 * kMaxBitmapWords + 8) * 4 + kLongThreads * 16 + 16;

template <int kOut, bool kStats>
__global__ void __launch_bounds__(kLongThreads) long_slice_kernel(const KParams p,
                                                                  const uint64_t seg_lo,
                                                                  const uint64_t seg_hi) {
    extern __shared__ __align__(16) uint32_t lsh[];
    // bitmap capacity BW words: the collection's widest possible probe range (long_words, a
    // multiple of 4), so narrow-universe collections fit more CTAs per SM
    const uint32_t BW = p.long_words ? p.long_words : kMaxBitmapWords;
    uint32_t* const bits = lsh;                          // [BW + 4]
    uint32_t* const rank = lsh + BW + 4;                 // [BW + 4]
    uint4* const llist = reinterpret_cast<uint4*>(rank + BW + 4);  // [kLongThreads]
    uint32_t* const lcount = reinterpret_cast<uint32_t*>(llist + kLongThreads);
    const uint32_t bits_s = (uint32_t)__cvta_generic_to_shared(bits);
    const uint32_t rank_s = (uint32_t)__cvta_generic_to_shared(rank);
    using Scan = cub::BlockScan<uint32_t, kLongThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t W = kLongThreads / 32;
    const uint64_t n_items = min((uint64_t)*p.defer_n, p.defer_cap);
    unsigned count = 0, prunes = 0, verified = 0;
#if SSJB_LONG_DYN_SLICES
    // slices taken dynamically (p.defer_n[3] counts them out): their long-pair work varies by
    // orders of magnitude, so a static round-robin leaves SMs idle in the launch's tail
    __shared__ unsigned long long s_it;
    for (;;) {
        if (tid == 0) s_it = atomicAdd(p.defer_n + 3, 1ull);
        __syncthreads();
        const uint64_t it = s_it;  // read by all before the slice's first barrier below
        if (it >= n_items) break;
#else
    for (uint64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
#endif
        const uint32_t e = __ldg(p.defer + it);
        const uint4 d0 = __ldg(reinterpret_cast<const uint4*>(p.slices + e));
        const uint32_t m = d0.z;
        const uint32_t* r = p.tokens + (size_t)d0.y * 8;
        const uint64_t b0 = e ? __ldg(p.C_O + 2 * (size_t)e - 1) : 0;
        const uint64_t begin = max(b0, seg_lo), end = min((uint64_t)d0.x, seg_hi);
        const uint32_t lo = m ? (__ldg(r) & ~31u) : 0u;
        const uint32_t hi = m ? __ldg(r + m - 1) : 0u;
        const uint32_t nw = m ? ((hi - lo) >> 5) + 1 : 0u;
        const bool use_bm = m && nw <= BW && hi != 0xFFFFFFFFu;  // CTA-uniform
        const uint32_t nbits = nw * 32u;
        __syncthreads();  // previous slice's readers are done with the bitmap
        if (use_bm) {
            for (uint32_t w = tid; w <= nw; w += kLongThreads) bits[w] = 0;
            __syncthreads();
            for (uint32_t i = tid; i < m; i += kLongThreads) {
                const uint32_t d = __ldg(r + i) - lo;
                atomicOr(bits + (d >> 5), 1u << (d & 31));
            }
            __syncthreads();
            // rank: thread t owns words [t*per, t*per + per) of the nw words
            const uint32_t per = (nw + kLongThreads - 1) / kLongThreads;
            uint32_t tot = 0;
            for (uint32_t q = 0, w = tid * per; q < per && w < nw; ++q, ++w) tot += __popc(bits[w]);
            uint32_t x;
            Scan(scan_tmp).ExclusiveSum(tot, x);
            for (uint32_t q = 0, w = tid * per; q < per && w < nw; ++q, ++w) {
                rank[w] = x;
                x += __popc(bits[w]);
            }
            if (tid == 0) rank[nw] = m;  // the guard word (tokens above the range): all of r
            __syncthreads();
        }
        // the slice's long pairs, kLongThreads slots at a time: compacted into a shared list,
        // then one warp per listed pair
        for (uint64_t cb = begin; cb < end; cb += kLongThreads) {
            const uint64_t myslot = cb + tid;
            uint32_t n = 0, req = 0, pos = 0;
            bool want = false;
            if (myslot < end) {
                const uint32_t cand = __ldg(p.C + myslot);
                if (cand < p.n_sets) {  // out-of-range ids were flagged by the first pass
                    const uint2 sd = __ldg(p.sets + cand);
                    n = sd.y;
                    pos = sd.x;
                    req = dev_required_fast(p.pred, m, n);
                    want = n > kLongPair && req >= 1 && req <= min(m, n);
                }
            }
            if (tid == 0) *lcount = 0;
            __syncthreads();
            const unsigned wm = __ballot_sync(0xffffffffu, want);
            uint32_t wbase = 0;
            if (lane == 0 && wm) wbase = atomicAdd(lcount, (uint32_t)__popc(wm));
            wbase = __shfl_sync(0xffffffffu, wbase, 0);
            if (want)
                llist[wbase + __popc(wm & ((1u << lane) - 1u))] =
                    make_uint4((uint32_t)(myslot - cb), pos, n, req);
            __syncthreads();
            const uint32_t nl = *lcount;
            for (uint32_t li = warp; li < nl; li += W) {
                const uint4 ent = llist[li];
                const uint64_t slot = cb + ent.x;
                const uint32_t sn = ent.z, sreq = ent.w;
                const uint32_t* s = p.tokens + (size_t)ent.y * 8;
                bool met;
                uint32_t ov = 0;
                if (use_bm) {
#if SSJB_LONG_V2
                    // 32 * kLongPerLane candidate tokens per step (token j + u*32 + lane in
                    // lane `lane`, coalesced); per-lane counts summed with one warp reduction.
                    // Full steps run without per-token predicates: the next step's loads are
                    // issued (volatile, so they are not sunk past the exits) before this
                    // step's lookups, reading past |s| inside the padded CSR
                    // (SSJ_TOKEN_TAIL_PAD); the last, partial step masks tokens past |s| to
                    // 0xFFFFFFFF, which clamps onto the bitmap's zero guard word.
                    constexpr uint32_t U = kLongPerLane;
                    static_assert(2 * 32 * U <= SSJ_TOKEN_TAIL_PAD, "prefetch past the tail pad");
                    const uint32_t slack_r = m - sreq, slack_s = sn - sreq;
                    const uint32_t* sl = s + lane;
                    uint32_t bs;  // bitmap base, opaque: kept in a register, not rematerialised
                    asm volatile("mov.b32 %0, %1;" : "=r"(bs) : "r"(bits_s));
                    const uint32_t rs = bs + (rank_s - bits_s);
                    // one step at token j: lookups of cur, next step's loads into nxt, the
                    // verdict checks; the r-side position after the step's last token (rank +
                    // popc, verify.hpp:58) is computed by every lane for its own last token
                    // from the word its lookup already read, and taken from lane 31
                    uint32_t j = 0;
                    auto step = [&](uint32_t (&cur)[U], uint32_t (&nxt)[U], bool last) -> bool {
                        const uint32_t jn = j + 32 * U;
                        if (!last) {
#pragma unroll
                            for (uint32_t u = 0; u < U; ++u) nxt[u] = ldg_nc_v(sl + jn + u * 32);
                        }
                        uint32_t c = 0, il = 0;
#pragma unroll
                        for (uint32_t u = 0; u < U; ++u) {
                            const uint32_t e = min(cur[u] - lo, nbits);
                            const uint32_t w = lds_u32(bs + ((e >> 5) << 2));
                            c += (w >> (e & 31)) & 1u;
                            if (u == U - 1 && !last)
                                il = cur[u] < lo ? 0u
                                                 : lds_u32(rs + ((e >> 5) << 2)) +
                                                       __popc(w & ((2u << (e & 31)) - 1u));
                        }
                        ov += __reduce_add_sync(0xffffffffu, c);
                        if (last || jn == sn) {
                            met = ov >= sreq;
                            return true;
                        }
                        if (kOut != kOutResults && ov >= sreq) {
                            met = true;
                            return true;
                        }
                        const uint32_t i = __shfl_sync(0xffffffffu, il, 31);
                        if (ov < sreq && (i - ov > slack_r || jn - ov > slack_s)) return true;
                        j = jn;
                        return false;
                    };
                    uint32_t A[U], B[U];
#pragma unroll
                    for (uint32_t u = 0; u < U; ++u) A[u] = ldg_nc_v(sl + u * 32);
                    met = false;
                    bool done = false;
                    for (;;) {  // full steps, ping-pong buffers
                        if (j + 32 * U > sn) break;
                        if (step(A, B, false)) {
                            done = true;
                            break;
                        }
                        if (j + 32 * U > sn) {
#pragma unroll
                            for (uint32_t u = 0; u < U; ++u) A[u] = B[u];
                            break;
                        }
                        if (step(B, A, false)) {
                            done = true;
                            break;
                        }
                    }
                    if (!done) {  // j < |s| < j + 32U: the last, partial step
#pragma unroll
                        for (uint32_t u = 0; u < U; ++u)
                            if (j + u * 32 + lane >= sn) A[u] = 0xFFFFFFFFu;
                        step(A, B, true);
                    }
                    if (!met) ov = 0;
#else
                    // 32 * kLongPerLane candidate tokens per step (token j + u*32 + lane in
                    // lane `lane`, coalesced), the next step's in flight; tokens past |s| read
                    // as 0xFFFFFFFF and clamp onto the bitmap's zero word; per-lane counts are
                    // summed with one warp reduction
                    // the first step covers SSJB_LONG_FIRST tokens, the following ones
                    // 32 * kLongPerLane
                    constexpr uint32_t U = kLongPerLane;
                    const uint32_t slack_r = m - sreq, slack_s = sn - sreq;
                    uint32_t j = 0, width = SSJB_LONG_FIRST;
                    bool decided = false;
                    met = false;
                    uint32_t a[U];
                    const uint32_t* sl = s + lane;  // loads at sl + j + u*32: immediate offsets
#pragma unroll
                    for (uint32_t u = 0; u < U; ++u)
                        a[u] = u * 32 < width && u * 32 + lane < sn ? __ldg(sl + u * 32) : 0xFFFFFFFFu;
                    for (;;) {
                        const uint32_t jn = j + width;  // next step: [jn, jn + 32 * U)
                        const int rem = (int)sn - (int)(jn + lane);  // tokens left for this lane
                        const uint32_t* ps = sl + jn;
                        uint32_t nx[U];
#pragma unroll
                        for (uint32_t u = 0; u < U; ++u)
                            nx[u] = (int)(u * 32) < rem ? __ldg(ps + u * 32) : 0xFFFFFFFFu;
                        uint32_t c = 0;
#pragma unroll
                        for (uint32_t u = 0; u < U; ++u) {
                            const uint32_t e = min(a[u] - lo, nbits);
                            c += (lds_u32(bits_s + ((e >> 5) << 2)) >> (e & 31)) & 1u;
                        }
                        ov += __reduce_add_sync(0xffffffffu, c);
                        j = jn;
                        if (j >= sn) break;
                        if (kOut != kOutResults && ov >= sreq) {
                            met = true;
                            decided = true;
                            break;
                        }
                        if (ov < sreq) {
                            const uint32_t tl = __shfl_sync(0xffffffffu, width == 32 * U ? a[U - 1] : a[0], 31);
                            const uint32_t dl = tl - lo;
                            uint32_t i;
                            if (tl < lo) i = 0;
                            else if (dl >= nbits) i = m;
                            else i = lds_u32(rank_s + ((dl >> 5) << 2)) +
                                     __popc(lds_u32(bits_s + ((dl >> 5) << 2)) & ((2u << (dl & 31)) - 1u));
                            if (i - ov > slack_r || j - ov > slack_s) {
                                decided = true;
                                break;
                            }
                        }
#pragma unroll
                        for (uint32_t u = 0; u < U; ++u) a[u] = nx[u];
                        width = 32 * U;
                    }
                    if (!decided) met = ov >= sreq;
                    if (!met) ov = 0;
#endif
                } else {
                    met = path_pair<32, kOut == kOutResults>(r, m, s, sn, sreq, lane, 0xffffffffu, &ov);
                }
                if (lane == 0) {
                    if (kOut == kOutFlags) p.flags[slot] = met ? 1 : 0;
                    count += met;
                    if (kStats) {
                        ++verified;
                        prunes += (!met && (m + sn) > 0);
                    }
                }
                if (kOut == kOutResults) warp_append(p, met && lane == 0, slot, ov);
            }
            __syncthreads();  // list consumed
        }
    }
    acc_add(p.acc, 0, count);
    if (kStats) {
        acc_add(p.acc, 2, verified);
        acc_add(p.acc, 3, prunes);
    }
}

// ---------------------------------------------------------------------------------------
// Diagnostic: streaming read bandwidth of a device buffer (16-byte loads, grid-stride),
// used by the benchmark for the L2-resident and HBM roofline denominators.
__global__ void read_bw_kernel(const uint4* __restrict__ a, uint64_t n, uint32_t reps,
                               unsigned* __restrict__ sink) {
    uint32_t x = 0;
    for (uint32_t r = 0; r < reps; ++r) {
        for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
             i += (uint64_t)gridDim.x * blockDim.x) {
            const uint4 v = __ldcg(a + i);
            x ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    }
    if (x == 0x9E3779B9u) sink[0] = x;  // keeps the loads alive
}

// ---------------------------------------------------------------------------------------
// H2 on the GPU (pipeline.hpp:79-92 decode_pairs): qualifying slot -> (max(orig), min(orig))
// original input ids, packed as a 64-bit key (r_id << 32 | s_id) so that a radix sort gives
// write_pairs order (report.hpp:39-42).
__global__ void pairs_kernel(const KParams p, const uint32_t* __restrict__ oid, uint64_t n,
                             unsigned long long* __restrict__ keys) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t slot = p.res_slots[k];
    const uint32_t e = upper_bound_ends(p.C_O, 0, p.n_slices, slot);
    const uint32_t a = __ldg(oid + __ldg(p.C_O + 2 * (size_t)e));
    const uint32_t b = __ldg(oid + __ldg(p.C + slot));
    keys[k] = ((unsigned long long)max(a, b) << 32) | min(a, b);
}

// ---------------------------------------------------------------------------------------
// Instrumentation: algorithmic bytes under the reference loop
// verify.hpp:56-69, replayed exactly per pair.
__global__ void bytes_kernel(const KParams p, unsigned long long* out) {
    const uint64_t idx = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long b = 0;
    if (idx < p.n_slices) {
        const uint32_t probe = p.C_O[2 * idx];
        const uint32_t m = probe < p.n_sets ? p.sets[probe].y : 0;
        b += 8 + 8 + 4ull * m;
    }
    if (idx < p.nC) {
        const uint32_t e = upper_bound_ends(p.C_O, 0, p.n_slices, idx);
        const uint32_t cand = p.C[idx];
        if (e < p.n_slices && cand < p.n_sets) {
            const uint32_t probe = p.C_O[2 * (size_t)e];
            if (probe < p.n_sets) {
                const uint2 rd = p.sets[probe], sd = p.sets[cand];
                const uint32_t* r = p.tokens + (size_t)rd.x * 8;
                const uint32_t* s = p.tokens + (size_t)sd.x * 8;
                const uint32_t m = rd.y, n = sd.y;
                const uint64_t req = dev_required(p.pred, m, n);
                uint64_t ov = 0;
                uint32_t i = 0, j = 0;
                while (i < m && j < n) {
                    if (ov >= req) break;
                    if (ov + min(m - i, n - j) < req) break;
                    if (r[i] == s[j]) {
                        ++ov; ++i; ++j;
                    } else if (r[i] < s[j]) {
                        ++i;
                    } else {
                        ++j;
                    }
                }
                const uint32_t touched = min(j + 1, n);
                b += 4 + 8 + 1 + 4ull * touched;
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) b += __shfl_xor_sync(0xffffffffu, b, off);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(out, b);
}

template <int G, int kOut>
cudaError_t launch_path_g(const KParams& p, uint32_t grid, uint32_t rcap, size_t smem,
                          cudaStream_t st) {
    auto k = path_kernel<G, kOut>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<grid, 256, smem, st>>>(p, rcap);
    return cudaGetLastError();
}

template <int G>
cudaError_t launch_path_out(const KParams& p, int out, uint32_t grid, uint32_t rcap, size_t smem,
                            cudaStream_t st) {
    switch (out) {
        case kOutFlags: return launch_path_g<G, kOutFlags>(p, grid, rcap, smem, st);
        case kOutResults: return launch_path_g<G, kOutResults>(p, grid, rcap, smem, st);
        default: return launch_path_g<G, kOutCount>(p, grid, rcap, smem, st);
    }
}

uint32_t slice_grid(uint32_t n_slices) {
    // One CTA per probe slice (the paper's launch shape), capped; CTAs grid-stride.
    const uint32_t cap = 148u * 64u;
    return n_slices < cap ? (n_slices ? n_slices : 1) : cap;
}

constexpr uint32_t kSliceRCap = 12288;  // tokens staged per CTA in strategies B/C (48 KB)

}  // namespace

cudaError_t launch_prep(const KParams& p, cudaStream_t st, int* launches) {
    if (p.n_slices) {
        prep_kernel<<<(uint32_t)((p.n_slices + kPrepThreads - 1) / kPrepThreads), kPrepThreads, 0, st>>>(p);
    } else {
        prep_empty_kernel<<<1, 32, 0, st>>>(p);
    }
    int n = 1;
    if (p.slices && p.bm_cap && p.n_slices) {
        const uint64_t warps = p.n_slices < 148ull * 64 ? p.n_slices : 148ull * 64;
        bitmap_kernel<<<(uint32_t)((warps * 32 + 255) / 256), 256, 0, st>>>(p);
        ++n;
    }
    if (launches) *launches = n;
    return cudaGetLastError();
}

__global__ void build_heads_kernel(const uint32_t* __restrict__ tokens, const uint2* __restrict__ sets,
                                   uint32_t n_sets, uint4* __restrict__ heads,
                                   unsigned* __restrict__ max_token) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_sets) return;
    const uint2 sd = sets[i];
    const uint32_t* t = tokens + (size_t)sd.x * 8;
    uint32_t v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t info = q < 4 ? (sd.x >> (8 * q)) & 0xFFu : (sd.y >> (8 * (q - 4))) & 0xFFu;
        const uint32_t tok = (uint32_t)q < sd.y ? (t[q] & kHeadTokenMask) : kHeadTokenMask;
        v[q] = tok | (info << 24);
    }
    heads[2 * (size_t)i] = make_uint4(v[0], v[1], v[2], v[3]);
    heads[2 * (size_t)i + 1] = make_uint4(v[4], v[5], v[6], v[7]);
    if (sd.y) atomicMax(max_token, t[sd.y - 1]);  // sets are sorted: the last token is the largest
}

int sm_count() {
    static int cached[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cached[dev]) {
        int n = 0;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = n > 0 ? n : 148;
    }
    return cached[dev];
}

// cudaFuncSetAttribute applies on the current device: set the dynamic shared memory limit
// once per (kernel, device); `done` holds one bit per device id.
template <typename K>
cudaError_t ensure_smem_attr(K kernel, int bytes, std::atomic<uint64_t>& done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
    return e;
}

template <int kOut, bool kStats>
cudaError_t launch_tiles_t(const KParams& p, uint32_t tile_begin, uint32_t tile_end,
                           cudaStream_t st, cudaStream_t aux, cudaEvent_t fork, cudaEvent_t join) {
    (void)tile_begin;
    (void)tile_end;
    const int sms = sm_count();
    // short slices (a map per run or two): three map buffers, so the next map is built while
    // the current one is in use
    const double avg = (double)p.nC / (double)max(p.n_slices, 1u);
    const uint32_t mb = avg < SSJB_RUN_MB3_BELOW ? 3u : 2u;
    auto rk = p.heads ? (mb == 3 ? run_kernel<kOut, kStats, true, 3> : run_kernel<kOut, kStats, true, 2>)
                      : (mb == 3 ? run_kernel<kOut, kStats, false, 3> : run_kernel<kOut, kStats, false, 2>);
    const size_t smem = run_smem_bytes(mb);
    static std::atomic<uint64_t> attr[4];  // per instantiation and device
    cudaError_t err = ensure_smem_attr(rk, (int)smem, attr[(p.heads ? 1 : 0) + 2 * (mb - 2)]);
    if (err != cudaSuccess) return err;
    cudaStream_t ts = st;
    if (aux && fork && join) {
        if ((err = cudaEventRecord(fork, st)) != cudaSuccess) return err;
        if ((err = cudaStreamWaitEvent(aux, fork, 0)) != cudaSuccess) return err;
        ts = aux;
    }
    if (p.heads)
        warp_tile_kernel<kOut, kStats, true><<<sms * kTileMinBlocks, kThreadsA, 0, ts>>>(p);
    else
        warp_tile_kernel<kOut, kStats, false><<<sms * kTileMinBlocks, kThreadsA, 0, ts>>>(p);
    rk<<<sms * kRunMinBlocks, kRunThreads, smem, st>>>(p);
    if (ts != st) {
        if ((err = cudaEventRecord(join, ts)) != cudaSuccess) return err;
        if ((err = cudaStreamWaitEvent(st, join, 0)) != cudaSuccess) return err;
    }
    return cudaGetLastError();
}

cudaError_t launch_tiles(const KParams& p, int out, bool stats, uint32_t tile_begin,
                         uint32_t tile_end, cudaStream_t st, cudaStream_t aux, cudaEvent_t fork,
                         cudaEvent_t join) {
    if (tile_end <= tile_begin) return cudaSuccess;
    switch (out * 2 + (stats ? 1 : 0)) {
        case 0: return launch_tiles_t<kOutCount, false>(p, tile_begin, tile_end, st, aux, fork, join);
        case 1: return launch_tiles_t<kOutCount, true>(p, tile_begin, tile_end, st, aux, fork, join);
        case 2: return launch_tiles_t<kOutFlags, false>(p, tile_begin, tile_end, st, aux, fork, join);
        case 3: return launch_tiles_t<kOutFlags, true>(p, tile_begin, tile_end, st, aux, fork, join);
        case 4: return launch_tiles_t<kOutResults, false>(p, tile_begin, tile_end, st, aux, fork, join);
        default: return launch_tiles_t<kOutResults, true>(p, tile_begin, tile_end, st, aux, fork, join);
    }
}

template <int kOut, bool kStats>
cudaError_t launch_long_t(const KParams& p, uint64_t seg_lo, uint64_t seg_hi, cudaStream_t st) {
    auto k = long_slice_kernel<kOut, kStats>;
    static std::atomic<uint64_t> attr;  // per device
    cudaError_t err = ensure_smem_attr(k, (int)kLongSmemBytes, attr);
    if (err != cudaSuccess) return err;
    const uint32_t W = p.long_words ? p.long_words : kMaxBitmapWords;
    const size_t smem = (size_t)(2 * W + 8) * 4 + kLongThreads * 16 + 16;
    k<<<sm_count() * (1024 / kLongThreads) * 2, kLongThreads, smem, st>>>(p, seg_lo, seg_hi);
    return cudaGetLastError();
}

cudaError_t launch_long(const KParams& p, int out, bool stats, uint32_t tile_begin,
                        uint32_t tile_end, cudaStream_t st) {
    if (!p.defer) return cudaSuccess;
    const uint64_t lo = (uint64_t)tile_begin * kTile;
    const uint64_t hi = min((uint64_t)tile_end * kTile, p.nC);
    switch (out * 2 + (stats ? 1 : 0)) {
        case 0: return launch_long_t<kOutCount, false>(p, lo, hi, st);
        case 1: return launch_long_t<kOutCount, true>(p, lo, hi, st);
        case 2: return launch_long_t<kOutFlags, false>(p, lo, hi, st);
        case 3: return launch_long_t<kOutFlags, true>(p, lo, hi, st);
        case 4: return launch_long_t<kOutResults, false>(p, lo, hi, st);
        default: return launch_long_t<kOutResults, true>(p, lo, hi, st);
    }
}

cudaError_t launch_block(const KParams& p, int out, bool stats, uint32_t threads,
                         cudaStream_t st) {
    threads = threads < 32 ? 32 : (threads > 1024 ? 1024 : threads);
    const uint32_t grid = slice_grid(p.n_slices);
    const size_t smem = kSliceRCap * sizeof(uint32_t);
    const uint32_t rcap = kSliceRCap;
#define SSJB_LAUNCH_B(O, S)                                                                   \
    do {                                                                                      \
        auto k = block_kernel<O, S>;                                                          \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
        k<<<grid, threads, smem, st>>>(p, rcap);                                              \
    } while (0)
    switch (out * 2 + (stats ? 1 : 0)) {
        case 0: SSJB_LAUNCH_B(kOutCount, false); break;
        case 1: SSJB_LAUNCH_B(kOutCount, true); break;
        case 2: SSJB_LAUNCH_B(kOutFlags, false); break;
        case 3: SSJB_LAUNCH_B(kOutFlags, true); break;
        case 4: SSJB_LAUNCH_B(kOutResults, false); break;
        default: SSJB_LAUNCH_B(kOutResults, true); break;
    }
#undef SSJB_LAUNCH_B
    return cudaGetLastError();
}

cudaError_t launch_path(const KParams& p, int out, uint32_t group, cudaStream_t st) {
    const uint32_t grid = slice_grid(p.n_slices);
    const size_t smem = kSliceRCap * sizeof(uint32_t);
    const uint32_t rcap = kSliceRCap;
    if (group >= 32) return launch_path_out<32>(p, out, grid, rcap, smem, st);
    if (group >= 16) return launch_path_out<16>(p, out, grid, rcap, smem, st);
    if (group >= 8) return launch_path_out<8>(p, out, grid, rcap, smem, st);
    if (group >= 4) return launch_path_out<4>(p, out, grid, rcap, smem, st);
    if (group >= 2) return launch_path_out<2>(p, out, grid, rcap, smem, st);
    return launch_path_out<1>(p, out, grid, rcap, smem, st);
}

cudaError_t launch_read_bw(const void* buf, uint64_t bytes, uint32_t reps, unsigned* sink,
                           cudaStream_t st) {
    read_bw_kernel<<<148 * 8, 512, 0, st>>>(static_cast<const uint4*>(buf), bytes / 16, reps, sink);
    return cudaGetLastError();
}

cudaError_t launch_build_heads(const uint32_t* tokens, const uint2* sets, uint32_t n_sets,
                               uint4* heads, unsigned* max_token, cudaStream_t st) {
    if (!n_sets) return cudaSuccess;
    build_heads_kernel<<<(n_sets + 255) / 256, 256, 0, st>>>(tokens, sets, n_sets, heads, max_token);
    return cudaGetLastError();
}

cudaError_t launch_pairs(const KParams& p, const uint32_t* oid, uint64_t n,
                         unsigned long long* keys, cudaStream_t st) {
    if (!n) return cudaSuccess;
    pairs_kernel<<<(uint32_t)((n + 255) / 256), 256, 0, st>>>(p, oid, n, keys);
    return cudaGetLastError();
}

cudaError_t launch_bytes(const KParams& p, unsigned long long* d_bytes, cudaStream_t st) {
    const uint64_t work = p.nC > p.n_slices ? p.nC : p.n_slices;
    const uint32_t threads = 256;
    const uint64_t grid = (work + threads - 1) / threads;
    bytes_kernel<<<(uint32_t)(grid ? grid : 1), threads, 0, st>>>(p, d_bytes);
    return cudaGetLastError();
}

}  // namespace ssjb
