// gpu_filter.cu -- device candidate generation (see gpu_filter.cuh for the algorithm).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gpu_filter.cuh"

namespace ssjb {

namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ uint64_t ceil_div128(u128 a, u128 b) { return (uint64_t)((a + b - 1) / b); }

// similarity.hpp:135-164 size_bounds(...).min, raised to 1 when zero (:162).
__device__ __forceinline__ uint64_t dev_size_lower_bound(const PredDev& p, uint64_t r) {
    uint64_t lo;
    switch (p.fn) {
        case kFnJaccard: lo = ceil_div128((u128)p.num * r, p.den); break;
        case kFnCosine: lo = ceil_div128((u128)p.num * p.num * r, (u128)p.den * p.den); break;
        case kFnDice: lo = ceil_div128((u128)p.num * r, 2 * p.den - p.num); break;
        default: lo = p.ovt; break;
    }
    return lo == 0 ? 1 : lo;
}

// filters.hpp:148-159 prefix_lengths: {probe, index}.
__device__ __forceinline__ uint2 dev_prefix_lengths(const PredDev& p, uint32_t size) {
    auto clamp = [size](uint64_t len) -> uint32_t {
        if (len < 1) return 1;
        return (uint32_t)(len < size ? len : size);
    };
    const uint64_t minsize = dev_size_lower_bound(p, size);
    const uint32_t probe = clamp(minsize >= size ? 1 : size - minsize + 1);
    const uint64_t self = dev_required(p, size, size);
    const uint32_t index = clamp(self >= size ? 1 : size - self + 1);
    return make_uint2(probe, index);
}

__device__ __forceinline__ uint32_t set_size(const FilterIndex& ix, uint32_t s) {
    return __ldg(&ix.sets[s].y);
}
__device__ __forceinline__ const uint32_t* set_tokens(const FilterIndex& ix, uint32_t s) {
    return ix.tokens + (size_t)__ldg(&ix.sets[s].x) * 8;
}

// First set whose size is >= minsize (sets are size-ascending).
__device__ __forceinline__ uint32_t first_set_of_size(const FilterIndex& ix, uint64_t minsize) {
    uint32_t lo = 0, hi = ix.n_sets;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if ((uint64_t)set_size(ix, mid) < minsize) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// First posting in [lo, hi) with set >= key.
__device__ __forceinline__ uint32_t posting_lower_bound(const FilterIndex& ix, uint32_t lo,
                                                        uint32_t hi, uint32_t key) {
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(&ix.post[mid].x) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---- index build -------------------------------------------------------------------------
__global__ void ilen_kernel(const FilterIndex ix, uint32_t* ilen, uint32_t* max_token) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ix.n_sets) return;
    const uint32_t n = set_size(ix, s);
    ilen[s] = n ? dev_prefix_lengths(ix.pred, n).y : 0u;
    if (n) atomicMax(max_token, __ldg(set_tokens(ix, s) + n - 1));
}

__global__ void entries_kernel(const FilterIndex ix, const uint32_t* ilen, const uint32_t* off,
                               uint32_t* keys, unsigned long long* vals, uint32_t* count) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= ix.n_sets) return;
    const uint32_t* r = set_tokens(ix, s);
    const uint32_t base = off[s];
    for (uint32_t q = 0; q < ilen[s]; ++q) {
        const uint32_t t = __ldg(r + q);
        keys[base + q] = t;
        vals[base + q] = ((unsigned long long)s << 32) | q;
        atomicAdd(count + t, 1u);
    }
}

__global__ void unpack_kernel(const unsigned long long* vals, uint64_t n, uint2* post) {
    const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) post[k] = make_uint2((uint32_t)(vals[k] >> 32), (uint32_t)vals[k]);
}

// ---- probing -------------------------------------------------------------------------------
// Warp per probe. Lanes take prefix positions p (strided); range of token r[p]'s postings
// usable by probe i: [first set >= S_min, first set >= i).
__global__ void bounds_kernel(const FilterIndex ix, uint32_t a, uint32_t b,
                              unsigned long long* bound) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = w; k < (uint64_t)(b - a); k += nw) {
        const uint32_t i = a + (uint32_t)k;
        const uint32_t m = set_size(ix, i);
        unsigned long long tot = 0;
        if (m) {
            const uint32_t P = dev_prefix_lengths(ix.pred, m).x;
            const uint32_t smin = first_set_of_size(ix, dev_size_lower_bound(ix.pred, m));
            const uint32_t* r = set_tokens(ix, i);
            for (uint32_t p = lane; p < P; p += 32) {
                const uint32_t t = __ldg(r + p);
                if (t >= ix.universe) continue;
                const uint32_t h0 = __ldg(ix.head + t), h1 = __ldg(ix.head + t + 1);
                const uint32_t lo = posting_lower_bound(ix, h0, h1, smin);
                const uint32_t hi = posting_lower_bound(ix, lo, h1, i);
                tot += hi - lo;
            }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, off);
        if (lane == 0) bound[k] = tot;
    }
}

// Warp per probe: for p = 0..P-1 the warp sweeps the range of r[p]'s postings 32 at a time;
// a lane keeps its set s unless s was already reached at an earlier prefix position (one of
// s's index-prefix tokens below r[p] is in r) and, for PPJoin, unless the positional filter
// rejects it at this first match. Kept sets are appended in order (ballot compaction).
// The posting ranges of 32 prefix positions are found at once (one binary-search pair per
// lane), r's first kGenRStage tokens are staged in the warp's shared memory for the dedup
// searches, and s's first 8 tokens come from its packed head record in one 256-bit load.
constexpr uint32_t kGenThreads = 256;
constexpr uint32_t kGenRStage = 256;
// Per-warp membership filter over the probe prefix r[0..P): a token of s below r[p] is in
// r[0..p) iff it is in r at all (r is sorted), so one filter per probe serves every p.
// Exact mode (the prefix's token range fits kGenFilterWords - 1 words): bit v - lo, tokens
// outside the range clamp onto a zero guard word -- a hit is a member. Otherwise a Bloom
// filter (hashed bits) screens the exact binary search.
constexpr uint32_t kGenFilterBits = 13;
constexpr uint32_t kGenFilterWords = (1u << kGenFilterBits) / 32;

__device__ __forceinline__ uint32_t bloom_hash(uint32_t v) {
    return (v * 0x9E3779B1u) >> (32 - kGenFilterBits);
}
template <bool kExact>
__device__ __forceinline__ bool filter_hit(const uint32_t* __restrict__ bm, uint32_t v,
                                           uint32_t lo, uint32_t nbits) {
    const uint32_t h = kExact ? min(v - lo, nbits) : bloom_hash(v);
    return (bm[h >> 5] >> (h & 31)) & 1u;
}

__device__ __forceinline__ void ld8(const uint32_t* __restrict__ s, uint32_t t[8]) {
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(t[0]), "=r"(t[1]), "=r"(t[2]), "=r"(t[3]), "=r"(t[4]), "=r"(t[5]),
                   "=r"(t[6]), "=r"(t[7])
                 : "l"(s));
}

// is v one of r[lo..p)? r staged in rs (first kGenRStage tokens) or global. Returns the
// lower-bound position (>= lo) through *pos.
__device__ __forceinline__ bool in_r(const uint32_t* __restrict__ rs,
                                     const uint32_t* __restrict__ r, uint32_t lo, uint32_t p,
                                     uint32_t v, uint32_t* pos) {
    uint32_t l = lo, h = p;
    while (l < h) {
        const uint32_t mid = (l + h) >> 1;
        const uint32_t x = mid < kGenRStage ? rs[mid] : __ldg(r + mid);
        if (x < v) l = mid + 1;
        else h = mid;
    }
    *pos = l;
    return l < p && (l < kGenRStage ? rs[l] : __ldg(r + l)) == v;
}

#ifndef SSJB_GEN_POS_FIRST
#define SSJB_GEN_POS_FIRST 1
#endif
// Keep posting q of probe r (size m) at prefix position p? *s_out = the posting's set.
// Duplicate iff an index-prefix token of s below r[p] is in r (then it is in r[0..p), where s
// was already emitted); PPJoin also applies the positional filter at this first match.
template <bool kExact>
__device__ __forceinline__ bool candidate_keep(const FilterIndex& ix, const uint32_t* __restrict__ rs,
                                               const uint32_t* __restrict__ r,
                                               const uint32_t* __restrict__ bm, uint32_t flo,
                                               uint32_t fbits, uint32_t m, uint32_t p,
                                               uint32_t q, bool positional, uint32_t* s_out) {
    const uint2 pe = __ldg(&ix.post[q]);
    const uint32_t s = pe.x;
    *s_out = s;
    bool keep = true;
    // member of r: exact filter hit, or Bloom hit confirmed by the binary search
    auto member = [&](uint32_t v) {
        uint32_t pos;
        return filter_hit<kExact>(bm, v, flo, fbits) && (kExact || in_r(rs, r, 0, p, v, &pos));
    };
    uint32_t ns = 0;  // |s| when the head record was read
#if SSJB_GEN_POS_FIRST
    // PPJoin: the positional filter (filters.hpp:174-181, current_overlap = 1,
    // joiners.hpp:94) first -- keep = first occurrence AND positional, so the order of the two
    // tests does not change the stream, and the candidates it rejects skip the dedup
    if (positional) {
        ns = set_size(ix, s);
        const uint64_t a = m - p - 1, b = ns - pe.y - 1;
        if (1 + (a < b ? a : b) < dev_required_fast(ix.pred, m, ns)) return false;
    }
#endif
    if (p && pe.y) {  // pe.y = position of r[p] in s: the tokens before it are < r[p]
        if (ix.heads) {
            uint32_t hv[8];
            ld8(reinterpret_cast<const uint32_t*>(ix.heads + 2 * (size_t)s), hv);
            // pos8 / |s| from the record's top bytes (build_heads_kernel): no descriptor load
            const uint32_t pos8 = __byte_perm(__byte_perm(hv[0], hv[1], 0x0073), __byte_perm(hv[2], hv[3], 0x0073), 0x5410);
            ns = __byte_perm(__byte_perm(hv[4], hv[5], 0x0073), __byte_perm(hv[6], hv[7], 0x0073), 0x5410);
            // 8 tokens at a time: all lookups branch-free, the hits below the position decide
            // (Bloom hits are confirmed by the exact search); tokens 8.. come from the CSR by
            // 32-byte loads (reads past |s| stay inside the padded token array)
            auto dup8 = [&](const uint32_t (&t)[8], uint32_t lim, uint32_t mask) -> bool {
                uint32_t hit = 0;
#pragma unroll
                for (uint32_t u = 0; u < 8; ++u)
                    hit |= (uint32_t)filter_hit<kExact>(bm, t[u] & mask, flo, fbits) << u;
                hit &= lim >= 8 ? 0xFFu : (1u << lim) - 1u;
                if (kExact || !hit) return hit != 0;
                bool d = false;
#pragma unroll
                for (uint32_t u = 0; u < 8; ++u) {
                    uint32_t pos;
                    if ((hit >> u & 1u) && !d && in_r(rs, r, 0, p, t[u] & mask, &pos)) d = true;
                }
                return d;
            };
            keep = !dup8(hv, pe.y, kHeadTokenMask);
            if (keep && pe.y > 8) {
                const uint32_t* st = ix.tokens + (size_t)pos8 * 8;
                for (uint32_t u0 = 8; u0 < pe.y; u0 += 8) {
                    uint32_t tv[8];
                    ld8(st + u0, tv);
                    if (dup8(tv, pe.y - u0, 0xFFFFFFFFu)) {
                        keep = false;
                        break;
                    }
                }
            }
        } else {
            const uint32_t* st = set_tokens(ix, s);
            for (uint32_t u = 0; u < pe.y; ++u) {
                if (member(__ldg(st + u))) {
                    keep = false;
                    break;
                }
            }
        }
    }
    if (!SSJB_GEN_POS_FIRST && keep && positional) {
        // filters.hpp:174-181 positional_filter with current_overlap = 1 (joiners.hpp:94)
        if (!ns) ns = set_size(ix, s);  // sets in an index are never empty
        const uint64_t a = m - p - 1, b = ns - pe.y - 1;
        keep = 1 + (a < b ? a : b) >= dev_required_fast(ix.pred, m, ns);
    }
    return keep;
}

#ifndef SSJB_GEN_EXACT
#define SSJB_GEN_EXACT 1
#endif
#ifndef SSJB_GEN_DYN
#define SSJB_GEN_DYN 1
#endif
#ifndef SSJB_GEN_MINB
#define SSJB_GEN_MINB 4
#endif
__global__ void __launch_bounds__(kGenThreads, SSJB_GEN_MINB)
    generate_kernel(const FilterIndex ix, uint32_t a, uint32_t b, const unsigned long long* base,
                    unsigned long long base0, uint32_t* C, unsigned long long* count,
                    uint32_t* flag) {
    __shared__ uint32_t rstage[kGenThreads / 32][kGenRStage];
    __shared__ uint32_t bloom[kGenThreads / 32][kGenFilterWords];
    const uint32_t lane = threadIdx.x & 31;
    uint32_t* const rs = rstage[threadIdx.x >> 5];
    uint32_t* const bm = bloom[threadIdx.x >> 5];
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const bool positional = ix.algorithm == 1;
#if SSJB_GEN_DYN
    // dynamic schedule, largest probes first (sizes ascend with the set id): a warp takes the
    // next probe when it is done, so a few heavy probes do not make the launch's tail
    (void)w;
    (void)nw;
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(ix.work, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= (unsigned long long)(b - a)) break;
        const uint64_t k = (uint64_t)(b - a) - 1 - t;
#else
    for (uint64_t k = w; k < (uint64_t)(b - a); k += nw) {
#endif
        const uint32_t i = a + (uint32_t)k;
        const uint32_t m = set_size(ix, i);
        uint32_t n_out = 0;
        if (m) {
            const uint32_t P = dev_prefix_lengths(ix.pred, m).x;
            const uint32_t smin = first_set_of_size(ix, dev_size_lower_bound(ix.pred, m));
            const uint32_t* r = set_tokens(ix, i);
            // the prefix's token range decides the filter mode (warp-uniform)
            const uint32_t flo = __ldg(r) & ~31u, fhi = __ldg(r + P - 1);
            const uint32_t fnw = ((fhi - flo) >> 5) + 1;
            const bool exact = SSJB_GEN_EXACT && fnw < kGenFilterWords;
            const uint32_t fbits = fnw * 32u;
            __syncwarp();
            for (uint32_t u = lane; u < (exact ? fnw + 1 : kGenFilterWords); u += 32) bm[u] = 0;
            __syncwarp();
            for (uint32_t u = lane; u < P; u += 32) {
                const uint32_t v = __ldg(r + u);
                if (u < kGenRStage) rs[u] = v;
                const uint32_t h = exact ? v - flo : bloom_hash(v);
                atomicOr(&bm[h >> 5], 1u << (h & 31));
            }
            __syncwarp();
            uint32_t* out = C + (base[k] - base0);
            for (uint32_t p0 = 0; p0 < P; p0 += 32) {
                // ranges of prefix positions p0 + lane
                uint32_t my_lo = 0, my_hi = 0;
                if (p0 + lane < P) {
                    const uint32_t t = __ldg(r + p0 + lane);
                    if (t < ix.universe) {
                        const uint32_t h0 = __ldg(ix.head + t), h1 = __ldg(ix.head + t + 1);
                        my_lo = posting_lower_bound(ix, h0, h1, smin);
                        my_hi = posting_lower_bound(ix, my_lo, h1, i);
                    }
                }
                const uint32_t pend = min(32u, P - p0);
                for (uint32_t pl = 0; pl < pend; ++pl) {
                    const uint32_t lo = __shfl_sync(0xffffffffu, my_lo, pl);
                    const uint32_t hi = __shfl_sync(0xffffffffu, my_hi, pl);
                    for (uint32_t q0 = lo; q0 < hi; q0 += 32) {
                        const uint32_t q = q0 + lane;
                        bool keep = false;
                        uint32_t s = 0;
                        if (q < hi)
                            keep = exact ? candidate_keep<true>(ix, rs, r, bm, flo, fbits, m, p0 + pl, q, positional, &s)
                                         : candidate_keep<false>(ix, rs, r, bm, flo, fbits, m, p0 + pl, q, positional, &s);
                        const unsigned km = __ballot_sync(0xffffffffu, keep);
                        if (keep) out[n_out + __popc(km & ((1u << lane) - 1u))] = s;
                        n_out += __popc(km);
                    }
                }
            }
        }
        if (lane == 0) {
            count[k] = n_out;
            flag[k] = n_out ? 1u : 0u;
        }
    }
}

__global__ void compact_kernel(uint32_t a, uint32_t b, const unsigned long long* base,
                               unsigned long long base0, const uint32_t* C,
                               const unsigned long long* count,
                               const unsigned long long* out_base, const uint32_t* slot,
                               uint32_t* outC, uint32_t* outCO) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = w; k < (uint64_t)(b - a); k += nw) {
        const uint32_t n = (uint32_t)count[k];
        if (!n) continue;
        const uint32_t* src = C + (base[k] - base0);
        uint32_t* dst = outC + out_base[k];
        uint32_t q = lane;
        for (; q + 96 < n; q += 128) {  // 4 loads in flight per lane
            const uint32_t v0 = src[q], v1 = src[q + 32], v2 = src[q + 64], v3 = src[q + 96];
            dst[q] = v0;
            dst[q + 32] = v1;
            dst[q + 64] = v2;
            dst[q + 96] = v3;
        }
        for (; q < n; q += 32) dst[q] = src[q];
        if (lane == 0) {
            outCO[2 * (size_t)slot[k]] = a + (uint32_t)k;
            outCO[2 * (size_t)slot[k] + 1] = (uint32_t)(out_base[k] + n);
        }
    }
}

uint32_t warps_grid(uint64_t items) {
    const uint64_t warps = items < 148ull * 64 ? (items ? items : 1) : 148ull * 64;
    return (uint32_t)((warps * 32 + 255) / 256);
}

}  // namespace

cudaError_t filter_index_build(FilterIndex* ix, const uint32_t* d_tokens, const uint2* d_sets,
                               uint32_t n_sets, const PredDev& pred, int algorithm,
                               cudaStream_t st) {
    filter_index_free(ix);
    ix->tokens = d_tokens;
    ix->sets = d_sets;
    ix->n_sets = n_sets;
    ix->pred = pred;
    ix->algorithm = algorithm;
    ix->universe = 0;
    if (cudaMalloc(&ix->work, sizeof(unsigned long long)) != cudaSuccess) return cudaErrorMemoryAllocation;
    if (!n_sets) return cudaSuccess;
    uint32_t *ilen = nullptr, *off = nullptr, *mx = nullptr, *keys = nullptr, *keys2 = nullptr,
             *count = nullptr;
    unsigned long long *vals = nullptr, *vals2 = nullptr;
    void* tmp = nullptr;
    cudaError_t err = cudaSuccess;
    auto ck = [&](cudaError_t e) {
        if (err == cudaSuccess && e != cudaSuccess) err = e;
        return err == cudaSuccess;
    };
    const uint32_t g = (n_sets + 255) / 256;
    if (!ck(cudaMalloc(&ilen, (size_t)n_sets * 4)) || !ck(cudaMalloc(&off, ((size_t)n_sets + 1) * 4)) ||
        !ck(cudaMalloc(&mx, 4)) || !ck(cudaMemsetAsync(mx, 0, 4, st)))
        goto done;
    ilen_kernel<<<g, 256, 0, st>>>(*ix, ilen, mx);
    if (!ck(cudaGetLastError())) goto done;
    {
        size_t tb = 0;
        if (!ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, ilen, off, (int)n_sets, st)) ||
            !ck(cudaMalloc(&tmp, tb)) ||
            !ck(cub::DeviceScan::ExclusiveSum(tmp, tb, ilen, off, (int)n_sets, st)))
            goto done;
        cudaFree(tmp);
        tmp = nullptr;
        uint32_t last_off = 0, last_len = 0, max_tok = 0;
        if (!ck(cudaMemcpyAsync(&last_off, off + n_sets - 1, 4, cudaMemcpyDeviceToHost, st)) ||
            !ck(cudaMemcpyAsync(&last_len, ilen + n_sets - 1, 4, cudaMemcpyDeviceToHost, st)) ||
            !ck(cudaMemcpyAsync(&max_tok, mx, 4, cudaMemcpyDeviceToHost, st)) ||
            !ck(cudaStreamSynchronize(st)))
            goto done;
        const uint64_t E = (uint64_t)last_off + last_len;
        if (E > 0x7FFFFFFFull) {  // cub item counts are int
            err = cudaErrorInvalidValue;
            goto done;
        }
        // joiners.hpp:21-24 (every set non-empty here or max 0); the per-token heads and cub's
        // int item counts need universe + 1 < 2^31 (refused: cudaErrorInvalidValue)
        if (max_tok >= 0x7FFFFFFEu) {
            err = cudaErrorInvalidValue;
            goto done;
        }
        ix->universe = max_tok + 1;
        ix->n_post = E;
        if (!ck(cudaMalloc(&count, ((size_t)ix->universe + 1) * 4)) ||
            !ck(cudaMemsetAsync(count, 0, ((size_t)ix->universe + 1) * 4, st)) ||
            !ck(cudaMalloc(&ix->head, ((size_t)ix->universe + 1) * 4)) ||
            !ck(cudaMalloc(&ix->post, (size_t)(E ? E : 1) * sizeof(uint2))))
            goto done;
        if (E) {
            if (!ck(cudaMalloc(&keys, E * 4)) || !ck(cudaMalloc(&keys2, E * 4)) ||
                !ck(cudaMalloc(&vals, E * 8)) || !ck(cudaMalloc(&vals2, E * 8)))
                goto done;
            entries_kernel<<<g, 256, 0, st>>>(*ix, ilen, off, keys, vals, count);
            if (!ck(cudaGetLastError())) goto done;
            int bits = 1;
            while (bits < 32 && (1ull << bits) < ix->universe) ++bits;
            tb = 0;
            // stable: postings of a token stay set-ascending
            if (!ck(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys2, vals, vals2, (int)E,
                                                    0, bits, st)) ||
                !ck(cudaMalloc(&tmp, tb)) ||
                !ck(cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys2, vals, vals2, (int)E, 0,
                                                    bits, st)))
                goto done;
            unpack_kernel<<<(uint32_t)((E + 255) / 256), 256, 0, st>>>(vals2, E, ix->post);
            if (!ck(cudaGetLastError())) goto done;
            cudaFree(tmp);
            tmp = nullptr;
        }
        tb = 0;
        if (!ck(cub::DeviceScan::ExclusiveSum(nullptr, tb, count, ix->head, (int)ix->universe + 1, st)) ||
            !ck(cudaMalloc(&tmp, tb)) ||
            !ck(cub::DeviceScan::ExclusiveSum(tmp, tb, count, ix->head, (int)ix->universe + 1, st)))
            goto done;
        ck(cudaStreamSynchronize(st));
    }
done:
    cudaFree(ilen);
    cudaFree(off);
    cudaFree(mx);
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(vals);
    cudaFree(vals2);
    cudaFree(count);
    cudaFree(tmp);
    if (err != cudaSuccess) filter_index_free(ix);
    return err;
}

void filter_index_free(FilterIndex* ix) {
    cudaFree(ix->head);
    cudaFree(ix->post);
    cudaFree(ix->work);
    ix->head = nullptr;
    ix->post = nullptr;
    ix->work = nullptr;
    ix->n_post = 0;
}

cudaError_t filter_bounds(const FilterIndex& ix, uint32_t a, uint32_t b,
                          unsigned long long* d_bound, cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    bounds_kernel<<<warps_grid(b - a), 256, 0, st>>>(ix, a, b, d_bound);
    return cudaGetLastError();
}

cudaError_t filter_generate(const FilterIndex& ix, uint32_t a, uint32_t b,
                            const unsigned long long* d_base, unsigned long long base0,
                            uint32_t* d_C, unsigned long long* d_count, uint32_t* d_flag,
                            cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    if (SSJB_GEN_DYN) {
        if (!ix.work) return cudaErrorInvalidValue;
        cudaError_t e = cudaMemsetAsync(ix.work, 0, sizeof(unsigned long long), st);
        if (e != cudaSuccess) return e;
    }
    generate_kernel<<<warps_grid(b - a), kGenThreads, 0, st>>>(ix, a, b, d_base, base0, d_C,
                                                                d_count, d_flag);
    return cudaGetLastError();
}

cudaError_t filter_compact(uint32_t a, uint32_t b, const unsigned long long* d_base,
                           unsigned long long base0, const uint32_t* d_C,
                           const unsigned long long* d_count,
                           const unsigned long long* d_out_base, const uint32_t* d_slot,
                           uint32_t* d_outC, uint32_t* d_outCO, cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    compact_kernel<<<warps_grid(b - a), 256, 0, st>>>(a, b, d_base, base0, d_C, d_count,
                                                       d_out_base, d_slot, d_outC, d_outCO);
    return cudaGetLastError();
}

}  // namespace ssjb

// ---- GroupJoin -------------------------------------------------------------------------------
namespace ssjb {

namespace {

__global__ void group_flags_kernel(const uint32_t* __restrict__ tokens, const uint2* __restrict__ sets,
                                   uint32_t n, const PredDev pred, uint32_t* flag) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t f = 1;
    if (i) {
        const uint2 a = sets[i], b = sets[i - 1];
        if (a.y == b.y) {
            // equal sizes -> equal probe-prefix lengths; compare the prefixes (joiners.hpp:125-129)
            const uint32_t P = a.y ? dev_prefix_lengths(pred, a.y).x : 0u;
            const uint32_t* ta = tokens + (size_t)a.x * 8;
            const uint32_t* tb = tokens + (size_t)b.x * 8;
            uint32_t q = 0;
            while (q < P && ta[q] == tb[q]) ++q;
            f = q < P;
        }
    }
    flag[i] = f;
}

__global__ void group_fill_kernel(const uint2* __restrict__ sets, uint32_t n, const uint32_t* flag,
                                  const uint32_t* gid_incl, uint32_t* first, uint2* rep) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    const uint32_t g = gid_incl[i] - 1;
    first[g] = i;
    rep[g] = sets[i];
}

__global__ void group_heads_kernel(const uint4* __restrict__ heads, const uint32_t* first,
                                   uint32_t G, uint4* rep_heads) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    rep_heads[2 * (size_t)g] = heads[2 * (size_t)first[g]];
    rep_heads[2 * (size_t)g + 1] = heads[2 * (size_t)first[g] + 1];
}

__global__ void group_count_kernel(const uint32_t* first, uint32_t G, uint32_t n, uint32_t* count,
                                   uint2* fc) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const uint32_t c = (g + 1 < G ? first[g + 1] : n) - first[g];
    count[g] = c;
    fc[g] = make_uint2(first[g], c);
}

__global__ void group_sizes_kernel(const GroupIndex gi, uint32_t a, uint32_t b,
                                   const unsigned long long* base, unsigned long long base0,
                                   const uint32_t* M, const unsigned long long* mcnt,
                                   unsigned long long* per, unsigned long long* cand,
                                   uint32_t* nbat) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = w; k < (uint64_t)(b - a); k += nw) {
        const uint32_t* m = M + (base[k] - base0);
        const uint32_t nm = (uint32_t)mcnt[k];
        unsigned long long S = 0;
        for (uint32_t q = lane; q < nm; q += 32) S += gi.count[m[q]];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
        if (lane == 0) {
            const uint32_t c = gi.count[a + k];
            per[k] = S;
            cand[k] = nm ? (unsigned long long)c * S : 0ull;
            nbat[k] = nm ? c : 0u;
        }
    }
}

__global__ void group_expand_kernel(const GroupIndex gi, uint32_t a, uint32_t b,
                                    const unsigned long long* base, unsigned long long base0,
                                    const uint32_t* M, const unsigned long long* mcnt,
                                    const unsigned long long* per, const unsigned long long* coff,
                                    const uint32_t* soff, uint32_t* C, uint32_t* CO) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = w; k < (uint64_t)(b - a); k += nw) {
        const uint32_t nm = (uint32_t)mcnt[k];
        if (!nm) continue;
        const uint32_t g = a + (uint32_t)k;
        const uint32_t* m = M + (base[k] - base0);
        const uint32_t c = gi.count[g], f = gi.first[g];
        const unsigned long long S = per[k];
        // the matched groups' members, 32 matched groups at a time: one {first, count}
        // gather per matched group, written once per member of g (joiners.hpp:160-170)
        unsigned long long run = 0;
        for (uint32_t q0 = 0; q0 < nm; q0 += 32) {
            const uint32_t q = q0 + lane;
            const uint2 fh = q < nm ? gi.fc[m[q]] : make_uint2(0u, 0u);
            uint32_t incl = fh.y;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, off);
                if (lane >= (uint32_t)off) incl += v;
            }
            for (uint32_t mm = 0; mm < c; ++mm) {
                uint32_t* dst = C + coff[k] + (unsigned long long)mm * S + run + (incl - fh.y);
                for (uint32_t j = 0; j < fh.y; ++j) dst[j] = fh.x + j;
            }
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        for (uint32_t mm = lane; mm < c; mm += 32) {
            const size_t sl = (size_t)soff[k] + mm;
            CO[2 * sl] = f + mm;
            CO[2 * sl + 1] = (uint32_t)(coff[k] + (unsigned long long)mm * S + S);
        }
    }
}

__global__ void group_intra_sizes_kernel(const GroupIndex gi, uint32_t a, uint32_t b,
                                         unsigned long long* icand, uint32_t* islc) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= b - a) return;
    const unsigned long long c = gi.count[a + k];
    icand[k] = c * (c - 1) / 2;
    islc[k] = c ? (uint32_t)(c - 1) : 0u;
}

__global__ void group_intra_kernel(const GroupIndex gi, uint32_t a, uint32_t b,
                                   const unsigned long long* coff, const uint32_t* soff,
                                   uint32_t* C, uint32_t* CO) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t k = w; k < (uint64_t)(b - a); k += nw) {
        const uint32_t c = gi.count[a + k], f = gi.first[a + k];
        for (uint32_t i = 1; i < c; ++i) {
            const unsigned long long o = coff[k] + (unsigned long long)i * (i - 1) / 2;
            for (uint32_t j = lane; j < i; j += 32) C[o + j] = f + j;
            if (lane == 0) {
                const size_t sl = (size_t)soff[k] + (i - 1);
                CO[2 * sl] = f + i;
                CO[2 * sl + 1] = (uint32_t)(o + i);
            }
        }
    }
}

uint32_t warps_grid2(uint64_t items) {
    const uint64_t warps = items < 148ull * 64 ? (items ? items : 1) : 148ull * 64;
    return (uint32_t)((warps * 32 + 255) / 256);
}

}  // namespace

cudaError_t group_index_build(GroupIndex* gi, const uint32_t* d_tokens, const uint2* d_sets,
                              const uint4* d_heads, uint32_t n, const PredDev& pred,
                              cudaStream_t st) {
    group_index_free(gi);
    if (!n) return cudaSuccess;
    uint32_t *flag = nullptr, *incl = nullptr;
    void* tmp = nullptr;
    cudaError_t err = cudaSuccess;
    auto ck = [&](cudaError_t e) {
        if (err == cudaSuccess && e != cudaSuccess) err = e;
        return err == cudaSuccess;
    };
    size_t tb = 0;
    uint32_t G = 0;
    const uint32_t g256 = (n + 255) / 256;
    if (!ck(cudaMalloc(&flag, (size_t)n * 4)) || !ck(cudaMalloc(&incl, (size_t)n * 4))) goto done;
    group_flags_kernel<<<g256, 256, 0, st>>>(d_tokens, d_sets, n, pred, flag);
    if (!ck(cudaGetLastError())) goto done;
    if (!ck(cub::DeviceScan::InclusiveSum(nullptr, tb, flag, incl, (int)n, st)) ||
        !ck(cudaMalloc(&tmp, tb)) || !ck(cub::DeviceScan::InclusiveSum(tmp, tb, flag, incl, (int)n, st)) ||
        !ck(cudaMemcpyAsync(&G, incl + n - 1, 4, cudaMemcpyDeviceToHost, st)) ||
        !ck(cudaStreamSynchronize(st)))
        goto done;
    gi->n_groups = G;
    if (!ck(cudaMalloc(&gi->first, (size_t)G * 4)) || !ck(cudaMalloc(&gi->count, (size_t)G * 4)) ||
        !ck(cudaMalloc(&gi->fc, (size_t)G * sizeof(uint2))) ||
        !ck(cudaMalloc(&gi->rep, (size_t)G * sizeof(uint2))))
        goto done;
    group_fill_kernel<<<g256, 256, 0, st>>>(d_sets, n, flag, incl, gi->first, gi->rep);
    group_count_kernel<<<(G + 255) / 256, 256, 0, st>>>(gi->first, G, n, gi->count, gi->fc);
    if (!ck(cudaGetLastError())) goto done;
    // PPJoin over the representatives (joiners.hpp:144-160)
    if (!ck(filter_index_build(&gi->ix, d_tokens, gi->rep, G, pred, 1, st))) goto done;
    gi->ix.heads = nullptr;
    if (d_heads) {  // the representatives' head records, indexed by group like the index
        if (!ck(cudaMalloc(&gi->rep_heads, (size_t)G * 2 * sizeof(uint4)))) goto done;
        group_heads_kernel<<<(G + 255) / 256, 256, 0, st>>>(d_heads, gi->first, G, gi->rep_heads);
        if (!ck(cudaGetLastError())) goto done;
        gi->ix.heads = gi->rep_heads;
    }
done:
    cudaFree(flag);
    cudaFree(incl);
    cudaFree(tmp);
    if (err != cudaSuccess) group_index_free(gi);
    return err;
}

void group_index_free(GroupIndex* gi) {
    cudaFree(gi->rep_heads);
    gi->rep_heads = nullptr;
    cudaFree(gi->first);
    cudaFree(gi->count);
    cudaFree(gi->fc);
    gi->fc = nullptr;
    cudaFree(gi->rep);
    gi->first = gi->count = nullptr;
    gi->rep = nullptr;
    gi->n_groups = 0;
    filter_index_free(&gi->ix);
}

cudaError_t group_sizes(const GroupIndex& gi, uint32_t a, uint32_t b,
                        const unsigned long long* d_base, unsigned long long base0,
                        const uint32_t* d_M, const unsigned long long* d_mcnt,
                        unsigned long long* d_per, unsigned long long* d_cand, uint32_t* d_nbat,
                        cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    group_sizes_kernel<<<warps_grid2(b - a), 256, 0, st>>>(gi, a, b, d_base, base0, d_M, d_mcnt,
                                                            d_per, d_cand, d_nbat);
    return cudaGetLastError();
}

cudaError_t group_expand(const GroupIndex& gi, uint32_t a, uint32_t b,
                         const unsigned long long* d_base, unsigned long long base0,
                         const uint32_t* d_M, const unsigned long long* d_mcnt,
                         const unsigned long long* d_per, const unsigned long long* d_coff,
                         const uint32_t* d_soff, uint32_t* d_C, uint32_t* d_CO, cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    group_expand_kernel<<<warps_grid2(b - a), 256, 0, st>>>(gi, a, b, d_base, base0, d_M, d_mcnt,
                                                             d_per, d_coff, d_soff, d_C, d_CO);
    return cudaGetLastError();
}

cudaError_t group_intra_sizes(const GroupIndex& gi, uint32_t a, uint32_t b,
                              unsigned long long* d_icand, uint32_t* d_islc, cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    group_intra_sizes_kernel<<<(b - a + 255) / 256, 256, 0, st>>>(gi, a, b, d_icand, d_islc);
    return cudaGetLastError();
}

cudaError_t group_intra(const GroupIndex& gi, uint32_t a, uint32_t b,
                        const unsigned long long* d_coff, const uint32_t* d_soff,
                        uint32_t* d_C, uint32_t* d_CO, cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    group_intra_kernel<<<warps_grid2(b - a), 256, 0, st>>>(gi, a, b, d_coff, d_soff, d_C, d_CO);
    return cudaGetLastError();
}

}  // namespace ssjb
