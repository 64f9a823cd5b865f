// ssj_device.cuh -- device-side arithmetic and intersection primitives for sm_100a.
//
// Layout in HBM (uploaded once per engine, see engine.cu):
//   tokens : u32, padded CSR. Set i starts at tokens[8 * sets[i].x] (32-byte aligned, so
//            the first 8 tokens of every set are exactly one DRAM/L2 sector) and is
//            followed by 0xFFFFFFFF padding up to the next multiple of 8 tokens.
//   sets   : uint2 {pos8, size} per set (8 B, one random sector per candidate lookup;
//            8 MB for 1M sets, so it stays L2-resident across chunks).
// The reference layout it replaces is collection.hpp:76-94 (tokens + offsets[n+1]).
#pragma once

#include <cstdint>

namespace ssjb {

constexpr uint32_t kFnJaccard = 0, kFnCosine = 1, kFnDice = 2, kFnOverlap = 3;

// Error bits written to result word SSJ_RESULT_ERROR.
constexpr unsigned long long kErrOutOfRange = 1ull;  // set index >= n_sets
constexpr unsigned long long kErrBadOffsets = 2ull;  // C_O end offsets decreasing / > nC

// Predicate in the form the kernels evaluate. For Jaccard and Dice the required overlap is
// ceil(A * (r + s) / B) with A = num and B = num + den (Jaccard, similarity.hpp:113-114)
// or B = 2 * den (Dice, :117-118), B computed in u64 exactly like the reference.
struct PredDev {
    int32_t fn;
    int32_t wide;  // 1 -> u128 path needed (A >= 2^30 or B >= 2^32)
    uint64_t A, B;
    uint64_t num, den, ovt;
    uint32_t A32, B32, Binv;  // Jaccard/Dice, !wide: A, B and floor((2^32 - 1) / B)
    uint32_t pad;
};

// Jaccard / Dice required overlap ceil(A * sum / B) in 32-bit arithmetic when A * sum < 2^32
// (exact: q0 = umulhi(x, floor((2^32-1)/B)) is within 2 below floor(x / B)); else the
// reference formula. Returns min(required, 2^32 - 1).
__device__ __forceinline__ uint32_t dev_required_fast(const PredDev& p, uint32_t r, uint32_t s);

typedef unsigned __int128 u128;

// similarity.hpp:93-102 ceil_scaled_sqrt: smallest k >= 0 with k^2 den^2 >= num^2 r s.
// The double estimate minus 2 is never above the answer for any size pair a u32 CSR can
// hold, so stepping up reproduces the reference's long-double search exactly.
__device__ __forceinline__ uint64_t dev_ceil_scaled_sqrt(uint64_t num, uint64_t den, uint64_t r,
                                                         uint64_t s) {
    u128 rhs = (u128)num * num * r * s;
    if (rhs == 0) return 0;
    double est = (double)num / (double)den * sqrt((double)r * (double)s);
    uint64_t k = est > 2.0 ? (uint64_t)est - 2 : 0;
    while ((u128)k * k * den * den < rhs) ++k;
    return k;
}

// similarity.hpp:108-123 equivalent_overlap, bit-exact.
__device__ __forceinline__ uint64_t dev_required(const PredDev& p, uint32_t r, uint32_t s) {
    switch (p.fn) {
        case kFnJaccard:
        case kFnDice: {
            const uint64_t sum = (uint64_t)r + (uint64_t)s;
            if (!p.wide) {
                // A < 2^30, sum < 2^33, B < 2^32: A*sum + B - 1 < 2^64.
                const uint64_t a = p.A * sum;
                return (a + p.B - 1) / p.B;
            }
            const u128 a = (u128)p.A * sum;
            return (uint64_t)((a + (u128)p.B - 1) / (u128)p.B);
        }
        case kFnCosine: return dev_ceil_scaled_sqrt(p.num, p.den, r, s);
        default: return p.ovt;
    }
}

__device__ __forceinline__ uint32_t dev_required_fast(const PredDev& p, uint32_t r, uint32_t s) {
    if ((p.fn == kFnJaccard || p.fn == kFnDice) && !p.wide) {
        const uint64_t sum = (uint64_t)r + s;
        const uint64_t x64 = (uint64_t)p.A32 * sum;
        if (x64 <= 0xFFFFFFFFull) {
            const uint32_t x = (uint32_t)x64;
            uint32_t q = __umulhi(x, p.Binv);
            uint32_t rem = x - q * p.B32;
            if (rem >= p.B32) { ++q; rem -= p.B32; }
            if (rem >= p.B32) { ++q; rem -= p.B32; }
            return q + (rem != 0);
        }
    }
    const uint64_t v = dev_required(p, r, s);
    return v > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)v;
}

// Exactness argument used by every kernel below (verify.hpp:50-72):
// the reference's verdict is met <=> |r ∩ s| >= required (its early exits only stop when
// the verdict is already decided). With miss_r / miss_s = tokens of r / s consumed without
// a match, the reference's bound  overlap + min(m - i, n - j) < required  is exactly
// miss_r > m - required  or  miss_s > n - required. The kernels stop on the same bounds
// (possibly at a later point of the path, never earlier than sound), so their flags equal
// the reference's flags bit for bit.

// Thread-per-pair merge with two-sided early exit.
//   r   : probe tokens (shared or global memory, generic pointer), m = |r| >= 1
//   s4  : candidate tokens as 16-byte vectors (32-byte aligned), n = |s| >= 1
//   w0,w1 : s[0..8) already loaded by the caller (software prefetch)
//   req : required overlap, 1 <= req <= min(m, n)
// Returns met. With kFull the merge runs to the end for met pairs and *ov_out is the
// true |r ∩ s|; otherwise it stops at ov == req.
template <bool kFull>
__device__ __forceinline__ bool merge_thread(const uint32_t* __restrict__ r, uint32_t m,
                                             const uint4* __restrict__ s4, uint32_t n,
                                             uint32_t req, uint4 w0, uint4 w1,
                                             uint32_t* ov_out) {
    const uint32_t slack_r = m - req;
    const uint32_t slack_s = n - req;
    uint32_t i = 0, ov = 0, miss_s = 0;
    uint32_t a = r[0];
    uint32_t j = 0;
    uint32_t t[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    for (;;) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (j + q >= n) goto done;
            const uint32_t b = t[q];
            while (a < b) {
                ++i;
                if (i - ov > slack_r) goto reject;
                if (i >= m) goto done;
                a = r[i];
            }
            if (a == b) {
                ++ov;
                if (!kFull && ov >= req) goto done;
                ++i;
                if (i >= m) goto done;
                a = r[i];
            } else {
                ++miss_s;
                if (miss_s > slack_s) goto reject;
            }
        }
        j += 8;
        if (j >= n) break;
        {
            const uint4 v0 = __ldg(s4 + (j >> 2));
            const uint4 v1 = __ldg(s4 + (j >> 2) + 1);
            t[0] = v0.x; t[1] = v0.y; t[2] = v0.z; t[3] = v0.w;
            t[4] = v1.x; t[5] = v1.y; t[6] = v1.z; t[7] = v1.w;
        }
    }
done:
    if (kFull) *ov_out = ov;
    return ov >= req;
reject:
    if (kFull) *ov_out = 0;
    return false;
}

// Full overlap (no early exit) for a qualifying pair: used by the cooperative kernels'
// results mode, thread-sequential over global memory.
__device__ __forceinline__ uint32_t full_overlap_seq(const uint32_t* __restrict__ r, uint32_t m,
                                                     const uint32_t* __restrict__ s, uint32_t n) {
    uint32_t i = 0, j = 0, ov = 0;
    while (i < m && j < n) {
        const uint32_t a = r[i], b = s[j];
        ov += (a == b);
        i += (a <= b);
        j += (b <= a);
    }
    return ov;
}

// verify.hpp:86-103 merge_path_split: the (i, j), i + j = d, consistent with the merge
// order that consumes r[i] before s[j] iff r[i] <= s[j].
__device__ __forceinline__ uint32_t dev_merge_path_split(const uint32_t* __restrict__ r, uint32_t m,
                                                         const uint32_t* __restrict__ s, uint32_t n,
                                                         uint32_t d) {
    uint32_t lo = d > n ? d - n : 0;
    uint32_t hi = d < m ? d : m;
    while (lo < hi) {
        const uint32_t i = lo + (hi - lo) / 2;
        const uint32_t j = d - i;
        if (i < m && j > 0 && r[i] <= s[j - 1]) {
            lo = i + 1;
        } else if (i > 0 && j < n && r[i - 1] > s[j]) {
            hi = i - 1;
        } else {
            lo = hi = i;
        }
    }
    return lo;
}

}  // namespace ssjb
