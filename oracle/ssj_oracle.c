/*
 * ssj_oracle.c -- TEST INFRASTRUCTURE ONLY: plain-C restatement of the reference's
 * verification path, used as the parity checker (see ssj_oracle.h for the contract).
 * Every function cites the reference file:line it follows; paths are relative to
 * /root/reference/proj/include/ssjoin/.
 */
#include "ssj_oracle.h"

#include <math.h>
#include <string.h>

typedef unsigned __int128 u128;

/* similarity.hpp:88-90 ceil_div over u128, truncated to u64 */
static uint64_t ceil_div128(u128 a, u128 b) { return (uint64_t)((a + b - 1) / b); }

/* similarity.hpp:58-62 Threshold::reduce (Euclid, divide both by the gcd when > 1) */
void ssjo_threshold_reduce(uint64_t* num, uint64_t* den) {
    uint64_t a = *num, b = *den;
    while (b) {
        uint64_t r = a % b;
        a = b;
        b = r;
    }
    if (a > 1) {
        *num /= a;
        *den /= a;
    }
}

static int parse_u64(const char* p, const char* end, uint64_t* out) {
    /* std::stoull semantics for the digit strings this parser sees: leading digits only,
     * at least one digit required. */
    uint64_t v = 0;
    const char* q = p;
    while (q < end && *q >= '0' && *q <= '9') {
        v = v * 10 + (uint64_t)(*q - '0');
        ++q;
    }
    if (q == p) return -1;
    *out = v;
    return 0;
}

/* similarity.hpp:30-56 Threshold::parse: "0.8", ".85", "1", "1.0", "4/5". */
int ssjo_threshold_parse(const char* text, uint64_t* num_out, uint64_t* den_out) {
    size_t len = strlen(text);
    if (len == 0) return -1;
    const char* end = text + len;
    const char* slash = memchr(text, '/', len);
    uint64_t num = 0, den = 1;
    if (slash) {
        if (parse_u64(text, slash, &num) || parse_u64(slash + 1, end, &den)) return -1;
    } else {
        const char* dot = memchr(text, '.', len);
        const char* int_end = dot ? dot : end;
        if (int_end == text) {
            num = 0; /* digits.empty() -> "0" */
        } else if (parse_u64(text, int_end, &num)) {
            return -1;
        }
        if (dot) {
            for (const char* c = dot + 1; c < end; ++c) {
                if (*c < '0' || *c > '9') return -1;
                num = num * 10 + (uint64_t)(*c - '0');
                den *= 10;
            }
        }
    }
    if (den == 0) return -1;
    ssjo_threshold_reduce(&num, &den);
    *num_out = num;
    *den_out = den;
    return 0;
}

/* similarity.hpp:74-81 */
int ssjo_pred_validate(const ssjo_pred* p) {
    if (p->function != SSJO_OVERLAP) {
        if (p->num == 0 || p->num > p->den) return -1;
    } else if (p->overlap_threshold < 1) {
        return -1;
    }
    return 0;
}

/* similarity.hpp:93-102 ceil_scaled_sqrt: smallest k with k^2 den^2 >= num^2 r s */
static uint64_t ceil_scaled_sqrt(uint64_t num, uint64_t den, uint64_t r, uint64_t s) {
    u128 rhs = (u128)num * num * r * s;
    if (rhs == 0) return 0;
    long double est = (long double)num / den * sqrtl((long double)r * (long double)s);
    uint64_t k = est > 2.0L ? (uint64_t)est - 2 : 0;
    while ((u128)k * k * den * den < rhs) ++k;
    return k;
}

/* similarity.hpp:108-123 equivalent_overlap */
uint64_t ssjo_equivalent_overlap(const ssjo_pred* p, uint64_t size_r, uint64_t size_s) {
    const uint64_t num = p->num, den = p->den;
    switch (p->function) {
        case SSJO_JACCARD: return ceil_div128((u128)num * (size_r + size_s), den + num);
        case SSJO_COSINE: return ceil_scaled_sqrt(num, den, size_r, size_s);
        case SSJO_DICE: return ceil_div128((u128)num * (size_r + size_s), 2 * den);
        case SSJO_OVERLAP: return p->overlap_threshold;
    }
    return 0;
}

/* similarity.hpp:167-188 meets_threshold */
int ssjo_meets_threshold(const ssjo_pred* p, uint64_t o, uint64_t r, uint64_t s) {
    const uint64_t num = p->num, den = p->den;
    switch (p->function) {
        case SSJO_JACCARD: return (u128)o * den >= (u128)num * (r + s - o);
        case SSJO_COSINE: return (u128)o * o * den * den >= (u128)num * num * r * s;
        case SSJO_DICE: return (u128)2 * o * den >= (u128)num * (r + s);
        case SSJO_OVERLAP: return o >= p->overlap_threshold;
    }
    return 0;
}

/* similarity.hpp:135-164 size_bounds */
void ssjo_size_bounds(const ssjo_pred* p, uint64_t r, uint64_t* mn, uint64_t* mx) {
    const uint64_t num = p->num, den = p->den;
    uint64_t lo = 0, hi = UINT64_MAX;
    switch (p->function) {
        case SSJO_JACCARD:
            lo = ceil_div128((u128)num * r, den);
            hi = (uint64_t)((u128)den * r / num);
            break;
        case SSJO_COSINE:
            lo = ceil_div128((u128)num * num * r, (u128)den * den);
            hi = (uint64_t)((u128)den * den * r / ((u128)num * num));
            break;
        case SSJO_DICE:
            lo = ceil_div128((u128)num * r, 2 * den - num);
            hi = (uint64_t)((u128)(2 * den - num) * r / num);
            break;
        case SSJO_OVERLAP: lo = p->overlap_threshold; break;
    }
    if (lo == 0) lo = 1;
    *mn = lo;
    *mx = hi;
}

/* verify.hpp:50-72 verify_pair_count: the merge loop with two-sided early exit.
 * Exit order is the reference's: the met check, then the reachability bound, then a
 * comparison. */
ssjo_verify_result ssjo_verify_pair_count(const uint32_t* r, size_t m, const uint32_t* s,
                                          size_t n, uint64_t required) {
    ssjo_verify_result res = {0, 0, 0, 0, 0};
    size_t i = 0, j = 0;
    while (i < m && j < n) {
        if (res.overlap >= required) break;
        size_t rest = (m - i) < (n - j) ? (m - i) : (n - j);
        if (res.overlap + rest < required) break;
        ++res.comparisons;
        if (r[i] == s[j]) {
            ++res.overlap;
            ++i;
            ++j;
        } else if (r[i] < s[j]) {
            ++i;
        } else {
            ++j;
        }
    }
    res.met = res.overlap >= required;
    res.i_exit = (uint32_t)i;
    res.j_exit = (uint32_t)j;
    return res;
}

/* oracle.hpp:48-60: full merge without early exit */
uint64_t ssjo_full_overlap(const uint32_t* r, size_t m, const uint32_t* s, size_t n) {
    uint64_t o = 0;
    size_t a = 0, b = 0;
    while (a < m && b < n) {
        if (r[a] == s[b]) {
            ++o;
            ++a;
            ++b;
        } else if (r[a] < s[b]) {
            ++a;
        } else {
            ++b;
        }
    }
    return o;
}

/* verify.hpp:86-103 merge_path_split: ties consume r first (r[i] <= s[j]). */
uint32_t ssjo_merge_path_split(const uint32_t* r, size_t m, const uint32_t* s, size_t n,
                               size_t d) {
    size_t lo = d > n ? d - n : 0;
    size_t hi = d < m ? d : m;
    while (lo < hi) {
        size_t i = lo + (hi - lo) / 2;
        size_t j = d - i;
        if (i < m && j > 0 && r[i] <= s[j - 1]) {
            lo = i + 1;
        } else if (i > 0 && j < n && r[i - 1] > s[j]) {
            hi = i - 1;
        } else {
            lo = hi = i;
        }
    }
    return (uint32_t)lo;
}

/* verify.hpp:135-146 intersect_path_partition */
void ssjo_intersect_path_partition(const uint32_t* r, size_t m, const uint32_t* s, size_t n,
                                   uint32_t workers, uint32_t k, uint32_t* start_r,
                                   uint32_t* start_s, uint32_t* hops) {
    size_t total = m + n;
    size_t spacing = (total + workers - 1) / workers;
    size_t d = (size_t)k * spacing;
    if (total == 0 || d >= total) {
        *start_r = (uint32_t)m;
        *start_s = (uint32_t)n;
        *hops = 0;
        return;
    }
    uint32_t i = ssjo_merge_path_split(r, m, s, n, d);
    *start_r = i;
    *start_s = (uint32_t)(d - i);
    size_t h = total - d < spacing ? total - d : spacing;
    *hops = (uint32_t)h;
}

/* verify.hpp:151-166 partition_count: a common value counts at its r-side hop. */
uint64_t ssjo_partition_count(const uint32_t* r, size_t m, const uint32_t* s, size_t n,
                              uint32_t start_r, uint32_t start_s, uint32_t hops) {
    size_t i = start_r, j = start_s;
    uint64_t count = 0;
    for (uint32_t h = 0; h < hops && (i < m || j < n); ++h) {
        if (j >= n || (i < m && r[i] <= s[j])) {
            if (j < n && r[i] == s[j]) ++count;
            ++i;
        } else {
            ++j;
        }
    }
    return count;
}

/* chunk.hpp:36-48 decode: slices (probe, [prev, end)). Validation is ours: the reference
 * would read out of bounds on a malformed C_O. */
static int check_chunk(uint64_t nC, const uint32_t* C_O, uint64_t nCO) {
    uint64_t prev = 0;
    for (uint64_t e = 0; e + 1 < nCO; e += 2) {
        uint64_t end = C_O[e + 1];
        if (end < prev || end > nC) return -2;
        prev = end;
    }
    return 0;
}

/* verify.hpp:257-275 verify_chunk + :213-228 verify_slice_range + :188-194 record */
int ssjo_verify_chunk(const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                      const uint32_t* C, uint64_t nC, const uint32_t* C_O, uint64_t nCO,
                      const ssjo_pred* pred, uint8_t* flags, uint32_t* overlaps,
                      uint32_t* touched_s, uint64_t* count_out, ssjo_stats* stats) {
    if (check_chunk(nC, C_O, nCO)) return -2;
    if (flags) memset(flags, 0, nC);
    uint64_t count = 0;
    uint64_t prev = 0;
    for (uint64_t e = 0; e + 1 < nCO; e += 2) {
        uint32_t probe = C_O[e];
        uint64_t end = C_O[e + 1];
        if (end > prev && probe >= n_sets) return -1; /* set_view(probe) throws */
        const uint32_t* r = tokens + offsets[probe < n_sets ? probe : 0];
        size_t m = probe < n_sets ? offsets[probe + 1] - offsets[probe] : 0;
        for (uint64_t slot = prev; slot < end; ++slot) {
            uint32_t cand = C[slot];
            if (cand >= n_sets) return -1;
            const uint32_t* s = tokens + offsets[cand];
            size_t n = offsets[cand + 1] - offsets[cand];
            uint64_t required = ssjo_equivalent_overlap(pred, m, n);
            ssjo_verify_result res = ssjo_verify_pair_count(r, m, s, n, required);
            if (stats) {
                stats->pairs_verified++;
                if (res.comparisons > m + n) stats->comparison_budget_violations++;
                if (!res.met && res.comparisons < m + n) stats->early_exit_prunes++;
            }
            if (flags) flags[slot] = res.met ? 1 : 0;
            if (overlaps) overlaps[slot] = res.met ? (uint32_t)ssjo_full_overlap(r, m, s, n) : 0;
            if (touched_s) touched_s[slot] = (uint32_t)(res.j_exit + 1 < n ? res.j_exit + 1 : n);
            if (res.met) ++count;
        }
        prev = end;
    }
    if (count_out) *count_out = count;
    return 0;
}

uint64_t ssjo_chunk_algorithmic_bytes(const uint32_t* tokens, const uint32_t* offsets,
                                      uint32_t n_sets, const uint32_t* C, uint64_t nC,
                                      const uint32_t* C_O, uint64_t nCO, const ssjo_pred* pred) {
    if (check_chunk(nC, C_O, nCO)) return UINT64_MAX;
    uint64_t bytes = 0, prev = 0;
    for (uint64_t e = 0; e + 1 < nCO; e += 2) {
        uint32_t probe = C_O[e];
        uint64_t end = C_O[e + 1];
        if (probe >= n_sets) return UINT64_MAX;
        const uint32_t* r = tokens + offsets[probe];
        size_t m = offsets[probe + 1] - offsets[probe];
        bytes += 8 + 8 + 4 * (uint64_t)m;
        for (uint64_t slot = prev; slot < end; ++slot) {
            uint32_t cand = C[slot];
            if (cand >= n_sets) return UINT64_MAX;
            const uint32_t* s = tokens + offsets[cand];
            size_t n = offsets[cand + 1] - offsets[cand];
            uint64_t required = ssjo_equivalent_overlap(pred, m, n);
            ssjo_verify_result res = ssjo_verify_pair_count(r, m, s, n, required);
            uint64_t touched = res.j_exit + 1 < n ? res.j_exit + 1 : n;
            bytes += 4 + 8 + 1 + 4 * touched;
        }
        prev = end;
    }
    return bytes;
}

/* oracle.hpp:36-67 brute_force_join (guard omitted) */
uint64_t ssjo_brute_force_join(const uint32_t* tokens, const uint32_t* offsets, uint32_t n_sets,
                               const ssjo_pred* pred, uint32_t* out, uint64_t cap) {
    uint64_t total = 0;
    for (uint32_t i = 1; i < n_sets; ++i) {
        const uint32_t* r = tokens + offsets[i];
        size_t m = offsets[i + 1] - offsets[i];
        for (uint32_t j = 0; j < i; ++j) {
            const uint32_t* s = tokens + offsets[j];
            size_t n = offsets[j + 1] - offsets[j];
            uint64_t o = ssjo_full_overlap(r, m, s, n);
            if (ssjo_meets_threshold(pred, o, m, n)) {
                if (total < cap) {
                    out[3 * total] = i;
                    out[3 * total + 1] = j;
                    out[3 * total + 2] = (uint32_t)o;
                }
                ++total;
            }
        }
    }
    return total;
}
