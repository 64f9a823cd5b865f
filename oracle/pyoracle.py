"""ctypes bindings of the parity oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

C restatement (always available once `make -C oracle` ran):
    equivalent_overlap, meets_threshold, threshold_parse, verify_pair_count,
    full_overlap, intersect_path_partition, partition_count, verify_chunk,
    chunk_algorithmic_bytes, brute_force_join
Reference shim (available when oracle/_ref/libssjref.so exists): class `Ref`.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libssj_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libssjref.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)

JACCARD, COSINE, DICE, OVERLAP = 0, 1, 2, 3


class _Pred(C.Structure):
    _fields_ = [("function", C.c_int32), ("num", C.c_uint64), ("den", C.c_uint64),
                ("overlap_threshold", C.c_uint64)]


class _VerifyResult(C.Structure):
    _fields_ = [("overlap", C.c_uint64), ("met", C.c_int32), ("comparisons", C.c_uint32),
                ("i_exit", C.c_uint32), ("j_exit", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [("pairs_verified", C.c_uint64), ("early_exit_prunes", C.c_uint64),
                ("comparison_budget_violations", C.c_uint64)]


class _SsjPred(C.Structure):  # ssj_predicate (include/ssjoin_b200.h), for work_shim.cpp
    _fields_ = [("function", C.c_int32), ("reserved", C.c_uint32), ("num", C.c_uint64),
                ("den", C.c_uint64), ("overlap_threshold", C.c_uint64)]


class _SynthConfig(C.Structure):  # ssj_synth_config (include/ssjoin_b200.h)
    _fields_ = [("seed", C.c_uint64), ("n_sets", C.c_uint32), ("min_size", C.c_uint32),
                ("max_size", C.c_uint32), ("zipf_sizes", C.c_int32), ("size_skew", C.c_double),
                ("universe", C.c_uint32), ("zipf_tokens", C.c_int32), ("token_skew", C.c_double),
                ("duplicate_fraction", C.c_double), ("max_edits", C.c_uint32),
                ("distinct_tokens", C.c_int32), ("threads", C.c_uint32)]


def _ptr(a, t=u32p):
    return a.ctypes.data_as(t) if a is not None and a.size else None


def _u32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.check_call(["make", "-C", HERE, "-s", "all"])
        L = C.CDLL(ORACLE_SO)
        L.ssjo_equivalent_overlap.restype = C.c_uint64
        L.ssjo_equivalent_overlap.argtypes = [C.POINTER(_Pred), C.c_uint64, C.c_uint64]
        L.ssjo_meets_threshold.restype = C.c_int
        L.ssjo_meets_threshold.argtypes = [C.POINTER(_Pred), C.c_uint64, C.c_uint64, C.c_uint64]
        L.ssjo_threshold_parse.restype = C.c_int
        L.ssjo_threshold_parse.argtypes = [C.c_char_p, u64p, u64p]
        L.ssjo_verify_pair_count.restype = _VerifyResult
        L.ssjo_verify_pair_count.argtypes = [u32p, C.c_size_t, u32p, C.c_size_t, C.c_uint64]
        L.ssjo_full_overlap.restype = C.c_uint64
        L.ssjo_full_overlap.argtypes = [u32p, C.c_size_t, u32p, C.c_size_t]
        L.ssjo_intersect_path_partition.restype = None
        L.ssjo_intersect_path_partition.argtypes = [u32p, C.c_size_t, u32p, C.c_size_t,
                                                    C.c_uint32, C.c_uint32, u32p, u32p, u32p]
        L.ssjo_partition_count.restype = C.c_uint64
        L.ssjo_partition_count.argtypes = [u32p, C.c_size_t, u32p, C.c_size_t, C.c_uint32,
                                           C.c_uint32, C.c_uint32]
        L.ssjo_verify_chunk.restype = C.c_int
        L.ssjo_verify_chunk.argtypes = [u32p, u32p, C.c_uint32, u32p, C.c_uint64, u32p,
                                        C.c_uint64, C.POINTER(_Pred), u8p, u32p, u32p, u64p,
                                        C.POINTER(_Stats)]
        L.ssjo_chunk_algorithmic_bytes.restype = C.c_uint64
        L.ssjo_chunk_algorithmic_bytes.argtypes = [u32p, u32p, C.c_uint32, u32p, C.c_uint64,
                                                   u32p, C.c_uint64, C.POINTER(_Pred)]
        L.ssjo_brute_force_join.restype = C.c_uint64
        L.ssjo_brute_force_join.argtypes = [u32p, u32p, C.c_uint32, C.POINTER(_Pred), u32p,
                                            C.c_uint64]
        _lib = L
    return _lib


def pred(function=JACCARD, num=4, den=5, overlap_threshold=1):
    return _Pred(int(function), int(num), int(den), int(overlap_threshold))


def equivalent_overlap(p, r, s):
    return lib().ssjo_equivalent_overlap(C.byref(p), r, s)


def meets_threshold(p, o, r, s):
    return bool(lib().ssjo_meets_threshold(C.byref(p), o, r, s))


def threshold_parse(text):
    n, d = C.c_uint64(), C.c_uint64()
    if lib().ssjo_threshold_parse(text.encode(), C.byref(n), C.byref(d)):
        raise ValueError("bad threshold: " + text)
    return n.value, d.value


def verify_pair_count(r, s, required):
    r, s = _u32(r), _u32(s)
    res = lib().ssjo_verify_pair_count(_ptr(r), r.size, _ptr(s), s.size, required)
    return res


def full_overlap(r, s):
    r, s = _u32(r), _u32(s)
    return lib().ssjo_full_overlap(_ptr(r), r.size, _ptr(s), s.size)


def intersect_path_partition(r, s, workers, k):
    r, s = _u32(r), _u32(s)
    a, b, h = C.c_uint32(), C.c_uint32(), C.c_uint32()
    lib().ssjo_intersect_path_partition(_ptr(r), r.size, _ptr(s), s.size, workers, k,
                                        C.byref(a), C.byref(b), C.byref(h))
    return a.value, b.value, h.value


def partition_count(r, s, part):
    r, s = _u32(r), _u32(s)
    return lib().ssjo_partition_count(_ptr(r), r.size, _ptr(s), s.size, *part)


def verify_chunk(tokens, offsets, C_, C_O, p, want_flags=True, want_overlaps=False,
                 want_touched=False):
    """Strategy-A verify_chunk restatement. Returns dict(flags, count, stats, overlaps,
    touched). Raises IndexError / ValueError like the reference's exceptions."""
    tokens, offsets, C_, C_O = _u32(tokens), _u32(offsets), _u32(C_), _u32(C_O)
    n_sets = offsets.size - 1
    flags = np.zeros(C_.size, np.uint8) if want_flags else None
    ovs = np.zeros(C_.size, np.uint32) if want_overlaps else None
    tch = np.zeros(C_.size, np.uint32) if want_touched else None
    count = C.c_uint64()
    st = _Stats()
    rc = lib().ssjo_verify_chunk(_ptr(tokens), _ptr(offsets), n_sets, _ptr(C_), C_.size,
                                 _ptr(C_O), C_O.size, C.byref(p), _ptr(flags, u8p), _ptr(ovs),
                                 _ptr(tch), C.byref(count), C.byref(st))
    if rc == -1:
        raise IndexError("set index out of range")
    if rc == -2:
        raise ValueError("malformed C_O")
    return dict(flags=flags, count=count.value, overlaps=ovs, touched=tch,
                stats=(st.pairs_verified, st.early_exit_prunes, st.comparison_budget_violations))


def chunk_algorithmic_bytes(tokens, offsets, C_, C_O, p):
    tokens, offsets, C_, C_O = _u32(tokens), _u32(offsets), _u32(C_), _u32(C_O)
    return lib().ssjo_chunk_algorithmic_bytes(_ptr(tokens), _ptr(offsets), offsets.size - 1,
                                              _ptr(C_), C_.size, _ptr(C_O), C_O.size,
                                              C.byref(p))


def brute_force_join(tokens, offsets, p):
    """oracle.hpp:36-67: (r, s, overlap) triples in loop order (r > s)."""
    tokens, offsets = _u32(tokens), _u32(offsets)
    n = offsets.size - 1
    total = lib().ssjo_brute_force_join(_ptr(tokens), _ptr(offsets), n, C.byref(p), None, 0)
    out = np.zeros(3 * max(total, 1), np.uint32)
    lib().ssjo_brute_force_join(_ptr(tokens), _ptr(offsets), n, C.byref(p), _ptr(out), total)
    return out[: 3 * total].reshape(-1, 3)


def oracle_pairs(original_id, triples):
    """helpers.hpp:41-51 oracle_pairs: normalized (max, min) original ids, sorted."""
    if len(triples) == 0:
        return np.zeros((0, 2), np.uint32)
    a = np.asarray(original_id, np.uint32)[triples[:, 0]]
    b = np.asarray(original_id, np.uint32)[triples[:, 1]]
    pairs = np.stack([np.maximum(a, b), np.minimum(a, b)], axis=1)
    order = np.lexsort((pairs[:, 1], pairs[:, 0]))
    return pairs[order]


# ---------------------------------------------------------------------------------------
# The reference itself (oracle/_ref/libssjref.so), when available.

def ref_available():
    return os.path.exists(REF_SO)


class Ref:
    """Bindings of oracle/ref_shim.cpp (the unmodified reference headers)."""

    def __init__(self):
        L = C.CDLL(REF_SO)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_synth.restype = vp
        L.ref_synth.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int,
                                C.c_double, C.c_uint32, C.c_int, C.c_double, C.c_double]
        L.ref_coll_from_csr.restype = vp
        L.ref_coll_from_csr.argtypes = [u32p, u32p, C.c_uint32, u32p]
        L.ref_coll_sizes.argtypes = [vp, u64p, u64p]
        L.ref_coll_copy.argtypes = [vp, u32p, u32p, u32p]
        L.ref_coll_free.argtypes = [vp]
        L.ref_equivalent_overlap.restype = C.c_uint64
        L.ref_equivalent_overlap.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                             C.c_uint64, C.c_uint64]
        L.ref_meets_threshold.restype = C.c_int
        L.ref_meets_threshold.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_uint64, C.c_uint64, C.c_uint64]
        L.ref_threshold_parse.restype = C.c_int
        L.ref_threshold_parse.argtypes = [C.c_char_p, u64p, u64p]
        L.ref_verify_pair_count.argtypes = [u32p, C.c_uint64, u32p, C.c_uint64, C.c_uint64,
                                            u64p, C.POINTER(C.c_int), u32p]
        L.ref_intersect_path_partitions.argtypes = [u32p, C.c_uint64, u32p, C.c_uint64,
                                                    C.c_uint32, u32p, u64p]
        L.ref_pool_create.restype = vp
        L.ref_pool_create.argtypes = [C.c_uint]
        L.ref_pool_workers.restype = C.c_uint
        L.ref_pool_workers.argtypes = [vp]
        L.ref_pool_free.argtypes = [vp]
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_verify_chunk.restype = C.c_int
        L.ref_verify_chunk.argtypes = [vp, vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                       C.c_int, C.c_uint32, C.c_int, u32p, C.c_uint64, u32p,
                                       C.c_uint64, u8p, u64p, u64p, C.POINTER(C.c_int), u32p]
        L.ref_time_verify_chunk.restype = C.c_double
        L.ref_time_verify_chunk.argtypes = [vp, vp, C.c_int, C.c_uint64, C.c_uint64,
                                            C.c_uint64, C.c_int, C.c_uint32, C.c_int, u32p,
                                            C.c_uint64, u32p, C.c_uint64, C.c_int, u64p, u8p]
        L.ref_work_last_error.restype = C.c_char_p
        L.ref_work_synth.restype = vp
        L.ref_work_synth.argtypes = [C.POINTER(_SynthConfig), u64p, u64p]
        L.ref_work_synth_copy.argtypes = [vp, u32p, u32p, u32p]
        L.ref_work_generate_windows.restype = vp
        L.ref_work_generate_windows.argtypes = [u32p, u32p, C.c_uint32, C.POINTER(_SsjPred),
                                                C.c_int32, u32p, C.c_uint32, C.c_uint32, u64p,
                                                u64p]
        L.ref_work_candidates_copy.argtypes = [vp, u32p, u32p]
        L.ref_run_join.restype = vp
        L.ref_run_join.argtypes = [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                   C.c_uint64, C.c_int, C.c_uint32, C.c_int, C.c_uint, C.c_int]
        L.ref_join_report.argtypes = [vp, u64p, C.POINTER(C.c_double)]
        L.ref_join_pairs.argtypes = [vp, u32p]
        L.ref_join_pairs_unsorted.argtypes = [vp, u32p]
        L.ref_join_chunk_count.restype = C.c_uint64
        L.ref_join_chunk_count.argtypes = [vp]
        L.ref_join_chunk_sizes.argtypes = [vp, C.c_uint64, u64p, u64p, u64p]
        L.ref_join_chunk_copy.argtypes = [vp, C.c_uint64, u32p, u32p, u8p]
        L.ref_join_free.argtypes = [vp]
        L.ref_brute_force.restype = C.c_int64
        L.ref_brute_force.argtypes = [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, u32p,
                                      C.c_uint64]
        L.ref_generate.restype = vp
        L.ref_generate.argtypes = [vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        L.ref_cands_sizes.argtypes = [vp, u64p, u64p, u64p]
        L.ref_cands_copy.argtypes = [vp, u32p, u32p, u32p]
        L.ref_cands_free.argtypes = [vp]
        self.L = L

    def err(self):
        return self.L.ref_last_error().decode()

    # collections -------------------------------------------------------------------
    def synth(self, seed, sets=100, min_size=1, max_size=50, zipf_sizes=False, size_skew=1.0,
              universe=1000, zipf_tokens=False, token_skew=1.0, duplicate_fraction=0.0):
        h = self.L.ref_synth(seed, sets, min_size, max_size, int(zipf_sizes), size_skew,
                             universe, int(zipf_tokens), token_skew, duplicate_fraction)
        if not h:
            raise RuntimeError(self.err())
        return self._take(h)

    def _take(self, h):
        n, t = C.c_uint64(), C.c_uint64()
        self.L.ref_coll_sizes(h, C.byref(n), C.byref(t))
        tokens = np.zeros(max(t.value, 1), np.uint32)
        offsets = np.zeros(n.value + 1, np.uint32)
        oid = np.zeros(max(n.value, 1), np.uint32)
        self.L.ref_coll_copy(h, _ptr(tokens), _ptr(offsets), _ptr(oid))
        self.L.ref_coll_free(h)
        return tokens[: t.value], offsets, oid[: n.value]

    def coll(self, tokens, offsets, original_id=None):
        tokens, offsets = _u32(tokens), _u32(offsets)
        oid = _u32(original_id) if original_id is not None else None
        if tokens.size == 0:
            tokens = np.zeros(1, np.uint32)
        return self.L.ref_coll_from_csr(_ptr(tokens), _ptr(offsets), offsets.size - 1,
                                        _ptr(oid) if oid is not None else None)

    # primitives --------------------------------------------------------------------
    def equivalent_overlap(self, fn, num, den, ovt, r, s):
        return self.L.ref_equivalent_overlap(fn, num, den, ovt, r, s)

    def meets_threshold(self, fn, num, den, ovt, o, r, s):
        return bool(self.L.ref_meets_threshold(fn, num, den, ovt, o, r, s))

    def threshold_parse(self, text):
        n, d = C.c_uint64(), C.c_uint64()
        if self.L.ref_threshold_parse(text.encode(), C.byref(n), C.byref(d)):
            raise ValueError(self.err())
        return n.value, d.value

    def verify_pair_count(self, r, s, required):
        r, s = _u32(r), _u32(s)
        ov, met, cmp_ = C.c_uint64(), C.c_int(), C.c_uint32()
        self.L.ref_verify_pair_count(_ptr(r), r.size, _ptr(s), s.size, required, C.byref(ov),
                                     C.byref(met), C.byref(cmp_))
        return ov.value, bool(met.value), cmp_.value

    def intersect_path_partitions(self, r, s, workers):
        r, s = _u32(r), _u32(s)
        out = np.zeros(3 * workers, np.uint32)
        cnt = np.zeros(workers, np.uint64)
        self.L.ref_intersect_path_partitions(_ptr(r), r.size, _ptr(s), s.size, workers,
                                             _ptr(out), _ptr(cnt, u64p))
        return out.reshape(-1, 3), cnt

    # engine ------------------------------------------------------------------------
    def pool(self, workers=0):
        return self.L.ref_pool_create(workers)

    def verify_chunk(self, coll, pool, fn, num, den, ovt, kind, group, pairs_mode, C_, C_O):
        C_, C_O = _u32(C_), _u32(C_O)
        flags = np.zeros(max(C_.size, 1), np.uint8)
        count = C.c_uint64()
        stats = np.zeros(3, np.uint64)
        rk, rg = C.c_int(), C.c_uint32()
        rc = self.L.ref_verify_chunk(coll, pool, fn, num, den, ovt, kind, group, int(pairs_mode),
                                     _ptr(C_), C_.size, _ptr(C_O), C_O.size, _ptr(flags, u8p),
                                     C.byref(count), _ptr(stats, u64p), C.byref(rk), C.byref(rg))
        if rc:
            raise RuntimeError(self.err())
        return flags[: C_.size], count.value, stats, (rk.value, rg.value)

    def time_verify_chunk(self, coll, pool, fn, num, den, ovt, kind, group, pairs_mode, C_, C_O,
                          reps=3, flags_out=None):
        """Best-of-`reps` seconds of verify_chunk and its count; flags_out (uint8[|C|],
        Pairs mode) receives the last run's flags."""
        C_, C_O = _u32(C_), _u32(C_O)
        count = C.c_uint64()
        fp = _ptr(flags_out, u8p) if flags_out is not None else None
        sec = self.L.ref_time_verify_chunk(coll, pool, fn, num, den, ovt, kind, group,
                                           int(pairs_mode), _ptr(C_), C_.size, _ptr(C_O),
                                           C_O.size, reps, C.byref(count), fp)
        if sec < 0:
            raise RuntimeError(self.err())
        return sec, count.value

    # benchmark workload (work_shim.cpp: synth.cpp + candidates.cpp linked into this library,
    # so the reference arm never loads the product library) -----------------------------
    def work_synth(self, seed, sets=100, min_size=1, max_size=50, zipf_sizes=False,
                   size_skew=1.0, universe=1000, zipf_tokens=False, token_skew=1.0,
                   duplicate_fraction=0.0, max_edits=0, distinct_tokens=False, threads=0):
        """The product's deterministic synthetic collection (ssj_synth_collection):
        (tokens, offsets, original_id)."""
        cfg = _SynthConfig(seed, sets, min_size, max_size, int(zipf_sizes), size_skew, universe,
                           int(zipf_tokens), token_skew, duplicate_fraction, max_edits,
                           int(distinct_tokens), threads)
        n, t = C.c_uint64(), C.c_uint64()
        h = self.L.ref_work_synth(C.byref(cfg), C.byref(n), C.byref(t))
        if not h:
            raise RuntimeError(self.L.ref_work_last_error().decode())
        tokens = np.zeros(max(t.value, 1), np.uint32)
        offsets = np.zeros(n.value + 1, np.uint32)
        oid = np.zeros(max(n.value, 1), np.uint32)
        self.L.ref_work_synth_copy(h, _ptr(tokens), _ptr(offsets), _ptr(oid))
        return tokens[: t.value], offsets, oid[: n.value]

    def work_generate_windows(self, tokens, offsets, fn, num, den, ovt, algorithm, windows,
                              threads=0):
        """ssj_generate_candidates_windows: AllPairs (0) / PPJoin (1) candidates of the probe
        windows [(lo, hi), ...] as one chunk (C, C_O)."""
        tokens = _u32(tokens) if np.asarray(tokens).size else np.zeros(1, np.uint32)
        offsets = _u32(offsets)
        w = _u32(np.asarray(windows, np.int64).reshape(-1))
        p = _SsjPred(fn, 0, num, den, ovt)
        nC, nCO = C.c_uint64(), C.c_uint64()
        h = self.L.ref_work_generate_windows(_ptr(tokens), _ptr(offsets), offsets.size - 1,
                                             C.byref(p), algorithm, _ptr(w), w.size // 2,
                                             threads, C.byref(nC), C.byref(nCO))
        if not h:
            raise RuntimeError(self.L.ref_work_last_error().decode())
        c = np.zeros(max(nC.value, 1), np.uint32)
        co = np.zeros(max(nCO.value, 1), np.uint32)
        self.L.ref_work_candidates_copy(h, _ptr(c), _ptr(co))
        return c[: nC.value], co[: nCO.value]

    def run_join(self, coll, fn, num, den, ovt, algorithm=1, budget=64 << 20, kind=3, group=32,
                 pairs_mode=True, workers=1, record_chunks=False, sort_pairs=True):
        """The reference run_join: (report dict, pairs (sorted like write_pairs, or in
        JoinReport::pairs order when sort_pairs=False), recorded chunks)."""
        h = self.L.ref_run_join(coll, fn, num, den, ovt, algorithm, budget, kind, group,
                                int(pairs_mode), workers, int(record_chunks))
        if not h:
            raise RuntimeError(self.err())
        rep = np.zeros(11, np.uint64)
        tim = (C.c_double * 4)()
        self.L.ref_join_report(h, _ptr(rep, u64p), tim)
        pairs = np.zeros(2 * max(int(rep[8]), 1), np.uint32)
        if sort_pairs:
            self.L.ref_join_pairs(h, _ptr(pairs))
        else:
            self.L.ref_join_pairs_unsorted(h, _ptr(pairs))
        chunks = []
        for i in range(self.L.ref_join_chunk_count(h)):
            nC, nCO, cnt = C.c_uint64(), C.c_uint64(), C.c_uint64()
            self.L.ref_join_chunk_sizes(h, i, C.byref(nC), C.byref(nCO), C.byref(cnt))
            c = np.zeros(max(nC.value, 1), np.uint32)
            co = np.zeros(max(nCO.value, 1), np.uint32)
            f = np.zeros(max(nC.value, 1), np.uint8)
            self.L.ref_join_chunk_copy(h, i, _ptr(c), _ptr(co), _ptr(f, u8p))
            chunks.append((c[: nC.value], co[: nCO.value], f[: nC.value], cnt.value))
        self.L.ref_join_free(h)
        report = dict(count=int(rep[0]), chunk_count=int(rep[1]), candidate_count=int(rep[2]),
                      host_verified_pairs=int(rep[3]), max_live_candidate_bytes=int(rep[4]),
                      pairs_verified=int(rep[5]), early_exit_prunes=int(rep[6]),
                      comparison_budget_violations=int(rep[7]), resolved_kind=int(rep[9]),
                      resolved_group=int(rep[10]), filtering_ms=tim[0], serialization_ms=tim[1],
                      verification_ms=tim[2], join_ms=tim[3])
        return report, pairs[: 2 * int(rep[8])].reshape(-1, 2), chunks

    def brute_force(self, coll, fn, num, den, ovt):
        total = self.L.ref_brute_force(coll, fn, num, den, ovt, None, 0)
        if total < 0:
            raise RuntimeError(self.err())
        out = np.zeros(3 * max(total, 1), np.uint32)
        self.L.ref_brute_force(coll, fn, num, den, ovt, _ptr(out), total)
        return out[: 3 * total].reshape(-1, 3)

    def generate(self, coll, fn, num, den, ovt, algorithm):
        h = self.L.ref_generate(coll, fn, num, den, ovt, algorithm)
        if not h:
            raise RuntimeError(self.err())
        nC, nCO, nH = C.c_uint64(), C.c_uint64(), C.c_uint64()
        self.L.ref_cands_sizes(h, C.byref(nC), C.byref(nCO), C.byref(nH))
        c = np.zeros(max(nC.value, 1), np.uint32)
        co = np.zeros(max(nCO.value, 1), np.uint32)
        hp = np.zeros(2 * max(nH.value, 1), np.uint32)
        self.L.ref_cands_copy(h, _ptr(c), _ptr(co), _ptr(hp))
        self.L.ref_cands_free(h)
        return c[: nC.value], co[: nCO.value], hp[: 2 * nH.value].reshape(-1, 2)
