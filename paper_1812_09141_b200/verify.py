"""The B200 verification engine (mirror of proj/include/ssjoin/verify.hpp:241-351).

`VerificationEngine` has the reference's constructor and `verify_chunk` surface; every
call goes through the C ABI (include/ssjoin_b200.h) into the sm_100a kernels. There is no
CPU path: constructing an engine without a CUDA device raises RuntimeError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .collection import CandidateChunk, Collection
from .similarity import SimilarityPredicate


class StrategyKind(IntEnum):
    """verify.hpp:18"""
    A = 0
    B = 1
    C = 2
    Auto = 3


class OutputMode(IntEnum):
    """verify.hpp:31"""
    Count = 0
    Pairs = 1


@dataclass
class Strategy:
    """verify.hpp:21-29"""
    kind: StrategyKind = StrategyKind.Auto
    group_size: int = 32

    def validate(self) -> None:
        s = N.ssj_strategy(int(self.kind), self.group_size)
        N.check(N.lib().ssj_strategy_validate(C.byref(s)))


@dataclass
class VerificationOutput:
    """verify.hpp:36-39: flags (Pairs mode, slot order = C order) + count."""
    flags: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))
    count: int = 0


@dataclass
class VerifyStats:
    """verify.hpp:183-195 (accumulated across calls)."""
    pairs_verified: int = 0
    early_exit_prunes: int = 0
    comparison_budget_violations: int = 0


def _vp(a: Optional[np.ndarray]):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else None


class VerificationEngine:
    """verify.hpp:241-351 on a B200.

    VerificationEngine(collection, pred, mode, strategy[, device]) uploads the collection
    once (padded CSR); verify_chunk(chunk[, pool, stats]) returns VerificationOutput with
    byte-identical flags and the same count as the reference. `pool` is accepted for
    signature parity and ignored (the grid replaces the WorkerPool).
    """

    def __init__(self, collection: Collection, pred: SimilarityPredicate, mode: OutputMode,
                 strategy: Strategy, device: int = 0, devices: Optional[Sequence[int]] = None):
        """devices: several GPUs behind one engine (ssj_engine_create_multi: one upload,
        NVLink fan-out, every chunk split by probe-slice ranges); `device` otherwise."""
        self._lib = N.lib()
        self._h = C.c_void_p()
        self.collection = collection
        self.pred = pred
        self.mode = OutputMode(mode)
        p = pred._c()
        s = N.ssj_strategy(int(strategy.kind), strategy.group_size)
        tokens = collection.tokens if collection.tokens.size else np.zeros(1, np.uint32)
        if devices is not None:
            devs = (C.c_int32 * len(devices))(*devices)
            N.check(self._lib.ssj_engine_create_multi(
                C.byref(self._h), devs, len(devices), tokens.ctypes.data_as(N.u32p),
                collection.offsets.ctypes.data_as(N.u32p), collection.size(), C.byref(p),
                int(self.mode), C.byref(s)))
            device = int(devices[0])
        else:
            N.check(self._lib.ssj_engine_create(
                C.byref(self._h), device, tokens.ctypes.data_as(N.u32p),
                collection.offsets.ctypes.data_as(N.u32p), collection.size(), C.byref(p),
                int(self.mode), C.byref(s)))
        r = N.ssj_strategy()
        N.check(self._lib.ssj_engine_strategy(self._h, C.byref(r)))
        self._strategy = Strategy(StrategyKind(r.kind), r.group_size)
        self.device = device

    @classmethod
    def from_device(cls, d_tokens: int, n_padded: int, d_sets: int, n_sets: int, n_tokens: int,
                    pred: SimilarityPredicate, mode: OutputMode, strategy: Strategy,
                    device: int = 0) -> "VerificationEngine":
        """Engine over a collection already resident on `device` in the padded layout
        (e.g. NCCL-broadcast from another rank's engine)."""
        self = cls.__new__(cls)
        self._lib = N.lib()
        self._h = C.c_void_p()
        self.collection = None
        self.pred = pred
        self.mode = OutputMode(mode)
        p = pred._c()
        s = N.ssj_strategy(int(strategy.kind), strategy.group_size)
        N.check(self._lib.ssj_engine_create_from_device(
            C.byref(self._h), device, C.c_void_p(d_tokens), n_padded, C.c_void_p(d_sets),
            n_sets, n_tokens, C.byref(p), int(self.mode), C.byref(s)))
        r = N.ssj_strategy()
        N.check(self._lib.ssj_engine_strategy(self._h, C.byref(r)))
        self._strategy = Strategy(StrategyKind(r.kind), r.group_size)
        self.device = device
        return self

    def devices(self) -> Tuple[list, float]:
        """(the engine's CUDA devices, collection fan-out ms)."""
        buf = (C.c_int32 * 64)()
        n = C.c_uint32()
        ms = C.c_double()
        N.check(self._lib.ssj_engine_devices(self._h, buf, 64, C.byref(n), C.byref(ms)))
        return [buf[i] for i in range(min(n.value, 64))], ms.value

    def device_collection(self) -> Tuple[int, int, int]:
        """(d_tokens, n_padded_tokens, d_sets) of the engine's resident collection."""
        t, s = C.c_void_p(), C.c_void_p()
        n = C.c_uint64()
        N.check(self._lib.ssj_engine_device_collection(self._h, C.byref(t), C.byref(n),
                                                       C.byref(s)))
        return t.value, n.value, s.value

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            self._lib.ssj_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def strategy(self) -> Strategy:
        """verify.hpp:255: the resolved strategy (never Auto), resolved like the reference
        (verify.hpp:249-253)."""
        return self._strategy

    def kernel_strategy(self) -> Strategy:
        """The kernel family that runs (Auto: strategy A's kernels)."""
        r = N.ssj_strategy()
        N.check(self._lib.ssj_engine_kernel_strategy(self._h, C.byref(r)))
        return Strategy(StrategyKind(r.kind), r.group_size)

    # -- the hot call ----------------------------------------------------------------
    def verify_chunk(self, chunk: CandidateChunk, pool=None,
                     stats: Optional[VerifyStats] = None,
                     flags_out: Optional[np.ndarray] = None) -> VerificationOutput:
        """verify.hpp:257-275. `flags_out` (optional, uint8[nC], e.g. pinned) receives the
        flags in place instead of a fresh array."""
        out = VerificationOutput()
        nC = chunk.candidate_count()
        flags = None
        if self.mode == OutputMode.Pairs:
            flags = flags_out if flags_out is not None else np.zeros(nC, np.uint8)
            assert flags.size >= nC and flags.dtype == np.uint8
        cnt = C.c_uint64()
        st = N.ssj_stats()
        N.check(self._lib.ssj_verify_chunk(self._h, _vp(chunk.C), nC, _vp(chunk.C_O),
                                           chunk.C_O.size, _vp(flags) if nC else None,
                                           C.byref(cnt), C.byref(st)))
        if flags is not None:
            out.flags = flags[:nC]
        out.count = cnt.value
        if stats is not None:
            stats.pairs_verified += st.pairs_verified
            stats.early_exit_prunes += st.early_exit_prunes
            stats.comparison_budget_violations += st.comparison_budget_violations
        return out

    def submit_chunk(self, chunk: CandidateChunk, flags: Optional[np.ndarray] = None) -> int:
        """Asynchronous half of verify_chunk (<= 2 in flight). Keep `chunk` and `flags`
        alive until wait_chunk returns."""
        t = C.c_uint64()
        N.check(self._lib.ssj_submit_chunk(self._h, _vp(chunk.C), chunk.candidate_count(),
                                           _vp(chunk.C_O), chunk.C_O.size, _vp(flags),
                                           C.byref(t)))
        return t.value

    def wait_chunk(self, ticket: int, stats: Optional[VerifyStats] = None) -> int:
        cnt = C.c_uint64()
        st = N.ssj_stats()
        N.check(self._lib.ssj_wait_chunk(self._h, ticket, C.byref(cnt), C.byref(st)))
        if stats is not None:
            stats.pairs_verified += st.pairs_verified
            stats.early_exit_prunes += st.early_exit_prunes
            stats.comparison_budget_violations += st.comparison_budget_violations
        return cnt.value

    def verify_chunk_results(self, chunk: CandidateChunk) -> Tuple[np.ndarray, np.ndarray]:
        """Qualifying slots (ascending) and their true overlaps |r ∩ s|."""
        nC = chunk.candidate_count()
        slots = np.zeros(max(nC, 1), np.uint32)
        ovs = np.zeros(max(nC, 1), np.uint32)
        n = C.c_uint64()
        N.check(self._lib.ssj_verify_chunk_results(self._h, _vp(chunk.C), nC, _vp(chunk.C_O),
                                                   chunk.C_O.size, _vp(slots), _vp(ovs), nC,
                                                   C.byref(n)))
        return slots[: n.value], ovs[: n.value]

    def set_original_ids(self, original_id: Optional[np.ndarray] = None) -> None:
        """Original input ids for verify_chunk_pairs (identity when None)."""
        oid = None if original_id is None else np.ascontiguousarray(original_id, np.uint32)
        N.check(self._lib.ssj_engine_set_original_ids(self._h, _vp(oid)))

    def verify_chunk_pairs(self, chunk: CandidateChunk, sorted_: bool = True,
                           stats: Optional[VerifyStats] = None) -> Tuple[np.ndarray, np.ndarray]:
        """Qualifying pairs decoded on the GPU: ((k, 2) uint32 (r_id, s_id) with r_id > s_id,
        in write_pairs order when sorted_), and their true overlaps."""
        nC = chunk.candidate_count()
        pairs = np.zeros(2 * max(nC, 1), np.uint32)
        ovs = np.zeros(max(nC, 1), np.uint32)
        n = C.c_uint64()
        st = N.ssj_stats()
        N.check(self._lib.ssj_verify_chunk_pairs(self._h, _vp(chunk.C), nC, _vp(chunk.C_O),
                                                 chunk.C_O.size, _vp(pairs), _vp(ovs), nC,
                                                 C.byref(n), int(sorted_), C.byref(st)))
        if stats is not None:
            stats.pairs_verified += st.pairs_verified
            stats.early_exit_prunes += st.early_exit_prunes
            stats.comparison_budget_violations += st.comparison_budget_violations
        return pairs[: 2 * n.value].reshape(-1, 2), ovs[: n.value]

    # -- candidate generation and the whole join on the GPU ----------------------------
    def gpu_generate_candidates(self, algorithm: int, probe_begin: int = 0,
                                probe_end: Optional[int] = None) -> CandidateChunk:
        """AllPairs / PPJoin candidates of probes [probe_begin, probe_end) generated on the
        device (the same stream as the reference generators), copied to the host."""
        probe_end = 0xFFFFFFFF if probe_end is None else probe_end
        nC, nCO = C.c_uint64(), C.c_uint64()
        rc = self._lib.ssj_gpu_generate_candidates(self._h, int(algorithm), probe_begin,
                                                   probe_end, None, 0, C.byref(nC), None, 0,
                                                   C.byref(nCO))
        if rc != N.SSJ_OK and not (nC.value or nCO.value):
            N.check(rc)
        Cs = np.zeros(max(nC.value, 1), np.uint32)
        COs = np.zeros(max(nCO.value, 1), np.uint32)
        N.check(self._lib.ssj_gpu_generate_candidates(self._h, int(algorithm), probe_begin,
                                                      probe_end, _vp(Cs), nC.value,
                                                      C.byref(nC), _vp(COs), nCO.value,
                                                      C.byref(nCO)))
        return CandidateChunk(Cs[: nC.value], COs[: nCO.value])

    def gpu_join(self, algorithm: int, max_chunk_candidates: int = 0, pairs: bool = True,
                 pairs_cap: int = 1 << 24, shard: int = 0, n_shards: int = 1):
        """Self-join (or shard `shard` of `n_shards` of it) entirely on the device. Returns
        (pairs (k, 2) uint32 in write_pairs order or None, report dict)."""
        rep = N.ssj_gpu_join_report()
        n = C.c_uint64()
        buf = np.zeros(2 * max(pairs_cap, 1), np.uint32) if pairs else None
        N.check(self._lib.ssj_gpu_join_shard(self._h, int(algorithm), shard, n_shards,
                                             max_chunk_candidates,
                                             _vp(buf) if pairs else None,
                                             pairs_cap if pairs else 0, C.byref(n),
                                             C.byref(rep)))
        out = {k: getattr(rep, k) for k, _ in rep._fields_}
        return (buf[: 2 * n.value].reshape(-1, 2) if pairs else None), out

    # -- device-resident (kernel-only) path --------------------------------------------
    def verify_chunk_device(self, d_C: int, nC: int, d_C_O: int, nCO: int, d_flags: int,
                            d_result: int, stream: int = 0) -> None:
        """Enqueue verification of a device-resident chunk on `stream` (cudaStream_t as
        int). d_result: device uint64[8] -> [count, error bits, stats...]."""
        N.check(self._lib.ssj_verify_chunk_device(self._h, C.c_void_p(d_C), nC,
                                                  C.c_void_p(d_C_O), nCO,
                                                  C.c_void_p(d_flags) if d_flags else None,
                                                  C.c_void_p(d_result),
                                                  C.c_void_p(stream) if stream else None))

    def set_profiling(self, enabled: bool) -> None:
        N.check(self._lib.ssj_engine_set_profiling(self._h, int(enabled)))

    def kernel_time(self) -> Tuple[float, int]:
        """(summed verification-kernel ms, launches) since the last call (profiling on)."""
        ms = C.c_double()
        n = C.c_uint64()
        N.check(self._lib.ssj_engine_kernel_time(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def export_collection(self, d_tokens: int, d_sets: int, stream: int = 0) -> None:
        N.check(self._lib.ssj_engine_export_collection(
            self._h, C.c_void_p(d_tokens), C.c_void_p(d_sets),
            C.c_void_p(stream) if stream else None))

    def launches_per_chunk(self, nC: int, nCO: int) -> int:
        return self._lib.ssj_launches_per_chunk(self._h, nC, nCO)

    def chunk_algorithmic_bytes_device(self, d_C: int, nC: int, d_C_O: int, nCO: int,
                                       d_bytes: int, stream: int = 0) -> None:
        N.check(self._lib.ssj_chunk_algorithmic_bytes_device(
            self._h, C.c_void_p(d_C), nC, C.c_void_p(d_C_O), nCO, C.c_void_p(d_bytes),
            C.c_void_p(stream) if stream else None))


def result_error(words) -> None:
    """Raise for the error bits of a device result block (ssj_verify_chunk_device)."""
    bits = int(words[1])
    if bits & 1:
        raise IndexError("set index out of range")
    if bits & 2:
        raise ValueError("malformed C_O: end offsets decreasing or beyond C")


def measure_read_bandwidth(device: int, nbytes: int, reps: int = 20) -> float:
    """Streaming read GB/s of an nbytes device buffer (diagnostic, see the C ABI)."""
    g = C.c_double()
    N.check(N.lib().ssj_measure_read_bandwidth(device, nbytes, reps, C.byref(g)))
    return g.value


def chunk_split(set_sizes: np.ndarray, parts: int, C_O: np.ndarray, nC: int) -> np.ndarray:
    """The probe-slice split a multi-device engine applies to a chunk (host only):
    (parts, 4) uint64 rows {first slice, end slice, first slot, end slot}."""
    sz = np.ascontiguousarray(np.asarray(set_sizes, np.uint32))
    co = np.ascontiguousarray(np.asarray(C_O, np.uint32))
    out = np.zeros(4 * parts, np.uint64)
    N.check(N.lib().ssj_chunk_split(sz.ctypes.data_as(N.u32p) if sz.size else None, sz.size,
                                    parts, co.ctypes.data_as(N.u32p) if co.size else None,
                                    co.size, nC, out.ctypes.data_as(N.u64p)))
    return out.reshape(parts, 4)


def device_count() -> int:
    return N.lib().ssj_device_count()


class PinnedBuffer:
    """Pinned host memory from ssj_host_alloc viewed as a numpy array."""

    def __init__(self, nbytes: int):
        self.ptr = N.lib().ssj_host_alloc(nbytes)
        if not self.ptr:
            raise MemoryError(N.last_error())
        self.nbytes = nbytes

    def view(self, dtype, count: int) -> np.ndarray:
        arr_t = C.c_uint8 * self.nbytes
        raw = np.frombuffer(arr_t.from_address(self.ptr), dtype=np.uint8)
        return raw.view(dtype)[:count]

    def close(self):
        if self.ptr:
            N.lib().ssj_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
