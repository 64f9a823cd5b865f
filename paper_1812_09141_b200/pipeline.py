"""The join driver and the host-side producers (mirror of pipeline.hpp and joiners.hpp).

run_join(collection, pred, config) -> JoinReport runs the reference's three roles natively
(C++ in libssjoin_b200.so): H0 generation + serialization into pinned chunks, H1 GPU
verification, H2 pair decoding.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Callable, Optional, Tuple, Sequence

import numpy as np

from . import _native as N
from .collection import CandidateChunk, Collection
from .similarity import SimilarityPredicate
from .verify import OutputMode, Strategy, StrategyKind, VerificationOutput


FILTER_ON_GPU = 0xFFFFFFFF  # PipelineConfig.filter_threads: generate candidates on the device


class Algorithm(IntEnum):
    """pipeline.hpp:25"""
    AllPairs = 0
    PPJoin = 1
    GroupJoin = 2


@dataclass
class PipelineConfig:
    """pipeline.hpp:36-51 (+ device, filter_threads)."""
    algorithm: Algorithm = Algorithm.PPJoin
    chunk_budget: int = 64 << 20
    strategy: Strategy = field(default_factory=Strategy)
    mode: OutputMode = OutputMode.Count
    workers: int = 1
    chunk_observer: Optional[Callable[[CandidateChunk, VerificationOutput], None]] = None
    device: int = 0
    filter_threads: int = 1  # FILTER_ON_GPU: candidate generation on the device too
    devices: Optional[Sequence[int]] = None  # several GPUs behind the engine (probe-slice split)
    max_inflight: int = 1    # chunks the dispatcher keeps on the GPU (1 = the reference's)


@dataclass
class PhaseTimings:
    """pipeline.hpp:53-58 (+ handoff_wait_ms, setup_ms)."""
    filtering_ms: float = 0.0
    serialization_ms: float = 0.0
    verification_ms: float = 0.0
    join_ms: float = 0.0
    handoff_wait_ms: float = 0.0
    setup_ms: float = 0.0


@dataclass
class JoinReport:
    """pipeline.hpp:63-75. `pairs` is an (n, 2) uint32 array of (r_id, s_id), r_id > s_id."""
    count: int = 0
    pairs: np.ndarray = field(default_factory=lambda: np.zeros((0, 2), np.uint32))
    timings: PhaseTimings = field(default_factory=PhaseTimings)
    chunk_count: int = 0
    candidate_count: int = 0
    host_verified_pairs: int = 0
    max_live_candidate_bytes: int = 0
    pairs_verified: int = 0
    early_exit_prunes: int = 0
    comparison_budget_violations: int = 0
    resolved_strategy: Strategy = field(default_factory=Strategy)


def _u32p(a: np.ndarray):
    return a.ctypes.data_as(N.u32p)


def run_join(collection: Collection, pred: SimilarityPredicate,
             config: Optional[PipelineConfig] = None) -> JoinReport:
    """pipeline.hpp:150-361 on the GPU (raises like the reference on bad configs)."""
    config = config or PipelineConfig()
    L = N.lib()
    cfg = N.ssj_join_config()
    L.ssj_join_config_init(C.byref(cfg))
    cfg.algorithm = int(config.algorithm)
    cfg.mode = int(config.mode)
    cfg.chunk_budget = min(int(config.chunk_budget), (1 << 64) - 1)
    cfg.strategy = N.ssj_strategy(int(config.strategy.kind), config.strategy.group_size)
    cfg.workers = max(0, int(config.workers))
    cfg.device = config.device
    cfg.filter_threads = config.filter_threads
    cfg.max_inflight = config.max_inflight
    devs = None
    if config.devices is not None:
        devs = (C.c_int32 * len(config.devices))(*config.devices)
        cfg.devices = C.cast(devs, C.POINTER(C.c_int32))
        cfg.n_devices = len(config.devices)
    errors = []
    if config.chunk_observer is not None:
        def _obs(user, Cp, nC, COp, nCO, flagsp, count):
            try:
                c_arr = np.ctypeslib.as_array(Cp, (nC,)).copy() if nC else np.zeros(0, np.uint32)
                co_arr = np.ctypeslib.as_array(COp, (nCO,)).copy() if nCO else np.zeros(0, np.uint32)
                fl = (np.ctypeslib.as_array(flagsp, (nC,)).copy() if (flagsp and nC)
                      else np.zeros(0, np.uint8))
                config.chunk_observer(CandidateChunk(c_arr, co_arr), VerificationOutput(fl, count))
            except Exception as e:  # surfaced after the join
                errors.append(e)
        cb = N.OBSERVER(_obs)
        cfg.observer = cb
    p = pred._c()
    tokens = collection.tokens if collection.tokens.size else np.zeros(1, np.uint32)
    oid = collection.original_id if collection.original_id.size else np.zeros(1, np.uint32)
    h = C.c_void_p()
    N.check(L.ssj_run_join(_u32p(tokens), _u32p(collection.offsets), collection.size(),
                           _u32p(oid) if collection.original_id.size else None, C.byref(p),
                           C.byref(cfg), C.byref(h)))
    try:
        rep = N.ssj_join_report()
        N.check(L.ssj_join_result_report(h, C.byref(rep)))
        pairs = np.zeros(2 * max(rep.n_pairs, 1), np.uint32)
        N.check(L.ssj_join_result_pairs(h, C.c_void_p(pairs.ctypes.data)))
    finally:
        L.ssj_join_result_free(h)
    if errors:
        raise errors[0]
    return JoinReport(
        count=rep.count, pairs=pairs[: 2 * rep.n_pairs].reshape(-1, 2),
        timings=PhaseTimings(rep.filtering_ms, rep.serialization_ms, rep.verification_ms,
                             rep.join_ms, rep.handoff_wait_ms, rep.setup_ms),
        chunk_count=rep.chunk_count, candidate_count=rep.candidate_count,
        host_verified_pairs=rep.host_verified_pairs,
        max_live_candidate_bytes=rep.max_live_candidate_bytes,
        pairs_verified=rep.pairs_verified, early_exit_prunes=rep.early_exit_prunes,
        comparison_budget_violations=rep.comparison_budget_violations,
        resolved_strategy=Strategy(StrategyKind(rep.resolved_strategy.kind),
                                   rep.resolved_strategy.group_size))


def sorted_pairs(pairs: np.ndarray) -> np.ndarray:
    """report.hpp:39-42 write_pairs order."""
    if len(pairs) == 0:
        return pairs.reshape(-1, 2)
    return pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]


def write_pairs(pairs: np.ndarray) -> str:
    """report.hpp:39-42: "r_id\\ts_id\\n" lines, sorted."""
    return "".join(f"{a}\t{b}\n" for a, b in sorted_pairs(pairs))


def generate_candidates(collection: Collection, pred: SimilarityPredicate,
                        algorithm: Algorithm = Algorithm.PPJoin, probe_begin: int = 0,
                        probe_end: Optional[int] = None, threads: int = 0
                        ) -> Tuple[CandidateChunk, np.ndarray]:
    """The reference generators' candidate stream (joiners.hpp:47-183) for probes
    [probe_begin, probe_end) as one unbounded chunk, plus GroupJoin's intra-group host pairs
    (k, 2). threads == 1 (or GroupJoin) runs the reference's sequential loop."""
    L = N.lib()
    n = collection.size()
    probe_end = n if probe_end is None else probe_end
    p = pred._c()
    tokens = collection.tokens if collection.tokens.size else np.zeros(1, np.uint32)
    h = C.c_void_p()
    N.check(L.ssj_generate_candidates(_u32p(tokens), _u32p(collection.offsets), n, C.byref(p),
                                      int(algorithm), probe_begin, probe_end, threads,
                                      C.byref(h)))
    return _take_candidates(h)


def generate_candidates_windows(collection: Collection, pred: SimilarityPredicate,
                                algorithm: Algorithm, windows, threads: int = 0) -> CandidateChunk:
    """Probe windows [(lo, hi), ...] concatenated into one chunk (one shared static index)."""
    L = N.lib()
    w = np.ascontiguousarray(np.asarray(windows, np.uint32).reshape(-1))
    p = pred._c()
    tokens = collection.tokens if collection.tokens.size else np.zeros(1, np.uint32)
    h = C.c_void_p()
    N.check(L.ssj_generate_candidates_windows(_u32p(tokens), _u32p(collection.offsets),
                                              collection.size(), C.byref(p), int(algorithm),
                                              _u32p(w), w.size // 2, threads, C.byref(h)))
    return _take_candidates(h)[0]


def _take_candidates(h):
    L = N.lib()
    try:
        nC, nCO, nH = C.c_uint64(), C.c_uint64(), C.c_uint64()
        N.check(L.ssj_candidates_sizes(h, C.byref(nC), C.byref(nCO), C.byref(nH)))
        Carr = np.zeros(max(nC.value, 1), np.uint32)
        COarr = np.zeros(max(nCO.value, 1), np.uint32)
        H = np.zeros(2 * max(nH.value, 1), np.uint32)
        N.check(L.ssj_candidates_copy(h, C.c_void_p(Carr.ctypes.data),
                                      C.c_void_p(COarr.ctypes.data), C.c_void_p(H.ctypes.data)))
    finally:
        L.ssj_candidates_free(h)
    return (CandidateChunk(Carr[: nC.value], COarr[: nCO.value]),
            H[: 2 * nH.value].reshape(-1, 2))


def _take_collection(h) -> Collection:
    L = N.lib()
    try:
        n, t, d = C.c_uint64(), C.c_uint64(), C.c_uint64()
        N.check(L.ssj_collection_sizes(h, C.byref(n), C.byref(t), C.byref(d)))
        tokens = np.zeros(max(t.value, 1), np.uint32)
        offsets = np.zeros(n.value + 1, np.uint32)
        oid = np.zeros(max(n.value, 1), np.uint32)
        N.check(L.ssj_collection_copy(h, C.c_void_p(tokens.ctypes.data),
                                      C.c_void_p(offsets.ctypes.data),
                                      C.c_void_p(oid.ctypes.data)))
    finally:
        L.ssj_collection_free(h)
    c = Collection(tokens[: t.value], offsets, oid[: n.value])
    c.dropped_empty = d.value
    return c


@dataclass
class SynthConfig:
    """Synthetic workload knobs (oracle.hpp:71-81 + near-duplicates, distinct draws)."""
    sets: int = 100
    min_size: int = 1
    max_size: int = 50
    zipf_sizes: bool = False
    size_skew: float = 1.0
    universe: int = 1000
    zipf_tokens: bool = False
    token_skew: float = 1.0
    duplicate_fraction: float = 0.0
    max_edits: int = 0
    distinct_tokens: bool = False
    threads: int = 0


def synth_collection(seed: int, cfg: SynthConfig) -> Collection:
    """Deterministic synthetic collection, preprocessed like preprocess_precoded."""
    c = N.ssj_synth_config(seed, cfg.sets, cfg.min_size, cfg.max_size, int(cfg.zipf_sizes),
                           cfg.size_skew, cfg.universe, int(cfg.zipf_tokens), cfg.token_skew,
                           cfg.duplicate_fraction, cfg.max_edits, int(cfg.distinct_tokens),
                           cfg.threads)
    h = C.c_void_p()
    N.check(N.lib().ssj_synth_collection(C.byref(c), C.byref(h)))
    return _take_collection(h)


def preprocess_precoded_native(records) -> Collection:
    """collection.hpp:134-168 in C++ (records: sequence of integer sequences)."""
    lens = [len(r) for r in records]
    offs = np.zeros(len(records) + 1, np.uint64)
    offs[1:] = np.cumsum(lens)
    toks = (np.concatenate([np.asarray(r, np.uint32) for r in records]) if sum(lens)
            else np.zeros(1, np.uint32))
    h = C.c_void_p()
    N.check(N.lib().ssj_preprocess_precoded(C.c_void_p(toks.ctypes.data),
                                            C.c_void_p(offs.ctypes.data), len(records),
                                            C.byref(h)))
    return _take_collection(h)
