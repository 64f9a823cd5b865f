"""ctypes binding of the in-tree C-ABI library libssjoin_b200.so (include/ssjoin_b200.h).

The library is built in-tree by `make` (or __graft_entry__.build()). There is no fallback:
if the library is missing, importing the engine raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libssjoin_b200.so")

u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
u8p = C.POINTER(C.c_uint8)
vp = C.c_void_p

SSJ_OK = 0
SSJ_ERR_INVALID_ARGUMENT = 1
SSJ_ERR_OUT_OF_RANGE = 2
SSJ_ERR_CUDA = 3
SSJ_ERR_RUNTIME = 4
SSJ_ERR_NO_DEVICE = 5
SSJ_RESULT_WORDS = 8


class ssj_predicate(C.Structure):
    _fields_ = [("function", C.c_int32), ("reserved", C.c_uint32), ("num", C.c_uint64),
                ("den", C.c_uint64), ("overlap_threshold", C.c_uint64)]


class ssj_strategy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("group_size", C.c_uint32)]


class ssj_stats(C.Structure):
    _fields_ = [("pairs_verified", C.c_uint64), ("early_exit_prunes", C.c_uint64),
                ("comparison_budget_violations", C.c_uint64)]


class ssj_synth_config(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_sets", C.c_uint32), ("min_size", C.c_uint32),
                ("max_size", C.c_uint32), ("zipf_sizes", C.c_int32), ("size_skew", C.c_double),
                ("universe", C.c_uint32), ("zipf_tokens", C.c_int32), ("token_skew", C.c_double),
                ("duplicate_fraction", C.c_double), ("max_edits", C.c_uint32),
                ("distinct_tokens", C.c_int32), ("threads", C.c_uint32)]


OBSERVER = C.CFUNCTYPE(None, C.c_void_p, u32p, C.c_uint64, u32p, C.c_uint64, u8p, C.c_uint64)


class ssj_join_config(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("mode", C.c_int32), ("chunk_budget", C.c_uint64),
                ("strategy", ssj_strategy), ("workers", C.c_uint32), ("device", C.c_int32),
                ("filter_threads", C.c_uint32), ("reserved", C.c_uint32),
                ("observer", OBSERVER), ("observer_user", C.c_void_p),
                ("devices", C.POINTER(C.c_int32)), ("n_devices", C.c_uint32),
                ("max_inflight", C.c_uint32)]


class ssj_join_report(C.Structure):
    _fields_ = [("count", C.c_uint64), ("chunk_count", C.c_uint64),
                ("candidate_count", C.c_uint64), ("host_verified_pairs", C.c_uint64),
                ("max_live_candidate_bytes", C.c_uint64), ("pairs_verified", C.c_uint64),
                ("early_exit_prunes", C.c_uint64), ("comparison_budget_violations", C.c_uint64),
                ("n_pairs", C.c_uint64), ("resolved_strategy", ssj_strategy),
                ("filtering_ms", C.c_double), ("serialization_ms", C.c_double),
                ("verification_ms", C.c_double), ("join_ms", C.c_double),
                ("handoff_wait_ms", C.c_double), ("setup_ms", C.c_double)]


class ssj_gpu_join_report(C.Structure):
    _fields_ = [("count", C.c_uint64), ("candidate_count", C.c_uint64),
                ("intra_group_pairs", C.c_uint64),
                ("chunk_count", C.c_uint64), ("index_ms", C.c_double),
                ("filtering_ms", C.c_double), ("verification_ms", C.c_double),
                ("join_ms", C.c_double)]


# name -> (restype, argtypes); every symbol declared in include/ssjoin_b200.h
SIGNATURES = {
    "ssj_abi_version": (C.c_int, []),
    "ssj_last_error": (C.c_char_p, []),
    "ssj_device_count": (C.c_int, []),
    "ssj_threshold_parse": (C.c_int, [C.c_char_p, u64p, u64p]),
    "ssj_predicate_validate": (C.c_int, [C.POINTER(ssj_predicate)]),
    "ssj_strategy_validate": (C.c_int, [C.POINTER(ssj_strategy)]),
    "ssj_equivalent_overlap": (C.c_uint64, [C.POINTER(ssj_predicate), C.c_uint64, C.c_uint64]),
    "ssj_engine_create": (C.c_int, [C.POINTER(vp), C.c_int, u32p, u32p, C.c_uint32,
                                    C.POINTER(ssj_predicate), C.c_int32,
                                    C.POINTER(ssj_strategy)]),
    "ssj_engine_create_from_device": (C.c_int, [C.POINTER(vp), C.c_int, vp, C.c_uint64, vp,
                                                C.c_uint32, C.c_uint64, C.POINTER(ssj_predicate),
                                                C.c_int32, C.POINTER(ssj_strategy)]),
    "ssj_engine_create_multi": (C.c_int, [C.POINTER(vp), C.POINTER(C.c_int32), C.c_uint32, u32p,
                                          u32p, C.c_uint32, C.POINTER(ssj_predicate), C.c_int32,
                                          C.POINTER(ssj_strategy)]),
    "ssj_engine_devices": (C.c_int, [vp, C.POINTER(C.c_int32), C.c_uint32, C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_double)]),
    "ssj_chunk_split": (C.c_int, [u32p, C.c_uint32, C.c_uint32, u32p, C.c_uint64, C.c_uint64,
                                  u64p]),
    "ssj_engine_device_collection": (C.c_int, [vp, C.POINTER(vp), u64p, C.POINTER(vp)]),
    "ssj_engine_destroy": (None, [vp]),
    "ssj_engine_strategy": (C.c_int, [vp, C.POINTER(ssj_strategy)]),
    "ssj_engine_kernel_strategy": (C.c_int, [vp, C.POINTER(ssj_strategy)]),
    "ssj_engine_device": (C.c_int, [vp]),
    "ssj_verify_chunk": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, u64p,
                                   C.POINTER(ssj_stats)]),
    "ssj_submit_chunk": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, u64p]),
    "ssj_wait_chunk": (C.c_int, [vp, C.c_uint64, u64p, C.POINTER(ssj_stats)]),
    "ssj_verify_chunk_results": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp,
                                           C.c_uint64, u64p]),
    "ssj_engine_set_original_ids": (C.c_int, [vp, vp]),
    "ssj_verify_chunk_pairs": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp, C.c_uint64,
                                         u64p, C.c_int, C.POINTER(ssj_stats)]),
    "ssj_verify_chunk_device": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp]),
    "ssj_launches_per_chunk": (C.c_int, [vp, C.c_uint64, C.c_uint64]),
    "ssj_engine_set_profiling": (C.c_int, [vp, C.c_int]),
    "ssj_engine_kernel_time": (C.c_int, [vp, C.POINTER(C.c_double), u64p]),
    "ssj_engine_export_collection": (C.c_int, [vp, vp, vp, vp]),
    "ssj_chunk_algorithmic_bytes_device": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp,
                                                     vp]),
    "ssj_generate_candidates": (C.c_int, [u32p, u32p, C.c_uint32, C.POINTER(ssj_predicate),
                                          C.c_int32, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.POINTER(vp)]),
    "ssj_generate_candidates_windows": (C.c_int, [u32p, u32p, C.c_uint32,
                                                  C.POINTER(ssj_predicate), C.c_int32, u32p,
                                                  C.c_uint32, C.c_uint32, C.POINTER(vp)]),
    "ssj_candidates_sizes": (C.c_int, [vp, u64p, u64p, u64p]),
    "ssj_candidates_copy": (C.c_int, [vp, vp, vp, vp]),
    "ssj_candidates_free": (None, [vp]),
    "ssj_synth_collection": (C.c_int, [C.POINTER(ssj_synth_config), C.POINTER(vp)]),
    "ssj_preprocess_precoded": (C.c_int, [vp, vp, C.c_uint64, C.POINTER(vp)]),
    "ssj_collection_sizes": (C.c_int, [vp, u64p, u64p, u64p]),
    "ssj_collection_copy": (C.c_int, [vp, vp, vp, vp]),
    "ssj_collection_free": (None, [vp]),
    "ssj_join_config_init": (None, [C.POINTER(ssj_join_config)]),
    "ssj_run_join": (C.c_int, [u32p, u32p, C.c_uint32, u32p, C.POINTER(ssj_predicate),
                               C.POINTER(ssj_join_config), C.POINTER(vp)]),
    "ssj_join_result_report": (C.c_int, [vp, C.POINTER(ssj_join_report)]),
    "ssj_join_result_pairs": (C.c_int, [vp, vp]),
    "ssj_join_result_free": (None, [vp]),
    "ssj_gpu_generate_candidates": (C.c_int, [vp, C.c_int32, C.c_uint32, C.c_uint32, vp,
                                              C.c_uint64, u64p, vp, C.c_uint64, u64p]),
    "ssj_gpu_join": (C.c_int, [vp, C.c_int32, C.c_uint64, vp, C.c_uint64, u64p,
                               C.POINTER(ssj_gpu_join_report)]),
    "ssj_gpu_join_shard": (C.c_int, [vp, C.c_int32, C.c_uint32, C.c_uint32, C.c_uint64, vp,
                                     C.c_uint64, u64p, C.POINTER(ssj_gpu_join_report)]),
    "ssj_measure_read_bandwidth": (C.c_int, [C.c_int, C.c_uint64, C.c_uint32,
                                             C.POINTER(C.c_double)]),
    "ssj_host_alloc": (vp, [C.c_size_t]),
    "ssj_host_free": (None, [vp]),
}

_lib = None


def lib():
    """Load libssjoin_b200.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
                "the B200 engine has no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().ssj_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    """Map an ssj_status to the reference's exception classes."""
    if rc == SSJ_OK:
        return
    msg = last_error()
    if rc == SSJ_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)        # std::invalid_argument
    if rc == SSJ_ERR_OUT_OF_RANGE:
        raise IndexError(msg)        # std::out_of_range
    raise RuntimeError(f"ssjoin_b200 error {rc}: {msg}")
