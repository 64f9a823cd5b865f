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
    "ssj_engine_device_collection": (C.c_int, [vp, C.POINTER(vp), u64p, C.POINTER(vp)]),
    "ssj_engine_destroy": (None, [vp]),
    "ssj_engine_strategy": (C.c_int, [vp, C.POINTER(ssj_strategy)]),
    "ssj_engine_device": (C.c_int, [vp]),
    "ssj_verify_chunk": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, u64p,
                                   C.POINTER(ssj_stats)]),
    "ssj_submit_chunk": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, u64p]),
    "ssj_wait_chunk": (C.c_int, [vp, C.c_uint64, u64p, C.POINTER(ssj_stats)]),
    "ssj_verify_chunk_results": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp,
                                           C.c_uint64, u64p]),
    "ssj_verify_chunk_device": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp]),
    "ssj_launches_per_chunk": (C.c_int, [vp, C.c_uint64, C.c_uint64]),
    "ssj_chunk_algorithmic_bytes_device": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp,
                                                     vp]),
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
