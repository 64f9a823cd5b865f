"""Multi-GPU plumbing: one process per GPU, probe-sharded weak scaling.

Verification has no exchange step: every candidate pair is independent and a probe slice only
reads the read-only collection. The one collective is the one-time broadcast of the padded
device collection from rank 0 over NVLink (NCCL); chunks are then sharded by probe windows.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


TOKEN_TAIL_PAD = 512  # SSJ_TOKEN_TAIL_PAD (include/ssjoin_b200.h)


def padded_layout(offsets: np.ndarray) -> Tuple[int, np.ndarray]:
    """The engine's device layout (engine.cu, ssj_engine_create): set i starts at token
    8 * pos8[i] (32-byte aligned), padded to a multiple of 8 tokens, plus TOKEN_TAIL_PAD
    sentinel tokens.
    Returns (n_padded_tokens, sets) with sets = uint32[2n] of (pos8, size) pairs."""
    offsets = np.asarray(offsets, np.int64)
    sizes = np.diff(offsets)
    padded = (sizes + 7) // 8 * 8
    pos = np.zeros(sizes.size, np.int64)
    if sizes.size:
        pos[1:] = np.cumsum(padded)[:-1]
    sets = np.stack([pos // 8, sizes], 1).astype(np.uint32).reshape(-1)
    return int(padded.sum()) + TOKEN_TAIL_PAD, sets


def padded_tokens(tokens: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Host copy of the padded token array (0xFFFFFFFF padding) matching padded_layout."""
    n_pad, sets = padded_layout(offsets)
    out = np.full(n_pad, 0xFFFFFFFF, np.uint32)
    offsets = np.asarray(offsets, np.int64)
    pos8 = sets[0::2].astype(np.int64)
    sizes = sets[1::2].astype(np.int64)
    # scatter every set: index of token k of set i = 8*pos8[i] + (k - offsets[i])
    if tokens.size:
        set_of = np.repeat(np.arange(sizes.size), sizes)
        within = np.arange(tokens.size) - np.repeat(offsets[:-1], sizes)
        out[8 * pos8[set_of] + within] = tokens
    return out


def shard_probe_windows(n_sets: int, windows: int, width: int, rank: int,
                        world: int) -> List[Tuple[int, int]]:
    """Stratified probe windows for `rank`: the collection is cut into `windows` strides and
    each rank takes its own `width`-wide window inside every stride, so every rank gets the
    same mix of set sizes (weak scaling) and no probe is verified twice."""
    stride = n_sets // windows
    width = min(width, stride // max(world, 1))
    return [(k * stride + rank * width, min(k * stride + rank * width + width, n_sets))
            for k in range(windows)]


def broadcast_device_collection(engine, n_sets: int, n_tokens: int, offsets: np.ndarray,
                                pred, mode, strategy, device: int, rank: int):
    """Rank 0 exports its engine's padded collection into device tensors and NCCL-broadcasts
    them; every other rank builds its engine on the received buffers. Returns
    (engine, keepalive_tensors)."""
    import torch
    import torch.distributed as dist

    from .verify import VerificationEngine

    n_pad, _ = padded_layout(offsets)
    dev = torch.device("cuda", device)
    d_tok = torch.empty(n_pad, dtype=torch.int32, device=dev)
    d_sets = torch.empty(2 * max(n_sets, 1), dtype=torch.int32, device=dev)
    if rank == 0:
        engine.export_collection(d_tok.data_ptr(), d_sets.data_ptr(),
                                 torch.cuda.current_stream(dev).cuda_stream)
        torch.cuda.synchronize(dev)
    dist.broadcast(d_tok, 0)
    dist.broadcast(d_sets, 0)
    torch.cuda.synchronize(dev)
    if rank == 0:
        return engine, (d_tok, d_sets)
    eng = VerificationEngine.from_device(d_tok.data_ptr(), n_pad, d_sets.data_ptr(), n_sets,
                                         n_tokens, pred, mode, strategy, device=device)
    return eng, (d_tok, d_sets)
