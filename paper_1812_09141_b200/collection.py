"""Collection and candidate-chunk containers (mirror of collection.hpp and chunk.hpp).

Host-side data only (numpy arrays in the reference's exact CSR / C / C_O layouts); the
device layout is built by the engine (include/ssjoin_b200.h, ssj_engine_create).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, NamedTuple, Sequence

import numpy as np

KUNBOUNDED_BUDGET = (1 << 64) - 1  # chunk.hpp:13 kUnboundedBudget


@dataclass
class Collection:
    """collection.hpp:76-94: tokens u32, offsets u32[n+1], original_id u32[n]."""
    tokens: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    offsets: np.ndarray = field(default_factory=lambda: np.zeros(1, np.uint32))
    original_id: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    dropped_empty: int = 0

    def __post_init__(self):
        self.tokens = np.ascontiguousarray(self.tokens, dtype=np.uint32)
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.uint32)
        self.original_id = np.ascontiguousarray(self.original_id, dtype=np.uint32)

    def size(self) -> int:
        return int(self.offsets.size) - 1

    def set_size(self, i: int) -> int:
        return int(self.offsets[i + 1]) - int(self.offsets[i])

    def set_view(self, i: int) -> np.ndarray:
        """collection.hpp:86-89 (raises IndexError like std::out_of_range)."""
        if i < 0 or i >= self.size():
            raise IndexError("set index out of range")
        return self.tokens[self.offsets[i]:self.offsets[i + 1]]

    def average_set_size(self) -> int:
        """collection.hpp:91-93 (integer division)."""
        return int(self.tokens.size) // self.size() if self.size() else 0

    @staticmethod
    def from_sets(sets: Sequence[Sequence[int]]) -> "Collection":
        """tests/helpers.hpp:15-23: verbatim, original_id = position."""
        sizes = [len(s) for s in sets]
        offsets = np.zeros(len(sets) + 1, np.uint32)
        offsets[1:] = np.cumsum(sizes, dtype=np.uint64).astype(np.uint32)
        tokens = (np.concatenate([np.asarray(s, np.uint32) for s in sets])
                  if sets and sum(sizes) else np.zeros(0, np.uint32))
        return Collection(tokens, offsets, np.arange(len(sets), dtype=np.uint32))


def preprocess_precoded(records: Sequence[Sequence[int]]) -> Collection:
    """collection.hpp:134-168: per-set dedup + sort, drop empties, order sets by
    (size, lexicographic, input line)."""
    sets = []
    dropped = 0
    for line, rec in enumerate(records):
        coded = sorted(set(int(t) for t in rec))
        if not coded:
            dropped += 1
            continue
        sets.append((len(coded), coded, line))
    sets.sort()
    c = Collection.from_sets([s[1] for s in sets])
    c.original_id = np.array([s[2] for s in sets], np.uint32)
    c.dropped_empty = dropped
    return c


@dataclass
class CandidateChunk:
    """chunk.hpp:20-28: C = candidate set indices, C_O = (probe, cumulative end) pairs."""
    C: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    C_O: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))

    def __post_init__(self):
        self.C = np.ascontiguousarray(self.C, dtype=np.uint32)
        self.C_O = np.ascontiguousarray(self.C_O, dtype=np.uint32)

    def candidate_count(self) -> int:
        return int(self.C.size)

    def byte_size(self) -> int:
        return 4 * int(self.C.size) + 4 * int(self.C_O.size)


class DecodedSlice(NamedTuple):
    probe: int
    begin: int
    candidates: np.ndarray


def decode(chunk: CandidateChunk) -> List[DecodedSlice]:
    """chunk.hpp:36-48"""
    out, prev = [], 0
    for e in range(0, chunk.C_O.size - 1, 2):
        end = int(chunk.C_O[e + 1])
        out.append(DecodedSlice(int(chunk.C_O[e]), prev, chunk.C[prev:end]))
        prev = end
    return out


class ChunkBuilder:
    """chunk.hpp:52-93: accumulates batches until the M_c byte budget."""
    kEntryBytes = 8
    kCandidateBytes = 4
    kMinBudget = kEntryBytes + kCandidateBytes

    def __init__(self, budget: int = KUNBOUNDED_BUDGET):
        assert budget >= self.kMinBudget
        self._budget = budget
        self._C: List[np.ndarray] = []
        self._CO: List[int] = []
        self._n = 0

    def byte_size(self) -> int:
        return 4 * self._n + 4 * len(self._CO)

    def capacity(self) -> int:
        used = self.byte_size()
        if used + self.kEntryBytes > self._budget:
            return 0
        return (self._budget - used - self.kEntryBytes) // self.kCandidateBytes

    def entry_fits(self) -> bool:
        return self.byte_size() + self.kEntryBytes <= self._budget

    def append(self, probe: int, candidates) -> None:
        cands = np.asarray(candidates, np.uint32)
        self._C.append(cands)
        self._n += int(cands.size)
        self._CO += [int(probe), self._n]

    def empty(self) -> bool:
        return not self._CO

    def budget(self) -> int:
        return self._budget

    def seal(self) -> CandidateChunk:
        assert not self.empty()
        C = np.concatenate(self._C) if self._C else np.zeros(0, np.uint32)
        chunk = CandidateChunk(C, np.array(self._CO, np.uint32))
        self._C, self._CO, self._n = [], [], 0
        return chunk
