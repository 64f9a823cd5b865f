"""B200-native verification phase of exact set-similarity self-joins (arXiv 1812.09141).

Public surface mirrors the reference (proj/include/ssjoin/):
  similarity.hpp -> SimilarityFunction, Threshold, SimilarityPredicate, equivalent_overlap
  collection.hpp -> Collection, preprocess_precoded
  chunk.hpp      -> CandidateChunk, ChunkBuilder, decode
  verify.hpp     -> StrategyKind, Strategy, OutputMode, VerificationOutput, VerifyStats,
                    VerificationEngine (sm_100a kernels behind include/ssjoin_b200.h)
"""
from .collection import (KUNBOUNDED_BUDGET, CandidateChunk, ChunkBuilder, Collection,
                         DecodedSlice, decode, preprocess_precoded)
from .similarity import (SimilarityFunction, SimilarityPredicate, Threshold,
                         equivalent_overlap, jaccard)
from .verify import (OutputMode, PinnedBuffer, Strategy, StrategyKind, VerificationEngine,
                     VerificationOutput, VerifyStats, device_count, result_error)

__all__ = [
    "KUNBOUNDED_BUDGET", "CandidateChunk", "ChunkBuilder", "Collection", "DecodedSlice",
    "decode", "preprocess_precoded", "SimilarityFunction", "SimilarityPredicate", "Threshold",
    "equivalent_overlap", "jaccard", "OutputMode", "PinnedBuffer", "Strategy", "StrategyKind",
    "VerificationEngine", "VerificationOutput", "VerifyStats", "device_count", "result_error",
]
