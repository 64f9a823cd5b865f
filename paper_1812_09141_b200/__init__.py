"""B200-native verification phase of exact set-similarity self-joins (arXiv 1812.09141).

Public surface mirrors the reference (proj/include/ssjoin/):
  similarity.hpp -> SimilarityFunction, Threshold, SimilarityPredicate, equivalent_overlap
  collection.hpp -> Collection, preprocess_precoded
  chunk.hpp      -> CandidateChunk, ChunkBuilder, decode
  pipeline.hpp   -> Algorithm, PipelineConfig, JoinReport, run_join (H0/H1/H2 natively)
  joiners.hpp    -> generate_candidates (identical streams; parallel AllPairs/PPJoin)
  verify.hpp     -> StrategyKind, Strategy, OutputMode, VerificationOutput, VerifyStats,
                    VerificationEngine (sm_100a kernels behind include/ssjoin_b200.h)
"""
from .collection import (KUNBOUNDED_BUDGET, CandidateChunk, ChunkBuilder, Collection,
                         DecodedSlice, decode, preprocess_precoded)
from .similarity import (SimilarityFunction, SimilarityPredicate, Threshold,
                         equivalent_overlap, jaccard)
from .pipeline import (FILTER_ON_GPU, Algorithm, JoinReport, PhaseTimings, PipelineConfig, SynthConfig,
                       generate_candidates, generate_candidates_windows, preprocess_precoded_native, run_join, sorted_pairs,
                       synth_collection, write_pairs)
from .verify import (OutputMode, PinnedBuffer, Strategy, StrategyKind, VerificationEngine,
                     VerificationOutput, VerifyStats, device_count, result_error)

__all__ = [
    "KUNBOUNDED_BUDGET", "CandidateChunk", "ChunkBuilder", "Collection", "DecodedSlice",
    "decode", "preprocess_precoded", "SimilarityFunction", "SimilarityPredicate", "Threshold",
    "equivalent_overlap", "jaccard", "OutputMode", "PinnedBuffer", "Strategy", "StrategyKind",
    "VerificationEngine", "VerificationOutput", "VerifyStats", "device_count", "result_error",
    "Algorithm", "JoinReport", "PhaseTimings", "PipelineConfig", "SynthConfig",
    "generate_candidates", "generate_candidates_windows", "preprocess_precoded_native", "run_join", "sorted_pairs",
    "synth_collection", "write_pairs",
]
