"""Similarity predicates (mirror of proj/include/ssjoin/similarity.hpp).

Exact rational thresholds; the arithmetic is done by the C ABI (the same code path the
kernels' host side uses), never in floating point.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

from . import _native as N


class SimilarityFunction(IntEnum):
    """similarity.hpp:11"""
    Jaccard = 0
    Cosine = 1
    Dice = 2
    Overlap = 3


@dataclass
class Threshold:
    """similarity.hpp:26-65: normalized threshold kept as num/den."""
    num: int = 1
    den: int = 1

    @staticmethod
    def parse(text: str) -> "Threshold":
        """similarity.hpp:30-56: "0.8", ".85", "1", "1.0", "4/5" (reduced)."""
        n, d = C.c_uint64(), C.c_uint64()
        N.check(N.lib().ssj_threshold_parse(text.encode(), C.byref(n), C.byref(d)))
        return Threshold(n.value, d.value)

    def reduce(self) -> None:
        """similarity.hpp:58-62"""
        a, b = self.num, self.den
        while b:
            a, b = b, a % b
        if a > 1:
            self.num //= a
            self.den //= a

    def value(self) -> float:
        return self.num / self.den


@dataclass
class SimilarityPredicate:
    """similarity.hpp:67-82"""
    function: SimilarityFunction = SimilarityFunction.Jaccard
    threshold: Threshold = field(default_factory=Threshold)
    overlap_threshold: int = 1

    def normalized(self) -> bool:
        return self.function != SimilarityFunction.Overlap

    def _c(self) -> N.ssj_predicate:
        return N.ssj_predicate(int(self.function), 0, self.threshold.num, self.threshold.den,
                               self.overlap_threshold)

    def validate(self) -> None:
        """similarity.hpp:74-81 (raises ValueError like std::invalid_argument)."""
        p = self._c()
        N.check(N.lib().ssj_predicate_validate(C.byref(p)))


def jaccard(num: int, den: int) -> SimilarityPredicate:
    """tests/helpers.hpp:31-37"""
    t = Threshold(num, den)
    t.reduce()
    return SimilarityPredicate(SimilarityFunction.Jaccard, t)


def equivalent_overlap(pred: SimilarityPredicate, size_r: int, size_s: int) -> int:
    """similarity.hpp:108-123 (exact, u128)."""
    p = pred._c()
    return int(N.lib().ssj_equivalent_overlap(C.byref(p), size_r, size_s))
