"""The C-ABI library (CPU-side checks): it loads, exports every symbol include/ssjoin_b200.h
declares, its host-side arithmetic matches the reference's golden vectors, and without a
GPU it refuses to verify (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ssjoin_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ssj_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(ssj):
    from paper_1812_09141_b200 import _native
    L = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_native.SIGNATURES), "python binding out of sync with the header"
    assert L.ssj_abi_version() == 1


def test_library_is_sm100a(ssj):
    """The fatbin carries sm_100a SASS (cuobjdump)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    from paper_1812_09141_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_threshold_parse(ssj):
    g = golden("similarity")
    for text, (n, d) in zip(g["parse_in"], g["parse_out"]):
        t = ssj.Threshold.parse(str(text))
        assert (t.num, t.den) == (int(n), int(d))
    for bad in ("", "0.x8", "1/0"):
        with pytest.raises(ValueError):
            ssj.Threshold.parse(bad)


def test_predicate_and_strategy_validation(ssj):
    # similarity.hpp:74-81, verify.hpp:25-28, test_verify.cpp:203-211
    ssj.jaccard(4, 5).validate()
    with pytest.raises(ValueError):
        ssj.SimilarityPredicate(ssj.SimilarityFunction.Jaccard, ssj.Threshold(0, 1)).validate()
    with pytest.raises(ValueError):
        ssj.SimilarityPredicate(ssj.SimilarityFunction.Jaccard, ssj.Threshold(6, 5)).validate()
    with pytest.raises(ValueError):
        ssj.SimilarityPredicate(ssj.SimilarityFunction.Overlap, overlap_threshold=0).validate()
    ssj.Strategy(ssj.StrategyKind.A, 32).validate()
    for bad in (0, 48, 3):
        with pytest.raises(ValueError):
            ssj.Strategy(ssj.StrategyKind.B, bad).validate()


def test_equivalent_overlap_host_matches_reference(ssj):
    g = golden("similarity")
    grid = g["eqo_grid"]
    for fi, fn in enumerate((ssj.SimilarityFunction.Jaccard, ssj.SimilarityFunction.Cosine,
                             ssj.SimilarityFunction.Dice)):
        for tn in (1, 7, 14, 19, 20):
            p = ssj.SimilarityPredicate(fn, ssj.Threshold(tn, 20))
            for r in range(1, 51, 7):
                for s in range(1, 51, 3):
                    assert ssj.equivalent_overlap(p, r, s) == grid[fi, tn - 1, r - 1, s - 1]
    for fn, num, den, r, s, want in g["big_cases"]:
        p = ssj.SimilarityPredicate(ssj.SimilarityFunction(int(fn)), ssj.Threshold(int(num), int(den)))
        assert ssj.equivalent_overlap(p, int(r), int(s)) == int(want)


def test_no_cpu_fallback_without_device(ssj):
    if ssj.device_count() > 0:
        pytest.skip("a device is present")
    coll = ssj.Collection.from_sets([[1, 2], [1, 2]])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ssj.VerificationEngine(coll, ssj.jaccard(1, 2), ssj.OutputMode.Pairs,
                               ssj.Strategy(ssj.StrategyKind.A, 1))


def test_engine_rejects_bad_config_before_touching_device(ssj):
    coll = ssj.Collection.from_sets([[1, 2], [1, 2]])
    with pytest.raises(ValueError):
        ssj.VerificationEngine(coll, ssj.jaccard(1, 2), ssj.OutputMode.Pairs,
                               ssj.Strategy(ssj.StrategyKind.B, 3))
    bad = ssj.SimilarityPredicate(ssj.SimilarityFunction.Jaccard, ssj.Threshold(0, 1))
    with pytest.raises(ValueError):
        ssj.VerificationEngine(coll, bad, ssj.OutputMode.Pairs, ssj.Strategy())
