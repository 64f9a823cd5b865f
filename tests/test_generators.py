"""The host-side producers (CPU): candidate streams identical to the reference's generators
(golden streams the reference produced), the parallel generator equal to the sequential one,
the synthetic generator deterministic, and precoded preprocessing ordered like
collection.hpp:134-168."""
import numpy as np
import pytest

from conftest import golden

FIXTURES = ["verify_s41", "verify_s42", "verify_s43", "medium_s101", "medium_s202",
            "medium_s707", "sweep_s1000", "sweep_s1001", "sweep_s1002"]


@pytest.mark.parametrize("name", FIXTURES)
def test_candidate_streams_match_reference(ssj, name):
    g = golden(name)
    coll = ssj.Collection(g["tokens"], g["offsets"], g["original_id"])
    for k in g.files:
        if not k.startswith("C_"):
            continue
        key = k[2:]
        fn, num, den = (int(x) for x in key.split("_")[:3])
        alg = int(key.split("_a")[1])
        pred = ssj.SimilarityPredicate(ssj.SimilarityFunction(fn), ssj.Threshold(num, den))
        for threads in ([1, 3] if alg != 2 else [1]):
            chunk, host = ssj.generate_candidates(coll, pred, ssj.Algorithm(alg), threads=threads)
            assert np.array_equal(chunk.C, g["C_" + key]), (key, threads)
            assert np.array_equal(chunk.C_O, g["CO_" + key]), (key, threads)
            assert np.array_equal(host.reshape(-1), g["host_" + key].reshape(-1)), key


def test_parallel_windows_concatenate(ssj):
    """Probe windows generated independently concatenate to the full stream."""
    c = ssj.synth_collection(5, ssj.SynthConfig(sets=4000, min_size=5, max_size=40, universe=800,
                                                zipf_tokens=True, duplicate_fraction=0.05,
                                                max_edits=2))
    pred = ssj.jaccard(3, 5)
    for alg in (ssj.Algorithm.AllPairs, ssj.Algorithm.PPJoin):
        full, _ = ssj.generate_candidates(c, pred, alg, threads=1)
        parts_C, parts_CO, base = [], [], 0
        for lo in range(0, c.size(), 700):
            ch, _ = ssj.generate_candidates(c, pred, alg, lo, min(lo + 700, c.size()), threads=4)
            co = ch.C_O.astype(np.int64).reshape(-1, 2)
            co[:, 1] += base
            base += ch.C.size
            parts_C.append(ch.C)
            parts_CO.append(co.reshape(-1))
        assert np.array_equal(np.concatenate(parts_C), full.C)
        assert np.array_equal(np.concatenate(parts_CO).astype(np.uint32), full.C_O)


def test_synth_deterministic_and_shaped(ssj):
    cfg = ssj.SynthConfig(sets=20000, min_size=40, max_size=120, universe=7200, zipf_tokens=True,
                          duplicate_fraction=0.01, max_edits=2, distinct_tokens=True)
    a = ssj.synth_collection(1812, cfg)
    cfg.threads = 1
    b = ssj.synth_collection(1812, cfg)
    assert np.array_equal(a.tokens, b.tokens) and np.array_equal(a.original_id, b.original_id)
    sizes = np.diff(a.offsets.astype(np.int64))
    assert np.all(np.diff(sizes) >= 0)
    assert 75 <= a.tokens.size / a.size() <= 85
    for i in range(0, a.size(), 997):
        assert np.all(np.diff(a.set_view(i).astype(np.int64)) > 0)


def test_preprocess_precoded_native_matches_python(ssj):
    rng = np.random.default_rng(0)
    recs = [rng.integers(0, 50, size=int(rng.integers(0, 12))).tolist() for _ in range(3000)]
    a = ssj.preprocess_precoded(recs)
    b = ssj.preprocess_precoded_native(recs)
    assert np.array_equal(a.tokens, b.tokens)
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.original_id, b.original_id)
    assert a.dropped_empty == b.dropped_empty
