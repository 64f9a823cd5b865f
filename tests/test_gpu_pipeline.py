"""run_join on the GPU engine, restating proj/tests/test_pipeline.cpp and acceptance.cpp
criterion 4 (30,092-byte golden) against the oracle and the reference's golden streams."""
import hashlib

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

J = 0


def coll_of(ssj, g):
    return ssj.Collection(g["tokens"], g["offsets"], g["original_id"])


def truth_pairs(oracle, g, num, den, fn=J):
    tri = oracle.brute_force_join(g["tokens"], g["offsets"], oracle.pred(fn, num, den))
    return oracle.oracle_pairs(g["original_id"], tri)


def cfg(ssj, **kw):
    c = ssj.PipelineConfig()
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def test_run_join_matches_oracle_every_algorithm(ssj, gpu, oracle):
    # test_pipeline.cpp:23-40
    g = golden("medium_s101")
    c = coll_of(ssj, g)
    for num, den in ((1, 2), (4, 5)):
        truth = truth_pairs(oracle, g, num, den)
        for alg in ssj.Algorithm:
            for ft in (1, 4):
                rep = ssj.run_join(c, ssj.jaccard(num, den),
                                   cfg(ssj, algorithm=alg, mode=ssj.OutputMode.Pairs, workers=2,
                                       filter_threads=ft))
                assert rep.count == len(truth), (alg, num, den)
                assert np.array_equal(ssj.sorted_pairs(rep.pairs), truth), (alg, num, den)
                if alg == ssj.Algorithm.GroupJoin:
                    assert rep.host_verified_pairs <= rep.count


def test_count_mode(ssj, gpu, oracle):
    # test_pipeline.cpp:42-50
    g = golden("medium_s101")
    rep = ssj.run_join(coll_of(ssj, g), ssj.jaccard(3, 4), cfg(ssj, mode=ssj.OutputMode.Count))
    assert rep.count == len(truth_pairs(oracle, g, 3, 4))
    assert len(rep.pairs) == 0


def test_invariance_to_budget_and_workers(ssj, gpu, oracle):
    # test_pipeline.cpp:52-71
    g = golden("medium_s202")
    c = coll_of(ssj, g)
    truth = truth_pairs(oracle, g, 2, 3)
    for budget in (256, 16 << 10, ssj.KUNBOUNDED_BUDGET):
        for workers in (1, 3):
            rep = ssj.run_join(c, ssj.jaccard(2, 3), cfg(ssj, chunk_budget=budget, workers=workers,
                                                         mode=ssj.OutputMode.Pairs))
            assert np.array_equal(ssj.sorted_pairs(rep.pairs), truth), (budget, workers)
            if budget == ssj.KUNBOUNDED_BUDGET:
                assert rep.chunk_count <= 1
            elif budget == 256:
                assert rep.chunk_count > 1


def test_min_budget_splits_batches(ssj, gpu, oracle):
    # test_pipeline.cpp:73-91
    g = golden("pipeline_s303")
    c = coll_of(ssj, g)
    seen = []

    def obs(chunk, out):
        assert chunk.byte_size() <= ssj.ChunkBuilder.kMinBudget
        seen.append(1)

    rep = ssj.run_join(c, ssj.jaccard(1, 2), cfg(ssj, chunk_budget=ssj.ChunkBuilder.kMinBudget,
                                                 mode=ssj.OutputMode.Pairs, chunk_observer=obs))
    assert rep.chunk_count == len(seen) > 100
    assert np.array_equal(ssj.sorted_pairs(rep.pairs), truth_pairs(oracle, g, 1, 2))


def test_chunk_stream_identical_to_reference(ssj, gpu):
    """The chunks run_join dispatches (C, C_O bytes and flags) equal the reference's
    (recorded through its chunk_observer), and the report counters agree."""
    g = golden("pipeline_s303")
    c = coll_of(ssj, g)
    for budget in (256, 16 << 10):
        got = []
        rep = ssj.run_join(c, ssj.jaccard(1, 2),
                           cfg(ssj, chunk_budget=budget, mode=ssj.OutputMode.Pairs,
                               strategy=ssj.Strategy(ssj.StrategyKind.A, 1),
                               chunk_observer=lambda ch, out: got.append((ch, out))))
        nC, nCO = g[f"nC_{budget}"], g[f"nCO_{budget}"]
        assert len(got) == len(nC) == int(g[f"nchunks_{budget}"][0])
        c0 = co0 = 0
        for i, (ch, out) in enumerate(got):
            assert np.array_equal(ch.C, g[f"C_{budget}"][c0:c0 + nC[i]])
            assert np.array_equal(ch.C_O, g[f"CO_{budget}"][co0:co0 + nCO[i]])
            assert np.array_equal(out.flags, g[f"flags_{budget}"][c0:c0 + nC[i]])
            assert out.flags.nbytes == ch.C.nbytes // 4  # test_pipeline.cpp:93-107
            c0 += int(nC[i])
            co0 += int(nCO[i])
        ref = [int(x) for x in g[f"report_{budget}"]]
        assert [rep.count, rep.chunk_count, rep.candidate_count, rep.pairs_verified,
                rep.early_exit_prunes] == ref
        assert np.array_equal(ssj.sorted_pairs(rep.pairs), g[f"pairs_{budget}"])


def test_live_memory_bound(ssj, gpu):
    # test_pipeline.cpp:109-121
    g = golden("medium_s101")
    for mode in (ssj.OutputMode.Count, ssj.OutputMode.Pairs):
        rep = ssj.run_join(coll_of(ssj, g), ssj.jaccard(1, 2),
                           cfg(ssj, chunk_budget=2 << 10, mode=mode, workers=3))
        assert rep.chunk_count > 2
        assert rep.max_live_candidate_bytes <= 2 * (2 << 10)


def test_timings_and_counters(ssj, gpu):
    # test_pipeline.cpp:123-148
    g = golden("medium_s707")
    c = coll_of(ssj, g)
    rep = ssj.run_join(c, ssj.jaccard(1, 2), cfg(ssj, mode=ssj.OutputMode.Pairs))
    t = rep.timings
    assert t.join_ms > 0 and t.filtering_ms >= 0 and t.serialization_ms >= 0
    assert t.verification_ms >= 0
    assert t.join_ms + 0.5 >= t.filtering_ms + t.serialization_ms
    rep = ssj.run_join(c, ssj.jaccard(4, 5),
                       cfg(ssj, algorithm=ssj.Algorithm.AllPairs,
                           strategy=ssj.Strategy(ssj.StrategyKind.B, 32)))
    assert rep.pairs_verified == rep.candidate_count
    assert rep.comparison_budget_violations == 0
    assert rep.early_exit_prunes >= 1
    assert rep.resolved_strategy.kind != ssj.StrategyKind.Auto


def test_configuration_errors(ssj, gpu):
    # test_pipeline.cpp:150-163
    c = coll_of(ssj, golden("medium_s101"))
    with pytest.raises(ValueError):
        ssj.run_join(c, ssj.jaccard(1, 2), cfg(ssj, chunk_budget=4))
    with pytest.raises(ValueError):
        ssj.run_join(c, ssj.jaccard(1, 2), cfg(ssj, strategy=ssj.Strategy(ssj.StrategyKind.B, 3)))
    zero = ssj.SimilarityPredicate(ssj.SimilarityFunction.Jaccard, ssj.Threshold(0, 1))
    with pytest.raises(ValueError):
        ssj.run_join(c, zero)


def test_empty_and_tiny(ssj, gpu):
    # test_pipeline.cpp:165-182
    rep = ssj.run_join(ssj.Collection(), ssj.jaccard(1, 2))
    assert rep.count == 0 and rep.chunk_count == 0
    assert ssj.run_join(ssj.Collection.from_sets([[1, 2, 3]]), ssj.jaccard(1, 2)).count == 0
    rep = ssj.run_join(ssj.Collection.from_sets([[1, 2], [1, 2]]), ssj.jaccard(1, 1),
                       cfg(ssj, mode=ssj.OutputMode.Pairs))
    assert rep.count == 1 and rep.pairs.tolist() == [[1, 0]]


def test_c4_invariance_golden(ssj, gpu):
    """acceptance.cpp:230-264: 9 configurations, identical 30,092-byte outputs."""
    g = golden("c4_s777")
    c = coll_of(ssj, g)
    outs = set()
    for budget in (64 << 10, 1 << 20, ssj.KUNBOUNDED_BUDGET):
        for ft in (1, 4, 0):
            rep = ssj.run_join(c, ssj.jaccard(1, 2), cfg(ssj, mode=ssj.OutputMode.Pairs,
                                                         chunk_budget=budget, filter_threads=ft))
            text = f"{rep.count}\n" + ssj.write_pairs(rep.pairs)
            outs.add(text)
    assert len(outs) == 1
    text = outs.pop()
    assert len(text.encode()) == 30092
    assert hashlib.sha256(text.encode()).hexdigest() == str(g["out_sha256"][0])


@pytest.mark.parametrize("name", ["sweep_s1000", "sweep_s1001", "sweep_s1002"])
def test_oracle_sweep_subset(ssj, gpu, oracle, name):
    """acceptance.cpp:55-148 criterion 1 on the first seeds: every algorithm x strategy x
    group size at several thresholds matches the brute-force oracle."""
    g = golden(name)
    c = coll_of(ssj, g)
    for tn in (10, 13, 16, 19):
        truth = truth_pairs(oracle, g, tn, 20)
        for alg in ssj.Algorithm:
            for kind in (ssj.StrategyKind.A, ssj.StrategyKind.B, ssj.StrategyKind.C):
                for group in (1, 32, 128):
                    rep = ssj.run_join(c, ssj.jaccard(tn, 20),
                                       cfg(ssj, algorithm=alg, mode=ssj.OutputMode.Pairs,
                                           strategy=ssj.Strategy(kind, group),
                                           chunk_budget=256 << 10))
                    assert rep.count == len(truth)
                    assert np.array_equal(ssj.sorted_pairs(rep.pairs), truth)


SHAPES = {
    # the five BASELINE configs at oracle-sized n (same generator knobs as bench.py)
    "cfg1": (dict(sets=3000, min_size=5, max_size=15, universe=1000, duplicate_fraction=0.10,
                  max_edits=1, distinct_tokens=True), (9, 10)),
    "cfg2": (dict(sets=3000, min_size=40, max_size=120, universe=7200, zipf_tokens=True,
                  token_skew=1.0, duplicate_fraction=0.05, max_edits=2, distinct_tokens=True),
             (4, 5)),
    "cfg3": (dict(sets=3000, min_size=2, max_size=2500, zipf_sizes=True, size_skew=1.9,
                  universe=41_000, zipf_tokens=True, token_skew=0.6, duplicate_fraction=0.05,
                  max_edits=2), (3, 4)),
    "cfg4": (dict(sets=2500, min_size=1, max_size=12_000, zipf_sizes=True, size_skew=1.3,
                  universe=200_000, zipf_tokens=True, token_skew=1.0, duplicate_fraction=0.05,
                  max_edits=3), (3, 5)),
    "cfg5": (dict(sets=3000, min_size=40, max_size=120, universe=7200, zipf_tokens=True,
                  token_skew=1.0, duplicate_fraction=0.05, max_edits=2, distinct_tokens=True),
             (17, 20)),
}


@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_config_shapes_join_vs_oracle(ssj, gpu, oracle, shape):
    """run_join over every config shape (small n) equals the brute-force oracle for every
    algorithm, in Pairs mode (GPU pair decoding) and Count mode, several budgets."""
    kw, (num, den) = SHAPES[shape]
    coll = ssj.synth_collection(1234, ssj.SynthConfig(**kw))
    tri = oracle.brute_force_join(coll.tokens, coll.offsets, oracle.pred(J, num, den))
    truth = oracle.oracle_pairs(coll.original_id, tri)
    for alg in ssj.Algorithm:
        for budget, ft in ((64 << 10, 1), (ssj.KUNBOUNDED_BUDGET, 0)):
            rep = ssj.run_join(coll, ssj.jaccard(num, den),
                               cfg(ssj, algorithm=alg, mode=ssj.OutputMode.Pairs,
                                   chunk_budget=budget, filter_threads=ft))
            assert rep.count == len(truth), (shape, alg, budget)
            assert np.array_equal(ssj.sorted_pairs(rep.pairs), truth), (shape, alg, budget)
        rep = ssj.run_join(coll, ssj.jaccard(num, den),
                           cfg(ssj, algorithm=alg, mode=ssj.OutputMode.Count))
        assert rep.count == len(truth)


@pytest.mark.parametrize("name", ["medium_s101", "medium_s202", "sweep_s1001", "c4_s777"])
def test_join_report_fields_match_reference(ssj, gpu, name):
    """The JoinReport of the default PipelineConfig (Auto/32, PPJoin, pipeline.hpp:36-51) and
    of the other generators equals the reference run_join's field for field: count, chunks,
    candidates, host-verified pairs, resolved_strategy (Auto resolved as verify.hpp:249-253),
    VerifyStats (C records none) and, in Pairs mode, the pairs in JoinReport::pairs order."""
    from oracle import pyoracle as po
    if not po.ref_available():
        pytest.skip("oracle/_ref/libssjref.so not built")
    R = po.Ref()
    g = golden(name)
    c = coll_of(ssj, g)
    h = R.coll(g["tokens"], g["offsets"], g["original_id"])
    for (num, den), group in (((1, 2), 32), ((4, 5), 1)):
        for alg in ssj.Algorithm:
            for mode in (ssj.OutputMode.Count, ssj.OutputMode.Pairs):
                for kind in (ssj.StrategyKind.Auto, ssj.StrategyKind.B):
                    ref, ref_pairs, _ = R.run_join(h, J, num, den, 1, algorithm=int(alg),
                                                   budget=16 << 10, kind=int(kind),
                                                   group=group,
                                                   pairs_mode=mode == ssj.OutputMode.Pairs,
                                                   sort_pairs=False)
                    rep = ssj.run_join(c, ssj.jaccard(num, den),
                                       cfg(ssj, algorithm=alg, mode=mode, chunk_budget=16 << 10,
                                           strategy=ssj.Strategy(kind, group)))
                    key = (name, num, alg, mode, kind)
                    assert rep.count == ref["count"], key
                    assert rep.chunk_count == ref["chunk_count"], key
                    assert rep.candidate_count == ref["candidate_count"], key
                    assert rep.host_verified_pairs == ref["host_verified_pairs"], key
                    assert (int(rep.resolved_strategy.kind), rep.resolved_strategy.group_size) \
                        == (ref["resolved_kind"], ref["resolved_group"]), key
                    assert rep.pairs_verified == ref["pairs_verified"], key
                    assert rep.early_exit_prunes == ref["early_exit_prunes"], key
                    assert rep.comparison_budget_violations == 0
                    if mode == ssj.OutputMode.Pairs:
                        if alg == ssj.Algorithm.GroupJoin:
                            # the reference appends intra-group pairs on H0 as they are
                            # verified (pipeline.hpp:299-312); here they come after the chunks
                            assert np.array_equal(ssj.sorted_pairs(rep.pairs),
                                                  ssj.sorted_pairs(ref_pairs)), key
                        else:
                            assert np.array_equal(rep.pairs, ref_pairs), key
    R.L.ref_coll_free(h)
