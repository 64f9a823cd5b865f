"""Candidate generation and the whole join on the GPU: the device
generator's streams are byte-identical to the reference generators' golden streams
(joiners.hpp:47-102), and the device join's result pairs equal the reference's brute-force
pairs and the host join's."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

FIXTURES = ["verify_s41", "verify_s42", "verify_s43", "medium_s101", "medium_s202",
            "medium_s707", "sweep_s1000", "sweep_s1001", "sweep_s1002"]


def coll_of(ssj, g):
    return ssj.Collection(g["tokens"], g["offsets"], g["original_id"])


def engine(ssj, coll, pred):
    return ssj.VerificationEngine(coll, pred, ssj.OutputMode.Pairs,
                                  ssj.Strategy(ssj.StrategyKind.A, 1))


@pytest.mark.parametrize("name", FIXTURES)
def test_gpu_streams_match_reference(ssj, gpu, name):
    g = golden(name)
    coll = coll_of(ssj, g)
    for k in g.files:
        if not k.startswith("C_"):
            continue
        key = k[2:]
        fn, num, den = (int(x) for x in key.split("_")[:3])
        alg = int(key.split("_a")[1])
        pred = ssj.SimilarityPredicate(ssj.SimilarityFunction(fn), ssj.Threshold(num, den))
        with engine(ssj, coll, pred) as eng:
            chunk = eng.gpu_generate_candidates(alg)
            assert np.array_equal(chunk.C, g["C_" + key]), key
            assert np.array_equal(chunk.C_O, g["CO_" + key]), key
            if alg == 2:  # GroupJoin: the stream is per group (no probe windows)
                continue
            # any probe window is the matching piece of the stream
            n = coll.size()
            lo, hi = n // 3, 2 * n // 3
            part = eng.gpu_generate_candidates(alg, lo, hi)
            host, _ = ssj.generate_candidates(coll, pred, ssj.Algorithm(alg), lo, hi, threads=1)
            assert np.array_equal(part.C, host.C) and np.array_equal(part.C_O, host.C_O), key


@pytest.mark.parametrize("name", FIXTURES)
def test_gpu_join_matches_brute_force(ssj, gpu, oracle, name):
    """Pairs of the device join == the reference's brute_force_join (oracle.hpp:36-67)."""
    g = golden(name)
    coll = coll_of(ssj, g)
    for k in g.files:
        if not k.startswith("bf_"):
            continue
        fn, num, den = (int(x) for x in k[3:].split("_"))
        pred = ssj.SimilarityPredicate(ssj.SimilarityFunction(fn), ssj.Threshold(num, den))
        want = oracle.oracle_pairs(g["original_id"], np.asarray(g[k]).reshape(-1, 3))
        for alg in (0, 1, 2):
            with engine(ssj, coll, pred) as eng:
                eng.set_original_ids(coll.original_id)
                pairs, rep = eng.gpu_join(alg, max_chunk_candidates=1000)
                assert np.array_equal(pairs, want), (k, alg)
                assert rep["count"] == len(want)


SHAPES = [
    # DBLP-like (cfg2 shape, smaller n), J 0.8
    (dict(sets=30_000, min_size=40, max_size=120, universe=7200, zipf_tokens=True,
          token_skew=1.0, duplicate_fraction=0.02, max_edits=2, distinct_tokens=True), (4, 5)),
    # cfg1 shape, J 0.9
    (dict(sets=100_000, min_size=5, max_size=15, universe=10_000, duplicate_fraction=0.10,
          max_edits=1, distinct_tokens=True), (9, 10)),
    # KOSARAK-like long tail, J 0.75
    (dict(sets=200_000, min_size=2, max_size=2500, zipf_sizes=True, size_skew=1.9,
          universe=41_000, zipf_tokens=True, token_skew=0.6, duplicate_fraction=0.05,
          max_edits=2), (3, 4)),
]


@pytest.mark.parametrize("shape,thr", SHAPES)
def test_gpu_join_matches_host_join(ssj, gpu, shape, thr):
    """Bench shapes: the device stream equals the host generator's, and the device join (in
    several probe blocks) returns the host run_join's pairs."""
    coll = ssj.synth_collection(2024, ssj.SynthConfig(**shape))
    pred = ssj.jaccard(*thr)
    for alg in (ssj.Algorithm.AllPairs, ssj.Algorithm.PPJoin, ssj.Algorithm.GroupJoin):
        host, host_pairs = ssj.generate_candidates(coll, pred, alg)
        with engine(ssj, coll, pred) as eng:
            dev = eng.gpu_generate_candidates(int(alg))
            assert np.array_equal(dev.C, host.C) and np.array_equal(dev.C_O, host.C_O), alg
            eng.set_original_ids(coll.original_id)
            pairs, rep = eng.gpu_join(int(alg), max_chunk_candidates=max(host.C.size // 5, 1))
            assert rep["candidate_count"] == host.C.size
            assert rep["intra_group_pairs"] == len(host_pairs.reshape(-1, 2))
            assert rep["chunk_count"] >= 2 or host.C.size < 10
            # count mode (no pair decoding) agrees
            _, rep_c = eng.gpu_join(int(alg), pairs=False)
            assert rep_c["count"] == len(pairs) == rep["count"]
        cfg = ssj.PipelineConfig(algorithm=alg, mode=ssj.OutputMode.Pairs)
        ref = ssj.run_join(coll, pred, cfg)
        want = ssj.sorted_pairs(ref.pairs)
        assert np.array_equal(pairs, want.reshape(-1, 2)), alg


def test_gpu_join_shards_partition_the_join(ssj, gpu):
    """Shards (one per GPU in a multi-GPU run) are disjoint and together give the join."""
    coll = ssj.synth_collection(7, ssj.SynthConfig(**SHAPES[0][0]))
    pred = ssj.jaccard(4, 5)
    with engine(ssj, coll, pred) as eng:
        eng.set_original_ids(coll.original_id)
        full, rep = eng.gpu_join(0)
        parts, cands = [], 0
        for k in range(3):
            pk, rk = eng.gpu_join(0, shard=k, n_shards=3)
            parts.append(pk)
            cands += rk["candidate_count"]
        assert cands == rep["candidate_count"]
        got = ssj.sorted_pairs(np.concatenate(parts))
        assert np.array_equal(got, full)
        with pytest.raises(ValueError):  # GroupJoin runs as one shard
            eng.gpu_join(2, shard=0, n_shards=2)


def test_gpu_generation_edge_cases(ssj, gpu):
    """Empty sets, large tokens (no packed head records: the dedup reads the CSR), a single
    set, and empty probe windows: device streams equal the host generator's."""
    rng = np.random.default_rng(3)
    sets = [sorted(rng.choice(5000, size=int(rng.integers(1, 30)), replace=False).tolist())
            for _ in range(800)]
    sets += [list(s) for s in sets[:200]]  # duplicates -> qualifying pairs
    # the reference's collection order (collection.hpp:115-119), plus empty sets first
    sets = [[], []] + sorted(sets, key=lambda x: (len(x), x))
    base = ssj.Collection.from_sets(sets)
    for shift in (0, 1 << 28):
        toks = (base.tokens.astype(np.uint64) + shift).astype(np.uint32)
        coll = ssj.Collection(toks, base.offsets, base.original_id)
        pred = ssj.jaccard(3, 5)
        for alg in (0, 1):
            host, _ = ssj.generate_candidates(coll, pred, ssj.Algorithm(alg), threads=1)
            with engine(ssj, coll, pred) as eng:
                dev = eng.gpu_generate_candidates(alg)
                assert np.array_equal(dev.C, host.C) and np.array_equal(dev.C_O, host.C_O)
                empty = eng.gpu_generate_candidates(alg, 5, 5)
                assert empty.C.size == 0 and empty.C_O.size == 0
                eng.set_original_ids(coll.original_id)
                pairs, rep = eng.gpu_join(alg, max_chunk_candidates=2000)
            ref = ssj.run_join(coll, pred, ssj.PipelineConfig(algorithm=ssj.Algorithm(alg),
                                                              mode=ssj.OutputMode.Pairs))
            assert np.array_equal(pairs, ssj.sorted_pairs(ref.pairs).reshape(-1, 2))
    one = ssj.Collection.from_sets([[1, 2, 3]])
    with engine(ssj, one, ssj.jaccard(1, 2)) as eng:
        pairs, rep = eng.gpu_join(0)
        assert pairs.shape == (0, 2) and rep["count"] == 0 and rep["candidate_count"] == 0


def test_gpu_join_requires_reference_order(ssj, gpu):
    """The generators rely on the preprocessed (size, lex) order like the reference's
    (collection.hpp:115-119); an unordered collection is rejected, not joined wrongly."""
    coll = ssj.Collection.from_sets([[1, 2, 3, 4], [1, 2]])
    with engine(ssj, coll, ssj.jaccard(1, 2)) as eng:
        with pytest.raises(ValueError):
            eng.gpu_join(0)


def test_run_join_with_gpu_filtering(ssj, gpu):
    """run_join (the reference's driver interface) with filter_threads = FILTER_ON_GPU gives
    the same report counts and pairs as with host filtering."""
    coll = ssj.synth_collection(11, ssj.SynthConfig(**SHAPES[0][0]))
    pred = ssj.jaccard(4, 5)
    for alg in (ssj.Algorithm.AllPairs, ssj.Algorithm.PPJoin, ssj.Algorithm.GroupJoin):
        for mode in (ssj.OutputMode.Pairs, ssj.OutputMode.Count):
            host = ssj.run_join(coll, pred, ssj.PipelineConfig(algorithm=alg, mode=mode))
            dev = ssj.run_join(coll, pred, ssj.PipelineConfig(algorithm=alg, mode=mode,
                                                              filter_threads=ssj.FILTER_ON_GPU))
            assert dev.count == host.count and dev.candidate_count == host.candidate_count
            assert dev.host_verified_pairs == host.host_verified_pairs
            assert np.array_equal(ssj.sorted_pairs(dev.pairs), ssj.sorted_pairs(host.pairs))
