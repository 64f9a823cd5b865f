"""One verification engine over several GPUs (ssj_engine_create_multi).

Only one GPU is available to the test box, so the device list repeats device 0: the
collection fan-out then runs as device-to-device copies, and every chunk is still split into
probe-slice ranges verified by separate per-device engines and reassembled in C order. The
results must be byte-identical to the one-device engine and to the reference's goldens."""
import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

J = 0
FIXTURES = ["verify_s41", "medium_s101", "sweep_s1002"]


def coll_of(ssj, g):
    return ssj.Collection(g["tokens"], g["offsets"], g["original_id"])


def chunk_keys(g):
    return [k[2:] for k in g.files if k.startswith("C_")]


def multi(ssj, coll, pred, kind="A", group=1, n=2, mode=None):
    mode = ssj.OutputMode.Pairs if mode is None else mode
    return ssj.VerificationEngine(coll, pred, mode, ssj.Strategy(ssj.StrategyKind[kind], group),
                                  devices=[0] * n)


@pytest.mark.parametrize("name", FIXTURES)
@pytest.mark.parametrize("n", [2, 3])
def test_multi_golden_chunks(ssj, gpu, name, n):
    """Flags byte-identical to the reference's, count and stats equal (test_verify.cpp:168-204
    through a 2- and 3-device engine), for every strategy kind incl. Auto."""
    g = golden(name)
    coll = coll_of(ssj, g)
    for key in chunk_keys(g):
        fn, num, den = (int(x) for x in key.split("_")[:3])
        pred = ssj.SimilarityPredicate(ssj.SimilarityFunction(fn), ssj.Threshold(num, den), 1)
        chunk = ssj.CandidateChunk(g["C_" + key], g["CO_" + key])
        for kind, group in (("A", 1), ("B", 32), ("C", 8), ("Auto", 32)):
            with multi(ssj, coll, pred, kind, group, n) as eng:
                devs, ms = eng.devices()
                assert devs == [0] * n and ms >= 0
                st = ssj.VerifyStats()
                out = eng.verify_chunk(chunk, None, st)
                assert out.count == int(g["count_" + key][0]), (key, kind)
                assert np.array_equal(out.flags, g["flags_" + key]), (key, kind)
                if eng.strategy().kind in (ssj.StrategyKind.A, ssj.StrategyKind.B):
                    assert [st.pairs_verified, st.early_exit_prunes,
                            st.comparison_budget_violations] == [int(x) for x in g["stats_" + key]]
                else:
                    assert st.pairs_verified == 0


def random_chunk(rng, n_sets, n_slices, max_k, trailing):
    probes = np.sort(rng.choice(np.arange(1, n_sets), size=n_slices, replace=True))
    C, CO = [], []
    for p in probes:
        k = int(rng.integers(0, max_k + 1))  # zero-width slices included
        C.extend(rng.integers(0, p, size=k).tolist())
        CO += [int(p), len(C)]
    C.extend(rng.integers(0, n_sets, size=trailing).tolist())  # slots no slice covers
    return np.array(C, np.uint32), np.array(CO, np.uint32)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_multi_random_vs_oracle(ssj, gpu, oracle, seed):
    rng = np.random.default_rng(seed)
    coll = ssj.synth_collection(seed, ssj.SynthConfig(sets=4000, min_size=1, max_size=200,
                                                      zipf_sizes=True, size_skew=1.2,
                                                      universe=3000, zipf_tokens=True,
                                                      duplicate_fraction=0.2, max_edits=2))
    C, CO = random_chunk(rng, coll.size(), 300, 400, 37)
    for num, den in ((1, 2), (4, 5)):
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, C, CO, oracle.pred(J, num, den))
        for n in (2, 4):
            with multi(ssj, coll, ssj.jaccard(num, den), "A", 32, n) as eng:
                out = eng.verify_chunk(ssj.CandidateChunk(C, CO))
                assert out.count == ref["count"]
                assert np.array_equal(out.flags, ref["flags"])
                assert out.flags[-37:].sum() == 0  # uncovered slots are never verified


def test_multi_double_buffering_and_results(ssj, gpu, oracle):
    rng = np.random.default_rng(9)
    coll = ssj.synth_collection(9, ssj.SynthConfig(sets=3000, min_size=5, max_size=90,
                                                   universe=2000, zipf_tokens=True,
                                                   duplicate_fraction=0.3, max_edits=1))
    chunks = [random_chunk(rng, coll.size(), 200, 300, 0) for _ in range(4)]
    pred = ssj.jaccard(3, 5)
    with multi(ssj, coll, pred, "A", 32, 3) as eng, \
            ssj.VerificationEngine(coll, pred, ssj.OutputMode.Pairs,
                                   ssj.Strategy(ssj.StrategyKind.A, 32)) as one:
        eng.set_original_ids(coll.original_id)
        one.set_original_ids(coll.original_id)
        flags = [np.zeros(c[0].size, np.uint8) for c in chunks]
        t0 = eng.submit_chunk(ssj.CandidateChunk(*chunks[0]), flags[0])
        t1 = eng.submit_chunk(ssj.CandidateChunk(*chunks[1]), flags[1])
        with pytest.raises(RuntimeError):  # two in flight already
            eng.submit_chunk(ssj.CandidateChunk(*chunks[2]), flags[2])
        counts = [eng.wait_chunk(t0), eng.wait_chunk(t1)]
        for k in range(2):
            ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunks[k][0], chunks[k][1],
                                      oracle.pred(J, 3, 5))
            assert counts[k] == ref["count"] and np.array_equal(flags[k], ref["flags"])
        for C, CO in chunks:
            ch = ssj.CandidateChunk(C, CO)
            s1, o1 = eng.verify_chunk_results(ch)
            s2, o2 = one.verify_chunk_results(ch)
            assert np.array_equal(s1, s2) and np.array_equal(o1, o2)
            for srt in (True, False):  # write_pairs order and decode_pairs (slot) order
                p1, v1 = eng.verify_chunk_pairs(ch, sorted_=srt)
                p2, v2 = one.verify_chunk_pairs(ch, sorted_=srt)
                assert np.array_equal(p1, p2) and np.array_equal(v1, v2), srt


def test_unsorted_pairs_follow_slot_order(ssj, gpu, oracle):
    """verify_chunk_pairs(sorted=False) returns decode_pairs order (pipeline.hpp:79-92):
    qualifying slots ascending, each as (max, min) of the original ids."""
    rng = np.random.default_rng(4)
    coll = ssj.synth_collection(4, ssj.SynthConfig(sets=2000, min_size=3, max_size=40,
                                                   universe=500, duplicate_fraction=0.4,
                                                   max_edits=1))
    C, CO = random_chunk(rng, coll.size(), 300, 200, 0)
    ref = oracle.verify_chunk(coll.tokens, coll.offsets, C, CO, oracle.pred(J, 1, 2))
    slots = np.nonzero(ref["flags"])[0]
    probe_of = np.repeat(CO[0::2], np.diff(np.concatenate([[0], CO[1::2]])))
    a, b = coll.original_id[probe_of[slots]], coll.original_id[C[slots]]
    want = np.stack([np.maximum(a, b), np.minimum(a, b)], 1)
    with ssj.VerificationEngine(coll, ssj.jaccard(1, 2), ssj.OutputMode.Pairs,
                                ssj.Strategy(ssj.StrategyKind.A, 1)) as eng:
        eng.set_original_ids(coll.original_id)
        got, _ = eng.verify_chunk_pairs(ssj.CandidateChunk(C, CO), sorted_=False)
        assert len(slots) > 50 and np.array_equal(got, want)


def test_multi_errors(ssj, gpu):
    coll = ssj.Collection.from_sets([[1, 2], [1, 2, 3], [2, 3]])
    with multi(ssj, coll, ssj.jaccard(1, 2), "A", 1, 2) as eng:
        with pytest.raises(ValueError):  # malformed C_O (ends decreasing)
            eng.verify_chunk(ssj.CandidateChunk([0, 1, 0], [1, 2, 2, 1]))
        with pytest.raises(IndexError):  # candidate index >= n (collection.hpp:87)
            eng.verify_chunk(ssj.CandidateChunk([0, 7], [1, 1, 2, 2]))
        with pytest.raises(ValueError):  # device pointers belong to one GPU
            eng.verify_chunk_device(0, 0, 0, 0, 0, 1)
        # still usable after the errors: {1,2,3}~{1,2}, {2,3}~{1,2}, {2,3}~{1,2,3} at J >= 1/2
        out = eng.verify_chunk(ssj.CandidateChunk([0, 0, 1], [1, 1, 2, 3]))
        assert out.flags.tolist() == [1, 0, 1] and out.count == 2
        out = eng.verify_chunk(ssj.CandidateChunk([], []))  # empty chunk
        assert out.count == 0 and out.flags.size == 0


def test_multi_run_join_and_gpu_join(ssj, gpu, oracle):
    """run_join with the engine over several devices (PipelineConfig.devices) and the
    dispatcher keeping 1 or 2 chunks in flight: pairs equal the brute-force oracle and the
    one-device join (same decode order); the all-GPU join shards over the devices."""
    coll = ssj.synth_collection(77, ssj.SynthConfig(sets=3000, min_size=5, max_size=60,
                                                    universe=1500, zipf_tokens=True,
                                                    duplicate_fraction=0.2, max_edits=1))
    tri = oracle.brute_force_join(coll.tokens, coll.offsets, oracle.pred(J, 7, 10))
    truth = oracle.oracle_pairs(coll.original_id, tri)
    pred = ssj.jaccard(7, 10)
    for alg in ssj.Algorithm:
        base = ssj.run_join(coll, pred, ssj.PipelineConfig(algorithm=alg,
                                                           mode=ssj.OutputMode.Pairs,
                                                           chunk_budget=64 << 10))
        assert np.array_equal(ssj.sorted_pairs(base.pairs), truth)
        for devs, inflight in (([0, 0], 1), ([0, 0, 0], 2)):
            for mode in (ssj.OutputMode.Pairs, ssj.OutputMode.Count):
                rep = ssj.run_join(coll, pred, ssj.PipelineConfig(
                    algorithm=alg, mode=mode, chunk_budget=64 << 10, devices=devs,
                    max_inflight=inflight))
                assert rep.count == len(truth), (alg, devs, inflight)
                assert rep.chunk_count == base.chunk_count
                assert rep.candidate_count == base.candidate_count
                if mode == ssj.OutputMode.Pairs:
                    assert np.array_equal(rep.pairs, base.pairs), (alg, devs)
    with multi(ssj, coll, pred, "Auto", 32, 3) as eng:
        eng.set_original_ids(coll.original_id)
        for alg in (0, 1, 2):
            pairs, rep = eng.gpu_join(alg, pairs=True, pairs_cap=1 << 20)
            assert np.array_equal(pairs, truth), alg
            assert rep["count"] == len(truth)


def test_inflight_with_observer(ssj, gpu):
    """max_inflight = 2 keeps the chunk observer's order and flags (pipeline.hpp:42-43)."""
    coll = ssj.synth_collection(5, ssj.SynthConfig(sets=2000, min_size=5, max_size=40,
                                                   universe=800, duplicate_fraction=0.3,
                                                   max_edits=1))
    seen = {1: [], 2: []}
    for inflight in (1, 2):
        def obs(chunk, out, k=inflight):
            seen[k].append((chunk.C.tobytes(), chunk.C_O.tobytes(), out.flags.tobytes(),
                            out.count))
        rep = ssj.run_join(coll, ssj.jaccard(3, 5), ssj.PipelineConfig(
            algorithm=ssj.Algorithm.AllPairs, mode=ssj.OutputMode.Pairs, chunk_budget=4 << 10,
            chunk_observer=obs, max_inflight=inflight))
        assert rep.chunk_count == len(seen[inflight]) > 4
    assert seen[1] == seen[2]
