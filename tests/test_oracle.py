"""Pin the C oracle (oracle/ssj_oracle.c) against the reference: its own known-answer tests
(restated from proj/tests/*.cpp) and the golden vectors the reference produced
(tests/golden/make_golden.py). CPU only."""
import hashlib

import numpy as np
import pytest

from conftest import golden

J, COS, DICE, OV = 0, 1, 2, 3


# ---- similarity.hpp ---------------------------------------------------------------------
def test_threshold_parse_known_answers(oracle):
    # test_similarity.cpp:18-29
    assert oracle.threshold_parse("0.8") == (4, 5)
    assert oracle.threshold_parse("1")[0] == 1
    assert oracle.threshold_parse("1.0")[1] == 1
    assert oracle.threshold_parse("4/5")[0] == 4
    assert oracle.threshold_parse(".85") == (17, 20)
    for bad in ("", "0.x8"):
        with pytest.raises(ValueError):
            oracle.threshold_parse(bad)


def test_threshold_parse_golden(oracle):
    g = golden("similarity")
    for text, (n, d) in zip(g["parse_in"], g["parse_out"]):
        assert oracle.threshold_parse(str(text)) == (int(n), int(d))


def test_equivalent_overlap_worked_values(oracle):
    # test_similarity.cpp:31-46
    assert oracle.equivalent_overlap(oracle.pred(J, 4, 5), 10, 10) == 9
    for n in (1, 2, 7, 100):
        assert oracle.equivalent_overlap(oracle.pred(J, 1, 1), n, n) == n
    assert oracle.equivalent_overlap(oracle.pred(COS, 1, 2), 4, 9) == 3
    assert oracle.equivalent_overlap(oracle.pred(OV, 1, 1, 5), 3, 100) == 5


def test_equivalent_overlap_grid_golden(oracle):
    g = golden("similarity")["eqo_grid"]
    for fi, fn in enumerate((J, COS, DICE)):
        for tn in range(1, 21):
            p = oracle.pred(fn, tn, 20)
            got = np.array([[oracle.equivalent_overlap(p, r, s) for s in range(1, 51)]
                            for r in range(1, 51)], np.uint8)
            assert np.array_equal(got, g[fi, tn - 1]), (fn, tn)


def test_equivalent_overlap_wide_golden(oracle):
    for fn, num, den, r, s, want in golden("similarity")["big_cases"]:
        assert oracle.equivalent_overlap(oracle.pred(int(fn), int(num), int(den)), int(r),
                                         int(s)) == int(want)


def test_meets_threshold_consistency_exhaustive(oracle):
    # test_similarity.cpp:79-102: meets_threshold <=> o >= eqo, and the reference's masks
    g = golden("similarity")
    for fi, fn in enumerate((J, COS, DICE)):
        for tn in range(1, 21, 3):
            p = oracle.pred(fn, tn, 20)
            for r in range(1, 51, 3):
                for s in range(1, 51, 2):
                    req = oracle.equivalent_overlap(p, r, s)
                    mask = 0
                    for o in range(0, min(r, s) + 1):
                        m = oracle.meets_threshold(p, o, r, s)
                        assert m == (o >= req)
                        mask |= int(m) << o
                    assert mask == int(g["meets_mask"][fi, tn - 1, r - 1, s - 1])


# ---- verify.hpp -------------------------------------------------------------------------
def test_verify_pair_count_worked_examples(oracle):
    # test_verify.cpp:35-57
    r = [1, 2, 3, 4, 5]
    s = [2, 3, 5, 7, 9]
    res = oracle.verify_pair_count(r, s, 3)
    assert res.met and res.overlap == 3
    hopeless = oracle.verify_pair_count(r, s, 6)
    assert not hopeless.met and hopeless.comparisons < 10
    early = oracle.verify_pair_count(r, [1, 2, 3, 4, 5], 2)
    assert early.met and early.overlap == 2 and early.comparisons == 2
    assert oracle.verify_pair_count(r, s, 0).met
    assert not oracle.verify_pair_count([], s, 1).met


def test_verify_pair_count_golden(oracle):
    g = golden("pair_count")
    ro, so = g["r_offsets"], g["s_offsets"]
    for k in range(len(g["required"])):
        r = g["r_tokens"][ro[k]:ro[k + 1]]
        s = g["s_tokens"][so[k]:so[k + 1]]
        res = oracle.verify_pair_count(r, s, int(g["required"][k]))
        assert (res.overlap, res.met, res.comparisons) == (
            int(g["overlap"][k]), bool(g["met"][k]), int(g["comparisons"][k]))
        truth = oracle.full_overlap(r, s)
        assert res.met == (truth >= int(g["required"][k]))


def test_intersect_path_partitions_golden(oracle):
    g = golden("partitions")
    ro, so = g["r_offsets"], g["s_offsets"]
    Bs = [int(b) for b in g["group_sizes"]]
    for k in range(len(ro) - 1):
        r = g["r_tokens"][ro[k]:ro[k + 1]]
        s = g["s_tokens"][so[k]:so[k + 1]]
        truth = oracle.full_overlap(r, s)
        row = 0
        for B in Bs:
            total = 0
            for w in range(B):
                part = oracle.intersect_path_partition(r, s, B, w)
                assert part == tuple(int(x) for x in g["parts"][k][row + w])
                c = oracle.partition_count(r, s, part)
                assert c == int(g["counts"][k][row + w])
                total += c
            assert total == truth
            row += B


def test_partition_equal_runs(oracle):
    # test_verify.cpp:120-132
    r = list(range(64))
    for B in (1, 2, 8, 64, 128):
        assert sum(oracle.partition_count(r, r, oracle.intersect_path_partition(r, r, B, k))
                   for k in range(B)) == 64


COLL_FIXTURES = ["verify_s41", "verify_s42", "verify_s43", "medium_s101", "medium_s202",
                 "medium_s707", "sweep_s1000", "sweep_s1001", "sweep_s1002"]


def chunk_keys(g):
    return [k[2:] for k in g.files if k.startswith("C_")]


@pytest.mark.parametrize("name", COLL_FIXTURES)
def test_verify_chunk_golden(oracle, name):
    """verify_chunk flags/count/stats and algorithmic bytes == the reference's."""
    g = golden(name)
    for key in chunk_keys(g):
        fn, num, den = (int(x) for x in key.split("_")[:3])
        p = oracle.pred(fn, num, den)
        res = oracle.verify_chunk(g["tokens"], g["offsets"], g["C_" + key], g["CO_" + key], p)
        assert res["count"] == int(g["count_" + key][0])
        assert np.array_equal(res["flags"], g["flags_" + key])
        assert tuple(res["stats"]) == tuple(int(x) for x in g["stats_" + key])
        assert oracle.chunk_algorithmic_bytes(g["tokens"], g["offsets"], g["C_" + key],
                                              g["CO_" + key], p) == int(g["bytes_" + key][0])


@pytest.mark.parametrize("name", COLL_FIXTURES)
def test_brute_force_golden(oracle, name):
    g = golden(name)
    for k in g.files:
        if not k.startswith("bf_"):
            continue
        fn, num, den = (int(x) for x in k[3:].split("_"))
        got = oracle.brute_force_join(g["tokens"], g["offsets"], oracle.pred(fn, num, den))
        assert np.array_equal(got, g[k].reshape(-1, 3))


def test_c4_golden_output_bytes(oracle):
    """acceptance.cpp:230-264 criterion 4: the oracle reproduces the 30,092-byte output."""
    g = golden("c4_s777")
    tri = oracle.brute_force_join(g["tokens"], g["offsets"], oracle.pred(J, 1, 2))
    pairs = oracle.oracle_pairs(g["original_id"], tri)
    text = f"{len(pairs)}\n" + "".join(f"{a}\t{b}\n" for a, b in pairs)
    assert len(text.encode()) == int(g["out_size"][0]) == 30092
    assert hashlib.sha256(text.encode()).hexdigest() == str(g["out_sha256"][0])


def test_oracle_errors(oracle):
    t = np.array([1, 2, 3], np.uint32)
    o = np.array([0, 3], np.uint32)
    p = oracle.pred(J, 1, 2)
    with pytest.raises(IndexError):
        oracle.verify_chunk(t, o, [5], [0, 1], p)
    with pytest.raises(ValueError):
        oracle.verify_chunk(t, o, [0, 0], [0, 2, 0, 1], p)


@pytest.mark.skipif("not __import__('oracle.pyoracle').pyoracle.ref_available()")
def test_oracle_matches_live_reference_random(oracle):
    """When the reference shim is present, cross-check on fresh random chunks."""
    R = oracle.Ref()
    rng = np.random.default_rng(99)
    for seed in range(3):
        t, o, oid = R.synth(500 + seed, sets=300, min_size=1, max_size=60, universe=300,
                            zipf_tokens=bool(seed % 2), duplicate_fraction=0.2)
        h = R.coll(t, o, oid)
        pool = R.pool(2)
        n = o.size - 1
        C_ = rng.integers(0, n, size=5000).astype(np.uint32)
        ends = np.sort(rng.integers(0, 5001, size=200)).astype(np.uint32)
        ends[-1] = 5000
        probes = rng.integers(0, n, size=200).astype(np.uint32)
        CO = np.stack([probes, ends], 1).reshape(-1)
        for fn, num, den in ((J, 1, 2), (COS, 3, 5), (DICE, 7, 10)):
            f, cnt, st, _ = R.verify_chunk(h, pool, fn, num, den, 1, 0, 1, True, C_, CO)
            res = oracle.verify_chunk(t, o, C_, CO, oracle.pred(fn, num, den))
            assert cnt == res["count"] and np.array_equal(f, res["flags"])
            assert tuple(st) == tuple(res["stats"])
