"""Parity of the sm_100a kernels (through the C ABI) with the reference: golden vectors the
reference produced, the C oracle on seeded random chunks, and the reference's edge cases.
Bit-exact flags, counts and overlaps (integer work)."""
import hashlib

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

J, COS, DICE, OV = 0, 1, 2, 3
COLL_FIXTURES = ["verify_s41", "verify_s42", "verify_s43", "medium_s101", "medium_s202",
                 "medium_s707", "sweep_s1000", "sweep_s1001", "sweep_s1002"]
STRATEGIES = [("A", 1), ("A", 32), ("B", 1), ("B", 4), ("B", 128), ("C", 1), ("C", 4),
              ("C", 32), ("C", 128)]


def make_pred(ssj, fn, num, den, ovt=1):
    return ssj.SimilarityPredicate(ssj.SimilarityFunction(fn), ssj.Threshold(num, den), ovt)


def engine(ssj, coll, pred, kind="A", group=1, mode=None):
    mode = ssj.OutputMode.Pairs if mode is None else mode
    return ssj.VerificationEngine(coll, pred, mode, ssj.Strategy(ssj.StrategyKind[kind], group))


def coll_of(ssj, g):
    return ssj.Collection(g["tokens"], g["offsets"], g["original_id"])


def chunk_keys(g):
    return [k[2:] for k in g.files if k.startswith("C_")]


@pytest.mark.parametrize("name", COLL_FIXTURES)
def test_golden_chunks_all_strategies(ssj, gpu, name):
    """verify_chunk flags byte-identical to the reference's, count and (A/B) stats equal
    (test_verify.cpp:168-204 on the GPU)."""
    g = golden(name)
    coll = coll_of(ssj, g)
    for key in chunk_keys(g):
        fn, num, den = (int(x) for x in key.split("_")[:3])
        pred = make_pred(ssj, fn, num, den)
        chunk = ssj.CandidateChunk(g["C_" + key], g["CO_" + key])
        for kind, group in STRATEGIES:
            with engine(ssj, coll, pred, kind, group) as eng:
                st = ssj.VerifyStats()
                out = eng.verify_chunk(chunk, None, st)
                assert out.count == int(g["count_" + key][0]), (key, kind, group)
                assert np.array_equal(out.flags, g["flags_" + key]), (key, kind, group)
                if kind != "C":
                    ref = [int(x) for x in g["stats_" + key]]
                    assert [st.pairs_verified, st.early_exit_prunes,
                            st.comparison_budget_violations] == ref
                else:
                    assert st.pairs_verified == 0  # verify.hpp:303-345 records nothing
        # Count mode reports the same tally without flags (test_verify.cpp:198-203)
        with engine(ssj, coll, pred, "B", 8, ssj.OutputMode.Count) as eng:
            out = eng.verify_chunk(chunk)
            assert out.count == int(g["count_" + key][0]) and out.flags.size == 0


@pytest.mark.parametrize("name", ["verify_s43", "medium_s101", "sweep_s1002"])
def test_results_mode_true_overlaps(ssj, gpu, oracle, name):
    """Qualifying slots with their true |r ∩ s| (oracle.hpp:48-62 semantics)."""
    g = golden(name)
    coll = coll_of(ssj, g)
    for key in chunk_keys(g):
        fn, num, den = (int(x) for x in key.split("_")[:3])
        ref = oracle.verify_chunk(g["tokens"], g["offsets"], g["C_" + key], g["CO_" + key],
                                  oracle.pred(fn, num, den), want_overlaps=True)
        want_slots = np.nonzero(ref["flags"])[0]
        for kind, group in (("A", 1), ("B", 32), ("C", 8)):
            with engine(ssj, coll, make_pred(ssj, fn, num, den), kind, group) as eng:
                slots, ovs = eng.verify_chunk_results(
                    ssj.CandidateChunk(g["C_" + key], g["CO_" + key]))
                assert np.array_equal(slots, want_slots), (key, kind)
                assert np.array_equal(ovs, ref["overlaps"][want_slots]), (key, kind)


def test_pipeline_chunk_streams(ssj, gpu):
    """Every chunk run_join dispatched under M_c = 256 B and 16 KiB (batches split across
    chunks, test_pipeline.cpp:52-91): GPU flags == the reference's per-chunk flags."""
    g = golden("pipeline_s303")
    coll = coll_of(ssj, g)
    pred = ssj.jaccard(1, 2)
    for budget in (256, 16 << 10):
        nC, nCO = g[f"nC_{budget}"], g[f"nCO_{budget}"]
        C_all, CO_all, F_all = g[f"C_{budget}"], g[f"CO_{budget}"], g[f"flags_{budget}"]
        counts = g[f"counts_{budget}"]
        with engine(ssj, coll, pred, "A", 1) as eng:
            c0 = co0 = 0
            total = 0
            for i in range(len(nC)):
                chunk = ssj.CandidateChunk(C_all[c0:c0 + nC[i]], CO_all[co0:co0 + nCO[i]])
                out = eng.verify_chunk(chunk)
                assert np.array_equal(out.flags, F_all[c0:c0 + nC[i]])
                assert out.count == int(counts[i])
                # ||O|| = ||C|| / 4 (verify.hpp:262-264, test_pipeline.cpp:93-107)
                assert out.flags.nbytes == chunk.C.nbytes // 4
                total += out.count
                c0 += int(nC[i])
                co0 += int(nCO[i])
            assert total == int(g[f"report_{budget}"][0])


# ---- seeded random chunks vs the C oracle --------------------------------------------------
def random_collection(ssj, rng, n_sets, max_size, universe, dup=0.3, zipf=False):
    sets = []
    for _ in range(n_sets):
        if sets and rng.random() < dup:
            base = list(sets[int(rng.integers(len(sets)))])
            for _ in range(int(rng.integers(0, 3))):
                if base:
                    base[int(rng.integers(len(base)))] = int(rng.integers(0, universe))
            sets.append(base)
        else:
            k = int(rng.integers(1, max_size + 1))
            if zipf:
                toks = np.unique((rng.zipf(1.3, size=3 * k) - 1) % universe)[:k]
            else:
                toks = rng.choice(universe, size=min(k, universe), replace=False)
            sets.append([int(t) for t in toks])
    return ssj.preprocess_precoded(sets)


def random_chunk(ssj, rng, coll, n_cands, n_slices, zero_width=0.0, trailing=0):
    n = coll.size()
    ends = np.sort(rng.integers(0, n_cands + 1, size=n_slices)).astype(np.int64)
    ends[-1] = n_cands
    if zero_width:
        dup = rng.random(n_slices) < zero_width
        for i in np.nonzero(dup)[0]:
            if i > 0:
                ends[i] = ends[i - 1]
        ends = np.maximum.accumulate(ends)
        ends[-1] = n_cands
    probes = rng.integers(0, n, size=n_slices)
    C_ = np.empty(n_cands + trailing, np.uint32)
    # candidates near the probe in (size, lex) order so that near-duplicates are met
    begin = 0
    for p, e in zip(probes, ends):
        k = int(e - begin)
        if k:
            lo = max(0, int(p) - 64)
            C_[begin:e] = rng.integers(lo, int(p) + 1, size=k)
        begin = int(e)
    if trailing:
        C_[n_cands:] = rng.integers(0, n, size=trailing)
    CO = np.stack([probes.astype(np.uint32), ends.astype(np.uint32)], 1).reshape(-1)
    return ssj.CandidateChunk(C_, CO)


CASES = [
    # (n_sets, max_size, universe, n_cands, n_slices, zipf)
    (3000, 12, 400, 50_000, 6_000, False),      # cfg1-like tiny sets, many slices per tile
    (3000, 12, 400, 50_000, 30_000, False),     # > kMaxTileSlices per tile: global search path
    (3000, 90, 2000, 200_000, 800, True),       # DBLP-like
    (600, 3000, 20000, 20_000, 40, True),       # long sets: probes beyond the staged cap
    (2000, 40, 150, 123_457, 1, False),         # one giant slice spanning many tiles
]


@pytest.mark.parametrize("case", CASES)
def test_random_chunks_vs_oracle(ssj, gpu, oracle, case):
    n_sets, max_size, universe, n_cands, n_slices, zipf = case
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    coll = random_collection(ssj, rng, n_sets, max_size, universe, zipf=zipf)
    chunk = random_chunk(ssj, rng, coll, n_cands, n_slices, zero_width=0.05)
    for fn, num, den, ovt in ((J, 4, 5, 1), (J, 1, 2, 1), (COS, 3, 4, 1), (DICE, 9, 10, 1),
                              (OV, 1, 1, 3)):
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                  oracle.pred(fn, num, den, ovt))
        for kind, group in (("A", 1), ("B", 64), ("C", 32), ("C", 4)):
            with engine(ssj, coll, make_pred(ssj, fn, num, den, ovt), kind, group) as eng:
                out = eng.verify_chunk(chunk)
                assert out.count == ref["count"], (fn, kind, group)
                assert np.array_equal(out.flags, ref["flags"]), (fn, kind, group)


TOKEN_RANGES = [
    # (scale, offset): tokens t -> t * scale + offset (monotone, so sets stay sorted)
    (1, 0x00FFFFE0 - 3000),        # largest tokens just below the packed-head limit
    (1, 0x00FFFFE0 - 1000),        # some tokens at/above the limit: descriptor + CSR path
    (1, 1 << 28),                  # all tokens large
    (131, 0),                      # probes spanning > 8160 tokens: bitmap read through L1
    (4099, 0),                     # probes spanning > 256K tokens: no bitmap, merge path
    (1, 0xFFFFFFFF - 2999),        # token 0xFFFFFFFF (the CSR padding value) is a real token
]


@pytest.mark.parametrize("scale,offset", TOKEN_RANGES)
def test_token_value_ranges(ssj, gpu, oracle, scale, offset):
    """Every token-value regime of the strategy-A path: packed head records (tokens below
    0x00FFFFE0), set descriptors + CSR sectors otherwise, the byte map / global bitmap / merge
    paths by probe span, and the padding value as a real token."""
    rng = np.random.default_rng(scale * 7 + (offset & 0xFFFF))
    base = random_collection(ssj, rng, 2500, 90, 3000, zipf=True)
    toks = (base.tokens.astype(np.uint64) * scale + offset).astype(np.uint32)
    coll = ssj.Collection(toks, base.offsets, base.original_id)
    chunk = random_chunk(ssj, rng, coll, 150_000, 600, zero_width=0.05)
    for fn, num, den, ovt in ((J, 4, 5, 1), (J, 1, 2, 1), (OV, 1, 1, 2)):
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                  oracle.pred(fn, num, den, ovt))
        with engine(ssj, coll, make_pred(ssj, fn, num, den, ovt), "A", 1) as eng:
            out = eng.verify_chunk(chunk)
            assert out.count == ref["count"], (fn, num, den)
            assert np.array_equal(out.flags, ref["flags"]), (fn, num, den)
        with engine(ssj, coll, make_pred(ssj, fn, num, den, ovt), "A", 1) as eng:
            ref2 = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                       oracle.pred(fn, num, den, ovt), want_overlaps=True)
            slots, ovs = eng.verify_chunk_results(chunk)
            want = np.nonzero(ref2["flags"])[0]
            assert np.array_equal(slots, want) and np.array_equal(ovs, ref2["overlaps"][want])


def test_wide_threshold_u128_path(ssj, gpu, oracle):
    """num >= 2^30 takes the device u128 path of equivalent_overlap."""
    rng = np.random.default_rng(5)
    coll = random_collection(ssj, rng, 1500, 60, 500)
    chunk = random_chunk(ssj, rng, coll, 60_000, 900)
    # Cosine / Dice with den > 2^32 (e.g. Threshold::parse("0.123456789012")): the device's
    # double estimate still starts the reference's upward search below the answer
    for fn, num, den in ((J, (1 << 40) + 3, (1 << 41) + 7), (DICE, (1 << 35) + 1, (1 << 36)),
                         (COS, 999983, 1000003), (COS, 30864197253, 250000000000),
                         (COS, (1 << 40) + 3, (1 << 41) + 7), (DICE, 30864197253, 250000000000)):
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                  oracle.pred(fn, num, den))
        with engine(ssj, coll, make_pred(ssj, fn, num, den)) as eng:
            out = eng.verify_chunk(chunk)
            assert np.array_equal(out.flags, ref["flags"]) and out.count == ref["count"]


def test_cosine_overflow_regime_refused(ssj, gpu):
    """num * max|s| + den >= 2^64 wraps the reference's u128 products (similarity.hpp:
    93-102): such a Cosine threshold is refused with std::invalid_argument, not reproduced."""
    coll = ssj.Collection.from_sets([list(range(100)), list(range(1, 101))])
    with pytest.raises(ValueError):
        engine(ssj, coll, make_pred(ssj, COS, (1 << 62) + 1, (1 << 63) + 5))
    with engine(ssj, coll, make_pred(ssj, COS, (1 << 56) + 1, (1 << 57) + 5)) as eng:
        assert eng.verify_chunk(ssj.CandidateChunk([0], [1, 1])).count == 1


def test_trailing_uncovered_slots(ssj, gpu, oracle):
    """Slots past the last C_O end are never verified (chunk.hpp:36-48 decode): flag 0."""
    rng = np.random.default_rng(11)
    coll = random_collection(ssj, rng, 800, 30, 200)
    chunk = random_chunk(ssj, rng, coll, 10_000, 300, trailing=5000)
    ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                              oracle.pred(J, 1, 2))
    # the same slots all covered first, so the engine's reused flag buffer holds verdicts
    # of the trailing slots (compute-sanitizer initcheck found strategies B / C copying
    # never-written flag bytes back)
    CO_full = chunk.C_O.copy()
    CO_full[-1] = chunk.C.size
    full = ssj.CandidateChunk(chunk.C, CO_full)
    ref_full = oracle.verify_chunk(coll.tokens, coll.offsets, full.C, full.C_O,
                                   oracle.pred(J, 1, 2))
    assert ref_full["flags"][10_000:].any()
    for kind, group in (("A", 1), ("B", 32), ("C", 8)):
        with engine(ssj, coll, ssj.jaccard(1, 2), kind, group) as eng:
            out = eng.verify_chunk(full)
            bad = np.flatnonzero(out.flags != ref_full["flags"])
            assert bad.size == 0 and out.count == ref_full["count"], (kind, bad[:10], bad.size)
            out = eng.verify_chunk(chunk)
            assert np.array_equal(out.flags, ref["flags"]) and out.count == ref["count"]
            assert not out.flags[10_000:].any()


# ---- edge cases ----------------------------------------------------------------------------
def test_empty_and_tiny(ssj, gpu):
    # test_pipeline.cpp:165-182 shapes at the engine level
    twins = ssj.Collection.from_sets([[1, 2], [1, 2]])
    with engine(ssj, twins, ssj.jaccard(1, 1)) as eng:
        out = eng.verify_chunk(ssj.CandidateChunk([0], [1, 1]))
        assert out.count == 1 and out.flags.tolist() == [1]
        out = eng.verify_chunk(ssj.CandidateChunk([], []))
        assert out.count == 0 and out.flags.size == 0
        out = eng.verify_chunk(ssj.CandidateChunk([], [0, 0, 1, 0]))  # zero-width entries
        assert out.count == 0
    empty = ssj.Collection()
    with engine(ssj, empty, ssj.jaccard(1, 2)) as eng:
        assert eng.verify_chunk(ssj.CandidateChunk([], [])).count == 0
        with pytest.raises(IndexError):
            eng.verify_chunk(ssj.CandidateChunk([0], [0, 1]))


def test_empty_sets_and_zero_requirement(ssj, gpu, oracle):
    """from_sets may hold empty sets: required 0 => met (verify.hpp:57, 70)."""
    sets = [[], [], [1, 2, 3], [], [4]]
    coll = ssj.Collection.from_sets(sets)
    chunk = ssj.CandidateChunk([0, 1, 3, 2, 4, 0], [1, 1, 3, 3, 4, 6])
    for fn, num, den, ovt in ((J, 1, 2, 1), (OV, 1, 1, 1), (COS, 1, 2, 1), (DICE, 1, 2, 1)):
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                  oracle.pred(fn, num, den, ovt), want_overlaps=True)
        for kind, group in STRATEGIES:
            with engine(ssj, coll, make_pred(ssj, fn, num, den, ovt), kind, group) as eng:
                st = ssj.VerifyStats()
                out = eng.verify_chunk(chunk, None, st)
                assert np.array_equal(out.flags, ref["flags"]), (fn, kind, group)
                if kind != "C":
                    assert (st.pairs_verified, st.early_exit_prunes) == tuple(ref["stats"][:2])
                slots, ovs = eng.verify_chunk_results(chunk)
                assert np.array_equal(slots, np.nonzero(ref["flags"])[0])
                assert np.array_equal(ovs, ref["overlaps"][slots])


def test_errors_like_the_reference(ssj, gpu):
    coll = ssj.Collection.from_sets([[1, 2, 3], [1, 2, 4], [2, 3]])
    for kind, group in (("A", 1), ("B", 32), ("C", 8)):
        with engine(ssj, coll, ssj.jaccard(1, 2), kind, group) as eng:
            with pytest.raises(IndexError):      # candidate out of range (collection.hpp:87)
                eng.verify_chunk(ssj.CandidateChunk([0, 7], [2, 2]))
            with pytest.raises(IndexError):      # probe out of range
                eng.verify_chunk(ssj.CandidateChunk([0], [9, 1]))
            with pytest.raises(ValueError):      # malformed C_O
                eng.verify_chunk(ssj.CandidateChunk([0, 1], [2, 2, 1, 1]))
            # the engine stays usable after an error
            out = eng.verify_chunk(ssj.CandidateChunk([0, 1], [2, 2]))
            assert out.flags.size == 2


def test_async_double_buffering_and_pinned(ssj, gpu, oracle):
    rng = np.random.default_rng(21)
    coll = random_collection(ssj, rng, 2000, 40, 300)
    chunks = [random_chunk(ssj, rng, coll, 300_000 + 1000 * i, 5000) for i in range(4)]
    refs = [oracle.verify_chunk(coll.tokens, coll.offsets, c.C, c.C_O, oracle.pred(J, 3, 5))
            for c in chunks]
    with engine(ssj, coll, ssj.jaccard(3, 5)) as eng:
        # pinned host buffers (ssj_host_alloc): copied without staging
        pins = []
        for c in chunks:
            pc = ssj.PinnedBuffer(c.C.nbytes + 16)
            pco = ssj.PinnedBuffer(c.C_O.nbytes + 16)
            pf = ssj.PinnedBuffer(c.C.size + 16)
            cv = pc.view(np.uint32, c.C.size)
            cv[:] = c.C
            cov = pco.view(np.uint32, c.C_O.size)
            cov[:] = c.C_O
            pins.append((pc, pco, pf, ssj.CandidateChunk.__new__(ssj.CandidateChunk)))
            pins[-1][3].C, pins[-1][3].C_O = cv, cov
        tickets = []
        for i, (pc, pco, pf, ch) in enumerate(pins):
            if len(tickets) == 2:
                t, j = tickets.pop(0)
                assert eng.wait_chunk(t) == refs[j]["count"]
                assert np.array_equal(pins[j][2].view(np.uint8, chunks[j].C.size),
                                      refs[j]["flags"])
            tickets.append((eng.submit_chunk(ch, pf.view(np.uint8, ch.C.size)), i))
        for t, j in tickets:
            assert eng.wait_chunk(t) == refs[j]["count"]
            assert np.array_equal(pins[j][2].view(np.uint8, chunks[j].C.size), refs[j]["flags"])


def test_device_api_and_algorithmic_bytes(ssj, gpu, oracle):
    import torch
    rng = np.random.default_rng(31)
    coll = random_collection(ssj, rng, 3000, 80, 1500, zipf=True)
    chunk = random_chunk(ssj, rng, coll, 250_000, 2500)
    ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                              oracle.pred(J, 4, 5))
    ref_bytes = oracle.chunk_algorithmic_bytes(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                               oracle.pred(J, 4, 5))
    dev = torch.device("cuda:0")
    dC = torch.from_numpy(chunk.C.view(np.int32)).to(dev)
    dCO = torch.from_numpy(chunk.C_O.view(np.int32)).to(dev)
    dF = torch.zeros(chunk.C.size, dtype=torch.uint8, device=dev)
    dR = torch.zeros(8, dtype=torch.int64, device=dev)
    dB = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    for kind, group in (("A", 1), ("B", 128), ("C", 32)):
        with engine(ssj, coll, ssj.jaccard(4, 5), kind, group) as eng:
            eng.verify_chunk_device(dC.data_ptr(), chunk.C.size, dCO.data_ptr(), chunk.C_O.size,
                                    dF.data_ptr(), dR.data_ptr(), stream)
            torch.cuda.synchronize()
            words = dR.cpu().numpy()
            ssj.result_error(words)
            assert int(words[0]) == ref["count"]
            assert np.array_equal(dF.cpu().numpy(), ref["flags"])
            eng.chunk_algorithmic_bytes_device(dC.data_ptr(), chunk.C.size, dCO.data_ptr(),
                                               chunk.C_O.size, dB.data_ptr(), stream)
            torch.cuda.synchronize()
            assert int(dB.item()) == ref_bytes


def test_every_flag_written(ssj, gpu, oracle):
    """Every slot's flag is stored by the kernels, covered or not: the device flag buffer is
    filled with 0xAB first, so a flag some kernel leaves unwritten cannot pass as a stale 0
    (long slices cut into runs, pairs longer than kLongPair, zero-width and trailing slices)."""
    import torch
    rng = np.random.default_rng(47)
    coll = random_collection(ssj, rng, 900, 300, 1200)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream().cuda_stream
    shapes = [dict(n_cands=10_000, n_slices=300, trailing=5000),
              dict(n_cands=60_000, n_slices=40, zero_width=0.2),
              dict(n_cands=3_000, n_slices=2000, trailing=700)]
    for kw in shapes:
        chunk = random_chunk(ssj, rng, coll, **kw)
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                  oracle.pred(J, 1, 2))
        dC = torch.from_numpy(chunk.C.view(np.int32)).to(dev)
        dCO = torch.from_numpy(chunk.C_O.view(np.int32)).to(dev)
        dR = torch.zeros(8, dtype=torch.int64, device=dev)
        for kind, group in (("A", 1), ("Auto", 32), ("B", 64), ("C", 8)):
            dF = torch.full((chunk.C.size,), 0xAB, dtype=torch.uint8, device=dev)
            with engine(ssj, coll, ssj.jaccard(1, 2), kind, group) as eng:
                eng.verify_chunk_device(dC.data_ptr(), chunk.C.size, dCO.data_ptr(),
                                        chunk.C_O.size, dF.data_ptr(), dR.data_ptr(), stream)
                torch.cuda.synchronize()
            got = dF.cpu().numpy()
            bad = np.flatnonzero(got != ref["flags"])
            assert bad.size == 0, (kw, kind, bad[:8], got[bad[:8]])
            assert int(dR[0].item()) == ref["count"]


def test_probe_map_protocol_stress(ssj, gpu, oracle):
    """run_kernel's probe maps are built by one warp and published through mbarriers (no CTA
    barrier): chunks whose runs change probe every run (3-buffer path, build-ahead) or every
    few runs (2-buffer path), re-verified several times into a 0xAB-filled buffer -- a reader
    that saw a half-built or recycled map would flip flags."""
    import torch
    rng = np.random.default_rng(2024)
    coll = random_collection(ssj, rng, 4000, 70, 3000, zipf=True)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream().cuda_stream
    n = coll.size()
    for per_slice, n_slices in ((200, 2500), (3000, 120)):
        lens = rng.integers(per_slice // 2, per_slice * 3 // 2, size=n_slices)
        ends = np.cumsum(lens)
        probes = rng.integers(64, n, size=n_slices)
        C_ = np.concatenate([rng.integers(max(0, int(p) - 300), int(p) + 1, size=int(k))
                             for p, k in zip(probes, lens)]).astype(np.uint32)
        CO = np.stack([probes.astype(np.uint32), ends.astype(np.uint32)], 1).reshape(-1)
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, C_, CO, oracle.pred(J, 1, 2))
        dC = torch.from_numpy(C_.view(np.int32)).to(dev)
        dCO = torch.from_numpy(CO.view(np.int32)).to(dev)
        dR = torch.zeros(8, dtype=torch.int64, device=dev)
        with engine(ssj, coll, ssj.jaccard(1, 2), "A", 32) as eng:
            for rep in range(5):
                dF = torch.full((C_.size,), 0xAB, dtype=torch.uint8, device=dev)
                eng.verify_chunk_device(dC.data_ptr(), C_.size, dCO.data_ptr(), CO.size,
                                        dF.data_ptr(), dR.data_ptr(), stream)
                torch.cuda.synchronize()
                got = dF.cpu().numpy()
                bad = np.flatnonzero(got != ref["flags"])
                assert bad.size == 0, (per_slice, rep, bad[:8])
                assert int(dR[0].item()) == ref["count"]


def test_c4_golden_on_gpu(ssj, gpu):
    """acceptance.cpp:230-264: the all-pairs chunk of seed 777 (12.5 M candidates) verified
    on the GPU reproduces the reference's 30,092-byte pairs output exactly."""
    g = golden("c4_s777")
    coll = coll_of(ssj, g)
    n = coll.size()
    ends = np.cumsum(np.arange(n, dtype=np.uint64)).astype(np.uint32)
    C_ = np.concatenate([np.arange(r, dtype=np.uint32) for r in range(n)])
    CO = np.stack([np.arange(n, dtype=np.uint32), ends], 1).reshape(-1)
    chunk = ssj.CandidateChunk(C_, CO)
    for kind, group in (("A", 1), ("C", 32)):
        with engine(ssj, coll, ssj.jaccard(1, 2), kind, group) as eng:
            out = eng.verify_chunk(chunk)
            slots = np.nonzero(out.flags)[0]
            probe = np.searchsorted(ends, slots, side="right")
            a = coll.original_id[probe]
            b = coll.original_id[C_[slots]]
            pairs = np.stack([np.maximum(a, b), np.minimum(a, b)], 1)
            pairs = pairs[np.lexsort((pairs[:, 1], pairs[:, 0]))]
            text = f"{out.count}\n" + "".join(f"{x}\t{y}\n" for x, y in pairs)
            assert len(text.encode()) == 30092
            assert hashlib.sha256(text.encode()).hexdigest() == str(g["out_sha256"][0])


def test_auto_resolution_like_the_reference(ssj, gpu):
    """verify.hpp:249-253: Auto reports B (average set size <= 10) or C with group >= 128,
    and the stats follow the reported strategy (C records none); the A kernels run."""
    small = ssj.Collection.from_sets([[1], [2, 3]])
    with engine(ssj, small, ssj.jaccard(1, 2), "Auto", 32) as eng:
        r = eng.strategy()
        assert (r.kind, r.group_size) == (ssj.StrategyKind.B, 32)
        assert eng.kernel_strategy().kind == ssj.StrategyKind.A
        st = ssj.VerifyStats()
        out = eng.verify_chunk(ssj.CandidateChunk([0], [1, 1]), None, st)
        assert out.count == 0 and st.pairs_verified == 1  # B records stats
    big = ssj.Collection.from_sets([list(range(1000)), list(range(3, 1003))])
    for group, want in ((32, 128), (256, 256)):
        with engine(ssj, big, ssj.jaccard(1, 2), "Auto", group) as eng:
            r = eng.strategy()
            assert (r.kind, r.group_size) == (ssj.StrategyKind.C, want)
            k = eng.kernel_strategy()
            assert (k.kind, k.group_size) == (ssj.StrategyKind.A, group)
            st = ssj.VerifyStats()
            out = eng.verify_chunk(ssj.CandidateChunk([0], [1, 1]), None, st)
            assert out.count == 1 and out.flags.tolist() == [1]
            assert st.pairs_verified == 0  # C records nothing (verify.hpp:303-345)


def test_long_sets_bitmaps_and_deferral(ssj, gpu, oracle):
    """ENRON-like long sets: probe bitmaps (slices >= 64 candidates), long pairs deferred to
    the warp-per-pair kernel, plus short slices on the merge path -- all strategies, flags,
    results mode overlaps and stats against the oracle."""
    coll = ssj.synth_collection(2019, ssj.SynthConfig(
        sets=6000, min_size=1, max_size=6000, zipf_sizes=True, size_skew=1.3, universe=60000,
        zipf_tokens=True, token_skew=1.0, duplicate_fraction=0.05, max_edits=3))
    for num, den in ((3, 5), (4, 5)):
        pred = ssj.jaccard(num, den)
        chunk, _ = ssj.generate_candidates(coll, pred, ssj.Algorithm.AllPairs, threads=4)
        assert chunk.C.size > 10_000
        ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                                  oracle.pred(J, num, den), want_overlaps=True)
        for kind, group in (("A", 1), ("B", 256), ("C", 32), ("C", 8)):
            with engine(ssj, coll, pred, kind, group) as eng:
                st = ssj.VerifyStats()
                out = eng.verify_chunk(chunk, None, st)
                assert out.count == ref["count"], (num, kind, group)
                assert np.array_equal(out.flags, ref["flags"]), (num, kind, group)
                if kind != "C":
                    assert (st.pairs_verified, st.early_exit_prunes) == tuple(ref["stats"][:2])
                slots, ovs = eng.verify_chunk_results(chunk)
                want = np.nonzero(ref["flags"])[0]
                assert np.array_equal(slots, want) and np.array_equal(ovs, ref["overlaps"][want])


@pytest.mark.parametrize("name", ["medium_s101", "sweep_s1002", "verify_s43"])
def test_gpu_pair_decoding(ssj, gpu, oracle, name):
    """H2 on the GPU (decode_pairs pipeline.hpp:79-92 + write_pairs order report.hpp:39-42):
    qualifying slots -> (max, min) original ids, radix-sorted on the device, with overlaps."""
    g = golden(name)
    coll = coll_of(ssj, g)
    for key in chunk_keys(g):
        fn, num, den = (int(x) for x in key.split("_")[:3])
        chunk = ssj.CandidateChunk(g["C_" + key], g["CO_" + key])
        ref = oracle.verify_chunk(g["tokens"], g["offsets"], chunk.C, chunk.C_O,
                                  oracle.pred(fn, num, den), want_overlaps=True)
        slots = np.nonzero(ref["flags"])[0]
        probe = chunk.C_O[0::2][np.searchsorted(chunk.C_O[1::2].astype(np.int64), slots,
                                                side="right")]
        a = coll.original_id[probe]
        b = coll.original_id[chunk.C[slots]]
        want = np.stack([np.maximum(a, b), np.minimum(a, b)], 1).astype(np.uint32)
        order = np.lexsort((want[:, 1], want[:, 0]))
        with engine(ssj, coll, make_pred(ssj, fn, num, den)) as eng:
            eng.set_original_ids(coll.original_id)
            st = ssj.VerifyStats()
            pairs, ovs = eng.verify_chunk_pairs(chunk, True, st)
            assert np.array_equal(pairs, want[order]), key
            assert np.array_equal(ovs, ref["overlaps"][slots][order]), key
            assert st.pairs_verified == chunk.C.size


@pytest.mark.parametrize("shape", [
    # DBLP-like: long slices -> runs, > 4M candidates -> the host path uploads C in segments
    dict(sets=45_000, min_size=40, max_size=120, universe=7200, zipf_tokens=True,
         token_skew=1.0, duplicate_fraction=0.02, max_edits=2, distinct_tokens=True),
    # KOSARAK-like: tiny slices of long-tailed sets -> short tiles + the long-pair pass
    dict(sets=500_000, min_size=2, max_size=2500, zipf_sizes=True, size_skew=1.9,
         universe=41_000, zipf_tokens=True, token_skew=0.6, duplicate_fraction=0.05,
         max_edits=2),
])
def test_large_segmented_chunks_vs_oracle(ssj, gpu, oracle, shape):
    """Whole-join AllPairs chunks of the bench shapes through every output path: the host
    call (C uploaded in segments, runs clipped at segment boundaries), the device call and
    results mode -- flags, counts and overlaps identical to the C oracle."""
    coll = ssj.synth_collection(99, ssj.SynthConfig(**shape))
    pred = ssj.jaccard(4, 5) if shape["universe"] == 7200 else ssj.jaccard(3, 4)
    chunk, _ = ssj.generate_candidates(coll, pred, ssj.Algorithm.AllPairs)
    assert chunk.C.size > 0
    ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O,
                              oracle.pred(J, pred.threshold.num, pred.threshold.den),
                              want_overlaps=True)
    with engine(ssj, coll, pred, "A", 1) as eng:
        out = eng.verify_chunk(chunk)
        assert out.count == ref["count"]
        assert np.array_equal(out.flags, ref["flags"])
        slots, ovs = eng.verify_chunk_results(chunk)
        want = np.nonzero(ref["flags"])[0]
        assert np.array_equal(slots, want) and np.array_equal(ovs, ref["overlaps"][want])
