"""Generate the golden vectors under tests/golden/ from the REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libssjref.so, compiled from the
read-only reference headers by `make -C oracle ref`). Every fixture is produced by calling
the reference's own functions (similarity.hpp, verify.hpp, chunk.hpp, joiners.hpp,
oracle.hpp, pipeline.hpp) through oracle/ref_shim.cpp; nothing here re-implements them.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402

J, COS, DICE, OV = 0, 1, 2, 3


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def pack_sets(sets):
    offs = np.zeros(len(sets) + 1, np.uint32)
    offs[1:] = np.cumsum([len(s) for s in sets])
    toks = np.concatenate([np.asarray(s, np.uint32) for s in sets]) if offs[-1] else np.zeros(0, np.uint32)
    return toks, offs


def main():
    R = po.Ref()

    # 1. similarity.hpp: equivalent_overlap grid (test_similarity.cpp:79-102 domain) and
    #    Threshold::parse cases (test_similarity.cpp:18-29).
    grid = np.zeros((3, 20, 50, 50), np.uint8)
    meets = np.zeros((3, 20, 50, 50), np.uint64)  # bitmask over overlap o in [0, 50]
    for fi, fn in enumerate((J, COS, DICE)):
        for tn in range(1, 21):
            for r in range(1, 51):
                for s in range(1, 51):
                    grid[fi, tn - 1, r - 1, s - 1] = R.equivalent_overlap(fn, tn, 20, 1, r, s)
                    m = 0
                    for o in range(0, min(r, s) + 1):
                        if R.meets_threshold(fn, tn, 20, 1, o, r, s):
                            m |= 1 << o
                    meets[fi, tn - 1, r - 1, s - 1] = m
    parse_in = ["0.8", ".85", "1", "1.0", "4/5", "0.95", "0.6", "3/4", "0.50", "19/20", "7/10",
                "2/4", "0.333"]
    parse_out = np.array([R.threshold_parse(t) for t in parse_in], np.uint64)
    # large / odd thresholds exercise the u128 paths
    big = [(J, (1 << 40) + 3, (1 << 41) + 7), (DICE, (1 << 35) + 1, (1 << 35) + 9),
           (COS, 999983, 1000003), (J, 4, 5), (COS, 1, 2), (DICE, 17, 20)]
    big_cases = []
    rng = np.random.default_rng(7)
    for fn, num, den in big:
        for _ in range(200):
            r = int(rng.integers(0, 20000))
            s = int(rng.integers(0, 20000))
            big_cases.append((fn, num, den, r, s, R.equivalent_overlap(fn, num, den, 1, r, s)))
    save("similarity", eqo_grid=grid, meets_mask=meets,
         parse_in=np.array(parse_in), parse_out=parse_out,
         big_cases=np.array(big_cases, np.uint64))

    # 2. verify.hpp:50-72 verify_pair_count on random pairs (test_verify.cpp:59-72 shape).
    rng = np.random.default_rng(17)
    rs, ss, req, out = [], [], [], []
    for _ in range(5000):
        r = np.sort(rng.choice(60, size=int(rng.integers(1, 31)), replace=False))
        s = np.sort(rng.choice(60, size=int(rng.integers(1, 31)), replace=False))
        q = int(rng.integers(0, min(r.size, s.size) + 2))
        rs.append(r)
        ss.append(s)
        req.append(q)
        out.append(R.verify_pair_count(r, s, q))
    rt, ro = pack_sets(rs)
    st, so = pack_sets(ss)
    save("pair_count", r_tokens=rt, r_offsets=ro, s_tokens=st, s_offsets=so,
         required=np.array(req, np.uint64),
         overlap=np.array([o[0] for o in out], np.uint64),
         met=np.array([o[1] for o in out], np.uint8),
         comparisons=np.array([o[2] for o in out], np.uint32))

    # 3. verify.hpp:86-166 intersect-path partitions (test_verify.cpp:86-118 shape).
    rng = np.random.default_rng(23)
    rs, ss, parts, counts = [], [], [], []
    Bs = [1, 2, 4, 8, 32, 128]
    for _ in range(300):
        uni = int(rng.integers(1, 301))
        m = min(int(rng.integers(0, 200)), uni)
        n = min(int(rng.integers(1, 200)), uni)
        r = np.sort(rng.choice(uni, size=m, replace=False))
        s = np.sort(rng.choice(uni, size=n, replace=False))
        rs.append(r)
        ss.append(s)
        pp, cc = [], []
        for B in Bs:
            p, c = R.intersect_path_partitions(r, s, B)
            pp.append(p)
            cc.append(c)
        parts.append(np.concatenate(pp))
        counts.append(np.concatenate(cc))
    rt, ro = pack_sets(rs)
    st, so = pack_sets(ss)
    save("partitions", r_tokens=rt, r_offsets=ro, s_tokens=st, s_offsets=so,
         group_sizes=np.array(Bs, np.uint32), parts=np.stack(parts), counts=np.stack(counts))

    # 4. Collections from the reference generator (oracle.hpp:83-125 + preprocess), with
    #    the reference's candidate streams, verify_chunk flags, stats and brute-force pairs.
    def coll_fixture(name, seed, preds, algs=(0, 1, 2), **cfg):
        t, o, oid = R.synth(seed, **cfg)
        h = R.coll(t, o, oid)
        pool = R.pool(4)
        arrays = dict(tokens=t, offsets=o, original_id=oid)
        for (fn, num, den) in preds:
            bf = R.brute_force(h, fn, num, den, 1)
            arrays[f"bf_{fn}_{num}_{den}"] = bf
            for alg in algs:
                C_, CO, hp = R.generate(h, fn, num, den, 1, alg)
                key = f"{fn}_{num}_{den}_a{alg}"
                arrays["C_" + key] = C_
                arrays["CO_" + key] = CO
                arrays["host_" + key] = hp
                flags, cnt, stats, _ = R.verify_chunk(h, pool, fn, num, den, 1, 0, 1, True, C_, CO)
                arrays["flags_" + key] = flags
                arrays["count_" + key] = np.array([cnt], np.uint64)
                arrays["stats_" + key] = stats
                arrays["bytes_" + key] = np.array(
                    [po.chunk_algorithmic_bytes(t, o, C_, CO, po.pred(fn, num, den))], np.uint64)
        save(name, **arrays)

    for seed in (41, 42, 43):  # test_verify.cpp:168-204
        coll_fixture(f"verify_s{seed}", seed, [(J, 7, 10), (J, 1, 2)], sets=200, min_size=1,
                     max_size=120 if seed == 43 else 25, universe=200)
    for seed in (101, 202, 707):  # test_pipeline.cpp:11-19 medium_collection
        coll_fixture(f"medium_s{seed}", seed, [(J, 1, 2), (J, 4, 5), (J, 2, 3), (COS, 3, 4),
                                               (DICE, 4, 5)],
                     sets=600, min_size=1, max_size=40, universe=150, duplicate_fraction=0.15)
    # acceptance.cpp:243-263 oracle sweep (first seeds): uniform, zipf, zipf+dups
    for i in range(3):
        cfg = dict(sets=100 * (1 + i % 10), min_size=1, max_size=50, universe=2000)
        if i % 3 == 1:
            cfg.update(zipf_tokens=True, token_skew=1.0)
        if i % 3 == 2:
            cfg.update(universe=500, zipf_tokens=True, token_skew=1.0, duplicate_fraction=0.4)
        coll_fixture(f"sweep_s{1000 + i}", 1000 + i, [(J, tn, 20) for tn in (10, 14, 17, 19)],
                     algs=(1,), **cfg)

    # 5. pipeline.hpp:150-361 run_join chunk streams under small budgets (chunk_observer),
    #    test_pipeline.cpp:52-91.
    t, o, oid = R.synth(303, sets=600, min_size=1, max_size=40, universe=150,
                        duplicate_fraction=0.15)
    h = R.coll(t, o, oid)
    arrays = dict(tokens=t, offsets=o, original_id=oid)
    for budget in (256, 16 << 10):
        rep, pairs, chunks = R.run_join(h, J, 1, 2, 1, algorithm=1, budget=budget, kind=0,
                                        group=1, pairs_mode=True, workers=2, record_chunks=True)
        arrays[f"pairs_{budget}"] = pairs
        arrays[f"nchunks_{budget}"] = np.array([len(chunks)], np.uint64)
        arrays[f"C_{budget}"] = np.concatenate([c[0] for c in chunks])
        arrays[f"CO_{budget}"] = np.concatenate([c[1] for c in chunks])
        arrays[f"flags_{budget}"] = np.concatenate([c[2] for c in chunks])
        arrays[f"nC_{budget}"] = np.array([c[0].size for c in chunks], np.uint64)
        arrays[f"nCO_{budget}"] = np.array([c[1].size for c in chunks], np.uint64)
        arrays[f"counts_{budget}"] = np.array([c[3] for c in chunks], np.uint64)
        arrays[f"report_{budget}"] = np.array(
            [rep["count"], rep["chunk_count"], rep["candidate_count"], rep["pairs_verified"],
             rep["early_exit_prunes"]], np.uint64)
    save("pipeline_s303", **arrays)

    # 6. acceptance.cpp:230-264 criterion 4: seed 777, 5000 sets, J = 1/2 -> 30,092 bytes.
    t, o, oid = R.synth(777, sets=5000, min_size=1, max_size=50, universe=400,
                        zipf_tokens=True, duplicate_fraction=0.2)
    h = R.coll(t, o, oid)
    rep, pairs, _ = R.run_join(h, J, 1, 2, 1, algorithm=1, budget=64 << 10, kind=3, group=32,
                               pairs_mode=True, workers=4)
    text = f"{rep['count']}\n" + "".join(f"{a}\t{b}\n" for a, b in pairs)
    save("c4_s777", tokens=t, offsets=o, original_id=oid,
         out_size=np.array([len(text.encode())], np.uint64),
         out_sha256=np.array([hashlib.sha256(text.encode()).hexdigest()]),
         count=np.array([rep["count"]], np.uint64))
    print("C4 golden size", len(text.encode()))


if __name__ == "__main__":
    main()
