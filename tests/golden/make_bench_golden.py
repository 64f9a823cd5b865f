"""Golden digests of bench.py's workloads, made by the REFERENCE (oracle/_ref/libssjref.so).

For every bench workload: the step batch (rank 0 / one GPU) is built exactly as bench.py
builds it (bench.RefWorkload + bench.batch_windows: the synthetic collection and the
candidate generator linked into libssjref.so), verified by the reference's own
VerificationEngine::verify_chunk (verify.hpp:257-275, strategy A, Pairs mode), and its flags
are recorded as a sha256 + count. For the join workload (cfg5) the reference run_join
(pipeline.hpp:150-361, Pairs mode) is run and its sorted pairs (report.hpp:39-42) recorded.

bench.py and tests/test_gpu_scale.py compare the GPU's flags / pairs with these digests at
full BASELINE size. Run in this container (needs /root/reference to build the shim):
    make -C oracle ref && python tests/golden/make_bench_golden.py [workload ...]
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import pyoracle as po  # noqa: E402

OUT = os.path.join(HERE, "bench_golden.json")
BATCHES = ["cfg1", "cfg2", "cfg2_085", "cfg2_090", "cfg2_095", "cfg3", "cfg4", "cfg5"]
JOINS = ["cfg5"]
SEED = 1812
WINDOWS = 64


def main(argv):
    want = set(argv) if argv else None
    R = po.Ref()
    try:
        with open(OUT) as f:
            gold = json.load(f)
    except Exception:
        gold = {}
    gold.setdefault("batches", {})
    gold.setdefault("join", {})
    gold["generator"] = ("tests/golden/make_bench_golden.py: reference verify_chunk / run_join "
                         "via oracle/_ref/libssjref.so")
    for name in BATCHES:
        if want and name not in want:
            continue
        t0 = time.time()
        w = bench.RefWorkload(name, SEED, 0, R)
        n = int(w.offsets.size - 1)
        target = 256e6 if name in bench.BIG else 0
        wins, width = bench.batch_windows(w.gen, n, 0, 1, target, WINDOWS)
        C, C_O = w.gen(wins)
        sec, cnt, flags, workers = bench.ref_verify(R, w, C, C_O, 1, True)
        gold["batches"][name] = {"seed": SEED, "windows": WINDOWS if name in bench.BIG else 1,
                                 "window_width": int(width), "candidates": int(C.size),
                                 "slices": int(C_O.size // 2), "count": int(cnt),
                                 "flags_sha256": bench.sha256(flags),
                                 "c_sha256": bench.sha256(C), "c_o_sha256": bench.sha256(C_O)}
        print(f"{name}: {C.size} candidates, {cnt} qualifying ({time.time() - t0:.1f}s, "
              f"verify {sec:.2f}s on {workers} threads)", flush=True)
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1, sort_keys=True)
    for name in JOINS:
        if want and "join:" + name not in want:
            continue
        j = bench.ref_join(R, name, SEED, 0)
        gold["join"][name] = {"seed": SEED, "count": j["count"], "pairs_sha256": j["pairs_sha256"],
                              "candidates": j["candidates"], "join_ms": j["join_ms"],
                              "join_workers": j["workers"]}
        print(f"join {name}: {j['count']} pairs, {j['candidates']} candidates, "
              f"{j['join_ms'] / 1e3:.1f}s on {j['workers']} workers", flush=True)
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])
