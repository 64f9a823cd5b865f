#!/usr/bin/env python
"""One all-GPU join of a bench workload (for profiling the device generator).
    python tools/gpu_join_once.py [--workload cfg5] [--alg 0]"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1812_09141_b200 as ssj  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg5")
ap.add_argument("--alg", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
kw, pt, alg, desc = bench.WORKLOADS[a.workload]
coll = ssj.synth_collection(1812, ssj.SynthConfig(**kw))
eng = ssj.VerificationEngine(coll, ssj.jaccard(*pt), ssj.OutputMode.Pairs,
                             ssj.Strategy(ssj.StrategyKind.Auto, 32))
for _ in range(a.reps):
    _, rep = eng.gpu_join(a.alg, pairs=False)
    print(json.dumps(rep))
