"""Full-size parity on the BASELINE configs: the bench batches (257.6M candidates for the
DBLP-like rows) verified on the GPU, flags compared byte for byte with the reference.

The golden digests (tests/golden/bench_golden.json) were made by the REFERENCE's own
VerificationEngine::verify_chunk on the same batches (tests/golden/make_bench_golden.py);
the batch itself is checked against the golden C / C_O digests first, so a mismatch cannot
hide in the workload generator. The reference shim (when built) is also run live on the whole
batch, and the C oracle on a stratified 3M-candidate subset of it."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "bench_golden.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).data).hexdigest()


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg2_085", "cfg2_090", "cfg2_095", "cfg3",
                                  "cfg4", "cfg5"])
def test_bench_batch_flags_match_reference(ssj, gpu, oracle, name):
    import bench
    g = GOLD["batches"][name]
    w = bench.OursWorkload(name, g["seed"], 0)
    target = 256e6 if name in bench.BIG else 0
    wins, width = bench.batch_windows(w.gen, w.coll.size(), 0, 1, target, g["windows"])
    C, CO = w.gen(wins)
    assert (int(C.size), sha(C), sha(CO)) == (g["candidates"], g["c_sha256"], g["c_o_sha256"])
    with ssj.VerificationEngine(w.coll, w.pred, ssj.OutputMode.Pairs,
                                ssj.Strategy(ssj.StrategyKind.Auto, 32)) as eng:
        out = eng.verify_chunk(ssj.CandidateChunk(C, CO))
    assert out.count == g["count"]
    assert sha(out.flags) == g["flags_sha256"]
    # the C oracle on every k-th slice (a stratified ~3M-candidate subset)
    sub_C, sub_CO, idx = bench_subset(C, CO, 3_000_000)
    ref = oracle.verify_chunk(w.tokens, w.offsets, sub_C, sub_CO, oracle.pred(0, *w.pred_t))
    assert np.array_equal(out.flags[idx], ref["flags"])
    # the reference itself, live, on the whole batch
    if oracle.ref_available():
        R = oracle.Ref()
        sec, cnt, flags, _ = bench.ref_verify(R, w, C, CO, 1, True)
        assert cnt == out.count and np.array_equal(flags, out.flags)


def bench_subset(C, CO, sample):
    CO = CO.reshape(-1, 2).astype(np.int64)
    ends = CO[:, 1]
    begins = np.concatenate([[0], ends[:-1]])
    k = max(1, int(np.ceil(ends[-1] / sample)))
    pick = np.arange(0, CO.shape[0], k)
    lens = ends[pick] - begins[pick]
    idx = np.concatenate([np.arange(b, e) for b, e in zip(begins[pick], ends[pick])])
    sub_CO = np.stack([CO[pick, 0], np.cumsum(lens)], 1).reshape(-1).astype(np.uint32)
    return C[idx], sub_CO, idx


def test_cfg5_join_pairs_match_reference_run_join(ssj, gpu):
    """The whole cfg5 self-join (1.65G AllPairs candidates) on the GPU, in Pairs mode: the
    sorted pairs equal the reference run_join's (write_pairs order, report.hpp:39-42)."""
    import bench
    g = GOLD["join"]["cfg5"]
    synth_kw, pred_t, algorithm, _ = bench.WORKLOADS["cfg5"]
    coll = ssj.synth_collection(g["seed"], ssj.SynthConfig(**synth_kw))
    with ssj.VerificationEngine(coll, ssj.jaccard(*pred_t), ssj.OutputMode.Pairs,
                                ssj.Strategy(ssj.StrategyKind.Auto, 32)) as eng:
        eng.set_original_ids(coll.original_id)
        pairs, rep = eng.gpu_join(0, pairs=True, pairs_cap=1 << 22)
    assert rep["candidate_count"] == g["candidates"]
    assert rep["count"] == g["count"] == len(pairs)
    assert sha(np.ascontiguousarray(pairs, np.uint32)) == g["pairs_sha256"]
