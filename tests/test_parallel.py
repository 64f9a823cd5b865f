"""Multi-process (N > 1) host logic on CPU with gloo, world_size 2: probe-window sharding is
disjoint and complete across ranks, the padded collection broadcast from rank 0 equals every
rank's own layout, and the max-over-ranks timing reduction. The GPU half (export ->
broadcast -> engine from device) is in test_gpu_parallel below."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_dir):
    import torch
    import torch.distributed as dist

    import paper_1812_09141_b200 as ssj
    from paper_1812_09141_b200.parallel import padded_layout, padded_tokens, shard_probe_windows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    coll = ssj.synth_collection(7, ssj.SynthConfig(sets=3000, min_size=3, max_size=40,
                                                   universe=500, zipf_tokens=True,
                                                   duplicate_fraction=0.05, max_edits=1))
    # sharding
    wins = shard_probe_windows(coll.size(), 16, 40, rank, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, wins)
    # broadcast of the padded collection (rank 0 -> all)
    n_pad, sets = padded_layout(coll.offsets)
    mine = padded_tokens(coll.tokens, coll.offsets).view(np.int32)
    buf = torch.from_numpy(mine.copy()) if rank == 0 else torch.zeros(n_pad, dtype=torch.int32)
    dist.broadcast(buf, 0)
    same = bool(np.array_equal(buf.numpy(), mine))
    # max over ranks
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    np.save(os.path.join(result_dir, f"r{rank}.npy"),
            np.array([same, t.item() == world, repr(gathered) != ""], dtype=object),
            allow_pickle=True)
    if rank == 0:
        import pickle
        with open(os.path.join(result_dir, "wins.pkl"), "wb") as f:
            pickle.dump(gathered, f)
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_and_broadcast(tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    import pickle
    for r in range(2):
        same, maxok, _ = np.load(tmp_path / f"r{r}.npy", allow_pickle=True)
        assert same and maxok
    wins = pickle.load(open(tmp_path / "wins.pkl", "rb"))
    probes = [set() for _ in range(2)]
    for r in range(2):
        for lo, hi in wins[r]:
            probes[r].update(range(lo, hi))
    assert probes[0] and probes[1] and not (probes[0] & probes[1])
    assert len(probes[0]) == len(probes[1])


def test_padded_layout_matches_definition(ssj):
    from paper_1812_09141_b200.parallel import TOKEN_TAIL_PAD, padded_layout, padded_tokens
    coll = ssj.Collection.from_sets([[1, 2, 3], [], list(range(9)), [7]])
    n_pad, sets = padded_layout(coll.offsets)
    assert sets.tolist() == [0, 3, 1, 0, 1, 9, 3, 1]
    assert n_pad == 8 + 0 + 16 + 8 + TOKEN_TAIL_PAD
    pt = padded_tokens(coll.tokens, coll.offsets)
    assert pt[:3].tolist() == [1, 2, 3] and pt[3] == 0xFFFFFFFF
    assert pt[8:17].tolist() == list(range(9)) and pt[24] == 7


@pytest.mark.gpu
def test_gpu_export_and_engine_from_device(ssj, gpu, oracle):
    """The engine's exported device collection equals the host layout, and an engine built
    on it (the NCCL-broadcast path) verifies identically."""
    import torch
    from paper_1812_09141_b200.parallel import padded_layout, padded_tokens
    coll = ssj.synth_collection(11, ssj.SynthConfig(sets=5000, min_size=5, max_size=60,
                                                    universe=900, zipf_tokens=True,
                                                    duplicate_fraction=0.05, max_edits=2))
    pred = ssj.jaccard(7, 10)
    chunk, _ = ssj.generate_candidates(coll, pred, ssj.Algorithm.AllPairs, threads=4)
    eng = ssj.VerificationEngine(coll, pred, ssj.OutputMode.Pairs, ssj.Strategy())
    n_pad, sets = padded_layout(coll.offsets)
    d_tok = torch.empty(n_pad, dtype=torch.int32, device="cuda:0")
    d_sets = torch.empty(sets.size, dtype=torch.int32, device="cuda:0")
    eng.export_collection(d_tok.data_ptr(), d_sets.data_ptr(), 0)
    torch.cuda.synchronize()
    assert np.array_equal(d_tok.cpu().numpy().view(np.uint32), padded_tokens(coll.tokens, coll.offsets))
    assert np.array_equal(d_sets.cpu().numpy().view(np.uint32), sets)
    eng2 = ssj.VerificationEngine.from_device(d_tok.data_ptr(), n_pad, d_sets.data_ptr(),
                                              coll.size(), coll.tokens.size, pred,
                                              ssj.OutputMode.Pairs, ssj.Strategy())
    a, b = eng.verify_chunk(chunk), eng2.verify_chunk(chunk)
    ref = oracle.verify_chunk(coll.tokens, coll.offsets, chunk.C, chunk.C_O, oracle.pred(0, 7, 10))
    assert np.array_equal(a.flags, ref["flags"]) and np.array_equal(b.flags, ref["flags"])
    eng2.close()
    # a device collection without the tail pad (the kernels read past a set's end) is refused
    with pytest.raises(Exception, match="tail pad"):
        ssj.VerificationEngine.from_device(d_tok.data_ptr(), n_pad - 1, d_sets.data_ptr(),
                                           coll.size(), coll.tokens.size, pred,
                                           ssj.OutputMode.Pairs, ssj.Strategy())
    eng.close()
