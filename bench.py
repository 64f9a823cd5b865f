#!/usr/bin/env python
"""Benchmark: candidate pairs verified per second on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the DBLP-like row): 1M synthetic sets, Zipf tokens over a
7,200-token universe (frequency-coded, rare first), 40..120 distinct tokens per set (avg 80),
1% near-duplicates; Jaccard 4/5; AllPairs candidates (the reference's generator,
joiners.hpp:47-71, run in parallel on the host). A full 1M-set join at 0.8 produces ~5e9
candidates, so one step verifies a fixed, stratified batch of it: `--windows` probe windows
spread evenly over the collection (so the batch has the full join's mix of set sizes),
~256M candidates = 1 GiB of C, i.e. one chunk at the paper's M_c regime (PAPER.md:827:
M_c = 4 GB). The chunk is larger than L2 (126 MB), so no L2 flush is needed between steps.

Arms:
  value  kernel-only: chunk resident in HBM, ssj_verify_chunk_device per step (CUDA events on
         the launching stream, max over ranks);
  e2e    through the C ABI with host buffers: ssj_verify_chunk from pinned C/C_O, H2D + kernels
         + D2H of the flags inside the timed region;
  parity the step's flags (all candidates) compared byte for byte with the reference's own
         VerificationEngine::verify_chunk on the same batch (the cpu_baseline leg) and with the
         committed golden digest (tests/golden/bench_golden.json); the whole-join pairs of
         `join` compared with the reference run_join's golden digest;
  --impl reference: the reference's own VerificationEngine::verify_chunk (strategy A, all host
         threads) compiled from its headers (oracle/_ref/libssjref.so) on the SAME batch, plus
         the reference run_join on the join workload. This arm never loads libssjoin_b200.so:
         its workload comes from the generator sources linked into libssjref.so
         (oracle/work_shim.cpp).

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU). Weak scaling -- every rank verifies its own
batch (different probe windows); the collection is uploaded by rank 0 and broadcast once over
NVLink (NCCL); no collective in the timed region.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "bench_golden.json")

_CFG2 = dict(sets=1_000_000, min_size=40, max_size=120, universe=7200, zipf_tokens=True,
             token_skew=1.0, duplicate_fraction=0.01, max_edits=2, distinct_tokens=True)
WORKLOADS = {
    # name: (synth kwargs, threshold, algorithm, description)
    "cfg2": (_CFG2, (4, 5), "allpairs",
             "DBLP-like Zipf self-join, 1M sets, avg 80 tokens, universe 7200, Jaccard 0.80"),
    "cfg2_085": (_CFG2, (17, 20), "allpairs",
                 "DBLP-like Zipf self-join, 1M sets, avg 80 tokens, universe 7200, Jaccard 0.85"),
    "cfg2_090": (_CFG2, (9, 10), "allpairs",
                 "DBLP-like Zipf self-join, 1M sets, avg 80 tokens, universe 7200, Jaccard 0.90"),
    "cfg2_095": (_CFG2, (19, 20), "allpairs",
                 "DBLP-like Zipf self-join, 1M sets, avg 80 tokens, universe 7200, Jaccard 0.95"),
    "cfg1": (dict(sets=100_000, min_size=5, max_size=15, universe=10_000, zipf_tokens=False,
                  duplicate_fraction=0.10, max_edits=1, distinct_tokens=True),
             (9, 10), "allpairs",
             "uniform self-join, 100K sets, avg 10 tokens, 10K-token universe, Jaccard 0.9"),
    "cfg3": (dict(sets=1_000_000, min_size=2, max_size=2500, zipf_sizes=True, size_skew=1.9,
                  universe=41_000, zipf_tokens=True, token_skew=0.6, duplicate_fraction=0.05,
                  max_edits=2),
             (3, 4), "allpairs",
             "KOSARAK-like sparse self-join, 1M sets, avg ~8 tokens, long tail, Jaccard 0.75"),
    "cfg4": (dict(sets=100_000, min_size=1, max_size=20_000, zipf_sizes=True, size_skew=1.3,
                  universe=200_000, zipf_tokens=True, token_skew=1.0, duplicate_fraction=0.02,
                  max_edits=3),
             (3, 5), "allpairs",
             "ENRON/ORKUT-like long-set self-join, 100K sets, avg ~180 tokens, max >10K, Jaccard 0.6"),
    "cfg5": (dict(sets=550_000, min_size=40, max_size=120, universe=7200, zipf_tokens=True,
                  token_skew=1.0, duplicate_fraction=0.01, max_edits=2, distinct_tokens=True),
             (4, 5), "allpairs",
             "~1B-candidate DBLP-like Zipf join, 550K sets, Jaccard 0.8 (probe-sharded)"),
}
L2_BYTES = 126 << 20  # B200 L2 (B200_PROFILING.md)
BIG = ("cfg2", "cfg2_085", "cfg2_090", "cfg2_095", "cfg5")  # stratified 256M-candidate batches
ALG = {"allpairs": 0, "ppjoin": 1, "groupjoin": 2}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def sha256(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).data).hexdigest()


def load_golden():
    try:
        with open(GOLDEN) as f:
            return json.load(f)
    except Exception:
        return {}


# ---- workload (shared by both arms; the generator is passed in) ---------------------------
def shard_probe_windows(n_sets, windows, width, rank, world):
    """Stratified probe windows for `rank` (paper_1812_09141_b200/parallel.py restated here so
    that the reference arm does not import the product package): the collection is cut into
    `windows` strides; each rank takes its own `width`-wide window inside every stride."""
    stride = n_sets // windows
    width = min(width, stride // max(world, 1))
    return [(k * stride + rank * width, min(k * stride + rank * width + width, n_sets))
            for k in range(windows)]


def batch_windows(gen, n, rank, world, target, windows):
    """The probe windows of rank `rank`'s step batch. gen(windows) -> (C, C_O). target <= 0:
    the whole join (probe shards of n / world); else `windows` stratified windows whose width is
    calibrated on a 64-probe sample to give ~target candidates."""
    if target <= 0:
        return (shard_probe_windows(n, world, n, rank, world) if world > 1 else [(0, n)]), n
    stride = n // windows
    sample_w = max(1, min(64, stride // max(world, 1)))
    cal_C, _ = gen([(k * stride, k * stride + sample_w) for k in range(windows)])
    per_probe = max(cal_C.size / (windows * sample_w), 1e-9)
    width = int(min(stride // max(world, 1), max(1, target / (per_probe * windows))))
    return shard_probe_windows(n, windows, width, rank, world), width


class OursWorkload:
    """The workload through the product library (GPU arm)."""

    def __init__(self, name, seed, threads):
        import paper_1812_09141_b200 as ssj
        self.ssj = ssj
        synth_kw, self.pred_t, self.algorithm, self.desc = WORKLOADS[name]
        self.coll = ssj.synth_collection(seed, ssj.SynthConfig(**synth_kw))
        self.tokens, self.offsets = self.coll.tokens, self.coll.offsets
        self.original_id = self.coll.original_id
        self.pred = ssj.jaccard(*self.pred_t)
        self.threads = threads

    def gen(self, wins):
        ch = self.ssj.generate_candidates_windows(self.coll, self.pred,
                                                  self.ssj.Algorithm(ALG[self.algorithm]), wins,
                                                  self.threads)
        return ch.C, ch.C_O


class RefWorkload:
    """The same workload through oracle/_ref/libssjref.so only (reference arm)."""

    def __init__(self, name, seed, threads, R):
        self.R = R
        synth_kw, self.pred_t, self.algorithm, self.desc = WORKLOADS[name]
        self.tokens, self.offsets, self.original_id = R.work_synth(seed, **synth_kw)
        self.threads = threads

    def gen(self, wins):
        return self.R.work_generate_windows(self.tokens, self.offsets, 0, self.pred_t[0],
                                            self.pred_t[1], 1, ALG[self.algorithm], wins,
                                            self.threads)


def workload_config(name, w, C, C_O, width, windows):
    """The `config` object both arms print (identical for the same workload and batch)."""
    n = int(w.offsets.size - 1)
    return {"workload": w.desc, "name": name, "n_sets": n,
            "avg_set_size": round(int(w.tokens.size) / max(n, 1), 2),
            "threshold": f"{w.pred_t[0]}/{w.pred_t[1]}", "algorithm": w.algorithm,
            "candidates_per_step_per_gpu": int(C.size), "slices_per_step": int(C_O.size // 2),
            "probe_windows": windows if name in BIG else 1, "window_width": int(width),
            "mode": "pairs (flags)",
            "l2": f"inputs larger than L2: C = {4 * C.size / 2**30:.2f} GiB per step"
                  if 4 * C.size > (126 << 20) else
                  "inputs smaller than L2 (126 MB): whole-join batch re-verified each step"}


# ---- clocks ----------------------------------------------------------------------------
class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML polled every ~2 ms
    (the timed region of a default run is tens of ms), nvidia-smi as the fallback."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = None
        self.source = "nvml"

    def _nvml_loop(self):
        import pynvml as nv
        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((float(sm), float(mx),
                                     [n for n, b in zip(self.NAMES, bits) if rs & b]))
                self._stop.wait(0.002)
        finally:
            nv.nvmlShutdown()

    def _smi_loop(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout
                f = [x.strip() for x in out.strip().split(",")]
                if len(f) >= 6:
                    self.samples.append((float(f[0]), float(f[1]),
                                         [n for n, v in zip(self.NAMES, f[2:6])
                                          if v.lower().startswith("active")]))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        def run():
            try:
                self._nvml_loop()
            except Exception:
                self.source = "nvidia-smi"
                self._smi_loop()
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        # the first sample (NVML initialised) before the timed region starts
        deadline = time.time() + 2.0
        while not self.samples and self._t.is_alive() and time.time() < deadline:
            time.sleep(0.001)
        return self

    def __exit__(self, *exc):
        # a timed region shorter than NVML's start-up still gets one sample (taken at its end,
        # while the clocks are still those of the region)
        deadline = time.time() + 2.0
        while not self.samples and self._t and self._t.is_alive() and time.time() < deadline:
            time.sleep(0.002)
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [x[0] for x in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(x[1] for x in self.samples),
                "reasons": sorted({r for x in self.samples for r in x[2]}),
                "samples": len(self.samples), "source": self.source}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(workload):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---- reference (CPU) pieces --------------------------------------------------------------
def ref_verify(R, w, C, C_O, reps, want_flags):
    """The reference's VerificationEngine::verify_chunk (strategy A, Pairs mode, all host
    threads) on the batch: (best seconds, count, flags or None, workers)."""
    h = R.coll(w.tokens, w.offsets, w.original_id)
    workers = int(R.L.ref_hardware_concurrency())
    pool = R.pool(workers)
    flags = np.zeros(max(C.size, 1), np.uint8) if want_flags else None
    sec, cnt = R.time_verify_chunk(h, pool, 0, w.pred_t[0], w.pred_t[1], 1, 0, 1, True, C, C_O,
                                   reps=reps, flags_out=flags)
    R.L.ref_pool_free(pool)
    R.L.ref_coll_free(h)
    return sec, cnt, (flags[: C.size] if want_flags else None), workers


def ref_join(R, name, seed, threads):
    """The reference's CPU run_join (pipeline.hpp:150-361) on the join workload: the same
    algorithm, Pairs mode, M_c = 64 MiB, strategy A, all host threads as workers."""
    w = RefWorkload(name, seed, threads, R)
    h = R.coll(w.tokens, w.offsets, w.original_id)
    workers = int(R.L.ref_hardware_concurrency())
    t0 = time.perf_counter()
    rep, pairs, _ = R.run_join(h, 0, w.pred_t[0], w.pred_t[1], 1, algorithm=ALG[w.algorithm],
                               budget=64 << 20, kind=0, group=1, pairs_mode=True,
                               workers=workers)
    wall = time.perf_counter() - t0
    R.L.ref_coll_free(h)
    pairs = np.ascontiguousarray(pairs, np.uint32)
    return {"workload": w.desc, "name": name, "n_sets": int(w.offsets.size - 1),
            "threshold": f"{w.pred_t[0]}/{w.pred_t[1]}", "algorithm": w.algorithm,
            "join_ms": rep["join_ms"], "wall_s": wall, "count": rep["count"],
            "candidates": rep["candidate_count"], "filtering_ms": rep["filtering_ms"],
            "serialization_ms": rep["serialization_ms"],
            "verification_ms": rep["verification_ms"], "workers": workers,
            "pairs_sha256": sha256(pairs), "n_pairs": int(pairs.shape[0]),
            "path": "reference run_join (pipeline.hpp:150-361), strategy A, Pairs mode, "
                    "M_c 64 MiB; pairs sorted like write_pairs (report.hpp:39-42)"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import pyoracle as po
    if not po.ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libssjref.so missing (reference not built)"}))
        return 0
    R = po.Ref()
    t0 = time.perf_counter()
    w = RefWorkload(args.workload, args.seed, args.threads, R)
    n = int(w.offsets.size - 1)
    wins, width = batch_windows(w.gen, n, 0, world, args.candidates, args.windows)
    C, C_O = w.gen(wins)
    config = workload_config(args.workload, w, C, C_O, width, args.windows)
    log(f"[reference] batch {C.size} candidates in {C_O.size // 2} slices "
        f"({time.perf_counter() - t0:.1f}s setup)")
    h = R.coll(w.tokens, w.offsets, w.original_id)
    workers = int(R.L.ref_hardware_concurrency())
    pool = R.pool(workers)
    for _ in range(args.warmup):
        R.time_verify_chunk(h, pool, 0, w.pred_t[0], w.pred_t[1], 1, 0, 1, True, C, C_O, reps=1)
    elapsed = 0.0
    flags = np.zeros(max(C.size, 1), np.uint8)
    cnt = 0
    for k in range(args.steps):  # each step: verify_chunk of the whole batch, timed in the shim
        sec, cnt = R.time_verify_chunk(h, pool, 0, w.pred_t[0], w.pred_t[1], 1, 0, 1, True, C,
                                       C_O, reps=1,
                                       flags_out=flags if k == args.steps - 1 else None)
        elapsed += sec
    R.L.ref_pool_free(pool)
    R.L.ref_coll_free(h)
    value = C.size * args.steps / elapsed
    join = None
    if args.join_workload != "none" and not args.no_ref_join:
        try:
            join = ref_join(R, args.join_workload, args.seed if args.join_workload != "cfg5"
                            else args.join_seed, args.threads)
        except Exception as e:  # reported, never fatal
            join = {"error": str(e)[:300]}
    line = {
        "impl": "reference", "metric": "candidate pairs verified/sec", "value": value,
        "unit": "pairs/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config,
        "arm": {"strategy": "A", "workers": workers, "mode": "Pairs",
                "path": "reference VerificationEngine::verify_chunk (verify.hpp:257-275), "
                        "oracle/_ref/libssjref.so (reference headers, -O3 -DNDEBUG)"},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": workers,
                         "kind": "reference",
                         "sample": f"the whole step batch ({C.size} candidates) per step"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "parity": {"count": int(cnt), "flags_sha256": sha256(flags[: C.size])},
        "join": join,
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- GPU arm -----------------------------------------------------------------------------
def gpu_join_shards(ssj, args, rank, world, local, dev):
    """BASELINE cfg5 (or --join-workload) self-join run entirely on the GPUs: rank r joins
    probe shard r of N (equal candidate upper bounds, no exchange step); counts summed, time
    = max over ranks of the join call (device filtering + verification + pair decoding);
    the pairs of all shards gathered on rank 0 and compared with the reference run_join's."""
    import torch
    synth_kw, pred_t, algorithm, desc = WORKLOADS[args.join_workload]
    seed = args.join_seed if args.join_workload == "cfg5" else args.seed
    coll = ssj.synth_collection(seed, ssj.SynthConfig(**synth_kw))
    pred = ssj.jaccard(*pred_t)
    alg = ALG[algorithm]
    eng = ssj.VerificationEngine(coll, pred, ssj.OutputMode.Pairs,
                                 ssj.Strategy(ssj.StrategyKind.Auto, 32), device=local)
    eng.set_original_ids(coll.original_id)
    # warm-up: the same call (static index build, bounds and buffer allocations are cached)
    eng.gpu_join(alg, pairs=True, pairs_cap=1 << 22, shard=rank, n_shards=world)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    pairs, rep = eng.gpu_join(alg, pairs=True, pairs_cap=1 << 22, shard=rank, n_shards=world)
    eng.close()
    vals = torch.tensor([rep["join_ms"], float(rep["count"]), float(rep["candidate_count"]),
                         rep["filtering_ms"], rep["verification_ms"]], dtype=torch.float64,
                        device=dev)
    if world > 1:
        import torch.distributed as dist
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        parts = [None] * world
        dist.all_gather_object(parts, pairs)
        allp = np.concatenate([p.reshape(-1, 2) for p in parts], 0)
        order = np.lexsort((allp[:, 1], allp[:, 0]))
        pairs = np.ascontiguousarray(allp[order], np.uint32)
    else:
        mx = sm = vals
    ms = float(mx[0].item())
    pairs = np.ascontiguousarray(pairs, np.uint32)
    digest = sha256(pairs)
    gold = load_golden().get("join", {}).get(args.join_workload)
    out = {"workload": desc, "name": args.join_workload, "n_sets": coll.size(),
           "threshold": f"{pred_t[0]}/{pred_t[1]}", "algorithm": algorithm, "n_gpus": world,
           "join_ms": ms, "count": int(sm[1].item()), "candidates": int(sm[2].item()),
           "candidates_per_s": float(sm[2].item()) / (ms / 1e3) if ms else None,
           "filtering_ms_max": float(mx[3].item()), "verification_ms_max": float(mx[4].item()),
           "pairs_sha256": digest, "n_pairs": int(pairs.shape[0]),
           "path": "ssj_gpu_join_shard: static index on the device, candidate generation and "
                   "verification in device-resident chunks, pairs decoded + sorted on the "
                   "device (pairs mode); rank r = probe shard r of N, no exchange step"}
    if gold:
        out["reference"] = {"join_ms": gold.get("join_ms"), "count": gold["count"],
                            "pairs_sha256": gold["pairs_sha256"],
                            "source": "tests/golden/bench_golden.json (reference run_join, "
                                      "made by tests/golden/make_bench_golden.py)"}
        out["pairs_match"] = (digest == gold["pairs_sha256"]
                              and int(pairs.shape[0]) == gold["count"])
        if gold.get("join_ms"):
            out["speedup_vs_reference_join"] = gold["join_ms"] / ms if ms else None
    return out


def spawn_ranks(args):
    """`--gpus N` outside torchrun: re-launch this script under torch.distributed.run with N
    ranks on 127.0.0.1 (one process per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--candidates", type=float, default=None,
                    help="candidates per step (default: 256M for the cfg2/cfg5 rows, the whole "
                         "join for the smaller configs)")
    ap.add_argument("--windows", type=int, default=64)
    ap.add_argument("--seed", type=int, default=1812)
    ap.add_argument("--join-seed", type=int, default=1812)
    ap.add_argument("--threads", type=int, default=0, help="host generator threads (0 = all)")
    ap.add_argument("--strategy", default="Auto")
    ap.add_argument("--group", type=int, default=32)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ref-join", action="store_true",
                    help="reference arm: skip the reference run_join on the join workload")
    ap.add_argument("--join-workload", default="cfg5",
                    help="workload of the extra whole-join measurement ('none' = off)")
    args = ap.parse_args()
    if args.candidates is None:
        args.candidates = 256e6 if args.workload in BIG else 0

    rank, world, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch "
                         "N ranks with torchrun, or run without torchrun to self-spawn)")
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import paper_1812_09141_b200 as ssj
    from paper_1812_09141_b200.parallel import broadcast_device_collection
    from paper_1812_09141_b200.verify import measure_read_bandwidth

    # one GPU per rank; with fewer visible GPUs than ranks (a functional check of the
    # multi-rank path on a single GPU) ranks share devices and use gloo instead of NCCL
    ndev = max(torch.cuda.device_count(), 1)
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if ndev >= world:
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    t0 = time.perf_counter()
    w = OursWorkload(args.workload, args.seed, args.threads)
    coll, pred, pred_t = w.coll, w.pred, w.pred_t
    wins, width = batch_windows(w.gen, coll.size(), rank, world, args.candidates, args.windows)
    C_h, CO_h = w.gen(wins)
    nC, nCO = int(C_h.size), int(CO_h.size)
    config = workload_config(args.workload, w, C_h, CO_h, width, args.windows)
    log(f"[rank {rank}] collection {coll.size()} sets avg {config['avg_set_size']}; "
        f"batch {nC} candidates in {nCO // 2} slices ({time.perf_counter() - t0:.1f}s setup)")

    strategy = ssj.Strategy(ssj.StrategyKind[args.strategy], args.group)
    mode = ssj.OutputMode.Pairs
    bcast_ms = None
    if world == 1:
        eng = ssj.VerificationEngine(coll, pred, mode, strategy, device=local)
    else:
        # rank 0 uploads once; the padded device collection is broadcast over NVLink (NCCL)
        eng0 = (ssj.VerificationEngine(coll, pred, mode, strategy, device=local)
                if rank == 0 else None)
        tb = time.perf_counter()
        eng, keep = broadcast_device_collection(eng0, coll.size(), int(coll.tokens.size),
                                                coll.offsets, pred, mode, strategy, local, rank)
        bcast_ms = 1e3 * (time.perf_counter() - tb)
    resolved = eng.strategy()          # as the reference resolves it (verify.hpp:249-253)
    kernels = eng.kernel_strategy()    # the kernel family that runs

    # ---- kernel-only arm ---------------------------------------------------------------
    dC = torch.from_numpy(C_h.view(np.int32)).to(dev)
    dCO = torch.from_numpy(CO_h.view(np.int32)).to(dev)
    dF = torch.empty(nC, dtype=torch.uint8, device=dev)
    dR = torch.zeros(8, dtype=torch.int64, device=dev)
    dB = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(device=dev)  # a real stream handle (not the legacy default)
    sp = stream.cuda_stream
    torch.cuda.synchronize()
    eng.chunk_algorithmic_bytes_device(dC.data_ptr(), nC, dCO.data_ptr(), nCO, dB.data_ptr(), sp)
    torch.cuda.synchronize()
    algo_bytes = int(dB.item())

    def step():
        eng.verify_chunk_device(dC.data_ptr(), nC, dCO.data_ptr(), nCO, dF.data_ptr(),
                                dR.data_ptr(), sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    words = dR.cpu().numpy()
    ssj.result_error(words)
    count = int(words[0])

    eng.set_profiling(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    kernel_ms, launches = eng.kernel_time()
    eng.set_profiling(False)
    if world > 1:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
        tot = torch.tensor([float(nC)], dtype=torch.float64, device=dev)
        dist.all_reduce(tot, op=dist.ReduceOp.SUM)
        total_pairs = float(tot.item()) * args.steps
    else:
        total_pairs = float(nC) * args.steps
    value = total_pairs / (elapsed_ms / 1e3)
    kernel_avg_ms = kernel_ms / max(launches, 1)
    gpu_flags = dF.cpu().numpy()
    assert int(gpu_flags.sum(dtype=np.int64)) == count
    flags_digest = sha256(gpu_flags)

    hbm_peak, peak_src = measured_peaks()
    achieved_gbs = algo_bytes / (kernel_avg_ms / 1e3) / 1e9
    l2_gbs = measure_read_bandwidth(local, 48 << 20, 50)
    hbm_read_gbs = measure_read_bandwidth(local, 4 << 30, 5)
    traffic = ncu_traffic(args.workload)
    # the working set decides the denominator: when the dominant kernel's measured DRAM bytes
    # are well below its algorithmic bytes (or, without an ncu capture, when the device
    # collection -- padded tokens, 32-byte head records, 8-byte descriptors -- fits in L2),
    # the data is served by L2 and L2 bounds it
    footprint = 4 * eng.device_collection()[1] + 40 * coll.size()
    l2_bound = (traffic < 0.5 * algo_bytes) if traffic is not None else footprint < L2_BYTES
    bound, peak = ("l2", l2_gbs) if l2_bound else ("hbm", hbm_peak)

    # ---- end-to-end arm: C ABI with pinned host buffers ---------------------------------
    pc = ssj.PinnedBuffer(4 * nC + 64)
    pco = ssj.PinnedBuffer(4 * nCO + 64)
    pf = ssj.PinnedBuffer(nC + 64)
    hC = pc.view(np.uint32, nC)
    hC[:] = C_h
    hCO = pco.view(np.uint32, nCO)
    hCO[:] = CO_h
    hF = pf.view(np.uint8, nC)
    host_chunk = ssj.CandidateChunk.__new__(ssj.CandidateChunk)
    host_chunk.C, host_chunk.C_O = hC, hCO
    for _ in range(2):  # warm-up: both chunk slots of the engine (double buffering)
        eng.verify_chunk(host_chunk, flags_out=hF)
    if world > 1:
        dist.barrier()
    te = time.perf_counter()
    for _ in range(args.e2e_steps):
        out = eng.verify_chunk(host_chunk, flags_out=hF)
    e2e_s = time.perf_counter() - te
    assert out.count == count, (out.count, count)
    e2e_flags_identical = bool(np.array_equal(hF, gpu_flags))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = (total_pairs / args.steps) * args.e2e_steps / e2e_s
    launches_per_step = int(eng.launches_per_chunk(nC, nCO))
    eng.close()

    # ---- the whole join on the GPU(s): device filtering + verification, probe shards -----
    join = None
    if args.join_workload != "none":
        try:
            join = gpu_join_shards(ssj, args, rank, world, local, dev)
        except Exception as e:  # reported, never fatal
            join = {"error": str(e)[:300]}

    # ---- CPU baseline + full-batch parity (rank 0) --------------------------------------
    cpu = None
    gold = load_golden().get("batches", {}).get(args.workload)
    parity = {"count": count, "flags_sha256": flags_digest,
              "e2e_flags_identical": e2e_flags_identical}
    if gold and gold.get("seed") == args.seed and gold.get("candidates") == nC and rank == 0:
        parity["golden"] = {"count": gold["count"], "flags_sha256": gold["flags_sha256"],
                            "source": "tests/golden/bench_golden.json (reference verify_chunk, "
                                      "made by tests/golden/make_bench_golden.py)"}
        parity["golden_match"] = (gold["flags_sha256"] == flags_digest
                                  and gold["count"] == count)
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle import pyoracle as po
            if not po.ref_available():
                raise RuntimeError("oracle/_ref/libssjref.so missing")
            R = po.Ref()
            sec, ref_count, ref_flags, cores = ref_verify(R, w, C_h, CO_h, args.cpu_reps, True)
            cpu = {"value": nC / sec, "unit": "pairs/s", "cores": cores, "kind": "reference",
                   "sample": f"the whole step batch of rank 0 ({nC} candidates), reference "
                             f"VerificationEngine::verify_chunk strategy A, Pairs mode, "
                             f"best of {args.cpu_reps}"}
            parity.update({"reference_count": int(ref_count),
                           "reference_flags_sha256": sha256(ref_flags),
                           "candidates_compared": nC,
                           "flags_match": bool(np.array_equal(ref_flags, gpu_flags))
                           and int(ref_count) == count})
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "pairs/s", "cores": 0, "kind": "unavailable",
                   "sample": str(e)[:200]}
    if world > 1:
        dist.barrier()

    if rank == 0:
        line = {
            "metric": "candidate pairs verified/sec", "value": value, "unit": "pairs/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config,
            "parallelism": f"probe-window shards x{world}, no data-path collective",
            "arm": {"strategy": f"{resolved.kind.name}/{resolved.group_size}",
                    "kernels": f"{kernels.kind.name}/{kernels.group_size}",
                    "qualifying_per_step": count, "collection_broadcast_ms": bcast_ms},
            "roofline": {
                "bound": bound, "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
                "frac": achieved_gbs / peak, "traffic": traffic,
                "kernel": "strategy-A verification pass (prep + bitmap + run_kernel + "
                          "warp_tile_kernel + long_slice_kernel; run_kernel dominant)"
                          if kernels.kind.name == "A" else
                          f"strategy {kernels.kind.name} kernel",
                "algorithmic_bytes_per_launch": algo_bytes,
                "kernel_ms_avg": kernel_avg_ms,
                "kernel_share_of_step": kernel_ms / elapsed_ms if elapsed_ms else None,
                "bound_rule": "l2 when the dominant kernel's ncu DRAM bytes < 0.5 x its "
                              "algorithmic bytes (profiles/ncu_traffic.json) or, without a "
                              "capture, when the device collection fits in L2; else hbm",
                "collection_footprint_bytes": footprint,
                "l2_peak_gbs": l2_gbs, "l2_frac": achieved_gbs / l2_gbs,
                "l2_peak_source": "measured in this run: streaming 16-byte reads of a 48 MiB "
                                  "L2-resident buffer (ssj_measure_read_bandwidth)",
                "hbm_peak_gbs": hbm_peak, "hbm_frac": achieved_gbs / hbm_peak,
                "hbm_peak_source": peak_src, "hbm_read_measured_gbs": hbm_read_gbs,
            },
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": "pairs/s",
                    "h2d_bytes_per_step": int(4 * nC + 4 * nCO),
                    "d2h_bytes_per_step": int(nC + 64), "steps": args.e2e_steps,
                    "path": "ssj_verify_chunk (C ABI) from pinned host buffers, flags D2H"},
            "gpu_launches": int(args.steps * launches_per_step),
            "join": join,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
