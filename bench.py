#!/usr/bin/env python3
"""Benchmark of the LCP-indexed top-k hot path (BASELINE.json metric).

Workload (N=1): BASELINE config 3 — N=2,000,000 items, L=32, sigma=4, k=10,
complete-mode top-k over batches of 4,096 queries.  A "step" is one batch
through the fused query kernel (pack -> 64-ary search -> window d* -> range
scan -> warp top-k), inputs resident in HBM.  L2 is flushed (256 MiB memset)
before every timed step and each step is bracketed by its own CUDA events on
the launching stream.  Inputs come from the reference generator restated in
paper_2602_04936_b200.datagen (byte-identical Philox streams).

N>1 (torchrun): row-block shards of 2M items per rank (weak scaling; rank g
holds generate_dataset(2M, 32, 4, seed=3+g) with ids offset by 2M*g), the
query batch is broadcast, and each step is local query -> encode ->
NCCL all_gather -> merge kernel.  value = queries/s over the whole corpus.

``--impl reference`` times the reference's own algorithm on the host CPU
(the pinned C restatement in oracle/, all host threads) on the same config.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "top-k LCP queries/sec at N=2M, L=32, k=10 (HBM GB/s frac); p50 latency; J/query"
N_ITEMS, SEQ_LEN, SIGMA, K, BATCH = 2_000_000, 32, 4, 10, 4096
FALLBACK_HBM_GBS = 6650.0


def algorithmic_key_bytes(length: int, sigma: int) -> int:
    """K_b = ceil(L * ceil(log2 sigma) / 8)   (SURVEY §8 notation)."""
    bits = max(1, int(np.ceil(np.log2(sigma))))
    return (length * bits + 7) // 8


def indexed_bytes_per_query(n: int, length: int, sigma: int, k: int, rsize: np.ndarray) -> np.ndarray:
    """K_b*ceil(log2(N+1)) + |R(d*)|*(K_b+4) + K_b + 6k."""
    kb = algorithmic_key_bytes(length, sigma)
    return kb * int(np.ceil(np.log2(n + 1))) + rsize.astype(np.float64) * (kb + 4) + kb + 6 * k


def hbm_peak() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int = 0):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.15)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        time.sleep(0.1)
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def nvml_energy():
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("LOCAL_RANK", "0")))
        return lambda: pynvml.nvmlDeviceGetTotalEnergyConsumption(h) / 1000.0  # J
    except Exception:
        return None


# --------------------------------------------------------------------------
def cpu_reference(ds, queries: np.ndarray, k: int, budget_s: float, nthreads: int):
    """Time the reference algorithm (C port in oracle/) on the host cores."""
    import oracle

    oracle.build()
    trie = oracle.OracleTrie(ds.items, SIGMA)
    trie.query_batch(queries[:256], k, "complete", nthreads=nthreads)  # warm
    done, t0 = 0, time.perf_counter()
    nb = queries.shape[0] // BATCH
    i = 0
    while True:
        qb = queries[(i % nb) * BATCH:((i % nb) + 1) * BATCH]
        trie.query_batch(qb, k, "complete", nthreads=nthreads)
        done += qb.shape[0]
        i += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    return done / el, done, el, trie


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2602_04936_b200.datagen as dg
    import oracle

    ds = dg.generate_dataset(N_ITEMS, SEQ_LEN, SIGMA, seed=3)
    qs = dg.generate_queries(ds, BATCH * 4, seed=4)
    nthreads = os.cpu_count() or 1
    oracle.build()
    trie = oracle.OracleTrie(ds.items, SIGMA)
    for w in range(args.warmup):
        trie.query_batch(qs[(w % 4) * BATCH:(w % 4 + 1) * BATCH], K, "complete", nthreads=nthreads)
    times = []
    for s in range(args.steps):
        qb = qs[(s % 4) * BATCH:(s % 4 + 1) * BATCH]
        t0 = time.perf_counter()
        trie.query_batch(qb, K, "complete", nthreads=nthreads)
        times.append(time.perf_counter() - t0)
    total = float(np.sum(times))
    value = BATCH * args.steps / total
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16",
        "data": "synthetic: generate_dataset(2_000_000, 32, 4, seed=3), generate_queries(seed=4)",
        "config": {"workload": "config 3: indexed complete-mode top-k, 4096-query batches",
                   "n_items": N_ITEMS, "seq_len": SEQ_LEN, "alphabet": SIGMA, "k": K,
                   "batch": BATCH, "mode": "complete", "parallelism": "host threads"},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": nthreads, "kind": "port",
                         "sample": f"{args.steps} batches x {BATCH} queries; C restatement of "
                                   "trie.build/TrieIndex.query (oracle/lcp_oracle.c), pthreads"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def time_steps(fn, flush, steps: int, stream):
    """Per-step CUDA events on `stream`, L2 flushed before each step."""
    import torch

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        if flush is not None:
            flush()
        evs[i][0].record(stream)
        fn(i)
        evs[i][1].record(stream)
    return evs


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget-s", type=float, default=10.0)
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2602_04936_b200 as lg
    from paper_2602_04936_b200 import _build
    from paper_2602_04936_b200.engine import NativeIndex

    if _build.needs_build():
        _build.build_native()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)

    ds = lg.generate_dataset(N_ITEMS, SEQ_LEN, SIGMA, seed=3 + rank)
    n_pool = 8
    qs = lg.generate_queries(ds, BATCH * n_pool, seed=4)  # uniform queries: identical on every rank
    stream = torch.cuda.Stream(device=dev)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    kbytes = algorithmic_key_bytes(SEQ_LEN, SIGMA)

    with torch.cuda.stream(stream):
        t_build = time.perf_counter()
        if world == 1:
            idx = lg.build(ds)
            native = idx.native
        else:
            from paper_2602_04936_b200.sharded import ShardedIndex

            sh = ShardedIndex(ds.items, SEQ_LEN, SIGMA, id_offset=N_ITEMS * rank)
            native = sh.local
        torch.cuda.synchronize()
        t_build = time.perf_counter() - t_build

        dq = torch.from_numpy(qs).to(dev).view(n_pool, BATCH, SEQ_LEN)
        stride = min(K, N_ITEMS * world)
        ids = torch.empty((BATCH, stride), dtype=torch.int32, device=dev)
        lcps = torch.empty((BATCH, stride), dtype=torch.int16, device=dev)
        hits = torch.empty(BATCH, dtype=torch.int32, device=dev)
        md = torch.empty(BATCH, dtype=torch.int16, device=dev)
        aux = torch.empty((n_pool, BATCH, 2), dtype=torch.int64, device=dev)
        st = stream.cuda_stream

        if world == 1:
            def step(i):
                native.query_device(dq[i % n_pool], K, "complete", ids, lcps, hits, md, aux[i % n_pool], stream=st)
        else:
            def step(i):
                sh.query_device(dq[i % n_pool], K, ids, lcps, hits)

        def flush():
            flush_buf.zero_()

        for i in range(args.warmup):
            flush()
            step(i)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(local_rank)
        sampler.start()
        evs = time_steps(step, flush, args.steps, stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = sampler.stop()
        step_ms = np.array([a.elapsed_time(b) for a, b in evs])
        total_ms = float(step_ms.sum())
        if world > 1:
            t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            total_ms = float(t.item())
        value = BATCH * args.steps / (total_ms / 1e3)

        # roofline of the dominant kernel (k_query_warp): algorithmic bytes / event time
        rsize = (aux[:, :, 1].cpu().numpy().astype(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
        per_batch = np.array([indexed_bytes_per_query(N_ITEMS, SEQ_LEN, SIGMA, K, rsize[b]).sum() for b in range(n_pool)])
        bytes_per_launch = float(np.mean([per_batch[i % n_pool] for i in range(args.steps)]))
        peak, peak_src = hbm_peak()
        achieved = bytes_per_launch / (np.mean(step_ms) / 1e3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("k_query_warp", {}).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 5), "traffic": traffic,
                    "kernel": "k_query_warp<1>", "bytes_per_launch": round(bytes_per_launch, 1),
                    "peak_source": peak_src,
                    "bytes_formula": "sum_q K_b*ceil(log2(N+1)) + |R(d*)|*(K_b+4) + K_b + 6k, K_b=8"}

    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": ("synthetic: reference Philox generator, generate_dataset(2_000_000, 32, 4, seed=3+rank), "
                 "generate_queries(seed=4), 8 distinct 4096-query batches cycled"),
        "config": {"workload": "config 3: indexed complete-mode top-k serving, 4096-query batches",
                   "n_items_per_rank": N_ITEMS, "n_items_total": N_ITEMS * world, "seq_len": SEQ_LEN,
                   "alphabet": SIGMA, "k": K, "batch": BATCH, "mode": "complete",
                   "l2": "flushed before every timed step (256 MiB memset), step = own CUDA event pair",
                   "parallelism": "single GPU" if world == 1 else f"row-block shards x{world} + NCCL all_gather merge"},
        "roofline": roofline,
        "gpu_launches": args.steps * (1 if world == 1 else 3),
        "clocks": clocks,
        "build_s": round(t_build, 3),
        "p50_batch_latency_ms": float(np.median(step_ms)),
    }

    if world == 1 and rank == 0:
        line["e2e"] = e2e_leg(idx, qs, args, stream)
        cpu_qps, cpu_done, cpu_el, trie = cpu_reference(ds, qs, K, args.cpu_budget_s, os.cpu_count() or 1)
        line["cpu_baseline"] = {
            "value": cpu_qps, "unit": "queries/s", "cores": os.cpu_count() or 1, "kind": "port",
            "sample": (f"{cpu_done} complete-mode k=10 queries ({cpu_el:.1f} s) of the same workload; "
                       "C restatement of trie.build/TrieIndex.query (oracle/lcp_oracle.c), one pthread per core")}
        if not args.no_extras:
            line["extras"] = extras(idx, ds, qs, stream, flush_buf, step_ms)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def e2e_leg(idx, qs, args, stream) -> dict:
    """Public API, host buffers: pinned queries in, results out, every step."""
    from paper_2602_04936_b200._native import PinnedArray

    n_pool = qs.shape[0] // BATCH
    pin = PinnedArray((n_pool, BATCH, SEQ_LEN), np.uint16)
    pin.array[:] = qs.reshape(n_pool, BATCH, SEQ_LEN)
    out = idx.native.alloc_batch(BATCH, K, "complete", pinned=True)
    for i in range(args.warmup):
        idx.query_batch(pin.array[i % n_pool], K, "complete", out=out)
    steps = min(args.steps, 1000)
    t = []
    for i in range(steps):
        t0 = time.perf_counter()
        idx.query_batch(pin.array[i % n_pool], K, "complete", out=out)
        t.append(time.perf_counter() - t0)
    stride = out.ids.shape[1]
    return {"value": BATCH * steps / float(np.sum(t)), "unit": "queries/s",
            "h2d_bytes_per_step": BATCH * SEQ_LEN * 2,
            "d2h_bytes_per_step": BATCH * (stride * 6 + 4 + 2 + 16),
            "steps": steps, "p50_ms": 1e3 * float(np.median(t)),
            "api": "TrieIndex.query_batch(pinned uint16 (4096, 32), k=10, 'complete', out=pinned)"}


def extras(idx, ds, qs, stream, flush_buf, step_ms) -> dict:
    import torch

    import paper_2602_04936_b200 as lg

    dev = flush_buf.device
    st = stream.cuda_stream
    out: dict = {}
    n_pool = qs.shape[0] // BATCH
    dq = torch.from_numpy(qs).to(dev).view(n_pool, BATCH, SEQ_LEN)
    ids = torch.empty((BATCH, K), dtype=torch.int32, device=dev)
    lcps = torch.empty((BATCH, K), dtype=torch.int16, device=dev)
    hits = torch.empty(BATCH, dtype=torch.int32, device=dev)

    def timed(fn, steps, flush=True):
        with torch.cuda.stream(stream):
            for i in range(3):
                fn(i)
            torch.cuda.synchronize()
            evs = time_steps(fn, (lambda: flush_buf.zero_()) if flush else None, steps, stream)
            torch.cuda.synchronize()
        return np.array([a.elapsed_time(b) for a, b in evs])

    # warm-L2 serving steady state (index resident in the 126 MB L2)
    warm = timed(lambda i: idx.native.query_device(dq[i % n_pool], K, "complete", ids, lcps, hits, stream=st), 500, flush=False)
    out["indexed_warm_l2_qps"] = BATCH / (warm.mean() / 1e3)
    # prefix-16 query variant
    qp = lg.generate_queries(ds, BATCH, seed=5, prefix_len=16)
    dqp = torch.from_numpy(qp).to(dev)
    pre = timed(lambda i: idx.native.query_device(dqp, K, "complete", ids, lcps, hits, stream=st), 200)
    out["indexed_prefix16_qps"] = BATCH / (pre.mean() / 1e3)
    # brute-force full-scan kernel on the same batch
    fs = timed(lambda i: idx.native.fullscan_device(dq[i % n_pool], K, ids, lcps, hits, stream=st), 20)
    out["fullscan_qps"] = BATCH / (fs.mean() / 1e3)
    out["fullscan_ms_per_batch"] = float(fs.mean())
    out["fullscan_stream_gbs"] = N_ITEMS * 8 / (fs.mean() / 1e3) / 1e9
    # TAL B=256 (paper's bounded-range scan)
    tal = lg.build_tal(ds, 256)
    tl = timed(lambda i: tal.native.query_device(dq[i % n_pool], K, "tal", ids, lcps, hits, stream=st), 50)
    out["tal256_qps"] = BATCH / (tl.mean() / 1e3)
    # energy: NVML counter over >= 3 s loops (gross, and net of idle power)
    energy = nvml_energy()
    if energy is not None:
        def joules_per_query(fn, seconds=3.0):
            with torch.cuda.stream(stream):
                fn(0)
                torch.cuda.synchronize()
                e0, t0, done, i = energy(), time.perf_counter(), 0, 0
                while time.perf_counter() - t0 < seconds:
                    for _ in range(20):
                        fn(i)
                        i += 1
                        done += BATCH
                    torch.cuda.synchronize()
                el = time.perf_counter() - t0
                return (energy() - e0) / done, done / el
        time.sleep(0.5)
        e0 = energy()
        time.sleep(2.0)
        idle_w = (energy() - e0) / 2.0
        jq_idx, qps_idx = joules_per_query(lambda i: idx.native.query_device(dq[i % n_pool], K, "complete", ids, lcps, hits, stream=st))
        jq_fs, qps_fs = joules_per_query(lambda i: idx.native.fullscan_device(dq[i % n_pool], K, ids, lcps, hits, stream=st))
        jq_tal, qps_tal = joules_per_query(lambda i: tal.native.query_device(dq[i % n_pool], K, "tal", ids, lcps, hits, stream=st))
        out["energy"] = {
            "idle_w": idle_w,
            "indexed_j_per_query": jq_idx, "indexed_net_j_per_query": jq_idx - idle_w / qps_idx,
            "fullscan_j_per_query": jq_fs, "fullscan_net_j_per_query": jq_fs - idle_w / qps_fs,
            "tal256_j_per_query": jq_tal, "tal256_net_j_per_query": jq_tal - idle_w / qps_tal,
            "method": "NVML total-energy delta over >=3 s back-to-back batches (warm L2)",
        }
    # GNC config 2: N=100k, L=24, k=5, one query per call through the public API
    g = lg.generate_dataset(100_000, 24, SIGMA, seed=4)
    gi = lg.build(g)
    readings = lg.generate_queries(g, 1000, seed=5, prefix_len=12)
    for q in readings[:20]:
        gi.query(q, 5, "complete")
    lat = []
    for q in readings:
        t0 = time.perf_counter()
        gi.query(q, 5, "complete")
        lat.append(time.perf_counter() - t0)
    out["gnc_single_query"] = {"hz": len(lat) / float(np.sum(lat)), "p50_ms": 1e3 * float(np.median(lat)),
                               "p99_ms": 1e3 * float(np.percentile(lat, 99)),
                               "api": "TrieIndex.query(q, 5, 'complete') per step, N=100k, L=24"}
    return out


if __name__ == "__main__":
    main()
