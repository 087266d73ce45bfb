#!/usr/bin/env python3
"""Benchmark of the LCP-indexed top-k hot path (BASELINE.json metric).

Workload (N=1): BASELINE config 3 — N=2,000,000 items, L=32, sigma=4, k=10,
complete-mode top-k over batches of 4,096 queries.  A "step" is one batch
through the fused query kernel (pack -> 64-ary search -> leaf region ->
d* -> rank selection), inputs resident in HBM.

Timing: the steps are captured once in a CUDA graph and replayed, so the
GPU is never starved by Python-side launch cost.  Step i runs on index
replica i % 8 (8 identical replicas, 8 x 24 MB > 126 MB L2, so every step's
index reads miss L2) and on CUDA stream i % 4 (four batches in flight, as a
serving loop keeps them); the whole K-step region is bracketed by CUDA
events on the capture stream.  The same loop on one stream (one batch in
flight) is reported beside it, and its per-step time is the kernel duration
used for the roofline.

N>1 (torchrun): BASELINE config 5, the north-star scheme (config5_leg):
the 200M-row corpus is split into row blocks that each rank draws itself,
re-split by lexicographic range; every step all-gathers the ranks' 4096-query
client batches, routes each query on the device to the shard owning its key
range (plus the neighbours its top-k may spill into), answers locally,
exchanges candidates with NCCL and merges them on the device.  The whole step
is captured in a CUDA graph; time = max over ranks, value = all ranks'
client queries/s ("scaling": "weak": 4096 queries per rank per step).  The
row-block scheme and query-partitioned config-3 replicas are side fields.

``--impl reference`` times the reference's own algorithm on the host CPU
(the pinned C restatement in oracle/, all host threads) on the same config.
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "top-k LCP queries/sec at N=2M, L=32, k=10 (HBM GB/s frac); p50 latency; J/query"
N_ITEMS, SEQ_LEN, SIGMA, K, BATCH = 2_000_000, 32, 4, 10, 4096
INFLIGHT = 4  # batches in flight in the headline timed loop (streams); swept 2..5: 1.02/1.44/1.49/1.49 G q/s
INFLIGHT = int(os.environ.get("LCP_BENCH_INFLIGHT", INFLIGHT))  # sweep hook
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
    """NVML-polled SM clocks + throttle reasons (2 ms period) around the timed
    region (started before the warm-up replays, stopped after timing)."""

    REASONS = {  # nvmlClocksEventReason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
        0x4: "sw_power_cap",
    }

    def __init__(self, device: int = 0):
        self.device = device
        self.samples: list[tuple[float, float, int]] = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        rs = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                        self.samples.append((time.perf_counter(), sm, rs))
                    except Exception:
                        pass
                    time.sleep(0.002)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None

    def stop(self, t0: float | None = None, t1: float | None = None) -> dict:
        if self._t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self._stop.set()
        self._t.join(timeout=1)
        inside = [x for x in self.samples if t0 is None or t0 <= x[0] <= t1]
        use = inside if inside else self.samples
        reasons = set()
        for _, _, rs in use:
            for bit, nm in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": float(np.median([x[1] for x in use])) if use else None,
                "sm_max_mhz": self._max, "reasons": sorted(reasons),
                "samples": len(use), "samples_in_timed_region": len(inside),
                "source": "NVML clock/event-reason polling, 2 ms"}


def nvml_energy():
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(int(os.environ.get("LOCAL_RANK", "0")))
        return lambda: pynvml.nvmlDeviceGetTotalEnergyConsumption(h) / 1000.0  # J
    except Exception:
        return None


def bench_config(world: int) -> dict:
    """The workload both arms (--impl ours / reference) run, as one dict, so
    the two JSON lines name the same config."""
    return {"workload": "config 3: indexed complete-mode top-k serving, 4096-query batches",
            "n_items": N_ITEMS, "seq_len": SEQ_LEN, "alphabet": SIGMA, "k": K, "batch": BATCH,
            "batch_per_rank": BATCH, "mode": "complete",
            "l2": "inputs larger than L2: 8 index replicas (8 x 24 MB > 126 MB) cycled step to step",
            "launch": f"CUDA graph replay; {INFLIGHT} batches in flight on {INFLIGHT} streams",
            "parallelism": ("single GPU" if world == 1 else
                            f"query-partitioned x{world}: every rank holds the full 2M index "
                            "(24 MB) and answers its own batches; no data-path collective")}


# --------------------------------------------------------------------------
def cpu_reference(ds, queries: np.ndarray, k: int, budget_s: float, nthreads: int, trie=None):
    """Time the reference algorithm (C port in oracle/) on the host cores."""
    import oracle

    if trie is None:
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


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def python_reference(n_queries: int = 2048) -> dict:
    """The reference's OWN Python path on the host cores (BASELINE.md §2,
    SURVEY §8d): the unmodified lcpsearch installed in baseline/_ref
    (tools/install_reference.sh), trie.build + the bench's own query loop
    _query_stream(index, queries, 10, "complete", workers=w) for w in
    {1, 2, 4, cpu_count} (pkg/src/lcpsearch/bench.py:245-270)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "lcpsearch")):
        return {"unavailable": "reference not installed in baseline/_ref (tools/install_reference.sh)"}
    sys.path.insert(0, ref)
    try:
        import lcpsearch
        from lcpsearch.bench import _query_stream
    finally:
        sys.path.remove(ref)
    ds = lcpsearch.generate_dataset(N_ITEMS, SEQ_LEN, SIGMA, seed=3)
    t0 = time.perf_counter()
    index = lcpsearch.build(ds)
    build_s = time.perf_counter() - t0
    qs = lcpsearch.generate_queries(ds, n_queries, seed=4)
    out = {"build_s": round(build_s, 3), "queries": n_queries, "unit": "queries/s",
           "api": "lcpsearch.bench._query_stream(trie.build(ds), q, 10, 'complete', workers=w)"}
    sweep = {}
    for w in sorted({1, 2, 4, os.cpu_count() or 1}):
        _, _, el = _query_stream(index, qs, K, "complete", w)
        sweep[str(w)] = round(n_queries / el, 1)
    out["workers_sweep"] = sweep
    out["value"] = max(sweep.values())
    return out


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
        "config": bench_config(args.gpus),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": nthreads, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"{args.steps} batches x {BATCH} queries; C restatement of "
                                   "trie.build/TrieIndex.query (oracle/lcp_oracle.c), pthreads"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=200)
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

    if _build.needs_build():
        _build.build_native()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # functional test hook only (numbers meaningless): all ranks on cuda:0,
    # gloo for the host-level barrier / max-reduce
    share = os.environ.get("LCP_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            # bounded collective timeout: a failed rank ends the run instead of hanging it
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank),
                                    timeout=datetime.timedelta(seconds=300))
    dev = torch.device("cuda", local_rank)

    # every rank serves the config-3 corpus from its own replica of the index
    # (query-partitioned: rank r answers its own query stream; no data-path
    # collective).  Rank 0's stream is the N=1 stream.
    ds = lg.generate_dataset(N_ITEMS, SEQ_LEN, SIGMA, seed=3)
    n_pool = 8
    qs = lg.generate_queries(ds, BATCH * n_pool, seed=4 + 1000 * rank)
    main_stream = torch.cuda.Stream(device=dev)
    sampler = ClockSampler(local_rank)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with torch.cuda.stream(main_stream):
        t_build = time.perf_counter()
        idx = lg.build(ds)
        torch.cuda.synchronize()
        t_build = time.perf_counter() - t_build
        dq = torch.from_numpy(qs).to(dev).view(n_pool, BATCH, SEQ_LEN)

        def out_bufs():
            return (torch.empty((BATCH, K), dtype=torch.int32, device=dev),
                    torch.empty((BATCH, K), dtype=torch.int16, device=dev),
                    torch.empty(BATCH, dtype=torch.int32, device=dev),
                    torch.empty(BATCH, dtype=torch.int16, device=dev),
                    torch.empty((n_pool, BATCH, 2), dtype=torch.int64, device=dev))

        from paper_2602_04936_b200._native import Workspace, workspace

        workspace()  # created outside graph capture (it allocates)
        t_rep = time.perf_counter()
        replicas = [idx] + [lg.build(ds) for _ in range(7)]
        torch.cuda.synchronize()
        build_ms_steady = 1e3 * (time.perf_counter() - t_rep) / 7
        R = len(replicas)
        # steps per captured graph: the whole timed region in one graph up to
        # 8192 steps (a multiple of R * n_pool, so the replica / batch cycle
        # stays aligned across replays beyond that); measured: per-step time
        # is the same as with 64-step graphs replayed back to back, minus the
        # graph-boundary gaps
        G_MAX = 8192

        def capture(n_steps: int, n_streams: int):
            streams = [torch.cuda.Stream(device=dev) for _ in range(n_streams)]
            wss = [Workspace() for _ in range(n_streams)]  # one per stream (lcp_b200.h contract)
            bufs = [out_bufs() for _ in range(n_streams)]
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=main_stream):
                for x in streams:
                    x.wait_stream(main_stream)
                for i in range(n_steps):
                    x, (ids, lcps, hits, md, aux) = streams[i % n_streams], bufs[i % n_streams]
                    b = (i // R) % n_pool
                    replicas[i % R].native.query_device(dq[b], K, "complete", ids, lcps, hits, md,
                                                       aux[b], stream=x.cuda_stream,
                                                       ws=wss[i % n_streams])
                for x in streams:
                    main_stream.wait_stream(x)
            g.workspaces = wss  # the graph holds their scratch pointers: keep them alive
            return g, bufs

        def run_steps(n_streams: int, steps: int, warmup: int):
            G = min(steps, G_MAX)
            g, bufs = capture(G, n_streams)
            tail = steps % G
            gt = capture(tail, n_streams)[0] if tail else None
            # W warm-up steps, and at least ~0.3 s so SM clocks leave idle.  Both
            # graphs the timed region replays are warmed (their first replay
            # uploads the graph), the tail one last, as in the timed region
            t_w, reps = time.perf_counter(), 0
            while reps * G < warmup or time.perf_counter() - t_w < 0.3:
                g.replay()
                if gt is not None:
                    gt.replay()
                reps += 1
                if reps % 16 == 0:
                    torch.cuda.synchronize()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # one more untimed replay queued right ahead of the start event keeps
            # the GPU busy while the host enqueues the timed graph, so no host
            # launch latency lands inside the region.  The region itself still
            # starts at that replay's join, with an empty pipeline: a short
            # --steps run includes one fill and one drain (about one batch's
            # latency), which a long run amortises
            (gt if gt is not None else g).replay()
            t0 = time.perf_counter()
            a.record(main_stream)
            for _ in range(steps // G):
                g.replay()
            if gt is not None:
                gt.replay()
            b.record(main_stream)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            barrier()
            return max_over_ranks(a.elapsed_time(b)), bufs, (t0, t1)

        # one batch in flight (kernel duration for the roofline)
        single_ms, bufs1, _ = run_steps(1, args.steps, args.warmup)
        # per-launch duration = the single-stream step: launches are graph
        # nodes back to back (event nodes around each launch were measured to
        # add ~5 us each, so they are not used)
        kernel_ms = single_ms / args.steps
        kernel_src = "CUDA events over the graph-replayed single-stream step loop"
        # headline: three batches in flight (a serving pipeline)
        sampler.start()
        total_ms, bufs2, (t0, t1) = run_steps(INFLIGHT, args.steps, args.warmup)
        clocks = sampler.stop(t0, t1)
        gpu_launches = args.steps * world
        value = world * BATCH * args.steps / (total_ms / 1e3)
        # |R(d*)| of every batch of the pool (a short timed region may not have
        # touched all of them): one untimed launch per batch
        ids_a, lcps_a, hits_a, md_a, aux_all = out_bufs()
        for bb in range(n_pool):
            idx.native.query_device(dq[bb], K, "complete", ids_a, lcps_a, hits_a, md_a, aux_all[bb],
                                    stream=main_stream.cuda_stream)
        torch.cuda.synchronize()

        # roofline of the dominant kernel (k_query_w1): algorithmic bytes / duration
        rsize = (aux_all[:, :, 1].cpu().numpy().astype(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
        per_batch = np.array([indexed_bytes_per_query(N_ITEMS, SEQ_LEN, SIGMA, K, rsize[bb]).sum()
                              for bb in range(n_pool)])
        bytes_per_launch = float(per_batch.mean())
        kernel_s = kernel_ms / 1e3
        peak, peak_src = hbm_peak()
        achieved = bytes_per_launch / kernel_s / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
        if os.path.exists(prof):
            try:
                traffic = json.load(open(prof)).get("k_query_w1", {}).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 5), "traffic": traffic,
                    "kernel": "k_query_w1<u32,2>", "bytes_per_launch": round(bytes_per_launch, 1),
                    "launch_us": round(kernel_s * 1e6, 3),
                    "peak_source": peak_src,
                    "duration_source": kernel_src,
                    "bytes_formula": "sum_q K_b*ceil(log2(N+1)) + |R(d*)|*(K_b+4) + K_b + 6k, K_b=8"}
        # the same algorithmic bytes over the pipelined (4-in-flight) per-step time
        step_s = total_ms / 1e3 / args.steps
        roofline["pipelined"] = {"achieved": round(bytes_per_launch / step_s / 1e9, 2), "unit": "GB/s",
                                 "frac": round(bytes_per_launch / step_s / 1e9 / peak, 5),
                                 "step_us": round(step_s * 1e6, 3),
                                 "note": "algorithmic bytes per batch / headline per-step time "
                                         f"({INFLIGHT} batches in flight); frac above is per launch"}
        # the kernel is issue-bound, not HBM-bound: instruction roofline from the
        # committed ncu capture (warp instructions per query) and the live rate
        try:
            prof_q = json.load(open(prof))["k_query_w1"]
            ipq = prof_q["warp_instructions"] / BATCH
            mhz = clocks.get("sm_mhz") or clocks.get("sm_max_mhz")
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            peak_gi = sms * 4 * mhz * 1e6 / 1e9  # 4 schedulers x 1 warp instruction / clock
            ach_gi = value / world * ipq / 1e9   # per GPU
            roofline["issue"] = {
                "warp_instructions_per_query": round(ipq, 1), "achieved": round(ach_gi, 1),
                "peak": round(peak_gi, 1), "unit": "G warp-instructions/s per GPU",
                "frac": round(ach_gi / peak_gi, 4),
                "source": "profiles/ncu_summary.json smsp__inst_executed.sum / 4096 queries; "
                          "peak = SMs x 4 schedulers x median SM clock in the timed region"}
        except Exception:
            pass

    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": ("synthetic: reference Philox generator, generate_dataset(2_000_000, 32, 4, seed=3), "
                 "generate_queries(seed=4 + 1000*rank), 8 distinct 4096-query batches cycled per rank"),
        "config": bench_config(world),
        "roofline": roofline,
        "gpu_launches": gpu_launches,
        "clocks": clocks,
        "build_s": round(t_build, 3),
        "build_ms_steady": round(build_ms_steady, 2),  # mean of 7 replica builds from host rows
        "one_batch_in_flight": {"value": world * BATCH * args.steps / (single_ms / 1e3), "unit": "queries/s",
                                "ms_per_step": single_ms / args.steps},
    }
    line["e2e"] = e2e_leg(idx, qs, args, world, barrier, max_over_ranks)
    if world > 1:
        # N > 1: the headline is BASELINE config 5 on the north-star scheme
        # (corpus sharded by lexicographic range, device routing, NCCL
        # exchanges, merge kernel); config-3 replicas stay as a side field
        del replicas, idx
        torch.cuda.empty_cache()
        c5 = config5_leg(args, world, rank, dev, barrier, max_over_ranks, "range")
        line["replicas"] = {k: line[k] for k in ("value", "ms_per_step", "one_batch_in_flight", "e2e")}
        line["replicas"]["parallelism"] = line["config"]["parallelism"]
        line["value"], line["ms_per_step"] = c5["value"], c5["ms_per_step"]
        line["e2e"] = c5.pop("e2e")
        line["config"] = config5_dict(world)
        line["sharded"] = c5
        line["gpu_launches"] = c5["steps"] * SHARD_LAUNCHES_PER_STEP
        line["rowblock_sharded"] = config5_leg(args, world, rank, dev, barrier, max_over_ranks, "rowblock")
    if world == 1 and rank == 0:
        line["p50_batch_latency_ms"] = cold_batch_latency(idx, dq, dev)
        cpu_qps, cpu_done, cpu_el, trie = cpu_reference(ds, qs, K, args.cpu_budget_s, os.cpu_count() or 1)
        line["cpu_baseline"] = {
            "value": cpu_qps, "unit": "queries/s", "cores": os.cpu_count() or 1, "kind": "port",
            "sample": (f"{cpu_done} complete-mode k=10 queries ({cpu_el:.1f} s) of the same workload; "
                       "C restatement of trie.build/TrieIndex.query (oracle/lcp_oracle.c), one pthread per core")}
        # host-thread scaling of the same CPU path (w in {1, 2, 4, all})
        sweep = {}
        for w in sorted({1, 2, 4, os.cpu_count() or 1}):
            if w == (os.cpu_count() or 1):
                sweep[str(w)] = cpu_qps
                continue
            sweep[str(w)] = cpu_reference(ds, qs, K, min(1.5, args.cpu_budget_s), w, trie=trie)[0]
        line["cpu_baseline"]["threads_sweep"] = sweep
        line["cpu_baseline"]["cpu_model"] = cpu_model()
        line["cpu_baseline"]["python_reference"] = python_reference()
        if not args.no_extras:
            # side measurements: a failure is recorded in the line, never
            # allowed to suppress the headline line itself
            try:
                flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
                line["extras"] = extras(idx, ds, qs, main_stream, flush_buf)
                del flush_buf, replicas
                torch.cuda.empty_cache()
            except Exception as e:  # pragma: no cover - reported in the line
                line["extras"] = {"error": f"{type(e).__name__}: {e}"}
            # config 5 on one GPU through the same sharded step the N > 1 runs
            # time (one range shard, local exchange): the N = 1 point of the
            # config-5 scaling curve
            try:
                line["extras"]["config5_single_gpu"] = config5_leg(args, 1, 0, dev, barrier, max_over_ranks,
                                                                   "range")
            except Exception as e:  # pragma: no cover - reported in the line
                line["extras"]["config5_single_gpu"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


C5_ITEMS = int(os.environ.get("LCP_BENCH_C5_ITEMS", 200_000_000))  # BASELINE config 5 (override: functional checks only)
# candidate exchange of the range-sharded step: "all_to_all" (NCCL) or "p2p"
# (symmetric memory: peers signal, the merge kernel reads their candidates over
# NVLink).  p2p is tested at one rank; no multi-GPU box was available to
# validate it, so NCCL stays the default (LCP_BENCH_EXCHANGE=p2p to select it)
EXCHANGE = os.environ.get("LCP_BENCH_EXCHANGE", "all_to_all")
# sharded steps in flight per rank (tools/c5_probe.py at 25M rows, one GPU:
# 2 / 4 / 8 slots -> 204 / 344 / 411 M q/s); under NCCL each slot holds its own
# communicator, so fewer of them there
C5_INFLIGHT = int(os.environ.get("LCP_BENCH_C5_INFLIGHT", "8"))
C5_INFLIGHT_NCCL = int(os.environ.get("LCP_BENCH_C5_INFLIGHT_NCCL", "4"))
# our kernels per range-sharded step: pack + route (own), counted query,
# thresholds, encode, pack + route (consult), counted query, encode, merge
SHARD_LAUNCHES_PER_STEP = 10


def config5_dict(world: int) -> dict:
    return {"workload": "config 5: corpus sharded by lexicographic range over the ranks, "
                        "complete-mode top-k of each rank's 4096-query client batches",
            "n_items": C5_ITEMS, "seq_len": SEQ_LEN, "alphabet": SIGMA, "k": K, "batch": BATCH * world,
            "batch_per_rank": BATCH, "mode": "complete",
            "l2": "inputs larger than L2: the 200M-row index (about 7 GB over the ranks)",
            "launch": "CUDA graph replay of the whole sharded step, NCCL collectives inside",
            "parallelism": f"range shards x{world} (north star, SURVEY §8e)"}


def config5_leg(args, world, rank, dev, barrier, max_over_ranks, scheme: str = "range",
                n_total: int = C5_ITEMS) -> dict:
    """BASELINE config 5 (N=200M, L=32, sigma=4, k=10), the north-star
    multi-GPU path: the corpus is split into row blocks over the ranks (each
    rank draws its own block with datagen.generate_row_block, byte-identical
    to slicing generate_dataset(200M, 32, 4, seed=6)), then
      scheme "range": re-split by lexicographic range (RangeShardedIndex):
          a step all-gathers the ranks' 4096-query client batches, routes every
          query to the shard owning its key range on the device, answers,
          exchanges owner thresholds (all_reduce), lets neighbouring ranges
          answer where the top-k may spill over, and all-to-alls the
          candidates back to the client's rank for the merge kernel;
      scheme "rowblock": every rank answers the whole gathered batch on its
          row block, candidates all-to-all to the client's rank, merge.
    Every step is graph-captured (NCCL collectives inside the graph) and
    replayed; no host synchronisation inside the timed region.  value = all
    ranks' client queries / max-over-ranks device time.  world = 1 runs the
    same code path on one GPU (local exchange)."""
    import torch
    import torch.distributed as dist

    from paper_2602_04936_b200.core import Alphabet, Dataset
    from paper_2602_04936_b200.datagen import generate_queries, generate_row_block
    from paper_2602_04936_b200.sharded import RowBlockShardStep, ShardPlan

    lo, hi = ShardPlan(n_total, world).bounds(rank)
    t0 = time.perf_counter()
    rows = generate_row_block(n_total, SEQ_LEN, SIGMA, 6, lo, hi)
    gen_s = time.perf_counter() - t0
    n_pool = 8  # each rank's own client stream: uniform queries (generate_queries, seed 4 + 1000*rank)
    qs = generate_queries(Dataset(alphabet=Alphabet(SIGMA), length=SEQ_LEN, items=rows[:1]),
                          BATCH * n_pool, seed=4 + 1000 * rank)
    barrier()
    t0 = time.perf_counter()
    if scheme == "range":
        from paper_2602_04936_b200.rangeshard import RangeShardedIndex

        sh = RangeShardedIndex(rows, SEQ_LEN, SIGMA, id_offset=lo)
        n_local = sh.n_local
    else:
        sh = RowBlockShardStep(rows, SEQ_LEN, SIGMA, id_offset=lo, n_total=n_total)
        n_local = sh.native.n
    del rows
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    stream = torch.cuda.Stream(device=dev)
    nccl = world > 1 and dist.get_backend() == "nccl"
    # C5_INFLIGHT steps in flight, each on its own stream with its own step
    # buffers (slot) and, under NCCL, its own communicator (process group):
    # one step is a chain of small dependent launches and exchanges, so its
    # latency, not any one kernel, bounds a single stream
    n_slots = C5_INFLIGHT if world == 1 else (min(C5_INFLIGHT, C5_INFLIGHT_NCCL) if nccl else 1)
    # slot 0 keeps the default group (the p2p leg's symmetric-memory
    # rendezvous runs on it); slots 1.. get their own communicators
    groups = [dist.new_group(list(range(world))) if nccl and s_ > 0 else None for s_ in range(n_slots)]
    slot_streams = [torch.cuda.Stream(device=dev) for _ in range(n_slots)]
    with torch.cuda.stream(stream):
        pool = torch.from_numpy(qs).to(dev).view(n_pool, BATCH, SEQ_LEN)
        gqs = [torch.empty((world * BATCH, SEQ_LEN), dtype=torch.uint16, device=dev) for _ in range(n_slots)]
        outs = [(torch.empty((BATCH, K), dtype=torch.int32, device=dev),
                 torch.empty((BATCH, K), dtype=torch.int16, device=dev),
                 torch.empty(BATCH, dtype=torch.int32, device=dev)) for _ in range(n_slots)]
        out = outs[0]

        # the uint16 rows travel as int32 pairs (NCCL and gloo have no 16-bit integer type)
        def step(i, exchange=EXCHANGE if scheme == "range" else "all_to_all", slot=0, rows=None):
            rows = pool[i % n_pool] if rows is None else rows
            src = rows.view(torch.int32)
            gq = gqs[slot]
            if nccl:
                dist.all_gather_into_tensor(gq.view(torch.int32), src, group=groups[slot])
            elif world > 1:  # gloo (LCP_BENCH_SHARE_GPU functional check): host staging
                h = torch.empty((world, BATCH, SEQ_LEN // 2), dtype=torch.int32)
                dist.all_gather(list(h.unbind(0)), src.cpu())
                gq.view(torch.int32).copy_(h.view(-1, SEQ_LEN // 2))
            else:
                gq.copy_(rows)
            sh.query_device(gq, K, "complete", out=outs[slot], exchange=exchange, group=groups[slot],
                            slot=slot)

        def timed(exchange, inflight=1):
            """Graph-capture G steps spread round-robin over `inflight` slot
            streams (eager if capture fails), warm, time ceil(steps / G)
            replays; returns (ms over ranks, steps, launch)."""
            S = max(1, min(inflight, n_slots))

            def run_steps(count):
                for x in slot_streams[:S]:
                    x.wait_stream(stream)
                for i in range(count):
                    with torch.cuda.stream(slot_streams[i % S]):
                        step(i, exchange, i % S)
                for x in slot_streams[:S]:
                    stream.wait_stream(x)

            for _ in range(3):  # eager warm-up (allocates every slot's step buffers)
                run_steps(S)
            torch.cuda.synchronize()
            G = min(64, max(8, args.steps))
            G = (G + S - 1) // S * S
            launch = (f"CUDA graph replay (NCCL collectives captured), {S} step(s) in flight"
                      + (", one communicator per stream" if nccl and S > 1 else ""))
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    run_steps(G)
                run = lambda: g.replay()
            except Exception as e:  # capture unsupported here: eager, still no host sync
                torch.cuda.synchronize()
                launch = f"eager stream-ordered launches (graph capture failed: {type(e).__name__})"
                run = lambda: run_steps(G)
            reps = max(1, (args.steps + G - 1) // G)
            for _ in range(max(1, args.warmup // G + 1)):
                run()
            barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                run()
            b.record(stream)
            torch.cuda.synchronize()
            ms = max_over_ranks(a.elapsed_time(b))
            barrier()
            return ms, reps * G, launch

        ms, steps, launch = timed(EXCHANGE if scheme == "range" else "all_to_all", n_slots)
        ms1, steps1, _ = timed(EXCHANGE if scheme == "range" else "all_to_all", 1)
        p2p = None
        if scheme == "range" and nccl and EXCHANGE != "p2p":
            # the peer-memory exchange beside it, when every rank can map its
            # peers' symmetric buffers (agreed by an all-reduce first)
            ok = torch.tensor([1], dtype=torch.int32, device=dev)
            try:
                import torch.distributed._symmetric_memory as symm_mem

                probe = symm_mem.empty((16,), dtype=torch.int64, device=dev)
                symm_mem.rendezvous(probe, dist.group.WORLD)
            except Exception:
                ok.zero_()
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if int(ok.item()):
                p_ms, p_steps, p_launch = timed("p2p")
                p2p = {"value": world * BATCH * p_steps / (p_ms / 1e3), "unit": "queries/s",
                       "steps": p_steps, "ms_per_step": p_ms / p_steps, "launch": p_launch,
                       "exchange": "p2p: symmetric-memory candidates, signal + merge kernel reading the peers"}
            else:
                p2p = {"unavailable": "symmetric memory rendezvous failed on some rank"}
        elif scheme == "range" and world == 1:  # the same kernels, the one rank its own peer
            p_ms, p_steps, p_launch = timed("p2p")
            p2p = {"value": BATCH * p_steps / (p_ms / 1e3), "unit": "queries/s", "steps": p_steps,
                   "ms_per_step": p_ms / p_steps, "launch": p_launch,
                   "exchange": "p2p kernels (signal + merge reading the candidate buffer), one rank"}
        kernel = kernel_leg(sh.engine.native, pool, dev, stream) if scheme == "range" and world == 1 else None
        # end to end: each step copies the rank's pinned client batch in and
        # its merged answers out (wall clock, max over ranks)
        from paper_2602_04936_b200._native import PinnedArray

        pin_q = PinnedArray((n_pool, BATCH, SEQ_LEN), np.uint16)
        pin_q.array[:] = qs.reshape(n_pool, BATCH, SEQ_LEN)
        host_q = torch.from_numpy(pin_q.array)
        # one graph per (slot, client batch): H2D of the pinned batch, the
        # step, D2H of the answers into the slot's pinned block; n_slots
        # steps in flight, a slot is reused once its previous step's answers
        # have landed (event wait)
        e_in = [torch.empty((BATCH, SEQ_LEN), dtype=torch.uint16, device=dev) for _ in range(n_slots)]
        host_outs = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in outs[s_]]
                     for s_ in range(n_slots)]
        exch = EXCHANGE if scheme == "range" else "all_to_all"

        def e2e_step(i, s_):
            e_in[s_].copy_(host_q[i % n_pool], non_blocking=True)
            step(i, exch, s_, rows=e_in[s_])
            for h, d in zip(host_outs[s_], outs[s_]):
                h.copy_(d, non_blocking=True)

        e_graphs = {}
        e_launch = "one CUDA graph per (slot, client batch)"
        try:
            for s_ in range(n_slots):
                for j in range(n_pool):
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=slot_streams[s_]):
                        e2e_step(j, s_)
                    e_graphs[(s_, j)] = g
        except Exception as e:
            torch.cuda.synchronize()
            e_graphs = {}
            e_launch = f"eager launches (graph capture failed: {type(e).__name__})"

        def e2e_submit(i, s_):
            with torch.cuda.stream(slot_streams[s_]):
                if e_graphs:
                    e_graphs[(s_, i % n_pool)].replay()
                else:
                    e2e_step(i, s_)

        e_steps = min(max(args.steps, 100), 400)
        e_steps = (e_steps + n_slots * n_pool - 1) // (n_slots * n_pool) * (n_slots * n_pool)
        events = [torch.cuda.Event() for _ in range(n_slots)]
        for i in range(n_slots * n_pool):
            e2e_submit(i, i % n_slots)
        torch.cuda.synchronize()
        barrier()
        t_e = time.perf_counter()
        for i in range(e_steps):
            s_ = i % n_slots
            if i >= n_slots:
                events[s_].synchronize()
            e2e_submit(i, s_)
            events[s_].record(slot_streams[s_])
        torch.cuda.synchronize()
        e_el = max_over_ranks(time.perf_counter() - t_e)
        barrier()
    e2e = {"value": world * BATCH * e_steps / e_el, "unit": "queries/s", "steps": e_steps,
           "ms_per_step": 1e3 * e_el / e_steps, "h2d_bytes_per_step": BATCH * SEQ_LEN * 2,
           "d2h_bytes_per_step": int(sum(t.numel() * t.element_size() for t in out)),
           "api": f"{type(sh).__name__}.query_device per step, pinned client batch in / answers out, "
                  f"{n_slots} step(s) in flight ({e_launch}), wall clock"}
    return {"value": world * BATCH * steps / (ms / 1e3), "unit": "queries/s", "steps": steps, "e2e": e2e,
            "ms_per_step": ms / steps, "steps_in_flight": n_slots,
            "one_step_in_flight": {"value": world * BATCH * steps1 / (ms1 / 1e3), "unit": "queries/s",
                                   "ms_per_step": ms1 / steps1},
            "n_items_total": n_total, "n_items_local": int(n_local),
            "scheme": scheme, "batch_per_rank": BATCH, "launch": launch,
            "exchange": EXCHANGE if scheme == "range" else "all_to_all",
            "gen_s": round(gen_s, 2), "build_s": round(build_s, 2), "p2p": p2p, "query_kernel": kernel,
            "parallelism": (f"{scheme} shards x{world}: all_gather client batches, device routing, "
                            "local top-k, NCCL exchange, k_merge" if scheme == "range" else
                            f"row-block shards x{world}: all_gather client batches, every shard answers, "
                            "all_to_all candidates, k_merge")}


def kernel_leg(native, pool, dev, stream, n_graph: int = 64, reps: int = 20) -> dict:
    """The bare query kernel on an index far larger than L2 (config 5 on one
    GPU: 200M rows, 7 GB): CUDA-graph replays of 4096-query batches, one and
    four in flight, and the per-launch roofline over the SURVEY §8d
    algorithmic bytes (|R(d*)| from the kernel's own aux words)."""
    import torch

    from paper_2602_04936_b200._native import Workspace

    n_pool = pool.shape[0]
    res = {}
    aux_all = torch.empty((n_pool, BATCH, 2), dtype=torch.int64, device=dev)
    for nst in (1, INFLIGHT):
        streams = [torch.cuda.Stream(device=dev) for _ in range(nst)]
        wss = [Workspace() for _ in range(nst)]
        bufs = [(torch.empty((BATCH, K), dtype=torch.int32, device=dev), torch.empty((BATCH, K), dtype=torch.int16, device=dev),
                 torch.empty(BATCH, dtype=torch.int32, device=dev), torch.empty(BATCH, dtype=torch.int16, device=dev))
                for _ in range(nst)]
        with torch.cuda.stream(stream):
            for b in range(n_pool):
                native.query_device(pool[b], K, "complete", *bufs[0], aux_all[b], stream=stream.cuda_stream, ws=wss[0])
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for x in streams:
                    x.wait_stream(stream)
                for i in range(n_graph):
                    j = i % nst
                    native.query_device(pool[i % n_pool], K, "complete", *bufs[j], aux_all[i % n_pool],
                                        stream=streams[j].cuda_stream, ws=wss[j])
                for x in streams:
                    stream.wait_stream(x)
            g.workspaces = wss
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                g.replay()
            b.record(stream)
            torch.cuda.synchronize()
        res[nst] = a.elapsed_time(b) / (n_graph * reps)  # ms per batch
    rsize = (aux_all[:, :, 1].cpu().numpy().astype(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
    per_batch = float(np.mean([indexed_bytes_per_query(native.n, SEQ_LEN, SIGMA, K, rsize[bb]).sum()
                               for bb in range(n_pool)]))
    peak = hbm_peak()[0]
    return {"n_items": native.n, "one_in_flight_us": round(res[1] * 1e3, 3),
            f"{INFLIGHT}_in_flight_us": round(res[INFLIGHT] * 1e3, 3),
            "qps_one_in_flight": BATCH / (res[1] / 1e3), f"qps_{INFLIGHT}_in_flight": BATCH / (res[INFLIGHT] / 1e3),
            "bytes_per_launch": round(per_batch, 1),
            "roofline_frac_per_launch": round(per_batch / (res[1] / 1e3) / 1e9 / peak, 5),
            "roofline_frac_pipelined": round(per_batch / (res[INFLIGHT] / 1e3) / 1e9 / peak, 5),
            "note": "k_query_w1<u64,2,1> (ids need 28 bits), index 7 GB >> L2: every search block and leaf "
                    "region read comes from DRAM"}


def cold_batch_latency(idx, dq, dev) -> float:
    """Median event-timed latency of one batch launched right after a 256 MiB
    L2-flushing memset (includes the launch; conservative)."""
    import torch

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    ids = torch.empty((BATCH, K), dtype=torch.int32, device=dev)
    lcps = torch.empty((BATCH, K), dtype=torch.int16, device=dev)
    hits = torch.empty(BATCH, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for i in range(60):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        idx.native.query_device(dq[i % dq.shape[0]], K, "complete", ids, lcps, hits, stream=st)
        b.record()
        torch.cuda.synchronize()
        if i >= 10:
            ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def e2e_leg(idx, qs, args, world=1, barrier=lambda: None, max_over_ranks=lambda x: x) -> dict:
    """Public API, host buffers: pinned queries in, results out, every step.
    At N GPUs every rank runs the same loop on its own stream of batches;
    value = all ranks' queries / the slowest rank's wall clock."""
    from paper_2602_04936_b200._native import PinnedArray

    n_pool = qs.shape[0] // BATCH
    pin = PinnedArray((n_pool, BATCH, SEQ_LEN), np.uint16)
    pin.array[:] = qs.reshape(n_pool, BATCH, SEQ_LEN)
    out = idx.native.alloc_batch(BATCH, K, "complete", pinned=True)
    for i in range(20):
        idx.query_batch(pin.array[i % n_pool], K, "complete", out=out)
    # e2e runs its own loop of at least 1000 batches (wall clock around a
    # depth-8 pipeline): a 20-batch region would mostly time the fill / drain
    steps = min(max(args.steps, 1000), 2000)
    t = []
    for i in range(steps):
        t0 = time.perf_counter()
        idx.query_batch(pin.array[i % n_pool], K, "complete", out=out)
        t.append(time.perf_counter() - t0)
    sync = {"value": world * BATCH * steps / max_over_ranks(float(np.sum(t))),
            "p50_ms": 1e3 * float(np.median(t)),
            "api": "TrieIndex.query_batch (synchronous, one batch at a time)"}
    # pipelined serving: up to 3 batches in flight, each with its own H2D and D2H
    from paper_2602_04936_b200 import _native

    depth = _native.ASYNC_DEPTH
    outs = [idx.native.alloc_batch(BATCH, K, "complete", pinned=True, with_work=False)
            for _ in range(depth)]
    # warm every (ring workspace, query batch, output block) triple the timed
    # loop will use, so each workspace's graph cache already holds its
    # submission: the async ring advances once per call, so starting the timed
    # loop on a multiple of lcm(depth, n_pool) keeps slot i % depth paired with
    # batch i % n_pool and block i % depth, exactly as during the warm-up
    period = depth * n_pool // np.gcd(depth, n_pool)
    _native.reset_async_ring()
    for i in range(2 * period):
        idx.query_batch_async(pin.array[i % n_pool], K, "complete", out=outs[i % depth]).result()
    pending = []
    barrier()
    t0 = time.perf_counter()
    for i in range(steps):
        if len(pending) == depth:
            pending.pop(0).result()
        pending.append(idx.query_batch_async(pin.array[i % n_pool], K, "complete", out=outs[i % depth]))
    for p in pending:
        p.result()
    el = max_over_ranks(time.perf_counter() - t0)
    barrier()
    return {"value": world * BATCH * steps / el, "unit": "queries/s",
            "h2d_bytes_per_step": BATCH * SEQ_LEN * 2,
            "d2h_bytes_per_step": int(outs[0].ids.nbytes + outs[0].lcps.nbytes + outs[0].hits.nbytes),
            "steps": steps, "ms_per_step": 1e3 * el / steps,
            "api": (f"TrieIndex.query_batch_async(pinned uint16 (4096, 32), k=10, 'complete', "
                    f"out=pinned packed block without work counters), {depth} batches in flight; wall clock"),
            "synchronous": sync}


def extras(idx, ds, qs, stream, flush_buf) -> dict:
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

    def graph_of(fn, n):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            fn(0)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for i in range(n):
                    fn(i)
        return g

    def per_step_ms(fn, n_graph, reps):
        g = graph_of(fn, n_graph)
        with torch.cuda.stream(stream):  # replay() launches on the current stream
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                g.replay()
            b.record(stream)
            torch.cuda.synchronize()
        return a.elapsed_time(b) / (n_graph * reps), g

    idx_fn = lambda i: idx.native.query_device(dq[i % n_pool], K, "complete", ids, lcps, hits, stream=st)
    # prefix-16 query variant, one batch in flight
    qp = lg.generate_queries(ds, BATCH, seed=5, prefix_len=16)
    dqp = torch.from_numpy(qp).to(dev)
    ms, _ = per_step_ms(lambda i: idx.native.query_device(dqp, K, "complete", ids, lcps, hits, stream=st), 64, 20)
    out["indexed_prefix16_qps"] = BATCH / (ms / 1e3)
    # strict mode on the same batches
    ms, _ = per_step_ms(lambda i: idx.native.query_device(dq[i % n_pool], K, "strict", ids, lcps, hits, stream=st), 64, 20)
    out["indexed_strict_qps"] = BATCH / (ms / 1e3)
    # brute-force full-scan kernel on the same batches
    fs_fn = lambda i: idx.native.fullscan_device(dq[i % n_pool], K, ids, lcps, hits, stream=st)
    ms, _ = per_step_ms(fs_fn, 4, 3)
    out["fullscan_qps"] = BATCH / (ms / 1e3)
    out["fullscan_ms_per_batch"] = ms
    out["fullscan_key_stream_gbs"] = N_ITEMS * 8 / (ms / 1e3) / 1e9
    # the single-query full scan (the reference's oracle_top_k(dataset, q, k)
    # call): the small-batch streaming kernel, HBM-bound on large corpora
    fs1_fn = lambda i: idx.native.fullscan_device(dq[i % n_pool][i % BATCH:i % BATCH + 1], K, ids[:1],
                                                  lcps[:1], hits[:1], stream=st)
    ms1, _ = per_step_ms(fs1_fn, 32, 5)
    alg = N_ITEMS * algorithmic_key_bytes(SEQ_LEN, SIGMA) + (algorithmic_key_bytes(SEQ_LEN, SIGMA) + 6 * K)
    peak = hbm_peak()[0]
    out["fullscan_single_query"] = {
        "us_per_query": ms1 * 1e3, "algorithmic_gbs": alg / (ms1 / 1e3) / 1e9,
        "frac": alg / (ms1 / 1e3) / 1e9 / peak, "kernel": "k_fullscan_smallq<u32,1>",
        "note": "N*K_b + K_b + 6k algorithmic bytes per call; the kernel reads the 4-byte hi plane "
                "(half of K_b) and the rare survivors' lo words; 2M keys are one 8 MB pass, so the "
                "launch, the seed and the merges dominate here (at N=200M: profiles/README.md)"}
    # TAL B=256 (paper's bounded-range scan)
    tal = lg.build_tal(ds, 256)
    tal_fn = lambda i: tal.native.query_device(dq[i % n_pool], K, "tal", ids, lcps, hits, stream=st)
    ms, _ = per_step_ms(tal_fn, 8, 5)
    out["tal256_qps"] = BATCH / (ms / 1e3)
    # SURVEY §8d TAL bytes: keys + ids of every distinct bucket the batch hits,
    # plus 8 + K_b + 6k per query.  That is the TAL algorithm's traffic (it
    # scans the bucket); the kernel gets the same answer and counters without
    # sweeping it, so this fraction credits the algorithm, not bytes moved
    try:
        qs0 = qs[:BATCH].astype(np.int64)
        code = np.zeros(BATCH, np.int64)
        for j in range(tal.bucket_depth):
            code = code * SIGMA + qs0[:, j]
        dirs = tal.directory
        uniq = np.unique(code)
        kb = algorithmic_key_bytes(SEQ_LEN, SIGMA)
        tal_bytes = float((dirs[uniq + 1] - dirs[uniq]).sum()) * (kb + 4) + BATCH * (8 + kb + 6 * K)
        out["tal256_roofline"] = {
            "bytes_per_batch": tal_bytes, "buckets_hit": int(uniq.size), "batch_us": ms * 1e3,
            "achieved_gbs": tal_bytes / (ms / 1e3) / 1e9, "frac": tal_bytes / (ms / 1e3) / 1e9 / peak,
            "formula": "SURVEY §8d: sum over distinct buckets hit of |B|*(K_b+4) + Q*(8 + K_b + 6k); "
                       "one batch in flight, back-to-back graph replays"}
    except Exception as e:  # pragma: no cover - reporting only
        out["tal256_roofline"] = {"unavailable": f"{type(e).__name__}: {e}"}
    # energy: NVML counter over >= 3 s of graph-replayed batches (gross, and net of idle)
    energy = nvml_energy()
    if energy is not None:
        def joules_per_query(fn, n_graph, seconds=3.0):
            g = graph_of(fn, n_graph)
            with torch.cuda.stream(stream):
                g.replay()
                torch.cuda.synchronize()
                e0, t0, done = energy(), time.perf_counter(), 0
                while time.perf_counter() - t0 < seconds:
                    g.replay()
                    done += BATCH * n_graph
                    torch.cuda.synchronize()
                el = time.perf_counter() - t0
                return (energy() - e0) / done, done / el
        time.sleep(0.5)
        e0 = energy()
        time.sleep(2.0)
        idle_w = (energy() - e0) / 2.0
        jq_idx, qps_idx = joules_per_query(idx_fn, 256)
        jq_fs, qps_fs = joules_per_query(fs_fn, 4)
        jq_tal, qps_tal = joules_per_query(tal_fn, 16)
        out["energy"] = {
            "idle_w": idle_w,
            "indexed_j_per_query": jq_idx, "indexed_net_j_per_query": jq_idx - idle_w / qps_idx,
            "fullscan_j_per_query": jq_fs, "fullscan_net_j_per_query": jq_fs - idle_w / qps_fs,
            "tal256_j_per_query": jq_tal, "tal256_net_j_per_query": jq_tal - idle_w / qps_tal,
            "fullscan_over_indexed": jq_fs / jq_idx,
            "method": "NVML total-energy delta over >=3 s of CUDA-graph-replayed batches (one in flight)",
        }
    # config 3 with sigma = 65536: W = 8 (64-byte keys), index 2M x 76 B > L2
    d8 = lg.generate_dataset(N_ITEMS, SEQ_LEN, 65536, seed=3)
    i8 = lg.build(d8)
    q8 = torch.from_numpy(lg.generate_queries(d8, BATCH, seed=4, prefix_len=2)).to(dev)
    ms8, _ = per_step_ms(lambda i: i8.native.query_device(q8, K, "complete", ids, lcps, hits, stream=st), 16, 10)
    out["indexed_sigma65536_qps"] = BATCH / (ms8 / 1e3)
    out["indexed_sigma65536_device_bytes"] = i8.nbytes
    # its roofline (SURVEY §8d bytes with K_b = 64 B; |R(d*)| from the aux words)
    md8 = torch.empty(BATCH, dtype=torch.int16, device=dev)
    aux8 = torch.empty((BATCH, 2), dtype=torch.int64, device=dev)
    i8.native.query_device(q8, K, "complete", ids, lcps, hits, md8, aux8, stream=st)
    torch.cuda.synchronize()
    rs8 = (aux8[:, 1].cpu().numpy().astype(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)
    # a query whose d* is 0 has R(d*) = the whole corpus; the formula's
    # |R(d*)| * (K_b + 4) would charge it 136 MB although the answer comes from
    # the id sketch, so runs are charged at most the 64-key leaf region
    b8 = float(indexed_bytes_per_query(N_ITEMS, SEQ_LEN, 65536, K, np.minimum(rs8, 64)).sum())
    out["indexed_sigma65536_roofline"] = {
        "bytes_per_batch": b8, "batch_us": ms8 * 1e3, "achieved_gbs": b8 / (ms8 / 1e3) / 1e9,
        "frac": b8 / (ms8 / 1e3) / 1e9 / peak, "kernel": "k_query_warp<8>",
        "queries_with_run_over_64": int((rs8 > 64).sum()),
        "note": "one batch in flight, back-to-back graph replays; SURVEY §8d indexed bytes with K_b = 64 "
                "and |R(d*)| capped at the 64-key region (longer runs are served by the id sketch)"}
    del i8, d8
    # config 3, clustered stress (datagen.py:42-52: skew 1.1, depth 8): long
    # shared prefixes make R(d*) wide for many queries
    dc = lg.generate_dataset(N_ITEMS, SEQ_LEN, SIGMA, seed=3, distribution="clustered")
    ic = lg.build(dc)
    for tag, pl in (("uniform", None), ("prefix16", 16)):
        qc = torch.from_numpy(lg.generate_queries(dc, BATCH, seed=4, prefix_len=pl)).to(dev)
        msc, _ = per_step_ms(lambda i: ic.native.query_device(qc, K, "complete", ids, lcps, hits,
                                                             stream=st), 32, 20)
        out[f"indexed_clustered_{tag}_qps"] = BATCH / (msc / 1e3)
    del ic, dc
    # config 4: the N x N materialisation wall vs the index (PAPER.md:493-496,
    # reference bench.memory_wall: n*n*2 bytes of fp16 similarities)
    n4 = 500_000
    free_b, total_b = torch.cuda.mem_get_info()
    mat_b = n4 * n4 * 2
    try:
        wall = torch.empty((n4, n4), dtype=torch.float16, device=dev)
        alloc = "succeeded (unexpected)"
        del wall
    except torch.OutOfMemoryError as e:
        alloc = "torch.OutOfMemoryError: " + str(e).split("\n")[0][:120]
    d4 = lg.generate_dataset(n4, 32, SIGMA, seed=5)
    i4 = lg.build(d4)
    q4 = torch.from_numpy(lg.generate_queries(d4, BATCH, seed=6)).to(dev)
    ms4, _ = per_step_ms(lambda i: i4.native.query_device(q4, K, "complete", ids, lcps, hits, stream=st), 64, 20)
    out["oom_boundary_config4"] = {
        "n": n4, "materialization_bytes": mat_b, "materialization_gib": mat_b / 2**30,
        "free_hbm_bytes": int(free_b), "feasible": mat_b <= free_b, "nxn_fp16_alloc": alloc,
        "index_device_bytes": i4.nbytes, "reference_arena_bytes": i4.arena_nbytes,
        "materialization_over_index": mat_b / i4.nbytes,
        "indexed_qps": BATCH / (ms4 / 1e3),
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
    # the same loop in latency mode: a resident warp answers through mailboxes
    # in page-locked host memory (no launch, copy or event per query); every
    # answer is checked against the batch API (nothing in the block
    # synchronises the device: the warp stays resident while it is in use)
    ref = gi.query_batch(readings, 5, "complete")
    lat = []
    with gi.low_latency(5, "complete"):
        for q in readings[:20]:
            gi.query(q, 5, "complete")
        for i, q in enumerate(readings):
            t0 = time.perf_counter()
            r = gi.query(q, 5, "complete")
            lat.append(time.perf_counter() - t0)
            if r.pairs() != ref.pairs(i):
                raise RuntimeError(f"latency-mode answer {i} differs from the batch API")
    out["gnc_single_query_low_latency"] = {
        "hz": len(lat) / float(np.sum(lat)), "p50_ms": 1e3 * float(np.median(lat)),
        "p99_ms": 1e3 * float(np.percentile(lat, 99)),
        "api": "with TrieIndex.low_latency(5, 'complete'): TrieIndex.query(q, 5, 'complete') per step, "
               "N=100k, L=24 (csrc/serve_kernels.cuh)"}
    return out


if __name__ == "__main__":
    main()
