#!/usr/bin/env python3
"""Benchmark: batched bicluster-fitness evaluation on B200 (EBIC hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c2|c4|c5|spec] [--shard rows|pop|replica]
                    [--l2 auto|stream|flush]

A STEP is one pass of the hot path over one batch: evaluate_population of P
candidates against all R rows (trend.cpp:56-72), i.e. P fitness evals and P*R
row-checks.  Metric (BASELINE.json): candidate fitness evals/s (row-checks/s
reported alongside), % of the HBM roofline.

Default workload = BASELINE configs[2] ("c3"): 20k x 1000 planted-trend float32
matrix, P = 16384 (L uniform in [3,5]), approx 0.03.  BASELINE's metric and both
of its numeric targets (>= 60% HBM roofline at 20k x 1000; >= 6x at 8 GPUs
row-sharded) are quoted on this configuration.

--gpus N > 1 without WORLD_SIZE in the environment re-launches this script
under torch.distributed.run with N ranks (one per GPU; it fails unless N GPUs
are visible, or --share-gpu lets the ranks share GPUs for testing).  Under
torchrun WORLD_SIZE must equal N.  N > 1, --shard:
  rows (default) -- BASELINE config 3: the matrix rows are sharded, every rank
           evaluates the whole population on its shard and the partial counts
           are summed over NVLink peer memory (ebic_xchg.cuh; --exchange nccl:
           an NCCL all_reduce).  Steps are pipelined: step k's exchange runs on
           the exchange stream while step k+1's count kernel runs.  Strong
           scaling: the whole job evaluates P candidates per step.
  pop      -- one population split across ranks, counts all-gathered (strong).
  replica  -- every rank evaluates its own P-candidate population against the
           replicated matrix, no collective (weak scaling; secondary mode).

Timing (--l2): `stream` (default when the per-rank index is larger than twice
the 126 MB L2) -- K steps issued back to back, populations cycled from a pool
whose pair vectors cover more than twice the L2, so no step finds its inputs
in L2 and nothing is flushed; `flush` -- a 512 MiB device read before every
step (outside the step's events).  Both are CUDA events on the launching
stream, max over ranks.

value    : device-resident populations, whole job's evals / step time.
e2e      : the same metric through the public host API (ebic_eval_counts,
           or ShardedEvaluator for N > 1): host arrays in, counts out, every
           step's H2D / D2H inside the timed region.
roofline : the count kernel's PHYSICAL HBM bytes (pair vectors it must stream:
           4 B x wp words x (L-1) pairs per candidate, x2 with negatives) over
           its measured time (sum bytes / sum time), vs the measured HBM peak.
           SURVEY 8(d)'s 4*L*R algorithmic bytes are reported separately as
           `effective_algorithmic` (the index kernel never reads the matrix).
amortized: the one-time upload + rank plane + index build spread over the
           timed steps and over a declared GA run.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "candidate fitness evals/s & row-checks/s at 1/2/4/8 B200; % of HBM roofline"
L2_BYTES = 126 * 1024 * 1024
GA_GENERATIONS = 200  # the declared GA run of the amortized fields: BASELINE config 1's iteration count

CONFIGS = {
    # name: rows, cols, population, len range, approx, negative, planted (rows, cols)
    "c2": dict(rows=10_000, cols=500, pop=4096, len_min=3, len_max=5, approx=0.03, negative=False, bic=(500, 20),
               label="c2: 10k x 500 planted-trend f32 matrix, P=4096 (L in [3,5]), approx 0.03"),
    "c3": dict(rows=20_000, cols=1000, pop=16384, len_min=3, len_max=5, approx=0.03, negative=False, bic=(500, 20),
               label="c3: 20k x 1000 planted-trend f32 matrix, P=16384 (L in [3,5]), approx 0.03"),
    "c4": dict(rows=200_000, cols=2000, pop=32768, len_min=3, len_max=5, approx=0.03, negative=False,
               bic=(5000, 20),
               label="c4: 200k x 2000 planted-trend f32 matrix (1.6 GB), P=32768 (L in [3,5]), approx 0.03"),
    "c5": dict(rows=1_000_000, cols=64, pop=1024, len_min=16, len_max=16, approx=0.03, negative=False,
               bic=(10_000, 16),
               label="c5 microbench point: 1M x 64 f32, P=1024, L=16, approx 0.03"),
    # SPEC.md:593's performance shape at the reference's own GA batch size
    # (P=400, evolution.hpp:21; 392 offspring per generation, evolution.cpp:291)
    "spec": dict(rows=20_000, cols=250, pop=392, len_min=3, len_max=5, approx=0.03, negative=False,
                 bic=(500, 20),
                 label="spec: 20k x 250 planted-trend f32 matrix, P=392 (one GA generation at the reference "
                       "defaults), L in [3,5], approx 0.03"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config: str, world: int):
    """dram read+write bytes per launch of the fitness kernel from the committed ncu capture."""
    p = REPO / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        rec = d.get(config)
        if rec and world == 1:
            return rec["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled DURING the timed region.

    NVML (nvidia-ml-py) polled every ~1 ms from a thread -- the timed region is
    only tens of milliseconds, too short for `nvidia-smi -lms`; nvidia-smi is
    the fallback when NVML is unavailable.
    """

    HW_SLOWDOWN, SW_POWER_CAP, SW_THERMAL, HW_THERMAL = 0x8, 0x4, 0x20, 0x40

    def __init__(self, torch_device_index: int):
        self.dev_index = torch_device_index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self._handle = None
        self._nvml = None

    def _open(self):
        import pynvml

        pynvml.nvmlInit()
        self._nvml = pynvml
        handle = None
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.dev_index).uuid)
            handle = pynvml.nvmlDeviceGetHandleByUUID(uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            cvd = [x for x in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if x.strip()]
            idx = cvd[self.dev_index] if self.dev_index < len(cvd) else str(self.dev_index)
            handle = (pynvml.nvmlDeviceGetHandleByUUID(idx) if idx.startswith("GPU-")
                      else pynvml.nvmlDeviceGetHandleByIndex(int(idx)))
        self._handle = handle
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(handle, pynvml.NVML_CLOCK_SM)

    def _reasons(self):
        f = getattr(self._nvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            self._nvml.nvmlDeviceGetCurrentClocksThrottleReasons
        return f(self._handle)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append((self._nvml.nvmlDeviceGetClockInfo(self._handle, self._nvml.NVML_CLOCK_SM),
                                     self._reasons()))
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        try:
            self._open()
            self._stop.clear()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self._handle = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._handle is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0}
        mask = 0
        for _, r in self.samples:
            mask |= int(r)
        reasons = [name for bit, name in ((self.HW_SLOWDOWN, "hw_slowdown"), (self.HW_THERMAL, "hw_thermal_slowdown"),
                                          (self.SW_THERMAL, "sw_thermal_slowdown"), (self.SW_POWER_CAP, "sw_power_cap"))
                   if mask & bit]
        return {"sm_mhz": statistics.median(c for c, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml, ~1 ms polling"}


def make_inputs(cfg, n_pops: int, seed0: int = 42):
    from paper_2105_01196_b200 import synth

    m, _ = synth.planted_trend_matrix(cfg["rows"], cfg["cols"], 3, cfg["bic"][0], cfg["bic"][1], seed=1)
    if cfg["len_min"] == cfg["len_max"]:
        pops = [synth.exact_len_population(cfg["pop"], cfg["cols"], cfg["len_min"], seed=seed0 + i)
                for i in range(n_pops)]
    else:
        pops = [synth.random_population(cfg["pop"], cfg["cols"], cfg["len_min"], cfg["len_max"], seed=seed0 + i)
                for i in range(n_pops)]
    return m, pops


# ---------------------------------------------------------------------------
# CPU baseline: the reference's own evaluate_population on a WorkerPool
# (oracle/_ref, "reference") or the C restatement ("port"), all host threads.
# ---------------------------------------------------------------------------
def cpu_eval_setup(m: np.ndarray):
    import oracle

    if oracle.reference_available():
        mat = oracle.RefMatrix(m.astype(np.float64))
        pool = oracle.RefPool(0)

        def run(pop):
            rp = oracle.RefPopulation(pop.cols, pop.offsets)
            return oracle.ref_evaluate(mat, rp, CUR_APPROX[0], CUR_NEG[0], pool)

        return run, "reference", pool.size
    threads = oracle.port().oracle_threads()

    def run(pop):
        return oracle.evaluate_population(m, pop.cols, pop.offsets, CUR_APPROX[0], CUR_NEG[0], threads=threads)

    return run, "port", threads


CUR_APPROX = [0.03]
CUR_NEG = [False]


def cpu_sample(run, pops, budget_s: float, cap=None):
    """Evaluate whole populations (then a prefix of the next one) until ~budget_s
    seconds of CPU work; returns (n_candidates, seconds, counts of pops[0] prefix)."""
    from paper_2105_01196_b200.shard import slice_population

    if not isinstance(pops, (list, tuple)):
        pops = [pops]
    probe_n = min(len(pops[0]), 64)
    t0 = time.perf_counter()
    run(slice_population(pops[0], 0, probe_n))
    per_cand = max((time.perf_counter() - t0) / probe_n, 1e-9)
    want = int(max(1, budget_s / per_cand))
    if cap:
        want = min(want, cap)
    n_done, secs, first = 0, 0.0, None
    i = 0
    while n_done < want:
        pop = pops[i % len(pops)]
        take = min(len(pop), want - n_done)
        sub = slice_population(pop, 0, take)
        t0 = time.perf_counter()
        out = run(sub)
        secs += time.perf_counter() - t0
        if first is None:
            first = out
        n_done += take
        i += 1
    return n_done, secs, first


def bench_reference(args, cfg, rank):
    if rank != 0:
        return 0
    CUR_APPROX[0], CUR_NEG[0] = cfg["approx"], cfg["negative"]
    m, pops = make_inputs(cfg, 1)
    run, kind, cores = cpu_eval_setup(m)
    pop = pops[0]
    per_step = float(os.environ.get("EBIC_REF_STEP_S", "3.0"))
    for _ in range(args.warmup):
        cpu_sample(run, pop, min(per_step, 1.0), cap=len(pop))
    tot_n, tot_t = 0, 0.0
    n_step = None
    for _ in range(args.steps):
        n, t, _ = cpu_sample(run, pop, per_step, cap=len(pop) if n_step is None else n_step)
        n_step = n
        tot_n += n
        tot_t += t
    value = tot_n / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak" if args.shard == "replica" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (planted-trend f32 matrix, random populations; no dataset)",
        "row_checks_per_s": value * cfg["rows"],
        "config": {"workload": cfg["label"], "rows": cfg["rows"], "cols": cfg["cols"], "population": cfg["pop"],
                   "parallelism": f"cpu: the reference's WorkerPool on {cores} host threads (rank 0 only)",
                   "shard": args.shard},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": kind,
                         "sample": f"{n_step} of {cfg['pop']} candidates x all {cfg['rows']} rows per step "
                                   f"(reference evaluate_population on WorkerPool({cores}))" if kind == "reference"
                         else f"{n_step} of {cfg['pop']} candidates per step (C restatement, {cores} threads)"},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def index_kernel_name(wp, n_cand, n_sms=148, lazy=False):
    """The index kernel launch_table picks (ebic_capi.cu) for this vector length
    and candidate count, with the default EBIC_TABLE_KERNEL."""
    if wp // 4 <= 32 and not lazy:
        return "table_count_group_kernel"
    if wp // 4 <= 256:
        return "table_count_tma_kernel"
    if lazy:
        return "table_count_warp_multi_kernel"
    return "table_count_warp_multi_kernel" if n_cand >= n_sms * 6 else "table_count_kernel"


def distinct_pairs(pop, n_cols: int, neg: bool) -> int:
    """Distinct pair vectors a batch reads (consecutive (a, b) pairs; (b, a)
    too with negatives): the DRAM bytes it must move at least once when the
    index does not stay in L2 (repeats within a launch may hit L2)."""
    cols = pop.cols.astype(np.int64)
    if cols.size < 2:
        return 0
    starts = np.zeros(cols.size, dtype=bool)
    starts[pop.offsets[:-1][pop.offsets[:-1] < cols.size].astype(np.int64)] = True
    k = np.nonzero(~starts[1:])[0] + 1  # positions k with a pair (k-1 -> k) in the same candidate
    keys = cols[k - 1] * n_cols + cols[k]
    if neg:
        keys = np.concatenate([keys, cols[k] * n_cols + cols[k - 1]])
    return int(np.unique(keys).size)


def table_wp(rows: int) -> int:
    """Words per pair vector (ebic_capi.cu table_wp)."""
    words = (rows + 31) // 32
    return (words + 127) // 128 * 128 if words > 128 else (words + 3) // 4 * 4


def pool_size(cfg, rows_rank: int, want_bytes: float) -> int:
    """Populations to cycle so the distinct pair vectors they touch cover
    `want_bytes` (expected over random draws of the C^2 ordered pairs)."""
    c2 = cfg["cols"] ** 2
    pairs = cfg["pop"] * ((cfg["len_min"] + cfg["len_max"]) / 2 - 1)
    vec = 4 * table_wp(rows_rank)
    for n in range(4, 65):
        if c2 * vec * (1 - math.exp(-n * pairs / c2)) >= want_bytes:
            return n
    return 64


class Collective:
    """Barrier / max / sum over ranks on whatever device the backend needs."""

    def __init__(self, dist, dev):
        self.dist = dist
        self.dev = dev if (dist is not None and dist.get_backend() == "nccl") else "cpu"

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def all_reduce_sum_(self, t):
        if self.dist is None:
            return t
        if self.dev == "cpu":
            c = t.cpu()
            self.dist.all_reduce(c, op=self.dist.ReduceOp.SUM)
            t.copy_(c)
        else:
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t


def bench_ours(args, cfg, rank, world, local_rank, dist):
    import torch

    from paper_2105_01196_b200 import Evaluator, Population, TrendParams
    from paper_2105_01196_b200.shard import ShardedEvaluator, pop_range, row_range, slice_population

    n_dev = max(torch.cuda.device_count(), 1)
    local_rank = local_rank % n_dev  # --share-gpu: ranks may share a GPU
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    coll = Collective(dist, dev)
    tp = TrendParams(approx=cfg["approx"], negative_trends=cfg["negative"])
    shard = args.shard
    R, Ccols, P = cfg["rows"], cfg["cols"], cfg["pop"]
    b, e = row_range(R, rank, world) if shard == "rows" else (0, R)
    replica = shard == "replica"
    p2p = shard == "rows" and args.exchange == "p2p"
    neg_factor = 2 if cfg["negative"] else 1

    # ---- populations: a pool large enough that the stream mode never finds
    # a step's pair vectors in L2 (see pool_size)
    want = 2.0 * L2_BYTES
    n_pops = args.pops or pool_size(cfg, e - b, want)
    m, pops = make_inputs(cfg, n_pops, seed0=42 + (1000 * rank if replica else 0))
    if shard == "pop":
        pops_local = [slice_population(pp, *pop_range(P, rank, world)) for pp in pops]
    else:
        pops_local = pops

    # ---- one-time: upload + (matrix, approx) index --------------------------
    ev = Evaluator(local_rank)
    ev.set_path({"auto": 0, "value": 1, "plane": 2, "table": 4}[args.path])
    if args.index_budget_gb is not None:
        ev.set_table_budget(int(args.index_budget_gb * (1 << 30)))
    # process start-up (lazy CUDA module loading, the page-locked staging
    # buffers) is paid once per process, not per matrix: a 34-MB warm-up
    # upload (staged like the real one) and evaluation take it out of the
    # per-matrix one-time costs below (`cold_start` reports the cold figures)
    wm = np.random.default_rng(0).standard_normal((16800, 500)).astype(np.float32)
    ev.upload(wm)
    ev.evaluate_population(Population.from_sequences([[0, 1, 2], [3, 4]]), tp)
    del wm
    # the median of three uploads of the matrix: the host side (pageable
    # source pages, staging threads) varies by tens of ms between runs on a
    # shared host
    mine = np.ascontiguousarray(m[b:e])
    ups = []
    for _ in range(3):
        t0 = time.perf_counter()
        ev.upload(mine, row_base=b)
        ups.append((time.perf_counter() - t0) * 1e3)
    upload_ms = sorted(ups)[1]
    del mine
    t0 = time.perf_counter()
    ev.prepare(cfg["approx"])
    prepare_ms = (time.perf_counter() - t0) * 1e3
    build = ev.build_info()
    index_bytes, index_used = ev.index_info()
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ev.set_stream(stream.cuda_stream)
    exchange_note = None
    if p2p:
        # peer-memory exchange windows; if any rank cannot map its peers (no
        # P2P between the GPUs), every rank falls back to the NCCL all_reduce
        # and the line says so
        h = ev.xchg_create(world, rank, P)
        handles = [None] * world
        dist.all_gather_object(handles, h)
        err = ""
        try:
            ev.xchg_open(handles)
        except Exception as ex:  # noqa: BLE001 -- reported in the line
            err = str(ex)
        errs = [None] * world
        dist.all_gather_object(errs, err)
        if any(errs):
            p2p = False
            exchange_note = "p2p unavailable (%s): NCCL all_reduce" % next(e for e in errs if e)
            log("exchange:", exchange_note)
            ev.xchg_destroy()

    d_pops = [(torch.from_numpy(pp.cols.view(np.int32)).to(dev), torch.from_numpy(pp.offsets.view(np.int32)).to(dev),
               len(pp), int(pp.cols.size)) for pp in pops_local]
    n_local = d_pops[0][2]
    counts = torch.zeros(P, dtype=torch.int32, device=dev)

    def step(i, pipelined=True):
        dc, do, n, _ = d_pops[i % n_pops]
        if p2p:
            if pipelined:
                ev.evaluate_population_rows_sum_async(dc.data_ptr(), do.data_ptr(), n, counts.data_ptr(), tp,
                                                      stream=stream.cuda_stream)
            else:
                ev.evaluate_population_rows_sum_device(dc.data_ptr(), do.data_ptr(), n, counts.data_ptr(), tp,
                                                       stream=stream.cuda_stream)
            return
        out = counts[:n]
        ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), n, out.data_ptr(), tp, stream=stream.cuda_stream)
        if world > 1 and shard == "rows":  # --exchange nccl
            coll.all_reduce_sum_(counts)
        elif world > 1 and shard == "pop":
            gathered = [torch.empty_like(out) for _ in range(world)]
            dist.all_gather(gathered, out)

    def finish():
        if p2p:
            ev.xchg_fence(stream.cuda_stream)

    # ---- warmup -------------------------------------------------------------
    # every population of the pool twice: with the lazy index the first visit
    # of a population builds its new pair vectors (timed here and reported as
    # a one-time cost), the second settles the pool's size (it grows when a
    # batch's worst case may not fit); later visits only read it
    n_warm = max(args.warmup, 3, 2 * n_pops)
    w_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_warm)]
    for i in range(n_warm):
        if i == n_pops:
            # the host runs ahead of the device: sync once so that the pool's
            # size is settled (grown if a worst-case batch may not fit) here,
            # not on the first timed step
            torch.cuda.synchronize()
        w_ev[i][0].record(stream)
        step(i)
        w_ev[i][1].record(stream)
    finish()
    torch.cuda.synchronize()
    ev.sync()
    coll.barrier()
    warm_ms = [a.elapsed_time(z) for a, z in w_ev]
    index_mode = ev.index_stats()["mode"]
    lazy = index_mode == "lazy"
    index_used = index_mode in ("full", "lazy")
    if lazy:
        index_bytes = ev.index_stats()["lazy_bytes"]

    # L2 mode
    wp = (index_bytes // (4 * Ccols ** 2)) if (index_mode == "full" and index_bytes) else table_wp(e - b)
    per_rank_index = index_bytes if index_used else 0
    l2_mode = args.l2
    if l2_mode == "auto":
        l2_mode = "stream" if (index_used and per_rank_index > 2 * L2_BYTES) else "flush"
    flush = torch.ones(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if l2_mode == "flush" else None
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)

    def flush_l2():
        if flush is not None:
            torch.sum(flush, dim=0, out=flush_sink)

    # ---- timed region ---------------------------------------------------------
    launches0 = ev.launch_count()
    clocks = ClockSampler(local_rank)
    torch.cuda.synchronize()
    coll.barrier()
    with clocks:
        w0 = time.perf_counter()
        if l2_mode == "stream":
            t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t_start.record(stream)
            for i in range(args.steps):
                step(i)
            finish()
            t_end.record(stream)
            torch.cuda.synchronize()
            total_ms = t_start.elapsed_time(t_end)
        else:
            starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            for i in range(args.steps):
                flush_l2()  # outside the step events
                starts[i].record(stream)
                step(i, pipelined=False)
                ends[i].record(stream)
            torch.cuda.synchronize()
            total_ms = sum(s.elapsed_time(t) for s, t in zip(starts, ends))
        coll.barrier()
        wall = time.perf_counter() - w0
    launches = ev.launch_count() - launches0
    ev.sync()  # raises on any device-side error of the timed steps (bad column, exchange timeout / poison)
    total_ms = coll.max(total_ms)
    ms_per_step = total_ms / args.steps
    p_total = P * world if replica else P
    value = p_total / (ms_per_step / 1e3)

    # ---- kernel pass: the count kernel alone, events around every launch ----
    k0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    k1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    kout = torch.zeros(P, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    for i in range(args.steps):
        if l2_mode == "flush":
            flush_l2()
        dc, do, n, _ = d_pops[i % n_pops]
        k0[i].record(stream)
        ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), n, kout.data_ptr(), tp, stream=stream.cuda_stream)
        k1[i].record(stream)
    torch.cuda.synchronize()
    kern_ms = [a.elapsed_time(z) for a, z in zip(k0, k1)]
    per_rank = None
    if p2p:
        # unpipelined steps: count + exchange, serialised (exchange = the difference)
        s0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        s1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        coll.barrier()
        for i in range(args.steps):
            s0[i].record(stream)
            step(i, pipelined=False)
            s1[i].record(stream)
        torch.cuda.synchronize()
        ser = statistics.mean(a.elapsed_time(z) for a, z in zip(s0, s1))
        per_rank = {"rank": rank, "rows": [b, e], "kernel_us": 1e3 * statistics.mean(kern_ms),
                    "step_unpipelined_us": 1e3 * ser, "exchange_us": 1e3 * max(0.0, ser - statistics.mean(kern_ms)),
                    "step_pipelined_us": 1e3 * ms_per_step}
    ev.sync()

    # roofline of the count kernel on this rank
    n_pairs = [int(dp[3]) - int(dp[2]) for dp in d_pops]
    reads = [4.0 * wp * npair * neg_factor for npair in n_pairs]  # every pair read (L2 hits included)
    if index_used:  # the distinct pair vectors the kernel must stream from HBM
        phys = [4.0 * wp * distinct_pairs(pp, Ccols, cfg["negative"]) for pp in pops_local]
    else:  # the slab kernels stage the rank plane (the value kernel: the store) once per launch
        phys = [4.0 * (e - b) * Ccols for _ in n_pairs]
    alg = [4.0 * (e - b) * int(dp[3]) for dp in d_pops]
    kb = [phys[i % n_pops] for i in range(args.steps)]
    ka = [alg[i % n_pops] for i in range(args.steps)]
    ksum_s = sum(kern_ms) / 1e3
    peak, peak_src = measured_peak()
    phys_gbs = sum(kb) / ksum_s / 1e9
    alg_gbs = sum(ka) / ksum_s / 1e9
    kernel = ((index_kernel_name(wp, n_local, lazy=lazy) +
               (" (lazy pair-trend index)" if lazy else " (pair-trend index)")) if index_used else
              "slab_pair_kernel (packed rank pairs)" if Ccols <= 2048 else "slab_count_kernel (rank plane)") \
        if (args.path != "value" and Ccols <= 8192) else "fitness_count_kernel (value)"
    # first visits of the pool's populations with the lazy index: the extra time
    # over a steady-state step is the vector building (a one-time cost per pair)
    lazy_build_ms = coll.max(max(0.0, sum(warm_ms[:n_pops]) - n_pops * statistics.mean(kern_ms))) if lazy else 0.0

    # ---- e2e through the public host API -------------------------------------
    ev.set_stream(None)
    torch.cuda.set_stream(torch.cuda.default_stream(dev))
    keep = []

    def pinned(a):
        t = torch.empty(a.size, dtype=torch.int32, pin_memory=True)
        keep.append(t)
        v = t.numpy().view(np.uint32)
        v[:] = a
        return v

    def pinned_csr(pp):  # one page-locked block [offsets | cols]: the library DMAs it in one copy
        buf = pinned(np.concatenate([pp.offsets, pp.cols]))
        n1 = pp.offsets.size
        return Population(buf[n1:], buf[:n1])

    n_e2e = min(n_pops, 8)
    if world > 1 and not replica:
        # the context already holds this rank's shard and its exchange window
        sev = ShardedEvaluator.attach(ev, R, Ccols, mode=shard, dist=dist,
                                      exchange="p2p" if p2p else "collective", max_cand=P)
        e2e_pops = pops[:n_e2e]
        call = sev.evaluate_population
        api = f"ShardedEvaluator({shard}, exchange={sev.exchange}).evaluate_population"
    else:
        e2e_pops = [pinned_csr(pp) for pp in pops_local[:n_e2e]]
        out_pinned = pinned(np.zeros(P, dtype=np.uint32))

        def call(pop, params):
            return ev.evaluate_population(pop, params, out=out_pinned)
        api = "ebic_eval_counts (Evaluator.evaluate_population), pinned host arrays"
    for i in range(max(args.warmup, 8)):  # >= 2x the marshaller ring: every pinned slot allocated
        call(e2e_pops[i % n_e2e], tp)
    e2e_ms = []
    for i in range(args.steps):
        if l2_mode == "flush":
            flush_l2()
        torch.cuda.synchronize()
        coll.barrier()
        t0 = time.perf_counter()
        call(e2e_pops[i % n_e2e], tp)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_tot = coll.max(sum(e2e_ms))
    e2e_step = e2e_tot / args.steps
    e2e_value = p_total / (e2e_step / 1e3)
    # the same host-array steps through the asynchronous marshaller
    # (ebic_eval_submit / ebic_eval_wait, the API the GA driver uses): step
    # i + 1 is submitted before step i is waited for, so one step's copies and
    # host work overlap the other's kernel; every step's H2D and D2H are still
    # inside the timed region (one-rank layouts only)
    e2e_pipe = None
    if world == 1 or replica:
        outs = [pinned(np.zeros(P, dtype=np.uint32)) for _ in range(2)]
        for i in range(max(args.warmup, 8)):
            ev.wait(ev.submit(e2e_pops[i % n_e2e], outs[i % 2], tp))
        torch.cuda.synchronize()
        coll.barrier()
        t0 = time.perf_counter()
        prev = None
        for i in range(args.steps):
            t = ev.submit(e2e_pops[i % n_e2e], outs[i % 2], tp)
            if prev is not None:
                ev.wait(prev)
            prev = t
        ev.wait(prev)
        pipe_step = coll.max((time.perf_counter() - t0) * 1e3) / args.steps
        ok_pipe = bool(np.array_equal(outs[(args.steps - 1) % 2][:P],
                                      np.asarray(call(e2e_pops[(args.steps - 1) % n_e2e], tp))[:P]))
        e2e_pipe = {"value": p_total / (pipe_step / 1e3), "ms_per_step": pipe_step, "parity_vs_sync_call": ok_pipe,
                    "api": "ebic_eval_submit / ebic_eval_wait (Evaluator.submit / wait), two steps in flight, "
                           "pinned host arrays; host clock over all steps"}
    pop0 = e2e_pops[0]
    h2d = int(pop0.cols.nbytes + pop0.offsets.nbytes)
    d2h = 4 * (P if not (shard == "pop") else n_local)

    # ---- parity spot checks (no oracle here: two independent device paths) ---
    host0 = np.array(call(e2e_pops[0], tp), copy=True)
    dc, do, n, _ = d_pops[0]
    ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), n, kout.data_ptr(), tp)
    ev.sync()
    local0 = kout[:n].clone()
    if world > 1 and shard == "rows":
        coll.all_reduce_sum_(local0)  # the partial counts summed by the process group, not the exchange windows
    parity = bool(np.array_equal(local0.cpu().numpy().view(np.uint32)[:len(host0)], host0)) \
        if shard != "pop" else None

    # ---- one-time costs, amortized ---------------------------------------------
    one_time_ms = coll.max(upload_ms + prepare_ms) + lazy_build_ms
    k = args.steps
    amort = {
        "one_time_ms": {"total": one_time_ms, "upload": upload_ms, "prepare": prepare_ms,
                        "index_alloc": build["alloc_ms"], "plane": build["plane_ms"], "index": build["index_ms"],
                        "lazy_build": lazy_build_ms,
                        "note": "per-(matrix, approx) costs after a warm-up upload of another matrix (process "
                                "start-up -- lazy module loading, page-locked staging -- is in cold_start); "
                                "upload = H2D + finiteness/exactness check + transpose (host clock, median of "
                                "3 uploads); prepare = "
                                "index allocation (host clock) + rank plane + pair-trend index (CUDA events); "
                                "lazy_build = first visits of the cycled populations with the lazy index minus "
                                "as many steady-state kernel times (CUDA events); max over ranks"},
        "value_amortized": p_total * k / ((total_ms + one_time_ms) / 1e3),
        "e2e_amortized": p_total * k / ((e2e_tot + one_time_ms) / 1e3),
        "over_timed_steps": k,
        "ga_run": {"generations": GA_GENERATIONS, "population": p_total,
                   "value": p_total * GA_GENERATIONS / ((GA_GENERATIONS * ms_per_step + one_time_ms) / 1e3),
                   "e2e": p_total * GA_GENERATIONS / ((GA_GENERATIONS * e2e_step + one_time_ms) / 1e3),
                   "note": f"{GA_GENERATIONS} generations (BASELINE config 1's iteration count) of this "
                           f"step's population, one upload + index build"},
    }

    parallelism = ("1 GPU" if world == 1 else
                   f"rows-sharded x{world}: every rank holds R/{world} rows and evaluates the whole population; "
                   + ("partial counts summed over NVLink peer memory (exchange windows, pipelined)" if p2p
                      else "partial counts summed with an NCCL all_reduce") if shard == "rows" else
                   f"population split x{world}, counts all-gathered" if shard == "pop" else
                   f"replicas x{world}: every rank evaluates its own {P}-candidate population, no collective")
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if replica else "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (planted-trend f32 matrix, random populations; no dataset)",
        "row_checks_per_s": value * R,
        "config": {"workload": cfg["label"], "rows": R, "cols": Ccols, "population": P,
                   "population_per_step_total": p_total, "parallelism": parallelism, "shard": shard,
                   "path": args.path,
                   "exchange": (exchange_note or ("p2p" if p2p else "nccl")) if shard == "rows" and world > 1 else None,
                   "l2": ("stream: no flush; the per-rank pair-trend index (%.0f MB) exceeds 2x the 126 MB L2 and "
                          "populations are cycled from a pool of %d whose pair vectors cover >= %.0f MB, "
                          "steps issued back to back" % (per_rank_index / 1e6, n_pops, want / 1e6))
                   if l2_mode == "stream" else
                   "flushed before every timed step (512 MiB device read, outside the step events)",
                   "populations_cycled": n_pops},
        "roofline": {"bound": "hbm",
                     "achieved": phys_gbs,
                     "peak": peak, "unit": "GB/s",
                     "frac": phys_gbs / peak,
                     "traffic": ncu_traffic(args.config, world),
                     "kernel": kernel, "kernel_avg_ms": statistics.mean(kern_ms),
                     "bytes_per_launch": statistics.mean(phys),
                     "reads_gbs": (sum(reads[i % n_pops] for i in range(args.steps)) / ksum_s / 1e9
                                   if index_used else None),
                     "bytes": ("physical: the distinct pair vectors a launch must stream from HBM, 4 B x %d "
                               "words each (consecutive pairs%s, repeats within a launch counted once: they may "
                               "hit L2; reads_gbs counts every read); achieved = sum(bytes) / sum(kernel time) "
                               "over the kernel pass (CUDA events around each launch on its stream)"
                               % (wp, " in both directions (negatives)" if neg_factor == 2 else ""))
                     if index_used else
                     "physical: the rank plane (4 B x R x C) the slab kernel stages into shared memory once per "
                     "launch; the kernel is bound by its shared-memory pipe, not HBM (DESIGN 4.3), so this "
                     "fraction is low by construction",
                     "peak_source": peak_src,
                     "stream": ({"gbs": statistics.mean(phys) / (ms_per_step / 1e3) / 1e9,
                                 "frac": statistics.mean(phys) / (ms_per_step / 1e3) / 1e9 / peak,
                                 "what": "the same physical bytes over the timed region's step time: batches "
                                         "issued back to back overlap one kernel's tail with the next one's start "
                                         "(programmatic dependent launch), which the per-launch events of the "
                                         "kernel pass (and ncu, which serialises launches) exclude"}
                                if (index_used and l2_mode == "stream" and world == 1) else None),
                     "effective_algorithmic": {"bytes_per_launch": statistics.mean(alg), "gbs": alg_gbs,
                                               "x_of_peak": alg_gbs / peak,
                                               "what": "SURVEY 8(d) algorithmic bytes (4 B x L x R per eval, each "
                                                       "referenced f32 element once) over the same kernel time: "
                                                       "the bandwidth a matrix-reading kernel would need to match "
                                                       "this one; not a roofline fraction"}},
        "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_step, "api": api, "pipelined": e2e_pipe},
        "amortized": amort,
        "gpu_launches": int(launches),
        "store": {"upload_ms": upload_ms, "index_build_ms": prepare_ms,
                  "pair_trend_index_bytes": per_rank_index,
                  "index_budget_gb": args.index_budget_gb},
        "wall_ms_timed_region": wall * 1e3,
        "parity_device_vs_host_api": parity,
    }
    if per_rank is not None:
        gathered = [None] * world
        dist.all_gather_object(gathered, per_rank)
        line["per_rank"] = gathered
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        CUR_APPROX[0], CUR_NEG[0] = cfg["approx"], cfg["negative"]
        run, kind, cores = cpu_eval_setup(m)
        n, t, cpu_counts = cpu_sample(run, pops, float(os.environ.get("EBIC_CPU_BUDGET_S", "12")))
        gpu_counts = call(e2e_pops[0], tp)
        line["cpu_baseline"] = {
            "value": n / t, "unit": "evals/s", "cores": cores, "kind": kind,
            "sample": f"{n} candidates (whole {P}-candidate populations, cycled) x all {R} rows, {t:.1f} s "
                      + ("(unmodified reference evaluate_population on WorkerPool)" if kind == "reference"
                         else "(C restatement of trend.cpp, pthreads)"),
            "parity_with_gpu": bool(np.array_equal(cpu_counts, gpu_counts[:len(cpu_counts)])),
        }
    line["clocks"] = clocks.summary()
    line["index"] = ev.index_stats()
    if world == 1 and args.path == "auto":
        line["cold_start"] = cold_start(cfg, m, pops[0], tp, local_rank)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ev.close()
    return 0


def cold_start(cfg, m, pop, tp, device):
    """First-call latency on a fresh context with the library's default policy
    (no prepare(): AUTO picks the lazy index when the full one is large),
    host API with host arrays, then the next calls of the same population."""
    from paper_2105_01196_b200 import Evaluator

    import torch

    # the first batch's device work alone (device API, CUDA events): the
    # lazy index builds the population's pair vectors inside the count kernel.
    # Process-cold (first launch of the lazy kernel in this process: CUDA's
    # lazy module loading) is measured first on a tiny matrix, then a fresh
    # matrix in a fresh context (matrix-cold).
    from paper_2105_01196_b200 import synth
    from paper_2105_01196_b200._lib import EBIC_PATH_LAZY

    ev = Evaluator(device)
    try:
        ev.set_path(EBIC_PATH_LAZY)
        ev.upload(np.ascontiguousarray(m[:256, :64]))
        tiny = synth.random_population(64, 64, 3, 5, seed=3)
        t0 = time.perf_counter()
        ev.evaluate_population(tiny, tp)
        process_cold_ms = (time.perf_counter() - t0) * 1e3
    finally:
        ev.close()
    ev = Evaluator(device)
    try:
        ev.upload(m)
        dc = torch.from_numpy(pop.cols.view(np.int32)).cuda(device)
        do = torch.from_numpy(pop.offsets.view(np.int32)).cuda(device)
        out = torch.empty(len(pop), dtype=torch.int32, device=f"cuda:{device}")
        s = torch.cuda.Stream()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        for k in range(3):
            e[k].record(s)
            ev.evaluate_population_device(dc.data_ptr(), do.data_ptr(), len(pop), out.data_ptr(), tp,
                                          stream=s.cuda_stream)
        e[3].record(s)
        torch.cuda.synchronize()
        ev.sync()
        dev_ms = [e[k].elapsed_time(e[k + 1]) for k in range(3)]
    finally:
        ev.close()
    ev = Evaluator(device)
    try:
        t0 = time.perf_counter()
        ev.upload(m)
        upload_ms = (time.perf_counter() - t0) * 1e3
        calls = []
        for _ in range(3):
            t0 = time.perf_counter()
            ev.evaluate_population(pop, tp)
            calls.append((time.perf_counter() - t0) * 1e3)
        st = ev.index_stats()
        return {"upload_ms": upload_ms, "first_call_ms": calls[0], "second_call_ms": calls[1],
                "third_call_ms": calls[2], "device_first_batch_ms": dev_ms[0], "device_next_batches_ms": dev_ms[1:],
                "process_cold_tiny_call_ms": process_cold_ms,
                "index": st["mode"], "lazy_vectors": st["lazy_slots_used"],
                "index_bytes": st["lazy_bytes"] if st["mode"] == "lazy" else st["full_bytes"],
                "what": "fresh context, upload, then evaluate_population of one population three times through "
                        "the host API (the first call builds what the default policy needs: with the lazy index "
                        "only the population's own pair vectors)"}
    finally:
        ev.close()


# ---------------------------------------------------------------------------
# config 5: the fitness-kernel microbench sweep (BASELINE configs[4])
# ---------------------------------------------------------------------------
SWEEP_L = [2, 3, 4, 5, 8, 12, 16, 24, 32, 50]
SWEEP_R = [1_000, 4_000, 16_000, 64_000, 256_000, 1_000_000]
SWEEP_APPROX = [0.0, 0.03]
SWEEP_COLS = 64


def measured_l2():
    p = REPO / "profiles" / "measured_l2.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["l2_gbs"]), "measured (profiles/measured_l2.json, scripts/microbench/l2_bw.cu)"
        except Exception:
            pass
    return None, None


def bench_sweep(args):
    """One JSON line per (R, approx, L): the index count kernel on an N(0,1)
    background of R x 64 (datagen.cpp:64-70 shape, float32), exactly-L random
    distinct columns, P = ceil(1 GiB / (4 L R)) candidates (>= 1 GiB of
    algorithmic bytes per launch), full pair-trend index.  The fraction is
    against the L2 read roofline when the whole index fits in L2 (every launch
    touches nearly all 64 x 63 pairs), else against HBM."""
    import torch

    from paper_2105_01196_b200 import Evaluator, TrendParams, synth

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    hbm, hbm_src = measured_peak()
    l2, l2_src = measured_l2()
    ev = Evaluator(0)
    stream = torch.cuda.Stream(dev)
    Ls = [int(x) for x in args.sweep_l.split(",")] if args.sweep_l else SWEEP_L
    Rs = [int(x) for x in args.sweep_r.split(",")] if args.sweep_r else SWEEP_R
    for R in Rs:
        rng = np.random.default_rng(7)
        m = rng.standard_normal((R, SWEEP_COLS), dtype=np.float32)
        ev.upload(m)
        for approx in SWEEP_APPROX:
            ev.prepare(approx)
            index_bytes, used = ev.index_info()
            wp = index_bytes // (4 * SWEEP_COLS ** 2)
            tp = TrendParams(approx=approx)
            for L in Ls:
                if args.sweep_sizing == "algorithmic":  # 4 L R P >= 1 GiB
                    P = min(2_000_000, -(-(1 << 30) // (4 * L * R)))
                else:  # >= 512 MB of pair vectors per launch: a throughput, not a launch-latency, measurement
                    P = min(2_000_000, -(-(512 << 20) // (4 * wp * (L - 1))))
                pops = [synth.exact_len_population(P, SWEEP_COLS, L, seed=1000 * L + k) for k in range(2)]
                d = [(torch.from_numpy(pp.cols.view(np.int32)).to(dev), torch.from_numpy(pp.offsets.view(np.int32)).to(dev))
                     for pp in pops]
                out = torch.empty(P, dtype=torch.int32, device=dev)
                ev.set_stream(stream.cuda_stream)
                for i in range(3):
                    ev.evaluate_population_device(d[i % 2][0].data_ptr(), d[i % 2][1].data_ptr(), P, out.data_ptr(), tp,
                                                  stream=stream.cuda_stream)
                ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
                ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
                torch.cuda.synchronize()
                for i in range(args.steps):
                    ev0[i].record(stream)
                    ev.evaluate_population_device(d[i % 2][0].data_ptr(), d[i % 2][1].data_ptr(), P, out.data_ptr(), tp,
                                                  stream=stream.cuda_stream)
                    ev1[i].record(stream)
                torch.cuda.synchronize()
                ev.sync()
                ev.set_stream(None)
                ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev0, ev1))
                reads = 4.0 * wp * P * (L - 1)
                alg = 4.0 * L * R * P
                # L2 roofline while the whole index is at most 2x the L2 (the
                # main bench's stream/flush rule): a 132-MB index (256k rows)
                # is mostly served from L2 and measures above the HBM peak.
                # Against L2 every read counts; against HBM the distinct
                # vectors a launch must bring in (64 columns: 4096 pairs in all,
                # so big populations repeat them and the repeats hit L2)
                regime = "l2" if (l2 is not None and index_bytes <= 2 * L2_BYTES) else "hbm"
                phys = reads if regime == "l2" else 4.0 * wp * statistics.mean(
                    distinct_pairs(pp, SWEEP_COLS, False) for pp in pops)
                peak = l2 if regime == "l2" else hbm
                line = {"sweep": "c5", "sizing": args.sweep_sizing, "rows": R, "cols": SWEEP_COLS, "L": L,
                        "approx": approx, "population": P,
                        "kernel": index_kernel_name(wp, P), "kernel_ms": ms, "evals_per_s": P / (ms / 1e3),
                        "row_checks_per_s": P * R / (ms / 1e3), "index_bytes": index_bytes, "wp": int(wp),
                        "physical_bytes": phys, "physical_gbs": phys / (ms / 1e3) / 1e9, "regime": regime,
                        "reads_gbs": reads / (ms / 1e3) / 1e9,
                        "peak_gbs": peak, "peak_source": l2_src if regime == "l2" else hbm_src,
                        "frac": phys / (ms / 1e3) / 1e9 / peak,
                        "effective_algorithmic_gbs": alg / (ms / 1e3) / 1e9}
                print(json.dumps(line), flush=True)
                del d, out
    ev.close()
    return 0


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int:
    """--gpus N without torchrun: re-launch this script with N ranks, one per GPU."""
    import torch

    n_dev = torch.cuda.device_count()
    if n_dev < args.gpus and not args.share_gpu:
        log(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n_dev} "
            f"(--share-gpu runs the ranks on fewer GPUs, for testing only)")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd, cwd=str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--shard", choices=["rows", "pop", "replica"], default=None,
                    help="N > 1: rows (default; BASELINE config 3: row-sharded strong scaling with the pipelined "
                         "peer-memory exchange), pop (population split + all_gather) or replica (independent "
                         "populations, no collective; weak scaling)")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="rows mode: sum the partial counts over peer memory (default) or with an NCCL all_reduce")
    ap.add_argument("--l2", choices=["auto", "stream", "flush"], default="auto")
    ap.add_argument("--pops", type=int, default=0, help="populations cycled (0 = enough to exceed 2x L2)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default=None,
                    help="process-group backend for N > 1 (default nccl; gloo with --share-gpu)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="allow N ranks on fewer than N GPUs (tests the sharded path on a 1-GPU box; not scaling data)")
    ap.add_argument("--index-budget-gb", type=float, default=None,
                    help="pair-trend index budget (default: the library's, 40%% of free HBM)")
    ap.add_argument("--path", choices=["auto", "value", "plane", "table"], default="auto",
                    help="evaluation kernel: rank-plane slab kernel (auto for <= 8192 cols) or float value kernel")
    ap.add_argument("--sweep", action="store_true",
                    help="config 5: one JSON line per (rows, approx, L) point of the fitness-kernel microbench sweep")
    ap.add_argument("--sweep-l", default="", help="comma-separated L values (default: the BASELINE sweep)")
    ap.add_argument("--sweep-r", default="", help="comma-separated row counts (default: the BASELINE sweep)")
    ap.add_argument("--sweep-sizing", choices=["physical", "algorithmic"], default="physical",
                    help="population per point: >= 512 MB of pair vectors per launch (default), or SURVEY 8(d)'s "
                         ">= 1 GiB of algorithmic bytes (4 L R P), which the index compresses ~32x into 10-30 us launches")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.sweep:
        return bench_sweep(args)
    env_world = os.environ.get("WORLD_SIZE")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.shard is None:
        args.shard = "rows" if args.gpus > 1 else "none"

    if args.impl == "reference":
        return bench_reference(args, cfg, rank)

    if env_world is None and args.gpus > 1:
        return self_launch(args)
    world = int(env_world or "1")
    if world != args.gpus:
        log(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
        return 2
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        n_dev = torch.cuda.device_count()
        if n_dev < world and not args.share_gpu:
            log(f"bench.py: {world} ranks need {world} visible GPUs, found {n_dev}")
            return 2
        dev_idx = local_rank % max(n_dev, 1)
        torch.cuda.set_device(dev_idx)
        backend = args.backend or ("gloo" if n_dev < world else "nccl")
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            tdist.init_process_group("gloo")
        dist = tdist
    try:
        return bench_ours(args, cfg, rank, world, local_rank, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
