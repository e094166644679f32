"""Benchmark of the hot path (BASELINE.json: pairwise distances/sec and
achieved HBM GB/s per metric; kNN queries/sec).

Default workload (BASELINE configs[1], what the driver runs): cosine pairwise
distances of 10,000 query rows against the full MovieLens-25M-shaped
power-law index (162,541 x 59,047, ~154 nnz/row), fp32, synthetic data from
the reference's generator.  One step = the full 10,000 x 162,541 distance
matrix.  The same line carries the workload's other metrics (`per_metric`:
euclidean, manhattan), float64 lines (`per_metric_f64`), the dominant kernel's
roofline, the CPU reference baseline and GPU-vs-oracle agreement.  Other
BASELINE configs: --workload c1 | c3 | c4 | c5 (c5 = kNN).

Timing: W warm-up steps, then K steps between barrier + synchronize, CUDA
events on the launching stream, max over ranks.  Inputs and outputs exceed
the 126 MB L2 (C1 excepted, stated in `config`).

Multi-GPU: `--gpus N` launches N ranks itself (torch.distributed.run, NCCL)
when not already under torchrun, and fails loudly if the node has fewer GPUs.
Pairwise distances partition by query rows with the index replicated and no
collective, so they scale WEAK by default: every rank its own
batch of the workload's queries (seed 26 + rank), value = all ranks'
distances / the max-over-ranks step time.  `--scaling strong` splits the
fixed query set across ranks by work instead (DESIGN.md §6 has the per-rank
cost model: the hybrid path's index-sized costs do not shrink with the
rank's share).  kNN shards the index rows (fixed total work) and merges the
per-rank top-k with one NCCL all-gather.

--impl reference: the reference's CPU algorithm (the oracle's numpy port,
bitwise equal to the reference) on the host cores, bounded query sample.
"""

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    "c1": dict(desc="BASELINE configs[0]: 1k x 1k rows, 10k cols, 1% uniform density", ref_queries=1000,
               index=dict(n_rows=1000, n_cols=10000, degree_dist="uniform", degree=100, seed=2),
               queries=dict(n_rows=1000, n_cols=10000, degree_dist="uniform", degree=100, seed=1),
               metrics=["manhattan", "cosine"], n_queries=1000, kind="pairwise"),
    "c2": dict(desc="BASELINE configs[1]: MovieLens-25M-shaped power-law index 162,541 x 59,047, ~154 nnz/row",
               index=dict(n_rows=162541, n_cols=59047, degree_dist="zipf", zipf_s=1.544, zipf_max_degree=32000,
                          seed=25),
               metrics=["cosine", "euclidean", "manhattan"], f64_metrics=["cosine", "manhattan"],
               n_queries=10000, kind="pairwise"),
    "c3": dict(desc="BASELINE configs[2]: NYTimes-BoW-shaped index 300,000 x 102,660, ~232 nnz/row, tf-idf values",
               index=dict(n_rows=300000, n_cols=102660, degree_dist="zipf", zipf_s=1.309, zipf_max_degree=2000,
                          value_dist="tfidf", seed=3),
               metrics=["canberra", "chebyshev", "jensenshannon", "kl"], n_queries=4096, kind="pairwise"),
    "c4": dict(desc="BASELINE configs[3]: scRNA-shaped index 65,000 x 26,000, degrees lognormal in [501, 9600] "
                    "(mean ~1.8k, ~7% dense)",
               index=dict(n_rows=65000, n_cols=26000, degree_dist="lognormal", lognormal_mu=7.38,
                          lognormal_sigma=0.55, min_degree=501, max_degree=9600, value_dist="tfidf", seed=4),
               metrics=["hellinger", "jaccard"], n_queries=2048, kind="pairwise"),
    "c5": dict(desc="BASELINE configs[4]: brute-force kNN k=32 cosine, 1,000,000 x 100,000 power-law index "
                    "(~154 nnz/row)",
               index=dict(n_rows=1000000, n_cols=100000, degree_dist="zipf", zipf_s=1.50, zipf_max_degree=10000,
                          seed=5),
               metrics=["cosine"], n_queries=10000, kind="knn", k=32),
}
BINARY_METRICS = ("jaccard", "dice", "russelrao", "hamming")
DOT_FAMILY = ("cosine", "euclidean", "correlation", "dot", "dice", "jaccard", "hellinger", "russelrao")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ data

def make_index(wl):
    import paper_2104_06357_b200 as sd
    return sd.round_values_f32(sd.generate(sd.GenSpec(**wl["index"])))


def make_queries(wl, index, n_queries, seed=26):
    """The workload's query rows: its own matrix (C1) or index rows sampled
    without replacement (values already rounded to fp32 with the index)."""
    import paper_2104_06357_b200 as sd
    if "queries" in wl:
        return sd.round_values_f32(sd.generate(sd.GenSpec(**wl["queries"])))
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(index.n_rows, min(n_queries, index.n_rows), replace=False))
    return gather_rows(index, rows)


def binary(m):
    """Same pattern with values 1 (set-semantics metrics, BINARY_PREFERRED metrics.py:37)."""
    return m.with_values(np.ones(len(m.values)))


def gather_rows(m, rows):
    import paper_2104_06357_b200 as sd
    ptr = np.asarray(m.indptr)
    rows = np.asarray(rows)
    deg = ptr[rows + 1] - ptr[rows]
    newptr = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(deg, out=newptr[1:])
    starts = np.repeat(ptr[rows], deg)
    take = starts + (np.arange(newptr[-1]) - np.repeat(newptr[:-1], deg))
    return sd.CsrMatrix(len(rows), m.n_cols, newptr, np.asarray(m.indices)[take], np.asarray(m.values)[take])


_BINARY = {}


def operands_for(metric, index, queries):
    """The matrices a metric runs on (binary pattern for the set metrics), the
    same objects on every call so their device copies and index are cached."""
    if metric not in BINARY_METRICS:
        return index, queries
    for m in (index, queries):
        if id(m) not in _BINARY:
            _BINARY[id(m)] = (m, binary(m))
    return _BINARY[id(index)][1], _BINARY[id(queries)][1]


# ------------------------------------------------------------------ host / clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() in ("active", "1", "yes"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def host_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    aff = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": aff, "numpy": np.__version__,
            "python": platform.python_version(), "host": socket.gethostname()}


def load_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_tensor_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured (MEASURED_PEAKS.json bf16_tflops, burst cuBLAS)"
    except (OSError, KeyError, ValueError):
        return 1590.0, "fallback (B200_PROFILING.md)"


def load_traffic(workload, metric, dtype):
    """Per-launch DRAM bytes of the sweep kernel from the committed ncu capture
    of the same workload / metric / dtype (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(f"{workload}/{metric}/{dtype}")
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------ CPU reference (oracle port)

def _oracle_run(index, queries, metric, q, workers, k=None):
    from oracle import semidist_oracle as O
    oq = O.Csr.of(queries).slice(0, q)
    if k is not None:
        return O.kneighbors(O.Csr.of(index), oq, k, metric, workers=workers, batch_rows=q)
    return O.pairwise_distances(oq, O.Csr.of(index), metric, strict=metric != "kl", workers=workers)


def cpu_reference_rate(index, queries, metric, sample, budget_s=15.0, k=None):
    """The reference algorithm (oracle numpy port, bitwise = reference) on a
    query sample against the FULL index.  Worker count: best of a sweep over
    {1, 2, 4, ..., cores} on a calibration slice (the first 20,000 index rows,
    1 query) — engine.py:102-107's `workers` knob, SURVEY §8(d).  Returns a
    dict with units/s and what was run."""
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    import paper_2104_06357_b200 as sd
    calib = sd.slice_rows(index, 0, min(index.n_rows, 20000))
    sweep, w = {}, 1
    while True:
        t0 = time.perf_counter()
        _oracle_run(calib, queries, metric, 1, w, k=min(k, calib.n_rows) if k else None)
        sweep[w] = time.perf_counter() - t0
        if w >= cores:
            break
        w = min(cores, w * 2)
    best = min(sweep, key=sweep.get)
    # a small run, then one sized to the budget (two-pass metrics have a
    # per-call cost in the index size whatever the query count)
    q = int(min(2, sample, queries.n_rows))
    t0 = time.perf_counter()
    res = _oracle_run(index, queries, metric, q, best, k)
    dt = time.perf_counter() - t0
    if dt < budget_s / 3 and q < min(sample, queries.n_rows):
        q = int(max(q + 1, min(sample, queries.n_rows, q * budget_s / max(dt, 1e-3) / 2)))
        t0 = time.perf_counter()
        res = _oracle_run(index, queries, metric, q, best, k)
        dt = time.perf_counter() - t0
    units = q if k is not None else q * index.n_rows
    return {"value": units / dt, "q": q, "cores": best, "seconds": dt, "result": res,
            "worker_sweep_s": {str(a): round(b, 3) for a, b in sweep.items()}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    metric = args.metric or wl["metrics"][0]
    index = make_index(wl)
    queries = make_queries(wl, index, max(256, wl.get("ref_queries", 0)))
    index, queries = operands_for(metric, index, queries)
    k = wl.get("k") if wl["kind"] == "knn" else None
    rates, ref = [], None
    for step in range(args.warmup + args.steps):
        ref = cpu_reference_rate(index, queries, metric, sample=wl.get("ref_queries", args.ref_queries),
                                 budget_s=args.ref_budget, k=k)
        if step >= args.warmup:
            rates.append(ref["value"])
    value = statistics.median(rates)
    unit = "queries/s" if k else "distances/s"
    sample = f"{ref['q']} queries x {index.n_rows} index rows per step (oracle numpy port, fp64)"
    line = {
        "metric": "kNN queries/sec" if k else "pairwise distances/sec", "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": (ref["q"] if k else ref["q"] * index.n_rows) / value * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if (wl["kind"] == "knn" or args.scaling == "strong") else "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference generator, values rounded to fp32)", "impl": "reference",
        "config": {"workload": f"{args.workload}: {metric}, {ref['q']}-query sample vs the full index; {wl['desc']}",
                   "metric": metric, "index_rows": index.n_rows, "n_cols": index.n_cols, "index_nnz": index.nnz},
        "cpu_baseline": {"value": value, "unit": unit, "cores": ref["cores"], "kind": "port", "sample": sample,
                         "worker_sweep_s": ref["worker_sweep_s"], **host_info()},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def self_launch(args):
    """Run this script under torch.distributed.run with N ranks (one per GPU)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}")
        print(json.dumps({"error": f"--gpus {args.gpus} requested, {have} GPU(s) visible", "n_gpus": args.gpus}))
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def compulsory_bytes(m_rows, n, es, dq_nnz, m_all, di, ix, n_cols, knn_k=0):
    """DESIGN.md §4.1 byte model of one sweep launch: its output written once
    (m_rows x n distances, or the k-lists for kNN) + query CSR + index postings
    + (tile, column) pointers + per-row statistics read once."""
    post_b = 8 if es == 4 else 16
    n_tiles = -(-n // ix.tile_rows)
    inputs = dq_nnz * (4 + es) + (m_all + 1) * 8 + di.nnz * post_b + 4 * (n_tiles * n_cols + 1) + (m_all + n) * es
    out = m_all * knn_k * (es + 8) if knn_k else m_rows * n * es
    return out + inputs


def run_ours(args):
    import ctypes

    import torch
    import torch.distributed as dist

    import paper_2104_06357_b200 as sd
    from paper_2104_06357_b200 import _lib
    from paper_2104_06357_b200.distributed import gather_candidates, merge_candidates, shard_bounds

    wl = WORKLOADS[args.workload]
    knn = wl["kind"] == "knn"
    metrics = [args.metric] if args.metric else list(wl["metrics"])
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    t_setup = time.perf_counter()
    n_queries = args.queries or wl["n_queries"]
    index = make_index(wl)
    strong = args.scaling == "strong"
    if knn or strong:
        queries_all = make_queries(wl, index, n_queries)
    else:   # weak: every rank its own batch of n_queries
        queries_all = make_queries(wl, index, n_queries, seed=26 + rank)
    index_full_rows = index.n_rows
    shard_lo, q_lo, q_hi = 0, 0, queries_all.n_rows
    if knn and world > 1:   # index rows sharded across ranks, queries replicated
        shard_lo, shard_hi = shard_bounds(index.n_rows, world)[rank]
        index = sd.slice_rows(index, shard_lo, shard_hi)
    if not knn and strong and world > 1:   # query rows sharded by work, index replicated
        w = np.diff(np.asarray(queries_all.indptr)).astype(np.float64) + 16.0
        q_lo, q_hi = shard_bounds(queries_all.n_rows, world, weights=w)[rank]
    queries = sd.slice_rows(queries_all, q_lo, q_hi) if (q_lo, q_hi) != (0, queries_all.n_rows) else queries_all
    log(f"[rank {rank}] {args.workload}: index {index.n_rows}x{index.n_cols} nnz={index.nnz} "
        f"(mean deg {index.nnz / max(1, index.n_rows):.1f}); queries {queries.n_rows} nnz={queries.nnz} "
        f"({time.perf_counter() - t_setup:.1f}s)")
    m, n = queries.n_rows, index.n_rows
    k = wl.get("k", 0)
    stream = torch.cuda.current_stream(dev)
    sh = ctypes.c_void_p(stream.cuda_stream)
    strat = _lib.strategy_struct(_lib.STRAT_AUTO)
    rep = _lib.SdReport()
    flags = _lib.new_flags(dev)
    ldo = (n + 3) // 4 * 4   # 16-byte aligned rows: the epilogue stores 4 cells per lane
    bufs = {}
    operands = {}

    def out_buf(tdt):
        key = ("out", tdt)
        if key not in bufs:
            bufs[key] = (torch.empty((m, k), dtype=tdt, device=dev), torch.empty((m, k), dtype=torch.int64, device=dev)) \
                if knn else torch.empty((m, ldo), dtype=tdt, device=dev)
        return bufs[key]

    def prepare(metric, tdt):
        key = (metric, tdt)
        if key in operands:
            return operands[key]
        idx_m, q_m = operands_for(metric, index, queries)
        transform = "sqrt" if metric == "hellinger" else None
        t0 = time.perf_counter()
        di = sd.to_device(idx_m, tdt, dev, transform=transform)
        dq = sd.to_device(q_m, tdt, dev, transform=transform)
        ix = _lib.device_index(di)
        torch.cuda.synchronize()
        operands[key] = (di, dq, ix, _lib.metric_struct(metric, None, metric != "kl", transform is not None),
                         time.perf_counter() - t0)
        return operands[key]

    def step(metric, tdt, phases=None):
        di, dq, ix, md, _ = prepare(metric, tdt)
        ca, cb = _lib.csr_struct(dq), _lib.csr_struct(di)
        if knn:
            od, oi = out_buf(tdt)
            _lib.check(lib.sd_knn(ctypes.byref(ca), ctypes.byref(cb), ix.handle, _lib.dtype_code(tdt),
                                  ctypes.byref(md), k, shard_lo, od.data_ptr(), oi.data_ptr(), flags.data_ptr(), sh),
                       "sd_knn")
            if world > 1:
                cd, ci = gather_candidates(od, oi)
                merge_candidates(cd, ci, k)
        elif m > 0:
            _lib.check(lib.sd_pairwise(ctypes.byref(ca), ctypes.byref(cb), ix.handle, _lib.dtype_code(tdt),
                                       ctypes.byref(md), ctypes.byref(strat), out_buf(tdt).data_ptr(), ldo,
                                       flags.data_ptr(), ctypes.byref(rep), phases, sh), "sd_pairwise")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world > 1:
            t = torch.tensor([x], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        return x

    def timed(metric, tdt, steps, warmup):
        for _ in range(warmup):
            step(metric, tdt)
        barrier()
        l0 = lib.sd_launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            step(metric, tdt)
        e1.record(stream)
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / steps), lib.sd_launch_count() - l0

    # units per step over ALL ranks: queries answered (kNN) / distances
    def units_all():
        if knn:
            return queries_all.n_rows
        return (queries_all.n_rows if strong else queries_all.n_rows * world) * index_full_rows

    head = metrics[0]
    tdt0 = torch.float32 if args.dtype == "float32" else torch.float64
    es0 = 4 if tdt0 == torch.float32 else 8
    prepare(head, tdt0)
    # ---------------- headline: K timed steps of the workload's first metric
    clocks = ClockSampler(local)
    for _ in range(args.warmup):
        step(head, tdt0)
    barrier()
    clocks.start()
    ms, launches = timed(head, tdt0, args.steps, 0)
    clk = clocks.stop()
    value = units_all() / (ms / 1e3)
    assert int(flags.item()) == 0 or head == "kl", "domain flag raised during benchmark"

    # ---------------- roofline of the dominant kernel
    def roofline_of(metric, tdt, step_ms):
        es = 4 if tdt == torch.float32 else 8
        di, dq, ix, _, _ = prepare(metric, tdt)
        peak, peak_kind = load_peak()
        traffic = load_traffic(args.workload, metric, "f32" if es == 4 else "f64")
        if knn or m == 0:
            alg = compulsory_bytes(0, n, es, dq.nnz, m, di, ix, index.n_cols, knn_k=k)
            achieved = alg / (step_ms / 1e3) / 1e9
            return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                    "kernel": f"sd_knn: isect_kernel<{'float' if es == 4 else 'double'}, {metric}, top-k> + merge",
                    "kernel_ms": step_ms, "alg_bytes_per_launch": alg, "peak_source": peak_kind,
                    "note": "intersection-bound, not HBM-bound: the sweep reads L2-resident postings; "
                            "bytes = query CSR + postings + pointers + statistics + the k-lists"}
        phases = (ctypes.c_float * 4)()
        kern_ms = []
        for _ in range(max(3, min(args.steps, 10))):
            step(metric, tdt, phases)
            kern_ms.append(phases[1])
        kern = statistics.median(kern_ms)
        if "dense" in ix.hybrid_blocks:
            # dense-index mode (dense_tc.cu): one tcgen05 bf16 GEMM; tensor-bound.
            # FLOPs executed = 2 m n K' x the MMAs per K step (hi*hi [+ hi*lo]
            # [+ lo*hi]), K' = n_cols rounded to 64; `kernel_ms` includes the
            # query image build (phase pass1)
            qv = np.asarray(operands_for(metric, index, queries)[1].values, dtype=np.float32)
            pb = 1 if not (qv.view(np.uint32) & 0xFFFF).any() else 2
            pa = 2 if "dense_two_planes" in ix.hybrid_blocks else 1
            terms = 1 + (pb == 2) + (pa == 2)
            kp = -(-index.n_cols // 64) * 64
            flops = 2.0 * m * n * kp * terms
            tpeak, tpeak_kind = load_tensor_peak()
            achieved = flops / (kern / 1e3) / 1e12
            path_bytes = compulsory_bytes(m, n, es, dq.nnz, m, di, ix, index.n_cols)
            return {"bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s",
                    "frac": achieved / tpeak, "traffic": None,
                    "kernel": f"dense_tc_kernel<{metric}> (bf16 {'hi/lo ' if terms > 1 else ''}x{terms})",
                    "kernel_ms": kern, "flops_per_launch": flops, "mma_terms": terms, "peak_source": tpeak_kind,
                    "path": {"what": "whole timed step, HBM view: output + operands", "ms": step_ms,
                             "alg_bytes": path_bytes, "achieved": path_bytes / (step_ms / 1e3) / 1e9,
                             "frac": path_bytes / (step_ms / 1e3) / 1e9 / peak}}
        # query rows the dense heavy-row path serves instead of the sweep
        deg = np.diff(np.asarray(queries.indptr))
        theta = max(64, (index.n_cols + 31) // 32)
        n_tiles = -(-n // ix.tile_rows)
        blocks = ix.hybrid_blocks
        hybrid = ("dot" in blocks and metric in DOT_FAMILY) or ("minsum" in blocks and metric == "manhattan")
        heavy_q = min(1024, int((deg >= theta).sum())) if ix.heavy_rows > 0 and n_tiles >= 4 and hybrid else 0
        alg = compulsory_bytes(m - heavy_q, n, es, dq.nnz, m, di, ix, index.n_cols)
        achieved = alg / (kern / 1e3) / 1e9
        path_bytes = compulsory_bytes(m, n, es, dq.nnz, m, di, ix, index.n_cols)
        alg3 = m * di.nnz * (8 + es) + m * n * es   # every query streams all of B
        return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                "traffic_source": (traffic or {}).get("source"),
                "kernel": f"isect_kernel<{'float' if es == 4 else 'double'}, {metric}>", "kernel_ms": kern,
                "alg_bytes_per_launch": alg, "rows_swept": m - heavy_q, "peak_source": peak_kind,
                "alg3_stream_equiv_gbs": alg3 / (kern / 1e3) / 1e9,
                "path": {"what": "whole timed step (statistics + dense heavy-row path + sweep + heavy epilogue), "
                                 "all output rows",
                         "ms": step_ms, "alg_bytes": path_bytes, "achieved": path_bytes / (step_ms / 1e3) / 1e9,
                         "frac": path_bytes / (step_ms / 1e3) / 1e9 / peak}}

    roofline = roofline_of(head, tdt0, ms)

    # ---------------- the workload's other metrics, and float64 lines
    per_metric = {head: {"value": value, "ms_per_step": ms, "frac": roofline["frac"],
                         "path_frac": roofline.get("path", {}).get("frac")}}
    per_metric_f64 = {}
    if not args.no_extra:
        for metric in metrics[1:]:
            ms_x, _ = timed(metric, tdt0, max(3, args.steps // 2), 1)
            rl = roofline_of(metric, tdt0, ms_x)
            per_metric[metric] = {"value": units_all() / (ms_x / 1e3), "ms_per_step": ms_x, "frac": rl["frac"],
                                  "path_frac": rl.get("path", {}).get("frac"), "kernel_ms": rl["kernel_ms"]}
        if tdt0 == torch.float32:
            for metric in wl.get("f64_metrics", []):
                ms_x, _ = timed(metric, torch.float64, max(3, args.steps // 2), 1)
                rl = roofline_of(metric, torch.float64, ms_x)
                per_metric_f64[metric] = {"value": units_all() / (ms_x / 1e3), "ms_per_step": ms_x,
                                          "frac": rl["frac"], "path_frac": rl.get("path", {}).get("frac"),
                                          "kernel_ms": rl["kernel_ms"]}

    # ---------------- e2e: public API, host in / host out, pinned buffers
    di, dq, ix, md, build_s = prepare(head, tdt0)
    qh = operands_for(head, index, queries)[1]
    hp = torch.from_numpy(np.asarray(qh.indptr, dtype=np.int64)).pin_memory()
    hi = torch.from_numpy(np.asarray(qh.indices, dtype=np.int32)).pin_memory()
    hv = torch.from_numpy(np.asarray(qh.values)).to(tdt0).pin_memory()
    spec = sd.metric_registry(head, strict=head != "kl")
    h2d = hp.numel() * 8 + hi.numel() * 4 + hv.numel() * es0
    if knn:
        host_d = torch.empty((m, k), dtype=tdt0, pin_memory=True)
        host_i = torch.empty((m, k), dtype=torch.int64, pin_memory=True)
        d2h = m * k * (es0 + 8)
    else:
        host_out = torch.empty((m, n), dtype=tdt0, pin_memory=True)
        d2h = m * n * es0
    index_host = operands_for(head, index, queries)[0]

    def e2e_step(index_obj):
        q = sd.upload(m, queries.n_cols, hp, hi, hv, device=dev)
        if knn:
            from paper_2104_06357_b200.knn import knn_device
            d, i_, _ = knn_device(index_obj, q, k, spec, dtype=tdt0, index_base=shard_lo)
            if world > 1:
                cd, ci = gather_candidates(d, i_)
                d, i_ = merge_candidates(cd, ci, k)
            host_d.copy_(d, non_blocking=True)
            host_i.copy_(i_, non_blocking=True)
            torch.cuda.current_stream(dev).synchronize()
        elif m > 0:
            sd.pairwise_distances(q, index_obj, spec, dtype=tdt0, out=host_out)

    e2e_step(index_host)
    barrier()
    t0 = time.perf_counter()
    e_steps = max(2, min(args.steps, 5))
    for _ in range(e_steps):
        e2e_step(index_host)
    barrier()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / e_steps)
    # cold: a fresh index object — its upload and sd_index_build inside the timed call
    import paper_2104_06357_b200.sparse as sp
    cold_index = sp.CsrMatrix(index_host.n_rows, index_host.n_cols, index_host.indptr, index_host.indices,
                              index_host.values)
    barrier()
    t0 = time.perf_counter()
    e2e_step(cold_index)
    barrier()
    cold_ms = max_over_ranks((time.perf_counter() - t0) * 1e3)
    cold_index_bytes = index_host.nnz * (4 + es0) + (index_host.n_rows + 1) * 8
    del cold_index
    e2e = {"value": units_all() / (e2e_ms / 1e3), "unit": "queries/s" if knn else "distances/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
           "path": ("sd.upload(pinned CSR) -> fused kNN (+ all-gather merge) -> pinned host (dist, idx)" if knn else
                    "sd.upload(pinned CSR) -> sd.pairwise_distances(..., out=pinned host buffer)"),
           "cold": {"ms": cold_ms, "value": units_all() / (cold_ms / 1e3),
                    "h2d_bytes": h2d + cold_index_bytes,
                    "what": "first call on a new index matrix: index upload + sd_index_build + the step"}}

    # ---------------- CPU baseline (rank 0, N=1) and GPU-vs-oracle agreement
    cpu, agreement = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        idx_h, q_h = operands_for(head, index, queries)
        ref = cpu_reference_rate(idx_h, q_h, head, sample=wl.get("ref_queries", args.ref_queries),
                                 budget_s=args.ref_budget, k=k if knn else None)
        cpu = {"value": ref["value"], "unit": "queries/s" if knn else "distances/s", "cores": ref["cores"],
               "kind": "port", "sample": f"{ref['q']} queries x {index.n_rows} index rows "
                                         f"({ref['seconds']:.1f}s, oracle numpy port, fp64)",
               "worker_sweep_s": ref["worker_sweep_s"], **host_info()}
    if rank == 0 and world == 1 and not args.no_check:
        agreement = check_agreement(args.workload, head, index, queries, tdt0, step, out_buf, knn, k, m, n)

    if rank == 0:
        line = {
            "metric": "kNN queries/sec" if knn else "pairwise distances/sec", "value": value,
            "unit": "queries/s" if knn else "distances/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if (knn or strong) else "weak", "vs_baseline": None,
            "dtype": "f32" if tdt0 == torch.float32 else "f64",
            "data": "synthetic (reference generator, values rounded to fp32)",
            "config": {"workload": f"{args.workload}: {head}, {queries_all.n_rows} query rows vs the full "
                                   f"{index_full_rows} x {index.n_cols} index "
                                   f"({'k=%d, index rows sharded' % k if knn else 'query rows sharded by work' if strong else 'a query batch per rank'}"
                                   f" over {world} GPU(s)); {wl['desc']}",
                       "metric": head, "queries": queries_all.n_rows, "index_rows": index_full_rows,
                       "n_cols": index.n_cols, "index_nnz_per_rank": index.nnz, "query_nnz": queries_all.nnz,
                       "parallelism": (f"index-row shards x{world}" if knn else f"query-row shards x{world}"),
                       "l2": ("inputs + outputs exceed the 126 MB L2 (no flush needed)" if args.workload != "c1" else
                              "C1 is L2-resident (6 MB inputs, 4 MB output); timed back to back"),
                       "index_build": f"once, outside the timed region ({build_s:.3f}s incl. upload; "
                                      f"e2e.cold times it inside)",
                       "index_bytes": ix.bytes},
            "roofline": roofline, "cpu_baseline": cpu, "agreement": agreement, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk, "per_metric": per_metric,
        }
        if per_metric_f64:
            line["per_metric_f64"] = per_metric_f64
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def check_agreement(workload, metric, index, queries, tdt, step, out_buf, knn, k, m, n, sample=16):
    """GPU rows of the timed run for the first `sample` queries vs the C
    restatement of the reference (oracle/), judged by the parity rule of
    tests/parity.py (BASELINE rtol, conditioning-based magnitudes)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import semidist_oracle as O
    from parity import check_cells
    idx_h, q_h = operands_for(metric, index, queries)
    qs = O.Csr.of(q_h).slice(0, min(sample, m))
    dt = np.float32 if tdt == torch.float32 else np.float64
    t0 = time.perf_counter()
    step(metric, tdt)
    torch.cuda.synchronize()
    if knn:
        od, oi = out_buf(tdt)
        ref_d, ref_i, full = O.kneighbors_c(idx_h, qs, k, metric)
        got_i = oi[:qs.n_rows].cpu().numpy()
        same = got_i == ref_i
        tol = 1e-5 if dt == np.float32 else 1e-11
        alt = np.take_along_axis(full, got_i, axis=1)
        ties = np.abs(alt - ref_d) <= tol * (1 + np.abs(ref_d))
        return {"gpu_topk_index_agreement": float(same.mean()), "mismatches_outside_ties": int((~same & ~ties).sum()),
                "queries": qs.n_rows, "checker": "oracle/semidist_oracle.c (C restatement), stable argsort",
                "seconds": round(time.perf_counter() - t0, 2)}
    got = out_buf(tdt)[:qs.n_rows, :n].double().cpu().numpy()
    ref = O.pairwise_distances_c(qs, idx_h, metric, strict=metric != "kl")
    sat = ref >= 1e308
    ok = check_cells(got, np.where(sat, 0.0, ref), qs, idx_h, metric, dt) | sat
    ok &= sat == (got >= (1e308 if dt == np.float64 else np.inf))
    return {"gpu_rows_vs_port_max_abs_err": float(np.max(np.abs(np.where(sat, 0.0, got - ref)))),
            "parity_rule_cells_failed": int((~ok).sum()), "cells": int(ok.size), "queries": qs.n_rows,
            "checker": "oracle/semidist_oracle.c (C restatement), rule tests/parity.py",
            "seconds": round(time.perf_counter() - t0, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--metric", default=None, help="override the workload's headline metric")
    ap.add_argument("--dtype", choices=["float32", "float64"], default="float32")
    ap.add_argument("--queries", type=int, default=0)
    ap.add_argument("--scaling", choices=["strong", "weak"], default="weak",
                    help="pairwise multi-GPU: a query batch per rank (weak, default) or the fixed set split (strong)")
    ap.add_argument("--ref-queries", type=int, default=64)
    ap.add_argument("--ref-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the GPU-vs-oracle agreement check")
    ap.add_argument("--no-extra", action="store_true", help="skip the workload's secondary metrics")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        log(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
