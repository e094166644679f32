"""Per-launch device timeline of one pairwise step (CUPTI via torch.profiler):
start/end of every kernel and copy on every stream, relative to the step's
first GPU activity — the critical path that ncu's serialised launch list
cannot show.

    python tools/timeline.py --workload c2 --metric cosine [--dtype float32] [--steps 3]

Prints the last profiled step (earlier ones are warm-up).  Not a bench
number: the profiler adds a little launch overhead.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--metric", default="cosine")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--queries", type=int, default=0, help="query rows (default: the workload's)")
    ap.add_argument("--api", type=float, default=0.0,
                    help="also list CUDA runtime calls on the host longer than this many us")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_2104_06357_b200 as sd
    from paper_2104_06357_b200 import _lib

    wl = bench.WORKLOADS[args.workload]
    index = bench.make_index(wl)
    queries = bench.make_queries(wl, index, args.queries or wl["n_queries"])
    idx_m, q_m = bench.operands_for(args.metric, index, queries)
    tdt = torch.float32 if args.dtype == "float32" else torch.float64
    dev = torch.device("cuda", 0)
    transform = "sqrt" if args.metric == "hellinger" else None
    di = sd.to_device(idx_m, tdt, dev, transform=transform)
    dq = sd.to_device(q_m, tdt, dev, transform=transform)
    ix = _lib.device_index(di)
    lib = _lib.load()
    md = _lib.metric_struct(args.metric, None, args.metric != "kl", transform is not None)
    strat = _lib.strategy_struct(_lib.STRAT_AUTO)
    rep = _lib.SdReport()
    flags = _lib.new_flags(dev)
    m, n = dq.n_rows, di.n_rows
    ldo = (n + 3) // 4 * 4
    knn = wl["kind"] == "knn"
    k = wl.get("k", 0)
    out = torch.empty((m, k) if knn else (m, ldo), dtype=tdt, device=dev)
    oi = torch.empty((m, k), dtype=torch.int64, device=dev) if knn else None
    sh = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    ca, cb = _lib.csr_struct(dq), _lib.csr_struct(di)

    def step():
        if knn:
            _lib.check(lib.sd_knn(ctypes.byref(ca), ctypes.byref(cb), ix.handle, _lib.dtype_code(tdt),
                                  ctypes.byref(md), k, 0, out.data_ptr(), oi.data_ptr(), flags.data_ptr(), sh),
                       "sd_knn")
            return
        _lib.check(lib.sd_pairwise(ctypes.byref(ca), ctypes.byref(cb), ix.handle, _lib.dtype_code(tdt),
                                   ctypes.byref(md), ctypes.byref(strat), out.data_ptr(), ldo, flags.data_ptr(),
                                   ctypes.byref(rep), None, sh), "sd_pairwise")

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(args.steps):
            with torch.profiler.record_function("step"):
                step()
        torch.cuda.synchronize()
    evs, api = [], []
    for e in prof.events():
        if (args.api > 0 and e.device_type == torch.autograd.DeviceType.CPU and e.name.startswith("cuda")
                and e.time_range.end - e.time_range.start >= args.api):
            api.append((e.time_range.start, e.time_range.end, -1, "host " + e.name))
        if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.end > e.time_range.start:
            evs.append((e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0) or 0, e.name))
    evs.sort()
    if not evs:
        print("no CUDA activity recorded")
        return
    # split into steps at gaps: the last len/steps events form the last step
    per = len(evs) // args.steps
    last = evs[-per:]
    t0 = last[0][0]
    print(f"# {args.workload} {args.metric} {args.dtype}: last of {args.steps} profiled steps, "
          f"{len(last)} device activities, span {(last[-1][1] - t0) / 1e3:.3f} ms")
    last = sorted(last + [a for a in api if last[0][0] - 500 <= a[0] <= last[-1][1]])
    print(f"{'start_us':>9} {'end_us':>9} {'dur_us':>8} stream  name")
    for s, e, r, name in last:
        print(f"{(s - t0):9.1f} {(e - t0):9.1f} {(e - s):8.1f} {r:6d}  {name[:90]}")
    ends = np.array([e for _, e, r, _ in last if r >= 0])
    print(f"# step span {(ends.max() - t0) / 1e3:.3f} ms")


if __name__ == "__main__":
    main()
