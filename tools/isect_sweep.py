"""Tuning sweep for the fused intersection kernel (not part of the product):
kernel time of one C2 cosine/manhattan step for index tile sizes and plans."""
import ctypes, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2104_06357_b200 as sd
from paper_2104_06357_b200 import _lib

index, queries = bench.make_data(bench.WORKLOADS[os.environ.get("WL", "c2")], 0, int(os.environ.get("Q", "10000")))
dev = torch.device("cuda", 0)
lib = _lib.load()
res = {}
for tile in [int(t) for t in os.environ.get("TILES", "2048,4096,8192").split(",")]:
    os.environ["SD_TILE"] = str(tile)
    di = sd.to_device(index, torch.float32, dev)
    di.cache.clear()
    dq = sd.to_device(queries, torch.float32, dev)
    ix = _lib.device_index(di)
    m, n = queries.n_rows, index.n_rows
    ldo = (n + 3) // 4 * 4
    out = torch.empty((m, ldo), dtype=torch.float32, device=dev)
    flags = _lib.new_flags(dev)
    for plan in os.environ.get("BANDS", "auto").split(","):   # "auto" = library default, 0 = no bands
        if plan == "auto":
            os.environ.pop("SD_ISECT_BAND", None)
        else:
            os.environ["SD_ISECT_BAND"] = plan if int(plan) else "1000000"
        for metric in ("cosine", "manhattan"):
            md = _lib.metric_struct(metric)
            ph = (ctypes.c_float * 4)()
            times = []
            for it in range(4):
                ca, cb = _lib.csr_struct(dq), _lib.csr_struct(di)
                _lib.check(lib.sd_pairwise(ctypes.byref(ca), ctypes.byref(cb), ix.handle, 0, ctypes.byref(md),
                                           ctypes.byref(_lib.strategy_struct(3)), out.data_ptr(), ldo,
                                           flags.data_ptr(), None, ph, _lib.stream_handle(dev)), "pw")
                if it:
                    times.append(ph[1])
            res[(tile, plan, metric)] = statistics.median(times)
            print(f"tile {tile:5d} band {plan:>5} {metric:10s} kernel {statistics.median(times):7.3f} ms", flush=True)
    del ix, di
    index_cache = None
