"""Host-side cost of one sd_pairwise call: tiny query batch against the C2 index
(GPU work negligible), wall time per call with and without a sync."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2104_06357_b200 as sd
from paper_2104_06357_b200 import _lib

wl = bench.WORKLOADS["c2"]
index, queries = bench.make_data(wl, 0, 64)
dev = torch.device("cuda", 0)
lib = _lib.load()
di = sd.to_device(index, torch.float32, dev); dq = sd.to_device(queries, torch.float32, dev)
ix = _lib.device_index(di)
md = _lib.metric_struct("cosine", None, True, False)
strat = _lib.strategy_struct(_lib.STRAT_AUTO); rep = _lib.SdReport(); flags = _lib.new_flags(dev)
n = index.n_rows; ldo = (n + 3) // 4 * 4
out = torch.empty((queries.n_rows, ldo), dtype=torch.float32, device=dev)
sh = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
def call(q):
    ca, cb = _lib.csr_struct(q), _lib.csr_struct(di)
    _lib.check(lib.sd_pairwise(ctypes.byref(ca), ctypes.byref(cb), ix.handle, 0, ctypes.byref(md), ctypes.byref(strat),
                               out.data_ptr(), ldo, flags.data_ptr(), ctypes.byref(rep), None, sh), "sd_pairwise")
for nq in (1, 64):
    q = dq.slice_rows(0, nq) if hasattr(dq, "slice_rows") else dq
    for _ in range(3): call(q)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): call(q)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"queries={nq}: host {1e3*(t1-t0)/20:.3f} ms/call, wall incl. GPU {1e3*(t2-t0)/20:.3f} ms/call")
