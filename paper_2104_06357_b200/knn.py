"""Brute-force sparse kNN (reference: /root/reference/pkg/src/semidist/knn.py).

``kneighbors`` keeps the reference contract — ascending distances, ties to
the lower index id, self-matches kept, results independent of batching — and
runs as ONE fused launch (``sd_knn``): distances are reduced to the top-k in
registers inside the intersection kernel, so the m x n distance matrix is
never written.  Forced engine strategies materialise query batches and select
with ``sd_topk_rows``.
"""

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .engine import WorkspaceReport, resolve_strategy
from .errors import DimensionMismatch, KTooLarge
from .metrics import _engine_report, _metric_args, pairwise_distances_detail
from .sparse import DeviceCsr, _torch_dtype, to_device

DEFAULT_MEMORY_BUDGET_BYTES = 256 * (1 << 20)   # knn.py:13


@dataclass(frozen=True)
class NeighborResult:
    distances: np.ndarray  # (n_queries, k) float64
    indices: np.ndarray    # (n_queries, k) int64


@dataclass(frozen=True)
class BatchPlan:
    batch_rows: int
    n_batches: int
    batch_output_elements: int


def plan_batches(n_queries, n_index, batch_rows=None, memory_budget_bytes=DEFAULT_MEMORY_BUDGET_BYTES):
    """Query batch size keeping a dense batch output under budget (knn.py:31-38)."""
    if batch_rows is None:
        batch_rows = memory_budget_bytes // (8 * max(1, n_index))
    batch_rows = int(max(1, min(batch_rows, max(1, n_queries))))
    n_batches = -(-n_queries // batch_rows) if n_queries else 0
    return BatchPlan(batch_rows, n_batches, batch_rows * n_index)


def select_topk(row_distances, k, *, device=None):
    """k smallest in ascending order, ties by ascending index (knn.py:41-47), on device."""
    import torch
    row = np.asarray(row_distances, dtype=np.float64).reshape(-1)
    if k > row.size:
        raise KTooLarge(f"k={k} exceeds {row.size} candidates")
    if k < 0:
        raise ValueError("k must be non-negative")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    d = torch.from_numpy(row).to(dev)
    od = torch.empty(k, dtype=torch.float64, device=dev)
    oi = torch.empty(k, dtype=torch.int64, device=dev)
    if k:
        _lib.call(dev, "sd_topk_rows", d.data_ptr(), 1, row.size, row.size, _lib.SD_F64, int(k), 0, od.data_ptr(),
                  oi.data_ptr(), _lib.stream_handle(dev))
    return od.cpu().numpy(), oi.cpu().numpy()


def knn_device(index, queries, k, spec, *, dtype=np.float32, index_base=0, check_flags=True):
    """Fused kNN on device-resident operands; returns CUDA tensors (dist, idx).
    This is the building block of the sharded multi-GPU path."""
    import torch
    name, p, strict = _metric_args(spec)
    tdt = _torch_dtype(dtype)
    transform = "sqrt" if name == "hellinger" else None
    di = to_device(index, tdt, None, transform=transform)
    dq = di if queries is index else to_device(queries, tdt, di.device, transform=transform)
    if di.n_cols != dq.n_cols:
        raise DimensionMismatch(f"column counts differ: {dq.n_cols} vs {di.n_cols}")
    if k > di.n_rows:
        raise KTooLarge(f"k={k} exceeds {di.n_rows} index rows")
    if k < 0:
        raise ValueError("k must be non-negative")
    od = torch.empty((dq.n_rows, k), dtype=tdt, device=di.device)
    oi = torch.empty((dq.n_rows, k), dtype=torch.int64, device=di.device)
    flags = _lib.new_flags(di.device)
    if k and dq.n_rows:
        md = _lib.metric_struct(name, p, strict, pre_transformed=transform is not None)
        ix = _lib.device_index(di).handle if name != "chebyshev" else None
        cq, cb = _lib.csr_struct(dq), _lib.csr_struct(di)
        _lib.call(di.device, "sd_knn", ctypes.byref(cq), ctypes.byref(cb), ix, _lib.dtype_code(tdt), ctypes.byref(md),
                  int(k), int(index_base), od.data_ptr(), oi.data_ptr(), flags.data_ptr(),
                  _lib.stream_handle(di.device))
    if check_flags:
        _lib.raise_flags(int(flags.item()), name)
    return od, oi, flags


def kneighbors_detail(index, queries, k, spec, strategy=None, batch_rows=None, workers=None,
                      memory_budget_bytes=DEFAULT_MEMORY_BUDGET_BYTES, *, dtype=np.float64, device=None):
    """kneighbors + WorkspaceReport + timings + BatchPlan (knn.py:50-82)."""
    import torch
    if index.n_cols != queries.n_cols:
        raise DimensionMismatch(f"column counts differ: {queries.n_cols} vs {index.n_cols}")
    if k > index.n_rows:
        raise KTooLarge(f"k={k} exceeds {index.n_rows} index rows")
    if k < 0:
        raise ValueError("k must be non-negative")
    name, _, _ = _metric_args(spec)
    plan = plan_batches(queries.n_rows, index.n_rows, batch_rows, memory_budget_bytes)
    timings = {"norms": 0.0, "pass1": 0.0, "pass2": 0.0, "expansion": 0.0, "topk": 0.0}
    tdt = _torch_dtype(dtype)
    fused = strategy is None or (isinstance(strategy, str) and strategy == "auto")
    passes = getattr(spec, "passes", 1)
    report = WorkspaceReport()
    if fused:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if device is not None:
            with torch.cuda.device(torch.device(device)):
                od, oi, _ = knn_device(index, queries, k, spec, dtype=tdt)
        else:
            od, oi, _ = knn_device(index, queries, k, spec, dtype=tdt)
        torch.cuda.synchronize()
        timings["pass1"] = time.perf_counter() - t0
        for start in range(0, queries.n_rows, plan.batch_rows):
            stop = min(start + plan.batch_rows, queries.n_rows)
            report = report.merged(_batch_report(index, queries, start, stop, passes, name, strategy))
        return (NeighborResult(_lib.as_numpy_f64(od), oi.cpu().numpy().astype(np.int64)), report, timings, plan)
    dists = np.empty((queries.n_rows, k), dtype=np.float64)
    ids = np.empty((queries.n_rows, k), dtype=np.int64)
    dq = to_device(queries, tdt, device)
    dix = to_device(index, tdt, dq.device)
    for start in range(0, queries.n_rows, plan.batch_rows):
        stop = min(start + plan.batch_rows, queries.n_rows)
        batch = dq.slice_rows(start, stop)
        d, rep, times = pairwise_distances_detail(batch, dix, spec, strategy, dtype=tdt, return_device=True)
        report = report.merged(rep)
        for key, value in times.items():
            if key.startswith("device_"):   # footprints, not times: the largest batch's
                timings[key] = max(timings.get(key, 0), value)
            else:
                timings[key] += value
        t0 = time.perf_counter()
        bd = torch.empty((stop - start, k), dtype=tdt, device=d.device)
        bi = torch.empty((stop - start, k), dtype=torch.int64, device=d.device)
        if k and d.numel():
            _lib.call(d.device, "sd_topk_rows", d.data_ptr(), stop - start, index.n_rows, d.stride(0),
                      _lib.dtype_code(tdt), int(k), 0, bd.data_ptr(), bi.data_ptr(), _lib.stream_handle(d.device))
        dists[start:stop] = _lib.as_numpy_f64(bd)
        ids[start:stop] = bi.cpu().numpy()
        timings["topk"] += time.perf_counter() - t0
    return NeighborResult(dists, ids), report, timings, plan


def _batch_report(index, queries, start, stop, passes, name, strategy):
    """Reference accounting of one query batch (knn.py:71-73 -> metrics.py:340-366)."""
    from .engine import _degrees, reference_report

    class _Slice:
        def __init__(self, deg, n_cols):
            self.deg = deg
            self.n_cols = n_cols
            self.n_rows = len(deg)
            self.nnz = int(deg.sum())

    qdeg = _degrees(queries)[start:stop]
    ideg = _degrees(index)
    strat = resolve_strategy(strategy, _DegView(qdeg, queries.n_cols))
    rep = reference_report(qdeg, strat, int(ideg.sum()))
    if passes == 2 or name == "kl":
        rep = rep.merged(reference_report(ideg, strat, int(qdeg.sum())))
    return rep


class _DegView:
    """Minimal matrix view (n_rows, n_cols, degrees) for strategy resolution."""

    def __init__(self, deg, n_cols):
        self._deg = np.asarray(deg)
        self.n_rows = int(self._deg.size)
        self.n_cols = int(n_cols)
        self.indptr = np.concatenate(([0], np.cumsum(self._deg)))


def kneighbors(index, queries, k, spec, strategy=None, batch_rows=None, workers=None,
               memory_budget_bytes=DEFAULT_MEMORY_BUDGET_BYTES, **kw):
    """k nearest index rows per query (knn.py:85-94)."""
    result, _, _, _ = kneighbors_detail(index, queries, k, spec, strategy, batch_rows, workers,
                                        memory_budget_bytes, **kw)
    return result
