"""Multi-GPU execution (one process per GPU, torch.distributed for plumbing).

SURVEY.md §8(e):
* pairwise distances shard the QUERY rows (A) across ranks with the index (B)
  replicated — every output row has one owner, so there is no collective on
  the data path (``pairwise_distances_sharded``);
* kNN shards the INDEX rows (B) across ranks with the queries replicated;
  each rank runs the fused top-k over its shard with global row ids
  (index_base = shard start), the per-rank candidate lists are exchanged with
  ONE all-gather (NCCL over NVLink on GPUs, gloo in the CPU tests) and merged
  on device by ``sd_topk_merge`` with the same (distance, index) order as
  numpy's stable argsort (knn.py:77), so the result equals the single-GPU one.
"""

import ctypes

import numpy as np

from . import _lib
from .knn import NeighborResult, knn_device
from .metrics import pairwise_distances_detail
from .sparse import slice_rows


def shard_bounds(n_rows, world, weights=None):
    """Contiguous row ranges [lo, hi) per rank.  With ``weights`` (per-row
    cost, e.g. degree + constant) the cut points balance the cumulative cost
    instead of the row count."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    if weights is None:
        cuts = [(n_rows * r) // world for r in range(world + 1)]
    else:
        w = np.asarray(weights, dtype=np.float64)
        if w.size != n_rows:
            raise ValueError("one weight per row expected")
        cum = np.concatenate(([0.0], np.cumsum(w)))
        targets = cum[-1] * np.arange(world + 1) / world
        cuts = np.searchsorted(cum, targets, side="left").tolist()
        cuts[0], cuts[-1] = 0, n_rows
        for r in range(1, world + 1):
            cuts[r] = max(cuts[r], cuts[r - 1])
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def _rank_world(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def pairwise_distances_sharded(a, b, spec, *, group=None, dtype=np.float32, balance=True, **kw):
    """This rank's block of the distance matrix: rows [lo, hi) of ``a``
    against all of ``b``.  Returns (lo, hi, rows, report, timings)."""
    rank, world = _rank_world(group)
    weights = None
    if balance:
        weights = np.diff(np.asarray(a.indptr)).astype(np.float64) + 16.0
    lo, hi = shard_bounds(a.n_rows, world, weights)[rank]
    part = slice_rows(a, lo, hi)
    rows, report, timings = pairwise_distances_detail(part, b, spec, dtype=dtype, **kw)
    return lo, hi, rows, report, timings


def gather_candidates(dist_t, idx_t, group=None):
    """All-gather per-rank (m, k) candidate tensors -> (world, m, k) tensors."""
    import torch
    import torch.distributed as dist
    _, world = _rank_world(group)
    if world == 1:
        return dist_t.unsqueeze(0), idx_t.unsqueeze(0)
    if dist.get_backend(group) == "nccl":   # one NCCL all-gather per tensor over NVLink
        out_d = torch.empty((world,) + tuple(dist_t.shape), dtype=dist_t.dtype, device=dist_t.device)
        out_i = torch.empty((world,) + tuple(idx_t.shape), dtype=idx_t.dtype, device=idx_t.device)
        dist.all_gather_into_tensor(out_d, dist_t.contiguous(), group=group)
        dist.all_gather_into_tensor(out_i, idx_t.contiguous(), group=group)
        return out_d, out_i
    # gloo (CPU tests, or several ranks sharing one GPU): stage device
    # candidates through host memory, return them on the caller's device
    dev = dist_t.device
    hd, hi = dist_t.detach().to("cpu").contiguous(), idx_t.detach().to("cpu").contiguous()
    parts_d = [torch.empty_like(hd) for _ in range(world)]
    parts_i = [torch.empty_like(hi) for _ in range(world)]
    dist.all_gather(parts_d, hd, group=group)
    dist.all_gather(parts_i, hi, group=group)
    return torch.stack(parts_d).to(dev), torch.stack(parts_i).to(dev)


def merge_candidates(cand_d, cand_i, k):
    """Device merge of (lists, m, k) sorted candidate lists into the global top-k."""
    import torch
    lists, m, kk = cand_d.shape
    if kk != k:
        raise ValueError("candidate lists must have length k")
    od = torch.empty((m, k), dtype=cand_d.dtype, device=cand_d.device)
    oi = torch.empty((m, k), dtype=torch.int64, device=cand_d.device)
    if m and k:
        cd, ci = cand_d.contiguous(), cand_i.contiguous()
        _lib.call(cand_d.device, "sd_topk_merge", cd.data_ptr(), ci.data_ptr(), m, lists, int(k),
                  _lib.dtype_code(cand_d.dtype), od.data_ptr(), oi.data_ptr(), _lib.stream_handle(cand_d.device))
    return od, oi


def local_topk_padded(index_shard, queries, k, spec, *, index_base, dtype=np.float32):
    """Fused top-k over this rank's index shard, padded to k with (NaN, int64
    max) when the shard holds fewer than k rows, so all ranks gather equal shapes."""
    import torch
    kk = min(k, index_shard.n_rows)
    od, oi, _ = knn_device(index_shard, queries, kk, spec, dtype=dtype, index_base=index_base)
    if kk < k:
        pad_d = torch.full((od.shape[0], k - kk), float("nan"), dtype=od.dtype, device=od.device)
        pad_i = torch.full((oi.shape[0], k - kk), np.iinfo(np.int64).max, dtype=oi.dtype, device=oi.device)
        od, oi = torch.cat([od, pad_d], 1), torch.cat([oi, pad_i], 1)
    return od, oi


def kneighbors_sharded(index, queries, k, spec, *, group=None, dtype=np.float32, index_shard=None,
                       shard_lo=None):
    """Global kNN with the index sharded across ranks (one all-gather of k
    candidates per query per rank).  ``index_shard``/``shard_lo`` let callers
    pass a pre-built device shard (e.g. the benchmark); by default the shard is
    sliced from ``index`` with ``shard_bounds``."""
    from .errors import KTooLarge
    rank, world = _rank_world(group)
    if index_shard is None:
        lo, hi = shard_bounds(index.n_rows, world)[rank]
        index_shard, shard_lo = slice_rows(index, lo, hi), lo
    n_total = index.n_rows if index is not None else None
    if n_total is not None and k > n_total:
        raise KTooLarge(f"k={k} exceeds {n_total} index rows")
    od, oi = local_topk_padded(index_shard, queries, k, spec, index_base=shard_lo, dtype=dtype)
    cd, ci = gather_candidates(od, oi, group)
    md, mi = merge_candidates(cd, ci, k)
    return NeighborResult(_lib.as_numpy_f64(md), mi.cpu().numpy().astype(np.int64))
