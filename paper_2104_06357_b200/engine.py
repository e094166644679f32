"""Engine-level API: execution strategies and the two sweeps of the
generalized pairwise SpMV (reference: /root/reference/pkg/src/semidist/engine.py).

Host side keeps the reference's planning vocabulary (strategy resolution,
``plan_chunks``, WorkspaceReport accounting) so results and reports read the
same; every sweep runs in ``sd_pass`` (csrc/engine.cu) on the GPU.
"""

import ctypes
import os
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .errors import DimensionMismatch
from .semiring import device_id
from .sparse import DeviceCsr, to_device

DENSE_COLUMN_LIMIT = 16384   # engine.py:49
HASH_CAPACITY_CAP = 16384    # engine.py:50


class StrategyKind(Enum):
    NAIVE_MERGE = "naive"
    BALANCED_DENSE = "dense"
    BALANCED_HASH = "hash"


@dataclass(frozen=True)
class ExecutionStrategy:
    """engine.py:59-77."""

    kind: StrategyKind
    accumulator_capacity: int = 0
    max_load_factor: float = 0.5

    def __post_init__(self):
        if not 0.0 < self.max_load_factor <= 1.0:
            raise ValueError("max_load_factor must be in (0, 1]")
        if self.kind is StrategyKind.BALANCED_HASH:
            if self.accumulator_capacity < 1:
                raise ValueError("hash strategy needs accumulator_capacity >= 1")
            if self.chunk_budget < 1:
                raise ValueError("accumulator_capacity * max_load_factor must admit at least one entry")

    @property
    def chunk_budget(self):
        return int(self.max_load_factor * self.accumulator_capacity)


@dataclass
class WorkspaceReport:
    """engine.py:80-99 (same fields and merge rule)."""

    peak_accumulator_entries: int = 0
    workspace_elements: int = 0
    chunks_executed: int = 0

    def merged(self, other):
        return WorkspaceReport(max(self.peak_accumulator_entries, other.peak_accumulator_entries),
                               max(self.workspace_elements, other.workspace_elements),
                               self.chunks_executed + other.chunks_executed)


def resolve_workers(workers=None):
    """Kept for signature compatibility (engine.py:102-107); the GPU ignores it."""
    if workers is None:
        env = os.environ.get("WORKERS", "").strip()
        workers = int(env) if env else (os.cpu_count() or 1)
    return max(1, int(workers))


def _degrees(m):
    if isinstance(m, DeviceCsr):
        return m.host_degrees()
    return np.diff(np.asarray(m.indptr))


def auto_hash_capacity(m):
    """Smallest power of two >= 2 * max degree, capped (engine.py:110-115)."""
    deg = _degrees(m)
    mx = int(deg.max()) if deg.size else 0
    need = max(2, 2 * mx)
    return min(1 << (need - 1).bit_length(), HASH_CAPACITY_CAP)


def choose_strategy(a, b=None):
    """engine.py:118-125."""
    if a.n_cols <= DENSE_COLUMN_LIMIT:
        return ExecutionStrategy(StrategyKind.BALANCED_DENSE)
    return ExecutionStrategy(StrategyKind.BALANCED_HASH, accumulator_capacity=auto_hash_capacity(a))


def resolve_strategy(strategy, a, b=None, *, capacity=None, max_load_factor=0.5):
    """engine.py:128-140."""
    if isinstance(strategy, ExecutionStrategy):
        return strategy
    if hasattr(strategy, "kind") and hasattr(strategy, "max_load_factor"):  # the reference's class
        return ExecutionStrategy(StrategyKind(strategy.kind.value), int(strategy.accumulator_capacity),
                                 float(strategy.max_load_factor))
    if strategy is None or strategy == "auto":
        return choose_strategy(a, b)
    kind = StrategyKind(strategy)
    if kind is StrategyKind.BALANCED_HASH:
        cap = auto_hash_capacity(a) if capacity is None else int(capacity)
        return ExecutionStrategy(kind, accumulator_capacity=cap, max_load_factor=max_load_factor)
    return ExecutionStrategy(kind, max_load_factor=max_load_factor)


def plan_chunks(row_degree, strategy):
    """Near-equal spans of at most chunk_budget entries (engine.py:143-164)."""
    if strategy.kind is not StrategyKind.BALANCED_HASH:
        raise ValueError("chunk planning applies to the hash strategy only")
    d = int(row_degree)
    budget = strategy.chunk_budget
    if d <= budget:
        return [(0, d)]
    n = -(-d // budget)
    base, rem = divmod(d, n)
    out, s = [], 0
    for t in range(n):
        sz = base + (1 if t < rem else 0)
        out.append((s, s + sz))
        s += sz
    return out


def reference_report(staged_degrees, strategy, swept_nnz):
    """WorkspaceReport the reference engine reports for one balanced/naive
    sweep (engine.py:212-267, 323-333, 345-353), from staged-row degrees."""
    if strategy.kind is StrategyKind.NAIVE_MERGE:
        return WorkspaceReport(0, 0, 0)
    deg = np.asarray(staged_degrees, dtype=np.int64)
    if strategy.kind is StrategyKind.BALANCED_DENSE:
        return WorkspaceReport(int(deg.max()) if deg.size else 0, int(swept_nnz), int(deg.size))
    budget = strategy.chunk_budget
    n_chunks = np.where(deg <= budget, 1, -(-deg // budget))
    biggest = np.where(deg <= budget, deg, -(-deg // np.maximum(n_chunks, 1)))
    return WorkspaceReport(int(biggest.max()) if deg.size else 0, int(swept_nnz), int(n_chunks.sum()))


def _strategy_struct(strategy):
    if strategy is None:
        return _lib.strategy_struct(_lib.STRAT_AUTO)
    kind = {StrategyKind.NAIVE_MERGE: _lib.STRAT_NAIVE, StrategyKind.BALANCED_DENSE: _lib.STRAT_DENSE,
            StrategyKind.BALANCED_HASH: _lib.STRAT_HASH}[strategy.kind]
    return _lib.strategy_struct(kind, strategy.accumulator_capacity, strategy.max_load_factor)


def allocate_output(a, b, semiring, *, dtype=np.float64, device=None):
    """m x n output filled with the reduce identity (engine.py:167-169).
    Host float64 by default; a CUDA tensor when ``device`` is given."""
    if device is None:
        return np.full((a.n_rows, b.n_rows), semiring.reduce_identity, dtype=np.float64)
    import torch
    from .sparse import _torch_dtype
    out = torch.empty((a.n_rows, b.n_rows), dtype=_torch_dtype(dtype), device=device)
    if out.numel():
        _lib.call(out.device, "sd_fill", out.data_ptr(), a.n_rows, b.n_rows, b.n_rows, _lib.dtype_code(out.dtype),
                  float(semiring.reduce_identity), _lib.stream_handle(out.device))
    return out


def _check_inputs(a, b, out):
    if a.n_cols != b.n_cols:
        raise DimensionMismatch(f"column counts differ: {a.n_cols} vs {b.n_cols}")
    if tuple(out.shape) != (a.n_rows, b.n_rows):
        raise ValueError(f"output shape {tuple(out.shape)} != {(a.n_rows, b.n_rows)}")
    if isinstance(out, np.ndarray) and out.dtype != np.float64:
        raise ValueError("output must be float64")


def _run_pass(a, b, semiring, strategy, out, pass_no):
    import torch
    strategy = resolve_strategy(strategy, a, b)
    if out is None:
        raise ValueError("pass 1 needs a pre-initialized output accumulator" if pass_no == 1
                         else "pass 2 accumulates into the pass 1 output")
    _check_inputs(a, b, out)
    host_out = isinstance(out, np.ndarray)
    dtype = torch.float64 if host_out else out.dtype
    device = None if host_out else out.device
    da = to_device(a, dtype, device)
    db = to_device(b, dtype, da.device)
    dev_out = torch.from_numpy(np.ascontiguousarray(out)).to(da.device) if host_out else out
    if dev_out.dim() != 2 or (dev_out.numel() and dev_out.stride(1) != 1):
        raise ValueError("device output must be a row-major matrix (unit column stride)")
    sid, p = device_id(semiring)
    ca, cb = _lib.csr_struct(da), _lib.csr_struct(db)
    strat = _strategy_struct(strategy)
    rep = _lib.SdReport()
    if dev_out.numel():
        _lib.call(da.device, "sd_pass", ctypes.byref(ca), ctypes.byref(cb), _lib.dtype_code(dtype), sid, p, pass_no,
                  ctypes.byref(strat), dev_out.data_ptr(), dev_out.stride(0), ctypes.byref(rep),
                  _lib.stream_handle(da.device))
    if host_out:
        out[...] = dev_out.cpu().numpy()
    staged = da if pass_no == 1 else db
    swept = db if pass_no == 1 else da
    return reference_report(_degrees(staged), strategy, swept.nnz)


def pairwise_spmv_pass1(a, b, semiring, strategy=None, out=None, workers=None):
    """Sweep B's stored columns: out[i, j] ⊕= ⊗(A_i[c] or 0, b_jc) (engine.py:314-333).
    ``out`` (numpy float64, updated in place, or a CUDA tensor) holds the
    reduce identity on entry."""
    return _run_pass(a, b, semiring, strategy, out, 1)


def pairwise_spmv_pass2(a, b, semiring, strategy=None, out=None, workers=None):
    """Complement sweep: out[i, j] ⊕= ⊗(a_ic, 0) for c in A_i \\ B_j (engine.py:336-353)."""
    return _run_pass(a, b, semiring, strategy, out, 2)


def pairwise_generalized(a, b, semiring, strategy=None, workers=None, *, dtype=np.float64,
                         device=None, return_device=False):
    """Pass 1, plus pass 2 for non-annihilating products (engine.py:356-368).
    Returns (out, WorkspaceReport); out is host float64 unless return_device."""
    import torch
    if a.n_cols != b.n_cols:
        raise DimensionMismatch(f"column counts differ: {a.n_cols} vs {b.n_cols}")
    strategy = resolve_strategy(strategy, a, b)
    da = to_device(a, dtype, device)
    db = to_device(b, dtype, da.device)
    out = allocate_output(a, b, semiring, dtype=dtype, device=da.device)
    report = pairwise_spmv_pass1(da, db, semiring, strategy, out)
    if not semiring.annihilating:
        report = report.merged(pairwise_spmv_pass2(da, db, semiring, strategy, out))
    if return_device:
        return out, report
    return _lib.as_numpy_f64(out), report
