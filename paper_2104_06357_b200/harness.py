"""Benchmark and verification harness of the drop-in (reference:
/root/reference/pkg/src/semidist/bench.py and verification.py).

``run_bench`` times the kNN query phase through ``kneighbors_detail`` and
reports the reference's JSON fields, including the tolerance-quantized
checksum (values rounded to 1e-8 before hashing) that lets a GPU run and a
CPU reference run be compared directly.  ``verify_metric`` checks the sparse
engine against an independent dense brute-force arbiter — here a separate
CUDA kernel (``sd_dense_pairwise``, the textbook formulas over all columns)
that shares no code with the sparse kernels.
"""

import ctypes
import hashlib
import time
from dataclasses import asdict, dataclass

import numpy as np

from . import _lib
from .engine import ExecutionStrategy
from .errors import DomainError, SizeOverflow
from .knn import kneighbors_detail
from .metrics import BINARY_PREFERRED, metric_registry, pairwise_distances
from .sparse import from_dense

CHECKSUM_QUANTUM_DECIMALS = 8   # bench.py:15
RTOL = 1e-6                     # verification.py:12
ATOL = 1e-9                     # verification.py:13
DENSE_ELEMENT_CAP = 1 << 26     # oracle.py:13


def quantized_checksum(arr):
    """SHA-256 of the values rounded to 1e-8 (-0.0 normalised): reduction-order
    noise below the quantum does not change it (bench.py:18-23)."""
    q = np.round(np.ascontiguousarray(arr, dtype=np.float64), CHECKSUM_QUANTUM_DECIMALS) + 0.0
    return hashlib.sha256(q.tobytes()).hexdigest()


def _strategy_label(strategy):
    if isinstance(strategy, ExecutionStrategy):
        label = strategy.kind.value
        if strategy.accumulator_capacity:
            label += f"(capacity={strategy.accumulator_capacity},load={strategy.max_load_factor:g})"
        return label
    return str(strategy or "auto")


def run_bench(index, queries, spec, strategy=None, k=10, batch_rows=None, repeat=1, workers=None, **kw):
    """Median query time over ``repeat`` runs plus workspace accounting and the
    distance checksum, as JSON-ready dict (bench.py:34-68)."""
    import torch
    runs = []
    result = report = timings = plan = None
    for _ in range(max(1, int(repeat))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        result, report, timings, plan = kneighbors_detail(index, queries, k, spec, strategy, batch_rows, workers, **kw)
        torch.cuda.synchronize()
        runs.append(time.perf_counter() - t0)
    return {
        "metric": spec.name, "params": dict(spec.params), "strategy": _strategy_label(strategy), "k": k,
        "index_rows": index.n_rows, "query_rows": queries.n_rows, "n_cols": index.n_cols,
        "index_nnz": index.nnz, "query_nnz": queries.nnz,
        "batch_rows": plan.batch_rows, "n_batches": plan.n_batches,
        "timings": dict(timings), "query_seconds": float(np.median(runs)), "runs": runs,
        "workspace": asdict(report), "checksum": quantized_checksum(result.distances),
    }


def densify(m, element_cap=DENSE_ELEMENT_CAP):
    """Dense float64 copy of a CSR matrix, capped like oracle.densify."""
    if m.n_rows * m.n_cols > element_cap:
        raise SizeOverflow(f"{m.n_rows} x {m.n_cols} exceeds the {element_cap}-element cap")
    out = np.zeros((m.n_rows, m.n_cols))
    deg = np.diff(np.asarray(m.indptr))
    out[np.repeat(np.arange(m.n_rows), deg), np.asarray(m.indices)] = np.asarray(m.values)
    return out


def dense_pairwise(a, b, name, *, p=None, strict=True, device=None):
    """m x n matrix of the textbook distance formulas on the densified rows
    (oracle.py:170-190 contract), evaluated by the sd_dense_pairwise kernel."""
    import torch
    da = a if isinstance(a, np.ndarray) else densify(a)
    db = b if isinstance(b, np.ndarray) else densify(b)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ta = torch.from_numpy(np.ascontiguousarray(da, dtype=np.float64)).to(dev)
    tb = torch.from_numpy(np.ascontiguousarray(db, dtype=np.float64)).to(dev)
    out = torch.empty((da.shape[0], db.shape[0]), dtype=torch.float64, device=dev)
    flags = _lib.new_flags(dev)
    md = _lib.metric_struct(name, p, strict)
    if out.numel():
        _lib.call(dev, "sd_dense_pairwise", ta.data_ptr(), tb.data_ptr(), da.shape[0], db.shape[0], da.shape[1],
                  ctypes.byref(md), out.data_ptr(), flags.data_ptr(), _lib.stream_handle(dev))
    f = int(flags.item())
    if f & _lib.SD_FLAG_NEGATIVE:
        raise DomainError(f"{name} requires non-negative inputs")
    if f & _lib.SD_FLAG_KL_UNCOVERED:
        raise DomainError("kl: support of the left vector is not covered by the right")
    return out.cpu().numpy()


@dataclass
class VerifyResult:
    metric: str
    trials: int
    failures: int
    max_abs_err: float

    @property
    def passed(self):
        return self.failures == 0


def random_instance(rng, name, max_rows=40, max_cols=32, density_range=(0.05, 0.5)):
    """A random matrix pair in the metric's domain, drawn in the reference's
    order so a seed gives the same instances (verification.py:28-51): binary
    patterns for the set metrics, values in [0.1, 1) otherwise, and a fully
    dense right side for kl (every query support covered)."""
    m, n, k = (int(rng.integers(1, hi + 1)) for hi in (max_rows, max_rows, max_cols))
    density = float(rng.uniform(*density_range))
    mask_a, mask_b = rng.random((m, k)) < density, rng.random((n, k)) < density
    if name in BINARY_PREFERRED:
        return from_dense(mask_a.astype(np.float64)), from_dense(mask_b.astype(np.float64))
    da = np.where(mask_a, rng.uniform(0.1, 1.0, (m, k)), 0.0)
    db = rng.uniform(0.1, 1.0, (n, k)) if name == "kl" else np.where(mask_b, rng.uniform(0.1, 1.0, (n, k)), 0.0)
    return from_dense(da), from_dense(db)


def verify_metric(name, trials=20, max_rows=40, max_cols=32, seed=0, strategy=None, rtol=RTOL, atol=ATOL):
    """Sparse GPU engine vs the dense GPU arbiter on random instances (verification.py:54-71)."""
    rng = np.random.default_rng(seed)
    failures, worst, p = 0, 0.0, None
    for _ in range(int(trials)):
        a, b = random_instance(rng, name, max_rows, max_cols)
        if name == "minkowski":
            p = float(rng.choice([1.0, 1.5, 2.0, 3.0]))
        got = pairwise_distances(a, b, metric_registry(name, p=p), strategy=strategy)
        want = dense_pairwise(a, b, name, p=p)
        if got.size:
            worst = max(worst, float(np.max(np.abs(got - want))))
        failures += 0 if np.allclose(got, want, rtol=rtol, atol=atol) else 1
    return VerifyResult(name, int(trials), failures, worst)
