"""Distance catalog and the pairwise-distance entry points
(reference: /root/reference/pkg/src/semidist/metrics.py).

``pairwise_distances[_detail]`` keep the reference signature and contract
(dense m x n float64, C-contiguous, per-phase timings, WorkspaceReport) and add
keyword-only ``dtype`` (float64 default, float32 for throughput), ``device``
and ``return_device`` (keep the result as a CUDA tensor).  The computation is
one call of ``sd_pairwise`` (csrc/api.cu): the fused intersection kernel for
every (+)-reduced metric under the default strategy, the two-pass engine for
chebyshev or when a strategy is forced.
"""

import ctypes
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from . import semiring as sr
from .engine import (StrategyKind, WorkspaceReport, _degrees, _strategy_struct, reference_report,
                     resolve_strategy)
from .errors import DimensionMismatch, DomainError, MissingParam, UnknownMetric
from .semiring import Semiring
from .sparse import NormKind, NormVector, _torch_dtype, to_device

NEGATIVE_RADICAND_TOLERANCE = 1e-9   # metrics.py:27
KL_SATURATION = 1e308                # metrics.py:29

METRIC_NAMES = (
    "correlation", "cosine", "dice", "dot", "euclidean", "hellinger",
    "jaccard", "kl", "russelrao",
    "canberra", "chebyshev", "hamming", "jensenshannon", "manhattan", "minkowski",
)

BINARY_PREFERRED = frozenset({"dice", "jaccard", "russelrao", "hamming"})


class _Epilogue:
    """One catalog row's expansion (``(dots, stats_a, stats_b, k) -> matrix``)
    or post-scale (``(matrix, k) -> matrix``) stage, evaluated on device by
    sd_expand (csrc/metric.cuh ``expand_stage``) — the same per-cell code the
    fused kernels apply inside ``sd_pairwise``."""

    def __init__(self, metric, stage, p=None):
        self.metric = metric
        self.stage = stage
        self.p = p

    def __call__(self, x, *args):
        if self.stage == "expansion":
            stats_a, stats_b, k = args
            return _device_expand(x, stats_a, stats_b, self.metric, self.p, int(k), stages=1)
        (k,) = args
        return _device_expand(x, None, None, self.metric, self.p, int(k), stages=2)

    def __repr__(self):
        return f"<device {self.stage} of {self.metric}>"


@dataclass(frozen=True)
class MetricSpec:
    """One Table-1 row (metrics.py:40-52)."""

    name: str
    semiring: Semiring
    passes: int
    norms_needed: tuple
    expansion: Optional[Callable] = None
    post_scale: Optional[Callable] = None
    value_transform: Optional[Callable] = None
    requires_nonnegative: bool = False
    params: dict = field(default_factory=dict)


@dataclass(frozen=True)
class SideStats:
    """Per-row statistics of one side (metrics.py:55-90)."""

    l0: Optional[np.ndarray] = None
    l1: Optional[np.ndarray] = None
    l2: Optional[np.ndarray] = None
    l2sq: Optional[np.ndarray] = None
    signed_sum: Optional[np.ndarray] = None

    @classmethod
    def from_norms(cls, norms, signed_sum=None):
        f = {"signed_sum": None if signed_sum is None else np.asarray(signed_sum, dtype=np.float64)}
        for nv in norms:
            f[NormKind(nv.kind).value] = np.asarray(nv.values, dtype=np.float64)
        if "l2" in f and "l2sq" not in f:
            f["l2sq"] = f["l2"] ** 2
        if "l2sq" in f and "l2" not in f:
            f["l2"] = np.sqrt(f["l2sq"])
        return cls(**f)

    def require(self, attr, metric):
        v = getattr(self, attr)
        if v is None:
            raise ValueError(f"{metric} expansion needs per-row '{attr}' statistics")
        return v

    def sums(self, metric):
        return self.signed_sum if self.signed_sum is not None else self.require("l1", metric)


def _spec(name, ring, passes, norms, expansion=False, post=False, transform=None, nonneg=False, params=None):
    p = (params or {}).get("p")
    return MetricSpec(name, ring, passes, norms,
                      _Epilogue(name, "expansion", p) if expansion else None,
                      _Epilogue(name, "post_scale", p) if post else None,
                      transform, nonneg, dict(params or {}))


def metric_registry(name, *, p=None, strict=True):
    """Catalog lookup (metrics.py:254-284)."""
    key = str(name).lower()
    if key not in METRIC_NAMES:
        raise UnknownMetric(f"unknown metric '{name}'; supported: " + ", ".join(METRIC_NAMES))
    L0, L2, L2SQ, L1 = NormKind.L0, NormKind.L2, NormKind.L2_SQUARED, NormKind.L1
    dot = sr.dot_product()
    if key == "correlation":
        return _spec(key, dot, 1, (L1, L2SQ), expansion=True)
    if key == "cosine":
        return _spec(key, dot, 1, (L2,), expansion=True)
    if key in ("dice", "jaccard"):
        return _spec(key, dot, 1, (L0,), expansion=True)
    if key in ("dot", "russelrao"):
        return _spec(key, dot, 1, (), expansion=True)
    if key == "euclidean":
        return _spec(key, dot, 1, (L2SQ,), expansion=True, post=True)
    if key == "hellinger":
        return _spec(key, dot, 1, (), expansion=True, transform=np.sqrt, nonneg=True)
    if key == "kl":
        return _spec(key, sr.kl_divergence_term(), 1, (), expansion=True, nonneg=True,
                     params={"strict": bool(strict)})
    if key == "canberra":
        return _spec(key, sr.canberra_ratio(), 2, ())
    if key == "chebyshev":
        return _spec(key, sr.max_absolute_difference(), 2, ())
    if key == "hamming":
        return _spec(key, sr.mismatch_indicator(), 2, (), post=True)
    if key == "jensenshannon":
        return _spec(key, sr.jensen_shannon_term(), 2, (), post=True, nonneg=True)
    if key == "manhattan":
        return _spec(key, sr.absolute_difference(), 2, ())
    # minkowski
    if p is None:
        raise MissingParam("minkowski requires the order parameter p")
    p = float(p)
    if not np.isfinite(p) or p < 1.0:
        raise DomainError("minkowski requires finite p >= 1")
    return _spec(key, sr.absolute_difference_power(p), 2, (), post=True, params={"p": p})


def _metric_args(spec):
    """(name, p, strict) of our MetricSpec or the reference's (duck-typed)."""
    name = str(spec.name).lower()
    if name not in _lib.METRIC_IDS:
        raise UnknownMetric(f"unknown metric '{spec.name}'")
    params = getattr(spec, "params", {}) or {}
    return name, params.get("p"), bool(params.get("strict", True))


def _stats_layout(name):
    """Which per-row statistics sd_expand reads, in order (csrc/metric.cuh)."""
    return {"correlation": ("signed_sum", "l2sq"), "cosine": ("l2",), "dice": ("l0",),
            "jaccard": ("l0",), "euclidean": ("l2sq",)}.get(name, ())


def _device_expand(dots, stats_a, stats_b, name, p, k, stages, *, dtype=np.float64, device=None):
    """sd_expand over a host matrix: stage 1 = expansion, 2 = post-scale, 0 = both."""
    import torch
    dots = np.asarray(dots, dtype=np.float64)
    shape = dots.shape
    d2 = dots.reshape(1, -1) if dots.ndim == 1 else dots.reshape(-1, shape[-1]) if dots.ndim else dots.reshape(1, 1)
    tdt = _torch_dtype(dtype)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    d = torch.from_numpy(np.ascontiguousarray(d2)).to(dev).to(tdt).contiguous()
    keep = []

    def arrays(st):
        if st is None or stages == 2:
            return None
        ptrs = []
        for attr in _stats_layout(name):
            v = st.sums(name) if attr == "signed_sum" else st.require(attr, name)
            t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(dev).to(tdt)
            keep.append(t)
            ptrs.append(t.data_ptr())
        return (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs) if ptrs else None

    pa, pb = arrays(stats_a), arrays(stats_b)
    flags = _lib.new_flags(dev)
    md = _lib.metric_struct(name, p, True, stages=stages)
    if d.numel():
        m, n = d.shape
        _lib.call(dev, "sd_expand", d.data_ptr(), m, n, n, _lib.dtype_code(tdt), ctypes.byref(md), int(k),
                  pa, pb, flags.data_ptr(), _lib.stream_handle(dev))
    _lib.raise_flags(int(flags.item()), name)
    return _lib.as_numpy_f64(d).reshape(shape)


def expansion_apply(dots, norms_a, norms_b, spec, *, n_cols, sums_a=None, sums_b=None,
                    dtype=np.float64, device=None):
    """Expansion + post-scale over a dots matrix (metrics.py:287-300), on device
    in one sd_expand launch.  ``spec`` may be the reference's MetricSpec: only
    its name and params are read (its numpy callables are never run)."""
    name, p, strict = _metric_args(spec)
    sa = SideStats.from_norms(norms_a, signed_sum=sums_a)
    sb = SideStats.from_norms(norms_b, signed_sum=sums_b)
    return _device_expand(dots, sa, sb, name, p, n_cols, stages=0, dtype=dtype, device=device)


def _engine_report(da, db, spec_passes, name, strategy, a, b):
    """WorkspaceReport the reference reports for this call (metrics.py:340-366)."""
    strat = resolve_strategy(strategy, a, b)
    rep = reference_report(_degrees(da), strat, db.nnz)
    if spec_passes == 2 or name == "kl":
        rep = rep.merged(reference_report(_degrees(db), strat, da.nnz))
    return rep


def pairwise_distances_detail(a, b, spec, strategy=None, workers=None, *, dtype=np.float64, device=None,
                              return_device=False, check_flags=True, out=None):
    """Distances + WorkspaceReport + per-phase device times (metrics.py:320-375).

    ``strategy`` None/"auto" runs the fused intersection kernel (two-pass
    engine for chebyshev); "naive"/"dense"/"hash"/ExecutionStrategy force the
    engine with the reference's chunking semantics.  ``workers`` is accepted
    for compatibility and ignored.  ``out`` (host numpy array or CPU torch
    tensor, ideally pinned, shape (m, n)) receives the result by one
    device->host copy and is returned instead of a new array.
    """
    import torch
    if a.n_cols != b.n_cols:
        raise DimensionMismatch(f"column counts differ: {a.n_cols} vs {b.n_cols}")
    name, p, strict = _metric_args(spec)
    tdt = _torch_dtype(dtype)
    transform = "sqrt" if name == "hellinger" else None
    da = to_device(a, tdt, device, transform=transform)
    db = da if b is a else to_device(b, tdt, da.device, transform=transform)
    passes = getattr(spec, "passes", 2 if name in METRIC_NAMES[9:] else 1)
    fused = strategy is None or (isinstance(strategy, str) and strategy == "auto")
    report = _engine_report(da, db, passes, name, strategy, a, b)
    host_out = out
    # 16-byte aligned rows let the kernel store 4 cells per lane; a host `out`
    # is filled by one contiguous D2H copy, so it gets an unpadded buffer
    ldo = b.n_rows if out is not None else (b.n_rows + 3) // 4 * 4
    out_buf = torch.empty((a.n_rows, ldo), dtype=tdt, device=da.device)
    out = out_buf[:, :b.n_rows]
    flags = _lib.new_flags(da.device)
    md = _lib.metric_struct(name, p, strict, pre_transformed=transform is not None)
    phases = (ctypes.c_float * 4)()
    ca, cb = _lib.csr_struct(da), _lib.csr_struct(db)
    if fused:
        strat = _lib.strategy_struct(_lib.STRAT_AUTO)
        index = _lib.device_index(db).handle if (a.n_rows and b.n_rows and name != "chebyshev") else None
    else:
        strat = _strategy_struct(resolve_strategy(strategy, a, b))
        index = None
    rep = _lib.SdReport()
    _lib.call(da.device, "sd_pairwise", ctypes.byref(ca), ctypes.byref(cb), index, _lib.dtype_code(tdt),
              ctypes.byref(md), ctypes.byref(strat), out_buf.data_ptr() if out.numel() else None, ldo,
              flags.data_ptr(), ctypes.byref(rep), phases, _lib.stream_handle(da.device))
    if check_flags:
        _lib.raise_flags(int(flags.item()), name)
    timings = {"norms": phases[0] / 1e3, "pass1": phases[1] / 1e3, "pass2": phases[2] / 1e3,
               "expansion": phases[3] / 1e3,
               # device footprint beside the reference-shaped WorkspaceReport (which restates the
               # reference's CPU staging plan): the cached index of b and this call's output
               "device_index_bytes": _lib.device_index(db).bytes if index is not None else 0,
               "device_output_bytes": int(out_buf.numel() * out_buf.element_size())}
    if host_out is not None:
        dst = host_out if isinstance(host_out, torch.Tensor) else torch.from_numpy(host_out)
        if tuple(dst.shape) != (a.n_rows, b.n_rows):
            raise ValueError(f"out has shape {tuple(dst.shape)}, expected {(a.n_rows, b.n_rows)}")
        src = out if dst.dtype == out.dtype else out.to(dst.dtype)
        dst.copy_(src, non_blocking=dst.is_pinned())
        torch.cuda.current_stream(da.device).synchronize()
        return host_out, report, timings
    if return_device:
        return out, report, timings
    return _lib.as_numpy_f64(out), report, timings


def pairwise_distances(a, b, spec, strategy=None, workers=None, **kw):
    """Dense m x n matrix of ``spec``'s distance between rows of a and b (metrics.py:378-381)."""
    result, _, _ = pairwise_distances_detail(a, b, spec, strategy, workers, **kw)
    return result
