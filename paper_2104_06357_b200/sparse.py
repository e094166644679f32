"""Host-side CSR containers and their device mirrors.

Host side (numpy, immutable) — the reference's container contract
(/root/reference/pkg/src/semidist/sparse.py:56-109):
``CsrMatrix`` with int64 ``indptr``/``indices`` and float64 ``values``, each
row's columns strictly ascending, no stored zeros.  Canonicalisation and the
CSR<->COO conversions are host preconditions of the hot path and stay in
numpy here, as SURVEY.md §2 ("keep in Python") prescribes.

Device side — ``DeviceCsr``: the layout the sm_100a kernels read
(DESIGN.md §3): int64 ``indptr``, int32 ``indices``, float32/float64
``values``, all in HBM as torch tensors (torch is only the allocator).
Every derived per-matrix structure (row statistics, the J-blocked inverted
index) is cached on the ``DeviceCsr`` the same way the reference caches
``coo_row_ids`` on its matrix (sparse.py:78-81).
"""

import ctypes
from dataclasses import dataclass
from enum import Enum
from functools import cached_property
import weakref

import numpy as np

from .errors import IndexOutOfBounds, NegativeOffset, NonMonotonicIndptr


def _ro(arr):
    arr.setflags(write=False)
    return arr


def _as_index(x):
    return np.ascontiguousarray(x, dtype=np.int64)


def _as_value(x):
    return np.ascontiguousarray(x, dtype=np.float64)


_UFUNCS = {"add": 0, "maximum": 1, "minimum": 2, "multiply": 3}   # sd_ufunc


def segment_reduce(values, boundaries, ufunc, identity, *, device=None):
    """Reduce ``values`` over consecutive segments on device (sparse.py:31-53).

    Segment ``t`` covers ``values[boundaries[t]:boundaries[t+1]]``; the
    segments must tile ``values``; empty segments yield ``identity``.  The
    device kernel associates exactly like numpy's ``ufunc.reduceat``
    (``v[0] + pairwise_sum(v[1:])`` for add), so results are bitwise the
    reference's.  Supported ufuncs: add, maximum, minimum, multiply.
    """
    import torch
    from . import _lib
    boundaries = np.asarray(boundaries)
    n_segments = boundaries.size - 1
    result = np.full(max(n_segments, 0), identity, dtype=np.float64)
    if n_segments <= 0:
        return result
    values = np.asarray(values)
    if boundaries[0] != 0 or boundaries[-1] != len(values):
        raise ValueError("segment boundaries must tile the value array")
    if len(values) == 0:
        return result
    code = _UFUNCS.get(getattr(ufunc, "__name__", ""))
    if code is None or not isinstance(ufunc, np.ufunc):
        raise NotImplementedError(f"segment_reduce on device supports {sorted(_UFUNCS)}, not {ufunc!r}")
    if values.dtype != np.float32:
        values = values.astype(np.float64)   # integer / bool sums stay exact below 2**53
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    v = torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    b = torch.from_numpy(np.ascontiguousarray(boundaries, dtype=np.int64)).to(dev)
    out = torch.empty(n_segments, dtype=v.dtype, device=dev)
    _lib.call(dev, "sd_segment_reduce", v.data_ptr(), int(values.size), b.data_ptr(), n_segments,
              _lib.dtype_code(v.dtype), code, float(identity), out.data_ptr(), _lib.stream_handle(dev))
    return out.cpu().numpy().astype(np.float64)


@dataclass(frozen=True, eq=False)
class CsrMatrix:
    """Compressed sparse rows (sparse.py:56-94): row ``i`` stores columns
    ``indices[indptr[i]:indptr[i+1]]`` with the matching ``values``."""

    n_rows: int
    n_cols: int
    indptr: np.ndarray
    indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self):
        return int(self.indptr[-1]) if len(self.indptr) else 0

    @cached_property
    def row_degrees(self):
        return _ro(np.diff(self.indptr))

    @cached_property
    def coo_row_ids(self):
        return _ro(np.repeat(np.arange(self.n_rows, dtype=np.int64), self.row_degrees))

    def row_slice(self, i):
        lo, hi = int(self.indptr[i]), int(self.indptr[i + 1])
        return self.indices[lo:hi], self.values[lo:hi]

    def with_values(self, values):
        values = _as_value(values)
        if values.size != self.indices.size:
            raise ValueError("replacement values must match nnz")
        return CsrMatrix(self.n_rows, self.n_cols, self.indptr, self.indices,
                         _ro(values.copy()))


@dataclass(frozen=True, eq=False)
class CooMatrix:
    """Coordinate view sorted by (row, col) (sparse.py:97-109)."""

    n_rows: int
    n_cols: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    @property
    def nnz(self):
        return int(self.rows.size)


class NormKind(str, Enum):
    """Row statistics of Table 1's "Norm" column (sparse.py:112-116)."""

    L0 = "l0"
    L1 = "l1"
    L2 = "l2"
    L2_SQUARED = "l2sq"


@dataclass(frozen=True, eq=False)
class NormVector:
    kind: NormKind
    values: np.ndarray


@dataclass(frozen=True, eq=False)
class DegreeStats:
    min_degree: int
    max_degree: int
    mean_degree: float
    histogram: np.ndarray


def validate_and_canonicalize(indptr, indices, values, *, n_cols, n_rows=None, device=None):
    """Check a raw CSR triple and return its canonical form (sparse.py:135-202):
    columns sorted per row, duplicates summed, zeros dropped.  Errors name the
    offending row.  Runs on the GPU (sd_canonicalize: validation kernels, CUB
    radix sort, duplicates summed in input order with numpy's reduceat
    association — bitwise the reference's result); returns a host CsrMatrix."""
    import torch
    from . import _lib
    indptr = _as_index(indptr)
    indices = _as_index(indices)
    values = _as_value(values)
    n_rows = indptr.size - 1 if n_rows is None else int(n_rows)
    n_cols = int(n_cols)
    if n_rows < 0 or n_cols < 0:
        raise ValueError("matrix dimensions must be non-negative")
    if indptr.size != n_rows + 1:
        raise ValueError(f"indptr length {indptr.size} does not match {n_rows} rows")
    if indices.size != values.size:
        raise ValueError("indices and values must have equal length")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    nnz = int(indices.size)
    d_ptr = torch.from_numpy(indptr).to(dev)
    d_idx = torch.from_numpy(indices).to(dev) if nnz else None
    d_val = torch.from_numpy(values).to(dev) if nnz else None
    o_ptr = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    o_idx = torch.empty(max(1, nnz), dtype=torch.int64, device=dev)
    o_val = torch.empty(max(1, nnz), dtype=torch.float64, device=dev)
    out_nnz = ctypes.c_int64(0)
    why = _lib.SdInvalid()
    with torch.cuda.device(dev):
        rc = _lib.load().sd_canonicalize(n_rows, n_cols, nnz, d_ptr.data_ptr(),
                                         d_idx.data_ptr() if nnz else None, d_val.data_ptr() if nnz else None,
                                         o_ptr.data_ptr(), o_idx.data_ptr(), o_val.data_ptr(), ctypes.byref(out_nnz),
                                         ctypes.byref(why), _lib.stream_handle(dev))
    if rc == _lib.SD_E_INVALID and why.kind:
        _raise_invalid(why, nnz)
    _lib.check(rc, "sd_canonicalize")
    k = int(out_nnz.value)
    return CsrMatrix(n_rows, n_cols, _ro(o_ptr.cpu().numpy()), _ro(o_idx[:k].cpu().numpy()),
                     _ro(o_val[:k].cpu().numpy()))


def _raise_invalid(why, nnz):
    """sd_invalid -> the reference's exception (sparse.py:148-170)."""
    kind = int(why.kind)
    if kind == 1:
        raise NegativeOffset(row=int(why.row), offset=int(why.value))
    if kind == 2:
        raise NonMonotonicIndptr(0, f"indptr[0] is {int(why.value)}, expected 0")
    if kind == 3:
        raise NonMonotonicIndptr(int(why.row), f"indptr decreases at row {int(why.row)}")
    if kind == 4:
        raise ValueError(f"indptr[-1] = {int(why.value)} but {nnz} entries supplied")
    raise IndexOutOfBounds(row=int(why.row), column=int(why.column), n_cols=int(why.value))


def canonicalize_host(indptr, indices, values, *, n_cols, n_rows=None):
    """validate_and_canonicalize evaluated with numpy on the host: for CPU-only
    tooling (data preparation without a GPU) and as the device version's
    parity reference in tests/test_gpu_boundary.py."""
    indptr = _as_index(indptr)
    indices = _as_index(indices)
    values = _as_value(values)
    n_rows = indptr.size - 1 if n_rows is None else int(n_rows)
    n_cols = int(n_cols)
    if n_rows < 0 or n_cols < 0:
        raise ValueError("matrix dimensions must be non-negative")
    if indptr.size != n_rows + 1:
        raise ValueError(f"indptr length {indptr.size} does not match {n_rows} rows")
    if indices.size != values.size:
        raise ValueError("indices and values must have equal length")
    bad = np.flatnonzero(indptr < 0)
    if bad.size:
        pos = int(bad[0])
        raise NegativeOffset(row=max(0, min(pos, n_rows - 1)), offset=int(indptr[pos]))
    if indptr[0] != 0:
        raise NonMonotonicIndptr(0, f"indptr[0] is {int(indptr[0])}, expected 0")
    deg = np.diff(indptr)
    bad = np.flatnonzero(deg < 0)
    if bad.size:
        row = int(bad[0])
        raise NonMonotonicIndptr(row, f"indptr decreases at row {row}")
    if int(indptr[-1]) != indices.size:
        raise ValueError(f"indptr[-1] = {int(indptr[-1])} but {indices.size} entries supplied")
    bad = np.flatnonzero((indices < 0) | (indices >= n_cols))
    if bad.size:
        pos = int(bad[0])
        row = int(np.searchsorted(indptr, pos, side="right") - 1)
        raise IndexOutOfBounds(row=row, column=int(indices[pos]), n_cols=n_cols)

    rows = np.repeat(np.arange(n_rows, dtype=np.int64), deg)
    key = rows * max(1, n_cols) + indices
    order = np.argsort(key, kind="stable")
    key, vals = key[order], values[order]
    if key.size:
        first = np.ones(key.size, dtype=bool)
        first[1:] = key[1:] != key[:-1]
        starts = np.flatnonzero(first)
        vals = np.add.reduceat(vals, starts)
        key = key[first]
        keep = vals != 0.0
        key, vals = key[keep], vals[keep]
    rows = key // max(1, n_cols)
    cols = key - rows * max(1, n_cols)
    out_ptr = np.zeros(n_rows + 1, dtype=np.int64)
    if rows.size:
        np.cumsum(np.bincount(rows, minlength=n_rows), out=out_ptr[1:])
    return CsrMatrix(n_rows, n_cols, _ro(out_ptr), _ro(cols.astype(np.int64)),
                     _ro(vals.astype(np.float64)))


def from_dense(dense):
    """Sparsify a 2-D array; zeros become structurally absent (sparse.py:205-217)."""
    dense = np.asarray(dense, dtype=np.float64)
    if dense.ndim != 2:
        raise ValueError("expected a 2-D array")
    r, c = np.nonzero(dense)
    ptr = np.zeros(dense.shape[0] + 1, dtype=np.int64)
    if r.size:
        np.cumsum(np.bincount(r, minlength=dense.shape[0]), out=ptr[1:])
    return CsrMatrix(dense.shape[0], dense.shape[1], _ro(ptr),
                     _ro(c.astype(np.int64)), _ro(dense[r, c].astype(np.float64)))


def csr_to_coo(m):
    """CSR -> COO row expansion (sparse.py:220-225)."""
    return CooMatrix(m.n_rows, m.n_cols, _ro(np.array(m.coo_row_ids, copy=True)),
                     _ro(np.array(m.indices, dtype=np.int64, copy=True)),
                     _ro(np.array(m.values, dtype=np.float64, copy=True)))


def coo_to_csr(coo):
    """Canonical COO -> CSR (sparse.py:228-244)."""
    rows, cols, vals = _as_index(coo.rows), _as_index(coo.cols), _as_value(coo.values)
    if rows.size:
        if (cols < 0).any() or (cols >= coo.n_cols).any() or \
           (rows < 0).any() or (rows >= coo.n_rows).any():
            raise ValueError("coordinate ids out of bounds")
        if (np.diff(rows * coo.n_cols + cols) <= 0).any():
            raise ValueError("coordinates must be sorted by (row, col) without duplicates")
    ptr = np.zeros(coo.n_rows + 1, dtype=np.int64)
    if rows.size:
        np.cumsum(np.bincount(rows, minlength=coo.n_rows), out=ptr[1:])
    return CsrMatrix(coo.n_rows, coo.n_cols, _ro(ptr), _ro(cols.copy()), _ro(vals.copy()))


def slice_rows(m, start, stop):
    """Rows [start, stop) sharing storage (sparse.py:247-254)."""
    if not (0 <= start <= stop <= m.n_rows):
        raise ValueError(f"invalid row range [{start}, {stop}) for {m.n_rows} rows")
    lo, hi = int(m.indptr[start]), int(m.indptr[stop])
    ptr = (np.asarray(m.indptr[start:stop + 1]) - lo).astype(np.int64)
    return CsrMatrix(stop - start, m.n_cols, _ro(ptr), m.indices[lo:hi], m.values[lo:hi])


def degree_stats(m):
    """Exact row-degree statistics (sparse.py:276-286)."""
    deg = np.diff(np.asarray(m.indptr))
    if deg.size == 0:
        return DegreeStats(0, 0, 0.0, _ro(np.zeros(1, dtype=np.int64)))
    return DegreeStats(int(deg.min()), int(deg.max()), float(deg.mean()),
                       _ro(np.bincount(deg)))


# --------------------------------------------------------------------------
# device mirror
# --------------------------------------------------------------------------

class DeviceCsr:
    """A CSR matrix resident in HBM, laid out for the kernels.

    ``indptr`` int64[n_rows+1], ``indices`` int32[nnz], ``values`` T[nnz]
    (T = float32 or float64).  Holds a per-matrix cache of derived device
    structures (row statistics by kind, the inverted index) so repeated
    queries against one index pay for them once.
    """

    def __init__(self, n_rows, n_cols, indptr, indices, values, row_offset=0):
        import torch
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.indptr = indptr
        self.indices = indices
        self.values = values
        self.row_offset = int(row_offset)
        if indptr.dtype != torch.int64 or indices.dtype != torch.int32:
            raise ValueError("DeviceCsr needs int64 indptr and int32 indices")
        if values.dtype not in (torch.float32, torch.float64):
            raise ValueError("DeviceCsr values must be float32 or float64")
        self.cache = {}
        self._host_degrees = None
        self.transform = None   # value transform these values already carry ("sqrt" for hellinger)

    @property
    def device(self):
        return self.values.device

    @property
    def dtype(self):
        return self.values.dtype

    @property
    def nnz(self):
        return int(self.indices.numel())

    def host_degrees(self):
        if self._host_degrees is None:
            self._host_degrees = np.diff(self.indptr.cpu().numpy())
        return self._host_degrees

    def slice_rows(self, start, stop):
        """Row range as a DeviceCsr view: indptr is rebased on device, columns and
        values are shared (no copy)."""
        if not (0 <= start <= stop <= self.n_rows):
            raise ValueError(f"invalid row range [{start}, {stop}) for {self.n_rows} rows")
        ptr = self.indptr[start:stop + 1]
        lo = int(ptr[0].item()) if stop >= start else 0
        hi = int(ptr[-1].item())
        sub = DeviceCsr(stop - start, self.n_cols, (ptr - lo).contiguous(),
                        self.indices[lo:hi], self.values[lo:hi],
                        row_offset=self.row_offset + start)
        if self._host_degrees is not None:
            sub._host_degrees = self._host_degrees[start:stop]
        sub.transform = self.transform
        return sub


_DEVICE_CACHE = weakref.WeakKeyDictionary()


def to_device(m, dtype="float64", device=None, transform=None):
    """Upload a host CSR (ours or the reference's, duck-typed) once per
    (dtype, device, transform); later calls return the cached DeviceCsr.

    ``transform`` names a value transform applied on device after upload
    ("sqrt" for Hellinger, metrics.py:205-207)."""
    import torch
    if isinstance(m, DeviceCsr):
        tdtype = _torch_dtype(dtype)
        if m.dtype != tdtype:   # compute dtype differs from the stored one: a converted copy, cached
            key = ("dtype", tdtype)
            conv = m.cache.get(key)
            if conv is None:
                conv = DeviceCsr(m.n_rows, m.n_cols, m.indptr, m.indices, m.values.to(tdtype),
                                 row_offset=m.row_offset)
                conv._host_degrees = m._host_degrees
                conv.transform = m.transform
                m.cache[key] = conv
            m = conv
        if transform is None or m.transform == transform:
            return m
        if m.transform is not None:
            raise ValueError(f"matrix already carries value transform {m.transform!r}")
        key = ("transform", transform)
        hit = m.cache.get(key)
        if hit is None:
            hit = _transformed(m, transform)
            m.cache[key] = hit
        return hit
    tdtype = _torch_dtype(dtype)
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    key = (tdtype, str(dev), transform)
    try:
        per = _DEVICE_CACHE.setdefault(m, {})
    except TypeError:
        per = {}
    hit = per.get(key)
    if hit is not None:
        return hit
    indptr = np.ascontiguousarray(m.indptr, dtype=np.int64)
    indices = np.asarray(m.indices)
    if indices.size and (int(indices.max()) >= 2 ** 31 or int(m.n_cols) >= 2 ** 31):
        raise ValueError("column ids must fit in int32 on device")
    d = DeviceCsr(
        int(m.n_rows), int(m.n_cols),
        torch.from_numpy(np.array(indptr, dtype=np.int64, copy=True)).to(dev),
        torch.from_numpy(np.array(indices, dtype=np.int32, copy=True)).to(dev),
        torch.from_numpy(np.array(m.values, dtype=np.float64, copy=True)).to(dev).to(tdtype),
    )
    d._host_degrees = np.diff(indptr)
    if transform is not None:
        d = _transformed(d, transform)
    per[key] = d
    return d


def _transformed(d, transform):
    """Value transform of a DeviceCsr on device, after the domain check on the
    raw values (metrics.py:308-311, 332-338)."""
    from . import _lib
    from .errors import DomainError
    if _lib.any_negative(d):
        raise DomainError("hellinger requires non-negative inputs")
    return _lib.transform_values(d, transform)


def _torch_dtype(dtype):
    import torch
    if dtype in (torch.float32, torch.float64):
        return dtype
    name = np.dtype(dtype).name
    if name == "float32":
        return torch.float32
    if name == "float64":
        return torch.float64
    raise ValueError(f"unsupported value dtype {dtype!r}; use float32 or float64")


def upload(n_rows, n_cols, indptr, indices, values, *, device=None, non_blocking=True):
    """DeviceCsr from host arrays (numpy or CPU torch tensors; pinned tensors
    make the H2D copies asynchronous).  ``values``' dtype (float32/float64)
    is the compute dtype."""
    import torch

    def dev_tensor(x, dt):
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        if t.dtype != dt:
            t = t.to(dt)
        return t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()),
                    non_blocking=non_blocking and t.is_pinned())

    vt = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(values))
    if vt.dtype not in (torch.float32, torch.float64):
        vt = vt.to(torch.float64)
    d = DeviceCsr(int(n_rows), int(n_cols), dev_tensor(indptr, torch.int64), dev_tensor(indices, torch.int32),
                  dev_tensor(vt, vt.dtype))
    host_ptr = indptr.numpy() if isinstance(indptr, torch.Tensor) else np.asarray(indptr)
    d._host_degrees = np.diff(host_ptr.astype(np.int64))
    return d
