"""ctypes binding of libsemidist_b200.so (include/semidist_b200.h).

This is the whole boundary between the Python mirror of the reference API
and the sm_100a kernels: device pointers (from torch tensors, used purely as
HBM allocations), sizes and the current CUDA stream go in; an integer status
comes back and is mapped onto the reference's exception classes
(/root/reference/pkg/src/semidist/errors.py).  There is no CPU fallback: if
the shared library is missing, every entry point raises.
"""

import ctypes
import os

import numpy as np

from .errors import DimensionMismatch, DomainError, KTooLarge

LIB_PATH = os.environ.get("SD_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "libsemidist_b200.so")

# sd_status (include/semidist_b200.h)
SD_OK, SD_E_DIM, SD_E_DOMAIN_NEG, SD_E_DOMAIN_RADICAND, SD_E_KL_UNCOVERED = 0, 1, 2, 3, 4
SD_E_K_TOO_LARGE, SD_E_INVALID, SD_E_UNSUPPORTED, SD_E_CUDA, SD_E_DOMAIN_PARAM = 5, 6, 7, 8, 9
SD_F32, SD_F64 = 0, 1
SD_FLAG_RADICAND, SD_FLAG_KL_UNCOVERED, SD_FLAG_NEGATIVE = 0x1, 0x2, 0x4
STRAT_NAIVE, STRAT_DENSE, STRAT_HASH, STRAT_AUTO = 0, 1, 2, 3
STAT_L0, STAT_L1, STAT_L2, STAT_L2SQ, STAT_SUM = 0, 1, 2, 3, 4

SEMIRING_IDS = {
    "dot": 0, "min-plus": 1, "abs-diff": 2, "abs-diff-pow": 3, "abs-diff-max": 4,
    "canberra-ratio": 5, "mismatch": 6, "jensen-shannon-term": 7, "kl-term": 8,
    "miss-count": 9,
}

METRIC_IDS = {
    "correlation": 0, "cosine": 1, "dice": 2, "dot": 3, "euclidean": 4, "hellinger": 5,
    "jaccard": 6, "kl": 7, "russelrao": 8, "canberra": 9, "chebyshev": 10, "hamming": 11,
    "jensenshannon": 12, "manhattan": 13, "minkowski": 14,
}


class SdCsr(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("indptr", ctypes.c_void_p), ("indices", ctypes.c_void_p), ("values", ctypes.c_void_p)]


class SdStrategy(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("accumulator_capacity", ctypes.c_int32),
                ("max_load_factor", ctypes.c_double)]


class SdReport(ctypes.Structure):
    _fields_ = [("peak_accumulator_entries", ctypes.c_int64), ("workspace_elements", ctypes.c_int64),
                ("chunks_executed", ctypes.c_int64)]


class SdMetricDesc(ctypes.Structure):
    _fields_ = [("metric", ctypes.c_int32), ("strict", ctypes.c_int32), ("p", ctypes.c_double),
                ("pre_transformed", ctypes.c_int32), ("stages", ctypes.c_int32)]


class SdInvalid(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad", ctypes.c_int32), ("row", ctypes.c_int64),
                ("column", ctypes.c_int64), ("value", ctypes.c_int64)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_CSR = ctypes.POINTER(SdCsr)

# (name, restype, argtypes) — exactly the declarations of include/semidist_b200.h
SIGNATURES = [
    ("sd_version", _I, []),
    ("sd_tune", _I, [_I, _I64, ctypes.POINTER(_I64)]),
    ("sd_last_error", ctypes.c_char_p, []),
    ("sd_launch_count", ctypes.c_uint64, []),
    ("sd_smem_budget", _I, [_I, ctypes.POINTER(_I64)]),
    ("sd_row_stat", _I, [_CSR, _I, _I, _P, _P]),
    ("sd_csr_to_coo", _I, [_CSR, _P, _P]),
    ("sd_check_nonnegative", _I, [_CSR, _I, _P, _P]),
    ("sd_sqrt_values", _I, [_CSR, _I, _P, _P]),
    ("sd_fill", _I, [_P, _I64, _I64, _I64, _I, _D, _P]),
    ("sd_pass", _I, [_CSR, _CSR, _I, _I, _D, _I, ctypes.POINTER(SdStrategy), _P, _I64,
                     ctypes.POINTER(SdReport), _P]),
    ("sd_index_build", _I, [_CSR, _I, _I, ctypes.POINTER(_P), _P]),
    ("sd_index_free", _I, [_P]),
    ("sd_index_bytes", _I64, [_P]),
    ("sd_index_tile_rows", _I, [_P]),
    ("sd_index_heavy_rows", _I64, [_P]),
    ("sd_index_hybrid_blocks", _I, [_P]),
    ("sd_pairwise", _I, [_CSR, _CSR, _P, _I, ctypes.POINTER(SdMetricDesc), ctypes.POINTER(SdStrategy),
                         _P, _I64, _P, ctypes.POINTER(SdReport), ctypes.POINTER(ctypes.c_float), _P]),
    ("sd_expand", _I, [_P, _I64, _I64, _I64, _I, ctypes.POINTER(SdMetricDesc), _I64,
                       ctypes.POINTER(_P), ctypes.POINTER(_P), _P, _P]),
    ("sd_knn", _I, [_CSR, _CSR, _P, _I, ctypes.POINTER(SdMetricDesc), _I, _I64, _P, _P, _P, _P]),
    ("sd_topk_rows", _I, [_P, _I64, _I64, _I64, _I, _I, _I64, _P, _P, _P]),
    ("sd_topk_merge", _I, [_P, _P, _I64, _I, _I, _I, _P, _P, _P]),
    ("sd_segment_reduce", _I, [_P, _I64, _P, _I64, _I, _I, _D, _P, _P]),
    ("sd_mix32", _I, [_P, _I64, _P, _P]),
    ("sd_hash_build", _I, [_P, _P, _I64, _I64, _P, _P, _P]),
    ("sd_hash_probe", _I, [_P, _P, _I64, _P, _I64, _P, _P, _P]),
    ("sd_semiring_apply", _I, [_I, _D, _P, _P, _I64, _P, _P]),
    ("sd_dense_pairwise", _I, [_P, _P, _I64, _I64, _I64, ctypes.POINTER(SdMetricDesc), _P, _P, _P]),
    ("sd_canonicalize", _I, [_I64, _I64, _I64, _P, _P, _P, _P, _P, _P, ctypes.POINTER(_I64),
                             ctypes.POINTER(SdInvalid), _P]),
]

TUNE_KNOBS = {
    "tile": 0, "isect_plan": 1, "cos_raw": 2, "isect_debug": 3, "isect_band": 4, "isect_l2_div": 5,
    "heavy_deg": 6, "hybrid": 7, "hybrid_max_mb": 8, "hybrid_max_queries": 9, "hgemm": 10,
    "dense": 11, "dense_max_mb": 12, "gather_shadow": 13, "gather_blocks": 14,
}

_LIB = None


def load():
    """Load the shared library once; raise loudly if it was not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2104_06357_b200.build` "
                "(there is no CPU fallback for the distance kernels)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def tune(name, value):
    """Set a tuning knob (include/semidist_b200.h sd_tune_knob); returns the previous value."""
    prev = ctypes.c_int64()
    check(load().sd_tune(TUNE_KNOBS[name], int(value), ctypes.byref(prev)), "sd_tune")
    return int(prev.value)


class tuned:
    """Context manager: ``with tuned(hybrid=2): ...`` restores the knobs on exit."""

    def __init__(self, **knobs):
        self.knobs = knobs
        self.saved = {}

    def __enter__(self):
        for name, value in self.knobs.items():
            self.saved[name] = tune(name, value)
        return self

    def __exit__(self, *exc):
        for name, value in self.saved.items():
            tune(name, value)
        return False


def last_error():
    return load().sd_last_error().decode(errors="replace")


def check(status, what=""):
    """Map an sd_status onto the reference's exception classes."""
    if status == SD_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == SD_E_DIM:
        raise DimensionMismatch(msg)
    if status in (SD_E_DOMAIN_NEG, SD_E_DOMAIN_RADICAND, SD_E_KL_UNCOVERED, SD_E_DOMAIN_PARAM):
        raise DomainError(msg)
    if status == SD_E_K_TOO_LARGE:
        raise KTooLarge(msg)
    if status == SD_E_INVALID:
        raise ValueError(msg)
    if status == SD_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"libsemidist_b200 status {status}: {msg}")


def call(device, name, *args):
    """Run C entry point ``name`` with ``device`` current (the library takes the
    SM count, shared-memory limit and side streams from the current device, and
    a launch into another device's stream fails) and map its status."""
    import torch
    fn = getattr(load(), name)
    if device is None:
        return check(fn(*args), name)
    with torch.cuda.device(device):
        return check(fn(*args), name)


def raise_flags(flags, metric_name=""):
    """Device flag word (SD_FLAG_*) -> the DomainError the reference raises."""
    if flags & SD_FLAG_NEGATIVE:
        raise DomainError(f"{metric_name} requires non-negative inputs")
    if flags & SD_FLAG_KL_UNCOVERED:
        raise DomainError("kl: some row pairs have query support not covered by the reference row")
    if flags & SD_FLAG_RADICAND:
        raise DomainError(f"{metric_name}: negative radicand beyond rounding tolerance")


# --------------------------------------------------------------- helpers

def dtype_code(tdtype):
    import torch
    if tdtype == torch.float32:
        return SD_F32
    if tdtype == torch.float64:
        return SD_F64
    raise ValueError(f"unsupported dtype {tdtype}")


def csr_struct(d):
    """SdCsr view of a DeviceCsr (no copies)."""
    return SdCsr(d.n_rows, d.n_cols, d.nnz, d.indptr.data_ptr(),
                 d.indices.data_ptr() if d.nnz else 0, d.values.data_ptr() if d.nnz else 0)


def stream_handle(device=None):
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def strategy_struct(kind, capacity=0, load=0.5):
    return SdStrategy(int(kind), int(capacity), float(load))


def metric_struct(name, p=None, strict=True, pre_transformed=False, stages=0):
    return SdMetricDesc(METRIC_IDS[name], 1 if strict else 0, float(p) if p is not None else 0.0,
                        1 if pre_transformed else 0, int(stages))


def new_flags(device):
    import torch
    return torch.zeros(1, dtype=torch.int32, device=device)


def any_negative(d):
    """True if any stored value of a DeviceCsr is negative (one 4-byte D2H)."""
    flags = new_flags(d.device)
    csr = csr_struct(d)
    call(d.device, "sd_check_nonnegative", ctypes.byref(csr), dtype_code(d.dtype), flags.data_ptr(),
         stream_handle(d.device))
    return bool(int(flags.item()) & SD_FLAG_NEGATIVE)


def transform_values(d, transform):
    """A DeviceCsr whose values carry a metric value transform (only "sqrt")."""
    import torch
    from .sparse import DeviceCsr
    if transform != "sqrt":
        raise ValueError(f"unknown value transform {transform!r}")
    out = torch.empty_like(d.values)
    csr = csr_struct(d)
    call(d.device, "sd_sqrt_values", ctypes.byref(csr), dtype_code(d.dtype), out.data_ptr() if d.nnz else None,
         stream_handle(d.device))
    t = DeviceCsr(d.n_rows, d.n_cols, d.indptr, d.indices, out, row_offset=d.row_offset)
    t._host_degrees = d._host_degrees
    t.transform = transform
    return t


class DeviceIndex:
    """Owner of an sd_index handle (the J-blocked inverted index of B)."""

    def __init__(self, dcsr):
        lib = load()
        handle = ctypes.c_void_p()
        csr = csr_struct(dcsr)
        call(dcsr.device, "sd_index_build", ctypes.byref(csr), dtype_code(dcsr.dtype), 0, ctypes.byref(handle),
             stream_handle(dcsr.device))
        self.handle = handle
        self.n_rows = dcsr.n_rows
        self.tile_rows = int(lib.sd_index_tile_rows(handle))

    @property
    def bytes(self):
        """Device memory held by the index (grows when the lazily built parts —
        cosine postings, chebyshev masks, hybrid block — are first needed)."""
        return int(load().sd_index_bytes(self.handle))

    @property
    def heavy_rows(self):
        """Index rows of the hybrid heavy block (0 until the first dot-family call)."""
        return int(load().sd_index_heavy_rows(self.handle))

    @property
    def hybrid_blocks(self):
        """Dense blocks built so far: subset of {"dot", "minsum"} (hybrid
        heavy-row blocks) and {"dense", "dense_two_planes", "dense_ints"}
        (dense-index mode image)."""
        bits = int(load().sd_index_hybrid_blocks(self.handle))
        return {n for b, n in ((1, "dot"), (2, "minsum"), (4, "dense"), (8, "dense_two_planes"),
                               (16, "dense_ints")) if bits & b}

    def __del__(self):
        try:
            if self.handle:
                load().sd_index_free(self.handle)
                self.handle = None
        except Exception:
            pass


def device_index(dcsr):
    """Inverted index of a DeviceCsr, cached on it (built once per index matrix)."""
    ix = dcsr.cache.get("index")
    if ix is None:
        ix = DeviceIndex(dcsr)
        dcsr.cache["index"] = ix
    return ix


def row_stat(dcsr, kind):
    import torch
    out = torch.empty(dcsr.n_rows, dtype=dcsr.dtype, device=dcsr.device)
    csr = csr_struct(dcsr)
    call(dcsr.device, "sd_row_stat", ctypes.byref(csr), dtype_code(dcsr.dtype), int(kind), out.data_ptr(),
         stream_handle(dcsr.device))
    return out


def coo_rows(dcsr):
    import torch
    out = torch.empty(dcsr.nnz, dtype=torch.int64, device=dcsr.device)
    csr = csr_struct(dcsr)
    call(dcsr.device, "sd_csr_to_coo", ctypes.byref(csr), out.data_ptr() if dcsr.nnz else None,
         stream_handle(dcsr.device))
    return out


def exported_symbols():
    return [name for name, _, _ in SIGNATURES]


def as_numpy_f64(t):
    return np.ascontiguousarray(t.detach().to("cpu").numpy(), dtype=np.float64)
