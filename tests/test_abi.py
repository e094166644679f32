"""The C-ABI library loads on a CPU-only host and exports exactly what
include/semidist_b200.h declares (no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

from paper_2104_06357_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "semidist_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^SD_API\s+[\w\s\*]+?\b(sd_\w+)\(", text, flags=re.M)))


def test_header_declares_entry_points():
    syms = header_symbols()
    assert "sd_pairwise" in syms and "sd_knn" in syms and "sd_pass" in syms
    assert len(syms) >= 18


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in header_symbols():
        assert hasattr(lib, name), name


def test_binding_table_matches_header():
    assert sorted(_lib.exported_symbols()) == header_symbols()


def test_version_and_error_calls_without_gpu():
    lib = _lib.load()
    assert lib.sd_version() == 1
    assert isinstance(lib.sd_last_error(), bytes)


def test_invalid_arguments_rejected_before_device_work():
    """Dimension / argument checks happen on the host side of the ABI."""
    lib = _lib.load()
    a = _lib.SdCsr(1, 3, 0, None, None, None)
    b = _lib.SdCsr(1, 4, 0, None, None, None)
    md = _lib.metric_struct("cosine")
    rc = lib.sd_pairwise(ctypes.byref(a), ctypes.byref(b), None, 0, ctypes.byref(md), None, None, 1,
                         None, None, None, None)
    assert rc in (_lib.SD_E_DIM, _lib.SD_E_INVALID)
    md = _lib.metric_struct("minkowski", p=0.5)
    rc = lib.sd_pairwise(ctypes.byref(a), ctypes.byref(a), None, 0, ctypes.byref(md), None, None, 1,
                         None, None, None, None)
    assert rc in (_lib.SD_E_DOMAIN_PARAM, _lib.SD_E_INVALID)
    with pytest.raises(Exception):
        _lib.check(_lib.SD_E_DIM)


def test_status_mapping():
    from paper_2104_06357_b200.errors import DimensionMismatch, DomainError, KTooLarge
    for code, exc in [(_lib.SD_E_DIM, DimensionMismatch), (_lib.SD_E_DOMAIN_RADICAND, DomainError),
                      (_lib.SD_E_K_TOO_LARGE, KTooLarge), (_lib.SD_E_INVALID, ValueError),
                      (_lib.SD_E_UNSUPPORTED, NotImplementedError), (_lib.SD_E_CUDA, RuntimeError)]:
        with pytest.raises(exc):
            _lib.check(code)


def test_sass_is_sm100a():
    """The shipped cubin targets sm_100a (checked with cuobjdump when present)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
