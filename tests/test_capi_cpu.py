"""The C-ABI libraries load on a GPU-less host and export every symbol include/*.h declares.
No compute calls (there is no GPU here); argument validation paths that fail before touching
the device are exercised."""

import ctypes
import os
import re

import pytest

from paper_2605_08639_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mbp?_[a-z0-9_]+)\s*\(", text)))


@pytest.mark.parametrize("header,loader", [("mb_kernels.h", _native.kernels), ("mb_planner.h", _native.planner)])
def test_every_declared_symbol_is_exported(header, loader):
    lib = loader()
    names = declared(header)
    assert len(names) >= 8
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_signatures_cover_headers():
    for header, sigs in (("mb_kernels.h", _native._KERNEL_SIGS), ("mb_planner.h", _native._PLANNER_SIGS)):
        assert set(declared(header)) <= set(sigs), set(declared(header)) - set(sigs)


def test_argument_errors_without_gpu():
    lib = _native.kernels()
    assert lib.mb_version() == 1
    # invalid shapes are rejected before any CUDA call
    rc = lib.mb_expert_histogram(None, 1, 10, 0, 8, None, None, 32, None)
    assert rc == 1 and b"bad histogram shape" in lib.mb_last_error()
    rc = lib.mb_grouped_gemm(0, None, 0, 0, None, 0, None, 0, 0, None, None, 1, 0, 256, 64, None, 0, 0, None, 0,
                             None, 0, None, None, 0, None)
    assert rc == 1
    p = _native.planner()
    out = (ctypes.c_int64 * 3)()
    assert p.mbp_static_plan(3, 2, out) == 1
    assert b"not divisible" in p.mbp_last_error()


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "LIB_DIR", tmp_path)
    monkeypatch.setattr(_native, "_libs", {})
    with pytest.raises(_native.NativeLibraryError):
        _native.kernels()
