"""CPU: the C-ABI library loads and exports every symbol include/*.h declares
(no compute calls without a GPU); the ctypes structs match the header."""

from __future__ import annotations

import ctypes
import os
import re

import pytest

from conftest import ROOT


def header_functions():
    names = []
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            src = open(os.path.join(inc, f)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names += re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(wm_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_abi():
    assert set(header_functions()) >= {"wm_graph_create", "wm_graph_create_device", "wm_run",
                                       "wm_graph_destroy", "wm_last_error", "wm_abi_version"}


def test_library_exports_every_declared_symbol():
    from paper_2212_04551_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        from paper_2212_04551_b200 import build
        build.build()
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in header_functions():
        assert hasattr(lib, name), name
    L = _native.load()
    assert L.wm_abi_version() == _native.ABI_VERSION == 2
    assert L.wm_last_error() == b""


def test_reduce_vector_layout():
    """wm_reduce_words and the WM_RED_* constants agree between header and
    binding (host-only call, no device work)."""
    from paper_2212_04551_b200 import _native
    src = open(os.path.join(ROOT, "include", "warpmine_b200.h")).read()
    consts = dict((k, int(v)) for k, v in re.findall(r"#define (WM_RED_\w+) (\d+)", src))
    for k, v in consts.items():
        assert getattr(_native, k) == v, k
    L = _native.load()
    assert L.wm_reduce_words(0, 1) == consts["WM_RED_HIST"] + consts["WM_RED_SLOT_WORDS"]
    assert L.wm_reduce_words(853, 8) == consts["WM_RED_HIST"] + 853 + 8 * consts["WM_RED_SLOT_WORDS"]


def test_struct_layouts_match_header():
    """Field order of the ctypes mirrors equals the C structs' declaration order."""
    from paper_2212_04551_b200 import _native
    src = open(os.path.join(ROOT, "include", "warpmine_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    for cname, py in (("wm_csr", _native.WmCsr), ("wm_app", _native.WmApp),
                      ("wm_cfg", _native.WmCfg), ("wm_result", _native.WmResult),
                      ("wm_listing", _native.WmListing), ("wm_csr_out", _native.WmCsrOut)):
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + cname + ";", src).group(1)
        fields = []
        for decl in body.split(";"):
            decl = re.sub(r"//.*", "", decl).strip()
            if not decl:
                continue
            for part in re.split(r",", decl):
                fields.append(re.findall(r"\**(\w+)\s*$", part.strip())[0])
        assert [f[0] for f in py._fields_] == fields, cname


def test_status_mapping():
    from paper_2212_04551_b200 import _native
    from paper_2212_04551_b200.errors import CapacityError, DeviceError, InternalInvariantError
    _native.load()
    for code, exc in ((_native.WM_EINVAL, ValueError), (_native.WM_ECAPACITY, CapacityError),
                      (_native.WM_EINVARIANT, InternalInvariantError),
                      (_native.WM_ECUDA, DeviceError)):
        with pytest.raises(exc):
            _native.check(code)
    from paper_2212_04551_b200.errors import GraphParseError, StoreShutdownError
    for code, exc in ((_native.WM_ESHUTDOWN, StoreShutdownError),
                      (_native.WM_EPARSE, GraphParseError)):
        with pytest.raises(exc):
            _native.check(code)
    _native.check(_native.WM_OK)
