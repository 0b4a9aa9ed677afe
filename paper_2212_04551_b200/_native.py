"""ctypes binding of ``libwm_b200.so`` (C-ABI in ``include/warpmine_b200.h``).

The library is built in-tree by ``paper_2212_04551_b200.build.build()``.
There is no fallback: if the shared object is missing or a call fails, an
exception is raised.  Status codes map onto the reference's exception
taxonomy (``pkg/src/warpmine/errors.py:4-31``).
"""

from __future__ import annotations

import ctypes
import os

from .errors import (CapacityError, DeviceError, GraphParseError, InternalInvariantError,
                     StoreShutdownError)

_HERE = os.path.dirname(os.path.abspath(__file__))
# WM_B200_LIB selects an alternative in-tree build (A/B kernel variants)
LIB_PATH = os.environ.get("WM_B200_LIB") or os.path.join(_HERE, "libwm_b200.so")

WM_OK, WM_EINVAL, WM_ECAPACITY, WM_EINVARIANT, WM_ECUDA, WM_ESHUTDOWN, WM_EPARSE = \
    0, -1, -2, -3, -4, -5, -6
WM_F_LOWER, WM_F_COMPACT, WM_F_CLIQUE, WM_F_CANONICAL = 1, 2, 4, 8
WM_AGG_COUNTER, WM_AGG_PATTERN, WM_AGG_STORE = 0, 1, 2
WM_LIST_ALL, WM_LIST_COMPLETE = 0, 1
WM_MODE_WC, WM_MODE_OPT, WM_MODE_DFS = 1, 2, 3
WM_ORDER_ID, WM_ORDER_DEGREE = 0, 1

EXPORTED = ("wm_graph_create", "wm_graph_create_device", "wm_run", "wm_run_listing",
            "wm_graph_destroy", "wm_last_error", "wm_abi_version", "wm_csr_build",
            "wm_edge_list_parse", "wm_csr_free", "wm_dictionary_build", "wm_reduce_words")
ABI_VERSION = 2
# device result vector layout (wm_cfg.reduce_out, include/warpmine_b200.h)
WM_RED_CLIQUES, WM_RED_LEAVES, WM_RED_ALG_BYTES, WM_RED_MIGRATIONS, WM_RED_DONATIONS, \
    WM_RED_TASKS, WM_RED_RECORDS, WM_RED_CHECKSUM, WM_RED_HIST = range(9)
WM_RED_SLOT_WORDS = 4


class WmCsr(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("offsets", ctypes.POINTER(ctypes.c_int64)),
                ("neighbors", ctypes.POINTER(ctypes.c_int32))]


class WmApp(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int), ("extend_all", ctypes.c_int), ("genedges", ctypes.c_int),
                ("aggregator", ctypes.c_int), ("filters", ctypes.c_uint32),
                ("dict_table", ctypes.POINTER(ctypes.c_uint32)), ("dict_len", ctypes.c_uint64),
                ("pattern_count", ctypes.c_uint32), ("dict_device", ctypes.c_void_p),
                ("dict_device_bits", ctypes.c_uint32)]


class WmCfg(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("lb_threshold", ctypes.c_double),
                ("lb_poll", ctypes.c_int), ("root_begin", ctypes.c_int64),
                ("root_end", ctypes.c_int64), ("shard_rank", ctypes.c_int),
                ("shard_count", ctypes.c_int), ("order", ctypes.c_int),
                ("count_bytes", ctypes.c_int), ("warps_per_block", ctypes.c_int),
                ("blocks_per_sm", ctypes.c_int), ("stream", ctypes.c_void_p),
                ("reduce_out", ctypes.c_void_p)]


class WmResult(ctypes.Structure):
    _fields_ = [("clique_count", ctypes.c_uint64), ("leaves", ctypes.c_uint64),
                ("alg_bytes", ctypes.c_uint64), ("rebalance_count", ctypes.c_uint64),
                ("migrations", ctypes.c_uint64), ("peak_ext", ctypes.c_uint64),
                ("pattern_counts", ctypes.POINTER(ctypes.c_uint64)),
                ("tasks", ctypes.c_uint64), ("launches", ctypes.c_uint64),
                ("nodes", ctypes.c_uint64), ("polls", ctypes.c_uint64),
                ("h2d_bytes", ctypes.c_uint64), ("d2h_bytes", ctypes.c_uint64),
                ("kernel_ms", ctypes.c_double), ("build_ms", ctypes.c_double),
                ("device_ms", ctypes.c_double),
                ("idle_warp_fraction", ctypes.c_double),
                ("idle_warp_fraction_tail", ctypes.c_double),
                ("warps", ctypes.c_int), ("bucket_words", ctypes.c_int)]


# int (*wm_sink_fn)(void *user, const uint32_t *records, uint64_t count, uint32_t stride)
SINK_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint32),
                           ctypes.c_uint64, ctypes.c_uint32)


class WmListing(ctypes.Structure):
    _fields_ = [("capacity", ctypes.c_uint32), ("filter", ctypes.c_uint32),
                ("sink", SINK_FN), ("user", ctypes.c_void_p),
                ("emitted", ctypes.c_uint64), ("checksum", ctypes.c_uint64),
                ("stride_words", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class WmCsrOut(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("offsets", ctypes.POINTER(ctypes.c_int64)),
                ("neighbors", ctypes.POINTER(ctypes.c_int32)),
                ("error_line", ctypes.c_int64), ("device_ms", ctypes.c_double)]


_LIB = None


def load():
    """Load libwm_b200.so (raises if it was not built — no CPU fallback)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError("libwm_b200.so not built: run paper_2212_04551_b200.build.build() "
                          "(nvcc -gencode arch=compute_100a,code=sm_100a)")
    L = ctypes.CDLL(LIB_PATH)
    L.wm_graph_create.argtypes = [ctypes.POINTER(WmCsr), ctypes.POINTER(ctypes.c_void_p)]
    L.wm_graph_create.restype = ctypes.c_int
    L.wm_graph_create_device.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
    L.wm_graph_create_device.restype = ctypes.c_int
    L.wm_run.argtypes = [ctypes.c_void_p, ctypes.POINTER(WmApp), ctypes.POINTER(WmCfg),
                         ctypes.POINTER(WmResult)]
    L.wm_run.restype = ctypes.c_int
    L.wm_run_listing.argtypes = [ctypes.c_void_p, ctypes.POINTER(WmApp), ctypes.POINTER(WmCfg),
                                 ctypes.POINTER(WmListing), ctypes.POINTER(WmResult)]
    L.wm_run_listing.restype = ctypes.c_int
    L.wm_csr_build.argtypes = [ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                               ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                               ctypes.POINTER(WmCsrOut)]
    L.wm_csr_build.restype = ctypes.c_int
    L.wm_edge_list_parse.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(WmCsrOut)]
    L.wm_edge_list_parse.restype = ctypes.c_int
    L.wm_csr_free.argtypes = [ctypes.POINTER(WmCsrOut)]
    L.wm_csr_free.restype = None
    L.wm_dictionary_build.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_uint32),
                                      ctypes.POINTER(ctypes.c_uint64), ctypes.c_uint32,
                                      ctypes.POINTER(ctypes.c_uint32)]
    L.wm_dictionary_build.restype = ctypes.c_int
    L.wm_graph_destroy.argtypes = [ctypes.c_void_p]
    L.wm_graph_destroy.restype = None
    L.wm_last_error.argtypes = []
    L.wm_last_error.restype = ctypes.c_char_p
    L.wm_abi_version.argtypes = []
    L.wm_abi_version.restype = ctypes.c_int
    L.wm_reduce_words.argtypes = [ctypes.c_uint32, ctypes.c_int]
    L.wm_reduce_words.restype = ctypes.c_uint64
    if L.wm_abi_version() != ABI_VERSION:
        raise ImportError("libwm_b200.so ABI %d, expected %d: rebuild it"
                          % (L.wm_abi_version(), ABI_VERSION))
    _LIB = L
    return L


def check(status: int) -> None:
    if status == WM_OK:
        return
    msg = load().wm_last_error().decode("utf-8", "replace")
    if status == WM_EINVAL:
        raise ValueError(msg)
    if status == WM_ECAPACITY:
        raise CapacityError(msg)
    if status == WM_EINVARIANT:
        raise InternalInvariantError(msg)
    if status == WM_ESHUTDOWN:
        raise StoreShutdownError(msg)
    if status == WM_EPARSE:
        raise GraphParseError(msg)
    raise DeviceError(msg or "libwm_b200 status %d" % status)
