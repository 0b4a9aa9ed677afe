"""ctypes front of the CPU restatement ``libwm_oracle.so``.

TEST INFRASTRUCTURE ONLY — the checker for parity tests, ``smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The product
package ``paper_2212_04551_b200`` never imports this module.
See ``wm_oracle.c`` for the reference file:line each function restates.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "libwm_oracle.so")


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libwm_oracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.wmo_clique_run.argtypes = [ctypes.c_int64, _i64p, _i32p, ctypes.c_int,
                                     ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int64,
                                     ctypes.c_int, ctypes.c_double,
                                     _u64p, _u64p, _u64p, _i64p, _u64p]
        L.wmo_motif_run.argtypes = [ctypes.c_int64, _i64p, _i32p, ctypes.c_int,
                                    _u32p, ctypes.c_uint32,
                                    ctypes.c_int64, ctypes.c_int64, _i64p, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_double,
                                    _u64p, _u64p, _u64p, _i64p, _u64p]
        L.wmo_clique_fast.argtypes = [ctypes.c_int64, _i64p, _i32p, ctypes.c_int, ctypes.c_int,
                                      _u64p, _u64p]
        L.wmo_list_run.argtypes = [ctypes.c_int64, _i64p, _i32p, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                   _u64p, _u64p, _u64p]
        _LIB = L
    return _LIB


_ERR = {-1: ValueError, -2: RuntimeError, -3: RuntimeError}


def _arrays(g):
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    nbr = np.ascontiguousarray(g.neighbors_array, dtype=np.int32)
    return off, nbr


def _roots(roots):
    if roots is None:
        return None, 0, None
    r = np.ascontiguousarray(roots, dtype=np.int64)
    return r.ctypes.data_as(_i64p), len(r), r


def clique_run(g, k, root_begin=-1, root_end=-1, roots=None, threads=None, time_budget_s=0.0):
    """Reference clique_app pipeline in id order.  Returns a dict with
    count, leaves, alg_bytes, roots_done, nodes."""
    off, nbr = _arrays(g)
    rp, nr, keep = _roots(roots)
    out = [ctypes.c_uint64() for _ in range(3)]
    done, nodes = ctypes.c_int64(), ctypes.c_uint64()
    st = lib().wmo_clique_run(g.n, off.ctypes.data_as(_i64p), nbr.ctypes.data_as(_i32p), k,
                              root_begin, root_end, rp, nr, threads or os.cpu_count(),
                              time_budget_s, *[ctypes.byref(o) for o in out],
                              ctypes.byref(done), ctypes.byref(nodes))
    if st:
        raise _ERR.get(st, RuntimeError)("oracle status %d" % st)
    return {"count": out[0].value, "leaves": out[1].value, "alg_bytes": out[2].value,
            "roots_done": done.value, "nodes": nodes.value}


def motif_run(g, k, table, pattern_count, root_begin=-1, root_end=-1, roots=None,
              threads=None, time_budget_s=0.0):
    """Reference motif_app pipeline.  Returns dict with hist (list), leaves,
    alg_bytes, roots_done, nodes."""
    off, nbr = _arrays(g)
    rp, nr, keep = _roots(roots)
    tab = np.ascontiguousarray(table, dtype=np.uint32)
    hist = np.zeros(pattern_count, dtype=np.uint64)
    leaves, ab, nodes = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    done = ctypes.c_int64()
    st = lib().wmo_motif_run(g.n, off.ctypes.data_as(_i64p), nbr.ctypes.data_as(_i32p), k,
                             tab.ctypes.data_as(_u32p), pattern_count, root_begin, root_end,
                             rp, nr, threads or os.cpu_count(), time_budget_s,
                             hist.ctypes.data_as(_u64p), ctypes.byref(leaves), ctypes.byref(ab),
                             ctypes.byref(done), ctypes.byref(nodes))
    if st:
        raise _ERR.get(st, RuntimeError)("oracle status %d" % st)
    return {"hist": [int(x) for x in hist], "leaves": leaves.value, "alg_bytes": ab.value,
            "roots_done": done.value, "nodes": nodes.value}


def list_run(g, k, complete_only=False, root_begin=-1, root_end=-1, threads=None):
    """Reference listing_app pipeline; returns dict with leaves, emitted and
    the order-independent record checksum (include/warpmine_b200.h)."""
    off, nbr = _arrays(g)
    lv, em, cs = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    st = lib().wmo_list_run(g.n, off.ctypes.data_as(_i64p), nbr.ctypes.data_as(_i32p), k,
                            int(complete_only), root_begin, root_end, threads or os.cpu_count(),
                            ctypes.byref(lv), ctypes.byref(em), ctypes.byref(cs))
    if st:
        raise _ERR.get(st, RuntimeError)("oracle status %d" % st)
    return {"leaves": lv.value, "emitted": em.value, "checksum": cs.value}


def record_checksum(records):
    """The checksum of include/warpmine_b200.h over (vertices, bits) records
    (pure Python; for golden fixtures and small cross-checks)."""
    M = (1 << 64) - 1

    def smix(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M
        return x ^ (x >> 31)

    total = 0
    for vertices, bits in records:
        h = 0
        for v in vertices:
            h = smix(h ^ int(v))
        h = smix(h ^ (bits & M))
        h = smix(h ^ (bits >> 64))
        total = (total + h) & M
    return total


def clique_fast(g, k, threads=None, with_bytes=False):
    """Independent degree-ordered kClist count (pins large clique counts).
    With ``with_bytes`` returns (count, B_alg in degree order)."""
    off, nbr = _arrays(g)
    c, b = ctypes.c_uint64(), ctypes.c_uint64()
    st = lib().wmo_clique_fast(g.n, off.ctypes.data_as(_i64p), nbr.ctypes.data_as(_i32p), k,
                               threads or os.cpu_count(), ctypes.byref(c), ctypes.byref(b))
    if st:
        raise _ERR.get(st, RuntimeError)("oracle status %d" % st)
    return (c.value, b.value) if with_bytes else c.value
