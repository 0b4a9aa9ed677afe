"""Undirected simple graphs in CSR form — the hot path's input contract.

Same contract as ``warpmine.graph.CsrGraph`` (reference
``pkg/src/warpmine/graph.py:28-136``): vertices ``0..n-1``, each row
``neighbors[offsets[v]:offsets[v+1]]`` strictly ascending, symmetric, no
self-loops, immutable after construction.

B200 layout differences:

* ``offsets`` is int64 (n+1) and ``neighbors_array`` is **int32** (2m) —
  the exact arrays uploaded to HBM by ``wm_graph_create``; the reference keeps
  int64 neighbours (``graph.py:67-78``).
* Construction is vectorised numpy (``np.unique`` over packed u64 edge keys)
  instead of the reference's ``sorted(set(pairs))`` tuple path
  (``graph.py:54-67``), so R-MAT scale-22 graphs build in seconds.
* ``save``/``load`` use a small binary file (``WMG1``) so the GPU run and the
  CPU baseline read the same graph bytes.
"""

from __future__ import annotations

import ctypes
import io
import os
import struct
from typing import Iterable, Iterator

import numpy as np

from .errors import GraphParseError

_COMMENT_PREFIXES = ("#", "%")
_MAGIC = b"WMG1"


class CsrGraph:
    """Immutable undirected simple graph in CSR layout."""

    __slots__ = ("n", "m", "offsets", "neighbors_array", "max_degree",
                 "_adj_lists", "_adj_sets", "_degrees", "__weakref__")

    def __init__(self, n: int, offsets: np.ndarray, neighbors: np.ndarray):
        self.n = int(n)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.neighbors_array = np.ascontiguousarray(neighbors, dtype=np.int32)
        self.m = len(self.neighbors_array) // 2
        self._degrees = np.diff(self.offsets)
        self.max_degree = int(self._degrees.max()) if self.n > 0 else 0
        self._adj_lists = None
        self._adj_sets = None
        self.offsets.setflags(write=False)
        self.neighbors_array.setflags(write=False)

    # -- construction ----------------------------------------------------

    @classmethod
    def from_edges(cls, n: int, edges) -> "CsrGraph":
        """Graph on ``0..n-1`` from an edge iterable or an (E,2) array.

        Duplicates and self-loops are dropped; ids are not remapped, so
        isolated vertices are representable (reference ``graph.py:44-61``).
        """
        if n < 1:
            raise ValueError("graph needs at least one vertex, got n=%d" % n)
        arr = np.asarray(list(edges) if not isinstance(edges, np.ndarray)
                         else edges, dtype=np.int64).reshape(-1, 2)
        if arr.size and (arr.min() < 0 or arr.max() >= n):
            bad = arr[(arr < 0).any(axis=1) | (arr >= n).any(axis=1)][0]
            raise ValueError("edge (%d, %d) outside vertex range 0..%d"
                             % (bad[0], bad[1], n - 1))
        return cls.from_arrays(n, arr[:, 0], arr[:, 1])

    @classmethod
    def from_arrays(cls, n: int, src, dst, device: bool = False) -> "CsrGraph":
        """Vectorised build from endpoint arrays (any direction, any
        multiplicity); symmetrises, dedups, drops self-loops.  With
        ``device=True`` the sort/unique/scan passes run on the current CUDA
        device (``wm_csr_build``); the arrays are identical."""
        if device:
            return _csr_build_device(n, src, dst)
        src = np.asarray(src, dtype=np.int64)
        dst = np.asarray(dst, dtype=np.int64)
        keep = src != dst
        lo = np.minimum(src[keep], dst[keep])
        hi = np.maximum(src[keep], dst[keep])
        key = np.unique(lo * np.int64(n) + hi)          # sorted, unique (u<v)
        u = key // n
        v = key - u * n
        s = np.concatenate([u, v])
        d = np.concatenate([v, u])
        order = np.lexsort((d, s))
        counts = np.bincount(s, minlength=n)
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=offsets[1:])
        return cls(n, offsets, d[order].astype(np.int32))

    @classmethod
    def from_csr(cls, offsets, neighbors, validate: bool = True) -> "CsrGraph":
        g = cls(len(offsets) - 1, offsets, neighbors)
        if validate:
            g.validate_fast()
        return g

    # -- accessors -------------------------------------------------------

    def neighbors(self, v: int) -> np.ndarray:
        if not (0 <= v < self.n):
            raise ValueError("vertex %d out of range 0..%d" % (v, self.n - 1))
        return self.neighbors_array[self.offsets[v]:self.offsets[v + 1]]

    def degree(self, v: int) -> int:
        if not (0 <= v < self.n):
            raise ValueError("vertex %d out of range 0..%d" % (v, self.n - 1))
        return int(self._degrees[v])

    def degrees(self) -> np.ndarray:
        return self._degrees

    def adjacency_lists(self) -> list:
        if self._adj_lists is None:
            flat = self.neighbors_array.tolist()
            off = self.offsets.tolist()
            self._adj_lists = [flat[off[v]:off[v + 1]] for v in range(self.n)]
        return self._adj_lists

    def adjacency_sets(self) -> list:
        if self._adj_sets is None:
            self._adj_sets = [set(a) for a in self.adjacency_lists()]
        return self._adj_sets

    def has_edge(self, u: int, v: int) -> bool:
        row = self.neighbors(u)
        i = int(np.searchsorted(row, v))
        return i < len(row) and int(row[i]) == v

    def edges(self) -> Iterator[tuple]:
        """Each undirected edge once as (u, v), u < v, sorted."""
        src = np.repeat(np.arange(self.n, dtype=np.int64), self._degrees)
        dst = self.neighbors_array.astype(np.int64)
        up = src < dst
        for a, b in zip(src[up].tolist(), dst[up].tolist()):
            yield (a, b)

    def edge_array(self) -> np.ndarray:
        src = np.repeat(np.arange(self.n, dtype=np.int64), self._degrees)
        dst = self.neighbors_array.astype(np.int64)
        up = src < dst
        return np.stack([src[up], dst[up]], axis=1)

    def to_edge_list(self) -> str:
        return "".join("%d %d\n" % e for e in self.edges())

    def induced_suffix(self, r0: int) -> "CsrGraph":
        """Induced subgraph on vertices ``r0..n-1`` relabelled to
        ``0..n-r0-1``.  Root-suffix runs enumerate exactly this graph:
        a subgraph lies in the subtree of its minimum-id vertex
        (reference ``engine.py:187`` roots ascending), so roots ``[r0,n)``
        own every subgraph whose vertices are all ``>= r0``."""
        e = self.edge_array()
        e = e[(e >= r0).all(axis=1)] - r0
        return CsrGraph.from_arrays(self.n - r0, e[:, 0], e[:, 1])

    # -- invariants ------------------------------------------------------

    def validate(self) -> None:
        """Check all CSR invariants (reference ``graph.py:122-133``)."""
        self.validate_fast()

    def validate_fast(self) -> None:
        off, nb = self.offsets, self.neighbors_array
        assert off[0] == 0 and off[-1] == len(nb), "offsets do not span neighbors"
        assert len(nb) % 2 == 0, "odd adjacency length"
        assert np.all(np.diff(off) >= 0), "offsets must be non-decreasing"
        if len(nb) == 0:
            return
        assert nb.min() >= 0 and nb.max() < self.n, "neighbor id out of range"
        src = np.repeat(np.arange(self.n, dtype=np.int64), self._degrees)
        same_row = src[1:] == src[:-1]
        assert np.all(nb[1:][same_row] > nb[:-1][same_row]), \
            "adjacency rows must be strictly ascending"
        assert not np.any(src == nb), "self-loop"
        fwd = src * self.n + nb
        rev = nb.astype(np.int64) * self.n + src
        assert np.array_equal(np.sort(fwd), np.sort(rev)), "adjacency not symmetric"

    # -- binary file -----------------------------------------------------

    def save(self, path) -> None:
        """``WMG1`` | u64 n | u64 nnz | i64 offsets[n+1] | i32 neighbors[nnz]."""
        with open(path, "wb") as fh:
            fh.write(_MAGIC)
            fh.write(struct.pack("<QQ", self.n, len(self.neighbors_array)))
            fh.write(self.offsets.astype("<i8").tobytes())
            fh.write(self.neighbors_array.astype("<i4").tobytes())

    @classmethod
    def load(cls, path, validate: bool = False) -> "CsrGraph":
        with open(path, "rb") as fh:
            blob = fh.read()
        if blob[:4] != _MAGIC:
            raise GraphParseError("bad graph file magic %r" % blob[:4])
        n, nnz = struct.unpack_from("<QQ", blob, 4)
        pos = 20
        offsets = np.frombuffer(blob, "<i8", n + 1, pos)
        neighbors = np.frombuffer(blob, "<i4", nnz, pos + 8 * (n + 1))
        return cls.from_csr(offsets.copy(), neighbors.copy(), validate=validate)

    def __repr__(self):
        return "CsrGraph(n=%d, m=%d, max_degree=%d)" % (self.n, self.m, self.max_degree)


def load_edge_list(source, device: bool = False) -> CsrGraph:
    """Parse whitespace edge-list text (reference ``graph.py:139-188``):
    '#'/'%' comments and blank lines skipped, ids remapped to ``0..n-1``
    preserving ascending order, duplicates and self-loops dropped.
    Raises GraphParseError with the line number on malformed input.
    ``device=True`` parses and builds on the current CUDA device
    (``wm_edge_list_parse``: one thread per line, sort/unique remap)."""
    if device:
        if isinstance(source, (str, bytes, os.PathLike)):
            with open(source, "rb") as fh:
                text = fh.read()
        else:
            text = "".join(source).encode("utf-8")
        return _parse_device(text)
    if isinstance(source, (str, bytes, os.PathLike)):
        with open(source, "r", encoding="utf-8") as fh:
            return _parse_lines(fh)
    return _parse_lines(source)


def _take_csr(out) -> CsrGraph:
    from . import _native
    try:
        n, nnz = int(out.n), int(out.nnz)
        off = np.ctypeslib.as_array(out.offsets, shape=(n + 1,)).copy()
        nbr = (np.ctypeslib.as_array(out.neighbors, shape=(nnz,)).copy() if nnz
               else np.zeros(0, np.int32))
    finally:
        _native.load().wm_csr_free(ctypes.byref(out))
    return CsrGraph(n, off, nbr)


def _csr_build_device(n, src, dst) -> CsrGraph:
    from . import _native
    src = np.ascontiguousarray(src, dtype=np.int64)
    dst = np.ascontiguousarray(dst, dtype=np.int64)
    if src.shape != dst.shape:
        raise ValueError("endpoint arrays differ in length")
    out = _native.WmCsrOut()
    p64 = ctypes.POINTER(ctypes.c_int64)
    _native.check(_native.load().wm_csr_build(int(n), src.ctypes.data_as(p64),
                                              dst.ctypes.data_as(p64), len(src),
                                              ctypes.byref(out)))
    return _take_csr(out)


def _parse_device(text: bytes) -> CsrGraph:
    from . import _native
    out = _native.WmCsrOut()
    st = _native.load().wm_edge_list_parse(text, len(text), ctypes.byref(out))
    if st == _native.WM_EPARSE:
        line = int(out.error_line)
        if line > 0:
            # re-raise through the host reader on the offending line so the
            # message and line number are exactly the reference's
            bad = text.split(b"\n")[line - 1].decode("utf-8", "replace")
            try:
                _parse_lines([""] * (line - 1) + [bad])
            except GraphParseError:
                raise
            raise GraphParseError("malformed input", line)
        raise GraphParseError("empty graph: no valid edges in input")
    _native.check(st)
    return _take_csr(out)


def _parse_lines(lines: Iterable[str]) -> CsrGraph:
    us: list = []
    vs: list = []
    for lineno, line in enumerate(lines, start=1):
        stripped = line.strip()
        if not stripped or stripped.startswith(_COMMENT_PREFIXES):
            continue
        tokens = stripped.split()
        if len(tokens) != 2:
            raise GraphParseError("expected two integer tokens, got %r" % stripped, lineno)
        try:
            u, v = int(tokens[0]), int(tokens[1])
        except ValueError:
            raise GraphParseError("non-integer token in %r" % stripped, lineno) from None
        if u < 0 or v < 0:
            raise GraphParseError("negative vertex id in %r" % stripped, lineno)
        if u == v:
            continue
        us.append(u)
        vs.append(v)
    if not us:
        raise GraphParseError("empty graph: no valid edges in input")
    ids, inv = np.unique(np.array(us + vs, dtype=np.int64), return_inverse=True)
    half = len(us)
    return CsrGraph.from_arrays(len(ids), inv[:half], inv[half:])


def neighbors(g: CsrGraph, v: int) -> np.ndarray:
    """Functional alias for ``g.neighbors(v)`` (reference ``graph.py:191``)."""
    return g.neighbors(v)
