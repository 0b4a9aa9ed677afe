"""The C-ABI boundary on the device: CsrGraph contract checks in
``wm_graph_create`` / ``wm_graph_create_device`` (reference
``graph.py:122-133``: offsets span nnz and never decrease, rows strictly
ascending, no self-loops, symmetric) and serialisation of concurrent callers
on one device (per-device workspace lock)."""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _create_host(n, off, nbr):
    from paper_2212_04551_b200 import _native
    off = np.ascontiguousarray(off, dtype=np.int64)
    nbr = np.ascontiguousarray(nbr, dtype=np.int32)
    csr = _native.WmCsr(n, len(nbr), off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                        nbr.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    h = ctypes.c_void_p()
    L = _native.load()
    _native.check(L.wm_graph_create(ctypes.byref(csr), ctypes.byref(h)))
    L.wm_graph_destroy(h)


def _create_device(n, off, nbr):
    import torch
    from paper_2212_04551_b200 import _native
    doff = torch.tensor(np.asarray(off, dtype=np.int64), device="cuda")
    dnbr = torch.tensor(np.asarray(nbr, dtype=np.int32), device="cuda")
    h = ctypes.c_void_p()
    L = _native.load()
    _native.check(L.wm_graph_create_device(n, len(nbr), doff.data_ptr(), dnbr.data_ptr(),
                                           ctypes.byref(h)))
    torch.cuda.synchronize()
    L.wm_graph_destroy(h)


# (n, offsets, neighbours, expected message fragment)
BAD = [
    # triangle 0-1-2 with row 1 unsorted
    (3, [0, 2, 4, 6], [1, 2, 2, 0, 0, 1], "adjacency of 1 not strictly ascending"),
    # duplicate neighbour (not strictly ascending)
    (3, [0, 2, 3, 4], [1, 1, 0, 0], "adjacency of 0 not strictly ascending"),
    # self-loop at 2
    (3, [0, 1, 2, 4], [1, 0, 1, 2], "self-loop at 2"),
    # edge (0,2) without (2,0)
    (3, [0, 2, 3, 4], [1, 2, 0, 1], "edge (0,2) not symmetric"),
    # neighbour id out of range
    (3, [0, 1, 2, 3], [1, 0, 7], "outside [0, 3)"),
    (3, [0, 1, 2, 3], [1, 0, -1], "outside [0, 3)"),
]


@pytest.mark.parametrize("n,off,nbr,msg", BAD)
def test_bad_csr_rejected_host(cuda, n, off, nbr, msg):
    with pytest.raises(ValueError, match=msg.replace("(", r"\(").replace(")", r"\)")
                       .replace("[", r"\[")):
        _create_host(n, off, nbr)


@pytest.mark.parametrize("n,off,nbr,msg", BAD)
def test_bad_csr_rejected_device(cuda, n, off, nbr, msg):
    with pytest.raises(ValueError, match=msg.replace("(", r"\(").replace(")", r"\)")
                       .replace("[", r"\[")):
        _create_device(n, off, nbr)


def test_bad_offsets_rejected(cuda):
    with pytest.raises(ValueError, match="offsets"):
        _create_host(3, [0, 2, 1, 2], [1, 0])
    with pytest.raises(ValueError, match="offsets"):
        _create_device(3, [0, 2, 1, 2], [1, 0])
    with pytest.raises(ValueError, match="offsets do not span"):
        _create_device(3, [0, 1, 2, 3], [1, 0, 0, 0])


def test_first_violation_in_reference_order(cuda):
    # vertex 1 has both a self-loop and an asymmetric edge; vertex 3 is
    # unsorted: the reference checks u = 0, 1, ... and per u ascending first
    n = 4
    rows = [[1], [0, 1, 3], [], [1, 0]]
    off = np.cumsum([0] + [len(r) for r in rows])
    nbr = sum(rows, [])
    with pytest.raises(ValueError, match="self-loop at 1"):
        _create_host(n, off, nbr)


def test_unsorted_row_reported_at_its_vertex(cuda):
    """Row 2 unsorted but symmetric: the reference's set-membership symmetry
    check passes at vertices 0 and 1 and the ascending check fails at 2."""
    rows = [[1, 2], [0, 2], [1, 0]]
    off = np.cumsum([0] + [len(r) for r in rows])
    with pytest.raises(ValueError, match="adjacency of 2 not strictly ascending"):
        _create_host(3, off, sum(rows, []))
    with pytest.raises(ValueError, match="adjacency of 2 not strictly ascending"):
        _create_device(3, off, sum(rows, []))


def test_good_graphs_accepted(cuda):
    from paper_2212_04551_b200 import gnp_random_graph, run_clique, synth
    g = gnp_random_graph(200, 0.1, 5)
    _create_host(g.n, g.offsets, g.neighbors_array)
    _create_device(g.n, g.offsets, g.neighbors_array)
    e = synth.path_graph(1)  # one vertex, no edges
    _create_host(e.n, e.offsets, e.neighbors_array)
    assert run_clique(g, 3).clique_count >= 0


def test_concurrent_calls_on_one_device(cuda):
    """Two Python threads (ctypes drops the GIL) share one device: the
    workspace lock serialises them, both results stay exact."""
    import oracle
    from paper_2212_04551_b200 import (BalanceConfig, build_dictionary, gnp_random_graph,
                                       run_clique, run_motifs)
    ga = gnp_random_graph(400, 0.05, 11)
    gb = gnp_random_graph(300, 0.06, 12)
    d = build_dictionary(4)
    want_a = oracle.clique_run(ga, 4)["count"]
    want_b = oracle.motif_run(gb, 4, d.table, d.pattern_count)["hist"]
    errors = []

    def worker(fn):
        try:
            for _ in range(20):
                fn()
        except BaseException as exc:  # pragma: no cover - surfaced below
            errors.append(exc)

    def a():
        assert run_clique(ga, 4, mode="opt",
                          balance_config=BalanceConfig(threshold=1.0)).clique_count == want_a

    def b():
        assert run_motifs(gb, 4, d, mode="opt",
                          balance_config=BalanceConfig(threshold=1.0)).pattern_counts == want_b

    ts = [threading.Thread(target=worker, args=(f,)) for f in (a, b, a, b)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
