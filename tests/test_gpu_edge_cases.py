"""GPU parity on edge-case graphs the golden corpus does not stress: no edges,
a single vertex, k beyond the largest clique, disconnected parts, and hub rows
far wider than a warp (multi-round 32-ary row searches, wide bitmap classes,
edge-hash probes against a hub).  The checker is the CPU restatement
(``oracle/``), itself pinned to the reference's golden vectors."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import dictionary

pytestmark = pytest.mark.gpu


def _graph(n, edges):
    from paper_2212_04551_b200.graph import CsrGraph
    ed = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    return CsrGraph.from_arrays(n, ed[:, 0], ed[:, 1])


def _hub_graph(leaves=5000, extra=6000, seed=5):
    """Vertex 0 adjacent to every leaf, plus random leaf-leaf edges and a second
    hub sharing half the leaves (rows of 5000 and 2500 entries)."""
    rng = np.random.default_rng(seed)
    n = leaves + 2
    e = [(0, v) for v in range(1, leaves + 1)]
    e += [(leaves + 1, v) for v in range(1, leaves + 1, 2)]
    a = rng.integers(1, leaves + 1, extra)
    b = rng.integers(1, leaves + 1, extra)
    e += [(int(x), int(y)) for x, y in zip(a, b) if x != y]
    return _graph(n, e)


def _check_motif(g, k, modes=("wc", "opt")):
    import oracle
    from paper_2212_04551_b200 import BalanceConfig, run_motifs
    d = dictionary(k)
    want = oracle.motif_run(g, k, d.table, d.pattern_count)
    for mode in modes:
        kw = {"balance_config": BalanceConfig(threshold=1.0, poll_interval=1)} if mode == "opt" else {}
        r = run_motifs(g, k, d, mode=mode, **kw)
        assert r.pattern_counts == want["hist"], (k, mode)
        assert r.aggregated_total == want["leaves"], (k, mode)


def _check_clique(g, k):
    import oracle
    from paper_2212_04551_b200 import BalanceConfig, run_clique
    want = oracle.clique_fast(g, k)
    assert run_clique(g, k, mode="wc").clique_count == want, k
    bc = BalanceConfig(threshold=1.0, poll_interval=1)
    assert run_clique(g, k, mode="opt", balance_config=bc).clique_count == want, k
    assert run_clique(g, k, mode="opt", balance_config=bc, order="id").clique_count == want, k


def test_graph_without_edges(cuda):
    from paper_2212_04551_b200 import run_clique, run_motifs
    g = _graph(7, np.zeros((0, 2), dtype=np.int64))
    for k in (3, 4, 6):
        assert run_clique(g, k).clique_count == 0
    for k in (3, 4, 5):
        r = run_motifs(g, k, dictionary(k), mode="opt")
        assert r.pattern_counts == [0] * dictionary(k).pattern_count
        assert r.aggregated_total == 0


def test_single_vertex_and_single_edge(cuda):
    from paper_2212_04551_b200 import run_clique, run_motifs
    for g in (_graph(1, np.zeros((0, 2), dtype=np.int64)), _graph(2, [(0, 1)])):
        assert run_clique(g, 3).clique_count == 0
        assert sum(run_motifs(g, 3, dictionary(3)).pattern_counts) == 0


def test_k_beyond_largest_clique(cuda):
    from paper_2212_04551_b200 import complete_graph, run_clique
    g = complete_graph(5)
    assert [run_clique(g, k).clique_count for k in (5, 6, 8, 12)] == [1, 0, 0, 0]


def test_disconnected_components(cuda):
    from paper_2212_04551_b200 import star_of_cliques
    g = star_of_cliques(3, 6)
    n = g.n
    src, dst = [], []
    off, nbr = np.asarray(g.offsets), np.asarray(g.neighbors_array)
    for u in range(n):
        for v in nbr[off[u]:off[u + 1]]:
            if u < v:
                src += [u, u + n]
                dst += [int(v), int(v) + n]
    two = _graph(2 * n, list(zip(src, dst)))
    for k in (3, 4, 5):
        _check_clique(two, k)
    _check_motif(two, 4)


@pytest.mark.parametrize("k,leaves,extra", [(3, 5000, 6000), (4, 400, 2000), (5, 120, 300)])
def test_hub_rows_motif(cuda, k, leaves, extra):
    # hub stars dominate: C(leaves, k-1) leaves per hub, kept to a few million
    _check_motif(_hub_graph(leaves, extra), k)


@pytest.mark.parametrize("leaves,extra", [(600, 40000), (1000, 50000), (1500, 60000)])
def test_hub_rows_clique(cuda, leaves, extra):
    # in id order the hub's out-row spans every leaf: wide bitmap classes up to
    # 1024 members, beyond that the wide-root path (induced subgraph of N+(v))
    g = _hub_graph(leaves=leaves, extra=extra, seed=9)
    for k in (3, 4, 5, 6):
        _check_clique(g, k)


@pytest.mark.parametrize("k", [3, 4])
def test_wide_roots_in_degree_order(cuda, k):
    """K_1040 under degree order (all degrees tie -> id order): roots 0..14 have
    > 1024 out-neighbours; their induced subgraphs recurse (k=4 nests once more,
    down to the k-1 = 2 edge count).  Sharded runs still partition them."""
    from math import comb
    from paper_2212_04551_b200 import complete_graph, run_clique
    g = complete_graph(1040)
    assert run_clique(g, k).clique_count == comb(1040, k)
    parts = [run_clique(g, k, shard=(r, 3), reduce=False).clique_count for r in range(3)]
    assert sum(parts) == comb(1040, k)
