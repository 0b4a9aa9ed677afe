"""GPU parity: k-clique counts (clique_app) through the C-ABI vs the
reference's own results (golden vectors) and the validated CPU restatement."""

from __future__ import annotations

import pytest

from conftest import golden_cases, graph_from_entry

pytestmark = pytest.mark.gpu


def _graphs(golden):
    cache = {}
    for e, r in golden_cases(golden, app="clique"):
        if e["name"] not in cache:
            cache[e["name"]] = graph_from_entry(e)
        yield cache[e["name"]], e, r


@pytest.mark.parametrize("order", ["degree", "id"])
@pytest.mark.parametrize("mode", ["wc", "opt"])
def test_clique_counts_match_reference(golden, cuda, order, mode):
    from paper_2212_04551_b200 import BalanceConfig, run_clique
    bad = []
    n = 0
    for g, e, r in _graphs(golden):
        kw = {}
        if mode == "opt":
            kw["balance_config"] = BalanceConfig(threshold=1.0, poll_interval=1)
        res = run_clique(g, r["k"], mode=mode, order=order, **kw)
        n += 1
        if res.clique_count != r["count"] or res.aggregated_total != r["leaves"]:
            bad.append((e["name"], r["k"], res.clique_count, r["count"]))
    assert n > 100
    assert not bad, bad[:10]


def test_clique_alg_bytes_id_order_match_reference(golden, cuda):
    """B_alg in the reference's id order equals the figure
    derived from the reference's own traversal tree."""
    from paper_2212_04551_b200 import run_clique
    for g, e, r in _graphs(golden):
        res = run_clique(g, r["k"], order="id", count_bytes=True)
        assert res.alg_bytes == r["alg_bytes"], (e["name"], r["k"], res.alg_bytes, r["alg_bytes"])


def test_known_answers(cuda):
    """Reference tests/test_apps.py:43-54 and test_output.txt:268."""
    from paper_2212_04551_b200 import (CsrGraph, clique_counting, complete_graph, path_graph,
                                       star_of_cliques)
    g1 = CsrGraph.from_edges(5, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3), (3, 4)])
    assert clique_counting(g1, 3) == 2
    assert clique_counting(complete_graph(5), 4) == 5
    assert clique_counting(complete_graph(5), 5) == 1
    assert clique_counting(path_graph(6), 3) == 0
    assert clique_counting(star_of_cliques(6, 7), 5) == 336


@pytest.mark.parametrize("k", [3, 6, 9, 12])
def test_complete_graph_binomials(cuda, k):
    from math import comb
    from paper_2212_04551_b200 import clique_counting, complete_graph
    sizes = [k, 20, 33] + ([64, 65] if k <= 9 else []) + ([100] if k <= 6 else [])
    for n in sizes:
        if n >= k:
            assert clique_counting(complete_graph(n), k) == comb(n, k), (n, k)


def test_forced_rebalance_conserves(golden, cuda):
    from paper_2212_04551_b200 import BalanceConfig, run_clique, star_of_cliques
    g = star_of_cliques(6, 7)
    want = golden["forced_rebalance_star_of_cliques_6_7"]["clique_5"]["count"]
    r = run_clique(g, 5, mode="opt", balance_config=BalanceConfig(threshold=1.0, poll_interval=1))
    assert r.clique_count == want


def test_cfg3_scale_counts(scale_golden, cuda):
    """Config 3 (power-law 100K / ~1M) against the pinned restatement."""
    from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
    from conftest import ROOT  # noqa: F401
    import hashlib
    import numpy as np
    g = synth.config_graph("cfg3")
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype="<i8").tobytes())
    h.update(np.asarray(g.neighbors_array, dtype="<i4").tobytes())
    assert h.hexdigest() == scale_golden["cfg3"]["digest"]
    for k in range(3, 9):
        want = scale_golden["cfg3"]["clique"][str(k)]
        for mode in ("wc", "opt"):
            kw = {"balance_config": BalanceConfig(threshold=1.0)} if mode == "opt" else {}
            r = run_clique(g, k, mode=mode, **kw)
            assert r.clique_count == want["count"], (k, mode, r.clique_count, want["count"])
    for k in range(9, 13):
        want = scale_golden["cfg3"]["clique"].get(str(k))
        if want:
            r = run_clique(g, k, mode="opt", balance_config=BalanceConfig(threshold=1.0))
            assert r.clique_count == want["count"], (k, r.clique_count, want["count"])
    for k in (5, 6):
        r = run_clique(g, k, count_bytes=True)
        assert r.alg_bytes == scale_golden["cfg3"]["clique"][str(k)]["alg_bytes_degree_order"]


def test_sharded_runs_sum_to_total(cuda):
    """Cyclic task shards partition the root tasks (multi-GPU path, run
    sequentially on one device)."""
    from paper_2212_04551_b200 import gnp_random_graph, run_clique
    g = gnp_random_graph(300, 0.1, 1)
    total = run_clique(g, 4).clique_count
    for n in (2, 3, 8):
        parts = [run_clique(g, 4, shard=(r, n), reduce=False).clique_count for r in range(n)]
        assert sum(parts) == total


@pytest.mark.parametrize("split", ["0", "1", "32", "1000000"])
def test_split_heavy_tasks_partition(scale_golden, cuda, monkeypatch, split):
    """The costliest tasks of each width class are split over all shards at
    level 1 (WM_CLIQUE_SPLIT per shard; 0 = whole-task dealing only): shard
    counts sum to the golden total for every split size, and every task is
    counted once."""
    from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
    monkeypatch.setenv("WM_CLIQUE_SPLIT", split)
    g = synth.config_graph("cfg3")
    lb = BalanceConfig(threshold=1.0)
    single = run_clique(g, 6, mode="opt", balance_config=lb)
    assert single.clique_count == scale_golden["cfg3"]["clique"]["6"]["count"]
    for n in (3, 8):
        rs = [run_clique(g, 6, mode="opt", balance_config=lb, shard=(r, n), reduce=False)
              for r in range(n)]
        assert sum(r.clique_count for r in rs) == single.clique_count, (split, n)
        assert sum(r.tasks for r in rs) == single.tasks
    # k = 4 with the id orientation (wider roots: the W > 4 classes)
    want = run_clique(g, 4, order="id").clique_count
    parts = [run_clique(g, 4, order="id", shard=(r, 4), reduce=False).clique_count
             for r in range(4)]
    assert sum(parts) == want == scale_golden["cfg3"]["clique"]["4"]["count"]


def test_root_range_is_induced_suffix(cuda):
    """roots=(r0, n) in id order enumerates exactly the induced subgraph on
    [r0, n) (reference roots ascend, engine.py:187)."""
    from paper_2212_04551_b200 import gnp_random_graph, run_clique
    g = gnp_random_graph(200, 0.15, 4)
    for r0 in (0, 50, 150):
        a = run_clique(g, 4, order="id", roots=(r0, g.n)).clique_count
        b = run_clique(g.induced_suffix(r0), 4, order="id").clique_count
        assert a == b


def test_errors_map_to_reference_exceptions(cuda):
    from paper_2212_04551_b200 import Application, complete_graph, run
    from paper_2212_04551_b200.apps import clique_app
    g = complete_graph(5)
    with pytest.raises(ValueError):
        run(g, clique_app(3), mode="bogus")
    with pytest.raises(ValueError):
        run(g, Application(name="x", k=3, extend_all=False, genedges=False,
                           pipeline=(("filter", lambda *a: True, ()),), aggregator="counter"))


def test_cfg5_rmat_s22_clique_counts(scale_golden, cuda):
    """Config 5 (R-MAT scale 22, ~33M edges): k-clique counts k=3..12 vs the
    pinned restatement (kClist, tests/golden/make_golden_scale.py --cfg5)."""
    import hashlib
    import numpy as np
    from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
    g = synth.config_graph("cfg5")
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype="<i8").tobytes())
    h.update(np.asarray(g.neighbors_array, dtype="<i4").tobytes())
    assert h.hexdigest() == scale_golden["cfg5"]["digest"]
    for k in range(3, 13):
        want = scale_golden["cfg5"]["clique"][str(k)]["count"]
        r = run_clique(g, k, mode="opt", balance_config=BalanceConfig(threshold=1.0))
        assert r.clique_count == want, (k, r.clique_count, want)
    r = run_clique(g, 6, mode="wc")
    assert r.clique_count == scale_golden["cfg5"]["clique"]["6"]["count"]
