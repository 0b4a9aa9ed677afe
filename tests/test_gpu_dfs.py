"""GPU parity of the DM_DFS ablation (mode "dfs": one thread per traversal,
reference engine.py:13-16) — the same counts, histograms and records as the
reference (golden vectors) and as the warp-centric kernels."""

from __future__ import annotations

import json
import os

import pytest

from conftest import GOLDEN_DIR, dictionary, golden_cases, graph_from_entry

pytestmark = pytest.mark.gpu


def test_dfs_clique_counts_match_reference(golden, cuda):
    from paper_2212_04551_b200 import run_clique
    cache, n = {}, 0
    for e, r in golden_cases(golden, app="clique"):
        g = cache.setdefault(e["name"], graph_from_entry(e))
        for order in ("id", "degree"):
            res = run_clique(g, r["k"], mode="dfs", order=order)
            assert res.clique_count == r["count"], (e["name"], r["k"], order)
        n += 1
    assert n > 100


def test_dfs_motif_histograms_match_reference(golden, cuda):
    from paper_2212_04551_b200 import run_motifs
    cache, n = {}, 0
    for e, r in golden_cases(golden, app="motif"):
        g = cache.setdefault(e["name"], graph_from_entry(e))
        res = run_motifs(g, r["k"], dictionary(r["k"]), mode="dfs")
        assert res.pattern_counts == r["hist"] and res.aggregated_total == r["leaves"], \
            (e["name"], r["k"])
        n += 1
    assert n > 100


def test_dfs_listing_matches_reference(cuda):
    """Reference test_apps.py:124-127: every mode lists the same family."""
    from paper_2212_04551_b200 import CsrGraph, listing_checksum, subgraph_listing
    with open(os.path.join(GOLDEN_DIR, "listing_golden.json")) as fh:
        lg = json.load(fh)
    g1 = CsrGraph.from_edges(5, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3), (3, 4)])
    sets = [{frozenset(v) for v, b in subgraph_listing(g1, 3, mode=m)}
            for m in ("dfs", "wc", "opt")]
    assert sets[0] == sets[1] == sets[2]
    for e in lg["graphs"]:
        g = graph_from_entry(e)
        for r in e["results"]:
            res = listing_checksum(g, r["k"], mode="dfs")
            assert (res.records_emitted, res.extra["checksum"]) == (r["count"], r["checksum"])
            res = listing_checksum(g, r["k"], complete_only=True, mode="dfs")
            assert res.records_emitted == r["complete_count"]


@pytest.mark.parametrize("cfg,app,k", [("cfg3", "clique", 5), ("cfg2", "motif", 5),
                                       ("cfg1", "motif", 6)])
def test_dfs_equals_warp_centric_at_scale(cuda, cfg, app, k):
    from paper_2212_04551_b200 import run_clique, run_motifs, synth
    g = synth.config_graph(cfg)
    if app == "clique":
        assert run_clique(g, k, mode="dfs").clique_count == run_clique(g, k).clique_count
    else:
        d = dictionary(k)
        assert run_motifs(g, k, d, mode="dfs").pattern_counts == \
            run_motifs(g, k, d).pattern_counts
