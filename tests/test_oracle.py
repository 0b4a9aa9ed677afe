"""CPU: pin the oracle (oracle/wm_oracle.c, a restatement of the reference
engine) against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and the reference's own known answers."""

from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from conftest import dictionary, golden_cases, graph_from_entry


@pytest.fixture(scope="module")
def graphs(golden):
    return {e["name"]: graph_from_entry(e) for e in golden["graphs"] if e["edges"] is not None}


def test_clique_restatement_matches_reference(golden, graphs):
    cases = golden_cases(golden, app="clique")
    assert len(cases) > 150
    for e, r in cases:
        got = oracle.clique_run(graphs[e["name"]], r["k"], threads=2)
        assert got["count"] == r["count"], (e["name"], r["k"])
        assert got["leaves"] == r["leaves"]
        assert got["alg_bytes"] == r["alg_bytes"], (e["name"], r["k"])


def test_motif_restatement_matches_reference(golden, graphs):
    cases = golden_cases(golden, app="motif")
    assert len(cases) > 150
    for e, r in cases:
        d = dictionary(r["k"])
        got = oracle.motif_run(graphs[e["name"]], r["k"], d.table, d.pattern_count, threads=2)
        assert got["hist"] == r["hist"], (e["name"], r["k"])
        assert got["leaves"] == r["leaves"]
        assert got["alg_bytes"] == r["alg_bytes"], (e["name"], r["k"])


def test_fast_clique_counter_agrees(golden, graphs):
    for e, r in golden_cases(golden, app="clique"):
        assert oracle.clique_fast(graphs[e["name"]], r["k"], threads=2) == r["count"]


def test_survey_reference_values(golden):
    """SURVEY §8(d) / BASELINE.md values measured on the reference."""
    by = {e["name"]: {(r["app"], r["k"]): r for r in e["results"]} for e in golden["graphs"]}
    assert by["cfg1_seed1"][("clique", 3)]["alg_bytes"] == 536
    assert by["cfg2_seed2"][("motif", 4)]["alg_bytes"] == 231776
    assert by["gnp_300_0.1_1"][("clique", 5)]["alg_bytes"] == 1752
    assert [by["cfg1_seed%d" % s][("clique", 3)]["count"] for s in range(5)] == [17, 17, 15, 19, 10]
    assert all(by["cfg1_seed%d" % s][("clique", 4)]["count"] == 0 for s in range(5))
    assert by["cfg2_seed2"][("motif", 4)]["hist"] == [9973, 29576, 19, 0, 7, 0]
    assert by["star_of_cliques_6_7"][("clique", 5)]["count"] == 336


def test_known_answers():
    """Reference tests/test_apps.py:43-72."""
    from paper_2212_04551_b200 import CsrGraph, complete_graph, path_graph
    g1 = CsrGraph.from_edges(5, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3), (3, 4)])
    assert oracle.clique_run(g1, 3)["count"] == 2
    assert oracle.clique_run(complete_graph(5), 4)["count"] == 5
    assert oracle.clique_run(complete_graph(5), 5)["count"] == 1
    assert oracle.clique_run(path_graph(6), 3)["count"] == 0
    d3 = dictionary(3)
    assert oracle.motif_run(g1, 3, d3.table, 2)["hist"] == [4, 2]
    assert oracle.motif_run(path_graph(4), 3, d3.table, 2)["hist"] == [2, 0]
    assert oracle.motif_run(complete_graph(4), 3, d3.table, 2)["hist"] == [0, 4]


def test_root_ranges_partition(graphs):
    """Root subsets partition the work (reference ctx.queue hook,
    tests/test_engine.py:300): per-range counts sum to the total."""
    g = graphs["gnp_60_0.3_5"]
    total = oracle.clique_run(g, 4)["count"]
    cuts = [0, 7, 20, 33, 60]
    assert sum(oracle.clique_run(g, 4, a, b)["count"] for a, b in zip(cuts, cuts[1:])) == total
    d = dictionary(4)
    tot = oracle.motif_run(g, 4, d.table, d.pattern_count)["hist"]
    parts = [oracle.motif_run(g, 4, d.table, d.pattern_count, a, b)["hist"]
             for a, b in zip(cuts, cuts[1:])]
    assert [sum(x) for x in zip(*parts)] == tot


def test_explicit_root_lists_and_budget(graphs):
    g = graphs["gnp_60_0.3_5"]
    roots = np.random.default_rng(1).permutation(g.n)
    r = oracle.clique_run(g, 4, roots=roots)
    assert r["count"] == oracle.clique_run(g, 4)["count"] and r["roots_done"] == g.n


def test_scale_golden_pinned(scale_golden):
    """BASELINE.md's survey-probe values for cfg3 reproduced by the pinned
    restatement (k=3..9), and the faithful id-order path agrees at k=3."""
    cl = scale_golden["cfg3"]["clique"]
    want = [2149007, 12110411, 77855834, 448767768, 2219264404, 9384222498, 34125264080]
    assert [cl[str(k)]["count"] for k in range(3, 10)] == want
    assert scale_golden["cfg3"]["id_order_k3"]["count"] == want[0]
    assert scale_golden["cfg3"]["m"] == 947479


def test_oracle_matches_reference_on_config_slices():
    """The C restatement against the REFERENCE's own results on slices of
    configs 3-5 (tests/golden/ref_scale_golden.json, make_golden_ref_scale.py)."""
    import json
    import numpy as np
    from conftest import GOLDEN_DIR, dictionary
    from paper_2212_04551_b200 import synth
    with open(os.path.join(GOLDEN_DIR, "ref_scale_golden.json")) as fh:
        ref = json.load(fh)
    g3 = synth.config_graph("cfg3")
    for key, want in ref["cfg3"]["clique_roots"].items():
        b, e = want["roots"]
        got = oracle.clique_run(g3, want["k"], roots=np.arange(b, e))
        assert got["count"] == want["count"], key
    g4 = synth.config_graph("cfg4")
    for key, want in ref["cfg4"]["motif_suffix"].items():
        k, s = want["k"], want["suffix"]
        d = dictionary(k)
        got = oracle.motif_run(g4, k, d.table, d.pattern_count, root_begin=g4.n - s,
                               root_end=g4.n)
        assert got["hist"] == want["hist"], key
