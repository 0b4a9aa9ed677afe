"""GPU parity: k-motif pattern histograms (motif_app) through the C-ABI vs the
reference's own results (golden vectors) and the validated CPU restatement."""

from __future__ import annotations

import pytest

from conftest import dictionary, golden_cases, graph_from_entry

pytestmark = pytest.mark.gpu


def _cases(golden):
    cache = {}
    for e, r in golden_cases(golden, app="motif"):
        if e["name"] not in cache:
            cache[e["name"]] = graph_from_entry(e)
        yield cache[e["name"]], e, r


@pytest.mark.parametrize("mode", ["wc", "opt"])
def test_motif_histograms_match_reference(golden, cuda, mode):
    from paper_2212_04551_b200 import BalanceConfig, run_motifs
    bad = []
    n = 0
    for g, e, r in _cases(golden):
        kw = {}
        if mode == "opt":
            kw["balance_config"] = BalanceConfig(threshold=1.0, poll_interval=1)
        res = run_motifs(g, r["k"], dictionary(r["k"]), mode=mode, **kw)
        n += 1
        if res.pattern_counts != r["hist"] or res.aggregated_total != r["leaves"]:
            bad.append((e["name"], r["k"], res.pattern_counts, r["hist"]))
    assert n > 100
    assert not bad, bad[:5]


def test_motif_alg_bytes_match_reference(golden, cuda):
    from paper_2212_04551_b200 import run_motifs
    for g, e, r in _cases(golden):
        res = run_motifs(g, r["k"], dictionary(r["k"]), count_bytes=True)
        assert res.alg_bytes == r["alg_bytes"], (e["name"], r["k"], res.alg_bytes, r["alg_bytes"])


def test_motif_alg_bytes_with_balancer(golden, scale_golden, cuda):
    """B_alg with the on-device balancer forced on (threshold 1.0, poll 1):
    productive nodes shared through donations are counted exactly once
    (claim slots), so it equals the LB-off / reference figure."""
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, synth
    lb = BalanceConfig(threshold=1.0, poll_interval=1)
    n = 0
    for g, e, r in _cases(golden):
        res = run_motifs(g, r["k"], dictionary(r["k"]), mode="opt", balance_config=lb,
                         count_bytes=True)
        assert res.alg_bytes == r["alg_bytes"], (e["name"], r["k"], res.alg_bytes, r["alg_bytes"])
        assert res.pattern_counts == r["hist"]
        n += 1
    assert n > 0
    migr = 0
    for name in ("cfg1", "cfg2"):
        g = synth.config_graph(name)
        for k, want in scale_golden[name]["motif"].items():
            res = run_motifs(g, int(k), dictionary(int(k)), mode="opt", balance_config=lb,
                             count_bytes=True)
            assert res.alg_bytes == want["alg_bytes"], (name, k, res.alg_bytes)
            assert res.pattern_counts == want["hist"]
            migr += res.migrations
    assert migr > 0  # donations happened


def test_known_answers(cuda):
    """Reference tests/test_apps.py:57-72."""
    from paper_2212_04551_b200 import CsrGraph, complete_graph, motif_counting, path_graph
    g1 = CsrGraph.from_edges(5, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3), (3, 4)])
    assert motif_counting(g1, 3, dictionary(3)) == {0: 4, 1: 2}
    assert motif_counting(path_graph(4), 3, dictionary(3)) == {0: 2, 1: 0}
    assert motif_counting(complete_graph(4), 3, dictionary(3)) == {0: 0, 1: 4}


@pytest.mark.parametrize("k", [3, 4, 5, 6, 7])
def test_cross_app_identity(cuda, k):
    """clique(k) == motif_hist(k)[last] (reference test_apps.py:85-88)."""
    from paper_2212_04551_b200 import clique_counting, gnp_random_graph, motif_counting
    g = gnp_random_graph(60, 0.3, 5)
    hist = motif_counting(g, k, dictionary(k))
    assert hist[max(hist)] == clique_counting(g, k)


def test_forced_rebalance_conserves(golden, cuda):
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, star_of_cliques
    g = star_of_cliques(6, 7)
    want = golden["forced_rebalance_star_of_cliques_6_7"]["motif_4"]["hist"]
    r = run_motifs(g, 4, dictionary(4), mode="opt",
                   balance_config=BalanceConfig(threshold=1.0, poll_interval=1))
    assert r.pattern_counts == want


def test_cfg_scale_histograms(scale_golden, cuda):
    """cfg1/cfg2 motif k=5,6 vs the pinned restatement."""
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, synth
    for name in ("cfg1", "cfg2"):
        g = synth.config_graph(name)
        for k, want in scale_golden[name]["motif"].items():
            k = int(k)
            for mode in ("wc", "opt"):
                kw = {"balance_config": BalanceConfig(threshold=1.0)} if mode == "opt" else {}
                r = run_motifs(g, k, dictionary(k), mode=mode, **kw)
                assert r.pattern_counts == want["hist"], (name, k, mode)


def test_cfg4_rmat_root_suffix(scale_golden, cuda):
    """Config 4 (skewed R-MAT s20): bounded root-suffix runs vs the pinned
    restatement; the suffix is exactly the induced subgraph on the last ids."""
    import hashlib
    import numpy as np
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, synth
    g = synth.config_graph("cfg4")
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype="<i8").tobytes())
    h.update(np.asarray(g.neighbors_array, dtype="<i4").tobytes())
    assert h.hexdigest() == scale_golden["cfg4"]["digest"]
    for key, want in scale_golden["cfg4"]["motif_suffix"].items():
        k, s = want["k"], want["suffix"]
        for mode in ("wc", "opt"):
            kw = {"balance_config": BalanceConfig(threshold=1.0)} if mode == "opt" else {}
            r = run_motifs(g, k, dictionary(k), mode=mode, roots=(g.n - s, g.n), **kw)
            assert r.pattern_counts == want["hist"], (key, mode)


def test_root_suffix_and_shards(cuda):
    """Root suffix == induced suffix graph; cyclic shards sum to the total."""
    from paper_2212_04551_b200 import gnp_random_graph, run_motifs
    g = gnp_random_graph(150, 0.06, 11)
    d = dictionary(5)
    full = run_motifs(g, 5, d).pattern_counts
    for r0 in (0, 40, 100):
        a = run_motifs(g, 5, d, roots=(r0, g.n)).pattern_counts
        b = run_motifs(g.induced_suffix(r0), 5, d).pattern_counts
        assert a == b
    parts = [run_motifs(g, 5, d, shard=(r, 3), reduce=False).pattern_counts for r in range(3)]
    assert [sum(x) for x in zip(*parts)] == full


@pytest.mark.parametrize("level", ["1", "2"])
def test_shards_partition_deep_motifs(scale_golden, cuda, monkeypatch, level):
    """k = 6 / 7 shards (level-1 edge tasks or level-2 (root, child,
    grandchild) tasks, WM_MOTIF_SHARD_LEVEL) partition the tree: their
    histograms sum to the golden one, with and without forced balancing."""
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, synth
    monkeypatch.setenv("WM_MOTIF_SHARD_LEVEL", level)
    lb = BalanceConfig(threshold=1.0, poll_interval=1)
    g = synth.config_graph("cfg2")
    for k in (6, 7) if "7" in scale_golden["cfg2"]["motif"] else (6,):
        want = scale_golden["cfg2"]["motif"][str(k)]["hist"]
        for n in (2, 5):
            parts = [run_motifs(g, k, dictionary(k), mode="opt", balance_config=lb,
                                shard=(r, n), reduce=False).pattern_counts for r in range(n)]
            assert [sum(x) for x in zip(*parts)] == want, (k, n)
    g4 = synth.config_graph("cfg4")
    want = scale_golden["cfg4"]["motif_suffix"]["k6_s4096"]["hist"]
    parts = [run_motifs(g4, 6, dictionary(6), mode="opt", balance_config=lb,
                        roots=(g4.n - 4096, g4.n), shard=(r, 4), reduce=False).pattern_counts
             for r in range(4)]
    assert [sum(x) for x in zip(*parts)] == want


def test_cfg5_rmat_s22_root_suffix(scale_golden, cuda):
    """Config 5 (R-MAT scale 22): k=5/6/7 motif histograms over root suffixes
    (the induced subgraph on the last s ids) vs the pinned restatement."""
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, synth
    g = synth.config_graph("cfg5")
    for key, want in scale_golden["cfg5"]["motif_suffix"].items():
        k, s = want["k"], want["suffix"]
        for mode in ("wc", "opt"):
            kw = {"balance_config": BalanceConfig(threshold=1.0)} if mode == "opt" else {}
            r = run_motifs(g, k, dictionary(k), mode=mode, roots=(g.n - s, g.n), **kw)
            assert r.pattern_counts == want["hist"], (key, mode)


def test_suffix_local_hash_matches_global(scale_golden, cuda, monkeypatch):
    """Root-suffix runs probe a per-run edge hash of the induced subgraph on
    [begin, n); the whole-graph table (WM_NO_LOCAL_HASH=1) gives the same
    histograms, with and without forced balancing."""
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, synth
    g = synth.config_graph("cfg4")
    lb = BalanceConfig(threshold=1.0, poll_interval=1)
    for key in ("k5_s4096", "k6_s4096", "k7_s2048"):
        want = scale_golden["cfg4"]["motif_suffix"][key]
        k, s = want["k"], want["suffix"]
        for local in ("0", "1"):
            monkeypatch.setenv("WM_NO_LOCAL_HASH", local)
            r = run_motifs(g, k, dictionary(k), mode="opt", balance_config=lb,
                           roots=(g.n - s, g.n))
            assert r.pattern_counts == want["hist"], (key, local)


def test_csr_probe_fallback_matches(golden, cuda, monkeypatch):
    """Without the edge hash set (allocation failure path) the CSR binary-search
    probes give the same histograms."""
    from paper_2212_04551_b200 import run_motifs
    monkeypatch.setenv("WM_NO_EDGE_HASH", "1")
    for i, (g, e, r) in enumerate(_cases(golden)):
        if i % 7:
            continue
        got = run_motifs(g, r["k"], dictionary(r["k"]), mode="opt")
        assert got.pattern_counts == r["hist"], (e["name"], r["k"])
