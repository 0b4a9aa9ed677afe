"""Generate golden parity fixtures by running the REFERENCE itself.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Writes ``tests/golden/reference_golden.json``.  Every number in it comes from
``warpmine`` (the reference package, imported read-only): ``engine.run`` in
mode "wc" for counts/histograms, ``build_dictionary(...).save`` for dictionary
digests, and a hook on ``engine.Lane.aggregate`` to record the leaf-bearing
traversals from which the SURVEY §8(d) algorithmic-byte figure B_alg is
derived.  Graph digests pin the exact input (our ``synth`` module regenerates
the same graphs; tests check the digest before comparing counts).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import warpmine  # noqa: E402  (the reference)
from warpmine import engine  # noqa: E402
from warpmine.apps import clique_app, motif_app  # noqa: E402
from warpmine.balance import BalanceConfig  # noqa: E402
from warpmine.graph import CsrGraph as RefGraph  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")


def graph_digest(offsets, neighbors) -> str:
    h = hashlib.sha256()
    h.update(np.asarray(offsets, dtype="<i8").tobytes())
    h.update(np.asarray(neighbors, dtype="<i4").tobytes())
    return h.hexdigest()


_LEAF_TRS: list = []


def _hooked_aggregate(self, _orig=engine.Lane.aggregate):
    before = self.warp.leaves
    _orig(self)
    found = self.warp.leaves - before
    if found:
        _LEAF_TRS.append(tuple(self.te.tr[:self.te.len]))


engine.Lane.aggregate = _hooked_aggregate


def b_alg(g, leaf_trs, motif: bool) -> int:
    """4 B * sum over productive nodes of deg+(last) (clique, id order) or
    deg(last) (motif).  Productive nodes = all prefixes of leaf-bearing
    (k-1)-traversals (each traversal is a unique tree node)."""
    nodes = set()
    for tr in leaf_trs:
        for L in range(1, len(tr) + 1):
            nodes.add(tr[:L])
    adj = g.adjacency_lists()
    total = 0
    for t in nodes:
        last = t[-1]
        total += len(adj[last]) if motif else sum(1 for u in adj[last] if u > last)
    return 4 * total


def run_case(g, k, app, dicts, mode="wc", **kw):
    _LEAF_TRS.clear()
    if app == "clique":
        r = engine.run(g, clique_app(k), mode=mode, **kw)
        rec = {"count": r.clique_count}
    else:
        r = engine.run(g, motif_app(k, dicts[k]), mode=mode, **kw)
        rec = {"hist": list(r.pattern_counts)}
    rec["leaves"] = r.aggregated_total
    rec["alg_bytes"] = b_alg(g, list(_LEAF_TRS), app == "motif")
    return rec


def entry(name, g, cases, dicts):
    out = {"name": name, "n": g.n, "m": g.m,
           "digest": graph_digest(g.offsets, g.neighbors_array),
           "edges": [list(e) for e in g.edges()] if g.m <= 5000 else None,
           "results": []}
    for app, k in cases:
        t = time.time()
        rec = run_case(g, k, app, dicts)
        rec.update({"app": app, "k": k})
        out["results"].append(rec)
        print("  %-28s %-6s k=%d leaves=%d (%.2fs)" % (name, app, k, rec["leaves"], time.time() - t),
              flush=True)
    return out


def main():
    dicts = {k: warpmine.build_dictionary(k) for k in range(3, 8)}
    golden = {"generator": "warpmine (reference) engine.run mode=wc", "dictionaries": {},
              "graphs": []}
    for k, d in dicts.items():
        path = "/tmp/_golden_dict_%d.dmcd" % k
        d.save(path)
        blob = open(path, "rb").read()
        golden["dictionaries"][str(k)] = {
            "sha256": hashlib.sha256(blob).hexdigest(), "bytes": len(blob),
            "pattern_count": d.pattern_count, "canonical_bitmaps": list(d.canonical_bitmaps)}
    S = warpmine.synth
    small = [
        ("G1", RefGraph.from_edges(5, [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3), (3, 4)])),
        ("K4", S.complete_graph(4)), ("K5", S.complete_graph(5)), ("K6", S.complete_graph(6)),
        ("K8", S.complete_graph(8)),
        ("P4", S.path_graph(4)), ("P6", S.path_graph(6)),
        ("star_of_cliques_4_5", S.star_of_cliques(4, 5)),
        ("star_of_cliques_6_7", S.star_of_cliques(6, 7)),
        ("isolated_plus_edge", RefGraph.from_edges(6, [(2, 4)])),
    ]
    for name, g in small:
        kmax = min(8, max(3, g.max_degree + 1))
        cases = [("clique", k) for k in range(3, kmax + 1)]
        cases += [("motif", k) for k in range(3, min(7, g.n) + 1)
                  if not (name.startswith("star_of_cliques_6") and k > 5)]
        golden["graphs"].append(entry(name, g, cases, dicts))
    # acceptance corpus (reference tests/test_acceptance.py:28-31)
    for n, p in [(20, 0.1), (14, 0.3), (10, 0.6)]:
        for seed in range(20):
            g = S.gnp_random_graph(n, p, seed=seed)
            cases = [(a, k) for k in (3, 4, 5) for a in ("clique", "motif")]
            if seed < 4:
                cases += [("motif", 6), ("motif", 7), ("clique", 6)]
            golden["graphs"].append(entry("gnp_%d_%.1f_%d" % (n, p, seed), g, cases, dicts))
    # medium graphs: more leaves, deeper trees
    for name, g, cases in [
        ("gnp_300_0.1_1", S.gnp_random_graph(300, 0.1, 1), [("clique", 3), ("clique", 4), ("clique", 5)]),
        ("gnp_40_0.2_7", S.gnp_random_graph(40, 0.2, 7), [("motif", 4), ("motif", 5), ("motif", 6)]),
        ("gnp_60_0.3_5", S.gnp_random_graph(60, 0.3, 5), [("clique", k) for k in range(3, 8)]
         + [("motif", 4), ("motif", 5)]),
        ("gnp_120_0.05_9", S.gnp_random_graph(120, 0.05, 9), [("motif", 3), ("motif", 4), ("motif", 5)]),
    ]:
        golden["graphs"].append(entry(name, g, cases, dicts))
    # BASELINE.json configs 1 and 2
    for seed in range(5):
        g = S.gnp_random_graph(516, 1200 / 132870, seed)
        golden["graphs"].append(entry("cfg1_seed%d" % seed, g,
                                      [("clique", 3), ("clique", 4), ("motif", 3), ("motif", 4)], dicts))
    for seed in range(3):
        g = S.gnp_random_graph(3300, 4500 / 5443350, seed)
        golden["graphs"].append(entry("cfg2_seed%d" % seed, g,
                                      [("motif", 4), ("clique", 3), ("motif", 3)], dicts))
    # forced rebalancing conserves results (reference test_acceptance.py:115-147)
    g = S.star_of_cliques(6, 7)
    forced = {}
    for app, k in [("clique", 5), ("motif", 4)]:
        _LEAF_TRS.clear()
        a = (clique_app(k) if app == "clique" else motif_app(k, dicts[k]))
        r = engine.run(g, a, mode="opt", warps=8,
                       balance_config=BalanceConfig(threshold=1.0, poll_interval=1))
        forced["%s_%d" % (app, k)] = {"count": r.clique_count, "hist": r.pattern_counts,
                                      "rebalance_count": r.rebalance_count,
                                      "migrations": r.migrations}
    golden["forced_rebalance_star_of_cliques_6_7"] = forced
    with open(OUT, "w") as fh:
        json.dump(golden, fh, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
