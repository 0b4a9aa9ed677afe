"""Expectations on the BASELINE config graphs produced by the REFERENCE itself
(``warpmine``, imported read-only from /root/reference), not by the C
restatement — SURVEY §8(c): "Python-feasible root suffixes run by the
reference".

The reference engine is exact on any graph but ~1e5x slower than the device,
so it runs on slices of configs 3-5 that finish in about a minute:

* cliques, cfg3 (ids NOT permuted: vertex 0 is the heaviest): a root-id
  range [b, e) of the FULL graph through the reference's own queue hook —
  ``_Context.queue`` replaced by ``deque(range(b, e))`` and the warp driven by
  ``run_warp`` (``engine.py:160-191``, ``:740-743``; the hook of
  ``pkg/tests/test_engine.py:300``).  The device reproduces it with
  ``run_clique(g, k, order="id", roots=(b, e))``.
* motifs, cfg4 / cfg5 (ids permuted): a root suffix [n - s, n).  Under the
  canonical rule every vertex of a traversal is >= its root
  (``canon.py:190-210``), so the suffix run IS the run on the induced
  subgraph of the last s ids; ids are relabeled order-preservingly
  (v -> v - (n - s)), which keeps the traversal tree identical, and the
  reference ``engine.run`` runs on that graph.  Device: ``run_motifs(g, k, d,
  roots=(n - s, n))`` on the full graph.
* cliques, cfg5: a root suffix in id order, likewise the induced subgraph.

    WM_HOST_BUILD=1 python tests/golden/make_golden_ref_scale.py

Writes ``tests/golden/ref_scale_golden.json`` (graph digests included).
"""

from __future__ import annotations

import collections
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF = "/root/reference/pkg/src"
sys.path.insert(0, ROOT)
sys.path.insert(0, REF)
os.environ.setdefault("WM_HOST_BUILD", "1")

from paper_2212_04551_b200 import synth  # noqa: E402
import warpmine  # noqa: E402
from warpmine import apps as ref_apps, canon as ref_canon, engine as ref_engine  # noqa: E402
from warpmine.graph import CsrGraph as RefGraph  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_scale_golden.json")


def digest(g) -> str:
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype="<i8").tobytes())
    h.update(np.asarray(g.neighbors_array, dtype="<i4").tobytes())
    return h.hexdigest()


def to_ref(g) -> "RefGraph":
    return RefGraph(g.n, np.asarray(g.offsets, dtype=np.int64).copy(),
                    np.asarray(g.neighbors_array, dtype=np.int64).copy())


def induced_suffix(g, s):
    """Induced subgraph on ids [n - s, n), relabeled v -> v - (n - s)."""
    lo = g.n - s
    src = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.offsets))
    dst = np.asarray(g.neighbors_array, dtype=np.int64)
    keep = (src >= lo) & (dst >= lo)
    src, dst = src[keep] - lo, dst[keep] - lo
    counts = np.bincount(src, minlength=s)
    off = np.zeros(s + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    order = np.lexsort((dst, src))
    return RefGraph(s, off, dst[order])


def ref_clique_roots(rg, k, b, e):
    """Reference engine over roots [b, e) of the full graph (queue hook)."""
    ctx = ref_engine._Context(rg, ref_apps.clique_app(k), ref_engine.DEFAULT_LANE_WIDTH)
    ctx.queue = collections.deque(range(b, e))
    w = ref_engine.WarpState(0, "wc", ctx)
    ref_engine.run_warp(w)
    return w.clique_count, w.leaves


def main():
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    out["reference"] = {"package": "warpmine %s" % getattr(warpmine, "__version__", "?"),
                        "path": REF}
    dicts = {}

    def dictionary(k):
        if k not in dicts:
            dicts[k] = ref_canon.build_dictionary(k)
        return dicts[k]

    def save():
        json.dump(out, open(OUT, "w"), indent=1)

    # cfg3 cliques: root-id ranges of the full graph, id order
    g3 = synth.config_graph("cfg3")
    r3 = out.setdefault("cfg3", {"digest": digest(g3), "n": g3.n, "m": g3.m})
    cl = r3.setdefault("clique_roots", {})
    rg3 = None
    for k, b, e in ((3, 50, 60), (4, 30, 31), (4, 100, 120), (5, 100, 120), (6, 100, 120)):
        key = "k%d_r%d_%d" % (k, b, e)
        if key in cl:
            continue
        if rg3 is None:
            rg3 = to_ref(g3)
        t = time.time()
        c, leaves = ref_clique_roots(rg3, k, b, e)
        cl[key] = {"k": k, "roots": [b, e], "count": c, "leaves": leaves,
                   "ref_s": round(time.time() - t, 1), "order": "id"}
        print("cfg3 clique %s count=%d %.1fs" % (key, c, time.time() - t), flush=True)
        save()
    # cfg4 / cfg5 motifs: root suffixes = induced subgraphs of the last s ids
    for name, plan in (("cfg4", ((5, 4096), (6, 4096), (7, 2048), (5, 6144))),
                       ("cfg5", ((5, 32768), (6, 16384), (7, 16384)))):
        g = synth.config_graph(name)
        rec = out.setdefault(name, {"digest": digest(g), "n": g.n, "m": g.m})
        mo = rec.setdefault("motif_suffix", {})
        for k, s in plan:
            key = "k%d_s%d" % (k, s)
            if key in mo:
                continue
            sub = induced_suffix(g, s)
            t = time.time()
            r = ref_engine.run(sub, ref_apps.motif_app(k, dictionary(k)), mode="wc")
            mo[key] = {"k": k, "suffix": s, "hist": list(r.pattern_counts),
                       "leaves": r.aggregated_total, "sub_m": sub.m,
                       "ref_s": round(time.time() - t, 1)}
            print("%s motif %s leaves=%d (sub m=%d) %.1fs" % (name, key, r.aggregated_total,
                                                              sub.m, time.time() - t), flush=True)
            save()
    g5 = synth.config_graph("cfg5")
    cq = out["cfg5"].setdefault("clique_suffix", {})
    for k, s in ((3, 262144), (4, 262144), (5, 524288)):
        key = "k%d_s%d" % (k, s)
        if key in cq:
            continue
        sub = induced_suffix(g5, s)
        t = time.time()
        r = ref_engine.run(sub, ref_apps.clique_app(k), mode="wc")
        cq[key] = {"k": k, "suffix": s, "count": r.clique_count, "sub_m": sub.m,
                   "ref_s": round(time.time() - t, 1), "order": "id"}
        print("cfg5 clique %s count=%d (sub m=%d) %.1fs" % (key, r.clique_count, sub.m,
                                                            time.time() - t), flush=True)
        save()
    save()


if __name__ == "__main__":
    main()
