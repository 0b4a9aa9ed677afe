"""Golden values at benchmark scale (configs 3-5), from the CPU restatement.

The Python reference is 1e5-1e6x too slow here, so these
numbers come from ``oracle/`` — ``wmo_clique_fast`` (degree-ordered kClist)
and ``wmo_motif_run`` (the engine restatement) — both pinned bit-exact to the
reference on the 508 cases of ``reference_golden.json`` (tests/test_oracle.py).
Where feasible the faithful id-order restatement ``wmo_clique_run`` re-derives
the same count as a second, independent path.

    python tests/golden/make_golden_scale.py [--kmax 9]

Writes ``tests/golden/scale_golden.json``.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2212_04551_b200 import canon, synth  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "scale_golden.json")


def digest(g) -> str:
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype="<i8").tobytes())
    h.update(np.asarray(g.neighbors_array, dtype="<i4").tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kmax", type=int, default=9)
    ap.add_argument("--cfg5", action="store_true", help="also the (long) cfg5 section")
    args = ap.parse_args()
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    g = synth.config_graph("cfg3")
    rec = out.setdefault("cfg3", {})
    rec.update({"n": g.n, "m": g.m, "max_degree": g.max_degree, "digest": digest(g),
                "recipe": "chung_lu(100000, 1000000, 2.3, seed=3)"})
    cl = rec.setdefault("clique", {})
    for k in range(3, args.kmax + 1):
        if str(k) in cl:
            continue
        t = time.time()
        c, b = oracle.clique_fast(g, k, with_bytes=True)
        cl[str(k)] = {"count": c, "alg_bytes_degree_order": b, "oracle": "wmo_clique_fast",
                      "cpu_s": round(time.time() - t, 2)}
        print("cfg3 clique k=%d count=%d bytes=%d %.1fs" % (k, c, b, time.time() - t), flush=True)
        json.dump(out, open(OUT, "w"), indent=1)
    if "id_order_k3" not in rec:
        t = time.time()
        r = oracle.clique_run(g, 3)
        rec["id_order_k3"] = {"count": r["count"], "alg_bytes_id_order": r["alg_bytes"],
                              "oracle": "wmo_clique_run", "cpu_s": round(time.time() - t, 2)}
        assert r["count"] == cl["3"]["count"], (r, cl["3"])
        json.dump(out, open(OUT, "w"), indent=1)
    # cfg2 (citeseer-sized) motif k=5,6 and cfg1 motif k=5: exhaustive
    for name, ks in (("cfg2", (5, 6)), ("cfg1", (5, 6))):
        gg = synth.config_graph(name)
        r2 = out.setdefault(name, {"digest": digest(gg), "n": gg.n, "m": gg.m})
        mo = r2.setdefault("motif", {})
        for k in ks:
            if str(k) in mo:
                continue
            d = canon.build_dictionary(k)
            t = time.time()
            r = oracle.motif_run(gg, k, d.table, d.pattern_count)
            mo[str(k)] = {"hist": r["hist"], "leaves": r["leaves"], "alg_bytes": r["alg_bytes"],
                          "cpu_s": round(time.time() - t, 2)}
            print("%s motif k=%d leaves=%d %.1fs" % (name, k, r["leaves"], time.time() - t), flush=True)
            json.dump(out, open(OUT, "w"), indent=1)
    # cfg4 (R-MAT s20 ef16, Graph500 skew, permuted ids): root suffixes
    # [n - s, n) == the induced subgraph on the last s ids
    g4 = synth.config_graph("cfg4")
    r4 = out.setdefault("cfg4", {})
    r4.update({"digest": digest(g4), "n": g4.n, "m": g4.m, "max_degree": g4.max_degree,
               "recipe": "rmat(20, 16, a=.57, b=.19, c=.19, seed=1), ids permuted (seed 20)"})
    suf = r4.setdefault("motif_suffix", {})
    for k, s in ((5, 16384), (6, 4096), (5, 4096), (7, 2048), (6, 8192), (6, 16384)):
        key = "k%d_s%d" % (k, s)
        if key in suf:
            continue
        d = canon.build_dictionary(k)
        t = time.time()
        r = oracle.motif_run(g4, k, d.table, d.pattern_count, root_begin=g4.n - s, root_end=g4.n)
        suf[key] = {"k": k, "suffix": s, "hist": r["hist"], "leaves": r["leaves"],
                    "cpu_s": round(time.time() - t, 2), "oracle": "wmo_motif_run"}
        print("cfg4 motif %s leaves=%d %.1fs" % (key, r["leaves"], time.time() - t), flush=True)
        json.dump(out, open(OUT, "w"), indent=1)
    # cfg5 (R-MAT s22 ef8, a=.52 b=c=.20, permuted ids): clique k=3..12
    # exhaustive (kClist), motif k=5/7 over root suffixes
    if args.cfg5:
        g5 = synth.config_graph("cfg5")
        r5 = out.setdefault("cfg5", {})
        r5.update({"digest": digest(g5), "n": g5.n, "m": g5.m, "max_degree": g5.max_degree,
                   "recipe": "rmat(22, 8, a=.52, b=.20, c=.20, seed=1), ids permuted (seed 22)"})
        cl5 = r5.setdefault("clique", {})
        for k in range(3, 13):
            if str(k) in cl5:
                continue
            t = time.time()
            c = oracle.clique_fast(g5, k)
            cl5[str(k)] = {"count": c, "oracle": "wmo_clique_fast", "cpu_s": round(time.time() - t, 2)}
            print("cfg5 clique k=%d count=%d %.1fs" % (k, c, time.time() - t), flush=True)
            json.dump(out, open(OUT, "w"), indent=1)
        suf5 = r5.setdefault("motif_suffix", {})
        # suffix sizes: the largest power of two whose induced subgraph has a
        # star lower bound sum_v C(deg_suffix(v), k-1) <= 2e9 (CPU-feasible)
        from math import comb
        src = np.repeat(np.arange(g5.n), np.diff(g5.offsets))
        dst = np.asarray(g5.neighbors_array)

        def stars(s, k):
            keep = (src >= g5.n - s) & (dst >= g5.n - s)
            deg = np.bincount(src[keep], minlength=g5.n)
            return sum(comb(int(d), k - 1) for d in deg[deg >= k - 1])

        plan = []
        for k in (5, 6, 7):
            s = 1 << 22
            while s > 1024 and stars(s, k) > 2e9:
                s >>= 1
            plan.append((k, s))
        for k, s in plan:
            key = "k%d_s%d" % (k, s)
            if key in suf5:
                continue
            d = canon.build_dictionary(k)
            t = time.time()
            r = oracle.motif_run(g5, k, d.table, d.pattern_count, root_begin=g5.n - s,
                                 root_end=g5.n)
            suf5[key] = {"k": k, "suffix": s, "hist": r["hist"], "leaves": r["leaves"],
                         "cpu_s": round(time.time() - t, 2), "oracle": "wmo_motif_run"}
            print("cfg5 motif %s leaves=%d %.1fs" % (key, r["leaves"], time.time() - t), flush=True)
            json.dump(out, open(OUT, "w"), indent=1)
    json.dump(out, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
