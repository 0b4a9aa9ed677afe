"""Small golden cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every product kernel family on graphs small enough for the
instrumented run, with the on-device balancer forced to fire (threshold 1.0,
poll 1) so donation records move between warps.  Each case is checked
against the oracle; exits non-zero on any mismatch.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2212_04551_b200 import (BalanceConfig, CsrGraph, build_dictionary,  # noqa: E402
                                   gnp_random_graph, listing_checksum, run_clique, run_motifs,
                                   star_of_cliques)

LB = BalanceConfig(threshold=1.0, poll_interval=1)
bad = []


def check(name, got, want):
    if got != want:
        bad.append((name, got, want))
    print("%-40s %s" % (name, "ok" if got == want else "MISMATCH %r != %r" % (got, want)),
          flush=True)


graphs = {"gnp60": gnp_random_graph(60, 0.25, 3), "soc": star_of_cliques(4, 6)}
for gname, g in graphs.items():
    for k in (3, 4, 5):
        want = oracle.clique_run(g, k, threads=2)["count"]
        for mode in ("wc", "opt"):
            kw = {"balance_config": LB} if mode == "opt" else {}
            check("clique %s k=%d %s" % (gname, k, mode),
                  run_clique(g, k, mode=mode, **kw).clique_count, want)
        check("clique %s k=%d id-order" % (gname, k),
              run_clique(g, k, mode="opt", balance_config=LB, order="id").clique_count, want)
    for k in (3, 4, 5, 6):
        d = build_dictionary(k)
        want = oracle.motif_run(g, k, d.table, d.pattern_count, threads=2)
        r = run_motifs(g, k, d, mode="opt", balance_config=LB)
        check("motif %s k=%d opt" % (gname, k), r.pattern_counts, want["hist"])
        # two shards (level-1 / level-2 dealing inside leaf_bulk): their sum
        parts = [run_motifs(g, k, d, mode="opt", balance_config=LB, shard=(r_, 2),
                            reduce=False).pattern_counts for r_ in range(2)]
        check("motif %s k=%d 2 shards" % (gname, k), [a + b for a, b in zip(*parts)],
              want["hist"])
        r = run_motifs(g, k, d, mode="opt", balance_config=LB, count_bytes=True)
        check("motif %s k=%d B_alg" % (gname, k), r.alg_bytes, want["alg_bytes"])
    for k in (3, 4):
        want = oracle.list_run(g, k, threads=2)
        r = listing_checksum(g, k, mode="opt", balance_config=LB)
        check("listing %s k=%d" % (gname, k), (r.records_emitted, r.extra["checksum"]),
              (want["emitted"], want["checksum"]))
# wide roots (> 1024 out-neighbours in id order): nested induced-subgraph runs
hub = 1100
src = np.concatenate([np.zeros(hub, np.int64), np.arange(1, hub, dtype=np.int64)])
dst = np.concatenate([np.arange(1, hub + 1, dtype=np.int64), np.arange(2, hub + 1, dtype=np.int64)])
gw = CsrGraph.from_arrays(hub + 1, src, dst)
check("clique wide root k=3 id-order", run_clique(gw, 3, order="id").clique_count,
      oracle.clique_run(gw, 3, threads=2)["count"])
# the C-ABI boundary rejects a malformed CSR (device validation pass)
try:
    from paper_2212_04551_b200 import _native
    import ctypes
    off = np.array([0, 2, 3, 4], np.int64)
    nbr = np.array([1, 2, 0, 1], np.int32)
    csr = _native.WmCsr(3, 4, off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                        nbr.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    h = ctypes.c_void_p()
    st = _native.load().wm_graph_create(ctypes.byref(csr), ctypes.byref(h))
    check("bad CSR rejected", st, _native.WM_EINVAL)
except Exception as exc:  # pragma: no cover
    bad.append(("bad CSR", repr(exc), None))
print("sanitize cases: %d mismatches" % len(bad), flush=True)
sys.exit(1 if bad else 0)
