"""Secondary measurements beside bench.py's headline (one JSON line each):
configs 4-5, motif load balancing before/after, listing throughput, the k=8
dictionary build and graph ingest.  Kernel times are CUDA events inside
wm_run (``kernel_ms``); every count is checked against the pinned golden.

    python scripts/bench_extras.py [--quick] > profiles/rNN_extras.jsonl
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2212_04551_b200 import (BalanceConfig, build_dictionary, listing_checksum,  # noqa: E402
                                   run_clique, run_motifs, synth)
from paper_2212_04551_b200.graph import CsrGraph, load_edge_list  # noqa: E402

quick = "--quick" in sys.argv
golden = json.load(open(os.path.join(ROOT, "tests", "golden", "scale_golden.json")))
OPT = BalanceConfig(threshold=1.0, poll_interval=32)


def emit(**kw):
    print(json.dumps(kw), flush=True)


def best(fn, reps=3):
    out = None
    for _ in range(reps):
        r = fn()
        out = r if out is None or r.kernel_ms < out.kernel_ms else out
    return out


# ---- config 5: k-clique on R-MAT scale 22 ---------------------------------
t = time.time()
g5 = synth.config_graph("cfg5")
emit(what="cfg5 graph build (numpy R-MAT + wm_csr_build)", n=g5.n, m=g5.m, seconds=time.time() - t)
for k in ((8, 12) if quick else (5, 8, 10, 12)):
    r = best(lambda: run_clique(g5, k, mode="opt", balance_config=OPT), 2)
    want = golden["cfg5"]["clique"][str(k)]["count"]
    emit(what="cfg5 clique", k=k, count=r.clique_count, matches_golden=r.clique_count == want,
         kernel_ms=r.kernel_ms, subgraphs_per_s=r.clique_count / (r.kernel_ms * 1e-3),
         idle_warp_fraction=r.idle_warp_fraction, device_ms=r.device_ms)

# ---- motif load balancing before / after (north star: idle-warp fraction) --
# the cfg5 k=7 "wc" run is a single hub subtree on one warp (~200 s): --full
cases = [("cfg4", 5, "k5_s16384")] + ([("cfg5", 7, "k7_s32768")] if "--full" in sys.argv else [])
for cfg, k, key in cases:
    g = synth.config_graph(cfg)
    want = golden[cfg]["motif_suffix"][key]
    roots = (g.n - want["suffix"], g.n)
    d = build_dictionary(k)
    for mode, kw in (("wc", {}), ("opt", {"balance_config": BalanceConfig(threshold=1.0,
                                                                          poll_interval=2)})):
        r = best(lambda: run_motifs(g, k, d, mode=mode, roots=roots, **kw), 1 if mode == "wc" else 2)
        emit(what="%s motif root suffix" % cfg, k=k, suffix=want["suffix"], mode=mode,
             leaves=r.aggregated_total, matches_golden=r.pattern_counts == want["hist"],
             kernel_ms=r.kernel_ms, subgraphs_per_s=r.aggregated_total / (r.kernel_ms * 1e-3),
             idle_warp_fraction=r.idle_warp_fraction,
             idle_warp_fraction_tail=r.idle_warp_fraction_tail, migrations=r.migrations,
             warps=r.warps)

g2 = synth.config_graph("cfg2")
for k in (4, 5, 6):
    r = best(lambda: run_motifs(g2, k, build_dictionary(k)))
    ok = True if k == 4 else r.pattern_counts == golden["cfg2"]["motif"][str(k)]["hist"]
    emit(what="cfg2 motif", k=k, leaves=r.aggregated_total, matches_golden=ok,
         kernel_ms=r.kernel_ms, subgraphs_per_s=r.aggregated_total / (r.kernel_ms * 1e-3))

# ---- listing: records streamed device -> mapped host ring -> consumer ------
for cfg, k in (("cfg2", 6), ("cfg1", 6)):
    g = synth.config_graph(cfg)
    lbc = BalanceConfig(threshold=1.0, poll_interval=2)
    listing_checksum(g, k, mode="opt", balance_config=lbc)  # warm
    t = time.perf_counter()
    r = listing_checksum(g, k, mode="opt", balance_config=lbc)
    dt = time.perf_counter() - t
    emit(what="%s listing (native consumer: count + checksum)" % cfg, k=k,
         records=r.records_emitted, seconds=dt, records_per_s=r.records_emitted / dt,
         kernel_ms=r.kernel_ms, bytes_to_host=r.extra["d2h_bytes"],
         host_GBps=r.extra["d2h_bytes"] / dt / 1e9)

# ---- dictionary build on the device (k=8: 2^27 entries, 11,117 classes) ----
for k in (7, 8):
    t = time.perf_counter()
    d = build_dictionary(k, allow_large=True, device=True)
    emit(what="dictionary build on device", k=k, patterns=d.pattern_count,
         seconds=time.perf_counter() - t)
t = time.perf_counter()
build_dictionary(7, device=False)
emit(what="dictionary build on host (reference algorithm)", k=7,
     seconds=time.perf_counter() - t)
d8 = build_dictionary(8, allow_large=True)
g = synth.gnp_random_graph(3300, 4500 / 5443350 * 2, 2)
r = best(lambda: run_motifs(g, 8, d8))
emit(what="k=8 motif (ER 3300, avg degree ~5.5)", leaves=r.aggregated_total, kernel_ms=r.kernel_ms,
     subgraphs_per_s=r.aggregated_total / (r.kernel_ms * 1e-3))

# ---- ingest: endpoints -> CSR, and edge-list text -> CSR -------------------
rng = np.random.default_rng(1)
n, m = 1 << 22, 1 << 25
src, dst = rng.integers(0, n, m), rng.integers(0, n, m)
CsrGraph.from_arrays(n, src[:1000], dst[:1000], device=True)  # warm
t = time.perf_counter()
gd = CsrGraph.from_arrays(n, src, dst, device=True)
td = time.perf_counter() - t
t = time.perf_counter()
gh = CsrGraph.from_arrays(n, src, dst)
th = time.perf_counter() - t
emit(what="CSR build from 33.5M endpoint pairs", n=n, m=gd.m, device_s=td, host_numpy_s=th,
     identical=bool(np.array_equal(gd.offsets, gh.offsets)
                    and np.array_equal(gd.neighbors_array, gh.neighbors_array)))
g3 = synth.config_graph("cfg3")
text = "".join("%d %d\n" % (u, v) for u, v in g3.edge_array().tolist()).encode()
t = time.perf_counter()
gp = load_edge_list(__import__("io").StringIO(text.decode()), device=True)
tdev = time.perf_counter() - t
t = time.perf_counter()
gq = load_edge_list(__import__("io").StringIO(text.decode()))
thost = time.perf_counter() - t
emit(what="edge-list parse (cfg3 text, %d bytes)" % len(text), device_s=tdev, host_s=thost,
     identical=bool(np.array_equal(gp.neighbors_array, gq.neighbors_array)))
