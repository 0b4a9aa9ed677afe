import sys, time
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import run_motifs, synth, BalanceConfig, build_dictionary
polls = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8]
runs = [("cfg2", k, 0) for k in (4, 5, 6, 7)] + [("cfg1", k, 0) for k in (5, 6, 7)] + \
       [("cfg4", 5, 16384), ("cfg4", 6, 8192), ("cfg4", 5, 65536)]
graphs = {}
for name, k, s in runs:
    if name not in graphs:
        graphs[name] = synth.config_graph(name)
    g = graphs[name]
    d = build_dictionary(k)
    roots = (g.n - s, g.n) if s else None
    for mode, p in [("wc", None)] + [("opt", p) for p in polls]:
        if mode == "wc" and s >= 65536:
            continue
        kw = {"balance_config": BalanceConfig(threshold=1.0, poll_interval=p)} if mode == "opt" else {}
        r = run_motifs(g, k, d, mode=mode, roots=roots, **kw)
        r = run_motifs(g, k, d, mode=mode, roots=roots, **kw)
        print(name, k, s, mode, p, r.aggregated_total, "kernel_ms=%.3f rate=%.3e idle=%.3f mig=%d dons=%d warps=%d nodes=%d" % (
            r.kernel_ms, r.subgraphs_per_second, r.idle_warp_fraction, r.migrations, r.rebalance_count, r.warps, r.extra["nodes"]), flush=True)
