import sys, time
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import run_motifs, synth, BalanceConfig, build_dictionary
for name, ks in (("cfg2", (4, 5, 6, 7)), ("cfg1", (4, 5, 6, 7))):
    g = synth.config_graph(name)
    for k in ks:
        d = build_dictionary(k)
        for mode in ("wc", "opt"):
            kw = {"balance_config": BalanceConfig(threshold=1.0, poll_interval=8)} if mode == "opt" else {}
            r = run_motifs(g, k, d, mode=mode, **kw)
            print(name, k, mode, r.aggregated_total, "kernel_ms=%.2f rate=%.3e idle=%.3f mig=%d warps=%d" % (
                r.kernel_ms, r.subgraphs_per_second, r.idle_warp_fraction, r.migrations, r.warps), r.extra, flush=True)
