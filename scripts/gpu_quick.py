import sys, time
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import run_clique, synth, BalanceConfig
g = synth.config_graph("cfg3")
ks = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [5, 6, 7, 8, 9]
polls = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8]
for k in ks:
    runs = [("wc", None)] + [("opt", p) for p in polls]
    for mode, p in runs:
        kw = {"balance_config": BalanceConfig(threshold=1.0, poll_interval=p)} if mode == "opt" else {}
        r = run_clique(g, k, mode=mode, **kw)
        print(k, mode, p, r.clique_count, "kernel_ms=%.2f dev_ms=%.2f rate=%.3e idle=%.3f tail=%.3f mig=%d dons=%d warps=%d" % (
            r.kernel_ms, r.device_ms, r.subgraphs_per_second, r.idle_warp_fraction,
            r.idle_warp_fraction_tail, r.migrations, r.rebalance_count, r.warps), r.extra, flush=True)
