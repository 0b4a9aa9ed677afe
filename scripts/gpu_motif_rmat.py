"""Root-suffix motif runs on config 4 (R-MAT scale 20, ef 16, Graph500 skew,
random id permutation): roots [n - s, n) for growing s."""
import sys, time
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import run_motifs, synth, BalanceConfig, build_dictionary
t = time.time()
g = synth.config_graph("cfg4")
print("cfg4", g, "%.1fs" % (time.time() - t), flush=True)
ks = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [5]
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1 << 12, 1 << 14, 1 << 16]
for k in ks:
    d = build_dictionary(k)
    for s in sizes:
        for mode in ("opt",):
            kw = {"balance_config": BalanceConfig(threshold=1.0, poll_interval=8)} if mode == "opt" else {}
            t = time.time()
            r = run_motifs(g, k, d, mode=mode, roots=(g.n - s, g.n), **kw)
            print(k, s, mode, r.aggregated_total, "kernel_ms=%.2f wall=%.2f rate=%.3e idle=%.3f mig=%d warps=%d" % (
                r.kernel_ms, time.time() - t, r.subgraphs_per_second, r.idle_warp_fraction, r.migrations, r.warps),
                r.extra, flush=True)
