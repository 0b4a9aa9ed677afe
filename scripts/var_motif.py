"""Run-to-run variance of motif kernel times: python scripts/var_motif.py CFG K REPS [SUFFIX]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
cfg, k, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
suffix = int(sys.argv[4]) if len(sys.argv) > 4 else 0
g = synth.config_graph(cfg)
d = build_dictionary(k)
roots = (g.n - suffix, g.n) if suffix else None
bc = BalanceConfig(threshold=0.9, poll_interval=8)
ms = []
for i in range(reps):
    r = run_motifs(g, k, d, mode="opt", balance_config=bc, roots=roots)
    ms.append(round(r.kernel_ms, 3))
print(cfg, k, "idle %.3f" % r.idle_warp_fraction, "warps", r.warps, ms, flush=True)
