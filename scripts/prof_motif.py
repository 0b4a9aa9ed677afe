"""Warm motif run for ncu capture: prof_motif.py CFG K [SUFFIX]."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
name, k = sys.argv[1], int(sys.argv[2])
suffix = int(sys.argv[3]) if len(sys.argv) > 3 else 0
g = synth.config_graph(name)
d = build_dictionary(k)
roots = (g.n - suffix, g.n) if suffix else None
bc = BalanceConfig(threshold=1.0, poll_interval=8)
for _ in range(2):
    r = run_motifs(g, k, d, mode="opt", balance_config=bc, roots=roots)
print(r.aggregated_total, r.kernel_ms)
