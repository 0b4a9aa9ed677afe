"""One warm k-clique run on cfg3 for ncu capture (the profiled launch is the
second enumeration kernel launch)."""
import sys
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = synth.config_graph("cfg3")
bc = BalanceConfig(threshold=1.0, poll_interval=32)
for _ in range(2):
    r = run_clique(g, k, mode="opt", balance_config=bc)
print(r.clique_count, r.kernel_ms)
