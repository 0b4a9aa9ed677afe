"""One k-clique run of a config graph for ncu capture: prof_clique_cfg.py CFG K [RUNS]"""
import sys
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
g = synth.config_graph(sys.argv[1])
k = int(sys.argv[2])
bc = BalanceConfig(threshold=1.0, poll_interval=32)
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    r = run_clique(g, k, mode="opt", balance_config=bc)
print(r.clique_count, r.kernel_ms)
