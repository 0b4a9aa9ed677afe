"""Warps-per-block sweep of the clique kernels (cfg5: the W=8 class is
register-limited at 2 x 8 warps per SM)."""
import json, sys
sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
bc = BalanceConfig(threshold=1.0, poll_interval=32)
for cfg, k in (("cfg5", 8), ("cfg3", 9)):
    g = synth.config_graph(cfg)
    for wpb in (8, 4, 2):
        rs = [run_clique(g, k, mode="opt", balance_config=bc, warps_per_block=wpb) for _ in range(3)]
        r = min(rs, key=lambda x: x.kernel_ms)
        print(json.dumps({"cfg": cfg, "k": k, "wpb": wpb, "kernel_ms": round(r.kernel_ms, 3),
                          "warps": r.warps, "count": r.clique_count}), flush=True)
