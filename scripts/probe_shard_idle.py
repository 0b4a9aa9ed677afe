"""Idle accounting of one clique shard vs the whole run (ramp/tail vs
replicated work): python scripts/probe_shard_idle.py CFG K N"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
cfg, k, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
g = synth.config_graph(cfg)
for poll in (32, 8):
    bc = BalanceConfig(threshold=1.0, poll_interval=poll)
    for sh in ((0, 1), (0, N), (N - 1, N)):
        r = min((run_clique(g, k, mode="opt", balance_config=bc, shard=sh, reduce=False)
                 for _ in range(3)), key=lambda r: r.kernel_ms)
        print(json.dumps({"poll": poll, "shard": sh, "kernel_ms": round(r.kernel_ms, 3),
                          "device_ms": round(r.device_ms, 3), "idle": round(r.idle_warp_fraction, 3),
                          "idle_tail": round(r.idle_warp_fraction_tail, 3), "tasks": r.tasks,
                          "migr": r.migrations, "don": r.rebalance_count,
                          "busy_warp_ms": round(r.kernel_ms * (1 - r.idle_warp_fraction), 3)}), flush=True)
