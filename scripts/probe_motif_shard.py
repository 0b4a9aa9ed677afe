"""Idle/phase accounting of one motif shard vs the whole run (cfg5 k=7 suffix
32768): python scripts/probe_motif_shard.py (WM_B200_LIB=<prof build> adds the
per-phase cycle line on stderr)"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
g = synth.config_graph("cfg5"); k = 7; d = build_dictionary(k)
mo = BalanceConfig(threshold=1.0, poll_interval=2)
for sh in ((0, 1), (0, 8), (3, 8)):
    for _ in range(2):
        r = run_motifs(g, k, d, mode="opt", balance_config=mo, roots=(g.n - 32768, g.n),
                       shard=sh, reduce=False)
    print(json.dumps({"shard": sh, "kernel_ms": round(r.kernel_ms, 3),
                      "idle": round(r.idle_warp_fraction, 3), "leaves": r.aggregated_total,
                      "tasks": r.tasks, "migr": r.migrations}), flush=True)
