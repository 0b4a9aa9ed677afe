"""Balancer knobs on a full and a 1/8-shard motif run (cfg5 k=7 suffix 32768):
python scripts/probe_motif_lb.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
cfg, k, suf = (sys.argv[1], int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else ("cfg5", 7, 32768)
g = synth.config_graph(cfg); d = build_dictionary(k)
for thr in (1.0, 0.95, 0.85):
    for poll in (2, 8):
        mo = BalanceConfig(threshold=thr, poll_interval=poll)
        out = {"thr": thr, "poll": poll}
        for sh in ((0, 1), (0, 8), (3, 8)):
            rs = [run_motifs(g, k, d, mode="opt", balance_config=mo, roots=(g.n - suf, g.n),
                             shard=sh, reduce=False) for _ in range(3)]
            r = min(rs[1:], key=lambda r: r.kernel_ms)
            out["%d/%d" % sh] = [round(r.kernel_ms, 3), round(r.idle_warp_fraction, 3), r.migrations]
        print(json.dumps(out), flush=True)
