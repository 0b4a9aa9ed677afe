"""Motif shard balance on one GPU, level-1 vs level-2 task dealing
(WM_MOTIF_SHARD_LEVEL): each of the N shards runs one after another; the
N-GPU step is the slowest shard.  python scripts/shard_motif_levels.py"""
import json, os, subprocess, sys
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
    cfg, k, suf = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    g = synth.config_graph(cfg)
    d = build_dictionary(k)
    mo = BalanceConfig(threshold=1.0, poll_interval=2)
    def best(sh):
        rs = [run_motifs(g, k, d, mode="opt", balance_config=mo, roots=(g.n - suf, g.n),
                         shard=sh, reduce=False) for _ in range(3)]
        return min(rs, key=lambda r: r.device_ms)
    base = None
    for N in (1, 2, 4, 8):
        rs = [best((r, N)) for r in range(N)]
        tot = sum(x.aggregated_total for x in rs)
        dmax = max(x.device_ms for x in rs)
        base = base or (dmax, tot)
        print(json.dumps({"workload": "%s k=%d suffix %d" % (cfg, k, suf),
                          "level": os.environ.get("WM_MOTIF_SHARD_LEVEL"), "shards": N,
                          "total_matches_1": tot == base[1],
                          "device_ms": [round(x.device_ms, 3) for x in rs],
                          "speedup_device": base[0] / dmax}), flush=True)
    sys.exit(0)
for cfg, k, suf in (("cfg5", 7, 32768), ("cfg4", 6, 16384), ("cfg4", 5, 16384)):
    for lvl in ("1", "2"):
        env = dict(os.environ, WM_MOTIF_SHARD_LEVEL=lvl)
        subprocess.run([sys.executable, __file__, "--one", cfg, str(k), str(suf)], env=env)
