"""A/B of library builds on a motif workload's full run and its N-shard balance
(slowest of N shards run one after another on one GPU):
    python scripts/ab_motif_shard.py CFG K SUFFIX N lib1.so lib2.so ..."""
import json, os, subprocess, sys
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
    cfg, k, suf, N = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    g = synth.config_graph(cfg); d = build_dictionary(k)
    mo = BalanceConfig(threshold=1.0, poll_interval=4 if k <= 5 else 8)
    def best(sh):
        rs = [run_motifs(g, k, d, mode="opt", balance_config=mo, roots=(g.n - suf, g.n),
                         shard=sh, reduce=False) for _ in range(3)]
        return min(rs[1:], key=lambda r: r.device_ms)
    one = best((0, 1))
    rs = [best((r, N)) for r in range(N)]
    print(json.dumps({"full_kernel_ms": round(one.kernel_ms, 3), "full_device_ms": round(one.device_ms, 3),
                      "max_shard_ms": round(max(r.device_ms for r in rs), 3),
                      "shard_ms": [round(r.device_ms, 3) for r in rs],
                      "speedup": round(one.device_ms / max(r.device_ms for r in rs), 3),
                      "ok": sum(r.aggregated_total for r in rs) == one.aggregated_total}))
    sys.exit(0)
cfg, k, suf, N = sys.argv[1:5]
for lib in sys.argv[5:]:
    env = dict(os.environ, WM_B200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, __file__, "--one", cfg, k, suf, N], env=env,
                         capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip() or out.stderr[-500:], flush=True)
