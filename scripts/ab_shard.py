"""A/B of library builds on the N-shard balance of a clique workload (slowest
shard of N run one after another on one GPU):
    python scripts/ab_shard.py CFG K N lib1.so lib2.so ..."""
import json, os, subprocess, sys
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
    cfg, k, N = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    g = synth.config_graph(cfg)
    bc = BalanceConfig(threshold=1.0, poll_interval=32)
    def best(sh):
        return min((run_clique(g, k, mode="opt", balance_config=bc, shard=sh, reduce=False)
                    for _ in range(3)), key=lambda r: r.device_ms)
    one = best((0, 1))
    rs = [best((r, N)) for r in range(N)]
    print(json.dumps({"k": k, "N": N, "single_ms": round(one.device_ms, 3),
                      "max_shard_ms": round(max(r.device_ms for r in rs), 3),
                      "kernel_ms": [round(r.kernel_ms, 3) for r in rs],
                      "speedup": one.device_ms / max(r.device_ms for r in rs),
                      "ok": sum(r.clique_count for r in rs) == one.clique_count}))
    sys.exit(0)
cfg, k, N = sys.argv[1], sys.argv[2], sys.argv[3]
for lib in sys.argv[4:]:
    env = dict(os.environ, WM_B200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, __file__, "--one", cfg, k, N], env=env,
                         capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip() or out.stderr[-500:], flush=True)
