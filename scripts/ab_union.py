"""Union-graph path for the wide clique classes vs the W = 8..32 kernels
(WM_CLIQUE_UNION=0), cfg5 and cfg3 (id order: wide hub rows)."""
import json, os, subprocess, sys
if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
    cfg, k, order = sys.argv[2], int(sys.argv[3]), sys.argv[4]
    g = synth.config_graph(cfg)
    bc = BalanceConfig(threshold=1.0, poll_interval=32)
    rs = [run_clique(g, k, mode="opt", balance_config=bc, order=order) for _ in range(3)]
    r = min(rs[1:], key=lambda x: x.device_ms)
    print(json.dumps({"cfg": cfg, "k": k, "order": order,
                      "union": os.environ.get("WM_CLIQUE_UNION", "1"),
                      "kernel_ms": round(r.kernel_ms, 3), "device_ms": round(r.device_ms, 3),
                      "first_device_ms": round(rs[0].device_ms, 3), "count": r.clique_count}))
    sys.exit(0)
for cfg, k, order in (("cfg5", 8, "degree"), ("cfg5", 12, "degree"), ("cfg5", 5, "degree"),
                      ("cfg3", 6, "id")):
    for u in ("0", "1"):
        env = dict(os.environ, WM_CLIQUE_UNION=u)
        out = subprocess.run([sys.executable, __file__, "--one", cfg, str(k), order], env=env,
                             capture_output=True, text=True)
        print(out.stdout.strip() or out.stderr[-800:], flush=True)
