"""A/B timing of clique kernel builds: [WM_AB_CFG=cfg5] python scripts/ab_clique.py K lib1.so ...
Each library runs in a fresh process (WM_B200_LIB); prints median kernel ms."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 2 and sys.argv[1] == "--one":
    sys.path.insert(0, "/root/repo")
    import statistics
    from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
    k = int(sys.argv[2])
    g = synth.config_graph(os.environ.get("WM_AB_CFG", "cfg3"))
    bc = BalanceConfig(threshold=1.0, poll_interval=int(os.environ.get("WM_POLL", "32")))
    ms, bms, dms = [], [], []
    for i in range(int(os.environ.get("WM_AB_REPS", "6"))):
        r = run_clique(g, k, mode="opt", balance_config=bc)
        if i:
            ms.append(r.kernel_ms)
            bms.append(r.extra["build_ms"])
            dms.append(r.device_ms)
    print(json.dumps({"k": k, "kernel_ms": statistics.median(ms), "min": min(ms),
                      "build_ms": statistics.median(bms), "device_ms": statistics.median(dms),
                      "count": r.clique_count, "warps": r.warps,
                      "idle": round(r.idle_warp_fraction, 3), "migr": r.migrations}))
    sys.exit(0)

k = sys.argv[1]
for lib in sys.argv[2:]:
    env = dict(os.environ, WM_B200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, __file__, "--one", k], env=env, capture_output=True,
                         text=True)
    print(lib, out.stdout.strip() or out.stderr[-500:], flush=True)
