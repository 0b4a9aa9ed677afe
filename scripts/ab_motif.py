"""A/B timing of motif kernel builds:
    python scripts/ab_motif.py CFG K SUFFIX lib1.so lib2.so ...   (SUFFIX 0 = all roots)
Each library runs in a fresh process (WM_B200_LIB); prints median kernel ms."""
import json
import os
import subprocess
import sys

if len(sys.argv) > 2 and sys.argv[1] == "--one":
    sys.path.insert(0, "/root/repo")
    import statistics
    from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth
    cfg, k, suffix = sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
    g = synth.config_graph(cfg)
    d = build_dictionary(k)
    roots = (g.n - suffix, g.n) if suffix else None
    bc = BalanceConfig(threshold=float(os.environ.get("WM_THR", "0.9")), poll_interval=int(os.environ.get("WM_POLL", "8")))
    ms = []
    for i in range(4):
        r = run_motifs(g, k, d, mode="opt", balance_config=bc, roots=roots)
        if i:
            ms.append(r.kernel_ms)
    print(json.dumps({"cfg": cfg, "k": k, "kernel_ms": statistics.median(ms), "min": min(ms),
                      "leaves": r.aggregated_total, "idle": round(r.idle_warp_fraction, 3),
                      "migr": r.migrations}))
    sys.exit(0)

cfg, k, suffix = sys.argv[1], sys.argv[2], sys.argv[3]
for lib in sys.argv[4:]:
    env = dict(os.environ, WM_B200_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, __file__, "--one", cfg, k, suffix], env=env,
                         capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip() or out.stderr[-500:], flush=True)
    prof = [l for l in out.stderr.splitlines() if l.startswith("[motif prof]")]
    if prof:
        print("   ", prof[-1], flush=True)
