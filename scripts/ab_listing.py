"""A/B listing throughput: python scripts/ab_listing.py lib1.so lib2.so ..."""
import json
import os
import subprocess
import sys
import time

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, "/root/repo")
    from paper_2212_04551_b200 import BalanceConfig, engine, listing_checksum, synth
    bc = BalanceConfig(threshold=0.9, poll_interval=8)
    engine.LISTING_RING = int(os.environ.get("WM_RING", str(engine.LISTING_RING)))
    out = {"ring": engine.LISTING_RING}
    for cfg, k in (("cfg2", 6), ("cfg1", 6)):
        g = synth.config_graph(cfg)
        listing_checksum(g, k, mode="opt", balance_config=bc)
        t = time.perf_counter()
        r = listing_checksum(g, k, mode="opt", balance_config=bc)
        dt = time.perf_counter() - t
        out[cfg] = {"records": r.records_emitted, "s": round(dt, 4),
                    "Mrec_per_s": round(r.records_emitted / dt / 1e6, 1),
                    "kernel_ms": round(r.kernel_ms, 2)}
    print(json.dumps(out))
    sys.exit(0)

for lib in sys.argv[1:]:
    env = dict(os.environ, WM_B200_LIB=os.path.abspath(lib))
    o = subprocess.run([sys.executable, __file__, "--one"], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), o.stdout.strip() or o.stderr[-400:], flush=True)
