"""Size the motif bench workloads: leaves / kernel time per root suffix,
LB off vs on (one-off exploration; results -> gpurun_out/)."""
import json, sys, time
sys.path.insert(0, ".")
import torch
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_motifs, synth

out = open("gpurun_out/explore_motif.jsonl", "a")
lb = BalanceConfig(threshold=1.0, poll_interval=2)
def go(cfg, k, s, mode, budget=None):
    g = synth.config_graph(cfg)
    d = build_dictionary(k)
    kw = {"balance_config": lb} if mode == "opt" else {}
    r = run_motifs(g, k, d, mode=mode, roots=(g.n - s, g.n), **kw)
    rec = {"cfg": cfg, "k": k, "suffix": s, "mode": mode, "leaves": r.aggregated_total,
           "kernel_ms": r.kernel_ms, "idle": r.idle_warp_fraction, "rate": r.subgraphs_per_second}
    print(json.dumps(rec), flush=True); out.write(json.dumps(rec) + "\n"); out.flush()
    return r
t=time.time(); synth.config_graph("cfg4"); print("cfg4 gen", time.time()-t, flush=True)
for s in (4096, 8192, 16384, 32768):
    r = go("cfg4", 6, s, "opt")
    if r.kernel_ms > 200: break
go("cfg4", 5, 16384, "wc")
go("cfg4", 6, 4096, "wc")
go("cfg4", 6, 8192, "wc")
t=time.time(); synth.config_graph("cfg5"); print("cfg5 gen", time.time()-t, flush=True)
for s in (4096, 8192, 16384, 32768):
    go("cfg5", 7, s, "opt")
for s in (4096, 8192):
    r = go("cfg5", 7, s, "wc")
    if r.kernel_ms > 20000: break
