"""DM_DFS vs DM_WC ablation (the paper's Table 4, on B200).

    python scripts/ablation_dfs.py            # timings (CUDA events), JSON lines
    ncu --metrics ... python scripts/ablation_dfs.py --once   # counter capture

Workloads: cfg3 (power-law Chung-Lu) clique k=4 and cfg2 (ER 3300) / cfg4
root suffix (R-MAT) motif k=4, each in mode dfs (thread per traversal) and
wc (warp per traversal, load balancing off), same tree, same counts.
"""
import json
import sys

sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import build_dictionary, run_clique, run_motifs, synth  # noqa: E402

once = "--once" in sys.argv
cases = [("cfg3", "clique", 4, None), ("cfg2", "motif", 4, None), ("cfg4", "motif", 4, 16384)]
graphs = {}
for cfg, app, k, suffix in cases:
    g = graphs.setdefault(cfg, synth.config_graph(cfg))
    roots = (g.n - suffix, g.n) if suffix else None
    out = {"workload": cfg, "app": app, "k": k, "root_suffix": suffix}
    for mode in ("dfs", "wc"):
        reps = 1 if once else 3
        best = None
        for _ in range(reps):
            if app == "clique":
                r = run_clique(g, k, mode=mode, roots=roots)
            else:
                r = run_motifs(g, k, build_dictionary(k), mode=mode, roots=roots)
            best = r if best is None or r.kernel_ms < best.kernel_ms else best
        out[mode] = {"kernel_ms": best.kernel_ms, "leaves": best.aggregated_total,
                     "warps": best.warps}
    out["speedup_wc_over_dfs"] = out["dfs"]["kernel_ms"] / max(1e-9, out["wc"]["kernel_ms"])
    assert out["dfs"]["leaves"] == out["wc"]["leaves"]
    print(json.dumps(out), flush=True)
