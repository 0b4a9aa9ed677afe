"""Shard balance on one GPU: run each of the N cyclic root shards of a workload
one after another (shard=(r, N), no all_reduce) and report every shard's kernel
and device time.  With one process per GPU the N-GPU step time is the slowest
shard, so t(N=1) / max_r t_r is the speed-up the sharding allows (the
measured multi-GPU numbers come from bench.py --gpus N under torchrun).

    python scripts/shard_scaling.py [cfg3:8 cfg5:12 motif:cfg5:7:32768 ...] \
        > profiles/rNN_shard_scaling.jsonl
"""
import json
import sys

sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_clique, run_motifs, synth

import os
CL = BalanceConfig(threshold=1.0, poll_interval=int(os.environ.get("WM_POLL", "32")))
MO = BalanceConfig(threshold=1.0, poll_interval=2)


def best(fn, reps=3):
    out = None
    for _ in range(reps):
        r = fn()
        out = r if out is None or r.device_ms < out.device_ms else out
    return out


def sweep(name, fn, count, reps=3):
    base = None
    for N in (1, 2, 4, 8):
        rs = [best(lambda: fn((r, N)), reps) for r in range(N)]
        tot = sum(count(x) for x in rs)
        kmax = max(x.kernel_ms for x in rs)
        dmax = max(x.device_ms for x in rs)
        if base is None:
            base = (kmax, dmax, tot)
        print(json.dumps({
            "workload": name, "shards": N, "total": tot, "total_matches_1": tot == base[2],
            "kernel_ms": [round(x.kernel_ms, 3) for x in rs],
            "device_ms": [round(x.device_ms, 3) for x in rs],
            "speedup_kernel": base[0] / kmax, "speedup_device": base[1] / dmax,
            "efficiency_device": base[1] / dmax / N}), flush=True)


WORKLOADS = sys.argv[1:] or ["cfg3:8", "cfg3:9", "cfg3:10", "cfg5:8", "cfg5:12",
                             "motif:cfg5:7:32768"]
for wl in WORKLOADS:
    parts = wl.split(":")
    if parts[0] == "motif":
        g = synth.config_graph(parts[1])
        k, suf = int(parts[2]), int(parts[3])
        d = build_dictionary(k)
        sweep("%s motif k=%d root suffix %d" % (parts[1], k, suf),
              lambda sh: run_motifs(g, k, d, mode="opt", balance_config=MO,
                                    roots=(g.n - suf, g.n), shard=sh, reduce=False),
              lambda r: r.aggregated_total)
    else:
        g = synth.config_graph(parts[0])
        k = int(parts[1])
        sweep("%s clique k=%d" % (parts[0], k),
              lambda sh: run_clique(g, k, mode="opt", balance_config=CL, shard=sh, reduce=False),
              lambda r: r.clique_count, reps=3 if k <= 10 else 1)
