"""Shard balance on one GPU: run each of the N cyclic root shards of a workload
one after another (shard=(r, N), no all_reduce) and report every shard's kernel
and device time.  With one process per GPU the N-GPU step time is the slowest
shard, so t(N=1) / max_r t_r is the speed-up the sharding allows (the
measured multi-GPU numbers come from bench.py --gpus N under torchrun).

    python scripts/shard_scaling.py > profiles/rNN_shard_scaling.jsonl
"""
import json
import sys

sys.path.insert(0, "/root/repo")
from paper_2212_04551_b200 import BalanceConfig, build_dictionary, run_clique, run_motifs, synth

CL = BalanceConfig(threshold=1.0, poll_interval=32)
MO = BalanceConfig(threshold=1.0, poll_interval=2)


def best(fn, reps=3):
    out = None
    for _ in range(reps):
        r = fn()
        out = r if out is None or r.device_ms < out.device_ms else out
    return out


def sweep(name, fn, count):
    base = None
    for N in (1, 2, 4, 8):
        rs = [best(lambda: fn((r, N))) for r in range(N)]
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


g3 = synth.config_graph("cfg3")
sweep("cfg3 clique k=8", lambda sh: run_clique(g3, 8, mode="opt", balance_config=CL, shard=sh,
                                               reduce=False), lambda r: r.clique_count)
g5 = synth.config_graph("cfg5")
sweep("cfg5 clique k=8", lambda sh: run_clique(g5, 8, mode="opt", balance_config=CL, shard=sh,
                                               reduce=False), lambda r: r.clique_count)
d7 = build_dictionary(7)
sweep("cfg5 motif k=7 root suffix 32768",
      lambda sh: run_motifs(g5, 7, d7, mode="opt", balance_config=MO, roots=(g5.n - 32768, g5.n),
                            shard=sh, reduce=False), lambda r: r.aggregated_total)
