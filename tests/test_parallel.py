"""CPU, world_size 2 over gloo: the multi-GPU host path — cyclic sharding of
the cost-sorted root tasks and the single all_reduce of counters — gives the
single-process result.  Each rank's shard is computed by the oracle (the
device kernel cannot run here); the sharding rule is the one wm_run applies
(task i goes to rank i mod N after the stable (degree desc, id asc) sort)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _task_order(g):
    deg = np.diff(g.offsets)
    return np.lexsort((np.arange(g.n), -deg))  # degree desc, id asc (stable)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2212_04551_b200 import gnp_random_graph, parallel
    from paper_2212_04551_b200.canon import build_dictionary
    from paper_2212_04551_b200.engine import RunResult
    g = gnp_random_graph(80, 0.15, 3)
    assert parallel.default_shard() == (rank, world)
    roots = parallel.shard_tasks(_task_order(g), rank, world)
    d = build_dictionary(4)
    c = oracle.clique_run(g, 4, roots=roots, threads=1)
    m = oracle.motif_run(g, 4, d.table, d.pattern_count, roots=roots, threads=1)
    res = RunResult(app="motifs", k=4, mode="wc", warps=1, lane_width=32,
                    clique_count=c["count"], pattern_counts=m["hist"], records_emitted=None,
                    aggregated_total=m["leaves"], ledgers=[], makespan_ticks=0,
                    wall_seconds=0.0, rebalance_count=0, migrations=0,
                    peak_extension_storage=0, kernel_ms=float(rank + 1), tasks=len(roots))
    red = parallel.allreduce_result(res)
    out[rank] = (red.clique_count, red.pattern_counts, red.aggregated_total, red.kernel_ms,
                 red.tasks, red.devices)
    dist.destroy_process_group()


def test_two_rank_gloo_reduce_matches_single_process():
    import oracle
    from paper_2212_04551_b200 import gnp_random_graph
    from paper_2212_04551_b200.canon import build_dictionary
    g = gnp_random_graph(80, 0.15, 3)
    d = build_dictionary(4)
    want_c = oracle.clique_run(g, 4)["count"]
    want_m = oracle.motif_run(g, 4, d.table, d.pattern_count)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for rank in range(2):
        cc, hist, leaves, kms, tasks, devices = out[rank]
        assert cc == want_c
        assert hist == want_m["hist"]
        assert leaves == want_m["leaves"]
        assert kms == 2.0          # max over ranks
        assert tasks == g.n        # the shards partition the roots
        assert devices == 2


def test_shards_partition_tasks():
    from paper_2212_04551_b200 import parallel
    tasks = list(range(101))
    parts = [parallel.shard_tasks(tasks, r, 4) for r in range(4)]
    assert sorted(sum(parts, [])) == tasks
