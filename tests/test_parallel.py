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


def _vec_worker(rank, world, port, out):
    """Each rank holds the device result vector wm_run would write (layout of
    include/warpmine_b200.h WM_RED_*); allreduce_device sums it once."""
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2212_04551_b200 import _native, parallel
    from paper_2212_04551_b200.engine import RunResult
    P = 6
    v = np.zeros(_native.WM_RED_HIST + P + _native.WM_RED_SLOT_WORDS * world, dtype=np.uint64)
    v[_native.WM_RED_LEAVES] = 100 + rank
    v[_native.WM_RED_ALG_BYTES] = (1 << 63) + rank      # sums wrap mod 2^64
    v[_native.WM_RED_MIGRATIONS] = 3
    v[_native.WM_RED_DONATIONS] = 2
    v[_native.WM_RED_TASKS] = 10 * (rank + 1)
    v[_native.WM_RED_HIST:_native.WM_RED_HIST + P] = np.arange(P) + rank
    slot = _native.WM_RED_HIST + P + _native.WM_RED_SLOT_WORDS * rank
    v[slot:slot + 4] = np.array([1.5 + rank, 2.0, 0.25 * (rank + 1), 0.5],
                                dtype=np.float64).view(np.uint64)
    res = RunResult(app="motifs", k=4, mode="opt", warps=1, lane_width=32,
                    clique_count=None, pattern_counts=[0] * P, records_emitted=None,
                    aggregated_total=0, ledgers=[], makespan_ticks=0, wall_seconds=0.0,
                    rebalance_count=0, migrations=0, peak_extension_storage=0)
    red = parallel.allreduce_device(res, torch.from_numpy(v.view(np.int64)))
    out[rank] = (red.aggregated_total, red.alg_bytes, red.migrations, red.rebalance_count,
                 red.tasks, red.pattern_counts, red.kernel_ms, red.device_ms,
                 red.idle_warp_fraction, red.devices, red.clique_count,
                 red.extra["collective"])
    dist.destroy_process_group()


def test_device_result_vector_single_allreduce():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_vec_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for rank in range(2):
        leaves, ab, mig, don, tasks, hist, kms, dms, idle, dev, cc, coll = out[rank]
        assert leaves == 201
        assert ab == 1                     # (2^63 + 0) + (2^63 + 1) mod 2^64
        assert (mig, don, tasks) == (6, 4, 30)
        assert hist == [2 * i + 1 for i in range(6)]
        assert (kms, dms, idle) == (2.5, 2.0, 0.5)   # max over ranks
        assert dev == 2 and cc is None
        assert coll.startswith("all_reduce(SUM) x1")
