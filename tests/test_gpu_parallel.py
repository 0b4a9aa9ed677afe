"""Multi-rank execution of the real device path.

Each rank calls ``engine.run(..., shard="auto")``: ``wm_run`` enumerates the
rank's cyclic share of the cost-sorted root tasks and writes its result
vector into a device buffer on the run's stream; ONE all_reduce(SUM) over
that buffer gives every rank the job totals (reference sum semantics,
``aggregate.py:39-55``; independent root subtrees, ``engine.py:187``).

* gloo, 2 ranks sharing cuda:0 — runs on a 1-GPU lease;
* NCCL, min(2, device_count) ranks on distinct GPUs — skipped on one GPU.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, backend, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        from paper_2212_04551_b200 import (BalanceConfig, build_dictionary, run_clique,
                                           run_motifs, synth)
        res = {}
        g3 = synth.config_graph("cfg3")
        r = run_clique(g3, 6, mode="opt", balance_config=BalanceConfig(threshold=1.0),
                       shard="auto")
        res["cfg3_k6"] = (r.clique_count, r.aggregated_total, r.tasks, r.devices,
                          r.extra.get("collective"), r.kernel_ms)
        res["cfg3_k6_single_tasks"] = run_clique(g3, 6).tasks  # default shard: local
        r = run_clique(g3, 5, mode="wc", shard="auto", count_bytes=True)
        res["cfg3_k5_bytes"] = (r.clique_count, r.alg_bytes)
        g4 = synth.config_graph("cfg4")
        d = build_dictionary(5)
        r = run_motifs(g4, 5, d, mode="opt", roots=(g4.n - 4096, g4.n),
                       balance_config=BalanceConfig(threshold=1.0, poll_interval=2),
                       shard="auto")
        res["cfg4_k5_s4096"] = (r.pattern_counts, r.aggregated_total, r.devices)
        # a plain call stays local (no collective, full result)
        r = run_clique(synth.config_graph("cfg1"), 3)
        res["cfg1_local"] = (r.clique_count, r.devices)
        out[rank] = res
    finally:
        dist.destroy_process_group()


def _check(out, world, scale_golden):
    c3 = scale_golden["cfg3"]["clique"]
    m4 = scale_golden["cfg4"]["motif_suffix"]["k5_s4096"]
    for rank in range(world):
        res = out[rank]
        cc, leaves, tasks, devices, coll, kms = res["cfg3_k6"]
        assert cc == c3["6"]["count"] and leaves == cc
        assert tasks == res["cfg3_k6_single_tasks"]  # the shards partition the tasks
        assert devices == world
        assert coll and coll.startswith("all_reduce(SUM) x1")
        assert kms > 0
        cc5, ab5 = res["cfg3_k5_bytes"]
        assert cc5 == c3["5"]["count"]
        assert ab5 == c3["5"]["alg_bytes_degree_order"]
        hist, leaves, devices = res["cfg4_k5_s4096"]
        assert hist == m4["hist"] and leaves == m4["leaves"] and devices == world
        assert res["cfg1_local"] == (17, 1)


def test_two_ranks_share_one_gpu_gloo(cuda, scale_golden):
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, _free_port(), "gloo", out), nprocs=2, join=True)
    _check(out, 2, scale_golden)


def test_nccl_ranks_on_distinct_gpus(cuda, scale_golden):
    world = min(2, torch.cuda.device_count())
    if world < 2:
        pytest.skip("needs >= 2 GPUs (one NCCL rank per GPU)")
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), "nccl", out), nprocs=world, join=True)
    _check(out, world, scale_golden)
