"""Multi-GPU plumbing: root-task sharding and the single count allreduce.

The path shards naturally: root subtrees are independent
(reference ``engine.py:187``, ``:809-816``) and results are plain sums
(``engine.py:821-826``, ``aggregate.py:39-55``).  One process per GPU;
rank ``r`` of ``N`` takes the cost-sorted root tasks ``i ≡ r (mod N)``
(computed identically on every rank inside ``wm_run``), runs its own
on-device load balancer, and the ranks combine their results with ONE
``all_reduce(SUM)``: ``wm_run`` writes ``[cliques, leaves, B_alg,
migrations, donations, tasks, records, checksum, hist[P], timing slots]``
into a device buffer on the run's stream (``wm_cfg.reduce_out``) and the
collective runs over that buffer on the same stream (NCCL), so nothing is
copied to the host or repacked before the reduction.  gloo (CPU tests, and
several ranks sharing one GPU) reduces a host copy of the same vector.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np


def _dist():
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return None
    return dist if dist.is_available() and dist.is_initialized() else None


def default_shard():
    """(rank, world) of the initialised process group, else (0, 1)."""
    dist = _dist()
    if dist is None:
        return (0, 1)
    return (dist.get_rank(), dist.get_world_size())


def shard_tasks(tasks, rank: int, count: int):
    """Host restatement of the device's cyclic task split (for tests)."""
    return list(tasks)[rank::count]


def _i64(x: int) -> int:
    """u64 -> two's-complement int64 (sums stay exact mod 2^64)."""
    x &= (1 << 64) - 1
    return x - (1 << 64) if x >= 1 << 63 else x


def pack(res) -> list:
    hist = res.pattern_counts or []
    return [res.clique_count or 0, res.aggregated_total, res.alg_bytes, res.migrations,
            res.rebalance_count, res.tasks, res.records_emitted or 0,
            _i64(res.extra.get("checksum", 0))] + list(hist)


def allreduce_result(res, group=None, device=None):
    """Sum the counters of every rank (one all_reduce).  Timing fields are
    max-reduced in a second tiny collective so ``kernel_ms`` is the job's
    critical path."""
    import torch
    dist = _dist()
    if dist is None:
        return res
    backend = dist.get_backend(group)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" \
            else torch.device("cpu")
    vals = torch.tensor(pack(res), dtype=torch.int64, device=device)
    dist.all_reduce(vals, op=dist.ReduceOp.SUM, group=group)
    t = torch.tensor([res.kernel_ms, res.device_ms, res.wall_seconds,
                      res.idle_warp_fraction, res.idle_warp_fraction_tail],
                     dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    v = [int(x) for x in vals.tolist()]
    tt = t.tolist()
    extra = dict(res.extra)
    if "checksum" in extra:
        extra["checksum"] = v[7] & ((1 << 64) - 1)
    return replace(res,
                   clique_count=v[0] if res.clique_count is not None else None,
                   aggregated_total=v[1], alg_bytes=v[2], migrations=v[3],
                   rebalance_count=v[4], tasks=v[5],
                   records_emitted=v[6] if res.records_emitted is not None else None,
                   pattern_counts=v[8:] if res.pattern_counts is not None else None,
                   extra=extra,
                   kernel_ms=tt[0], device_ms=tt[1], wall_seconds=tt[2],
                   idle_warp_fraction=tt[3], idle_warp_fraction_tail=tt[4],
                   devices=dist.get_world_size(group))


def reduce_buffer(pattern_count: int, world: int):
    """Device buffer for ``wm_cfg.reduce_out`` (``wm_reduce_words`` int64
    words on the current device), or None without a process group."""
    if _dist() is None:
        return None
    import torch
    from . import _native
    words = int(_native.load().wm_reduce_words(pattern_count, world))
    return torch.empty(words, dtype=torch.int64,
                       device=torch.device("cuda", torch.cuda.current_device()))


def _torch_stream(stream):
    import torch
    if stream is None:
        return torch.cuda.current_stream()
    if isinstance(stream, int):
        return torch.cuda.ExternalStream(stream)
    return stream


def allreduce_device(res, vec, stream=None, group=None):
    """ONE all_reduce(SUM) over the device result vector ``wm_run`` wrote
    on ``stream`` (layout: include/warpmine_b200.h ``WM_RED_*``), then one
    copy of the reduced vector to the host.  Counters are sums mod 2^64;
    each rank's timing slot survives the sum, so ``kernel_ms`` etc. are the
    max over ranks (the job's critical path)."""
    import torch
    from . import _native
    dist = _dist()
    if dist is None:
        return res
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        with torch.cuda.stream(_torch_stream(stream)):
            dist.all_reduce(vec, op=dist.ReduceOp.SUM, group=group)
            host = vec.cpu()
    else:  # gloo reduces host tensors
        if vec.is_cuda:
            with torch.cuda.stream(_torch_stream(stream)):
                host = vec.cpu()
        else:
            host = vec.clone()
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
    v = host.numpy()
    u = v.view(np.uint64)
    P = len(res.pattern_counts) if res.pattern_counts is not None else 0
    base = _native.WM_RED_HIST + P
    nslot = (v.size - base) // _native.WM_RED_SLOT_WORDS  # the shard count of the run
    slots = v[base:base + _native.WM_RED_SLOT_WORDS * nslot].view(np.float64)
    tmax = slots.reshape(nslot, _native.WM_RED_SLOT_WORDS).max(axis=0)
    return replace(res,
                   clique_count=int(u[_native.WM_RED_CLIQUES])
                   if res.clique_count is not None else None,
                   aggregated_total=int(u[_native.WM_RED_LEAVES]),
                   alg_bytes=int(u[_native.WM_RED_ALG_BYTES]),
                   migrations=int(u[_native.WM_RED_MIGRATIONS]),
                   rebalance_count=int(u[_native.WM_RED_DONATIONS]),
                   tasks=int(u[_native.WM_RED_TASKS]),
                   pattern_counts=[int(x) for x in u[_native.WM_RED_HIST:base]]
                   if res.pattern_counts is not None else None,
                   kernel_ms=float(tmax[0]), device_ms=float(tmax[1]),
                   idle_warp_fraction=float(tmax[2]), idle_warp_fraction_tail=float(tmax[3]),
                   devices=world,
                   extra=dict(res.extra, collective="all_reduce(SUM) x1 over %d words (%s)"
                              % (v.size, dist.get_backend(group))))
