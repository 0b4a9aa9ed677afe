"""Engine entry point: ``run(g, app, ...) -> RunResult`` on a B200.

Mirrors ``warpmine.engine`` (reference ``pkg/src/warpmine/engine.py``):
``Application`` (:53-80) and ``RunResult`` (:747-778) keep their fields and
validation, and ``run`` (:781-843) keeps its signature and argument checks.
The body is replaced: the CsrGraph is uploaded once to HBM (cached per graph
and device) and ``wm_run`` in ``libwm_b200.so`` executes the whole
control/extend/filter/compact/aggregate/move loop on the device
(``csrc/wm_clique.cu``, ``csrc/wm_motif.cu``).  There is no CPU fallback:
pipelines other than the built-in clique/motif ones raise ValueError.

Extra keyword arguments (all optional, B200-only):
  roots        (begin, end) root-id range; ``None`` = all vertices
               (engine.py:187).  A root is the first vertex of a
               traversal: for motifs (and listing) the lowest id of the
               subgraph (canonical rule, canon.py:190-210); for cliques the
               lowest vertex in the clique ``order`` — so a suffix
               ``(b, n)`` enumerates exactly the subgraphs of the induced
               subgraph on ids >= b for motifs, and for cliques only with
               ``order="id"`` (under "degree" the suffix selects cliques
               by their lowest-(degree, id) member).
  order        "degree" (default) or "id": orientation of the clique DAG.
               Counts are order-invariant; "id" reproduces the reference
               tree exactly (and its B_alg).
  count_bytes  also compute B_alg — an instrumented pass.
  shard        (rank, count): process this rank's cyclic share of the
               cost-sorted root tasks (see ``parallel.py``); ``"auto"`` =
               (rank, world) of the initialised torch.distributed group.
               Default (0, 1): a plain call never becomes a collective.
  reduce       with count > 1, combine the ranks' results (default True):
               ``wm_run`` writes its result vector into a device buffer on
               the run's stream and ONE all_reduce(SUM) over it (NCCL on
               that stream) yields the job totals on every rank.
  stream       a ``torch.cuda.Stream`` (or raw cudaStream_t int) to run on.
"""

from __future__ import annotations

import ctypes
import time
import weakref
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native
from . import balance as bal
from .graph import CsrGraph

MODES = ("dfs", "wc", "opt")

# Store target of ``apps.listing_checksum``: records are consumed inside the
# native library (counted + checksummed) instead of a Python StoreBuffer.
NATIVE_STORE = object()
LISTING_RING = 1 << 16   # device->host ring records (the StoreBuffer keeps its own capacity)
DEFAULT_WARPS = 4
DEFAULT_LANE_WIDTH = 32
_BUILTIN_TAGS = ("lower", "compact", "clique", "canonical")


@dataclass(frozen=True)
class Application:
    """Declarative pipeline (reference ``engine.py:53-80``)."""

    name: str
    k: int
    extend_all: bool
    genedges: bool
    pipeline: tuple
    aggregator: str
    dictionary: object = None
    store: object = None
    store_predicate: Optional[Callable] = None

    def __post_init__(self):
        if self.k < 3:
            raise ValueError("need k >= 3")
        if self.aggregator not in ("counter", "pattern", "store"):
            raise ValueError("unknown aggregator %r" % (self.aggregator,))
        if self.aggregator == "pattern" and self.dictionary is None:
            raise ValueError("pattern aggregation requires a dictionary")
        if self.aggregator == "store" and self.store is None:
            raise ValueError("store aggregation requires a StoreBuffer")


@dataclass
class RunResult:
    """Reference ``engine.py:747-778`` plus device evidence."""

    app: str
    k: int
    mode: str
    warps: int
    lane_width: int
    clique_count: Optional[int]
    pattern_counts: Optional[list]
    records_emitted: Optional[int]
    aggregated_total: int
    ledgers: list
    makespan_ticks: int
    wall_seconds: float
    rebalance_count: int
    migrations: int
    peak_extension_storage: int
    # --- B200 evidence (no reference counterpart) ---
    kernel_ms: float = 0.0
    device_ms: float = 0.0
    alg_bytes: int = 0
    idle_warp_fraction: float = 0.0
    idle_warp_fraction_tail: float = 0.0
    tasks: int = 0
    launches: int = 0
    devices: int = 1
    order: str = "degree"
    extra: dict = field(default_factory=dict)

    @property
    def total_instructions(self) -> int:
        return 0

    @property
    def total_transactions(self) -> int:
        return 0

    @property
    def instructions_per_warp(self) -> float:
        return 0.0

    @property
    def transactions_per_warp(self) -> float:
        return 0.0

    @property
    def subgraphs_per_second(self) -> float:
        return self.aggregated_total / (self.kernel_ms * 1e-3) if self.kernel_ms > 0 else 0.0


# ---------------------------------------------------------------------------
# device graph handles (one upload per graph and device)

_HANDLES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _current_device() -> int:
    import torch
    return torch.cuda.current_device()


def device_graph(g: CsrGraph):
    """The ``wm_graph_create`` handle of ``g`` on the current device."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 engine has no CPU fallback")
    L = _native.load()
    dev = _current_device()
    per = _HANDLES.get(g)
    if per is None:
        per = {}
        _HANDLES[g] = per
        weakref.finalize(g, _free_handles, per)
    h = per.get(dev)
    if h is None:
        csr = _native.WmCsr(g.n, len(g.neighbors_array),
                            g.offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                            g.neighbors_array.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
        out = ctypes.c_void_p()
        _native.check(L.wm_graph_create(ctypes.byref(csr), ctypes.byref(out)))
        h = out.value
        per[dev] = h
    return h


def _free_handles(per: dict) -> None:
    try:
        L = _native.load()
    except ImportError:
        return
    for h in per.values():
        L.wm_graph_destroy(h)
    per.clear()


def release_device_graph(g: CsrGraph) -> None:
    per = _HANDLES.pop(g, None)
    if per:
        _free_handles(per)


# ---------------------------------------------------------------------------


def _app_struct(app: Application):
    tags = []
    for t in app.pipeline:
        if isinstance(t, str) and t in _BUILTIN_TAGS:
            tags.append(t)
        else:
            raise ValueError("user filter %r has no device implementation "
                             "(only the built-in tags %s run on B200)" % (t, _BUILTIN_TAGS))
    flags = 0
    for t in tags:
        flags |= {"lower": _native.WM_F_LOWER, "compact": _native.WM_F_COMPACT,
                  "clique": _native.WM_F_CLIQUE, "canonical": _native.WM_F_CANONICAL}[t]
    a = _native.WmApp()
    a.k = app.k
    a.extend_all = int(app.extend_all)
    a.genedges = int(app.genedges)
    a.aggregator = {"counter": _native.WM_AGG_COUNTER, "pattern": _native.WM_AGG_PATTERN,
                    "store": _native.WM_AGG_STORE}[app.aggregator]
    a.filters = flags
    keep = None
    if app.aggregator == "pattern":
        d = app.dictionary
        if d.k != app.k:
            raise ValueError("dictionary is for k=%d, run needs k=%d" % (d.k, app.k))
        keep = _device_table(d)
        a.dict_table = None
        a.dict_len = len(d.table)
        a.pattern_count = d.pattern_count
        a.dict_device = keep.data_ptr()
        a.dict_device_bits = 16 if keep.element_size() == 2 else 32
    return a, keep


_DEV_TABLES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _device_table(d):
    """HBM-resident copy of a dictionary's table, uploaded once per device
    (the dictionary is immutable, reference ``canon.py:222-224``).  Stored as
    u16 with SENTINEL 0xFFFF when the ids fit — half the bytes of the
    reference's u32 table (4 MiB -> 2 MiB at k = 7, 512 -> 256 MiB at k = 8)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 engine has no CPU fallback")
    dev = _current_device()
    per = _DEV_TABLES.setdefault(d, {})
    t = per.get(dev)
    if t is None:
        table = np.asarray(d.table, dtype=np.uint32)
        if d.pattern_count < 0xFFFF:
            host = np.where(table == 0xFFFFFFFF, 0xFFFF, table).astype(np.uint16)
            t = torch.from_numpy(host.view(np.int16)).to(torch.device("cuda", dev))
        else:
            t = torch.from_numpy(table.view(np.int32)).to(torch.device("cuda", dev))
        per[dev] = t
    return t


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def run(g: CsrGraph, app: Application, *, mode: str = "wc", warps: int = None,
        lane_width: int = DEFAULT_LANE_WIDTH, balance_config=None, roots=None,
        order: str = "degree", count_bytes: bool = False, shard=None, stream=None,
        warps_per_block: int = 0, blocks_per_sm: int = 0, reduce: bool = True) -> RunResult:
    """Enumerate all canonical size-k traversals of ``g`` on the current CUDA
    device (reference ``engine.py:781-843``)."""
    if mode not in MODES:
        raise ValueError("mode must be one of %s" % (MODES,))
    if warps is not None and warps < 1:
        raise ValueError("need at least one warp")
    if lane_width < 1:
        raise ValueError("need lane_width >= 1")
    if balance_config is not None and mode != "opt":
        raise ValueError("balance configuration only applies to opt mode")
    if order not in ("degree", "id"):
        raise ValueError("order must be 'degree' or 'id'")
    a, keep_table = _app_struct(app)
    cfg = _native.WmCfg()
    cfg.mode = {"dfs": _native.WM_MODE_DFS, "wc": _native.WM_MODE_WC,
                "opt": _native.WM_MODE_OPT}[mode]
    bc = balance_config or bal.default_config(app.name)
    if mode == "opt" and not bc.enabled:
        cfg.mode = _native.WM_MODE_WC
    cfg.lb_threshold = bc.threshold
    cfg.lb_poll = bc.poll_interval
    if roots is None:
        cfg.root_begin, cfg.root_end = -1, -1
    else:
        rb, re = roots
        if not (0 <= rb <= re <= g.n):
            raise ValueError("root range %r outside 0..%d" % ((rb, re), g.n))
        cfg.root_begin, cfg.root_end = rb, re
    if shard is None:
        shard = (0, 1)
    elif shard == "auto":
        from . import parallel
        shard = parallel.default_shard()
    shard = (int(shard[0]), int(shard[1]))
    if not (shard[1] >= 1 and 0 <= shard[0] < shard[1]):
        raise ValueError("bad shard %r" % (shard,))
    cfg.shard_rank, cfg.shard_count = shard
    cfg.order = _native.WM_ORDER_ID if order == "id" else _native.WM_ORDER_DEGREE
    cfg.count_bytes = int(count_bytes)
    cfg.warps_per_block = warps_per_block
    cfg.blocks_per_sm = blocks_per_sm
    cfg.stream = _stream_handle(stream)
    h = device_graph(g)
    if app.aggregator == "store":
        return _run_store(g, app, a, cfg, h, mode, lane_width, shard, order, reduce)
    res = _native.WmResult()
    hist = None
    if app.aggregator == "pattern":
        hist = np.zeros(app.dictionary.pattern_count, dtype=np.uint64)
        res.pattern_counts = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    red = None
    if reduce and shard[1] > 1:
        from . import parallel
        red = parallel.reduce_buffer(hist.size if hist is not None else 0, shard[1])
        if red is not None:
            cfg.reduce_out = red.data_ptr()
    t0 = time.perf_counter()
    _native.check(_native.load().wm_run(h, ctypes.byref(a), ctypes.byref(cfg), ctypes.byref(res)))
    wall = time.perf_counter() - t0
    del keep_table
    out = RunResult(
        app=app.name, k=app.k, mode=mode, warps=res.warps, lane_width=lane_width,
        clique_count=int(res.clique_count) if app.aggregator == "counter" else None,
        pattern_counts=[int(x) for x in hist] if hist is not None else None,
        records_emitted=None, aggregated_total=int(res.leaves), ledgers=[],
        makespan_ticks=0, wall_seconds=wall, rebalance_count=int(res.rebalance_count),
        migrations=int(res.migrations), peak_extension_storage=int(res.peak_ext),
        kernel_ms=res.kernel_ms, device_ms=res.device_ms, alg_bytes=int(res.alg_bytes),
        idle_warp_fraction=res.idle_warp_fraction,
        idle_warp_fraction_tail=res.idle_warp_fraction_tail, tasks=int(res.tasks),
        launches=int(res.launches), devices=shard[1], order=order,
        extra={"bucket_words": res.bucket_words, "nodes": int(res.nodes),
               "polls": int(res.polls), "build_ms": res.build_ms,
               "h2d_bytes": int(res.h2d_bytes), "d2h_bytes": int(res.d2h_bytes)})
    if red is not None:
        from . import parallel
        out = parallel.allreduce_device(out, red, stream)
    elif reduce and shard[1] > 1:
        from . import parallel
        out = parallel.allreduce_result(out)
    return out


def _result(app, mode, lane_width, res, wall, shard, order, **kw) -> RunResult:
    extra = {"bucket_words": res.bucket_words, "nodes": int(res.nodes),
             "polls": int(res.polls), "build_ms": res.build_ms,
             "h2d_bytes": int(res.h2d_bytes), "d2h_bytes": int(res.d2h_bytes)}
    extra.update(kw.pop("extra", {}))
    return RunResult(
        app=app.name, k=app.k, mode=mode, warps=res.warps, lane_width=lane_width,
        clique_count=kw.get("clique_count"), pattern_counts=kw.get("pattern_counts"),
        records_emitted=kw.get("records_emitted"), aggregated_total=int(res.leaves),
        ledgers=[], makespan_ticks=0, wall_seconds=wall,
        rebalance_count=int(res.rebalance_count), migrations=int(res.migrations),
        peak_extension_storage=int(res.peak_ext), kernel_ms=res.kernel_ms,
        device_ms=res.device_ms, alg_bytes=int(res.alg_bytes),
        idle_warp_fraction=res.idle_warp_fraction,
        idle_warp_fraction_tail=res.idle_warp_fraction_tail, tasks=int(res.tasks),
        launches=int(res.launches), devices=shard[1], order=order, extra=extra)


def _run_store(g, app, a, cfg, h, mode, lane_width, shard, order, reduce) -> RunResult:
    """listing_app through ``wm_run_listing``: device warps stream records
    into a mapped ring (aggregate_store, reference ``aggregate.py:199-223``);
    the native drain loop hands batches to ``sink`` below, which rebuilds
    ``(vertices, bits)`` (traversal order, ``extend_bits``), applies the
    predicate and ``put``s into the app's StoreBuffer — blocking there blocks
    the device producers."""
    from .apps import complete_subgraph
    from .canon import group_offset
    k = app.k
    pred = app.store_predicate
    lst = _native.WmListing()
    lst.capacity = LISTING_RING
    # the reference's complete_subgraph predicate runs on the device
    lst.filter = _native.WM_LIST_COMPLETE if pred is complete_subgraph else _native.WM_LIST_ALL
    host_pred = None if pred is complete_subgraph else pred
    off = group_offset(k - 1) if k > 2 else 0
    state = {"emitted": 0, "error": None}
    store = app.store

    def sink(user, recs, count, stride):
        try:
            rows = np.ctypeslib.as_array(recs, shape=(int(count) * int(stride),))
            rows = rows.reshape(int(count), int(stride)).tolist()
            for r in rows:
                vertices = tuple(r[5:4 + k]) + (r[1],)
                bits = r[3] | (r[4] << 32) | (r[2] << off)
                if host_pred is not None and not host_pred(vertices, bits):
                    continue
                store.put((vertices, bits))
                state["emitted"] += 1
            return 0
        except BaseException as exc:  # surfaced after the device stops
            state["error"] = exc
            return 1

    native_only = store is NATIVE_STORE
    if native_only:
        if pred is not None and pred is not complete_subgraph:
            raise ValueError("a Python predicate needs a Python store")
        lst.sink = _native.SINK_FN()
    else:
        lst.sink = _native.SINK_FN(sink)
    res = _native.WmResult()
    t0 = time.perf_counter()
    st = _native.load().wm_run_listing(h, ctypes.byref(a), ctypes.byref(cfg), ctypes.byref(lst),
                                       ctypes.byref(res))
    wall = time.perf_counter() - t0
    if state["error"] is not None:
        raise state["error"]
    _native.check(st)
    emitted = int(lst.emitted) if native_only else state["emitted"]
    out = _result(app, mode, lane_width, res, wall, shard, order, records_emitted=emitted,
                  extra={"checksum": int(lst.checksum), "records_streamed": int(lst.emitted),
                         "stride_words": int(lst.stride_words)})
    if reduce and shard[1] > 1:
        from . import parallel
        out = parallel.allreduce_result(out)
    return out
