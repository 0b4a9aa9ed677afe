"""Reference applications over the B200 engine (reference
``pkg/src/warpmine/apps.py:43-118``): the same declarative pipelines, so
``run_clique`` / ``run_motifs`` / ``clique_counting`` / ``motif_counting``
calls written against ``warpmine`` run unchanged.  The brute-force oracle of
the reference (``apps.py:126-200``) is NOT part of the product; parity tests
use ``oracle/`` and golden vectors generated from the reference."""

from __future__ import annotations

from typing import Callable, Optional

from . import engine
from .aggregate import StoreBuffer
from .canon import CanonicalDictionary, stored_bits
from .graph import CsrGraph

K_MIN = 3
K_MAX = 12


def _check_k(k: int, upper: int = K_MAX) -> None:
    if not K_MIN <= k <= upper:
        raise ValueError("k must be in [%d, %d], got %d" % (K_MIN, upper, k))


def clique_app(k: int) -> engine.Application:
    """Reference ``apps.py:43-47``."""
    _check_k(k)
    return engine.Application(
        name="clique", k=k, extend_all=False, genedges=False,
        pipeline=("lower", "compact", "clique"), aggregator="counter")


def motif_app(k: int, dictionary: CanonicalDictionary) -> engine.Application:
    """Reference ``apps.py:50-58``."""
    _check_k(k, upper=8)
    if dictionary.k != k:
        raise ValueError("dictionary is for k=%d, run needs k=%d" % (dictionary.k, k))
    return engine.Application(
        name="motifs", k=k, extend_all=True, genedges=True,
        pipeline=("canonical",), aggregator="pattern", dictionary=dictionary)


def listing_app(k: int, store: StoreBuffer,
                predicate: Optional[Callable] = None) -> engine.Application:
    """Reference ``apps.py:61-67``: the motif pipeline with the store
    aggregator (k up to 12, no dictionary)."""
    _check_k(k)
    return engine.Application(
        name="list", k=k, extend_all=True, genedges=True,
        pipeline=("canonical",), aggregator="store",
        store=store, store_predicate=predicate)


def run_clique(g: CsrGraph, k: int, mode: str = "wc", **kwargs) -> engine.RunResult:
    return engine.run(g, clique_app(k), mode=mode, **kwargs)


def run_motifs(g: CsrGraph, k: int, dictionary: CanonicalDictionary,
               mode: str = "wc", **kwargs) -> engine.RunResult:
    return engine.run(g, motif_app(k, dictionary), mode=mode, **kwargs)


def clique_counting(g: CsrGraph, k: int, mode: str = "wc", **kwargs) -> int:
    """Number of k-cliques in g (reference ``apps.py:79-81``)."""
    return run_clique(g, k, mode, **kwargs).clique_count


def motif_counting(g: CsrGraph, k: int, dictionary: CanonicalDictionary,
                   mode: str = "wc", **kwargs) -> dict:
    """Connected induced k-subgraph counts keyed by pattern id, zeros
    included (reference ``apps.py:84-91``)."""
    return dict(enumerate(run_motifs(g, k, dictionary, mode, **kwargs).pattern_counts))


def subgraph_listing(g: CsrGraph, k: int, predicate: Optional[Callable] = None,
                     mode: str = "wc", *, capacity: int = 1024,
                     sink: Optional[Callable] = None, **kwargs):
    """Stream every connected induced k-subgraph passing ``predicate``
    (reference ``apps.py:94-118``): records ``(vertices, bits)`` flow from
    the device ring through a ``StoreBuffer`` of ``capacity`` to a consumer
    thread.  Returns the records (default sink) or ``records_emitted``."""
    store = StoreBuffer(capacity)
    records: list = []
    consumer = store.start_consumer(sink if sink is not None else records.append)
    try:
        result = engine.run(g, listing_app(k, store, predicate), mode=mode, **kwargs)
    finally:
        store.close()
        consumer.join(timeout=30.0)
    if store.failed:
        raise RuntimeError("listing sink failed")
    return records if sink is None else result.records_emitted


def listing_checksum(g: CsrGraph, k: int, complete_only: bool = False,
                     mode: str = "wc", **kwargs) -> engine.RunResult:
    """B200 extra: run the listing pipeline with the records consumed inside
    the native library (counted and checksummed, no Python sink) — the
    listing throughput path and its parity check at scale.
    ``result.records_emitted`` and ``result.extra["checksum"]`` (definition in
    ``include/warpmine_b200.h``)."""
    app = listing_app(k, engine.NATIVE_STORE,
                      complete_subgraph if complete_only else None)
    return engine.run(g, app, mode=mode, **kwargs)


def complete_subgraph(vertices, bits: int) -> bool:
    """Listing predicate: fully connected records (reference ``apps.py:121-123``)."""
    return bits == (1 << stored_bits(len(vertices))) - 1
