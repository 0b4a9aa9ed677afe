"""Reference applications over the B200 engine (reference
``pkg/src/warpmine/apps.py:43-118``): the same declarative pipelines, so
``run_clique`` / ``run_motifs`` / ``clique_counting`` / ``motif_counting``
calls written against ``warpmine`` run unchanged.  The brute-force oracle of
the reference (``apps.py:126-200``) is NOT part of the product; parity tests
use ``oracle/`` and golden vectors generated from the reference."""

from __future__ import annotations

from . import engine
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


def complete_subgraph(vertices, bits: int) -> bool:
    """Listing predicate: fully connected records (reference ``apps.py:121-123``)."""
    return bits == (1 << stored_bits(len(vertices))) - 1
