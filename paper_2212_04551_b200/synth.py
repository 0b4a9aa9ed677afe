"""Seeded synthetic graphs for the parity corpus and the benchmark configs.

``gnp_random_graph``, ``complete_graph``, ``path_graph`` and
``star_of_cliques`` reproduce the reference generators
(``pkg/src/warpmine/synth.py:10-50``) bit-for-bit — same PCG64 stream, same
edge set — so a graph built here is the graph the reference would mine.
``chung_lu`` and ``rmat`` are the SURVEY §8(d) / Appendix B recipes for
configs 3-5 (no reference counterpart: its O(n^2) ``triu_indices`` cannot
build them).
"""

from __future__ import annotations

import functools
import os

import numpy as np

from .graph import CsrGraph


def _device_build() -> bool:
    """Large generated graphs (configs 3-5) are assembled on the GPU
    (``wm_csr_build``) when one is present; the arrays are identical to the
    host build (tests/test_gpu_ingest.py).  WM_HOST_BUILD=1 forces the host."""
    if os.environ.get("WM_HOST_BUILD"):
        return False
    try:
        import torch
        from . import _native
        return torch.cuda.is_available() and os.path.exists(_native.LIB_PATH)
    except Exception:
        return False


def gnp_random_graph(n: int, p: float, seed: int) -> CsrGraph:
    """Erdos-Renyi G(n, p) (reference ``synth.py:10-20``)."""
    if n < 1:
        raise ValueError("need n >= 1")
    if not 0.0 <= p <= 1.0:
        raise ValueError("edge probability must be in [0, 1]")
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    mask = rng.random(len(iu)) < p
    return CsrGraph.from_arrays(n, iu[mask], ju[mask])


def complete_graph(n: int) -> CsrGraph:
    iu, ju = np.triu_indices(n, k=1)
    return CsrGraph.from_arrays(n, iu, ju)


def path_graph(n: int) -> CsrGraph:
    a = np.arange(max(n - 1, 0))
    return CsrGraph.from_arrays(n, a, a + 1)


def star_of_cliques(blobs: int, blob_size: int) -> CsrGraph:
    """Hub 0 joined to ``blobs`` disjoint ``blob_size``-cliques
    (reference ``synth.py:31-50``); adversarial for load balancing."""
    if blobs < 1 or blob_size < 2:
        raise ValueError("need blobs >= 1 and blob_size >= 2")
    src, dst = [], []
    for b in range(blobs):
        lo = 1 + b * blob_size
        members = np.arange(lo, lo + blob_size)
        src.append(np.zeros(blob_size, np.int64))
        dst.append(members)
        iu, ju = np.triu_indices(blob_size, k=1)
        src.append(members[iu])
        dst.append(members[ju])
    return CsrGraph.from_arrays(1 + blobs * blob_size, np.concatenate(src),
                                np.concatenate(dst))


def permute(g: CsrGraph, seed: int) -> CsrGraph:
    """Relabel vertices by a seeded uniform permutation (counts invariant,
    SURVEY §0 item 6)."""
    perm = np.random.default_rng(seed).permutation(g.n)
    e = g.edge_array()
    return CsrGraph.from_arrays(g.n, perm[e[:, 0]], perm[e[:, 1]], device=_device_build())


def chung_lu(n: int, m: int, gamma: float, seed: int, permute_seed=None) -> CsrGraph:
    """Power-law Chung-Lu graph: ``w_i = (i+1)^(-1/(γ-1))``,
    both endpoints drawn ``rng.choice(n, m, p=w/Σw)`` from ``default_rng(seed)``,
    simplified.  cfg3 = ``chung_lu(100000, 1000000, 2.3, 3)`` -> 947,479 edges."""
    rng = np.random.default_rng(seed)
    w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1))
    p = w / w.sum()
    src = rng.choice(n, size=m, p=p)
    dst = rng.choice(n, size=m, p=p)
    g = CsrGraph.from_arrays(n, src, dst, device=_device_build())
    return permute(g, permute_seed) if permute_seed is not None else g


def rmat(scale: int, edge_factor: int, a=0.57, b=0.19, c=0.19, seed: int = 1,
         permute_seed=None) -> CsrGraph:
    """R-MAT (Graph500 skew by default)."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = n * edge_factor
    src = np.zeros(m, np.int64)
    dst = np.zeros(m, np.int64)
    for bit in range(scale):
        r = rng.random(m)
        src |= (r >= a + b).astype(np.int64) << bit
        dst |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.int64) << bit
    g = CsrGraph.from_arrays(n, src, dst, device=_device_build())
    return permute(g, permute_seed) if permute_seed is not None else g


# The benchmark configs of BASELINE.json.  Graphs are
# immutable, so one build per process is shared (configs 4-5 take ~10-60 s
# of host RNG work).
@functools.lru_cache(maxsize=4)
def config_graph(name: str, seed: int = None) -> CsrGraph:
    if name == "cfg1":
        return gnp_random_graph(516, 1200 / 132870, 1 if seed is None else seed)
    if name == "cfg2":
        return gnp_random_graph(3300, 4500 / 5443350, 2 if seed is None else seed)
    if name == "cfg3":
        return chung_lu(100000, 1000000, 2.3, 3 if seed is None else seed)
    if name == "cfg4":
        return rmat(20, 16, seed=1 if seed is None else seed, permute_seed=20)
    if name == "cfg5":
        # Graph500 skew at scale 22 has ~1e18 12-cliques (a
        # 0.97-dense hub core); a = 0.52, b = c = 0.20, d = 0.08 keeps the
        # power-law skew (max degree ~41K) with ~1e11 12-cliques.
        return rmat(22, 8, a=0.52, b=0.20, c=0.20, seed=1 if seed is None else seed,
                    permute_seed=22)
    raise ValueError("unknown config %r" % name)
