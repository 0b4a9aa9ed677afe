"""Pattern dictionary built on the device (wm_dictionary_build, reference
build_dictionary canon.py:315-343) and k = 8 motif counting with it."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("k", [3, 4, 5, 6, 7])
def test_device_dictionary_bytes_equal_reference(golden, cuda, k):
    from paper_2212_04551_b200.canon import build_dictionary
    d = build_dictionary(k, device=True)
    assert hashlib.sha256(d.to_bytes()).hexdigest() == golden["dictionaries"][str(k)]["sha256"]
    assert d.to_bytes() == build_dictionary(k, device=False).to_bytes()


def test_k8_dictionary_is_the_canonical_map(cuda):
    from paper_2212_04551_b200.canon import (SENTINEL, build_dictionary, canonical_bits,
                                             group_offset, stored_bits)
    d = build_dictionary(8, allow_large=True)
    assert d.pattern_count == 11117          # connected graphs on 8 vertices
    reps = d.canonical_bitmaps
    assert all(b < c for b, c in zip(reps, reps[1:]))
    assert all(int(d.table[b]) == i for i, b in enumerate(reps))
    assert reps[-1] == (1 << stored_bits(8)) - 1   # K8 is the last id (SURVEY A)
    rng = np.random.default_rng(8)
    sample = rng.integers(0, 1 << stored_bits(8), 3000)
    for b in sample.tolist():
        ok = all((b >> group_offset(i)) & ((1 << i) - 1) for i in range(2, 8))
        if not ok:
            assert int(d.table[b]) == SENTINEL
            continue
        assert reps[int(d.table[b])] == canonical_bits(b, 8)


def test_k8_motifs(cuda):
    import oracle
    from paper_2212_04551_b200 import (BalanceConfig, clique_counting, complete_graph,
                                       gnp_random_graph, listing_checksum, run_motifs,
                                       star_of_cliques)
    from paper_2212_04551_b200.canon import build_dictionary
    d = build_dictionary(8, allow_large=True)
    r = run_motifs(complete_graph(9), 8, d)
    assert r.pattern_counts[-1] == 9 and sum(r.pattern_counts) == 9
    for g in (gnp_random_graph(20, 0.3, 1), gnp_random_graph(16, 0.6, 3), star_of_cliques(3, 8)):
        want = oracle.motif_run(g, 8, d.table, d.pattern_count)
        for mode, kw in (("wc", {}), ("opt", {"balance_config": BalanceConfig(threshold=1.0)}),
                         ("dfs", {})):
            got = run_motifs(g, 8, d, mode=mode, **kw)
            assert got.pattern_counts == want["hist"], mode
        assert sum(want["hist"]) == listing_checksum(g, 8).records_emitted
        assert want["hist"][-1] == clique_counting(g, 8)
