"""GPU parity on the BASELINE config graphs against expectations the
REFERENCE itself produced (tests/golden/make_golden_ref_scale.py imports
warpmine read-only): root-id ranges of cfg3 through the reference's queue
hook (``engine.py:160-191``) and root suffixes of cfg4 / cfg5 (the induced
subgraph of the last s ids, canonical rule ``canon.py:190-210``)."""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, dictionary

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref_scale():
    with open(os.path.join(GOLDEN_DIR, "ref_scale_golden.json")) as fh:
        return json.load(fh)


def _digest(g):
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype="<i8").tobytes())
    h.update(np.asarray(g.neighbors_array, dtype="<i4").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("mode", ["wc", "opt"])
def test_cfg3_clique_root_ranges(ref_scale, cuda, mode):
    from paper_2212_04551_b200 import BalanceConfig, run_clique, synth
    g = synth.config_graph("cfg3")
    rec = ref_scale["cfg3"]
    assert _digest(g) == rec["digest"]
    kw = {"balance_config": BalanceConfig(threshold=1.0)} if mode == "opt" else {}
    for key, want in rec["clique_roots"].items():
        b, e = want["roots"]
        r = run_clique(g, want["k"], mode=mode, order="id", roots=(b, e), **kw)
        assert r.clique_count == want["count"], (key, r.clique_count, want["count"])


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_motif_root_suffixes(ref_scale, cuda, name):
    from paper_2212_04551_b200 import BalanceConfig, run_motifs, synth
    g = synth.config_graph(name)
    rec = ref_scale[name]
    assert _digest(g) == rec["digest"]
    lb = BalanceConfig(threshold=1.0, poll_interval=1)
    for key, want in rec["motif_suffix"].items():
        k, s = want["k"], want["suffix"]
        for mode, kw in (("wc", {}), ("opt", {"balance_config": lb})):
            r = run_motifs(g, k, dictionary(k), mode=mode, roots=(g.n - s, g.n), **kw)
            assert r.pattern_counts == want["hist"], (name, key, mode)
            assert r.aggregated_total == want["leaves"]


def test_cfg5_clique_suffixes(ref_scale, cuda):
    from paper_2212_04551_b200 import run_clique, synth
    g = synth.config_graph("cfg5")
    for key, want in ref_scale["cfg5"]["clique_suffix"].items():
        s = want["suffix"]
        r = run_clique(g, want["k"], order="id", roots=(g.n - s, g.n))
        assert r.clique_count == want["count"], (key, r.clique_count, want["count"])
