"""GPU graph ingest (wm_csr_build / wm_edge_list_parse) produces exactly the
host CsrGraph (reference graph.py:44-78 construction, graph.py:139-188
reader semantics, GraphParseError line numbers)."""

from __future__ import annotations

import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _same(a, b):
    assert a.n == b.n
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.neighbors_array, b.neighbors_array)


def test_from_arrays_device_equals_host(cuda):
    from paper_2212_04551_b200 import CsrGraph
    rng = np.random.default_rng(5)
    for n, m in [(1, 0), (2, 1), (10, 40), (1000, 20000), (70000, 300000)]:
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        _same(CsrGraph.from_arrays(n, src, dst, device=True), CsrGraph.from_arrays(n, src, dst))
    with pytest.raises(ValueError):
        CsrGraph.from_arrays(5, [0, 7], [1, 2], device=True)


def test_config_graphs_device_equal_host(cuda, monkeypatch):
    from paper_2212_04551_b200 import synth
    build = synth.config_graph.__wrapped__  # bypass the per-process cache
    for name in ("cfg3",):
        dev = build(name)
        monkeypatch.setenv("WM_HOST_BUILD", "1")
        host = build(name)
        monkeypatch.delenv("WM_HOST_BUILD")
        _same(dev, host)


def test_edge_list_device_equals_host(cuda, tmp_path):
    from paper_2212_04551_b200 import gnp_random_graph
    from paper_2212_04551_b200.graph import load_edge_list
    g = gnp_random_graph(300, 0.05, 3)
    text = "# comment\n% other\n\n" + "".join("%d %d\n" % (3 * u + 7, 3 * v + 7)
                                             for u, v in g.edges())
    text += "5 5\n  12\t 30  \r\n1_000 2\n+4 9"  # self-loop, tabs/CR, underscore, sign, no EOL
    p = tmp_path / "g.txt"
    p.write_text(text)
    _same(load_edge_list(str(p), device=True), load_edge_list(str(p)))
    _same(load_edge_list(io.StringIO(text), device=True), load_edge_list(io.StringIO(text)))


@pytest.mark.parametrize("bad", ["1 2\n3\n", "1 2\n3 x\n", "1 2\n\n-1 4\n", "1 2 3\n", "# c\n"])
def test_edge_list_errors_match_host(cuda, bad):
    from paper_2212_04551_b200 import GraphParseError
    from paper_2212_04551_b200.graph import load_edge_list
    with pytest.raises(GraphParseError) as want:
        load_edge_list(io.StringIO(bad))
    with pytest.raises(GraphParseError) as got:
        load_edge_list(io.StringIO(bad), device=True)
    assert str(got.value) == str(want.value)
    assert got.value.line_number == want.value.line_number
