"""CPU: host-side mirror of the reference interface — graph contract,
dictionary bytes, generators, application/engine validation and error
behaviour (reference tests/test_graph.py, test_canon.py, test_apps.py)."""

from __future__ import annotations

import hashlib
import io
import itertools

import numpy as np
import pytest

from paper_2212_04551_b200 import (SENTINEL, Application, BalanceConfig, CanonicalDictionary,
                                   CsrGraph, DictionaryFormatError, EdgeBitmap, GraphParseError,
                                   build_dictionary, canonical_bits, clique_app, complete_graph,
                                   extend_bits, is_canonical_candidate, load_edge_list, motif_app,
                                   path_graph, run, star_of_cliques)
from paper_2212_04551_b200 import canon, synth
from paper_2212_04551_b200.balance import default_config, should_rebalance
from conftest import dictionary

G1 = [(0, 1), (0, 2), (1, 2), (1, 3), (2, 3), (3, 4)]


def digest(g):
    h = hashlib.sha256()
    h.update(np.asarray(g.offsets, dtype="<i8").tobytes())
    h.update(np.asarray(g.neighbors_array, dtype="<i4").tobytes())
    return h.hexdigest()


# -- graph (reference graph.py:28-188) ---------------------------------------

def test_g1_shape_and_rows():
    g = CsrGraph.from_edges(5, G1)
    assert (g.n, g.m, g.max_degree) == (5, 6, 3)
    assert g.neighbors(1).tolist() == [0, 2, 3]
    assert [g.degree(v) for v in range(5)] == [2, 3, 3, 3, 1]
    assert g.has_edge(0, 1) and g.has_edge(1, 0) and not g.has_edge(0, 3)
    g.validate()


def test_duplicates_self_loops_isolated():
    g = CsrGraph.from_edges(3, [(0, 1), (1, 0), (0, 1), (2, 2)])
    assert g.m == 1 and g.degree(2) == 0
    with pytest.raises(ValueError):
        CsrGraph.from_edges(2, [(0, 2)])
    with pytest.raises(ValueError):
        CsrGraph.from_edges(0, [])


def test_edge_list_parsing():
    g = load_edge_list(io.StringIO("# header\n\n0 1\n% c\n1 2\n"))
    assert (g.n, g.m) == (3, 2)
    g = load_edge_list(io.StringIO("5 7\n7 5\n5 5\n"))
    assert (g.n, g.m) == (2, 1)
    with pytest.raises(GraphParseError) as exc:
        load_edge_list(io.StringIO("0 1\nnot numbers\n"))
    assert exc.value.line_number == 2
    with pytest.raises(GraphParseError):
        load_edge_list(io.StringIO("# nothing\n"))
    with pytest.raises(GraphParseError):
        load_edge_list(io.StringIO("1 -2\n"))


def test_binary_roundtrip_and_suffix(tmp_path):
    g = synth.gnp_random_graph(200, 0.05, 3)
    p = tmp_path / "g.wmg"
    g.save(p)
    h = CsrGraph.load(p, validate=True)
    assert digest(h) == digest(g)
    s = g.induced_suffix(50)
    assert s.n == 150
    assert s.m == sum(1 for u, v in g.edges() if u >= 50 and v >= 50)


def test_reference_graphs_regenerate_bit_exact(golden):
    """Our generators rebuild the reference's exact graphs (digest of the CSR)."""
    want = {e["name"]: e["digest"] for e in golden["graphs"]}
    for s in range(5):
        assert digest(synth.gnp_random_graph(516, 1200 / 132870, s)) == want["cfg1_seed%d" % s]
    for s in range(3):
        assert digest(synth.gnp_random_graph(3300, 4500 / 5443350, s)) == want["cfg2_seed%d" % s]
    assert digest(star_of_cliques(6, 7)) == want["star_of_cliques_6_7"]
    assert digest(complete_graph(8)) == want["K8"]
    assert digest(path_graph(6)) == want["P6"]
    for n, p in [(20, 0.1), (14, 0.3), (10, 0.6)]:
        for seed in range(20):
            assert digest(synth.gnp_random_graph(n, p, seed)) == want["gnp_%d_%.1f_%d" % (n, p, seed)]


# -- canonical encoding and dictionary (reference canon.py) ------------------

def test_encoding():
    assert canon.group_offset(2) == 0 and canon.group_offset(3) == 2
    assert canon.stored_bits(4) == 5 and canon.stored_bits(7) == 20
    assert extend_bits(0, 1, 1) == 0
    assert extend_bits(0, 2, 0b11) == 0b11
    with pytest.raises(ValueError):
        extend_bits(0, 2, 0)
    with pytest.raises(ValueError):
        EdgeBitmap(0b100000, 4)


@pytest.mark.parametrize("k", [3, 4, 5, 6, 7])
def test_dictionary_bytes_identical_to_reference(golden, k):
    d = build_dictionary(k)
    g = golden["dictionaries"][str(k)]
    blob = d.to_bytes()
    assert hashlib.sha256(blob).hexdigest() == g["sha256"]
    assert d.pattern_count == g["pattern_count"]
    assert d.canonical_bitmaps == g["canonical_bitmaps"]


def test_dictionary_known_values():
    d3 = build_dictionary(3)
    assert d3.table.tolist() == [SENTINEL, 0, 0, 1]
    assert [build_dictionary(k).pattern_count for k in range(3, 8)] == [2, 6, 21, 112, 853]
    assert build_dictionary(4).canonical_bitmaps == [0b101, 0b110, 0b111, 0b1111, 0b10110, 0b11111]
    with pytest.raises(ValueError):
        build_dictionary(2)
    with pytest.raises(ValueError):
        build_dictionary(8)


def test_dictionary_file_validation(tmp_path):
    d = build_dictionary(3)
    p = tmp_path / "d.dmcd"
    d.save(p)
    e = CanonicalDictionary.load(p)
    assert e.table.tolist() == d.table.tolist() and e.canonical_bitmaps == d.canonical_bitmaps
    blob = bytearray(p.read_bytes())
    for mutate in (lambda b: b.__setitem__(slice(0, 4), b"XXXX"),
                   lambda b: b.__setitem__(4, 9)):
        bad = bytearray(blob)
        mutate(bad)
        with pytest.raises(DictionaryFormatError):
            CanonicalDictionary.from_bytes(bytes(bad))
    with pytest.raises(DictionaryFormatError):
        CanonicalDictionary.from_bytes(bytes(blob[:-3]))


def _relabel(bits, k, perm):
    full = [[False] * k for _ in range(k)]
    full[1][0] = full[0][1] = True
    for i in range(2, k):
        for j in range(i):
            if (bits >> canon.group_offset(i) + j) & 1:
                full[i][j] = full[j][i] = True
    img = [[full[perm.index(a)][perm.index(b)] for b in range(k)] for a in range(k)]
    if not img[1][0]:
        return None
    out = 0
    for i in range(2, k):
        grp = 0
        for j in range(i):
            if img[i][j]:
                grp |= 1 << j
        if not grp:
            return None
        out |= grp << canon.group_offset(i)
    return out


def test_canonical_form_is_relabel_invariant():
    d = build_dictionary(4)
    for bits in range(1 << canon.stored_bits(4)):
        if not canon.bitmap_is_valid(bits, 4):
            assert d.table[bits] == SENTINEL
            continue
        for perm in itertools.permutations(range(4)):
            img = _relabel(bits, 4, list(perm))
            if img is not None:
                assert d.table[img] == d.table[bits]
                assert canonical_bits(img, 4) == canonical_bits(bits, 4)


def test_canonical_candidate_rule():
    g = CsrGraph.from_edges(5, G1)
    assert is_canonical_candidate([0], 1, g)
    assert not is_canonical_candidate([1], 0, g)
    assert not is_canonical_candidate([0, 2], 1, g)   # 1 < 2 after first adjacent position
    assert is_canonical_candidate([0, 1], 3, g)


# -- applications, engine validation, balance config -------------------------

def test_app_validation():
    with pytest.raises(ValueError):
        clique_app(2)
    with pytest.raises(ValueError):
        clique_app(13)
    with pytest.raises(ValueError):
        motif_app(4, build_dictionary(3))
    with pytest.raises(ValueError):
        Application(name="x", k=2, extend_all=False, genedges=False, pipeline=(), aggregator="counter")
    with pytest.raises(ValueError):
        Application(name="x", k=3, extend_all=False, genedges=False, pipeline=(), aggregator="bogus")
    with pytest.raises(ValueError):
        Application(name="x", k=3, extend_all=True, genedges=True, pipeline=(), aggregator="pattern")


def test_run_argument_errors_before_device():
    g = complete_graph(5)
    for kw in ({"mode": "bogus"}, {"warps": 0}, {"lane_width": 0},
               {"mode": "wc", "balance_config": BalanceConfig()}, {"order": "random"},
               {"shard": (2, 2)}, {"shard": (0, 0)}, {"shard": (-1, 3)}):
        with pytest.raises(ValueError):
            run(g, clique_app(3), **kw)
    with pytest.raises(ValueError):
        run(g, Application(name="u", k=3, extend_all=False, genedges=False,
                           pipeline=(("filter", lambda *a: True, ()),), aggregator="counter"))


def test_default_shard_is_local():
    """A plain call never becomes a collective: without shard= the run is
    (0, 1) even inside an initialised process group; "auto" asks the group."""
    import inspect
    from paper_2212_04551_b200 import engine, parallel
    assert inspect.signature(engine.run).parameters["shard"].default is None
    assert parallel.default_shard() == (0, 1)  # no process group here


def test_balance_config():
    with pytest.raises(ValueError):
        BalanceConfig(threshold=0.0)
    with pytest.raises(ValueError):
        BalanceConfig(poll_interval=0)
    assert default_config("clique").threshold == 0.40
    assert default_config("motifs").threshold == 0.10
    assert should_rebalance(3, 10, BalanceConfig(threshold=0.4))
    assert not should_rebalance(4, 10, BalanceConfig(threshold=0.4))
    with pytest.raises(ValueError):
        should_rebalance(1, 0, BalanceConfig())


def test_product_never_imports_oracle():
    """The product package must not route through the CPU oracle."""
    import pathlib
    pkg = pathlib.Path(__file__).resolve().parent.parent / "paper_2212_04551_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p
