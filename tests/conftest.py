"""Shared fixtures.  GPU tests carry ``@pytest.mark.gpu``; everything else
runs on CPU (the driver runs ``-m "not gpu"`` in the build container)."""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN_DIR, "reference_golden.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def scale_golden():
    with open(os.path.join(GOLDEN_DIR, "scale_golden.json")) as fh:
        return json.load(fh)


def graph_from_entry(e):
    from paper_2212_04551_b200.graph import CsrGraph
    ed = np.array(e["edges"], dtype=np.int64).reshape(-1, 2)
    return CsrGraph.from_arrays(e["n"], ed[:, 0], ed[:, 1])


def golden_cases(golden, app=None, max_k=12, names=None):
    """(graph entry, result record) pairs with stored edges."""
    out = []
    for e in golden["graphs"]:
        if e["edges"] is None or (names is not None and e["name"] not in names):
            continue
        for r in e["results"]:
            if (app is None or r["app"] == app) and r["k"] <= max_k:
                out.append((e, r))
    return out


_DICTS = {}


def dictionary(k):
    from paper_2212_04551_b200.canon import build_dictionary
    if k not in _DICTS:
        _DICTS[k] = build_dictionary(k)
    return _DICTS[k]


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_04551_b200 import _native
    _native.load()  # fails loudly if the extension is missing
    return torch.device("cuda", 0)
