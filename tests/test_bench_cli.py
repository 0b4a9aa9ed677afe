"""CPU: bench.py's launch contract without a GPU — ``--gpus N`` refuses to
time fewer GPUs than asked (instead of silently timing one), a torchrun
environment whose WORLD_SIZE disagrees with --gpus is rejected, and the
reference arm (the CPU restatement, rank 0 only) prints one JSON line with
the contract's keys and never maps the product library."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True,
                          env=e, timeout=timeout, cwd=ROOT)


def test_too_few_gpus_is_an_error():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has >= 2 GPUs")
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 2
    assert "GPU(s) visible" in r.stderr


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "4"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=2 but --gpus 4" in r.stderr


def test_reference_arm_line_and_no_product_library():
    """k=5 keeps the slice short; the line carries the reference-arm keys."""
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "3", "--k", "5"],
             env={"WM_B200_LIB": "/nonexistent/libwm_b200.so"})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "config", "cpu_baseline", "e2e", "step_rate_cv"):
        assert key in d, key
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["value"] > 0


def test_reference_arm_other_ranks_exit_quietly():
    r = _run(["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "3"],
             env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r.returncode == 0
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
