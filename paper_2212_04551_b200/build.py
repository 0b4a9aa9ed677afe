"""In-tree build of ``libwm_b200.so`` for sm_100a (nvcc cross-compiles
without a GPU).  ``python -m paper_2212_04551_b200.build``.

Each ``csrc/*.cu`` compiles to its own object in ``build/`` (in parallel,
only when stale), then one link step produces the shared library."""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
OUT = os.path.join(HERE, "libwm_b200.so")
SOURCES = ["wm_api.cu", "wm_clique.cu", "wm_motif.cu", "wm_ingest.cu", "wm_dict.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-fopenmp", "-Xptxas", "-O3",
                "-I", os.path.join(ROOT, "include")]


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "warpmine_b200.h"))
    return hs


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.splitext(src)[0] + ".o")


def _stale_obj(src: str, hdr_t: float) -> bool:
    o = _obj(src)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    return os.path.getmtime(os.path.join(CSRC, src)) > t or hdr_t > t


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdr_t = max(os.path.getmtime(h) for h in _headers())
    todo = [s for s in SOURCES if force or _stale_obj(s, hdr_t)]
    if todo:
        with ThreadPoolExecutor(max_workers=len(todo)) as ex:
            futs = [ex.submit(_run, [NVCC, *FLAGS, "-c", "-o", _obj(s) + ".tmp",
                                     os.path.join(CSRC, s)], verbose) for s in todo]
            for f in futs:
                f.result()
        for s in todo:
            os.replace(_obj(s) + ".tmp", _obj(s))
    objs = [_obj(s) for s in SOURCES]
    if todo or not os.path.exists(OUT) or any(os.path.getmtime(o) > os.path.getmtime(OUT)
                                              for o in objs):
        tmp = OUT + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-Xcompiler", "-fopenmp", "-o", tmp, *objs, "-lgomp"],
             verbose)
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
