"""Build libpifb200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2605_10729_b200.build [--force]
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpifb200.so")
SOURCES = ["particles.cu", "fields.cu", "capi.cu", "probe.cu", "sampler.cu", "comm.cu"]
HEADERS = ["pif_internal.cuh", "es_fast.cuh", os.path.join("..", "..", "include", "pif_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
LIBS = ["-lcufft", "-ldl", "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-Xlinker", "-z,defs"]


OBJDIR = os.path.join(HERE, "build")
CFLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
          "-Xcompiler", "-fPIC"]


def _headers():
    return [os.path.join(CSRC, h) for h in HEADERS]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + _headers()
    return any(os.path.getmtime(d) > t for d in deps)


def _obj(src: str, force: bool, verbose: bool) -> str:
    """Compile one translation unit to build/<name>.o unless it is up to date
    (its source and every shared header older than the object)."""
    os.makedirs(OBJDIR, exist_ok=True)
    obj = os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")
    srcp = os.path.join(CSRC, src)
    if not force and os.path.exists(obj):
        t = os.path.getmtime(obj)
        if all(os.path.getmtime(d) <= t for d in [srcp, *_headers()]):
            return obj
    cmd = [NVCC, *CFLAGS, "-c", "-o", obj + ".tmp", srcp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile the translation units in parallel (stale ones only unless
    force) and link libpifb200.so."""
    if not force and not _stale():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _obj(s, force, verbose), SOURCES))
    tmp = OUT + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
           *LIBS]
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
