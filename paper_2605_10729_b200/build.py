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
SOURCES = ["particles.cu", "fields.cu", "capi.cu", "probe.cu", "sampler.cu"]
HEADERS = ["pif_internal.cuh", "es_fast.cuh", os.path.join("..", "..", "include", "pif_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared"]
LIBS = ["-lcufft", "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-Xlinker", "-z,defs"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    cmd = [NVCC, *FLAGS, "-o", OUT, *[os.path.join(CSRC, s) for s in SOURCES], *LIBS]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    tmp = OUT + ".tmp"
    cmd[cmd.index(OUT)] = tmp
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
