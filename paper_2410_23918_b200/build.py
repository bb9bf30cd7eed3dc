"""Build the in-tree CUDA library libbitstack.so for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbitstack.so")
SOURCES = ["bitstack.cu"]


def _deps():
    """Every CUDA source/header under csrc/ plus the public header (content-hashed)."""
    files = sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h")))
    return [os.path.join(CSRC, f) for f in files] + [os.path.join(ROOT, "include", "bitstack.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-lcublas", "-Xlinker", "-rpath=/usr/local/cuda/lib64",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _digest(extra=()) -> str:
    """Content hash of every source + the flags (mtimes do not survive a repo snapshot)."""
    h = hashlib.sha256(" ".join(NVCC_FLAGS + list(extra)).encode())
    for d in _deps():
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _stale(out: str, extra=()) -> bool:
    if not os.path.exists(out) or not os.path.exists(out + ".sha256"):
        return True
    with open(out + ".sha256") as f:
        return f.read().strip() != _digest(extra)


def build(force: bool = False, verbose: bool = False, extra=(), out: str = LIB) -> str:
    """Compile csrc/bitstack.cu into `out` (default: the in-tree libbitstack.so).
    `extra` nvcc flags are for debug variants (e.g. -DBS_DECODE_TRACE) written elsewhere."""
    extra = list(extra)
    if not force and not _stale(out, extra):
        return out
    tmp = out + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp] + [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(tmp, out)
    with open(out + ".sha256", "w") as f:
        f.write(_digest(extra))
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
