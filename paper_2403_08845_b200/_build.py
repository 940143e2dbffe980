"""Build libbifattn.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension: the .so is a plain C-ABI library loaded with ctypes)."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libbifattn.so")
SRC = os.path.join(HERE, "csrc", "bifattn_api.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",
    "-diag-suppress", "177",
]


def _sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*"))) + [os.path.join(ROOT, "include", "bifattn.h")]


def source_hash(extra=()) -> str:
    """sha256 over the sources, the nvcc flags and the nvcc path: the library is
    rebuilt whenever any of them changes (never reused on a newer mtime)."""
    h = hashlib.sha256()
    for s in _sources():
        h.update(os.path.basename(s).encode())
        with open(s, "rb") as f:
            h.update(f.read())
    h.update(" ".join([NVCC, *NVCC_FLAGS, *extra]).encode())
    return h.hexdigest()


def needs_build() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".srchash"):
        return True
    with open(LIB + ".srchash") as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if force or needs_build():
        cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp", SRC]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        os.replace(LIB + ".tmp", LIB)
        with open(LIB + ".srchash", "w") as f:
            f.write(source_hash() + "\n")
    return LIB



def build_variant(name: str, defines, force: bool = False) -> str:
    """An instrumented build of the same sources (e.g. -DBIFATTN_TRACE: the
    %globaltimer timeline of scripts/timeline.py) next to the product
    library: libbifattn_<name>.so.  Never loaded by the product binding."""
    out = os.path.join(HERE, f"libbifattn_{name}.so")
    stamp = out + ".srchash"
    h = source_hash(tuple(defines))
    if force or not os.path.exists(out) or not os.path.exists(stamp) or open(stamp).read().strip() != h:
        cmd = [NVCC, *NVCC_FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-o", out + ".tmp", SRC]
        subprocess.check_call(cmd)
        os.replace(out + ".tmp", out)
        with open(stamp, "w") as f:
            f.write(h + "\n")
    return out


if __name__ == "__main__":
    print(build(force=True, verbose=True))
