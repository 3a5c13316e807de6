"""Build the sm_100a shared library in-tree (no JIT cache, no site-packages).

`python -m paper_1802_06263_b200._build` or `__graft_entry__.build()`
compiles csrc/*.cu with nvcc for `-gencode arch=compute_100a,code=sm_100a`
into paper_1802_06263_b200/_mfb.so, which the ctypes loader (_lib.py) opens.
"""

import glob
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
SO_PATH = os.path.join(PKG, "_mfb.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def source_files():
    return sorted(sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) +
                  glob.glob(os.path.join(REPO, "include", "*.h")))


def source_hash():
    """16 hex digits of SHA-256 over the CUDA sources and the C-ABI header
    (names and contents): embedded in the library (mfb_version) at build
    time and checked against the tree when the library is loaded."""
    h = hashlib.sha256()
    for f in source_files():
        h.update(os.path.relpath(f, REPO).encode())
        with open(f, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def up_to_date():
    if not os.path.exists(SO_PATH) or not os.path.exists(SO_PATH + ".srchash"):
        return False
    with open(SO_PATH + ".srchash") as fh:
        return fh.read().strip() == source_hash()


def build(force=False, verbose=False):
    if not force and up_to_date():
        return SO_PATH
    tmp = SO_PATH + ".tmp"
    src_hash = source_hash()
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
           f"-DMFB_SOURCE_HASH=\"{src_hash}\"",
           "-Xcompiler", "-fPIC", "-I", os.path.join(REPO, "include"),
           "-I", os.path.join(PKG, "csrc"), "-o", tmp, *sources(), "-lcudart"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, SO_PATH)
    with open(SO_PATH + ".srchash", "w") as fh:
        fh.write(src_hash + "\n")
    return SO_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO_PATH)
