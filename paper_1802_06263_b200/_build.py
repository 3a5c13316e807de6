"""Build the sm_100a shared library in-tree (no JIT cache, no site-packages).

`python -m paper_1802_06263_b200._build` or `__graft_entry__.build()`
compiles csrc/*.cu with nvcc for `-gencode arch=compute_100a,code=sm_100a`
into paper_1802_06263_b200/_mfb.so, which the ctypes loader (_lib.py) opens.
"""

import glob
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


def up_to_date():
    if not os.path.exists(SO_PATH):
        return False
    t = os.path.getmtime(SO_PATH)
    deps = sources() + glob.glob(os.path.join(PKG, "csrc", "*.cuh")) + \
        glob.glob(os.path.join(REPO, "include", "*.h"))
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return SO_PATH
    tmp = SO_PATH + ".tmp"
    cmd = [nvcc_path(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
           "-Xcompiler", "-fPIC", "-I", os.path.join(REPO, "include"),
           "-I", os.path.join(PKG, "csrc"), "-o", tmp, *sources(), "-lcudart"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, SO_PATH)
    return SO_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(SO_PATH)
