"""Compile libetree.so in-tree for sm_100a (nvcc; no GPU needed)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libetree.so")
SOURCES = ["scan_s16.cu", "scan_s60.cu", "scan_s0.cu", "kernels.cu", "build_gpu.cu", "host.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "-diag-suppress", "550",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "etree.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False, out_dir: str = OUT_DIR, defines=()) -> str:
    """Compile libetree.so into out_dir (defines: extra -D macros for experiment builds)."""
    lib = os.path.join(out_dir, "libetree.so")
    if out_dir == OUT_DIR and not defines and not force and not _stale():
        return LIB
    os.makedirs(out_dir, exist_ok=True)
    objs, procs = [], []
    dflags = [f"-D{d}" for d in defines]
    for src in SOURCES:   # one nvcc per translation unit, in parallel
        obj = os.path.join(out_dir, src.rsplit(".", 1)[0] + ".o")
        cmd = [NVCC, *FLAGS, *dflags, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, *FLAGS, *dflags, "-x", "cu", "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd)))
        objs.append(obj)
    failed = [src for src, pr in procs if pr.wait() != 0]
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    tmp = lib + ".tmp"
    subprocess.run([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs,
                    "-Xlinker", "-z,defs", "-lpthread"], check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
