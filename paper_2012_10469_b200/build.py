"""Build libmegb200.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("megb200_kernels.cu", "megb200_coop.cu", "megb200_umma.cu", "megb200_step.cu", "megb200_rr.cu", "megb200_qm.cu", "megb200_runtime.cu")]
HEADERS = [os.path.join(HERE, "csrc", "megb200_internal.h"), os.path.join(HERE, "csrc", "megb200_umma.cuh"),
           os.path.join(HERE, "csrc", "megb200_jacobi.cuh"), os.path.join(os.path.dirname(HERE), "include", "megb200.h")]
TARGET = os.path.join(HERE, "libmegb200.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "174",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(TARGET):
        return False
    t = os.path.getmtime(TARGET)
    return all(os.path.getmtime(p) <= t for p in SOURCES + HEADERS)


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Each translation unit compiles in parallel (-c), then one shared link; the translation units
    share no device code, so no device link step is needed."""
    if not force and up_to_date():
        return TARGET
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [nvcc(), *cflags, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC", "-o",
           TARGET + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(TARGET + ".tmp", TARGET)
    return TARGET


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose=True))
