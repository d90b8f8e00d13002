"""Build libclipdetect.so in-tree with nvcc for sm_100a (no JIT cache)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libclipdetect.so")
SOURCES = ["hist.cu", "hist_nv12.cu", "cuts.cu", "merge.cu", "sample.cu", "api.cu"]
HEADERS = ["common.cuh", "binfn.cuh", "kernels.cuh"]
PUBLIC_HEADER = os.path.join(os.path.dirname(HERE), "include", "clip_detect.h")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def _inputs():
    return [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [PUBLIC_HEADER]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _inputs())


CHECKED_LIB = os.path.join(HERE, "build_checked", "libclipdetect_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Each source compiled to an object in parallel, then one shared-library link.
    checked: the bounds-checked build (-DCLIPDETECT_CHECKED, common.cuh CD_CHECK)
    in build_checked/ — a test tool, never the product library."""
    lib = CHECKED_LIB if checked else LIB
    if force or not os.path.exists(lib) or any(os.path.getmtime(p) > os.path.getmtime(lib)
                                               for p in _inputs()):
        from concurrent.futures import ThreadPoolExecutor

        objdir = os.path.join(HERE, "build_checked" if checked else "build")
        os.makedirs(objdir, exist_ok=True)
        cflags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DCLIPDETECT_CHECKED"] if checked else [])
        if verbose:
            cflags = ["-Xptxas=-v"] + cflags

        def compile_one(src):
            obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
            subprocess.check_call(["nvcc", *cflags, "-c", "-o", obj, os.path.join(CSRC, src)],
                                  cwd=CSRC)
            return obj

        with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
            objs = list(ex.map(compile_one, SOURCES))
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-Xcompiler", "-fPIC", "-o", lib, *objs], cwd=CSRC)
    return lib
