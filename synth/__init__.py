"""Seeded synthetic-input generator shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only frames/embeddings as pure integer
functions of (seed, video, frame, pixel, dim) (``synth.h``), the event
manifests (``manifest.py``) and a frame hash used to prove that host- and
device-generated inputs are identical.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import manifest  # noqa: F401
from .manifest import FRAME_DTYPE, Video  # noqa: F401

HERE = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(HERE, "libsynth.so")
DEV_LIB = os.path.join(HERE, "libsynthdev.so")
NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: str, *srcs: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(os.path.join(HERE, s)) > t for s in srcs)


def build(device: bool = True, force: bool = False) -> None:
    """Compile libsynth.so (gcc) and, if ``device``, libsynthdev.so (nvcc, sm_100a)."""
    if force or _stale(HOST_LIB, "synth_host.c", "synth.h"):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               "-o", HOST_LIB, os.path.join(HERE, "synth_host.c")])
    if device and (force or _stale(DEV_LIB, "synth_dev.cu", "synth.h")):
        subprocess.check_call(["nvcc", *NVCC_ARCH, "-O3", "-lineinfo", "-shared",
                               "-Xcompiler", "-fPIC", "-o", DEV_LIB,
                               os.path.join(HERE, "synth_dev.cu")])


_host = None
_dev = None


def _host_lib():
    global _host
    if _host is None:
        build(device=False)
        lib = ctypes.CDLL(HOST_LIB)
        lib.synth_gen_frames.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                         ctypes.c_uint32, ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.synth_gen_frames.restype = None
        lib.synth_gen_emb.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p,
                                      ctypes.c_void_p]
        lib.synth_gen_emb.restype = None
        lib.synth_frame_hash.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.synth_frame_hash.restype = ctypes.c_uint64
        lib.synth_pixel_ref.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                        ctypes.c_uint32, ctypes.c_void_p]
        lib.synth_pixel_ref.restype = None
        lib.synth_gen_nv12.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_uint32, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.synth_gen_nv12.restype = None
        _host = lib
    return _host


def dev_lib():
    """ctypes handle of libsynthdev.so (device generator)."""
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            raise RuntimeError("synth/libsynthdev.so missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(DEV_LIB)
        lib.synth_dev_gen_frames.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                             ctypes.c_uint32, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_dev_gen_frames.restype = ctypes.c_int
        lib.synth_dev_gen_emb.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_uint32, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_dev_gen_emb.restype = ctypes.c_int
        lib.synth_dev_frame_hash.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                             ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_dev_frame_hash.restype = ctypes.c_int
        lib.synth_dev_gen_nv12.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                           ctypes.c_uint32, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_dev_gen_nv12.restype = ctypes.c_int
        _dev = lib
    return _dev


def _ptr(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


def gen_frames(v: Video, t0: int = 0, n: int | None = None, nthreads: int | None = None,
               out: np.ndarray | None = None) -> np.ndarray:
    """Host frames t0..t0+n-1 of video ``v`` as u8 [n, H, W, 3]."""
    if n is None:
        n = v.n - t0
    assert 0 <= t0 and t0 + n <= v.n
    if out is None:
        out = np.empty((n, v.H, v.W, 3), dtype=np.uint8)
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    fr = np.ascontiguousarray(v.frames)
    _host_lib().synth_gen_frames(v.seed, v.id, v.W, v.H, t0, n, _ptr(fr), _ptr(out), nthreads)
    return out


def gen_nv12(v: Video, t0: int = 0, n: int | None = None, nthreads: int | None = None,
             out: np.ndarray | None = None) -> np.ndarray:
    """Host NV12 frames t0..t0+n-1 of video ``v`` as u8 [n, H*3/2, W] (Y rows then UV rows)."""
    if n is None:
        n = v.n - t0
    assert 0 <= t0 and t0 + n <= v.n and v.W % 2 == 0 and v.H % 2 == 0
    if out is None:
        out = np.empty((n, v.H * 3 // 2, v.W), dtype=np.uint8)
    if nthreads is None:
        nthreads = len(os.sched_getaffinity(0))
    fr = np.ascontiguousarray(v.frames)
    _host_lib().synth_gen_nv12(v.seed, v.id, v.W, v.H, t0, n, _ptr(fr), _ptr(out), nthreads)
    return out


def gen_emb(v: Video, D: int = manifest.EMB_DIM, t0: int = 0, n: int | None = None) -> np.ndarray:
    """Host per-frame embeddings (exact f32) of frames t0..t0+n-1, [n, D]."""
    if n is None:
        n = v.n - t0
    out = np.empty((n, D), dtype=np.float32)
    fr = np.ascontiguousarray(v.frames)
    _host_lib().synth_gen_emb(v.seed, v.id, t0, n, D, _ptr(fr), _ptr(out))
    return out


def frame_hash(frame: np.ndarray) -> int:
    """synth.h frame hash of one frame's bytes."""
    a = np.ascontiguousarray(frame)
    return int(_host_lib().synth_frame_hash(_ptr(a), a.nbytes))


def pixel_ref(v: Video, t: int, x: int, y: int) -> tuple:
    """Uncached synth_pixel() (for testing the memoised generators)."""
    rec = np.ascontiguousarray(v.frames[t:t + 1])
    out = (ctypes.c_uint8 * 3)()
    _host_lib().synth_pixel_ref(v.seed, v.id, t, _ptr(rec), v.W, x, y, out)
    return tuple(out)
