"""CPU ORACLE for shot-boundary clip splitting — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2503_12964_b200``) never imports it and shares no code
with it.  The arithmetic lives in ``oracle.c`` (plain C, one function per
reading O1..O9 of DESIGN.md §"Readings"; §2.1); this module only
marshals numpy arrays through ctypes.

Parity status: every function is pinned by tests/test_oracle_*.py against
values and properties fixed independently of this code (named colours, the
``colorsys`` library routine off exact bin edges, hand-computed 4x4 histograms,
brute force, closed forms, planted ground truth, the merge worked examples).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")


@dataclass
class Params:
    """Oracle parameters (defaults = DESIGN.md readings O1, O4, O5, O9)."""
    nh: int = 18
    ns: int = 3
    nv: int = 3
    tau_ppm: int = 300000
    l_min: int = 8
    theta: float = 0.90
    band_rel: float = 1e-5
    max_rounds: int = 0

    @property
    def nbins(self) -> int:
        return self.nh * self.ns * self.nv


class _CParams(ctypes.Structure):
    _fields_ = [("nh", ctypes.c_int32), ("ns", ctypes.c_int32), ("nv", ctypes.c_int32),
                ("tau_ppm", ctypes.c_int64), ("l_min", ctypes.c_int64),
                ("theta", ctypes.c_double), ("band_rel", ctypes.c_double),
                ("max_rounds", ctypes.c_int32)]


class _CResult(ctypes.Structure):
    _fields_ = [("n_candidates", ctypes.c_int64), ("n_detected", ctypes.c_int64),
                ("n_final", ctypes.c_int64), ("n_band_hits", ctypes.c_int64),
                ("rounds", ctypes.c_int32)]


def build(force: bool = False) -> None:
    """Compile liboracle.so with gcc (plain C, -O2, no -ffast-math)."""
    srcs = [os.path.join(HERE, "oracle.c"), os.path.join(HERE, "oracle.h")]
    if not force and os.path.exists(LIB) and all(
            os.path.getmtime(s) <= os.path.getmtime(LIB) for s in srcs):
        return
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off",
                           "-shared", "-fPIC", "-pthread", "-o", LIB, srcs[0], "-lm"])


_lib = None
P = ctypes.c_void_p
I32, I64, U64, F64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        sigs = {
            "oracle_bin": (I32, [I32, I32, I32, I32, I32, I32]),
            "oracle_bin_table": (None, [I32, I32, I32, P]),
            "oracle_hist": (None, [P, I64, I32, I32, I32, P]),
            "oracle_hist_frames": (None, [P, I64, I64, I32, I32, I32, P, ctypes.c_int]),
            "oracle_l1": (None, [P, I64, I32, I64, P, P]),
            "oracle_candidates": (I64, [P, I64, I64, I64, P]),
            "oracle_min_length": (I64, [P, I64, I64, I64, P]),
            "oracle_clip_sum": (None, [P, I64, I64, I64, P]),
            "oracle_cosine": (F64, [P, P, I64]),
            "oracle_merge": (I64, [P, I64, I64, P, I64, F64, F64, I32, P, P, P, P]),
            "oracle_merge_stride": (I64, [P, I64, I64, P, I64, F64, F64, I32, I64, P, P, P, P]),
            "oracle_video": (ctypes.c_int, [P, I64, I64, P, I64, P, ctypes.c_int, P, P, P, P,
                                            P, P, P]),
            "oracle_nv12_to_rgb": (None, [P, I64, I64, P]),
            "oracle_hist_nv12_frames": (None, [P, I64, I64, I64, I32, I32, I32, P, ctypes.c_int]),
            "oracle_sample_index": (I64, [I64, I64, I64, I64]),
            "oracle_distance": (F64, [P, P, I32, I64, I32]),
            "oracle_distances": (None, [P, I64, I32, I64, I32, P]),
            "oracle_candidates_f64": (I64, [P, I64, I64, P]),
            "oracle_candidates_adaptive": (I64, [P, I64, I64, I64, I64, I64, P]),
            "oracle_resize_linear": (None, [P, I64, I64, P, I64, I64]),
            "oracle_sample_clips": (None, [P, I64, I64, I64, P, I64, I64, I64, I64, P, P]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle inputs must be C-contiguous"
    return a.ctypes.data


def _nthreads(n: int | None) -> int:
    return n if n else len(os.sched_getaffinity(0))


# ---------------------------------------------------------------- O1 / O2
def pixel_bin(r: int, g: int, b: int, p: Params = Params()) -> int:
    return int(lib().oracle_bin(r, g, b, p.nh, p.ns, p.nv))


def bin_table(p: Params = Params()) -> np.ndarray:
    """O1 over all 2^24 colours, indexed (r<<16)|(g<<8)|b."""
    t = np.empty(1 << 24, dtype=np.uint8)
    lib().oracle_bin_table(p.nh, p.ns, p.nv, _p(t))
    return t


def hist(frame: np.ndarray, p: Params = Params()) -> np.ndarray:
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    assert f.size % 3 == 0
    out = np.empty(p.nbins, dtype=np.uint32)
    lib().oracle_hist(_p(f), f.size // 3, p.nh, p.ns, p.nv, _p(out))
    return out


def hist_frames(frames: np.ndarray, p: Params = Params(), nthreads: int | None = None) -> np.ndarray:
    f = np.ascontiguousarray(frames, dtype=np.uint8)
    n = f.shape[0]
    npix = f[0].size // 3 if n else 0
    out = np.empty((n, p.nbins), dtype=np.uint32)
    lib().oracle_hist_frames(_p(f), n, npix, p.nh, p.ns, p.nv, _p(out), _nthreads(nthreads))
    return out


# ---------------------------------------------------------------- O0 (NV12)
def nv12_to_rgb(frame: np.ndarray) -> np.ndarray:
    """One NV12 frame u8 [H*3/2, W] -> RGB24 u8 [H, W, 3] (reading O0)."""
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    H, W = f.shape[0] * 2 // 3, f.shape[1]
    out = np.empty((H, W, 3), dtype=np.uint8)
    lib().oracle_nv12_to_rgb(_p(f), H, W, _p(out))
    return out


def hist_nv12_frames(frames: np.ndarray, p: Params = Params(), nthreads: int | None = None) -> np.ndarray:
    """O0 + O2 for n NV12 frames u8 [n, H*3/2, W] -> [n, nbins]."""
    f = np.ascontiguousarray(frames, dtype=np.uint8)
    n = f.shape[0]
    H, W = f.shape[1] * 2 // 3, f.shape[2]
    out = np.empty((n, p.nbins), dtype=np.uint32)
    lib().oracle_hist_nv12_frames(_p(f), n, H, W, p.nh, p.ns, p.nv, _p(out), _nthreads(nthreads))
    return out


def run_video_nv12(frames: np.ndarray, emb: np.ndarray | None, p: Params = Params(),
                   nthreads: int | None = None) -> VideoResult:
    """The whole path (O0 then O1..O9) for one NV12 video u8 [n, H*3/2, W]."""
    h = hist_nv12_frames(frames, p, nthreads)
    n = h.shape[0]
    npix = frames.shape[2] * frames.shape[1] * 2 // 3
    l1_, sc = l1(h, npix)
    cand = candidates(l1_, npix, p)
    det = min_length(cand, n, p.l_min)
    if emb is None:
        return VideoResult(h, l1_, sc, int(cand.size), det, det.copy(), np.zeros(det.size), 0, 0)
    m = merge(emb, det, p)
    return VideoResult(h, l1_, sc, int(cand.size), det, m.final, m.cos, m.n_band_hits, m.rounds)


# ---------------------------------------------------------------- O3..O6
def l1(hist_: np.ndarray, npix: int) -> tuple:
    h = np.ascontiguousarray(hist_, dtype=np.uint32)
    n, nbins = h.shape
    out = np.empty(n, dtype=np.uint32)
    score = np.empty(n, dtype=np.float64)
    lib().oracle_l1(_p(h), n, nbins, npix, _p(out), _p(score))
    return out, score


def candidates(l1_: np.ndarray, npix: int, p: Params = Params()) -> np.ndarray:
    a = np.ascontiguousarray(l1_, dtype=np.uint32)
    out = np.empty(max(1, a.size), dtype=np.int64)
    k = lib().oracle_candidates(_p(a), a.size, npix, p.tau_ppm, _p(out))
    return out[:k].copy()


def min_length(cand: np.ndarray, n: int, l_min: int) -> np.ndarray:
    c = np.ascontiguousarray(cand, dtype=np.int64)
    out = np.empty(max(1, c.size), dtype=np.int64)
    k = lib().oracle_min_length(_p(c), c.size, n, l_min, _p(out))
    return out[:k].copy()


# ---------------------------------------------------------------- O8 / O9
def clip_sum(emb: np.ndarray, f0: int, f1: int) -> np.ndarray:
    e = np.ascontiguousarray(emb, dtype=np.float32)
    S = np.empty(e.shape[1], dtype=np.float64)
    lib().oracle_clip_sum(_p(e), e.shape[1], f0, f1, _p(S))
    return S


def cosine(a: np.ndarray, b: np.ndarray) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return float(lib().oracle_cosine(_p(a), _p(b), a.size))


@dataclass
class MergeResult:
    final: np.ndarray
    cos: np.ndarray
    n_band_hits: int
    rounds: int


def merge(emb: np.ndarray, cuts, p: Params = Params(), stride: int = 1) -> MergeResult:
    """O8 + O9 (stride > 1: O8' keyframe stride, NEXT f4)."""
    e = np.ascontiguousarray(emb, dtype=np.float32)
    n, dim = e.shape
    c = np.ascontiguousarray(np.asarray(cuts, dtype=np.int64))
    fin = np.empty(max(1, c.size), dtype=np.int64)
    cos = np.empty(max(1, c.size), dtype=np.float64)
    hits = ctypes.c_int64(0)
    rounds = ctypes.c_int32(0)
    k = lib().oracle_merge_stride(_p(e), n, dim, _p(c), c.size, p.theta, p.band_rel, p.max_rounds,
                                  stride, _p(fin), _p(cos), ctypes.byref(hits), ctypes.byref(rounds))
    return MergeResult(fin[:k].copy(), cos[:c.size].copy(), int(hits.value), int(rounds.value))


# ---------------------------------------------------------------- the path
@dataclass
class VideoResult:
    hist: np.ndarray
    l1: np.ndarray
    score: np.ndarray
    n_candidates: int
    detected: np.ndarray
    final: np.ndarray
    cos: np.ndarray
    n_band_hits: int
    rounds: int


def run_video(frames: np.ndarray, emb: np.ndarray | None, p: Params = Params(),
              nthreads: int | None = None) -> VideoResult:
    f = np.ascontiguousarray(frames, dtype=np.uint8)
    n = f.shape[0]
    npix = f[0].size // 3
    e = None if emb is None else np.ascontiguousarray(emb, dtype=np.float32)
    dim = 0 if e is None else e.shape[1]
    h = np.empty((n, p.nbins), dtype=np.uint32)
    l1_ = np.empty(n, dtype=np.uint32)
    sc = np.empty(n, dtype=np.float64)
    det = np.empty(max(1, n), dtype=np.int64)
    fin = np.empty(max(1, n), dtype=np.int64)
    cos = np.zeros(max(1, n), dtype=np.float64)
    cp = _CParams(p.nh, p.ns, p.nv, p.tau_ppm, p.l_min, p.theta, p.band_rel, p.max_rounds)
    res = _CResult()
    lib().oracle_video(_p(f), n, npix, _p(e), dim, ctypes.byref(cp), _nthreads(nthreads),
                       _p(h), _p(l1_), _p(sc), _p(det), _p(fin), _p(cos), ctypes.byref(res))
    nd = res.n_detected
    return VideoResult(h, l1_, sc, int(res.n_candidates), det[:nd].copy(),
                       fin[:res.n_final].copy(), cos[:nd].copy(), int(res.n_band_hits),
                       int(res.rounds))


# ---------------------------------------------------------------- O10/O11 (NEXT f3)
def sample_index(s: int, e: int, i: int, k: int) -> int:
    """O10: frame i of k sampled from clip [s, e)."""
    return int(lib().oracle_sample_index(s, e, i, k))


def resize_linear(frame: np.ndarray, H2: int, W2: int) -> np.ndarray:
    """O11: one RGB24 frame [H, W, 3] -> [H2, W2, 3]."""
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    out = np.empty((H2, W2, 3), dtype=np.uint8)
    lib().oracle_resize_linear(_p(f), f.shape[0], f.shape[1], _p(out), H2, W2)
    return out


def sample_clips(frames: np.ndarray, cuts, k: int, H2: int, W2: int) -> tuple:
    """O10 + O11 for one video: (out u8 [(n_cuts+1)*k, H2, W2, 3], index i64 [(n_cuts+1)*k])."""
    f = np.ascontiguousarray(frames, dtype=np.uint8)
    c = np.ascontiguousarray(np.asarray(cuts, dtype=np.int64))
    m = (c.size + 1) * k
    out = np.empty((m, H2, W2, 3), dtype=np.uint8)
    idx = np.empty(m, dtype=np.int64)
    lib().oracle_sample_clips(_p(f), f.shape[0], f.shape[1], f.shape[2], _p(c) if c.size else None,
                              c.size, k, H2, W2, _p(out), _p(idx))
    return out, idx


# ---------------------------------------------------------------- O3'/O4' (NEXT f4)
DIST_L1, DIST_CHI2, DIST_BHATTACHARYYA, DIST_CORREL = 0, 1, 2, 3


def distance(a: np.ndarray, b: np.ndarray, npix: int, kind: int) -> float:
    """O3': f64 distance of two histograms (kind 1 chi-square, 2 Bhattacharyya, 3 1 - correlation)."""
    x = np.ascontiguousarray(a, dtype=np.uint32)
    y = np.ascontiguousarray(b, dtype=np.uint32)
    return float(lib().oracle_distance(_p(x), _p(y), x.size, npix, kind))


def distances(hist_: np.ndarray, npix: int, kind: int) -> np.ndarray:
    h = np.ascontiguousarray(hist_, dtype=np.uint32)
    d = np.empty(h.shape[0], dtype=np.float64)
    lib().oracle_distances(_p(h), h.shape[0], h.shape[1], npix, kind, _p(d))
    return d


def candidates_f64(d: np.ndarray, p: Params = Params()) -> np.ndarray:
    x = np.ascontiguousarray(d, dtype=np.float64)
    out = np.empty(max(1, x.size), dtype=np.int64)
    k = lib().oracle_candidates_f64(_p(x), x.size, p.tau_ppm, _p(out))
    return out[:k].copy()


def candidates_adaptive(l1_: np.ndarray, npix: int, w: int, ratio_ppm: int,
                        p: Params = Params()) -> np.ndarray:
    x = np.ascontiguousarray(l1_, dtype=np.uint32)
    out = np.empty(max(1, x.size), dtype=np.int64)
    k = lib().oracle_candidates_adaptive(_p(x), x.size, npix, p.tau_ppm, w, ratio_ppm, _p(out))
    return out[:k].copy()


def run_video_variant(frames: np.ndarray, emb: np.ndarray | None, p: Params = Params(),
                      distance_kind: int = DIST_L1, adaptive_window: int = 0,
                      adaptive_ratio_ppm: int = 3000000, nv12: bool = False,
                      emb_stride: int = 1, nthreads: int | None = None) -> VideoResult:
    """The path with the f4 variants: O1/O2 (or O0 first for NV12), then O3 (L1)
    or O3' (distance_kind), O4 / O4' / O4'' (adaptive_window > 0, on L1), O5-O9."""
    h = hist_nv12_frames(frames, p, nthreads) if nv12 else hist_frames(frames, p, nthreads)
    n = h.shape[0]
    npix = (frames.shape[1] * 2 // 3) * frames.shape[2] if nv12 else frames[0].size // 3
    l1_, sc = l1(h, npix)
    if adaptive_window > 0:
        cand = candidates_adaptive(l1_, npix, adaptive_window, adaptive_ratio_ppm, p)
    elif distance_kind != DIST_L1:
        sc = distances(h, npix, distance_kind)
        cand = candidates_f64(sc, p)
    else:
        cand = candidates(l1_, npix, p)
    det = min_length(cand, n, p.l_min)
    if emb is None:
        return VideoResult(h, l1_, sc, int(cand.size), det, det.copy(), np.zeros(det.size), 0, 0)
    m = merge(emb, det, p, stride=emb_stride)
    return VideoResult(h, l1_, sc, int(cand.size), det, m.final, m.cos, m.n_band_hits, m.rounds)
