"""Thin Python binding of libclipdetect (include/clip_detect.h).

Argument marshalling only: every step of the path (rows a1-a9, PAPER.md:35
§2.1) runs in the library's CUDA kernels.  PyTorch provides device memory and
streams.  There is no fallback: if the shared library or a B200 is missing,
every call raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _build

LIB_PATH = _build.LIB

OK, E_INVALID, E_CAPACITY, E_CUDA, E_NOMEM, E_ARCH, E_STATE = range(7)
FLAG_TIMING = 1
ABI_VERSION = 2
DIST_L1, DIST_CHI2, DIST_BHATTACHARYYA, DIST_CORREL = 0, 1, 2, 3  # clip_params.distance (f4)


class ClipError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"clipdetect error {code}: {msg}")
        self.code = code


class ClipParams(ctypes.Structure):
    _fields_ = [("abi_version", ctypes.c_uint32), ("h_bins", ctypes.c_uint32),
                ("s_bins", ctypes.c_uint32), ("v_bins", ctypes.c_uint32),
                ("cut_threshold_ppm", ctypes.c_uint64), ("min_clip_frames", ctypes.c_uint32),
                ("max_merge_rounds", ctypes.c_uint32), ("merge_cos_threshold", ctypes.c_double),
                ("band_rel", ctypes.c_double), ("flags", ctypes.c_uint32),
                ("reserved", ctypes.c_uint32), ("distance", ctypes.c_uint32),
                ("adaptive_window", ctypes.c_uint32), ("adaptive_ratio_ppm", ctypes.c_uint64),
                ("emb_stride", ctypes.c_uint32), ("reserved2", ctypes.c_uint32)]


class ClipVideo(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int64), ("n_frames", ctypes.c_int64), ("height", ctypes.c_int32),
                ("width", ctypes.c_int32), ("dim", ctypes.c_int32), ("format", ctypes.c_int32),
                ("frames", ctypes.c_void_p), ("emb", ctypes.c_void_p)]


class ClipVideoResult(ctypes.Structure):
    _fields_ = [("id", ctypes.c_int64), ("n_candidates", ctypes.c_int64),
                ("n_detected", ctypes.c_int64), ("n_final", ctypes.c_int64),
                ("n_band_hits", ctypes.c_int64), ("detected_offset", ctypes.c_int64),
                ("final_offset", ctypes.c_int64), ("rounds", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class ClipRunOutputs(ctypes.Structure):
    _fields_ = [("hist", ctypes.c_void_p), ("l1", ctypes.c_void_p),
                ("detected_cos", ctypes.c_void_p)]


class ClipStats(ctypes.Structure):
    _fields_ = [("k1_ms", ctypes.c_double), ("k2_ms", ctypes.c_double),
                ("k3_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("k1_launches", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("k1_bytes", ctypes.c_int64), ("memcpy_h2d", ctypes.c_int64),
                ("memcpy_d2h", ctypes.c_int64)]


FILL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                           ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p)

EXPORTS = ["clip_params_default", "clip_detect_init", "clip_detect_destroy", "clip_last_error",
           "clip_frame_scores", "clip_cuts", "clip_merge", "clip_run_videos", "clip_get_stats",
           "clip_debug_binmap", "clip_debug_read_roofline", "clip_frame_scores_nv12",
           "clip_debug_nv12map", "clip_debug_read_roofline_nv12", "clip_sample_frames",
           "clip_hist_scores", "clip_sample_frames_nv12"]

FORMAT_RGB24 = 0
FORMAT_NV12 = 1

_lib = None


def load(build_if_missing: bool = False, path: str | None = None):
    """Load libclipdetect.so (raises if it is missing: no fallback path).
    ``path`` (before the first load only): another build of the same library,
    e.g. the bounds-checked one of tools/sanitize_run.py."""
    global _lib
    if _lib is not None:
        if path is not None and path != _lib._name:
            raise RuntimeError(f"libclipdetect already loaded from {_lib._name}")
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        if build_if_missing:
            _build.build()
        else:
            raise RuntimeError(f"{path} missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    L.clip_params_default.argtypes = [ctypes.POINTER(ClipParams)]
    L.clip_params_default.restype = None
    L.clip_detect_init.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(ClipParams), ctypes.c_int,
                                   ctypes.c_size_t]
    L.clip_detect_destroy.argtypes = [vp]
    L.clip_last_error.argtypes = [vp]
    L.clip_last_error.restype = ctypes.c_char_p
    L.clip_frame_scores.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, vp]
    L.clip_cuts.argtypes = [vp, vp, i64, i64, vp, vp, i64, ctypes.c_int]
    L.clip_merge.argtypes = [vp, vp, i64, i32, vp, i64, vp, ctypes.POINTER(i64), vp,
                             ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.clip_run_videos.argtypes = [vp, ctypes.POINTER(ClipVideo), i32, FILL_FN, vp, i64, vp, i64,
                                  ctypes.POINTER(ClipVideoResult), ctypes.POINTER(ClipRunOutputs)]
    L.clip_get_stats.argtypes = [vp, ctypes.POINTER(ClipStats), ctypes.c_int]
    L.clip_debug_binmap.argtypes = [vp, vp]
    L.clip_debug_read_roofline.argtypes = [vp, vp, i64, i32, i32]
    L.clip_frame_scores_nv12.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, vp]
    L.clip_debug_nv12map.argtypes = [vp, vp]
    L.clip_hist_scores.argtypes = [vp, vp, i64, i64, vp, vp, vp]
    L.clip_sample_frames.argtypes = [vp, vp, i64, i32, i32, vp, i64, i32, i32, i32, vp, vp]
    L.clip_sample_frames_nv12.argtypes = [vp, vp, i64, i32, i32, vp, i64, i32, i32, i32, vp, vp]
    L.clip_debug_read_roofline_nv12.argtypes = [vp, vp, i64, i32, i32]
    for name in EXPORTS:
        if name not in ("clip_params_default", "clip_last_error"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def default_params(**kw) -> ClipParams:
    p = ClipParams()
    load().clip_params_default(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    assert x.is_contiguous(), "tensors must be contiguous"
    return x.data_ptr()


@dataclass
class VideoResult:
    id: int
    n_candidates: int
    detected: np.ndarray
    final: np.ndarray
    detected_cos: np.ndarray | None
    n_band_hits: int
    rounds: int


class Ctx:
    """One libclipdetect context (clip_detect_init) on one GPU / stream."""

    def __init__(self, params: ClipParams | None = None, device: int = 0, stream=None,
                 timing: bool = False):
        import torch
        self._lib = load()
        self.params = params if params is not None else default_params()
        if timing:
            self.params.flags |= FLAG_TIMING
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        self.device = device
        h = ctypes.c_void_p()
        rc = self._lib.clip_detect_init(ctypes.byref(h), ctypes.byref(self.params), device,
                                        stream.cuda_stream)
        if rc != OK:
            raise ClipError(rc, "clip_detect_init failed" + (" (not a B200 / sm_100)" if rc == E_ARCH else ""))
        self._h = h

    # ------------------------------------------------------------ helpers
    @property
    def nbins(self) -> int:
        p = self.params
        return p.h_bins * p.s_bins * p.v_bins

    def _check(self, rc: int):
        if rc != OK:
            raise ClipError(rc, self._lib.clip_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.clip_detect_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ API
    def frame_scores(self, frames, prev_hist=None, hist=None, l1=None, score=None,
                     want_l1: bool = True, want_score: bool = True):
        """clip_frame_scores: rows a1-a4 for one chunk of one video."""
        import torch
        n, H, W, C = frames.shape
        assert C == 3 and frames.dtype == torch.uint8 and frames.is_cuda
        dev = frames.device
        if hist is None:
            hist = torch.empty((n, self.nbins), dtype=torch.int32, device=dev)
        if l1 is None and want_l1:
            l1 = torch.empty(n, dtype=torch.int32, device=dev)
        if score is None and want_score:
            score = torch.empty(n, dtype=torch.float32, device=dev)
        self._check(self._lib.clip_frame_scores(self._h, _ptr(frames), n, H, W, _ptr(prev_hist),
                                                _ptr(hist), _ptr(l1), _ptr(score)))
        return hist, l1, score

    def frame_scores_nv12(self, frames, prev_hist=None, hist=None, l1=None, score=None,
                          want_l1: bool = True, want_score: bool = True):
        """clip_frame_scores_nv12: rows a1-a4 for NV12 frames u8 [n, H*3/2, W] (reading O0)."""
        import torch
        n, H3, W = frames.shape
        assert H3 % 3 == 0 and frames.dtype == torch.uint8 and frames.is_cuda
        H = H3 * 2 // 3
        dev = frames.device
        if hist is None:
            hist = torch.empty((n, self.nbins), dtype=torch.int32, device=dev)
        if l1 is None and want_l1:
            l1 = torch.empty(n, dtype=torch.int32, device=dev)
        if score is None and want_score:
            score = torch.empty(n, dtype=torch.float32, device=dev)
        self._check(self._lib.clip_frame_scores_nv12(self._h, _ptr(frames), n, H, W, _ptr(prev_hist),
                                                     _ptr(hist), _ptr(l1), _ptr(score)))
        return hist, l1, score

    def hist_scores(self, hist, pixels_per_frame: int, prev_hist=None, l1=None, score=None):
        """clip_hist_scores: row a4 from existing histograms (device u32/i32 [n, nbins])."""
        import torch
        n = hist.shape[0]
        if l1 is None:
            l1 = torch.empty(n, dtype=torch.int32, device=hist.device)
        self._check(self._lib.clip_hist_scores(self._h, _ptr(hist), n, pixels_per_frame,
                                               _ptr(prev_hist), _ptr(l1), _ptr(score)))
        return l1, score

    def sample_frames(self, frames, cuts, k: int, out_h: int = 224, out_w: int = 224, out=None,
                      want_index: bool = True):
        """clip_sample_frames (NEXT f3): k frames per clip of one RGB24 video
        ([n, H, W, 3]) or NV12 video ([n, H*3/2, W]), resized to out_h x out_w.  ``cuts``: device int32 tensor of final cuts.
        Returns (out u8 [(n_cuts+1)*k, out_h, out_w, 3], index int32 tensor or None)."""
        import torch
        nv12 = frames.dim() == 3  # NV12 surfaces [n, H*3/2, W]
        if nv12:
            n, H3, W = frames.shape
            H = H3 * 2 // 3
        else:
            n, H, W, C = frames.shape
            assert C == 3
        assert frames.is_cuda
        n_cuts = 0 if cuts is None else cuts.numel()
        m = (n_cuts + 1) * k
        if out is None:
            out = torch.empty((m, out_h, out_w, 3), dtype=torch.uint8, device=frames.device)
        idx = torch.empty(m, dtype=torch.int32, device=frames.device) if want_index else None
        fn = self._lib.clip_sample_frames_nv12 if nv12 else self._lib.clip_sample_frames
        self._check(fn(self._h, _ptr(frames), n, H, W,
                                                 _ptr(cuts) if n_cuts else None, n_cuts, k, out_h,
                                                 out_w, _ptr(out), _ptr(idx)))
        return out, idx

    def cuts(self, l1, pixels_per_frame: int, state, cuts, is_final: bool):
        """clip_cuts: rows a5-a6 streaming; state is a device int64[4] tensor."""
        n = 0 if l1 is None else l1.numel()
        self._check(self._lib.clip_cuts(self._h, _ptr(l1), n, pixels_per_frame, _ptr(state),
                                        _ptr(cuts), cuts.numel(), int(bool(is_final))))

    def merge(self, emb, cuts, n_cuts: int | None = None, want_cos: bool = True):
        """clip_merge: rows a7-a9 for one video.  Returns (final cuts tensor,
        boundary cos tensor, band hits, rounds)."""
        import torch
        n, dim = emb.shape
        if n_cuts is None:
            n_cuts = cuts.numel()
        merged = torch.empty(max(1, n_cuts), dtype=torch.int32, device=emb.device)
        cos = torch.empty(max(1, n_cuts), dtype=torch.float64, device=emb.device) if want_cos else None
        nm = ctypes.c_int64(0)
        hits = ctypes.c_int64(0)
        rounds = ctypes.c_int32(0)
        self._check(self._lib.clip_merge(self._h, _ptr(emb), n, dim, _ptr(cuts), n_cuts,
                                         _ptr(merged), ctypes.byref(nm), _ptr(cos),
                                         ctypes.byref(hits), ctypes.byref(rounds)))
        return merged[:nm.value], (cos[:n_cuts] if cos is not None else None), hits.value, rounds.value

    def run_videos(self, videos: list, fill=None, chunk_frames: int = 0, hist=None, l1=None,
                   want_cos: bool = False, min_clip_frames: int | None = None) -> list:
        """clip_run_videos: rows a1-a9 for a batch.  ``videos``: dicts with
        keys n, H, W, frames (device tensor / numpy array / None), emb (device
        tensor or None), id, format (FORMAT_RGB24 default / FORMAT_NV12)."""
        nv = len(videos)
        arr = (ClipVideo * nv)()
        L = min_clip_frames or self.params.min_clip_frames
        cap = 0
        for i, v in enumerate(videos):
            e = v.get("emb")
            arr[i].id = v.get("id", i)
            arr[i].n_frames = v["n"]
            arr[i].height = v["H"]
            arr[i].width = v["W"]
            arr[i].dim = 0 if e is None else e.shape[1]
            arr[i].format = v.get("format", FORMAT_RGB24)
            arr[i].frames = _ptr(v.get("frames"))
            arr[i].emb = _ptr(e)
            cap += 2 * (v["n"] // L + 1)
        cut_buf = np.empty(max(1, cap), dtype=np.int32)
        cos_buf = np.empty(max(1, cap), dtype=np.float64) if want_cos else None
        res = (ClipVideoResult * nv)()
        outs = ClipRunOutputs(_ptr(hist), _ptr(l1), None if cos_buf is None else cos_buf.ctypes.data)
        if fill is None:
            cb = FILL_FN()
        else:
            def _cb(user, vi, t0, n, dst, stream):
                try:
                    return int(fill(int(vi), int(t0), int(n), int(dst), int(stream or 0)) or 0)
                except Exception as ex:  # pragma: no cover - surfaced as CLIP_E_INVALID
                    print("fill callback failed:", ex)
                    return 1
            cb = FILL_FN(_cb)
        self._check(self._lib.clip_run_videos(self._h, arr, nv, cb, None, chunk_frames,
                                              cut_buf.ctypes.data, cap, res, ctypes.byref(outs)))
        out = []
        for i in range(nv):
            r = res[i]
            det = cut_buf[r.detected_offset:r.detected_offset + r.n_detected].copy()
            fin = cut_buf[r.final_offset:r.final_offset + r.n_final].copy()
            dc = None if cos_buf is None else cos_buf[r.detected_offset:r.detected_offset + r.n_detected].copy()
            out.append(VideoResult(r.id, r.n_candidates, det, fin, dc, r.n_band_hits, r.rounds))
        return out

    def stats(self, reset: bool = False) -> dict:
        s = ClipStats()
        self._check(self._lib.clip_get_stats(self._h, ctypes.byref(s), int(reset)))
        return {k: getattr(s, k) for k, _ in ClipStats._fields_}

    def debug_binmap(self):
        import torch
        t = torch.empty(2 << 24, dtype=torch.uint8, device=f"cuda:{self.device}")
        self._check(self._lib.clip_debug_binmap(self._h, _ptr(t)))
        return t.view(2, 1 << 24)

    def debug_read_roofline(self, frames):
        n, H, W, _ = frames.shape
        self._check(self._lib.clip_debug_read_roofline(self._h, _ptr(frames), n, H, W))

    def debug_nv12map(self):
        """K5 for NV12: [2, 1<<24] bins of every (Y, U, V) in lane 0 / lane 1."""
        import torch
        t = torch.empty(2 << 24, dtype=torch.uint8, device=f"cuda:{self.device}")
        self._check(self._lib.clip_debug_nv12map(self._h, _ptr(t)))
        return t.view(2, 1 << 24)

    def debug_read_roofline_nv12(self, frames):
        n, H3, W = frames.shape
        self._check(self._lib.clip_debug_read_roofline_nv12(self._h, _ptr(frames), n, H3 * 2 // 3, W))


_run_ctx = {}


def run(frames, emb=None, params: ClipParams | None = None, want_detected: bool = False):
    """One video through rows a1-a9 (SURVEY.md §8(b) "Python shell"):
    ``frames`` u8 cuda [T, H, W, 3] (RGB24) or [T, H*3/2, W] (NV12), ``emb`` f32
    cuda [T, D] or None (no merge).  Uses a cached Ctx per (device, params) on the
    current stream.  Returns the final cut list (and the detected cuts if
    ``want_detected``)."""
    import torch
    dev = frames.device.index or 0
    key = (dev, None if params is None else bytes(params))
    ctx = _run_ctx.get(key)
    if ctx is None or ctx.stream != torch.cuda.current_stream(dev):
        ctx = Ctx(params, device=dev)
        _run_ctx[key] = ctx
    nv12 = frames.dim() == 3
    T = frames.shape[0]
    H = frames.shape[1] * 2 // 3 if nv12 else frames.shape[1]
    W = frames.shape[2]
    item = {"n": T, "H": H, "W": W, "frames": frames, "emb": emb,
            "format": FORMAT_NV12 if nv12 else FORMAT_RGB24}
    r = ctx.run_videos([item])[0]
    fin = [int(x) for x in r.final]
    return (fin, [int(x) for x in r.detected]) if want_detected else fin
