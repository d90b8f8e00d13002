"""Device-side input generation with torch tensors as buffers (bench/tests).

Thin wrapper of libsynthdev.so (synth/synth_dev.cu); holds no method arithmetic.
"""
from __future__ import annotations

import numpy as np

from . import dev_lib
from .manifest import Video


def frame_table(v: Video, device) -> "torch.Tensor":
    import torch
    raw = np.ascontiguousarray(v.frames).view(np.uint8)
    return torch.from_numpy(raw.copy()).to(device)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def gen_frames(v: Video, table, out, t0: int = 0, n: int | None = None, stream=None):
    """Frames t0..t0+n-1 of v into out (u8 cuda [n, H, W, 3])."""
    if n is None:
        n = v.n - t0
    rc = dev_lib().synth_dev_gen_frames(v.seed, v.id, v.W, v.H, t0, n, table.data_ptr(),
                                        out.data_ptr(), _stream(stream))
    if rc != 0:
        raise RuntimeError(f"synth_dev_gen_frames failed: cuda error {rc}")
    return out


def gen_nv12(v: Video, table, out, t0: int = 0, n: int | None = None, stream=None):
    """NV12 frames t0..t0+n-1 of v into out (u8 cuda [n, H*3/2, W])."""
    if n is None:
        n = v.n - t0
    rc = dev_lib().synth_dev_gen_nv12(v.seed, v.id, v.W, v.H, t0, n, table.data_ptr(),
                                      out.data_ptr(), _stream(stream))
    if rc != 0:
        raise RuntimeError(f"synth_dev_gen_nv12 failed: cuda error {rc}")
    return out


def gen_emb(v: Video, table, out, t0: int = 0, n: int | None = None, stream=None):
    """Embeddings of frames t0..t0+n-1 into out (f32 cuda [n, D])."""
    if n is None:
        n = v.n - t0
    rc = dev_lib().synth_dev_gen_emb(v.seed, v.id, t0, n, out.shape[1], table.data_ptr(),
                                     out.data_ptr(), _stream(stream))
    if rc != 0:
        raise RuntimeError(f"synth_dev_gen_emb failed: cuda error {rc}")
    return out


def frame_hashes(frames, stream=None) -> np.ndarray:
    """synth.h frame hash of every frame of a u8 cuda [n, H, W, 3] tensor."""
    import torch
    n = frames.shape[0]
    out = torch.empty(n, dtype=torch.int64, device=frames.device)
    rc = dev_lib().synth_dev_frame_hash(frames.data_ptr(), n, frames[0].numel(), out.data_ptr(),
                                        _stream(stream))
    if rc != 0:
        raise RuntimeError(f"synth_dev_frame_hash failed: cuda error {rc}")
    return out.cpu().numpy().view(np.uint64)
