#!/usr/bin/env python3
"""NV12 K1 micro-benchmark: the fused NV12 histogram kernel against the same
TMA pipeline without binning (NV12 read roofline), on C2 content (NV12
surfaces of the synthetic generator) and on uniform-noise NV12 frames.  CUDA
events on the ctx stream; inputs >> L2.  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx  # noqa: E402

from k1_micro import timeit  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--lib=")]
    libs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--lib=")]
    if libs:  # A/B of another build of the library (tools only)
        from paper_2503_12964_b200 import clipdetect
        clipdetect.load(path=os.path.abspath(libs[0]))
    n = int(args[0]) if args else 6000
    dev = torch.device("cuda:0")
    synth.build(device=True)
    stream = torch.cuda.Stream()
    ctx = Ctx(device=0, stream=stream)
    out = {}
    for name, v in [("c2", manifest.subsample(manifest.c2_video(0), n)),
                    ("c2_1080p_shape", None), ("noise", None)]:
        if v is None:
            W, H = (1920, 1080) if name == "c2_1080p_shape" else (1280, 720)
            g = torch.Generator(device=dev).manual_seed(5)
            frames = torch.randint(0, 256, (n * 720 * 1280 // (W * H), H * 3 // 2, W),
                                   dtype=torch.uint8, device=dev, generator=g)
            if name == "c2_1080p_shape":
                frames[:, :H] //= 64  # coarse luma levels: spatially coherent codes
                frames[:, :H] *= 64
        else:
            table = torch_dev.frame_table(v, dev)
            frames = torch.empty((v.n, v.H * 3 // 2, v.W), dtype=torch.uint8, device=dev)
            torch_dev.gen_nv12(v, table, frames)
        hist = torch.empty((frames.shape[0], 162), dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        nbytes = frames.numel()
        npix = nbytes * 2 // 3
        with torch.cuda.stream(stream):
            ms_k1 = timeit(lambda: ctx.frame_scores_nv12(frames, hist=hist, want_l1=False,
                                                         want_score=False), stream)
            ms_rd = timeit(lambda: ctx.debug_read_roofline_nv12(frames), stream)
        out[name] = {"frames": frames.shape[0], "bytes": nbytes, "k1_ms": round(ms_k1, 3),
                     "k1_gbs": round(nbytes / ms_k1 / 1e6, 1),
                     "k1_gpix_s": round(npix / ms_k1 / 1e6, 1),
                     "read_ms": round(ms_rd, 3), "read_gbs": round(nbytes / ms_rd / 1e6, 1),
                     "k1_frac_of_read": round(ms_rd / ms_k1, 3)}
        del frames, hist
        torch.cuda.empty_cache()
    out["lib"] = libs[0] if libs else "product"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
