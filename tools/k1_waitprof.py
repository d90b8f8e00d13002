#!/usr/bin/env python3
"""Diagnosis with the wait-profiling build (tools/ab/vW.so, not the product): the share
of K1 consumer time spent waiting on the ring's full barriers (clock64 around each wait,
summed over warps), on C2 content and on uniform noise."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx, clipdetect  # noqa: E402


def main():
    L = clipdetect.load(path=os.path.abspath(sys.argv[1]))
    dev = torch.device("cuda:0")
    synth.build(device=True)
    ctx = Ctx(device=0)
    out = {}
    for name, v in [("c2", manifest.subsample(manifest.c2_video(0), 6000)),
                    ("noise", manifest.noise_video(0, 1280, 720, 6000))]:
        table = torch_dev.frame_table(v, dev)
        frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
        torch_dev.gen_frames(v, table, frames)
        hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
        ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)
        buf = (ctypes.c_ulonglong * 2)()
        L.clip_debug_sink(ctx._h, buf)
        for _ in range(3):
            ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)
        L.clip_debug_sink(ctx._h, buf)
        out[name] = {"consumer_wait_share": round(buf[0] / buf[1], 4), "wait_cycles": buf[0], "total_cycles": buf[1]}
        del frames
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
