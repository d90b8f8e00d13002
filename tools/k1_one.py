#!/usr/bin/env python3
"""One launch of each hot kernel on C2 content, for ncu --set full captures:
K1 (RGB24) and K1-NV12 over the first N frames of the C2 video, K4 on the
final clips of a 2,000-frame prefix, and the K3 merge (clip_merge) of that
prefix.  Runs each once untimed (warm-up, module load) then once more.

usage: python tools/k1_one.py [n_frames] [which: k1,nv12,k4,k3,noise]
(noise: K1 over n_frames / 4 uniform-noise 1080p frames, the worst case)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    which = (sys.argv[2] if len(sys.argv) > 2 else "k1,nv12,k4,k3").split(",")
    dev = torch.device("cuda:0")
    synth.build(device=True)
    ctx = Ctx(device=0)
    v = manifest.subsample(manifest.c2_video(0), n)
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    if "k1" in which:
        for _ in range(2):
            ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)
    if "k4" in which or "k3" in which:
        emb = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
        torch_dev.gen_emb(v, table, emb)
        res = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": frames, "emb": emb}])[0]
        cuts = torch.from_numpy(res.detected.astype(np.int32)).to(dev)
        fin = torch.from_numpy(res.final.astype(np.int32)).to(dev)
        if "k3" in which:
            for _ in range(2):
                ctx.merge(emb, cuts)
        if "k4" in which:
            for _ in range(2):
                ctx.sample_frames(frames, fin, 8, 224, 224, want_index=False)
    if "noise" in which:
        nz = manifest.noise_video(1, n=max(1, n // 4))
        ft = torch_dev.frame_table(nz, dev)
        nf = torch.empty((nz.n, nz.H, nz.W, 3), dtype=torch.uint8, device=dev)
        torch_dev.gen_frames(nz, ft, nf)
        nh = torch.empty((nz.n, 162), dtype=torch.int32, device=dev)
        for _ in range(2):
            ctx.frame_scores(nf, hist=nh, want_l1=False, want_score=False)
        del nf
        torch.cuda.empty_cache()
    if "nv12" in which:
        del frames
        torch.cuda.empty_cache()
        nv = torch.empty((v.n, v.H * 3 // 2, v.W), dtype=torch.uint8, device=dev)
        torch_dev.gen_nv12(v, table, nv)
        for _ in range(2):
            ctx.frame_scores_nv12(nv, hist=hist, want_l1=False, want_score=False)
    torch.cuda.synchronize()
    print("k1_one ok", which, n)


if __name__ == "__main__":
    main()
