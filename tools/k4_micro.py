#!/usr/bin/env python3
"""K4 (f3) timing: k = 8 frames per final clip of the first 6,000 C2 frames,
resized to 224^2 (RGB24 and NV12), CUDA events; prints GB/s of algorithmic
bytes (source rows staged + output) and an output hash.
usage: python tools/k4_micro.py [--lib=path.so]"""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx, clipdetect  # noqa: E402


def main():
    libs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--lib=")]
    if libs:
        clipdetect.load(path=os.path.abspath(libs[0]))
    dev = torch.device("cuda:0")
    v = manifest.subsample(manifest.c2_video(0), 6000)
    t = torch_dev.frame_table(v, dev)
    fr = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, t, fr)
    e = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, t, e)
    ctx = Ctx(device=0)
    r = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": fr, "emb": e}])[0]
    cuts = torch.from_numpy(r.final.astype(np.int32)).to(dev)
    k, S = 8, 224
    m = (len(r.final) + 1) * k
    out = torch.empty((m, S, S, 3), dtype=torch.uint8, device=dev)
    for _ in range(3):
        ctx.sample_frames(fr, cuts, k, S, S, out=out, want_index=False)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream)
    for _ in range(20):
        ctx.sample_frames(fr, cuts, k, S, S, out=out, want_index=False)
    b.record(ctx.stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    # algorithmic bytes: per output frame the 2 source rows of each output row + the output
    alg = m * (S * 2 * v.W * 3 + S * S * 3)
    h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
    print(json.dumps({"lib": libs[0] if libs else "product", "frames_out": m, "k4_ms": round(ms, 4),
                      "gbs": round(alg / ms / 1e6, 1), "out_sha16": h}))


if __name__ == "__main__":
    main()
