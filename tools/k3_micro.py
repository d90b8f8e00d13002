#!/usr/bin/env python3
"""K2 + K3 per clip_run_videos step on the C2 video (resident) and clip_merge
of 20,000 near-constant 768-d boundaries, from the library's CUDA events.
usage: python tools/k3_micro.py [--lib=path.so]"""
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
    v = manifest.c2_video(0)
    t = torch_dev.frame_table(v, dev)
    fr = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, t, fr)
    e = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, t, e)
    ctx = Ctx(device=0, timing=True)
    item = [{"n": v.n, "H": v.H, "W": v.W, "frames": fr, "emb": e}]
    for _ in range(3):
        r = ctx.run_videos(item)
    ctx.stats(reset=True)
    for _ in range(10):
        r = ctx.run_videos(item)
    st = ctx.stats(reset=True)
    out = {"lib": libs[0] if libs else "product", "k2_ms": round(st["k2_ms"] / 10, 4),
           "k3_ms": round(st["k3_ms"] / 10, 4), "detected": len(r[0].detected), "final": len(r[0].final)}
    rng = np.random.default_rng(3)
    n = 2 * 20001
    base = rng.standard_normal(768)
    emb = torch.from_numpy((base[None, :] + 0.01 * rng.standard_normal((n, 768))).astype(np.float32)).to(dev)
    cuts = torch.tensor(list(range(2, n, 2)), dtype=torch.int32, device=dev)
    ts = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ctx.stream)
        ctx.merge(emb, cuts)
        b.record(ctx.stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out["merge20k_ms"] = round(float(np.median(ts[1:])), 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
