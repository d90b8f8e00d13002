#!/usr/bin/env python3
"""K4 (frame sampling + resize) micro-benchmark: C2 frames resident, final-cut
like clips (one every 127 frames), k = 8 at 224x224, per-CTA staging budget
swept through CLIPDETECT_K4_BUDGET_KB.  CUDA events; prints one JSON line."""
import json
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
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 18000
    dev = torch.device("cuda:0")
    synth.build(device=True)
    v = manifest.subsample(manifest.c2_video(0), n)
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    cuts = torch.arange(127, v.n, 127, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream()
    ctx = Ctx(device=0, stream=stream)
    S, k = 224, 8
    m = (cuts.numel() + 1) * k
    out = torch.empty((m, S, S, 3), dtype=torch.uint8, device=dev)
    alg = m * (448 * 3 * v.W + S * S * 3)  # 720 -> 224: 448 distinct source rows
    res = {}
    for kb in [int(x) for x in os.environ.get("K4_BUDGETS", "40,24,32,48,64,96").split(",")]:
        os.environ["CLIPDETECT_K4_BUDGET_KB"] = str(kb)
        with torch.cuda.stream(stream):
            for _ in range(3):
                ctx.sample_frames(frames, cuts, k, S, S, out=out, want_index=False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(10):
                ctx.sample_frames(frames, cuts, k, S, S, out=out, want_index=False)
            e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[f"budget_{kb}kb"] = {"ms": round(ms, 4), "gbs": round(alg / ms / 1e6, 1)}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
