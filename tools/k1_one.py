#!/usr/bin/env python3
"""One K1 launch per configuration in K1_CFGS on a C2 subsample (for ncu:
ncu -k regex:k1_hist ... python tools/k1_one.py 2000).  Tools only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    dev = torch.device("cuda:0")
    synth.build(device=True)
    v = manifest.subsample(manifest.c2_video(0), n)
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    for c in [int(x) for x in os.environ.get("K1_CFGS", "14").split(",")]:
        os.environ["CLIPDETECT_K1_CFG"] = str(c)
        ctx = Ctx(device=0)
        ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)
        torch.cuda.synchronize()
        ctx.close()
    print("ok")


if __name__ == "__main__":
    main()
