#!/usr/bin/env python3
"""A/B of K1 launch configurations on the full C2 video (the bench workload):
configurations interleaved, R rounds, median K1 GB/s per configuration.
CUDA events on the ctx stream; 49.8 GB input >> L2.  Prints one JSON line.
usage: K1_CFGS=14,32 python tools/k1_ab.py [n_frames] [rounds]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 18000
    rounds = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    dev = torch.device("cuda:0")
    synth.build(device=True)
    stream = torch.cuda.Stream()
    cfgs = [int(c) for c in os.environ.get("K1_CFGS", "14").split(",")]
    ctxs = {}
    for c in cfgs:
        os.environ["CLIPDETECT_K1_CFG"] = str(c)
        ctxs[c] = Ctx(device=0, stream=stream)
    os.environ.pop("CLIPDETECT_K1_CFG", None)
    which = os.environ.get("K1_VIDEO", "c2")  # c2: the C2 video; c3: C3 video 0 (1080p, fades, flashes)
    base = manifest.c3_videos()[0] if which == "c3" else manifest.c2_video(0)
    v = manifest.subsample(base, n) if n < base.n else base
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    torch.cuda.synchronize()
    res = {c: [] for c in cfgs}
    ref = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    try:
        import pynvml
        pynvml.nvmlInit()
        nvh = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        clk = lambda: pynvml.nvmlDeviceGetClockInfo(nvh, pynvml.NVML_CLOCK_SM)  # noqa: E731
    except Exception:
        clk = lambda: None  # noqa: E731
    clocks = []
    for r in range(rounds):
        order = cfgs[r % len(cfgs):] + cfgs[:r % len(cfgs)]  # rotate: no fixed position in a round
        clocks.append(clk())
        for c in order:
            ctx = ctxs[c]
            with torch.cuda.stream(stream):
                ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)  # warm
                e0.record(stream)
                for _ in range(2):
                    ctx.frame_scores(frames, hist=hist, want_l1=False, want_score=False)
                e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 2
            res[c].append(frames.numel() / ms / 1e6)
            if ref is None:
                ref = hist.clone()
            elif not torch.equal(ref, hist):
                res[c].append(float("nan"))
    out = {f"cfg{c}": {"median_gbs": round(statistics.median(x), 1), "all": [round(y, 1) for y in x]}
           for c, x in res.items()}
    import hashlib
    sha = hashlib.sha256(ref.cpu().numpy().tobytes()).hexdigest()[:16]  # compare across library builds
    print(json.dumps({"video": which, "frames": v.n, "bytes": frames.numel(), "sm_mhz_per_round": clocks,
                      "lib": os.environ.get("CLIPDETECT_LIB", "default"), "hist_sha": sha, **out}))


if __name__ == "__main__":
    main()
