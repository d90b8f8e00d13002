#!/usr/bin/env python3
"""K1 micro-benchmark: the histogram kernel against the same TMA pipeline
without binning (K6 read roofline), on C2 content and on uniform-noise
frames.  CUDA events on the ctx stream; inputs >> L2.  Prints one JSON line."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx  # noqa: E402


def timeit(fn, stream, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


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
                    ("c2v1", manifest.subsample(manifest.c2_video(1), n)),
                    ("noise", manifest.noise_video(0, 1280, 720, n))]:
        table = torch_dev.frame_table(v, dev)
        frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
        torch_dev.gen_frames(v, table, frames)
        hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        nbytes = frames.numel()
        with torch.cuda.stream(stream):
            ms_k1 = timeit(lambda: ctx.frame_scores(frames, hist=hist, want_l1=False,
                                                    want_score=False), stream)
            ms_rd = timeit(lambda: ctx.debug_read_roofline(frames), stream)
        import hashlib
        out[name] = {"frames": v.n, "bytes": nbytes, "k1_ms": round(ms_k1, 3),
                     "k1_gbs": round(nbytes / ms_k1 / 1e6, 1), "read_ms": round(ms_rd, 3),
                     "read_gbs": round(nbytes / ms_rd / 1e6, 1),
                     "k1_frac_of_read": round(ms_rd / ms_k1, 3),
                     "hist_sha16": hashlib.sha256(hist.cpu().numpy().tobytes()).hexdigest()[:16]}
        del frames, hist
        torch.cuda.empty_cache()
    out["lib"] = libs[0] if libs else "product"
    print(json.dumps(out))


if __name__ == "__main__":
    main()
