#!/usr/bin/env python3
"""Write tests/golden/<CONFIG>.json from the CPU ORACLE (and the shared input
generator) only — no CUDA code is imported or executed here.

Per video: resolution, length, sha256 of the oracle's hist [n][nbins] u32 and
L1 [n] u32 arrays, candidate count, detected and final cuts, the cosine of
every detected boundary at its last evaluation, band hits, rounds, and the
synth frame hash of three sampled frames (proves the device generator fed the
same bytes).  Frames are generated and histogrammed chunk by chunk so that
C2-C5 (50 GB - 1.6 TB of frames) fit in host memory; the arithmetic is
oracle.hist_frames / l1 / candidates / min_length / merge, i.e. oracle_video's
steps in order.

With --nv12 the frames are the generator's NV12 surfaces and the histogram
is oracle.hist_nv12_frames (reading O0 then O2); written as <CONFIG>_NV12.json.

usage: python tools/make_goldens.py C1 [C2 ...] [--threads N] [--nv12]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import manifest  # noqa: E402

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def golden_video(v, p, threads, chunk_bytes=2 << 30, buf=None, nv12=False):
    n = v.n
    fb = v.npix * 3 // 2 if nv12 else v.frame_bytes
    chunk = max(1, min(n, chunk_bytes // fb))
    if buf is None or buf.size < chunk * fb:
        buf = np.empty(chunk * fb, dtype=np.uint8)
    hist = np.empty((n, p.nbins), dtype=np.uint32)
    fh = {}
    sample = sorted({0, n // 2, n - 1})
    for t0 in range(0, n, chunk):
        m = min(chunk, n - t0)
        if nv12:
            fr = buf[:m * fb].reshape(m, v.H * 3 // 2, v.W)
            synth.gen_nv12(v, t0=t0, n=m, nthreads=threads, out=fr)
            hist[t0:t0 + m] = oracle.hist_nv12_frames(fr, p, nthreads=threads)
        else:
            fr = buf[:m * fb].reshape(m, v.H, v.W, 3)
            synth.gen_frames(v, t0=t0, n=m, nthreads=threads, out=fr)
            hist[t0:t0 + m] = oracle.hist_frames(fr, p, nthreads=threads)
        for t in sample:
            if t0 <= t < t0 + m:
                fh[str(t)] = str(synth.frame_hash(fr[t - t0]))
    l1, _ = oracle.l1(hist, v.npix)
    cand = oracle.candidates(l1, v.npix, p)
    det = oracle.min_length(cand, n, p.l_min)
    emb = synth.gen_emb(v, manifest.EMB_DIM)
    mr = oracle.merge(emb, det, p)
    rec = {
        "id": v.id, "W": v.W, "H": v.H, "n": n, "seed": v.seed,
        "hist_sha256": hashlib.sha256(hist.tobytes()).hexdigest(),
        "l1_sha256": hashlib.sha256(l1.tobytes()).hexdigest(),
        "n_candidates": int(cand.size),
        "detected": [int(x) for x in det],
        "final": [int(x) for x in mr.final],
        "cos": [float(x) for x in mr.cos],
        "n_band_hits": mr.n_band_hits,
        "rounds": mr.rounds,
        "frame_hash": fh,
        "planted_hard": [int(x) for x in v.hard],
        "planted_false": [int(x) for x in v.false],
    }
    return rec, buf


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
    ap.add_argument("--nv12", action="store_true")
    args = ap.parse_args()
    oracle.build()
    synth.build(device=False)
    p = oracle.Params()
    for name in args.configs:
        t0 = time.time()
        vids = manifest.config_videos(name)
        out = {"config": name, "format": "nv12" if args.nv12 else "rgb24", "params": p.__dict__, "emb_dim": manifest.EMB_DIM,
               "generator": "synth/synth.h + synth/manifest.py", "videos": []}
        buf = None
        for i, v in enumerate(vids):
            rec, buf = golden_video(v, p, args.threads, buf=buf, nv12=args.nv12)
            out["videos"].append(rec)
            if (i + 1) % max(1, len(vids) // 10) == 0:
                print(f"{name}: {i + 1}/{len(vids)} videos, {time.time() - t0:.0f}s", flush=True)
        out["total_frames"] = int(sum(v.n for v in vids))
        out["seconds"] = round(time.time() - t0, 1)
        path = os.path.join(GOLDEN_DIR, f"{name}_NV12.json" if args.nv12 else f"{name}.json")
        with open(path, "w") as f:
            json.dump(out, f, indent=0, separators=(",", ":"))
        print(f"wrote {path} in {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    main()
