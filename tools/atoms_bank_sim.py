#!/usr/bin/env python3
"""Shared-memory bank-conflict simulation of K1's code-histogram atomics
(ATOMS.POPC.INC: same-address lanes combine; distinct addresses in one bank
serialise) for the code layouts of binfn.cuh: the LUT layout (cfg14) and the
direct-offset layout with each table bank hash (lut_entry_dir).  Average
wavefronts per warp-wide atomic on C2 content and on uniform noise, for the
quad (4 px per lane) and octet (8 px per lane) lane layouts.
Run: PYTHONPATH=. python tools/atoms_bank_sim.py"""
import numpy as np

import synth
from synth import manifest

H, W = 720, 1280
rng = np.random.default_rng(0)
v = manifest.subsample(manifest.c2_video(0), 40)
c2 = synth.gen_frames(v)[::8].astype(np.int64)
noise = rng.integers(0, 256, (2, H, W, 3)).astype(np.int64)
DIRQ = {(0, 0): 0, (0, 3): 1, (0, 2): 2, (1, 2): 3, (1, 1): 4, (2, 1): 5, (2, 0): 6, (3, 0): 7}


def fields(rgb):
    r, g, b = rgb[..., 0], rgb[..., 1], rgb[..., 2]
    mx = rgb.max(-1); mn = rgb.min(-1); mid = rgb.sum(-1) - mx - mn
    d = mx - mn; na = mid - mn
    dd = np.maximum(d, 1)
    qr = np.where(d > 0, np.minimum(3, 3 * na // dd), 0)
    qf = np.where(d > 0, np.minimum(3, 3 * (d - na) // dd), 0)
    f = dict(A=(r >= g) * 1, B=(g >= b) * 1, C=(r >= b) * 1, qr=qr, qf=qf, v=(3 * mx) >> 8,
             s1=(3 * d >= mx) * 1, s2=(3 * d >= 2 * mx) * 1, d=d, na=na)
    q3 = np.zeros_like(d)
    for (a, bq), i in DIRQ.items():
        q3[(qr == a) & (qf == bq)] = i
    f["q3"] = q3
    return f


def index(f, layout):
    if layout == "lut":
        return (f["A"] | (f["qr"] | f["qf"] << 2) << 1 | f["v"] << 5 | f["s1"] << 7 | f["s2"] << 8
                | f["B"] << 9 | f["C"] << 12)
    h = {"dir-none": 0, "dir-d": f["d"] & 3, "dir-na": f["na"] & 3,
         "dir-dxna": (f["d"] ^ f["na"]) & 3, "dir-d6": f["d"] >> 6, "dir-d5": (f["d"] >> 5) & 3,
         "dir-d4": (f["d"] >> 4) & 3, "dir-d6xd": (f["d"] >> 6) ^ (f["d"] & 3),
         "dir-d5xna": ((f["d"] >> 5) ^ f["na"]) & 3}[layout]
    return (f["q3"] | h << 3 | f["v"] << 6 | f["s1"] << 8 | f["s2"] << 9 | f["A"] << 10
            | f["B"] << 11 | f["C"] << 12)


def wavefronts(idx_frames, ppl, n=3000):
    """ppl = pixels per lane (4 quads, 8 octets); one atomic = the same pixel of
    each lane's run across a warp's 32 consecutive runs."""
    flat = idx_frames.reshape(idx_frames.shape[0], -1)
    tot = 0
    for _ in range(n):
        fr = rng.integers(0, flat.shape[0])
        r0 = rng.integers(0, flat.shape[1] // ppl - 32)
        k = rng.integers(0, ppl)
        ids = flat[fr, (r0 + np.arange(32)) * ppl + k]
        banks = {}
        for a in np.unique(ids):
            banks[a & 31] = banks.get(a & 31, 0) + 1
        tot += max(banks.values())
    return tot / n


for name, frames in (("c2", c2), ("noise", noise)):
    f = fields(frames)
    for layout in ("lut", "dir-dxna", "dir-d6", "dir-d5", "dir-d4", "dir-d6xd", "dir-d5xna"):
        idx = index(f, layout)
        print(name, layout, "quad %.2f" % wavefronts(idx, 4), "octet %.2f" % wavefronts(idx, 8),
              "distinct/warp %.1f" % np.mean([len(np.unique(idx.reshape(idx.shape[0], -1)[0, s:s + 128:4]))
                                              for s in range(0, 100000, 997)]))
