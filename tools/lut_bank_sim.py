#!/usr/bin/env python3
"""Shared-memory bank-conflict simulation of the hue-table (LUT) lookups of K1 and
K1-NV12 for the table swizzles of binfn.cuh (lut_swizzle), on C2 content and noise:
average wavefronts per warp-wide LDS.U8.  Run: PYTHONPATH=. python tools/lut_bank_sim.py
(NV12 -> RGB through OpenCV's COLOR_YUV2RGB_NV12, the conversion reading O0 names.)"""
import cv2
import numpy as np

import synth
from synth import manifest
v = manifest.subsample(manifest.c2_video(0), 40)
nv = synth.gen_nv12(v)[::8]     # 5 frames
rgbs = np.stack([cv2.cvtColor(f, cv2.COLOR_YUV2RGB_NV12) for f in nv]).astype(np.int32)
rgb_direct = synth.gen_frames(v)[::8].astype(np.int32)

def dn(rgb):
    mx = rgb.max(-1); mn = rgb.min(-1); mid = rgb.sum(-1) - mx - mn
    return mx - mn, mid - mn
def idx_of(d, na, swz):
    if swz == 'xor': return d * 256 + (na ^ d)
    if swz == 'none': return d * 256 + na
    if swz == 'xor4': return d * 256 + ((na ^ (d << 2)) & 255)
    if swz == 'add4': return d * 256 + ((na + 4 * d) & 255)
def wavefronts(idx):  # idx: [n_instr, 32] byte indices
    words = idx >> 2
    bank = words & 31
    tot = 0
    for w, b in zip(words, bank):
        # per bank: number of distinct words
        m = {}
        for ww, bb in zip(w, b):
            m.setdefault(bb, set()).add(ww)
        tot += max(len(s) for s in m.values())
    return tot / len(words)

H, W = 720, 1280
rng = np.random.default_rng(0)
# NV12 tile layout: warp-instruction = 32 consecutive units u, pair (k, r), half h
def nv12_instrs(rgb, swz, n=4000):
    d, na = dn(rgb)
    wu = W // 8
    out = []
    for _ in range(n):
        f = rng.integers(0, rgb.shape[0]); u0 = rng.integers(0, (H // 2) * wu - 32) // 32 * 32
        us = u0 + np.arange(32); br, cx = us // wu, us % wu
        k = rng.integers(0, 4); r = rng.integers(0, 2); h = rng.integers(0, 2)
        y = 2 * br + r; x = 8 * cx + 2 * k + h
        out.append(idx_of(d[f, y, x], na[f, y, x], swz))
    return np.array(out)
def rgb_instrs(rgb, swz, n=4000):
    d, na = dn(rgb)
    dflat, naflat = d.reshape(d.shape[0], -1), na.reshape(na.shape[0], -1)
    out = []
    for _ in range(n):
        f = rng.integers(0, rgb.shape[0]); q0 = rng.integers(0, H * W // 4 - 32)
        qs = q0 + np.arange(32); p = rng.integers(0, 2); h = rng.integers(0, 2)
        px = 4 * qs + 2 * p + h
        out.append(idx_of(dflat[f, px], naflat[f, px], swz))
    return np.array(out)
noise = rng.integers(0, 256, (2, H, W, 3)).astype(np.int32)
for swz in ['xor', 'none', 'xor4', 'add4']:
    print(swz, 'NV12-c2', round(wavefronts(nv12_instrs(rgbs, swz)), 2), 'RGB-c2', round(wavefronts(rgb_instrs(rgb_direct, swz)), 2),
          'RGB-noise', round(wavefronts(rgb_instrs(noise, swz)), 2))
def nv12_instrs4(rgb, swz, n=4000):
    d, na = dn(rgb)
    wu = W // 4
    out = []
    for _ in range(n):
        f = rng.integers(0, rgb.shape[0]); u0 = rng.integers(0, (H // 2) * wu - 32) // 32 * 32
        us = u0 + np.arange(32); br, cx = us // wu, us % wu
        k = rng.integers(0, 2); r = rng.integers(0, 2); h = rng.integers(0, 2)
        y = 2 * br + r; x = 4 * cx + 2 * k + h
        out.append(idx_of(d[f, y, x], na[f, y, x], swz))
    return np.array(out)
for swz in ['xor', 'xor4']:
    print('2x4 units', swz, 'NV12-c2', round(wavefronts(nv12_instrs4(rgbs, swz)), 2))
nz12 = rng.integers(0, 256, (2, H * 3 // 2, W), dtype=np.uint8)
nzrgb = np.stack([cv2.cvtColor(f, cv2.COLOR_YUV2RGB_NV12) for f in nz12]).astype(np.int32)
for swz in ['xor', 'xor4']:
    print('NV12-noise', swz, round(wavefronts(nv12_instrs(nzrgb, swz)), 2))
