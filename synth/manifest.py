"""Event manifests for the synthetic workloads C1..C5 (BASELINE.json ``configs``).

Part of the seeded input-generator module (``synth/``), which holds none of the
method's arithmetic.  A manifest fixes, per video, the resolution, the length
and per-frame records (scene id, palette rotation / flash mode, fade weight);
the pixels themselves come from ``synth.h`` (host: ``libsynth.so``, device:
``libsynthdev.so``).  The recipe is DESIGN.md "Input recipe" (SURVEY.md §8(d),
PROPOSED; the paper gives none — PAPER.md:35 only says clips are split on colour
changes and merged by embedding similarity).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

FRAME_DTYPE = np.dtype([("scene", "<u4"), ("mode", "<u2"), ("fade_w", "<u2")])
assert FRAME_DTYPE.itemsize == 8

MODE_NORMAL, MODE_ROT1, MODE_ROT2, MODE_FLASH, MODE_NOISE = 0, 1, 2, 3, 4
FADE_LEN = 24
MIN_SPACING = 10
L_MIN_DEFAULT = 8

CONFIG_SEEDS = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C5": 5}
EMB_DIM = 768


@dataclass
class Video:
    id: int
    W: int
    H: int
    n: int
    seed: int
    frames: np.ndarray  # FRAME_DTYPE [n]
    hard: list = field(default_factory=list)   # planted hard-cut frames
    false: list = field(default_factory=list)  # planted false cuts (palette rotation)
    flashes: list = field(default_factory=list)  # (start, length)
    fades: list = field(default_factory=list)  # fade centres (scene switch frame)

    @property
    def npix(self) -> int:
        return self.W * self.H

    @property
    def frame_bytes(self) -> int:
        return 3 * self.W * self.H


def _blank(n: int) -> np.ndarray:
    fr = np.zeros(n, dtype=FRAME_DTYPE)
    fr["fade_w"] = 256
    return fr


def c1_video() -> Video:
    """C1: one 64-frame 320x240 video, hard cuts at 10, 32, 53; false cut
    (palette rotation) at 21; 2-frame flash at 43-44."""
    n = 64
    fr = _blank(n)
    fr["scene"][0:10] = 0
    fr["scene"][10:32] = 1
    fr["scene"][32:53] = 2
    fr["scene"][53:64] = 3
    fr["mode"][21:32] = MODE_ROT1
    fr["mode"][43:45] = MODE_FLASH
    return Video(id=0, W=320, H=240, n=n, seed=CONFIG_SEEDS["C1"], frames=fr,
                 hard=[10, 32, 53], false=[21], flashes=[(43, 2)], fades=[])


def random_video(seed: int, vid: int, W: int, H: int, n: int, p_hard: float,
                 p_false: float, p_fade: float, flashes_per_min: float) -> Video:
    """Random shots: lengths 10 + Geometric(1/110) (mean 120 frames); each
    boundary hard / false / fade with the given probabilities; flashes of 1-3
    frames placed >= L_min frames from any boundary or fade."""
    rng = np.random.default_rng([seed, vid])
    bounds = []
    pos = 0
    while True:
        L = MIN_SPACING + int(rng.geometric(1.0 / 110.0))
        if pos + L >= n:
            break
        if n - (pos + L) < MIN_SPACING:  # tail shorter than 10 merges into the last shot
            break
        pos += L
        bounds.append(pos)
    fr = _blank(n)
    hard, false, fades = [], [], []
    busy = np.zeros(n, dtype=bool)  # frames covered by a fade
    scene, rot = 0, 0
    kinds = []
    for b in bounds:
        u = rng.random()
        if u < p_hard:
            kind = "hard"
        elif u < p_hard + p_false:
            kind = "false"
        else:
            kind = "fade"
        if kind == "fade":
            lo, hi = b - FADE_LEN // 2, b + FADE_LEN // 2
            if lo < 0 or hi > n or busy[max(0, lo - 2):min(n, hi + 2)].any():
                kind = "hard"
            else:
                busy[lo:hi] = True
        kinds.append(kind)
    # scene ids / rotations per shot
    edges = [0] + bounds + [n]
    for i in range(len(edges) - 1):
        if i > 0:
            k = kinds[i - 1]
            if k == "false":
                rot = (rot + 1) % 3
                false.append(edges[i])
            else:
                scene += 1
                rot = 0
                (hard if k == "hard" else fades).append(edges[i])
        fr["scene"][edges[i]:edges[i + 1]] = scene
        fr["mode"][edges[i]:edges[i + 1]] = rot
    for c in fades:
        for j in range(FADE_LEN):
            t = c - FADE_LEN // 2 + j
            fr["fade_w"][t] = (256 * abs(2 * j - FADE_LEN)) // FADE_LEN
    flashes = []
    if flashes_per_min > 0:
        count = int(rng.poisson(flashes_per_min * n / 1800.0))
        near = np.zeros(n, dtype=bool)
        for b in bounds:
            near[max(0, b - L_MIN_DEFAULT - FADE_LEN // 2):min(n, b + L_MIN_DEFAULT + FADE_LEN // 2)] = True
        for _ in range(count):
            for _try in range(20):
                length = int(rng.integers(1, 4))
                s = int(rng.integers(L_MIN_DEFAULT, max(L_MIN_DEFAULT + 1, n - L_MIN_DEFAULT - length)))
                if s + length > n or near[s:s + length].any():
                    continue
                fr["mode"][s:s + length] = MODE_FLASH
                near[max(0, s - L_MIN_DEFAULT):min(n, s + length + L_MIN_DEFAULT)] = True
                flashes.append((s, length))
                break
    flashes.sort()
    return Video(id=vid, W=W, H=H, n=n, seed=seed, frames=fr, hard=hard, false=false,
                 flashes=flashes, fades=fades)


def c2_video(vid: int = 0) -> Video:
    """C2: single 10-minute 720p 30 fps video (18,000 frames), ~93% hard cuts and
    ~7% false cuts.  ``vid`` > 0 gives further independent C2-shaped videos (the
    bench's per-rank weak-scaling unit)."""
    return random_video(CONFIG_SEEDS["C2"], vid, 1280, 720, 18000, 0.93, 0.07, 0.0, 0.0)


def c3_videos() -> list:
    """C3: 64 one-minute 1080p videos with fades and flashes."""
    return [random_video(CONFIG_SEEDS["C3"], v, 1920, 1080, 1800, 0.75, 0.10, 0.15, 3.0)
            for v in range(64)]


def c4_videos() -> list:
    """C4: 16 two-minute 4K videos."""
    return [random_video(CONFIG_SEEDS["C4"], v, 3840, 2160, 3600, 0.75, 0.10, 0.15, 3.0)
            for v in range(16)]


C5_RES = [(854, 480), (1280, 720), (1920, 1080)]


def c5_shapes() -> list:
    """C5 resolutions and lengths, drawn first from default_rng(5) in video order."""
    rng = np.random.default_rng(CONFIG_SEEDS["C5"])
    out = []
    for _ in range(1000):
        W, H = C5_RES[int(rng.integers(0, 3))]
        n = int(rng.integers(60, 901))
        out.append((W, H, n))
    return out


def c5_videos() -> list:
    """C5: 1000 mixed-resolution (480p-1080p) videos of 60-900 frames."""
    return [random_video(CONFIG_SEEDS["C5"], v, W, H, n, 0.75, 0.10, 0.15, 3.0)
            for v, (W, H, n) in enumerate(c5_shapes())]


def noise_video(vid: int, W: int = 1920, H: int = 1080, n: int = 256) -> Video:
    """Uniform-random-colour stress frames for K1 (worst-case bin spread)."""
    fr = _blank(n)
    fr["mode"][:] = MODE_NOISE
    fr["scene"][:] = np.arange(n) // 64
    return Video(id=vid, W=W, H=H, n=n, seed=99, frames=fr)


def config_videos(name: str) -> list:
    name = name.upper()
    if name == "C1":
        return [c1_video()]
    if name == "C2":
        return [c2_video(0)]
    if name == "C3":
        return c3_videos()
    if name == "C4":
        return c4_videos()
    if name == "C5":
        return c5_videos()
    raise ValueError(f"unknown config {name}")


def subsample(video: Video, n: int) -> Video:
    """First n frames of a video (same seed/id, so the same bytes)."""
    fr = video.frames[:n].copy()
    keep = lambda xs: [x for x in xs if x < n]
    return Video(id=video.id, W=video.W, H=video.H, n=n, seed=video.seed, frames=fr,
                 hard=keep(video.hard), false=keep(video.false),
                 flashes=[f for f in video.flashes if f[0] + f[1] <= n],
                 fades=[c for c in video.fades if c + FADE_LEN // 2 <= n])
