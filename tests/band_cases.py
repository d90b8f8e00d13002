"""Planted merge inputs whose adjacent-clip cosines sit at chosen places
relative to the band |c - theta| <= band_rel * theta (north star: "any
threshold decision made within that band must be reported"; merge passage
PAPER.md:35 §2.1; reading O9 in DESIGN.md §2).

Every clip embedding is an INTEGER vector (exact in f32 and in the f64 sums),
so each cosine is dot / sqrt(|a|^2 |b|^2) of integers: the exact value is
checked here with 50-digit Decimal arithmetic and every planted cosine keeps
>= 3e-7 from each band edge, ~1e9 times the f64 rounding of either side.
The integer pairs (x, y) were found by a brute-force search for
x / sqrt(x^2 + y^2) near the target (cos of the angle between (1, 0) and
(x, y)).  No value here comes from the CUDA path or from the oracle.

Input generation only: no method arithmetic (tests/ and the GPU tests share it).
"""
from __future__ import annotations

from decimal import Decimal, getcontext

import numpy as np

getcontext().prec = 50

# (x, y) with cos((1,0), (x,y)) = x / sqrt(x^2 + y^2)
PAIRS = {
    "in_below": (1181, 572),      # 0.89999534  theta=0.9: |c-theta| = 4.66e-6 <= 9e-6, c < theta
    "in_above": (956, 463),       # 0.90000441  in band and c >= theta (merges)
    "out_above": (1369, 663),     # 0.90000953  9.53e-6 > 9e-6 (outside); <= 1e-5 (inside if *theta dropped)
    "out_below": (607, 294),      # 0.89999041  9.59e-6: outside; inside a band without *theta
    "half_out": (709, 1228),      # 0.50000734  theta=0.5: 7.34e-6 > 5e-6; <= 1e-5 without *theta
    "half_in": (892, 1545),       # 0.49999741  theta=0.5: 2.59e-6 <= 5e-6
}


def exact_cos(a, b) -> Decimal:
    """Exact (50-digit) cosine of two integer vectors."""
    dot = sum(int(x) * int(y) for x, y in zip(a, b))
    na = sum(int(x) * int(x) for x in a)
    nb = sum(int(y) * int(y) for y in b)
    return Decimal(dot) / (Decimal(na) * Decimal(nb)).sqrt()


def in_band(c: Decimal, theta: float, band_rel: float) -> bool:
    th = Decimal(theta)
    return abs(c - th) <= Decimal(band_rel) * th


def clips_to_emb(clips, frames_per_clip=None, dim: int = 16):
    """One integer vector per clip, repeated over its frames -> (emb f32 [n][dim], cuts)."""
    frames_per_clip = frames_per_clip or [1] * len(clips)
    n = sum(frames_per_clip)
    e = np.zeros((n, dim), dtype=np.float32)
    cuts, f = [], 0
    for v, m in zip(clips, frames_per_clip):
        for j in range(m):
            e[f + j, :len(v)] = v
        f += m
        cuts.append(f)
    return e, cuts[:-1]


def scale(v, k):
    return [k * x for x in v]


def case_two_rounds():
    """A | B | C | D, one frame each.  cos(A,B) in band below theta (not merged),
    cos(B,C) = 0, cos(C,D) = 5/sqrt(26) = 0.98 (merges in round 1).  Round 2
    re-evaluates A|B (same sums -> the same in-band cosine: a second hit) and
    B|CD (0): nothing merges.  Exact: final = [1, 2], rounds = 2, hits = 2."""
    x, y = PAIRS["in_below"]
    clips = [[1, 0, 0, 0], [x, y, 0, 0], [0, 0, 1, 0], [0, 0, 5, 1]]
    return clips_to_emb(clips)


def case_hit_that_merges():
    """A | B | C: cos(A,B) in band ABOVE theta (a hit that merges), cos(B,C) = 0.
    Round 1: 1 hit, merge A+B.  Round 2: cos(A+B, C) = 0, no hit, stop."""
    x, y = PAIRS["in_above"]
    clips = [[1, 0, 0], [x, y, 0], [0, 0, 1]]
    return clips_to_emb(clips)


def case_edges():
    """Eight clips a0 b0 a1 b1 a2 b2 a3 b3 (cuts 1..7); pair i lives in its own
    two dimensions, so b_i | a_{i+1} is orthogonal (cosine 0).  Planted
    (theta 0.9): cut 1 out_above, cut 3 out_below, cut 5 in_below, cut 7
    in_above.  Round 1: hits at cuts 5 and 7; cuts 1 and 7 merge (their
    cosines are >= theta).  Round 2: cuts 3 and 5 keep their cosines (sums
    unchanged): one more hit at cut 5; cuts 2 and 6 now face merged clips,
    still orthogonal; nothing merges.  Exact: final = [2..6], hits = 3,
    rounds = 2."""
    names = ["out_above", "out_below", "in_below", "in_above"]
    dim = 2 * len(names)
    clips = []
    for i, nm in enumerate(names):
        x, y = PAIRS[nm]
        a = [0] * dim
        b = [0] * dim
        a[2 * i] = 1
        b[2 * i], b[2 * i + 1] = x, y
        clips += [a, b]
    return clips_to_emb(clips, dim=dim)
