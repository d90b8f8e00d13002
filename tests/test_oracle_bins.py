"""Pins for oracle O1 (pixel -> HSV bin), independent of the oracle's code.

O1 is reading "exact integer hexcone HSV, floor bins" of DESIGN.md (the paper,
PAPER.md:35 §2.1, only says clips are split by "analyzing the color changes
between frames").  Pins:
  * named colours hand-computed from the textbook hue angle (tests/golden/named_colours.txt);
  * the library routine ``colorsys.rgb_to_hsv`` (float64) agrees with the
    oracle on every one of the 2^24 colours except where float rounding
    lands on the wrong side of an exact bin edge, and there the oracle equals
    the floor of the EXACT rational HSV (``fractions.Fraction``);
  * rotating channels (r,g,b) -> (b,r,g) turns the hue by exactly +120 deg, so
    the hue bin moves by nh/3 and s, v stay (a geometric invariant).
"""
import colorsys
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "named_colours.txt")
P = oracle.Params()


def _named():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            r, g, b, k = (int(x) for x in s.split()[:4])
            rows.append((r, g, b, k))
    return rows


def test_named_colours():
    rows = _named()
    assert len(rows) >= 15
    for r, g, b, k in rows:
        assert oracle.pixel_bin(r, g, b) == k, (r, g, b)


def _colorsys_vec(r, g, b):
    """numpy transcription of colorsys.rgb_to_hsv (same float64 operation
    order); verified equal to colorsys itself in test_colorsys_vec_matches."""
    r = r.astype(np.float64)
    g = g.astype(np.float64)
    b = b.astype(np.float64)
    maxc = np.maximum(np.maximum(r, g), b)
    minc = np.minimum(np.minimum(r, g), b)
    rangec = maxc - minc
    grey = minc == maxc
    safe = np.where(grey, 1.0, rangec)
    safe_max = np.where(maxc == 0, 1.0, maxc)
    s = np.where(grey, 0.0, rangec / safe_max)
    rc = (maxc - r) / safe
    gc = (maxc - g) / safe
    bc = (maxc - b) / safe
    h = np.where(r == maxc, bc - gc, np.where(g == maxc, 2.0 + rc - bc, 4.0 + gc - rc))
    h = np.mod(h / 6.0, 1.0)
    h = np.where(grey, 0.0, h)
    return h, s, maxc


def _float_bins(r, g, b):
    h, s, v = _colorsys_vec(r, g, b)
    hb = np.minimum(np.floor(h * P.nh), P.nh - 1).astype(np.int64)
    sb = np.minimum(np.floor(s * P.ns), P.ns - 1).astype(np.int64)
    vb = np.floor(v * P.nv / 256.0).astype(np.int64)
    return (hb * P.ns + sb) * P.nv + vb


def test_colorsys_vec_matches():
    rng = np.random.default_rng(7)
    c = rng.integers(0, 256, size=(20000, 3))
    h, s, v = _colorsys_vec(c[:, 0], c[:, 1], c[:, 2])
    for i in range(c.shape[0]):
        H, S, V = colorsys.rgb_to_hsv(int(c[i, 0]), int(c[i, 1]), int(c[i, 2]))
        assert (H, S, V) == (h[i], s[i], v[i])


def _exact_bin(r, g, b):
    """Floor of the exact rational textbook HSV (colorsys structure, Fractions)."""
    mx, mn = max(r, g, b), min(r, g, b)
    if mx == mn:
        H, S = Fraction(0), Fraction(0)
    else:
        rng_ = Fraction(mx - mn)
        S = rng_ / mx
        rc, gc, bc = (mx - r) / rng_, (mx - g) / rng_, (mx - b) / rng_
        if r == mx:
            H = bc - gc
        elif g == mx:
            H = 2 + rc - bc
        else:
            H = 4 + gc - rc
        H = (H / 6) % 1
    hb = min(int(H * P.nh), P.nh - 1)  # H*nh >= 0: int() is floor
    sb = min(int(S * P.ns), P.ns - 1)
    vb = (mx * P.nv) // 256
    return (hb * P.ns + sb) * P.nv + vb, H * P.nh, S * P.ns


def test_all_colours_vs_colorsys_and_exact():
    table = oracle.bin_table()
    idx = np.arange(1 << 24, dtype=np.int64)
    r, g, b = idx >> 16, (idx >> 8) & 255, idx & 255
    fb = _float_bins(r, g, b)
    mism = np.nonzero(fb != table.astype(np.int64))[0]
    # float rounding only ever goes wrong ON an exact edge (a few % of colours at most)
    assert 0 < mism.size < 200000
    for i in mism:
        ri, gi, bi = int(r[i]), int(g[i]), int(b[i])
        exact, h18, s3 = _exact_bin(ri, gi, bi)
        on_edge = (h18.denominator == 1) or (s3.denominator == 1)
        assert on_edge, (ri, gi, bi)
        assert int(table[i]) == exact, (ri, gi, bi)


def test_exact_on_random_sample():
    table = oracle.bin_table()
    rng = np.random.default_rng(11)
    for c in rng.integers(0, 256, size=(5000, 3)):
        r, g, b = (int(x) for x in c)
        assert table[(r << 16) | (g << 8) | b] == _exact_bin(r, g, b)[0]


def test_rotation_turns_hue_by_120_degrees():
    table = oracle.bin_table().astype(np.int64)
    idx = np.arange(1 << 24, dtype=np.int64)
    r, g, b = idx >> 16, (idx >> 8) & 255, idx & 255
    rot = (b << 16) | (r << 8) | g  # (r,g,b) -> (b,r,g): red -> green
    h, sv = table // (P.ns * P.nv), table % (P.ns * P.nv)
    h2, sv2 = table[rot] // (P.ns * P.nv), table[rot] % (P.ns * P.nv)
    grey = (r == g) & (g == b)
    assert np.array_equal(sv, sv2)
    assert np.array_equal(h2[~grey], (h[~grey] + P.nh // 3) % P.nh)
    assert np.all(h[grey] == 0)


def test_value_depends_on_max_only_and_bins_in_range():
    table = oracle.bin_table().astype(np.int64)
    assert table.max() < P.nbins
    assert len(np.unique(table)) == P.nbins  # every bin is reachable
    idx = np.arange(1 << 24, dtype=np.int64)
    mx = np.maximum(np.maximum(idx >> 16, (idx >> 8) & 255), idx & 255)
    assert np.array_equal(table % P.nv, (mx * P.nv) // 256)


@pytest.mark.parametrize("bins", [(12, 4, 4), (6, 2, 2), (18, 3, 3), (36, 4, 4)])
def test_other_bin_layouts_against_exact(bins):
    p = oracle.Params(nh=bins[0], ns=bins[1], nv=bins[2])
    rng = np.random.default_rng(sum(bins))
    for c in rng.integers(0, 256, size=(3000, 3)):
        r, g, b = (int(x) for x in c)
        mx, mn = max(r, g, b), min(r, g, b)
        if mx == mn:
            H, S = Fraction(0), Fraction(0)
        else:
            H = Fraction(colorsys.rgb_to_hsv(r, g, b)[0]).limit_denominator(10 ** 6)
            S = Fraction(mx - mn, mx)
        hb = min(int(H * p.nh), p.nh - 1)
        sb = min(int(S * p.ns), p.ns - 1)
        vb = (mx * p.nv) // 256
        want = (hb * p.ns + sb) * p.nv + vb
        got = oracle.pixel_bin(r, g, b, p)
        if got != want:  # only allowed exactly on a hue edge (float H recovered approximately)
            assert (H * p.nh).denominator == 1 or abs(float(H * p.nh) - round(float(H * p.nh))) < 1e-6
