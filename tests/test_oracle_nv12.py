"""Pins of the oracle's NV12 conversion (reading O0) and of the NV12 path.

O0 is the definition of OpenCV's COLOR_YUV2RGB_NV12 (BT.601 limited range,
20-bit fixed point), so the oracle is pinned (a) against that library routine
on every (Y, U, V), (b) against the textbook BT.601 real-valued equations
(R = 1.164 (Y-16) + 1.596 (V-128) ...) within one level, and (c) at anchors
(black, white, grey, primaries).  The NV12 histogram is pinned as O2 of the
converted frame, and the synthetic NV12 C1 video must reproduce its planted
cuts (the same ground truth as the RGB C1 video).
"""
import numpy as np
import pytest

import oracle
import synth
from synth import manifest

from nv12_helpers import all_yuv_image, random_nv12, yuv_rgb_table


@pytest.fixture(scope="module")
def rgb_all():
    return yuv_rgb_table()


def test_o0_matches_opencv_on_every_yuv():
    cv2 = pytest.importorskip("cv2")
    img, _ = all_yuv_image()
    got = oracle.nv12_to_rgb(img)
    want = cv2.cvtColor(img, cv2.COLOR_YUV2RGB_NV12)
    assert np.array_equal(got, want)


def test_o0_textbook_bt601_within_one_level(rgb_all):
    c = np.arange(1 << 24, dtype=np.int64)
    Y, U, V = (c >> 16).astype(np.float64), ((c >> 8) & 255).astype(np.float64), (c & 255).astype(np.float64)
    y = 1.164 * np.maximum(Y - 16, 0)
    ref = [y + 1.596 * (V - 128), y - 0.813 * (V - 128) - 0.391 * (U - 128), y + 2.018 * (U - 128)]
    for ch, r in enumerate(ref):
        got = (rgb_all >> (16 - 8 * ch)) & 255
        want = np.clip(np.round(r), 0, 255)
        assert np.abs(got - want).max() <= 1, ch


@pytest.mark.parametrize("yuv,rgb", [((16, 128, 128), (0, 0, 0)), ((235, 128, 128), (255, 255, 255)),
                                     ((0, 128, 128), (0, 0, 0)), ((255, 128, 128), (255, 255, 255)),
                                     ((126, 128, 128), (128, 128, 128)),
                                     ((81, 90, 240), (255, 0, 0)), ((41, 240, 110), (0, 0, 255))])
def test_o0_anchors(rgb_all, yuv, rgb):
    Y, U, V = yuv
    v = int(rgb_all[(Y << 16) | (U << 8) | V])
    got = (v >> 16, (v >> 8) & 255, v & 255)
    # anchors are the BT.601 studio-swing values; primaries land within 1 level
    assert all(abs(a - b) <= 1 for a, b in zip(got, rgb)), (yuv, got)


def test_o0_grey_axis_is_monotone_and_neutral(rgb_all):
    idx = (np.arange(256) << 16) | (128 << 8) | 128
    v = rgb_all[idx]
    r, g, b = v >> 16, (v >> 8) & 255, v & 255
    assert np.array_equal(r, g) and np.array_equal(g, b)
    assert np.all(np.diff(r) >= 0) and r[16] == 0 and r[235] == 255


def test_nv12_hist_is_o2_of_converted_frame():
    rng = np.random.default_rng(3)
    for H, W in [(8, 16), (36, 40), (64, 96)]:
        fr = random_nv12(rng, 3, H, W)
        rgb = np.stack([oracle.nv12_to_rgb(f) for f in fr])
        assert np.array_equal(oracle.hist_nv12_frames(fr), oracle.hist_frames(rgb))
        assert oracle.hist_nv12_frames(fr).sum(axis=1).tolist() == [H * W] * 3


def test_nv12_chroma_is_shared_by_the_2x2_block():
    # changing one UV sample changes exactly the four pixels of its block
    rng = np.random.default_rng(4)
    f = random_nv12(rng, 1, 8, 8)[0]
    a = oracle.nv12_to_rgb(f)
    g = f.copy()
    g[8 + 1, 2] ^= 0x55  # U of block (by=1, bx=1)
    b = oracle.nv12_to_rgb(g)
    diff = np.argwhere(np.any(a != b, axis=2))
    assert {tuple(x) for x in diff} <= {(2, 2), (2, 3), (3, 2), (3, 3)} and len(diff) > 0


def test_nv12_c1_planted_cuts():
    v = manifest.c1_video()
    fr = synth.gen_nv12(v)
    emb = synth.gen_emb(v)
    r = oracle.run_video_nv12(fr, emb)
    assert r.detected.tolist() == [10, 21, 32, 43, 53]
    assert r.final.tolist() == [10, 32, 53]
