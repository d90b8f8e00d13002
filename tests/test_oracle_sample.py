"""Pins of the frame-sampling / resize oracle (NEXT f3; readings O10, O11).

O11 is OpenCV's 8-bit INTER_LINEAR fixed point, so the oracle is pinned bit
for bit against cv2.resize on every workload resolution -> 224x224 and on
random downscales whose output rows OpenCV computes entirely in its vector
path (3*W2 % 16 == 0, where its scalar tail with a different rounding is never
used); plus closed forms: identity size, constant images, 2x2 means.  O10 is
pinned by brute force with exact rationals and its closed forms.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("W,H", [(854, 480), (1280, 720), (1920, 1080), (3840, 2160), (320, 240)])
def test_o11_matches_opencv_workload_resolutions(W, H):
    cv2 = pytest.importorskip("cv2")
    rng = np.random.default_rng(W + H)
    img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    assert np.array_equal(oracle.resize_linear(img, 224, 224),
                          cv2.resize(img, (224, 224), interpolation=cv2.INTER_LINEAR))


def test_o11_matches_opencv_random_downscales():
    cv2 = pytest.importorskip("cv2")
    rng = np.random.default_rng(7)
    for _ in range(40):
        W, H = int(rng.integers(232, 1500)), int(rng.integers(40, 900))
        W2 = int(rng.choice([16, 64, 112, 224]))
        H2 = int(rng.integers(8, min(H, 300)))
        img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        if rng.random() < 0.5:  # smooth content too
            img = np.repeat(np.repeat(img[::8, ::8], 8, 0), 8, 1)[:H, :W].copy()
            H, W = img.shape[:2]
        assert np.array_equal(oracle.resize_linear(img, H2, W2),
                              cv2.resize(img, (W2, H2), interpolation=cv2.INTER_LINEAR)), (W, H, W2, H2)


def test_o11_identity_constant_and_2x2_mean():
    rng = np.random.default_rng(8)
    img = rng.integers(0, 256, (48, 64, 3), dtype=np.uint8)
    assert np.array_equal(oracle.resize_linear(img, 48, 64), img)
    flat = np.full((90, 160, 3), (17, 200, 255), dtype=np.uint8)
    assert np.all(oracle.resize_linear(flat, 37, 53) == np.array([17, 200, 255], dtype=np.uint8))
    half = oracle.resize_linear(img, 24, 32).astype(np.int64)
    mean = img.reshape(24, 2, 32, 2, 3).astype(np.float64).mean(axis=(1, 3))
    assert np.abs(half - mean).max() <= 1


def test_o10_sampling_closed_forms_and_bruteforce():
    for s, e in [(0, 1), (5, 6), (0, 8), (10, 20), (3, 500), (100, 107)]:
        L = e - s
        for k in [1, 2, 3, 4, 8, 16]:
            t = [oracle.sample_index(s, e, i, k) for i in range(k)]
            assert t == [s + int(Fraction(2 * i + 1, 2 * k) * L) for i in range(k)]  # floor of midpoints
            assert all(s <= x < e for x in t) and t == sorted(t)
            assert all(t[i] - s + t[k - 1 - i] - s in (L - 1, L) for i in range(k))  # symmetric
            if k == L:
                assert t == list(range(s, e))
            if L == 1:
                assert t == [s] * k
            if k <= L:
                assert len(set(t)) == k  # distinct when the clip is long enough


def test_sample_clips_composes_o10_and_o11():
    rng = np.random.default_rng(9)
    frames = rng.integers(0, 256, (30, 36, 64, 3), dtype=np.uint8)
    cuts = [7, 15, 29]
    out, idx = oracle.sample_clips(frames, cuts, 3, 12, 16)
    bounds = [0] + cuts + [30]
    want = [oracle.sample_index(bounds[c], bounds[c + 1], i, 3) for c in range(4) for i in range(3)]
    assert idx.tolist() == want
    for j, t in enumerate(idx):
        assert np.array_equal(out[j], oracle.resize_linear(frames[t], 12, 16))
