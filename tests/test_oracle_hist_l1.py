"""Pins for oracle O2 (histogram) and O3 (adjacent-frame L1 / TV distance).

O2: hist_t[b] = #{pixels with bin b}, sum = N (reading O2).
O3: L1_t = sum_b |h_t[b] - h_{t-1}[b]|, score = L1 / 2N (total variation).
PAPER.md:35 (§2.1): "analyzing the color changes between frames".
Pins: hand-computed 4x4 frames, sum = N, invariance under any pixel
permutation, numpy.bincount of the (separately pinned) O1 table, brute-force
L1 by numpy, and the identities L1 = 2N - 2 sum min(h_t, h_{t-1}), L1 even,
symmetric, 0 for identical frames, 2N for disjoint supports.
"""
import numpy as np

import oracle

P = oracle.Params()
RED, BLUE = (255, 0, 0), (0, 0, 255)


def _frame(pixels, H=4, W=4):
    return np.array(pixels, dtype=np.uint8).reshape(H, W, 3)


def test_4x4_all_red():
    h = oracle.hist(_frame([RED] * 16))
    assert h[8] == 16 and h.sum() == 16


def test_4x4_half_red_half_blue():
    h = oracle.hist(_frame([RED] * 8 + [BLUE] * 8))
    assert h[8] == 8 and h[116] == 8 and h.sum() == 16


def test_4x4_distance_red_vs_half():
    a = _frame([RED] * 16)
    b = _frame([RED] * 8 + [BLUE] * 8)
    hs = np.stack([oracle.hist(a), oracle.hist(b)])
    l1, score = oracle.l1(hs, 16)
    assert l1[0] == 0 and l1[1] == 16
    assert score[1] == 0.5
    # tau = 0.30: 16 * 1e6 >= 300000 * 32  -> frame 1 is a candidate
    assert list(oracle.candidates(l1, 16)) == [1]


def test_sum_is_npix_and_permutation_invariant():
    rng = np.random.default_rng(3)
    f = rng.integers(0, 256, size=(37, 53, 3), dtype=np.uint8)
    h = oracle.hist(f)
    assert h.sum() == 37 * 53
    perm = rng.permutation(37 * 53)
    g = f.reshape(-1, 3)[perm].reshape(37, 53, 3)
    assert np.array_equal(oracle.hist(g), h)


def test_hist_equals_bincount_of_table():
    table = oracle.bin_table()
    rng = np.random.default_rng(4)
    frames = rng.integers(0, 256, size=(5, 24, 40, 3), dtype=np.uint8)
    hs = oracle.hist_frames(frames, nthreads=3)
    for t in range(5):
        px = frames[t].reshape(-1, 3).astype(np.int64)
        bins = table[(px[:, 0] << 16) | (px[:, 1] << 8) | px[:, 2]]
        assert np.array_equal(hs[t], np.bincount(bins, minlength=P.nbins).astype(np.uint32))


def test_threads_do_not_change_result():
    rng = np.random.default_rng(5)
    frames = rng.integers(0, 256, size=(9, 16, 16, 3), dtype=np.uint8)
    assert np.array_equal(oracle.hist_frames(frames, nthreads=1),
                          oracle.hist_frames(frames, nthreads=4))


def test_l1_brute_force_and_identities():
    rng = np.random.default_rng(6)
    N = 1000
    n = 40
    hs = np.stack([np.bincount(rng.integers(0, rng.integers(1, 162), size=N), minlength=162)
                   for _ in range(n)]).astype(np.uint32)
    l1, score = oracle.l1(hs, N)
    assert l1[0] == 0 and score[0] == 0.0
    for t in range(1, n):
        a, b = hs[t].astype(np.int64), hs[t - 1].astype(np.int64)
        want = np.abs(a - b).sum()
        assert l1[t] == want
        assert want == 2 * N - 2 * np.minimum(a, b).sum()
        assert want % 2 == 0
        assert score[t] == want / (2 * N)
    # symmetric: reversing the sequence gives the same distances
    l1r, _ = oracle.l1(np.ascontiguousarray(hs[::-1]), N)
    assert np.array_equal(l1r[1:], l1[1:][::-1])


def test_l1_identical_and_disjoint():
    a = np.zeros(162, np.uint32)
    a[3] = 10
    b = np.zeros(162, np.uint32)
    b[100] = 10
    l1, score = oracle.l1(np.stack([a, a, b]), 10)
    assert list(l1) == [0, 0, 20]
    assert score[2] == 1.0


def test_threshold_is_exact_integer_tie_cuts():
    # N = 10: tau_ppm * 2N = 300000 * 20 = 6e6 -> L1 >= 6 cuts, L1 = 5 (score 0.25) does not
    l1 = np.array([0, 6, 5, 4, 20], dtype=np.uint32)
    assert list(oracle.candidates(l1, 10)) == [1, 4]
    p = oracle.Params(tau_ppm=250000)  # 0.25 * 20 = 5 -> ties cut
    assert list(oracle.candidates(l1, 10, p)) == [1, 2, 4]
