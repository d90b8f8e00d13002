"""Pins of the f4 variants (NEXT f4; readings O3', O4''): histogram distances
against OpenCV's compareHist (a library routine computing the same textbook
definitions) and closed forms; the adaptive threshold by brute force with
exact rationals; the composed variant path on C1's planted truth."""
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from synth import manifest


def _pairs(rng, n=60, nbins=162, npix=921600):
    for _ in range(n):
        a = rng.multinomial(npix, rng.dirichlet(np.full(nbins, rng.uniform(0.05, 3)))).astype(np.uint32)
        if rng.random() < 0.3:
            b = a.copy()
            idx = rng.integers(0, nbins, 5)
            for i in idx:
                mv = min(int(b[i]), int(rng.integers(0, 2000)))
                b[i] -= mv
                b[(i + 1) % nbins] += mv
        else:
            b = rng.multinomial(npix, rng.dirichlet(np.full(nbins, rng.uniform(0.05, 3)))).astype(np.uint32)
        yield a, b, npix


def test_distances_match_opencv_comparehist():
    cv2 = pytest.importorskip("cv2")
    rng = np.random.default_rng(1)
    for a, b, N in _pairs(rng):
        fa, fb = a.astype(np.float32), b.astype(np.float32)
        chi = cv2.compareHist(fa, fb, cv2.HISTCMP_CHISQR_ALT) / (4.0 * N)
        bha = cv2.compareHist(fa, fb, cv2.HISTCMP_BHATTACHARYYA)
        cor = 1.0 - cv2.compareHist(fa, fb, cv2.HISTCMP_CORREL)
        assert oracle.distance(a, b, N, 1) == pytest.approx(chi, rel=1e-9, abs=1e-12)
        assert oracle.distance(a, b, N, 2) == pytest.approx(bha, rel=1e-6, abs=1e-6)
        assert oracle.distance(a, b, N, 3) == pytest.approx(cor, rel=1e-9, abs=1e-12)


def test_distance_closed_forms():
    N = 1000
    a = np.zeros(162, np.uint32)
    a[3] = N
    b = np.zeros(162, np.uint32)
    b[100] = N
    for k in (1, 2, 3):
        assert oracle.distance(a, a, N, k) == 0.0
    assert oracle.distance(a, b, N, 1) == 1.0 and oracle.distance(a, b, N, 2) == 1.0
    # two spikes: r = (162*0 - N^2) / (162 N^2 - N^2) = -1/161
    assert oracle.distance(a, b, N, 3) == pytest.approx(1 + 1 / 161, rel=1e-15)
    # chi-square of a half/half split vs a spike: bins (N/2 vs N) and (N/2 vs 0)
    c = np.zeros(162, np.uint32)
    c[3], c[4] = N // 2, N // 2
    want = (Fraction(N // 2) ** 2 / Fraction(3 * N // 2) + Fraction(N // 2)) / (2 * N)
    assert oracle.distance(a, c, N, 1) == pytest.approx(float(want), rel=1e-15)
    # symmetric
    rng = np.random.default_rng(2)
    for x, y, n in list(_pairs(rng, 10)):
        for k in (1, 2, 3):
            assert oracle.distance(x, y, n, k) == pytest.approx(oracle.distance(y, x, n, k), rel=1e-12, abs=1e-15)


def _adaptive_brute(l1, npix, tau_ppm, w, ratio_ppm):
    n = len(l1)
    out = []
    for t in range(1, n):
        nb = [u for u in range(t - w, t + w + 1) if 1 <= u <= n - 1 and u != t]
        if not nb:
            continue
        mean = Fraction(sum(int(l1[u]) for u in nb), len(nb))
        if Fraction(int(l1[t])) >= Fraction(ratio_ppm, 10 ** 6) * mean and \
                Fraction(int(l1[t]), 2 * npix) >= Fraction(tau_ppm, 10 ** 6):
            out.append(t)
    return out


def test_adaptive_bruteforce_and_closed_forms():
    rng = np.random.default_rng(3)
    npix = 1000
    for _ in range(80):
        n = int(rng.integers(1, 120))
        l1 = rng.integers(0, 2 * npix + 1, n).astype(np.uint32)
        if rng.random() < 0.5:
            l1 = (l1 // 40).astype(np.uint32)
            l1[rng.integers(0, n, max(1, n // 10))] = 2 * npix  # spikes
        w, ratio, tau = int(rng.integers(1, 5)), int(rng.choice([1000000, 2000000, 3000000])), int(rng.choice([0, 50000, 300000]))
        got = oracle.candidates_adaptive(l1, npix, w, ratio, oracle.Params(tau_ppm=tau)).tolist()
        assert got == _adaptive_brute(l1, npix, tau, w, ratio)
    # constant scores: ratio 1 -> every frame with a neighbour; ratio > 1 -> none
    c = np.full(50, 700, np.uint32)
    assert oracle.candidates_adaptive(c, npix, 2, 1000000, oracle.Params(tau_ppm=0)).tolist() == list(range(1, 50))
    assert oracle.candidates_adaptive(c, npix, 2, 1000001, oracle.Params(tau_ppm=0)).size == 0
    # an isolated spike in a flat sequence is the only candidate
    s = np.full(50, 10, np.uint32)
    s[20] = 900
    assert oracle.candidates_adaptive(s, npix, 2, 3000000, oracle.Params(tau_ppm=0)).tolist() == [20]


def test_variant_paths_find_c1_planted_cuts():
    v = manifest.c1_video()
    fr, emb = synth.gen_frames(v), synth.gen_emb(v)
    p = oracle.Params(tau_ppm=300000)
    for kind, tau in [(oracle.DIST_CHI2, 200000), (oracle.DIST_BHATTACHARYYA, 400000),
                      (oracle.DIST_CORREL, 500000)]:
        r = oracle.run_video_variant(fr, emb, oracle.Params(tau_ppm=tau), distance_kind=kind)
        assert r.final.tolist() == [10, 32, 53], kind
    r = oracle.run_video_variant(fr, emb, oracle.Params(tau_ppm=100000), adaptive_window=2,
                                 adaptive_ratio_ppm=3000000)
    assert r.final.tolist() == [10, 32, 53]
    # the default path through the variant composer is the default path
    r0 = oracle.run_video_variant(fr, emb, p)
    r1 = oracle.run_video(fr, emb, p)
    assert r0.detected.tolist() == r1.detected.tolist() and r0.final.tolist() == r1.final.tolist()


def test_keyframe_stride_merge():
    """O8': only every sigma-th frame of each detected clip enters the clip sums."""
    rng = np.random.default_rng(4)
    n, D = 60, 16
    emb = rng.standard_normal((n, D)).astype(np.float32)
    cuts = [11, 25, 40]
    p = oracle.Params(theta=0.0)  # merge everything with cos >= 0 ... decisions below use the sums
    # stride 1 is the plain merge
    a, b = oracle.merge(emb, cuts, p, stride=1), oracle.merge(emb, cuts, p)
    assert a.final.tolist() == b.final.tolist() and np.array_equal(a.cos, b.cos)
    # non-keyframes are never read: NaN there changes nothing
    for sigma in (2, 3, 7, 100):
        key = np.zeros(n, bool)
        for s0, s1 in zip([0] + cuts, cuts + [n]):
            key[s0:s1:sigma] = True
        poisoned = emb.copy()
        poisoned[~key] = np.nan
        r1 = oracle.merge(emb, cuts, oracle.Params(), stride=sigma)
        r2 = oracle.merge(poisoned, cuts, oracle.Params(), stride=sigma)
        assert r1.final.tolist() == r2.final.tolist() and np.array_equal(r1.cos, r2.cos)
        # first-round cosines are those of the keyframe sums (numpy, exact f64 sums of f32)
        bounds = [0] + cuts + [n]
        S = [emb[s0:s1][key[s0:s1]].astype(np.float64).sum(axis=0) for s0, s1 in zip(bounds[:-1], bounds[1:])]
        c0 = [float(np.dot(S[k], S[k + 1]) / np.linalg.norm(S[k]) / np.linalg.norm(S[k + 1])) for k in range(3)]
        r3 = oracle.merge(emb, cuts, oracle.Params(theta=2.0), stride=sigma)  # nothing merges: one round
        assert r3.rounds == 1
        np.testing.assert_allclose(r3.cos, c0, rtol=1e-12)
