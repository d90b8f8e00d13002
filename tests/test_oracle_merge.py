"""Pins for oracle O8 (clip embedding sums) and O9 (round-synchronous merge).

PAPER.md:35 (§2.1): the split "is smoothed out by computing the similarity
between image embeddings of adjacent clips to potentially merge them back
together".  Reading O9: remove every adjacent boundary with cosine
>= theta at once, recompute, repeat to a fixed point.  Pins: the worked
example (A = 4 u(0), B = u(20deg), C = u(-10deg), theta = 0.9: 1 clip after 2
rounds), the greedy counterexample, orthogonal clips -> nothing merges,
constant embeddings -> everything merges, idempotence, merged subset of
detected, fixed-point property and cosines against numpy.
"""
import math

import numpy as np

import oracle

P = oracle.Params()


def _emb_from_clips(vectors_per_frame, dim=768):
    e = np.zeros((len(vectors_per_frame), dim), dtype=np.float32)
    for i, v in enumerate(vectors_per_frame):
        e[i, :len(v)] = v
    return e


def _u(deg):
    return (math.cos(math.radians(deg)), math.sin(math.radians(deg)))


def test_worked_example_two_rounds():
    # frames: A = 4 frames of u(0), B = 1 frame of u(20), C = 1 frame of u(-10)
    frames = [_u(0)] * 4 + [_u(20)] + [_u(-10)]
    e = _emb_from_clips(frames)
    r = oracle.merge(e, [4, 5])
    # round 1: cos(A,B) = cos 20deg = 0.9397 >= 0.9 merges; cos(B,C) = cos 30deg = 0.866 does not
    assert abs(r.cos[0] - math.cos(math.radians(20))) < 1e-6
    # round 2: cos(A+B, C) = 0.9705 >= 0.9 merges -> one clip
    assert list(r.final) == []
    assert r.rounds == 2  # two evaluating rounds; the 2nd leaves one clip, so none is left to test
    assert abs(r.cos[1] - 0.9705) < 1e-3


def test_greedy_counterexample():
    # S = [(0.766, 1.086), (0.19, 0.088), (1.589, 1.803)], one frame per clip
    e = _emb_from_clips([(0.766, 1.086), (0.19, 0.088), (1.589, 1.803)])
    r = oracle.merge(e, [1, 2])
    assert list(r.final) == []  # round 1 merges clips 1+2, round 2 merges all
    r2 = oracle.merge(e, list(r.final))
    assert list(r2.final) == list(r.final)


def test_orthogonal_clips_never_merge():
    dim = 16
    frames = []
    cuts = []
    for k in range(6):
        v = np.zeros(dim)
        v[k] = 1.0
        frames += [v] * (3 + k)
        cuts.append(len(frames))
    cuts = cuts[:-1]
    e = np.array(frames, dtype=np.float32)
    r = oracle.merge(e, cuts)
    assert list(r.final) == cuts
    assert np.all(r.cos == 0.0)
    assert r.rounds == 1


def test_constant_embeddings_merge_all():
    e = np.ones((50, 32), dtype=np.float32)
    r = oracle.merge(e, [10, 20, 30, 40])
    assert list(r.final) == []


def test_zero_norm_gives_zero_cosine():
    e = np.zeros((20, 8), dtype=np.float32)
    e[10:] = 1.0
    r = oracle.merge(e, [10])
    assert r.cos[0] == 0.0 and list(r.final) == [10]


def _np_sum(e, a, b):
    return e[a:b].astype(np.float64).sum(axis=0)


def test_random_idempotent_subset_fixed_point_and_numpy_cosines():
    rng = np.random.default_rng(9)
    for trial in range(60):
        n = int(rng.integers(20, 200))
        dim = int(rng.integers(2, 40))
        k = int(rng.integers(0, 12))
        cuts = sorted(set(int(x) for x in rng.integers(1, n, size=k)))
        centres = rng.standard_normal((3, dim))
        # clustered directions so that some merges happen
        base = centres[rng.integers(0, 3, size=len(cuts) + 1)] + 0.3 * rng.standard_normal((len(cuts) + 1, dim))
        B = [0] + cuts + [n]
        e = np.zeros((n, dim), dtype=np.float32)
        for j in range(len(B) - 1):
            e[B[j]:B[j + 1]] = (base[j] + 0.05 * rng.standard_normal((B[j + 1] - B[j], dim))).astype(np.float32)
        r = oracle.merge(e, cuts)
        fin = list(r.final)
        assert set(fin) <= set(cuts)
        assert fin == sorted(fin)
        # fixed point: no remaining adjacent pair reaches theta (numpy cosines)
        F = [0] + fin + [n]
        for j in range(len(F) - 2):
            a, b = _np_sum(e, F[j], F[j + 1]), _np_sum(e, F[j + 1], F[j + 2])
            c = a @ b / (np.linalg.norm(a) * np.linalg.norm(b))
            assert c < P.theta
            assert abs(r.cos[cuts.index(F[j + 1])] - c) <= 1e-12
        # idempotent
        r2 = oracle.merge(e, fin)
        assert list(r2.final) == fin
        # first-round cosines equal numpy on the detected clips
        if cuts:
            r1 = oracle.merge(e, cuts, oracle.Params(max_rounds=1))
            for j in range(len(B) - 2):
                a, b = _np_sum(e, B[j], B[j + 1]), _np_sum(e, B[j + 1], B[j + 2])
                c = a @ b / (np.linalg.norm(a) * np.linalg.norm(b))
                assert abs(r1.cos[j] - c) <= 1e-12


def test_clip_sum_is_fp64_ascending():
    e = np.array([[1e8], [1.0], [-1e8], [1.0]], dtype=np.float32)
    # f64 accumulation keeps the 1.0 terms (f32 accumulation would not)
    assert oracle.clip_sum(e, 0, 4)[0] == 2.0
