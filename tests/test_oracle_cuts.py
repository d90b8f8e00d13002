"""Pins for oracle O5 (greedy minimum clip length) and O6 (tail rule).

Readings O5/O6 of DESIGN.md (PAPER.md:35 calls the split "aggressive"; the
minimum clip length is paper-silent).  Pins: the closed form for "every frame
is a candidate" (cuts exactly {L, 2L, ..., (floor(n/L)-1) L}), constant video
-> no cuts, n < 2L -> no cuts, and invariants on random candidate sets
(strictly increasing, gaps >= L, clips partition [0, n), cuts subset of
candidates, greedy maximality: every rejected candidate is closer than L to the
accepted cut before it).
"""
import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("n", list(range(1, 200, 7)) + [199])
@pytest.mark.parametrize("L", [1, 2, 3, 5, 8, 13, 19])
def test_all_candidates_closed_form(n, L):
    cand = np.arange(1, n, dtype=np.int64)
    cuts = list(oracle.min_length(cand, n, L))
    want = [k * L for k in range(1, n // L)]
    assert cuts == want


def test_no_candidates_and_short_videos():
    assert oracle.min_length(np.array([], np.int64), 100, 8).size == 0
    for n in range(1, 16):  # n < 2L -> no clip split is possible
        assert oracle.min_length(np.arange(1, n, dtype=np.int64), n, 8).size == 0


def _check_invariants(cand, n, L, cuts):
    cuts = list(cuts)
    cset = set(int(c) for c in cand)
    assert all(c in cset for c in cuts)
    assert all(b > a for a, b in zip(cuts, cuts[1:]))
    B = [0] + cuts + [n]
    assert all(b - a >= L for a, b in zip(B, B[1:])) or not cuts
    # greedy maximality up to the tail drop
    last, acc = 0, []
    for t in sorted(cset):
        if t - last >= L:
            acc.append(t)
            last = t
    if acc and n - acc[-1] < L:
        assert cuts == acc[:-1]
    else:
        assert cuts == acc


def test_random_candidate_sets():
    rng = np.random.default_rng(8)
    for _ in range(400):
        n = int(rng.integers(1, 300))
        L = int(rng.integers(1, 20))
        k = int(rng.integers(0, max(1, n)))
        cand = np.unique(rng.integers(1, max(2, n), size=k)).astype(np.int64)
        cand = cand[cand < n]
        cuts = oracle.min_length(cand, n, L)
        _check_invariants(cand, n, L, cuts)


def test_tail_drop_single():
    # candidates 8, 16 in n=20: 16 leaves a 4-frame tail -> dropped
    assert list(oracle.min_length(np.array([8, 16], np.int64), 20, 8)) == [8]
    assert list(oracle.min_length(np.array([8, 16], np.int64), 24, 8)) == [8, 16]
