"""Pins for the oracle's band-hit count (oracle/oracle.c oracle_merge_stride:
`fabs(c - theta) <= band_rel * theta`, counted at every evaluation of every
round).

North star: "Scores and cosines agree to within 1e-5 relative, and any
threshold decision made within that band must be reported"; merge passage
PAPER.md:35 (§2.1); reading O9.  The planted inputs
(tests/band_cases.py) are integer vectors whose exact cosines are known to 50
digits, so every expected count below is derived by hand from the exact
values, not from the oracle.  Each plausible mistake fails at least one test:
  * `* theta` dropped (band = band_rel absolute)  -> test_band_edges, test_band_scales_with_theta
  * `<` instead of `<=`                           -> test_band_edge_is_inclusive
  * only the last (or first) round counted        -> test_band_edges, test_two_rounds_recount
  * hits counted only for merged / unmerged pairs -> test_hit_that_merges, test_two_rounds_recount
"""
from decimal import Decimal

import numpy as np
import pytest

import oracle
from band_cases import PAIRS, case_edges, case_hit_that_merges, case_two_rounds, exact_cos, in_band


@pytest.mark.parametrize("name,theta,inside", [
    ("in_below", 0.9, True), ("in_above", 0.9, True), ("out_above", 0.9, False),
    ("out_below", 0.9, False), ("half_out", 0.5, False), ("half_in", 0.5, True)])
def test_planted_cosines_exact(name, theta, inside):
    """The fixtures themselves: exact cosine on the stated side of the band
    (band_rel 1e-5), >= 3e-7 from both edges of the true band and of the
    mutated absolute band |c - theta| <= 1e-5."""
    c = exact_cos((1, 0), PAIRS[name])
    th = Decimal(theta)
    assert in_band(c, theta, 1e-5) == inside
    for edge in (Decimal("1e-5") * th, Decimal("1e-5")):
        assert abs(abs(c - th) - edge) > Decimal("3e-7")
    if name in ("out_above", "out_below", "half_out"):
        assert abs(c - th) <= Decimal("1e-5")  # inside the band a dropped "* theta" would use


def test_band_edges():
    e, cuts = case_edges()
    assert cuts == [1, 2, 3, 4, 5, 6, 7]
    r = oracle.merge(e, cuts)
    assert list(r.final) == [2, 3, 4, 5, 6]  # out_above (c > theta) and in_above merge
    assert r.rounds == 2
    assert r.n_band_hits == 3  # cut 5 in rounds 1 and 2, cut 7 in round 1
    # cosines recorded at the round each boundary was last evaluated: exact values
    for cut, nm in [(1, "out_above"), (3, "out_below"), (5, "in_below"), (7, "in_above")]:
        assert abs(r.cos[cut - 1] - float(exact_cos((1, 0), PAIRS[nm]))) < 1e-14
    for cut in (2, 4, 6):
        assert r.cos[cut - 1] == 0.0
    # the mutated absolute band would count cuts 1, 3, 5, 7 in round 1 and 3, 5 in round 2
    assert sum(in_band(exact_cos((1, 0), PAIRS[nm]), 0.9, 1e-5 / 0.9)
               for nm in ["out_above", "out_below", "in_below", "in_above"]) == 4


def test_two_rounds_recount():
    e, cuts = case_two_rounds()
    r = oracle.merge(e, cuts)
    assert list(r.final) == [1, 2] and r.rounds == 2
    assert r.n_band_hits == 2  # the unmerged in-band boundary, once per round


def test_hit_that_merges():
    e, cuts = case_hit_that_merges()
    r = oracle.merge(e, cuts)
    assert list(r.final) == [2] and r.rounds == 2
    assert r.n_band_hits == 1


def test_band_scales_with_theta():
    """theta = 0.5: the band is 5e-6 wide.  half_out (7.34e-6 off) is outside,
    half_in (2.59e-6 off) inside; an absolute 1e-5 band would count both."""
    p = oracle.Params(theta=0.5)
    for nm, want in [("half_out", 0), ("half_in", 1)]:
        x, y = PAIRS[nm]
        e = np.zeros((2, 4), dtype=np.float32)
        e[0, 0] = 1
        e[1, :2] = (x, y)
        r = oracle.merge(e, [1], p)
        assert r.n_band_hits == want, nm


def test_band_scales_with_theta_merge_decisions():
    p = oracle.Params(theta=0.5)
    for nm, merged in [("half_out", True), ("half_in", False)]:
        x, y = PAIRS[nm]
        e = np.zeros((2, 4), dtype=np.float32)
        e[0, 0] = 1
        e[1, :2] = (x, y)
        r = oracle.merge(e, [1], p)
        assert (list(r.final) == []) == merged, nm


def test_band_edge_is_inclusive():
    """band_rel = 0 and theta = 63/65 (as the same f64): (3, 4) . (5, 12) / (5 * 13)
    is exactly 63/65 in f64 (integer dot and perfect-square norms: one rounding,
    the same as Python's 63/65).  |c - theta| = 0 <= 0 is a hit; `<` would count
    nothing.  c >= theta, so it also merges (ties merge, O9)."""
    p = oracle.Params(theta=63 / 65, band_rel=0.0)
    e = np.zeros((3, 4), dtype=np.float32)
    e[0, :2] = (3, 4)
    e[1, :2] = (5, 12)
    e[2, 2] = 1  # orthogonal third clip
    r = oracle.merge(e, [1, 2], p)
    assert r.cos[0] == 63 / 65
    assert r.n_band_hits == 1
    assert list(r.final) == [2]


# ---------------------------------------------------------------- the pins pin
_BAND_LINE = "if (fabs(c[k] - theta) <= band_rel * theta) hits += 1;"
_MUTANTS = {
    "theta dropped": "if (fabs(c[k] - theta) <= band_rel) hits += 1;",
    "strict <": "if (fabs(c[k] - theta) < band_rel * theta) hits += 1;",
    "last round only": "if (fabs(c[k] - theta) <= band_rel * theta) hits += 1; if (k == 0) hits = "
                       "(fabs(c[k] - theta) <= band_rel * theta);",
    "first round only": "if (r == 0 && fabs(c[k] - theta) <= band_rel * theta) hits += 1;",
    "merged pairs only": "if (c[k] >= theta && fabs(c[k] - theta) <= band_rel * theta) hits += 1;",
    "unmerged pairs only": "if (c[k] < theta && fabs(c[k] - theta) <= band_rel * theta) hits += 1;",
}


def _band_results(L):
    """(final, hits, rounds) of every band case through oracle_merge_stride of library L."""
    import ctypes
    f = L.oracle_merge_stride
    f.restype = ctypes.c_int64
    P, I32, I64, F64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    f.argtypes = [P, I64, I64, P, I64, F64, F64, I32, I64, P, P, P, P]
    cases = [case_edges() + ((0.9, 1e-5),), case_two_rounds() + ((0.9, 1e-5),),
             case_hit_that_merges() + ((0.9, 1e-5),)]
    for nm in ("half_out", "half_in"):
        e = np.zeros((2, 4), dtype=np.float32)
        e[0, 0] = 1
        e[1, :2] = PAIRS[nm]
        cases.append((e, [1], (0.5, 1e-5)))
    e = np.zeros((3, 4), dtype=np.float32)
    e[0, :2], e[1, :2], e[2, 2] = (3, 4), (5, 12), 1
    cases.append((e, [1, 2], (63 / 65, 0.0)))
    out = []
    for e, cuts, (theta, band) in cases:
        c = np.asarray(cuts, dtype=np.int64)
        fin = np.empty(len(cuts), dtype=np.int64)
        cos = np.empty(len(cuts), dtype=np.float64)
        hits, rounds = ctypes.c_int64(0), ctypes.c_int32(0)
        k = f(e.ctypes.data, e.shape[0], e.shape[1], c.ctypes.data, c.size, theta, band, 0, 1,
              fin.ctypes.data, cos.ctypes.data, ctypes.byref(hits), ctypes.byref(rounds))
        out.append((list(fin[:k]), hits.value, rounds.value))
    return out


# hand-derived expectations of the cases above (docstrings of band_cases / the tests)
_EXPECTED = [([2, 3, 4, 5, 6], 3, 2), ([1, 2], 2, 2), ([2], 1, 2), ([], 0, 1), ([1], 1, 1),
             ([2], 1, 2)]


def test_band_pins_reject_mutants(tmp_path):
    """Each plausible mistake in the band-hit line of oracle.c, compiled into a
    throw-away library, changes at least one hand-derived result above."""
    import ctypes
    import os
    import subprocess
    src = open(os.path.join(os.path.dirname(oracle.__file__), "oracle.c")).read()
    assert src.count(_BAND_LINE) == 1, "band-hit line moved: update the mutants"
    assert _band_results(oracle.lib()) == _EXPECTED
    for name, line in _MUTANTS.items():
        path = tmp_path / "m.c"
        path.write_text(src.replace(_BAND_LINE, line))
        so = tmp_path / f"m{abs(hash(name))}.so"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-shared", "-fPIC",
                               "-pthread", "-I", os.path.dirname(oracle.__file__), "-o", str(so),
                               str(path), "-lm"])
        assert _band_results(ctypes.CDLL(str(so))) != _EXPECTED, f"mutant survives: {name}"
