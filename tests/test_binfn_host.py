"""The device bin code (csrc/binfn.cuh: code_pair + code_to_bin, unpack4 and
bin_generic), compiled for the HOST with its CUDA intrinsics emulated, equals
the oracle's O1 bin on all 2^24 colours in both u16x2 lanes.  The same
functions are checked on the GPU by K5 (tests/test_gpu_parity.py)."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from nv12_helpers import yuv_rgb_table

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "binfn_host_check.cpp")
INC = os.path.join(ROOT, "paper_2503_12964_b200", "csrc")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("binfn") / "binfn_host_check")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-I", INC, "-o", out, SRC])
    return out


@pytest.mark.parametrize("bins", [(18, 3, 3), (12, 4, 4), (36, 3, 2)])
def test_device_bin_code_on_host_all_colours(exe, tmp_path, bins):
    path = str(tmp_path / "tables.bin")
    subprocess.check_call([exe, path, *map(str, bins)])
    raw = np.fromfile(path, dtype=np.uint8)
    n = 1 << 24
    t0, t1, tg, l0, l1, n0, n1, e0, e1, m0, m1 = (raw[i * n:(i + 1) * n] for i in range(11))
    p = oracle.Params(nh=bins[0], ns=bins[1], nv=bins[2])
    want = oracle.bin_table(p)
    assert np.array_equal(tg, want)
    if bins == (18, 3, 3):
        assert np.array_equal(t0, want), np.nonzero(t0 != want)[0][:10]
        assert np.array_equal(t1, want), np.nonzero(t1 != want)[0][:10]
        assert np.array_equal(l0, want), np.nonzero(l0 != want)[0][:10]
        assert np.array_equal(l1, want), np.nonzero(l1 != want)[0][:10]
        assert np.array_equal(e0, want), np.nonzero(e0 != want)[0][:10]  # direct-offset codes
        assert np.array_equal(e1, want), np.nonzero(e1 != want)[0][:10]
        yuv = want[yuv_rgb_table()]  # bin of every (Y, U, V): oracle O0 then O1
        assert np.array_equal(n0, yuv), np.nonzero(n0 != yuv)[0][:10]
        assert np.array_equal(n1, yuv), np.nonzero(n1 != yuv)[0][:10]
        assert np.array_equal(m0, yuv), np.nonzero(m0 != yuv)[0][:10]  # direct-offset codes
        assert np.array_equal(m1, yuv), np.nonzero(m1 != yuv)[0][:10]

