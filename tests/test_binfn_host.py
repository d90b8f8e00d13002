"""The device bin code (csrc/binfn.cuh: code_pair_dir_pre + the hue table +
code_to_bin_dir, unpack4, the NV12 conversion and bin_generic), compiled for
the HOST with its CUDA intrinsics emulated, equals the oracle's O1 bin (and
O0 then O1 for NV12) on all 2^24 inputs in both u16x2 lanes.  The same
functions are checked on the GPU by K5 (tests/test_gpu_parity.py,
tests/test_gpu_nv12.py)."""
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
    e0, e1, tg, m0, m1 = (raw[i * n:(i + 1) * n] for i in range(5))
    p = oracle.Params(nh=bins[0], ns=bins[1], nv=bins[2])
    want = oracle.bin_table(p)
    assert np.array_equal(tg, want)
    if bins == (18, 3, 3):
        assert np.array_equal(e0, want), np.nonzero(e0 != want)[0][:10]  # K1 codes, lane 0
        assert np.array_equal(e1, want), np.nonzero(e1 != want)[0][:10]  # lane 1
        yuv = want[yuv_rgb_table()]  # bin of every (Y, U, V): oracle O0 then O1
        assert np.array_equal(m0, yuv), np.nonzero(m0 != yuv)[0][:10]  # K1-NV12 codes
        assert np.array_equal(m1, yuv), np.nonzero(m1 != yuv)[0][:10]

