"""The C-ABI library loads (no GPU needed) and exports every symbol that
include/clip_detect.h declares; the Python binding is argument marshalling
over exactly those symbols; the product package never imports the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "clip_detect.h")


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(clip_\w+)\s*\(", src, re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2503_12964_b200 import _build
    _build.build()
    return _build.LIB


def test_header_declares_the_north_star_entry_points():
    d = _declared()
    for name in ["clip_detect_init", "clip_frame_scores", "clip_cuts", "clip_merge",
                 "clip_run_videos"]:
        assert name in d


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib_path], text=True)
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing


def test_library_loads_without_gpu(lib_path):
    L = ctypes.CDLL(lib_path)
    for s in _declared():
        assert getattr(L, s) is not None
    from paper_2503_12964_b200 import clipdetect
    p = clipdetect.default_params()
    assert (p.h_bins, p.s_bins, p.v_bins) == (18, 3, 3)
    assert p.cut_threshold_ppm == 300000 and p.min_clip_frames == 8
    assert p.merge_cos_threshold == 0.9 and p.band_rel == 1e-5


def test_binding_exports_match_header():
    from paper_2503_12964_b200 import clipdetect
    assert sorted(clipdetect.EXPORTS) == _declared()


def test_init_fails_loudly_without_b200(lib_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_12964_b200 import clipdetect
    L = clipdetect.load()
    h = ctypes.c_void_p()
    p = clipdetect.default_params()
    rc = L.clip_detect_init(ctypes.byref(h), ctypes.byref(p), 0, 0)
    assert rc != clipdetect.OK and not h.value


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2503_12964_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "oracle.h" not in text and "liboracle" not in text, f


def test_ctypes_struct_layouts_match_the_header(tmp_path):
    """Every struct the binding marshals has the header's size and field
    offsets (compiled with the system C compiler against include/clip_detect.h)."""
    from paper_2503_12964_b200 import clipdetect as cd
    structs = {"clip_params": cd.ClipParams, "clip_video": cd.ClipVideo,
               "clip_video_result": cd.ClipVideoResult, "clip_run_outputs": cd.ClipRunOutputs,
               "clip_stats": cd.ClipStats}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', 'int main(void) {']
    for cname, py in structs.items():
        lines.append(f'  printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {fname}));')
    lines.append('  return 0; }')
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-o", str(exe), str(src)])
    got = {}
    for line in subprocess.check_output([str(exe)], text=True).splitlines():
        c, f, v = line.split()
        got[(c, f)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)
