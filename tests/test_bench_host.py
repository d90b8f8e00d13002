"""Host-side logic of bench.py (no GPU): the ncu traffic files are used only when
they were captured from the current kernel sources, and the committed ones are."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_kernel_src_sha_is_a_content_hash():
    a = bench.kernel_src_sha("k1")
    assert len(a) == 16 and a == bench.kernel_src_sha("k1")
    assert a != bench.kernel_src_sha("k1_nv12")  # different source sets


def test_committed_traffic_files_match_the_sources():
    """profiles/k1*_traffic.json were captured from the kernels as they are now
    (else bench.py reports traffic as null with the reason)."""
    for kind in ("k1", "k1_nv12"):
        ratio, instr, src = bench.traffic_file(kind)
        assert ratio is not None, src
        assert 0.99 < ratio < 1.05 and 10 < instr < 40


def test_stale_traffic_file_is_refused(tmp_path, monkeypatch):
    prof = tmp_path / "profiles"
    prof.mkdir()
    (prof / "k1_traffic.json").write_text(json.dumps(
        {"dram_bytes_per_alg_byte": 1.0, "thread_instr_per_px": 19.0, "src_sha": "0" * 16}))
    csrc = tmp_path / "paper_2503_12964_b200" / "csrc"
    csrc.mkdir(parents=True)
    for f in bench.KERNEL_SOURCES["k1"]:
        (csrc / f).write_text(open(os.path.join(ROOT, "paper_2503_12964_b200", "csrc", f)).read())
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    ratio, instr, why = bench.traffic_file("k1")
    assert ratio is None and instr is None and "stale" in why
