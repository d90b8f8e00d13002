"""GPU parity of the NV12 input path (NEXT f1, reading O0): the fused
NV12 -> RGB -> bin -> histogram kernel (hist_nv12.cu) through the C ABI
against the CPU oracle (oracle_nv12_to_rgb + O1/O2), bit-exact."""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402

from nv12_helpers import random_nv12, yuv_bins  # noqa: E402

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
COS_RTOL = 1e-5


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    synth.build(device=True)
    return torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx(dev):
    from paper_2503_12964_b200 import Ctx
    c = Ctx(device=0)
    yield c
    c.close()


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def test_nv12map_every_yuv_fast(ctx):
    got = ctx.debug_nv12map().cpu().numpy()
    want = yuv_bins()
    for lane in range(2):
        bad = np.nonzero(got[lane] != want)[0]
        assert bad.size == 0, f"lane {lane}: {bad.size} (Y,U,V) differ, first {bad[:5]}"


@pytest.mark.parametrize("bins", [(12, 4, 4), (36, 3, 2)])
def test_nv12map_every_yuv_generic(dev, bins):
    from paper_2503_12964_b200 import Ctx, default_params
    c = Ctx(default_params(h_bins=bins[0], s_bins=bins[1], v_bins=bins[2]), device=0)
    got = c.debug_nv12map().cpu().numpy()
    c.close()
    want = yuv_bins(oracle.Params(nh=bins[0], ns=bins[1], nv=bins[2]))
    assert np.array_equal(got[0], want) and np.array_equal(got[1], want)


def _check(ctx, host, p=oracle.Params()):
    hist, l1, score = ctx.frame_scores_nv12(torch.from_numpy(host).to("cuda:0"))
    ref_h = oracle.hist_nv12_frames(host, p)
    npix = host.shape[2] * host.shape[1] * 2 // 3
    ref_l1, ref_sc = oracle.l1(ref_h, npix)
    assert np.array_equal(_u32(hist), ref_h)
    assert np.array_equal(_u32(l1), ref_l1)
    assert np.array_equal(score.cpu().numpy(), ref_sc.astype(np.float32))


# fast-path shapes (W % 16 == 0) with full and ragged last stages, one stage
# per frame, tall/narrow, 1080p and 4K rows; generic-path shapes (W % 16 != 0)
@pytest.mark.parametrize("W,H,n", [(1280, 720, 3), (1920, 1080, 2), (16, 2, 9), (64, 4, 5),
                                   (848, 480, 4), (3840, 16, 2), (8192, 4, 2), (32, 200, 3),
                                   (40, 36, 4), (854, 480, 2), (8208, 4, 1), (2, 16, 3),
                                   (10240, 4, 2), (13648, 4, 1), (20480, 2, 1), (20496, 2, 1)])
def test_nv12_scores_random(ctx, dev, W, H, n):
    rng = np.random.default_rng(W * 31 + H + n)
    if (H * W) % 32:
        pytest.skip("shape outside the NV12 contract")
    _check(ctx, random_nv12(rng, n, H, W))


def test_nv12_random_and_structured_with_map(dev):
    """K1-NV12 gives the oracle's histograms on random and structured surfaces
    in a fresh context, and the all-(Y,U,V) bin map equals the oracle's."""
    from paper_2503_12964_b200 import Ctx
    c = Ctx(device=0)
    rng = np.random.default_rng(106)
    _check(c, random_nv12(rng, 3, 720, 1280))
    _check(c, random_nv12(rng, 4, 240, 320, structured=True))
    got = c.debug_nv12map().cpu().numpy()
    want = yuv_bins()
    assert np.array_equal(got[0], want) and np.array_equal(got[1], want)
    c.close()


def test_nv12_scores_structured(ctx, dev):
    rng = np.random.default_rng(11)
    _check(ctx, random_nv12(rng, 6, 240, 320, structured=True))


def test_nv12_generic_bins_scores(dev):
    from paper_2503_12964_b200 import Ctx, default_params
    c = Ctx(default_params(h_bins=12, s_bins=4, v_bins=4), device=0)
    rng = np.random.default_rng(12)
    _check(c, random_nv12(rng, 3, 64, 96), oracle.Params(nh=12, ns=4, nv=4))
    c.close()


def test_nv12_prev_hist_chunk_carry(ctx, dev):
    v = manifest.c1_video()
    table = torch_dev.frame_table(v, dev)
    fr = torch.empty((v.n, v.H * 3 // 2, v.W), dtype=torch.uint8, device=dev)
    torch_dev.gen_nv12(v, table, fr)
    full_h, full_l1, _ = ctx.frame_scores_nv12(fr)
    for split in [1, 17, 63]:
        h1, a, _ = ctx.frame_scores_nv12(fr[:split].contiguous())
        h2, b, _ = ctx.frame_scores_nv12(fr[split:].contiguous(), prev_hist=h1[-1].contiguous())
        assert torch.equal(torch.cat([a, b]), full_l1) and torch.equal(torch.cat([h1, h2]), full_h)


def test_nv12_device_generator_matches_host(dev):
    v = manifest.c1_video()
    table = torch_dev.frame_table(v, dev)
    fr = torch.empty((v.n, v.H * 3 // 2, v.W), dtype=torch.uint8, device=dev)
    torch_dev.gen_nv12(v, table, fr)
    assert np.array_equal(fr.cpu().numpy(), synth.gen_nv12(v))


def _golden(name):
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    with open(path) as f:
        return json.load(f)


def _check_golden(g, res, hist, l1):
    assert list(res.detected) == g["detected"]
    assert list(res.final) == g["final"]
    assert res.n_candidates == g["n_candidates"]
    np.testing.assert_allclose(res.detected_cos, np.array(g["cos"]), rtol=COS_RTOL, atol=1e-12)
    assert hashlib.sha256(_u32(hist).tobytes()).hexdigest() == g["hist_sha256"]
    assert hashlib.sha256(_u32(l1).tobytes()).hexdigest() == g["l1_sha256"]


@pytest.mark.parametrize("name", ["C1_NV12", "C2_NV12"])
def test_nv12_run_videos_golden(ctx, dev, name):
    """Whole path a1-a9 on NV12 input through clip_run_videos (format = NV12),
    C2 at full size (18,000 720p frames, 24.9 GB NV12) resident in HBM."""
    from paper_2503_12964_b200.clipdetect import FORMAT_NV12
    g = _golden(name)["videos"][0]
    v = manifest.c1_video() if name == "C1_NV12" else manifest.c2_video()
    table = torch_dev.frame_table(v, dev)
    fr = torch.empty((v.n, v.H * 3 // 2, v.W), dtype=torch.uint8, device=dev)
    torch_dev.gen_nv12(v, table, fr)
    emb = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, table, emb)
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    l1 = torch.empty(v.n, dtype=torch.int32, device=dev)
    res = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": fr, "emb": emb,
                           "format": FORMAT_NV12}], hist=hist, l1=l1, want_cos=True)[0]
    _check_golden(g, res, hist, l1)
    del fr
    torch.cuda.empty_cache()


def test_nv12_mixed_sources_and_formats(ctx, dev):
    """RGB and NV12 videos, resident / host / callback sources, in one call:
    each equals the oracle for its own format."""
    from paper_2503_12964_b200.clipdetect import FORMAT_NV12, FORMAT_RGB24
    vids = [manifest.subsample(v, 120) for v in manifest.c5_videos()[:4]]
    items, refs, tables = [], [], {}
    for i, v in enumerate(vids):
        nv = i % 2 == 0
        host = synth.gen_nv12(v) if nv else synth.gen_frames(v)
        e_host = synth.gen_emb(v)
        src = [torch.from_numpy(host).to(dev), host, None, None][i]
        tables[i] = torch_dev.frame_table(v, dev)
        items.append({"n": v.n, "H": v.H, "W": v.W, "frames": src, "id": i,
                      "emb": torch.from_numpy(e_host).to(dev),
                      "format": FORMAT_NV12 if nv else FORMAT_RGB24})
        refs.append(oracle.run_video_nv12(host, e_host) if nv else oracle.run_video(host, e_host))

    def fill(vi, t0, n, dst, stream):
        v = vids[vi]
        gen = synth.dev_lib().synth_dev_gen_nv12 if vi % 2 == 0 else synth.dev_lib().synth_dev_gen_frames
        return gen(v.seed, v.id, v.W, v.H, t0, n, tables[vi].data_ptr(), dst, stream)

    res = ctx.run_videos(items, fill=fill, chunk_frames=29, want_cos=True)
    for r, ref in zip(res, refs):
        assert list(r.detected) == list(ref.detected)
        assert list(r.final) == list(ref.final)
        np.testing.assert_allclose(r.detected_cos, ref.cos, rtol=COS_RTOL, atol=1e-12)


def test_nv12_invalid_shapes(ctx, dev):
    from paper_2503_12964_b200 import ClipError
    bad = torch.zeros((2, 9, 6), dtype=torch.uint8, device=dev)  # H = 6, W = 6: H*W % 32 != 0
    with pytest.raises(ClipError) as e:
        ctx.frame_scores_nv12(bad)
    assert e.value.code == 1
    odd = torch.zeros((1, 48, 33), dtype=torch.uint8, device=dev)  # W odd
    with pytest.raises(ClipError):
        ctx.frame_scores_nv12(odd)
