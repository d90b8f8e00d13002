"""GPU parity of clip frame sampling + resize (NEXT f3, readings O10/O11):
K4 (sample.cu) through clip_sample_frames against oracle.sample_clips, bit-exact."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402

from nv12_helpers import random_nv12  # noqa: E402

pytestmark = pytest.mark.gpu


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


def _check(ctx, host, cuts, k, oh, ow):
    d = torch.from_numpy(host).to("cuda:0")
    c = torch.tensor(cuts, dtype=torch.int32, device="cuda:0") if len(cuts) else None
    out, idx = ctx.sample_frames(d, c, k, oh, ow)
    want, widx = oracle.sample_clips(host, cuts, k, oh, ow)
    assert idx.cpu().numpy().tolist() == widx.tolist()
    got = out.cpu().numpy()
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} bytes differ, first {bad[:3].tolist()}"


# resolutions of the workloads (854x480 rows are not 16-byte aligned), odd and
# upscaled outputs, tiny frames
@pytest.mark.parametrize("W,H,n,cuts,k,oh,ow", [
    (1280, 720, 40, [9, 17, 30], 3, 224, 224),
    (854, 480, 25, [8, 16], 4, 224, 224),
    (1920, 1080, 12, [5], 2, 224, 224),
    (3840, 2160, 4, [2], 1, 224, 224),
    (320, 240, 30, [1, 2, 29], 8, 37, 53),
    (64, 48, 10, [], 5, 96, 128),
    (16, 16, 6, [3], 2, 7, 5),
])
def test_sample_random_frames(ctx, dev, W, H, n, cuts, k, oh, ow):
    rng = np.random.default_rng(W + H + n)
    host = rng.integers(0, 256, (n, H, W, 3), dtype=np.uint8)
    _check(ctx, host, cuts, k, oh, ow)


def test_sample_c1_planted_clips(ctx, dev):
    v = manifest.c1_video()
    host = synth.gen_frames(v)
    _check(ctx, host, [10, 32, 53], 8, 224, 224)


def test_sample_after_run_videos_c2_prefix(ctx, dev):
    """The f3 step on the path's own output: final cuts of a 2,000-frame C2
    prefix from clip_run_videos, k = 8 frames per clip at 224x224."""
    v = manifest.subsample(manifest.c2_video(), 2000)
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    emb = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, table, emb)
    res = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": frames, "emb": emb}])[0]
    cuts = torch.from_numpy(res.final.astype(np.int32)).to(dev)
    out, idx = ctx.sample_frames(frames, cuts, 8, 224, 224)
    idx_h = idx.cpu().numpy()
    _, widx = oracle.sample_clips(np.zeros((v.n, 1, 1, 3), np.uint8), res.final.tolist(), 8, 1, 1)
    assert idx_h.tolist() == widx.tolist()
    got = out.cpu().numpy()
    for j in range(0, idx_h.size, 7):  # every 7th sampled frame against the oracle
        t = int(idx_h[j])
        fr = synth.gen_frames(v, t0=t, n=1)[0]
        assert np.array_equal(got[j], oracle.resize_linear(fr, 224, 224)), (j, t)


def test_sample_full_c2_in_bench_configuration(ctx, dev):
    """The whole C2 video (18,000 x 720p, resident) -> clip_run_videos -> final
    cuts -> K4 with k = 8 at 224x224, exactly as bench.py's f3_sample times it;
    every sampled index checked, every 13th output frame against the oracle."""
    v = manifest.c2_video()
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    emb = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, table, emb)
    res = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": frames, "emb": emb}])[0]
    cuts = torch.from_numpy(res.final.astype(np.int32)).to(dev)
    out, idx = ctx.sample_frames(frames, cuts, 8, 224, 224)
    idx_h = idx.cpu().numpy()
    bounds = [0] + res.final.tolist() + [v.n]
    want = [oracle.sample_index(bounds[c], bounds[c + 1], i, 8) for c in range(len(bounds) - 1)
            for i in range(8)]
    assert idx_h.tolist() == want
    got = out.cpu().numpy()
    for j in range(0, idx_h.size, 13):
        t = int(idx_h[j])
        fr = synth.gen_frames(v, t0=t, n=1)[0]
        assert np.array_equal(got[j], oracle.resize_linear(fr, 224, 224)), (j, t)
    del frames, out
    torch.cuda.empty_cache()


def test_sample_invalid(ctx, dev):
    from paper_2503_12964_b200 import ClipError
    fr = torch.zeros((4, 16, 16, 3), dtype=torch.uint8, device=dev)
    with pytest.raises(ClipError):
        ctx.sample_frames(fr, None, 0, 8, 8)
    with pytest.raises(ClipError):
        ctx.sample_frames(fr, None, 1, 8, 5000)


@pytest.mark.parametrize("W,H,n,cuts,k,oh,ow", [
    (1280, 720, 20, [9, 13], 3, 224, 224),
    (854, 480, 12, [5], 2, 224, 224),
    (1920, 1080, 6, [2], 2, 224, 224),
    (64, 48, 8, [], 3, 96, 128),
    (32, 16, 5, [1, 4], 2, 7, 9),
])
def test_sample_nv12_random_frames(ctx, dev, W, H, n, cuts, k, oh, ow):
    """NV12 input: every tap converted by O0, then O11 — equal to the oracle's
    resize of the oracle's full-frame conversion."""
    rng = np.random.default_rng(W * 3 + H + n)
    host = random_nv12(rng, n, H, W, structured=(W % 64 == 0))
    rgb = np.stack([oracle.nv12_to_rgb(f) for f in host])
    d = torch.from_numpy(host).to(dev)
    c = torch.tensor(cuts, dtype=torch.int32, device=dev) if cuts else None
    out, idx = ctx.sample_frames(d, c, k, oh, ow)
    want, widx = oracle.sample_clips(rgb, cuts, k, oh, ow)
    assert idx.cpu().numpy().tolist() == widx.tolist()
    assert np.array_equal(out.cpu().numpy(), want)
