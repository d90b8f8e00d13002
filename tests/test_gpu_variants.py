"""GPU parity of the f4 variants (NEXT f4; readings O3', O4''): distance scores
bit-identical (same IEEE f64 operations in the same order, rounded to f32) and
cut lists identical to the oracle, through clip_frame_scores / clip_run_videos."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402

from nv12_helpers import random_nv12  # noqa: E402

pytestmark = pytest.mark.gpu
COS_RTOL = 1e-5
KINDS = [(1, 200000), (2, 400000), (3, 500000)]


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    synth.build(device=True)
    return torch.device("cuda:0")


def _ctx(**kw):
    from paper_2503_12964_b200 import Ctx, default_params
    return Ctx(default_params(**kw), device=0)


@pytest.mark.parametrize("kind,tau", KINDS)
def test_variant_scores_bit_identical(dev, kind, tau):
    c = _ctx(distance=kind, cut_threshold_ppm=tau)
    rng = np.random.default_rng(kind)
    v = manifest.c1_video()
    c1 = synth.gen_frames(v)
    noise = rng.integers(0, 256, (9, 120, 160, 3), dtype=np.uint8)
    noise[3] = noise[2]  # identical pair: distance 0
    noise[5] = 128       # flat frame: correlation's zero-variance branch
    noise[6] = 128
    for host in (c1, noise):
        _, l1, score = c.frame_scores(torch.from_numpy(host).to(dev))
        h = oracle.hist_frames(host)
        want = oracle.distances(h, host[0].size // 3, kind).astype(np.float32)
        assert np.array_equal(score.cpu().numpy(), want)
        assert np.array_equal(l1.cpu().numpy().view(np.uint32), oracle.l1(h, host[0].size // 3)[0])
    c.close()


def _videos(dev, n_videos=4, n=240):
    vids = [manifest.subsample(v, n) for v in manifest.c5_videos()[:n_videos]] + [manifest.c1_video()]
    items, hosts = [], []
    for i, v in enumerate(vids):
        host = synth.gen_frames(v)
        emb = synth.gen_emb(v)
        items.append({"n": v.n, "H": v.H, "W": v.W, "frames": torch.from_numpy(host).to(dev),
                      "emb": torch.from_numpy(emb).to(dev), "id": i})
        hosts.append((host, emb))
    return items, hosts


@pytest.mark.parametrize("kind,tau", KINDS)
def test_variant_run_videos_matches_oracle(dev, kind, tau):
    items, hosts = _videos(dev)
    c = _ctx(distance=kind, cut_threshold_ppm=tau)
    res = c.run_videos(items, want_cos=True)
    c.close()
    for r, (host, emb) in zip(res, hosts):
        ref = oracle.run_video_variant(host, emb, oracle.Params(tau_ppm=tau), distance_kind=kind)
        assert r.n_candidates == ref.n_candidates
        assert list(r.detected) == list(ref.detected) and list(r.final) == list(ref.final)
        np.testing.assert_allclose(r.detected_cos, ref.cos, rtol=COS_RTOL, atol=1e-12)
    assert list(res[-1].final) == [10, 32, 53]  # C1's planted truth


@pytest.mark.parametrize("w,ratio,tau", [(2, 3000000, 100000), (1, 2000000, 0), (8, 1500000, 50000)])
def test_adaptive_run_videos_matches_oracle(dev, w, ratio, tau):
    items, hosts = _videos(dev)
    c = _ctx(adaptive_window=w, adaptive_ratio_ppm=ratio, cut_threshold_ppm=tau)
    res = c.run_videos(items, want_cos=True)
    c.close()
    for r, (host, emb) in zip(res, hosts):
        ref = oracle.run_video_variant(host, emb, oracle.Params(tau_ppm=tau), adaptive_window=w,
                                       adaptive_ratio_ppm=ratio)
        assert r.n_candidates == ref.n_candidates
        assert list(r.detected) == list(ref.detected) and list(r.final) == list(ref.final)


def test_variant_on_nv12_input(dev):
    from paper_2503_12964_b200.clipdetect import FORMAT_NV12
    v = manifest.c1_video()
    host = synth.gen_nv12(v)
    emb = synth.gen_emb(v)
    c = _ctx(distance=1, cut_threshold_ppm=200000)
    r = c.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": torch.from_numpy(host).to(dev),
                       "emb": torch.from_numpy(emb).to(dev), "format": FORMAT_NV12}])[0]
    c.close()
    ref = oracle.run_video_variant(host, emb, oracle.Params(tau_ppm=200000), distance_kind=1, nv12=True)
    assert list(r.detected) == list(ref.detected) and list(r.final) == list(ref.final) == [10, 32, 53]


def test_streaming_cuts_reject_variants(dev):
    from paper_2503_12964_b200 import ClipError
    c = _ctx(distance=2)
    l1 = torch.zeros(10, dtype=torch.int32, device=dev)
    st = torch.zeros(4, dtype=torch.int64, device=dev)
    cuts = torch.zeros(4, dtype=torch.int32, device=dev)
    with pytest.raises(ClipError):
        c.cuts(l1, 100, st, cuts, True)
    c.close()
    with pytest.raises(ClipError):  # adaptive needs the L1 distance
        _ctx(distance=1, adaptive_window=2)


@pytest.mark.parametrize("sigma", [2, 5, 16, 40])
def test_keyframe_stride_matches_oracle(dev, sigma):
    """O8': only every sigma-th frame of each detected clip is summed; the
    other embeddings are NaN here and must never be read."""
    items, hosts = _videos(dev)
    c = _ctx(emb_stride=sigma)
    ref0 = [oracle.run_video(h, e) for h, e in hosts]  # detected cuts (stride-independent)
    for it, (host, emb), r0 in zip(items, hosts, ref0):
        key = np.zeros(host.shape[0], bool)
        b = [0] + r0.detected.tolist() + [host.shape[0]]
        for s0, s1 in zip(b[:-1], b[1:]):
            key[s0:s1:sigma] = True
        poisoned = emb.copy()
        poisoned[~key] = np.nan
        it["emb"] = torch.from_numpy(poisoned).to(dev)
    res = c.run_videos(items, want_cos=True)
    c.close()
    for r, (host, emb) in zip(res, hosts):
        ref = oracle.run_video_variant(host, emb, oracle.Params(), emb_stride=sigma)
        assert list(r.detected) == list(ref.detected) and list(r.final) == list(ref.final)
        np.testing.assert_allclose(r.detected_cos, ref.cos, rtol=COS_RTOL, atol=1e-12)
        assert r.rounds == ref.rounds
