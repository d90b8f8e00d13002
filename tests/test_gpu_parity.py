"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bit-exact: bin map, histograms, L1, candidates, detected and final cuts.
Floating point: score is one f64 division rounded to f32 on both sides (exact);
cosines within 1e-5 relative (BASELINE.json north_star), and every decision
taken within that band is reported (band hits) rather than hidden.
"""
import hashlib
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402

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


@pytest.mark.gpu
def test_device_generator_matches_host(dev):
    """synth_dev_gen_frames (the bench's and the streamed tests' frame source)
    writes the host generator's bytes: tiny and odd widths (one CTA spanning
    many texture-cell rows), C1, 480p / 1080p with fades and flashes, noise
    frames and 4K."""
    vids = [manifest.c1_video(),
            manifest.random_video(7, 1, 16, 4, 40, 0.75, 0.10, 0.15, 3.0),
            manifest.random_video(7, 2, 48, 30, 40, 0.75, 0.10, 0.15, 3.0),
            manifest.random_video(7, 5, 40, 8, 30, 0.75, 0.10, 0.15, 3.0),
            manifest.random_video(7, 3, 854, 480, 64, 0.75, 0.10, 0.15, 3.0),
            manifest.subsample(manifest.c3_videos()[0], 90),
            manifest.noise_video(4, 64, 64, 8),
            manifest.subsample(manifest.c4_videos()[0], 2)]
    for v in vids:
        frames, _ = _dev_video(v, dev, emb=False)
        assert np.array_equal(frames.cpu().numpy(), synth.gen_frames(v)), (v.id, v.W, v.H)


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _dev_video(v, dev, emb=True):
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    e = None
    if emb:
        e = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
        torch_dev.gen_emb(v, table, e)
    return frames, e


# ------------------------------------------------------------------ a1-a2
def test_binmap_all_colours_fast(ctx):
    got = ctx.debug_binmap().cpu().numpy()
    want = oracle.bin_table()
    for lane in range(2):
        bad = np.nonzero(got[lane] != want)[0]
        assert bad.size == 0, f"lane {lane}: {bad.size} colours differ, first {bad[:5]}"


@pytest.mark.parametrize("bins", [(12, 4, 4), (6, 2, 2), (36, 3, 2), (8, 8, 4)])
def test_binmap_all_colours_generic(dev, bins):
    from paper_2503_12964_b200 import Ctx, default_params
    c = Ctx(default_params(h_bins=bins[0], s_bins=bins[1], v_bins=bins[2]), device=0)
    got = c.debug_binmap().cpu().numpy()
    want = oracle.bin_table(oracle.Params(nh=bins[0], ns=bins[1], nv=bins[2]))
    c.close()
    assert np.array_equal(got[0], want) and np.array_equal(got[1], want)


# ------------------------------------------------------------------ a3-a4
def _check_scores(ctx, frames_dev, frames_host, p=oracle.Params()):
    hist, l1, score = ctx.frame_scores(frames_dev)
    ref_h = oracle.hist_frames(frames_host, p)
    ref_l1, ref_sc = oracle.l1(ref_h, frames_host[0].size // 3)
    assert np.array_equal(_u32(hist), ref_h)
    assert np.array_equal(_u32(l1), ref_l1)
    assert np.array_equal(score.cpu().numpy(), ref_sc.astype(np.float32))


def test_scores_c1(ctx, dev):
    v = manifest.c1_video()
    frames, _ = _dev_video(v, dev, emb=False)
    _check_scores(ctx, frames, synth.gen_frames(v))


@pytest.mark.parametrize("W,H,n", [(854, 480, 5), (4, 4, 3), (16, 1, 40), (100, 36, 7),
                                   (1920, 1080, 2), (320, 240, 33)])
def test_scores_random_noise_ragged(ctx, dev, W, H, n):
    # uniform random colours: worst case for bin spread; shapes with a ragged
    # last stage (854x480, 1080p), tiny frames (1 group), many small frames
    rng = np.random.default_rng(W * 7 + H + n)
    host = rng.integers(0, 256, size=(n, H, W, 3), dtype=np.uint8)
    _check_scores(ctx, torch.from_numpy(host).to(dev), host)


def test_scores_flat_and_permuted(ctx, dev):
    rng = np.random.default_rng(5)
    base = rng.integers(0, 256, size=(240, 320, 3), dtype=np.uint8)
    perm = base.reshape(-1, 3)[rng.permutation(240 * 320)].reshape(240, 320, 3)
    flat = np.zeros_like(base)
    flat[:] = (12, 200, 77)
    host = np.stack([base, perm, flat, flat, base])
    hist, l1, _ = ctx.frame_scores(torch.from_numpy(host).to(dev))
    h = _u32(hist)
    assert np.array_equal(h[0], h[1])  # permutation invariance
    assert _u32(l1)[1] == 0 and _u32(l1)[3] == 0
    assert np.array_equal(h, oracle.hist_frames(host))


def test_scores_prev_hist_chunk_carry(ctx, dev):
    v = manifest.c1_video()
    frames, _ = _dev_video(v, dev, emb=False)
    full_h, full_l1, _ = ctx.frame_scores(frames)
    for split in [1, 10, 11, 33, 63]:
        h1, l1a, _ = ctx.frame_scores(frames[:split].contiguous())
        h2, l1b, _ = ctx.frame_scores(frames[split:].contiguous(), prev_hist=h1[-1].contiguous())
        assert torch.equal(torch.cat([l1a, l1b]), full_l1)
        assert torch.equal(torch.cat([h1, h2]), full_h)


# ------------------------------------------------------------------ a5-a6
def _stream_cuts(ctx, dev, l1_host, npix, chunks, cap=None):
    n = l1_host.size
    l1 = torch.from_numpy(l1_host.view(np.int32)).to(dev)
    state = torch.zeros(4, dtype=torch.int64, device=dev)
    cap = cap if cap is not None else n + 1
    cuts = torch.full((max(1, cap),), -1, dtype=torch.int32, device=dev)
    bounds = [0] + sorted(chunks) + [n]
    for i in range(len(bounds) - 1):
        a, b = bounds[i], bounds[i + 1]
        ctx.cuts(l1[a:b].contiguous() if b > a else None, npix, state, cuts, i == len(bounds) - 2)
    st = state.cpu().numpy()
    k = int(st[3])
    return cuts.cpu().numpy()[:min(k, cap)], st


def test_cuts_streaming_every_split(ctx, dev):
    rng = np.random.default_rng(12)
    npix = 100
    for trial in range(6):
        n = int(rng.integers(20, 300))
        l1 = np.where(rng.random(n) < 0.3, rng.integers(60, 201, n), rng.integers(0, 60, n)).astype(np.uint32)
        l1[0] = 0
        want = oracle.min_length(oracle.candidates(l1, npix), n, 8)
        for split in range(0, n + 1, max(1, n // 25)):
            got, st = _stream_cuts(ctx, dev, l1, npix, [split] if 0 < split < n else [])
            assert list(got) == list(want), (trial, split)
            assert st[0] == n and st[2] == oracle.candidates(l1, npix).size


def test_cuts_all_candidates_closed_form(ctx, dev):
    for n in [1, 7, 8, 15, 16, 17, 100, 1000, 4097]:
        l1 = np.full(n, 200, dtype=np.uint32)
        got, _ = _stream_cuts(ctx, dev, l1, 100, [n // 3, n // 2] if n > 4 else [])
        assert list(got) == [8 * k for k in range(1, n // 8)]


def test_cuts_capacity_overflow_reported(ctx, dev):
    l1 = np.full(200, 200, dtype=np.uint32)
    got, st = _stream_cuts(ctx, dev, l1, 100, [], cap=5)
    assert st[3] == 200 // 8 - 1 and list(got) == [8, 16, 24, 32, 40]


# ------------------------------------------------------------------ a7-a9
def test_merge_random_vs_oracle(ctx, dev):
    rng = np.random.default_rng(21)
    for trial in range(25):
        n = int(rng.integers(10, 700))
        dim = int(rng.choice([3, 64, 768, 1000]))
        k = int(rng.integers(0, 20))
        cuts = sorted(set(int(x) for x in rng.integers(1, n, size=k)))
        centres = rng.standard_normal((3, dim))
        B = [0] + cuts + [n]
        e = np.zeros((n, dim), dtype=np.float32)
        for j in range(len(B) - 1):
            c = centres[rng.integers(0, 3)] + 0.3 * rng.standard_normal(dim)
            e[B[j]:B[j + 1]] = (c + 0.1 * rng.standard_normal((B[j + 1] - B[j], dim))).astype(np.float32)
        ref = oracle.merge(e, cuts)
        m, cos, hits, rounds = ctx.merge(torch.from_numpy(e).to(dev),
                                         torch.tensor(cuts if cuts else [0], dtype=torch.int32, device=dev),
                                         n_cuts=len(cuts))
        assert list(m.cpu().numpy()) == list(ref.final), trial
        if cuts:
            np.testing.assert_allclose(cos.cpu().numpy(), ref.cos, rtol=COS_RTOL, atol=1e-12)
        assert hits == ref.n_band_hits and rounds == ref.rounds


def test_merge_worked_example(ctx, dev):
    import math
    e = np.zeros((6, 768), dtype=np.float32)
    for i, deg in enumerate([0, 0, 0, 0, 20, -10]):
        e[i, 0], e[i, 1] = math.cos(math.radians(deg)), math.sin(math.radians(deg))
    m, cos, hits, rounds = ctx.merge(torch.from_numpy(e).to(dev),
                                     torch.tensor([4, 5], dtype=torch.int32, device=dev))
    assert m.numel() == 0 and rounds == 2


# ------------------------------------------------------------------ a1-a9 end to end
def _golden(name):
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    with open(path) as f:
        return json.load(f)


def _check_against_golden(g, res, hist=None, l1=None):
    assert list(res.detected) == g["detected"], g["id"]
    assert list(res.final) == g["final"], g["id"]
    assert res.n_candidates == g["n_candidates"]
    if res.detected_cos is not None and g["detected"]:
        np.testing.assert_allclose(res.detected_cos, np.array(g["cos"]), rtol=COS_RTOL, atol=1e-12)
    if hist is not None:
        assert hashlib.sha256(np.ascontiguousarray(hist).tobytes()).hexdigest() == g["hist_sha256"]
    if l1 is not None:
        assert hashlib.sha256(np.ascontiguousarray(l1).tobytes()).hexdigest() == g["l1_sha256"]


def test_run_videos_c1_golden(ctx, dev):
    g = _golden("C1")["videos"][0]
    v = manifest.c1_video()
    frames, emb = _dev_video(v, dev)
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    l1 = torch.empty(v.n, dtype=torch.int32, device=dev)
    res = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": frames, "emb": emb}],
                         hist=hist, l1=l1, want_cos=True)[0]
    _check_against_golden(g, res, _u32(hist), _u32(l1))
    assert res.final.tolist() == [10, 32, 53]


def test_run_videos_c2_full_golden(ctx, dev):
    """C2 at full size (18,000 720p frames, 49.8 GB) in the launch configuration
    bench.py times: every histogram, L1, cut and cosine against the oracle."""
    g = _golden("C2")["videos"][0]
    v = manifest.c2_video()
    frames, emb = _dev_video(v, dev)
    fh = torch_dev.frame_hashes(frames[[int(t) for t in g["frame_hash"]]].contiguous())
    assert [str(int(x)) for x in fh] == list(g["frame_hash"].values())
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    l1 = torch.empty(v.n, dtype=torch.int32, device=dev)
    res = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": frames, "emb": emb}],
                         hist=hist, l1=l1, want_cos=True)[0]
    _check_against_golden(g, res, _u32(hist), _u32(l1))
    assert set(v.hard) <= set(res.final.tolist())
    del frames
    torch.cuda.empty_cache()


def _run_config_streamed(ctx, dev, name, max_videos=None):
    """Frames produced chunk by chunk by the device generator through the fill
    callback (C3/C4/C5 do not fit in HBM at once)."""
    gold = _golden(name)
    vids = manifest.config_videos(name)
    if max_videos:
        vids = vids[:max_videos]
    tables = [torch_dev.frame_table(v, dev) for v in vids]
    embs = []
    for v, t in zip(vids, tables):
        e = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
        torch_dev.gen_emb(v, t, e)
        embs.append(e)
    F = sum(v.n for v in vids)
    hist = torch.empty((F, 162), dtype=torch.int32, device=dev)
    l1 = torch.empty(F, dtype=torch.int32, device=dev)

    def fill(vi, t0, n, dst, stream):
        v = vids[vi]
        rc = synth.dev_lib().synth_dev_gen_frames(v.seed, v.id, v.W, v.H, t0, n,
                                                  tables[vi].data_ptr(), dst, stream)
        return rc

    res = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": None, "emb": e, "id": v.id}
                          for v, e in zip(vids, embs)], fill=fill, hist=hist, l1=l1, want_cos=True)
    h, l = _u32(hist), _u32(l1)
    off = 0
    for v, r in zip(vids, res):
        g = gold["videos"][v.id]
        _check_against_golden(g, r, h[off:off + v.n], l[off:off + v.n])
        # planted hard cuts survive unless a fade/flash exit within L_min+12 frames
        # before them already took the cut (a property of the method, O5)
        clear = [c for c in v.hard
                 if all(abs(c - f) > 20 for f in v.fades) and all(abs(c - s) > 20 for s, _ in v.flashes)]
        assert set(clear) <= set(r.final.tolist())
        off += v.n
    return res


def test_run_videos_c3_golden(ctx, dev):
    _run_config_streamed(ctx, dev, "C3")


def test_run_videos_c4_golden(ctx, dev):
    _run_config_streamed(ctx, dev, "C4")


def test_run_videos_c5_golden(ctx, dev):
    _run_config_streamed(ctx, dev, "C5")


def test_batch_mixed_sources_equal_single(ctx, dev):
    """Resident, host-pointer and callback videos in one call give the same
    per-video results as one call per video (and as the oracle)."""
    vids = [manifest.subsample(v, 150) for v in manifest.c5_videos()[:4]]
    items, refs = [], []
    for i, v in enumerate(vids):
        host = synth.gen_frames(v)
        emb = torch.from_numpy(synth.gen_emb(v)).to(dev)
        src = [torch.from_numpy(host).to(dev), host, None, torch.from_numpy(host).to(dev)][i]
        items.append({"n": v.n, "H": v.H, "W": v.W, "frames": src, "emb": emb, "id": i,
                      "_host": host})
        refs.append(oracle.run_video(host, synth.gen_emb(v)))
    tables = {i: torch_dev.frame_table(v, dev) for i, v in enumerate(vids)}

    def fill(vi, t0, n, dst, stream):
        v = vids[vi]
        return synth.dev_lib().synth_dev_gen_frames(v.seed, v.id, v.W, v.H, t0, n,
                                                    tables[vi].data_ptr(), dst, stream)

    res = ctx.run_videos(items, fill=fill, chunk_frames=37, want_cos=True)
    for r, ref in zip(res, refs):
        assert list(r.detected) == list(ref.detected)
        assert list(r.final) == list(ref.final)
        np.testing.assert_allclose(r.detected_cos, ref.cos, rtol=COS_RTOL, atol=1e-12)


def test_invalid_arguments_fail_without_side_effects(ctx, dev):
    from paper_2503_12964_b200 import ClipError
    bad = torch.zeros((2, 3, 5, 3), dtype=torch.uint8, device=dev)  # H*W = 15
    with pytest.raises(ClipError) as e:
        ctx.frame_scores(bad)
    assert e.value.code == 1
    with pytest.raises(ClipError):
        ctx.run_videos([{"n": 0, "H": 4, "W": 4, "frames": None, "emb": None}])
    # ctx still usable
    v = manifest.c1_video()
    frames, _ = _dev_video(v, dev, emb=False)
    ctx.frame_scores(frames)
    torch.cuda.synchronize()


# ------------------------------------------------------------------ K1 corner cases
def test_k1_corner_frames_and_ragged_stages(ctx, dev):
    """K1's fast path on the hue table's corner cases (black, grey, a yellow
    edge where q = 3 in the rising sector), uniform noise with a ragged last
    stage (854x480 = 25,620 groups = 32 stages + 20 groups), and C1."""
    rng = np.random.default_rng(55)
    host = rng.integers(0, 256, size=(6, 480, 854, 3), dtype=np.uint8)
    host[1] = 0            # black
    host[2] = 128          # grey
    host[3, :, :, :] = (200, 200, 10)  # yellow edge (q = 3 in the rising sector)
    c1 = synth.gen_frames(manifest.c1_video())
    for frames in (host, c1):
        hist, l1, _ = ctx.frame_scores(torch.from_numpy(frames).to(dev))
        assert np.array_equal(_u32(hist), oracle.hist_frames(frames))


@pytest.mark.parametrize("bins", [(12, 4, 4), (6, 2, 2), (36, 3, 2)])
def test_k1_generic_bins_frames(dev, bins):
    """Bin layouts other than 18x3x3 run K1's pipeline with bin_generic per
    pixel: histograms and L1 against the oracle at full stages (1280x720),
    ragged stages (854x480) and tiny frames."""
    from paper_2503_12964_b200 import Ctx, default_params
    p = oracle.Params(nh=bins[0], ns=bins[1], nv=bins[2])
    c = Ctx(default_params(h_bins=bins[0], s_bins=bins[1], v_bins=bins[2]), device=0)
    rng = np.random.default_rng(sum(bins))
    try:
        for n, H, W in [(3, 720, 1280), (4, 480, 854), (9, 4, 4)]:
            host = rng.integers(0, 256, size=(n, H, W, 3), dtype=np.uint8)
            hist, l1, _ = c.frame_scores(torch.from_numpy(host).to(dev))
            want = oracle.hist_frames(host, p)
            assert np.array_equal(_u32(hist), want), (bins, W, H)
            assert np.array_equal(_u32(l1), oracle.l1(want, H * W)[0])
    finally:
        c.close()


def test_run_to_run_determinism(ctx, dev):
    """Histograms, cuts and cosines are bit-identical across runs."""
    v = manifest.subsample(manifest.c3_videos()[1], 300)
    frames, emb = _dev_video(v, dev)
    item = [{"n": v.n, "H": v.H, "W": v.W, "frames": frames, "emb": emb}]
    a = ctx.run_videos(item, want_cos=True)[0]
    b = ctx.run_videos(item, want_cos=True)[0]
    assert list(a.detected) == list(b.detected) and list(a.final) == list(b.final)
    assert np.array_equal(a.detected_cos, b.detected_cos)  # bitwise, not approx


def test_tiny_and_cutless_videos(ctx, dev):
    """n = 1, n < 2 L_min, a flat video (no candidates) and a normal one in one
    batch: empty cut lists where the oracle has none, merge with K = 1 clip."""
    rng = np.random.default_rng(77)
    items, refs = [], []
    for n in [1, 3, 15, 40]:
        if n == 40:
            v = manifest.subsample(manifest.c1_video(), 40)
            host = synth.gen_frames(v)
        else:
            host = np.broadcast_to(rng.integers(0, 256, size=(1, 1, 1, 3), dtype=np.uint8),
                                   (n, 16, 32, 3)).copy()
        emb = rng.standard_normal((n, 8)).astype(np.float32)
        items.append({"n": n, "H": host.shape[1], "W": host.shape[2],
                      "frames": torch.from_numpy(host).to(dev), "emb": torch.from_numpy(emb).to(dev)})
        refs.append(oracle.run_video(host, emb))
    res = ctx.run_videos(items, want_cos=True)
    for r, ref in zip(res, refs):
        assert list(r.detected) == list(ref.detected)
        assert list(r.final) == list(ref.final)
        assert r.rounds == ref.rounds


def test_c2_full_through_per_step_api_in_chunks(ctx, dev):
    """C2 at full size through the per-step entry points, streamed in ~1 GiB
    chunks: clip_frame_scores (prev_hist carry) -> clip_cuts (device-resident
    state, tail rule on the last chunk) -> clip_merge; every histogram and L1
    value and both cut lists equal the oracle golden."""
    g = _golden("C2")["videos"][0]
    v = manifest.c2_video()
    table = torch_dev.frame_table(v, dev)
    emb = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, table, emb)
    chunk = 388
    buf = torch.empty((chunk, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    hist = torch.empty((v.n, 162), dtype=torch.int32, device=dev)
    l1 = torch.empty(v.n, dtype=torch.int32, device=dev)
    state = torch.zeros(4, dtype=torch.int64, device=dev)
    cuts = torch.empty(v.n // 8 + 2, dtype=torch.int32, device=dev)
    prev = None
    for t0 in range(0, v.n, chunk):
        m = min(chunk, v.n - t0)
        fr = buf[:m]
        torch_dev.gen_frames(v, table, fr, t0=t0, n=m)
        ctx.frame_scores(fr, prev_hist=prev, hist=hist[t0:t0 + m], l1=l1[t0:t0 + m],
                         want_score=False)
        ctx.cuts(l1[t0:t0 + m], v.W * v.H, state, cuts, t0 + m == v.n)
        prev = hist[t0 + m - 1]
    torch.cuda.synchronize()
    assert hashlib.sha256(_u32(hist).tobytes()).hexdigest() == g["hist_sha256"]
    assert hashlib.sha256(_u32(l1).tobytes()).hexdigest() == g["l1_sha256"]
    st = state.cpu().numpy()
    assert st[2] == g["n_candidates"] and st[0] == v.n
    det = cuts.cpu().numpy()[:st[3]].tolist()
    assert det == g["detected"]
    merged, cos, hits, rounds = ctx.merge(emb, cuts[:st[3]].contiguous(), n_cuts=int(st[3]))
    assert merged.cpu().numpy().tolist() == g["final"]
    np.testing.assert_allclose(cos.cpu().numpy(), np.array(g["cos"]), rtol=COS_RTOL, atol=1e-12)
    assert hits == g["n_band_hits"] and rounds == g["rounds"]


def test_8k_frames_rgb_and_nv12(ctx, dev):
    """Maximum-size frames of practical video (7680x4320, 99.5 MB RGB24): K1 and
    K1-NV12 (one frame spans ~4,050 stages, many CTAs per frame) equal the oracle."""
    rng = np.random.default_rng(8)
    H, W = 4320, 7680
    rgb = rng.integers(0, 256, (2, H, W, 3), dtype=np.uint8)
    rgb[1, : H // 2] = rgb[0, : H // 2]  # half the second frame repeats the first
    hist, l1, _ = ctx.frame_scores(torch.from_numpy(rgb).to(dev))
    want = oracle.hist_frames(rgb)
    assert np.array_equal(_u32(hist), want)
    assert np.array_equal(_u32(l1), oracle.l1(want, H * W)[0])
    del rgb
    from nv12_helpers import random_nv12
    nv = random_nv12(rng, 2, H, W)
    hist, l1, _ = ctx.frame_scores_nv12(torch.from_numpy(nv).to(dev))
    want = oracle.hist_nv12_frames(nv)
    assert np.array_equal(_u32(hist), want)
    torch.cuda.empty_cache()


def test_frame_count_limit_rejected_before_any_work(ctx, dev):
    """A batch of more than INT32_MAX frames is refused by validation (nothing is
    allocated, generated or launched: the fill callback is never called)."""
    from paper_2503_12964_b200 import ClipError
    called = []

    def fill(*a):
        called.append(a)
        return 1

    vids = [{"n": (1 << 30), "H": 16, "W": 16, "frames": None, "emb": None} for _ in range(3)]
    with pytest.raises(ClipError) as e:
        ctx.run_videos(vids, fill=fill)
    assert e.value.code == 1 and not called


def test_python_shell_run(dev):
    """clipdetect.run (SURVEY §8(b) Python shell) on C1: RGB and NV12."""
    from paper_2503_12964_b200 import run
    v = manifest.c1_video()
    frames, emb = _dev_video(v, dev)
    fin, det = run(frames, emb, want_detected=True)
    assert fin == [10, 32, 53] and det == [10, 21, 32, 43, 53]
    nv = torch.from_numpy(synth.gen_nv12(v)).to(dev)
    assert run(nv, emb) == [10, 32, 53]
    assert run(frames) == [10, 21, 32, 43, 53]  # no embeddings: no merge


# ------------------------------------------------------------------ packed streaming batches
@pytest.mark.parametrize("chunk_frames", [0, 7, 50])
def test_streamed_videos_packed_batches(ctx, dev, chunk_frames):
    """Host and callback videos of mixed resolutions go through the staging
    buffers as packed batches (several videos' chunks per K1 launch, one
    segment each): every frame's histogram, L1 and every video's cuts equal
    the oracle's, for chunk sizes that pack whole videos (0), many small pieces
    (7) and pieces straddling batch boundaries (50)."""
    vids = [manifest.subsample(v, 31 + 17 * k) for k, v in enumerate(manifest.c5_videos()[:6])]
    tables = {i: torch_dev.frame_table(v, dev) for i, v in enumerate(vids)}
    hosts = [synth.gen_frames(v) for v in vids]
    items, refs = [], []
    for i, v in enumerate(vids):
        e_host = synth.gen_emb(v)
        items.append({"n": v.n, "H": v.H, "W": v.W, "frames": hosts[i] if i % 3 == 2 else None,
                      "id": i, "emb": torch.from_numpy(e_host).to(dev)})
        refs.append(oracle.run_video(hosts[i], e_host))

    def fill(vi, t0, n, dst, stream):
        v = vids[vi]
        return synth.dev_lib().synth_dev_gen_frames(v.seed, v.id, v.W, v.H, t0, n,
                                                   tables[vi].data_ptr(), dst, stream)

    F = sum(v.n for v in vids)
    hist = torch.empty((F, 162), dtype=torch.int32, device=dev)
    l1 = torch.empty(F, dtype=torch.int32, device=dev)
    before = ctx.stats()["k1_launches"]
    res = ctx.run_videos(items, fill=fill, chunk_frames=chunk_frames, hist=hist, l1=l1,
                         want_cos=True)
    launches = ctx.stats()["k1_launches"] - before
    h, l = _u32(hist), _u32(l1)
    f0 = 0
    for r, ref, v in zip(res, refs, vids):
        assert np.array_equal(h[f0:f0 + v.n], ref.hist)
        assert np.array_equal(l[f0:f0 + v.n], ref.l1)
        assert list(r.detected) == list(ref.detected)
        assert list(r.final) == list(ref.final)
        np.testing.assert_allclose(r.detected_cos, ref.cos, rtol=COS_RTOL, atol=1e-12)
        f0 += v.n
    pieces = sum(-(-v.n // (chunk_frames or v.n + 1)) for v in vids)
    assert launches < pieces or chunk_frames == 0, (launches, pieces)  # chunks were packed


def test_k1_every_colour_frame(dev):
    """One 4096 x 4096 frame holding each of the 2^24 colours once, through K1's
    fast path: the histogram equals the oracle's bin table counted per bin —
    every code, table entry, bank hash and the frame flush exercised at once."""
    from paper_2503_12964_b200 import Ctx
    c = Ctx(device=0)
    col = torch.arange(1 << 24, dtype=torch.int32, device=dev)
    frame = torch.stack([(col >> 16) & 255, (col >> 8) & 255, col & 255], dim=-1)
    frame = frame.to(torch.uint8).reshape(1, 4096, 4096, 3)
    hist, _, _ = c.frame_scores(frame)
    want = np.bincount(oracle.bin_table(), minlength=162).astype(np.uint32)
    assert np.array_equal(_u32(hist)[0], want)
    c.close()


# ------------------------------------------------------------------ K3 at scale
def _walk_embeddings(n_clips, frames_per_clip, dim, seed, step_deg):
    """Clip k's frames share the unit vector at angle phi_k, phi a random walk
    with steps uniform in [-step_deg, step_deg]: adjacent cosines straddle
    theta = 0.9 (25.8 degrees), so merges cascade over several rounds."""
    rng = np.random.default_rng(seed)
    phi = np.cumsum(rng.uniform(-step_deg, step_deg, n_clips)) * np.pi / 180
    e = np.zeros((n_clips * frames_per_clip, dim), dtype=np.float32)
    v = np.stack([np.cos(phi), np.sin(phi)], axis=1).astype(np.float32)
    e[:, :2] = np.repeat(v, frames_per_clip, axis=0)
    cuts = [frames_per_clip * (k + 1) for k in range(n_clips - 1)]
    return e, cuts


@pytest.mark.parametrize("n_clips,step", [(2000, 40.0), (20001, 45.0)])
def test_merge_many_cuts_multi_round(ctx, dev, n_clips, step):
    """Thousands of boundaries merging over several rounds (the device-side
    round loop and the incremental range sums) against the oracle: final cuts,
    rounds and band hits exact, cosines within 1e-5."""
    e, cuts = _walk_embeddings(n_clips, 3, 8, n_clips, step)
    ref = oracle.merge(e, cuts)
    m, cos, hits, rounds = ctx.merge(torch.from_numpy(e).to(dev),
                                     torch.tensor(cuts, dtype=torch.int32, device=dev))
    assert ref.rounds >= 3, ref.rounds
    assert list(m.cpu().numpy()) == list(ref.final)
    assert rounds == ref.rounds and hits == ref.n_band_hits
    np.testing.assert_allclose(cos.cpu().numpy(), ref.cos, rtol=COS_RTOL, atol=1e-12)


def test_merge_20k_cuts_near_constant_under_5ms(ctx, dev):
    """A near-constant 768-d video with 20,000 detected cuts (every boundary
    merges): clip_merge (piece sums, clip sums, all rounds on the device,
    final cuts) in < 5 ms, and the oracle's result (one clip)."""
    rng = np.random.default_rng(3)
    n = 2 * 20001
    base = rng.standard_normal(768)
    e = (base[None, :] + 0.01 * rng.standard_normal((n, 768))).astype(np.float32)
    cuts = list(range(2, n, 2))
    assert len(cuts) == 20000
    ed = torch.from_numpy(e).to(dev)
    cd = torch.tensor(cuts, dtype=torch.int32, device=dev)
    times = []
    for _ in range(6):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(ctx.stream)
        m, cos, hits, rounds = ctx.merge(ed, cd)
        t1.record(ctx.stream)
        torch.cuda.synchronize()
        times.append(t0.elapsed_time(t1))
    ref = oracle.merge(e, cuts)
    assert list(m.cpu().numpy()) == list(ref.final) == []
    assert rounds == ref.rounds
    ms = float(np.median(times[1:]))
    print(f"clip_merge 20,000 cuts x 768: {ms:.3f} ms (median of 5)")
    assert ms < 5.0, times


def test_run_videos_at_the_cut_count_bound(ctx, dev):
    """Videos whose colour flips every L_min = 8 frames (a cut at every allowed
    frame: the clip count K reaches the n / L_min bound the host sizes K3's
    scratch and grids with, while K itself exists only on the device) batched
    with a one-frame and a short video; embeddings on a random walk so merges
    cascade over several rounds.  Every list, count and cosine against the
    oracle."""
    rng = np.random.default_rng(2024)
    pal = np.array([[250, 10, 10], [10, 10, 250]], dtype=np.uint8)
    items, refs = [], []
    for n in [400, 301, 1, 64, 1003]:
        host = np.ascontiguousarray(np.broadcast_to(
            pal[(np.arange(n) // 8) % 2][:, None, None, :], (n, 16, 16, 3)))
        phi = np.cumsum(rng.uniform(-40.0, 40.0, n // 8 + 1)) * np.pi / 180
        e = np.zeros((n, 8), dtype=np.float32)
        e[:, 0] = np.cos(phi[np.arange(n) // 8])
        e[:, 1] = np.sin(phi[np.arange(n) // 8])
        items.append({"n": n, "H": 16, "W": 16, "frames": torch.from_numpy(host).to(dev),
                      "emb": torch.from_numpy(e).to(dev)})
        refs.append(oracle.run_video(host, e))
    res = ctx.run_videos(items, want_cos=True)
    assert any(ref.rounds >= 3 for ref in refs)
    for n, r, ref in zip([400, 301, 1, 64, 1003], res, refs):
        c = (n - 1) // 8  # a candidate every 8 frames; the tail rule drops a last clip < 8
        assert len(ref.detected) == c - (1 if c > 0 and n - 8 * c < 8 else 0)
        assert list(r.detected) == list(ref.detected)
        assert list(r.final) == list(ref.final)
        assert r.rounds == ref.rounds and r.n_band_hits == ref.n_band_hits
        np.testing.assert_allclose(r.detected_cos, ref.cos, rtol=COS_RTOL, atol=1e-12)


def test_run_videos_thousands_of_tiny_videos(ctx, dev):
    """3,000 device-resident 16x16 videos in one call: more segment descriptors
    than the pinned upload buffer holds (the plain-copy fallback), and the
    device-side video-table and summary scans over several 1,024-video blocks.
    Every video's lists against the oracle."""
    rng = np.random.default_rng(9)
    n_vid, n = 3000, 24
    pal = rng.integers(0, 256, size=(n_vid, 3, 3), dtype=np.uint8)
    change = rng.integers(8, 17, size=n_vid)
    host = np.empty((n_vid, n, 16, 16, 3), dtype=np.uint8)
    for i in range(n_vid):
        idx = (np.arange(n) >= change[i]).astype(int) + (np.arange(n) >= change[i] + 8).astype(int)
        host[i] = pal[i][idx][:, None, None, :]
    emb = rng.standard_normal((n_vid, n, 8)).astype(np.float32)
    fr = torch.from_numpy(host).to(dev)
    ed = torch.from_numpy(emb).to(dev)
    items = [{"n": n, "H": 16, "W": 16, "frames": fr[i], "emb": ed[i], "id": i} for i in range(n_vid)]
    res = ctx.run_videos(items, want_cos=True)
    for i in range(0, n_vid, 7):
        ref = oracle.run_video(host[i], emb[i])
        assert list(res[i].detected) == list(ref.detected), i
        assert list(res[i].final) == list(ref.final), i
    assert sum(len(r.detected) for r in res) > 0


def test_run_videos_every_frame_a_candidate(ctx, dev):
    """Colours alternating every frame: every frame t >= 1 is a candidate, so
    every 128-frame compaction chunk is full (K2's greedy takes its per-chunk
    path, not the four-candidate prefetch) and the greedy keeps every L_min-th
    frame: detected = {8, 16, ...} by the closed form, and equal to the oracle,
    for two videos batched with a sparse one."""
    pal = np.array([[250, 10, 10], [10, 10, 250]], dtype=np.uint8)
    items, refs, ns = [], [], [1000, 259, 333]
    rng = np.random.default_rng(5)
    for vi, n in enumerate(ns):
        idx = np.arange(n) % 2 if vi != 1 else (np.arange(n) // 37) % 2
        host = np.ascontiguousarray(np.broadcast_to(pal[idx][:, None, None, :], (n, 16, 16, 3)))
        e = rng.standard_normal((n, 8)).astype(np.float32)
        items.append({"n": n, "H": 16, "W": 16, "frames": torch.from_numpy(host).to(dev),
                      "emb": torch.from_numpy(e).to(dev)})
        refs.append(oracle.run_video(host, e))
    res = ctx.run_videos(items, want_cos=True)
    for n, r, ref in zip(ns, res, refs):
        assert list(r.detected) == list(ref.detected)
        assert list(r.final) == list(ref.final)
        assert r.n_candidates == ref.n_candidates
    last = (1000 - 1) // 8 * 8
    want = list(range(8, last + 1, 8))
    if 1000 - want[-1] < 8:
        want = want[:-1]
    assert list(res[0].detected) == want
