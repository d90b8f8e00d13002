"""GPU band-hit reporting (north star: "any threshold decision made within that
band must be reported"; merge passage PAPER.md:35 §2.1, reading O9): the K3
merge through clip_merge and through clip_run_videos counts the same in-band
cosines as the oracle, on inputs planted inside, outside and on the edges of
the band (tests/band_cases.py; exact cosines known to 50 digits, each >= 3e-7
from every band edge), and its cosines agree within 1e-5 relative."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from band_cases import PAIRS, case_edges, case_hit_that_merges, case_two_rounds  # noqa: E402

pytestmark = pytest.mark.gpu
COS_RTOL = 1e-5


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda:0")


def _ctx(**kw):
    from paper_2503_12964_b200 import Ctx, default_params
    return Ctx(default_params(**kw), device=0)


def _gpu_merge(ctx, e, cuts, dev):
    emb = torch.from_numpy(np.ascontiguousarray(e)).to(dev)
    c = torch.tensor(cuts, dtype=torch.int32, device=dev)
    m, cos, hits, rounds = ctx.merge(emb, c)
    return list(m.cpu().numpy()), cos.cpu().numpy(), hits, rounds


CASES = {"edges": case_edges, "two_rounds": case_two_rounds, "hit_that_merges": case_hit_that_merges}


@pytest.mark.parametrize("name", sorted(CASES))
def test_band_hits_clip_merge(name, dev):
    e, cuts = CASES[name]()
    ref = oracle.merge(e, cuts)
    assert ref.n_band_hits > 0
    ctx = _ctx()
    try:
        final, cos, hits, rounds = _gpu_merge(ctx, e, cuts, dev)
    finally:
        ctx.close()
    assert final == list(ref.final)
    assert hits == ref.n_band_hits and rounds == ref.rounds
    np.testing.assert_allclose(cos, ref.cos, rtol=COS_RTOL, atol=1e-12)


def test_band_hits_scale_with_theta(dev):
    p = oracle.Params(theta=0.5)
    ctx = _ctx(merge_cos_threshold=0.5)
    try:
        for nm, want in [("half_out", 0), ("half_in", 1)]:
            e = np.zeros((2, 4), dtype=np.float32)
            e[0, 0] = 1
            e[1, :2] = PAIRS[nm]
            ref = oracle.merge(e, [1], p)
            final, cos, hits, rounds = _gpu_merge(ctx, e, [1], dev)
            assert hits == ref.n_band_hits == want, nm
            assert final == list(ref.final) and rounds == ref.rounds
    finally:
        ctx.close()


def test_band_hits_run_videos(dev):
    """The three planted cases as one batch of videos through clip_run_videos
    (merge on supplied cuts is not reachable there, so each case's frames are
    built so that K1/K2 detect exactly the planted cuts: a video whose clips
    alternate between two flat colours with every clip >= L_min frames)."""
    rows = []
    for name in sorted(CASES):
        e, cuts = CASES[name]()
        L = 8  # min_clip_frames default; stretch each clip to 8 frames
        n_clips = len(cuts) + 1
        n = L * n_clips
        emb = np.zeros((n, 16), dtype=np.float32)  # one dim for the whole batch
        bounds = [0] + list(cuts) + [e.shape[0]]
        for k in range(n_clips):
            emb[L * k:L * (k + 1), :e.shape[1]] = e[bounds[k]]  # every frame of clip k: its planted vector
        frames = np.zeros((n, 16, 16, 3), dtype=np.uint8)
        for k in range(n_clips):
            frames[L * k:L * (k + 1)] = (255, 0, 0) if k % 2 == 0 else (0, 0, 255)
        rows.append((frames, emb, [L * (k + 1) for k in range(n_clips - 1)]))
    ctx = _ctx()
    try:
        vids = [{"n": f.shape[0], "H": 16, "W": 16, "frames": torch.from_numpy(f).to(dev),
                 "emb": torch.from_numpy(em).to(dev)} for f, em, _ in rows]
        res = ctx.run_videos(vids, want_cos=True)
    finally:
        ctx.close()
    for (f, em, det), r in zip(rows, res):
        ref = oracle.run_video(f, em)
        assert list(r.detected) == det == list(ref.detected)
        assert list(r.final) == list(ref.final)
        assert r.n_band_hits == ref.n_band_hits > 0 and r.rounds == ref.rounds
        np.testing.assert_allclose(r.detected_cos, ref.cos, rtol=COS_RTOL, atol=1e-12)
