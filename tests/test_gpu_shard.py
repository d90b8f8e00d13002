"""GPU parity of NEXT f2: one long video split by frame ranges (the
context-parallel analogue on the frame axis, §4.4, SURVEY.md
§8(f) f2).  The real orchestration (paper_2503_12964_b200/dist.py
run_video_sharded) runs on real kernels: R virtual ranks are threads of one
process on one GPU, each with its own libclipdetect context and CUDA stream,
joined by an in-process all-gather (ThreadComm) in place of NCCL.  The seam
step (clip_hist_scores with prev_hist), the whole-video clip_cuts over the
gathered L1 and clip_merge over the gathered embeddings are exactly the calls
an N-GPU run makes.  Results must equal the oracle's goldens bit for bit
(histogram and L1 digests, detected and final cuts) and the cosines within 1e-5.
"""
import hashlib
import json
import os
import threading

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


class ThreadComm:
    """all_gather_into_tensor among `world` threads of one process (one GPU)."""

    class _Rank:
        def __init__(self, shared, rank):
            self.s, self.rank = shared, rank

        def get_world_size(self, group=None):
            return self.s.world

        def get_rank(self, group=None):
            return self.rank

        def all_gather_into_tensor(self, out, inp, group=None, async_op=False):
            s = self.s
            torch.cuda.current_stream().synchronize()  # inp complete before others read it
            s.slots[self.rank] = inp
            s.bar.wait()
            o = out.view(s.world, -1)
            for r in range(s.world):
                o[r].copy_(s.slots[r].view(-1))
            torch.cuda.current_stream().synchronize()
            s.bar.wait()  # nobody overwrites a slot before every rank has read it

            class _Done:
                def wait(self):
                    return None
            return _Done() if async_op else None

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world

    def rank(self, r):
        return ThreadComm._Rank(self, r)


def _sharded(frames, emb, world, nv12=False):
    """Run run_video_sharded on `world` virtual ranks; returns rank 0's result,
    the concatenated histograms and the whole-video L1."""
    from paper_2503_12964_b200 import Ctx
    from paper_2503_12964_b200 import dist as cdist
    torch.cuda.synchronize()  # inputs were made on the default stream; the ranks use their own
    n = frames.shape[0]
    shards = cdist.frame_shards(n, world)
    comm = ThreadComm(world)
    results, outs, errors = [None] * world, [dict() for _ in range(world)], []

    def work(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = Ctx(device=0, stream=s)
                a, b = shards[r]
                results[r] = cdist.run_video_sharded(ctx, frames[a:b], emb[a:b], n, a,
                                                     comm=comm.rank(r), out=outs[r])
                s.synchronize()
                ctx.close()
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            comm.bar.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    hist = torch.cat([o["hist"] for o in outs]).cpu().numpy().view(np.uint32)
    l1 = outs[0]["l1"].cpu().numpy().view(np.uint32)
    for o in outs[1:]:  # every rank holds the same whole-video L1
        assert np.array_equal(o["l1"].cpu().numpy().view(np.uint32), l1)
    for r in results[1:]:
        assert r[0] == results[0][0] and r[1] == results[0][1]
    return results[0], hist, l1


def _golden(name):
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    with open(path) as f:
        return json.load(f)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _dev_video(v, dev):
    table = torch_dev.frame_table(v, dev)
    frames = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    torch_dev.gen_frames(v, table, frames)
    emb = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
    torch_dev.gen_emb(v, table, emb)
    return frames, emb


@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_c2_prefix_vs_oracle(dev, world):
    """2,000 C2 frames (720p, random cuts): every seam L1, cut and cosine vs the oracle."""
    v = manifest.subsample(manifest.c2_video(0), 2000)
    frames, emb = _dev_video(v, dev)
    (det, fin, cos, hits, rounds), hist, l1 = _sharded(frames, emb, world)
    ref = oracle.run_video(synth.gen_frames(v), synth.gen_emb(v))
    assert np.array_equal(hist, ref.hist) and np.array_equal(l1, ref.l1)
    assert det == list(ref.detected) and fin == list(ref.final)
    assert hits == ref.n_band_hits and rounds == ref.rounds
    np.testing.assert_allclose(cos.cpu().numpy(), ref.cos, rtol=COS_RTOL, atol=1e-12)
    assert len(det) > 5


def test_sharded_c3_video_with_fades_golden(dev):
    """The first C3 video with fades and flashes (1,800 frames 1080p) in 3
    frame shards: the golden's histogram / L1 digests and cuts."""
    v = next(x for x in manifest.c3_videos() if x.fades and x.flashes)
    g = _golden("C3")["videos"][v.id]
    frames, emb = _dev_video(v, dev)
    (det, fin, cos, hits, rounds), hist, l1 = _sharded(frames, emb, 3)
    assert _sha(hist) == g["hist_sha256"] and _sha(l1) == g["l1_sha256"]
    assert det == g["detected"] and fin == g["final"]
    np.testing.assert_allclose(cos.cpu().numpy(), np.array(g["cos"]), rtol=COS_RTOL, atol=1e-12)


def test_sharded_c2_full_golden(dev):
    """The whole C2 video (18,000 x 720p, 49.8 GB) in 4 frame shards, as
    bench.py --shard-frames runs it at 4 GPUs: the C2 golden."""
    g = _golden("C2")["videos"][0]
    v = manifest.c2_video()
    frames, emb = _dev_video(v, dev)
    (det, fin, cos, hits, rounds), hist, l1 = _sharded(frames, emb, 4)
    assert _sha(hist) == g["hist_sha256"] and _sha(l1) == g["l1_sha256"]
    assert det == g["detected"] and fin == g["final"]
    np.testing.assert_allclose(cos.cpu().numpy(), np.array(g["cos"]), rtol=COS_RTOL, atol=1e-12)
    del frames
    torch.cuda.empty_cache()


def test_hist_scores_seam_vs_oracle(dev):
    """clip_hist_scores (the seam entry point) against oracle.l1 on random
    histograms, with and without prev_hist, at several pixel counts."""
    from paper_2503_12964_b200 import Ctx
    ctx = Ctx(device=0)
    rng = np.random.default_rng(7)
    try:
        for npix, n in [(16, 1), (921600, 37), (2073600, 300), (8294400, 5)]:
            h = np.zeros((n + 1, 162), dtype=np.uint32)
            for t in range(n + 1):
                h[t] = rng.multinomial(npix, rng.dirichlet(np.full(162, 0.3)))
            want, want_s = oracle.l1(h, npix)
            hd = torch.from_numpy(h.view(np.int32)).to(dev)
            l1 = torch.empty(n, dtype=torch.int32, device=dev)
            sc = torch.empty(n, dtype=torch.float32, device=dev)
            ctx.hist_scores(hd[1:].contiguous(), npix, prev_hist=hd[0].contiguous(), l1=l1, score=sc)
            torch.cuda.synchronize()
            assert np.array_equal(l1.cpu().numpy().view(np.uint32), want[1:])
            assert np.array_equal(sc.cpu().numpy(), want_s[1:].astype(np.float32))
            ctx.hist_scores(hd[1:].contiguous(), npix, l1=l1, score=sc)  # video start: L1_0 = 0
            w2, _ = oracle.l1(h[1:], npix)
            assert np.array_equal(l1.cpu().numpy().view(np.uint32), w2)
    finally:
        ctx.close()
