"""N>1 host-side path on CPU: LPT whole-video sharding and the single result
gather, with torch.distributed gloo at world_size 2 (and 4)."""
import os
import socket
from dataclasses import dataclass

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2503_12964_b200 import dist as cdist
from synth import manifest


@dataclass
class FakeResult:
    id: int
    n_candidates: int
    detected: np.ndarray
    final: np.ndarray
    n_band_hits: int
    rounds: int


def _fake(vid, n):
    rng = np.random.default_rng(vid)
    det = np.unique(rng.integers(8, max(9, n - 8), size=int(rng.integers(0, 12)))).astype(np.int32)
    fin = det[::2].copy()
    return FakeResult(vid, int(det.size + 3), det, fin, 0, 2)


def test_lpt_balances_and_is_deterministic():
    shapes = manifest.c5_shapes()
    costs = [W * H * n for W, H, n in shapes]
    for world in [1, 2, 4, 8]:
        a = cdist.lpt_assign(costs, world)
        assert sorted(i for r in a for i in r) == list(range(len(costs)))
        loads = [sum(costs[i] for i in r) for r in a]
        assert max(loads) / (sum(loads) / world) < 1.01  # LPT on 1000 items: near perfect
        assert a == cdist.lpt_assign(costs, world)
    # C3: 64 equal videos split into equal contiguous-size blocks
    a = cdist.lpt_assign([1920 * 1080 * 1800] * 64, 8)
    assert all(len(r) == 8 for r in a)


def test_pack_roundtrip():
    res = [_fake(v, 300) for v in range(7)]
    cap = cdist.capacity_ints([300] * 7, 8)
    back = cdist.unpack_results(cdist.pack_results(res, cap))
    for r, b in zip(res, back):
        assert b["id"] == r.id and list(b["detected"]) == list(r.detected)
        assert list(b["final"]) == list(r.final) and b["rounds"] == 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nvid, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lengths = [200 + 37 * v for v in range(nvid)]
    assign = cdist.lpt_assign([n * 100 for n in lengths], world)
    mine = [_fake(v, lengths[v]) for v in assign[rank]]
    cap = cdist.capacity_ints(lengths, 8)  # every rank uses the same capacity
    allr = cdist.gather_results(mine, cap)
    if rank == 0:
        q.put([(d["id"], list(map(int, d["detected"])), list(map(int, d["final"]))) for d in allr])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gather_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    nvid = 11
    procs = [ctx.Process(target=_worker, args=(r, world, port, nvid, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    lengths = [200 + 37 * v for v in range(nvid)]
    want = [(v, list(map(int, _fake(v, lengths[v]).detected)), list(map(int, _fake(v, lengths[v]).final)))
            for v in range(nvid)]
    assert got == want


# ---------------------------------------------------------------- intra-video sharding (f2)
class _OracleCtx:
    """CPU stand-in for the Ctx binding (oracle-backed) so that the sharded
    orchestration and its collectives can run under gloo without a GPU."""

    class _P:
        min_clip_frames = 8

    params = _P()

    def frame_scores(self, frames, prev_hist=None, want_score=True):
        import oracle
        import torch
        f = frames.numpy()
        h = oracle.hist_frames(f)
        npix = f[0].size // 3
        if prev_hist is not None:
            hh = np.concatenate([prev_hist.numpy().view(np.uint32)[None], h])
            l1, _ = oracle.l1(hh, npix)
            l1 = l1[1:]
        else:
            l1, _ = oracle.l1(h, npix)
        return (torch.from_numpy(h.view(np.int32).copy()), torch.from_numpy(l1.view(np.int32).copy()), None)

    def hist_scores(self, hist, npix, prev_hist=None, l1=None):
        import oracle
        import torch
        h = hist.numpy().view(np.uint32)
        if prev_hist is not None:
            h = np.concatenate([prev_hist.numpy().view(np.uint32)[None], h])
        v, _ = oracle.l1(h, npix)
        if prev_hist is not None:
            v = v[1:]
        l1.copy_(torch.from_numpy(v.view(np.int32).copy()))
        return l1, None

    def cuts(self, l1, npix, state, cuts, is_final):
        import oracle
        a = l1.numpy().view(np.uint32)
        det = oracle.min_length(oracle.candidates(a, npix), a.size, 8)
        cuts[:det.size] = __import__("torch").from_numpy(det.astype(np.int32))
        state[3] = det.size

    def merge(self, emb, cuts, n_cuts):
        import oracle
        import torch
        r = oracle.merge(emb.numpy(), cuts.numpy()[:n_cuts].astype(np.int64))
        return torch.from_numpy(r.final.astype(np.int32)), torch.from_numpy(r.cos), r.n_band_hits, r.rounds


def _shard_worker(rank, world, port, n, q):
    import torch
    import torch.distributed as dist

    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    v = manifest.subsample(manifest.c2_video(0), n)
    v = manifest.Video(id=0, W=64, H=48, n=n, seed=v.seed, frames=v.frames, hard=v.hard, false=v.false)
    a, b = cdist.frame_shards(n, world)[rank]
    frames = torch.from_numpy(synth.gen_frames(v, t0=a, n=b - a))
    emb = torch.from_numpy(synth.gen_emb(v, t0=a, n=b - a))
    det, fin, cos, hits, rounds = cdist.run_video_sharded(_OracleCtx(), frames, emb, n, a)
    if rank == 0:
        q.put((det, fin, rounds))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_video_equals_whole_video(world):
    import oracle
    import synth
    n = 700
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    det, fin, rounds = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    v = manifest.subsample(manifest.c2_video(0), n)
    v = manifest.Video(id=0, W=64, H=48, n=n, seed=v.seed, frames=v.frames)
    ref = oracle.run_video(synth.gen_frames(v), synth.gen_emb(v))
    assert det == list(ref.detected) and fin == list(ref.final) and rounds == ref.rounds
    assert len(det) > 3  # the split crosses real cuts
