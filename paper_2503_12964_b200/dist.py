"""Multi-GPU plumbing: whole-video sharding and the one result gather.

Videos are independent units of the path (the split and the merge never cross
videos, §2.1), so a batch shards by whole videos with no
data-path collective.  Every rank computes the same longest-processing-time
(LPT) assignment from the manifest; after each rank's clip_run_videos call the
per-video cut lists are gathered to rank 0 with ONE collective
(all_gather_into_tensor: a single native ncclAllGather over NVLink with the
NCCL backend; gloo in the CPU tests).  Host-side bookkeeping only — no step of
the method runs here.
"""
from __future__ import annotations

import numpy as np

HEADER = 6  # per video: id, n_candidates, n_detected, n_final, n_band_hits, rounds


def lpt_assign(costs, world: int) -> list:
    """Assign items (cost = frames*H*W) to ranks: sort by cost descending
    (ties by index), give each to the least-loaded rank (ties: lowest rank).
    Returns, per rank, its item indices in ascending order."""
    order = sorted(range(len(costs)), key=lambda i: (-int(costs[i]), i))
    load = [0] * world
    out = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        load[r] += int(costs[i])
        out[r].append(i)
    return [sorted(x) for x in out]


def capacity_ints(n_frames_list, l_min: int) -> int:
    """int32 words needed to pack the results of videos with these lengths."""
    return 1 + sum(HEADER + 2 * (n // l_min + 1) for n in n_frames_list)


def pack_results(results, capacity: int) -> np.ndarray:
    """[count, then per video: header, detected..., final...] as int32[capacity]."""
    buf = np.zeros(capacity, dtype=np.int32)
    buf[0] = len(results)
    p = 1
    for r in results:
        det = np.asarray(r.detected, dtype=np.int32)
        fin = np.asarray(r.final, dtype=np.int32)
        need = HEADER + det.size + fin.size
        if p + need > capacity:
            raise ValueError("result buffer capacity exceeded")
        buf[p:p + HEADER] = [r.id, r.n_candidates, det.size, fin.size, r.n_band_hits, r.rounds]
        p += HEADER
        buf[p:p + det.size] = det
        p += det.size
        buf[p:p + fin.size] = fin
        p += fin.size
    return buf


def unpack_results(buf: np.ndarray) -> list:
    """Inverse of pack_results: list of dicts."""
    out = []
    n = int(buf[0])
    p = 1
    for _ in range(n):
        vid, ncand, nd, nf, hits, rounds = (int(x) for x in buf[p:p + HEADER])
        p += HEADER
        det = buf[p:p + nd].copy()
        p += nd
        fin = buf[p:p + nf].copy()
        p += nf
        out.append({"id": vid, "n_candidates": ncand, "detected": det, "final": fin,
                    "n_band_hits": hits, "rounds": rounds})
    return out


def gather_results(results, capacity: int, device=None, group=None) -> list | None:
    """One all_gather_into_tensor of every rank's packed results; returns the
    union (sorted by video id) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    local = torch.from_numpy(pack_results(results, capacity))
    if device is not None:
        local = local.to(device)
    out = torch.empty(world * capacity, dtype=torch.int32, device=local.device)
    dist.all_gather_into_tensor(out, local, group=group)
    arr = out.cpu().numpy().reshape(world, capacity)
    allr = []
    for r in range(world):
        allr.extend(unpack_results(arr[r]))
    return sorted(allr, key=lambda d: d["id"])


# ---------------------------------------------------------------- intra-video sharding (NEXT f2)
def frame_shards(n: int, world: int) -> list:
    """Contiguous frame ranges [f0, f1) of one video over `world` ranks."""
    return [(n * r // world, n * (r + 1) // world) for r in range(world)]


def run_video_sharded(ctx, frames, emb, n_total: int, f0: int, group=None, emb_all=None,
                      marks=None, comm=None, out=None):
    """One long video split by frame ranges across the ranks of `group`
    (the context-parallel analogue on the frame axis).

    Every step of the path still runs in libclipdetect kernels; the exchanges are
    NCCL collectives over NVLink:
      1. K1 + L1 on the local shard (clip_frame_scores);
      2. all_gather of each shard's last histogram -> L1 of each shard's first
         frame against its predecessor (clip_frame_scores on that one frame
         with prev_hist);
      3. all_gather of the L1 arrays -> every rank runs clip_cuts on the whole
         video's L1 (identical detected cuts everywhere);
      4. all_gather of the embeddings -> clip_merge on the whole video.
    Results are identical to the single-GPU path (same kernels, same order).
    `frames`: u8 cuda [m, H, W, 3] (or NV12 [m, H*3/2, W]) = frames f0..f0+m-1;
    `emb`: f32 cuda [m, D].
    `marks`: optional list; CUDA events recorded after each phase are appended
    (diagnosis of the exchange overhead).
    `comm`: the collective provider (default torch.distributed; the GPU tests
    pass an in-process one so that several virtual ranks share one GPU).
    `out`: optional dict; receives this shard's histograms ("hist") and the
    whole video's L1 ("l1").
    Returns (detected list, final list, cos tensor, band hits, rounds)."""
    import torch
    if comm is None:
        import torch.distributed as comm
    dist = comm
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nv12 = frames.dim() == 3  # NV12 surfaces [m, H*3/2, W] (NEXT f1)
    if nv12:
        m, H3, W = frames.shape
        H = H3 * 2 // 3
    else:
        m, H, W, _ = frames.shape
    dev = frames.device
    shards = frame_shards(n_total, world)
    width = max(b - a for a, b in shards)
    # (4, issued first) the embeddings do not depend on the scan: their
    # all-gather runs on NCCL's stream while K1 scans the shard
    e_work = None
    if emb_all is None:
        D = emb.shape[1]
        epad = torch.zeros((width, D), dtype=emb.dtype, device=dev)
        epad[:m].copy_(emb)
        e_all = torch.empty(world * width * D, dtype=emb.dtype, device=dev)
        e_work = dist.all_gather_into_tensor(e_all, epad.view(-1), group=group, async_op=True)
    def mark():
        if marks is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(torch.cuda.current_stream(dev))
            marks.append(ev)

    mark()
    scores = ctx.frame_scores_nv12 if nv12 else ctx.frame_scores
    hist, l1, _ = scores(frames, want_score=False)
    mark()
    nb = hist.shape[1]
    # (2) last histograms of every shard; the seam frame's L1 from histograms (K2 only)
    lasts = torch.empty(world * nb, dtype=hist.dtype, device=dev)
    dist.all_gather_into_tensor(lasts, hist[m - 1].contiguous(), group=group)
    lasts = lasts.view(world, nb)
    if rank > 0:
        ctx.hist_scores(hist[:1], H * W, prev_hist=lasts[rank - 1].contiguous(), l1=l1[:1])
    mark()
    # (3) whole-video L1 on every rank; shards are padded to a common length
    pad = torch.zeros(width, dtype=l1.dtype, device=dev)
    pad[:m].copy_(l1)
    l1_all = torch.empty(world * width, dtype=l1.dtype, device=dev)
    dist.all_gather_into_tensor(l1_all, pad, group=group)
    l1_full = torch.cat([l1_all[r * width:r * width + (b - a)] for r, (a, b) in enumerate(shards)])
    state = torch.zeros(4, dtype=torch.int64, device=dev)
    cuts = torch.empty(n_total // ctx.params.min_clip_frames + 2, dtype=torch.int32, device=dev)
    ctx.cuts(l1_full, H * W, state, cuts, True)
    n_cuts = int(state[3].item())
    mark()
    # (4) embeddings of the whole video, then the merge
    if emb_all is None:
        e_work.wait()
        e_all = e_all.view(world * width, D)
        emb_all = torch.cat([e_all[r * width:r * width + (b - a)] for r, (a, b) in enumerate(shards)])
    mark()
    merged, cos, hits, rounds = ctx.merge(emb_all, cuts[:max(1, n_cuts)].contiguous(), n_cuts=n_cuts)
    mark()
    if out is not None:
        out["hist"], out["l1"] = hist, l1_full
    return (cuts[:n_cuts].cpu().tolist(), merged.cpu().tolist(), cos, hits, rounds)
