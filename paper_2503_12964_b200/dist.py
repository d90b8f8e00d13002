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
