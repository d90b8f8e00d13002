#!/usr/bin/env python3
"""Device frame generator throughput and the streamed clip_run_videos path on
C3 videos: generator alone, resident K1..K3, streamed (fill callback) wall."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from synth import manifest, torch_dev  # noqa: E402
from paper_2503_12964_b200 import Ctx  # noqa: E402


def ev_time(fn, reps=3):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    nv = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    dev = torch.device("cuda:0")
    vids = manifest.c3_videos()[:nv]
    tables = [torch_dev.frame_table(v, dev) for v in vids]
    v = vids[0]
    buf = torch.empty((600, v.H, v.W, 3), dtype=torch.uint8, device=dev)
    g_ms = ev_time(lambda: torch_dev.gen_frames(v, tables[0], buf, t0=0, n=600))
    out = {"gen_600_1080p_ms": round(g_ms, 3), "gen_gbs": round(buf.numel() / g_ms / 1e6, 1)}
    embs = []
    for v, t in zip(vids, tables):
        e = torch.empty((v.n, manifest.EMB_DIM), dtype=torch.float32, device=dev)
        torch_dev.gen_emb(v, t, e)
        embs.append(e)
    ctx = Ctx(device=0, timing=True)

    def fill(vi, t0, n, dst, stream):
        w = vids[vi]
        return synth.dev_lib().synth_dev_gen_frames(w.seed, w.id, w.W, w.H, t0, n,
                                                    tables[vi].data_ptr(), dst, stream)
    items = [{"n": v.n, "H": v.H, "W": v.W, "frames": None, "emb": e, "id": v.id}
             for v, e in zip(vids, embs)]
    ctx.stats(reset=True)
    s_ms = ev_time(lambda: ctx.run_videos(items, fill=fill), reps=2)
    st = ctx.stats(reset=True)
    frames = sum(v.n for v in vids)
    out.update({"videos": nv, "frames": frames, "streamed_wall_ms": round(s_ms, 2),
                "streamed_k1_ms": round(st["k1_ms"] / 3, 2)})
    # resident: one video at a time (HBM)
    r_ms = 0.0
    for v, t, e in zip(vids, tables, embs):
        f = torch.empty((v.n, v.H, v.W, 3), dtype=torch.uint8, device=dev)
        torch_dev.gen_frames(v, t, f)
        it = [{"n": v.n, "H": v.H, "W": v.W, "frames": f, "emb": e, "id": v.id}]
        r_ms += ev_time(lambda: ctx.run_videos(it), reps=2)
        del f
        torch.cuda.empty_cache()
    out["resident_wall_ms"] = round(r_ms, 2)
    out["gen_alone_est_ms"] = round(g_ms * frames / 600, 2)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
