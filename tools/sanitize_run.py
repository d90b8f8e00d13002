#!/usr/bin/env python3
"""Small invocations of every kernel of the path for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): C1 and an N-frame C2 slice
through clip_run_videos (K1, K2, K3) as RGB24 and NV12 (K1-NV12), the
per-step entry points (clip_frame_scores with prev_hist, clip_cuts,
clip_merge, clip_hist_scores), K4 frame sampling (RGB24 and NV12) and a
generic-bins context.  Results are checked against the oracle so a run that
the sanitizer perturbs still has to be correct.

usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [c2_frames]
       python tools/sanitize_run.py [c2_frames] --checked
The pool's compute-sanitizer is closed ("runs under it have left GPUs needing
a reset"), so --checked runs the same workload on the bounds-checked build of
the library (-DCLIPDETECT_CHECKED: every TMA source range, ring hand-off,
shared-memory code offset, code -> bin entry, K3 alive / run / chunk index and
K4 staged row is checked on the device; a failure prints the condition and
traps, which fails the call).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from synth import manifest  # noqa: E402
from paper_2503_12964_b200 import Ctx, default_params  # noqa: E402
from paper_2503_12964_b200 import _build, clipdetect  # noqa: E402
from paper_2503_12964_b200.clipdetect import FORMAT_NV12  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n_c2 = int(args[0]) if args else 200
    if "--checked" in sys.argv:
        import glob
        import re
        lib = _build.build(checked=True)
        clipdetect.load(path=lib)
        sites = sum(len(re.findall(r"\bCD_CHECK\(", open(f).read()))
                    for f in glob.glob(os.path.join(ROOT, "paper_2503_12964_b200", "csrc", "*.cu")))
        print(f"checked build {lib}: {sites} CD_CHECK sites compiled in")
    dev = torch.device("cuda:0")
    ctx = Ctx(device=0)
    vids = [manifest.c1_video(), manifest.subsample(manifest.c2_video(0), n_c2)]
    for v in vids:
        host = synth.gen_frames(v)
        emb = synth.gen_emb(v)
        ref = oracle.run_video(host, emb)
        fr = torch.from_numpy(host).to(dev)
        ed = torch.from_numpy(emb).to(dev)
        r = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": fr, "emb": ed}], want_cos=True)[0]
        assert list(r.detected) == list(ref.detected) and list(r.final) == list(ref.final), v.id
        # per-step entry points, two chunks with prev_hist
        h = v.n // 2
        h1, l1a, _ = ctx.frame_scores(fr[:h].contiguous())
        h2, l1b, _ = ctx.frame_scores(fr[h:].contiguous(), prev_hist=h1[-1].contiguous())
        l1 = torch.cat([l1a, l1b])
        assert np.array_equal(l1.cpu().numpy().view(np.uint32), ref.l1)
        ctx.hist_scores(h2, v.W * v.H, prev_hist=h1[-1].contiguous(), l1=l1b)
        state = torch.zeros(4, dtype=torch.int64, device=dev)
        cuts = torch.empty(v.n // 8 + 2, dtype=torch.int32, device=dev)
        ctx.cuts(l1, v.W * v.H, state, cuts, True)
        nc = int(state[3].item())
        m, cos, hits, rounds = ctx.merge(ed, cuts[:max(1, nc)].contiguous(), n_cuts=nc)
        assert list(m.cpu().numpy()) == list(ref.final)
        # K4 sampling of the final clips
        fc = torch.from_numpy(np.asarray(ref.final, dtype=np.int32)).to(dev)
        out, idx = ctx.sample_frames(fr, fc, 4, 64, 64)
        so, si = oracle.sample_clips(host, list(ref.final), 4, 64, 64)
        assert np.array_equal(out.cpu().numpy(), so)
        # NV12 surfaces of the same video through K1-NV12
        nv = synth.gen_nv12(v)
        rn = oracle.run_video_nv12(nv, emb)
        r2 = ctx.run_videos([{"n": v.n, "H": v.H, "W": v.W, "frames": torch.from_numpy(nv).to(dev),
                              "emb": ed, "format": FORMAT_NV12}])[0]
        assert list(r2.final) == list(rn.final)
        ctx.sample_frames(torch.from_numpy(nv).to(dev), fc, 2, 32, 48)
    # generic bins (K1 kModeGeneric, K1-NV12 generic kernel)
    g = Ctx(default_params(h_bins=12, s_bins=4, v_bins=4), device=0)
    host = synth.gen_frames(vids[0])
    hist, _, _ = g.frame_scores(torch.from_numpy(host).to(dev))
    assert np.array_equal(hist.cpu().numpy().view(np.uint32),
                          oracle.hist_frames(host, oracle.Params(nh=12, ns=4, nv=4)))
    g.frame_scores_nv12(torch.from_numpy(synth.gen_nv12(vids[0])).to(dev))
    torch.cuda.synchronize()
    g.close()
    ctx.close()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
