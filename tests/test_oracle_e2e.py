"""End-to-end pins of the oracle on planted-truth synthetic videos.

C1 (BASELINE.json configs[0]): 64 frames 320x240, hard cuts at 10, 32, 53, a
false cut (palette rotation) at 21, a 2-frame flash at 43-44.  By construction
(DESIGN.md "Input recipe"): detected = {10, 21, 32, 43, 53} (the flash exit at
45 is 2 < L_min frames after 43 and is suppressed), final = {10, 32, 53} (the
false cut and the flash keep their scene's embedding and merge back).
PAPER.md:35: the split is "aggressive" and "smoothed out" by the merge.
"""
import numpy as np

import oracle
import synth
from synth import manifest


def test_c1_planted_truth():
    v = manifest.c1_video()
    r = oracle.run_video(synth.gen_frames(v), synth.gen_emb(v))
    assert list(r.detected) == [10, 21, 32, 43, 53]
    assert list(r.final) == [10, 32, 53]
    assert r.n_band_hits == 0
    # margins far from both thresholds
    planted = set(v.hard) | set(v.false) | {43, 45}
    for t in range(1, v.n):
        if t in planted:
            assert r.score[t] > 0.8
        else:
            assert r.score[t] < 0.05
    assert np.all(np.abs(r.cos - 0.9) > 0.05)


def test_c2_prefix_planted_cuts_survive():
    v = manifest.subsample(manifest.c2_video(0), 1500)
    r = oracle.run_video(synth.gen_frames(v), synth.gen_emb(v))
    fin = set(int(x) for x in r.final)
    assert set(v.hard) <= fin
    assert not (set(v.false) & fin)
    det = [0] + list(r.detected) + [v.n]
    assert all(b - a >= 8 for a, b in zip(det, det[1:]))


def test_c3_video_with_fades_and_flashes():
    v = manifest.subsample(manifest.c3_videos()[0], 600)
    v = manifest.Video(id=v.id, W=480, H=270, n=v.n, seed=v.seed, frames=v.frames, hard=v.hard,
                       false=v.false, flashes=v.flashes, fades=v.fades)
    r = oracle.run_video(synth.gen_frames(v), synth.gen_emb(v))
    fin = set(int(x) for x in r.final)
    assert set(v.hard) <= fin
    for s, L in v.flashes:  # flashes never survive the merge
        assert not any(s <= c <= s + L for c in fin)
    # every fade leaves at most one cut inside its span (the scene switch)
    for c in v.fades:
        inside = [x for x in fin if c - 12 <= x < c + 12]
        assert len(inside) <= 1
