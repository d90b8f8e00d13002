"""The seeded input generator: memoised host loops equal the uncached
definition, manifests are deterministic and shaped like BASELINE.json's configs."""
import numpy as np

import synth
from synth import manifest


def test_memoised_frames_equal_uncached_pixels():
    rng = np.random.default_rng(1)
    for v in [manifest.c1_video(), manifest.subsample(manifest.c5_videos()[0], 30)]:
        fr = synth.gen_frames(v, nthreads=2)
        for _ in range(1500):
            t, x, y = int(rng.integers(v.n)), int(rng.integers(v.W)), int(rng.integers(v.H))
            assert tuple(int(c) for c in fr[t, y, x]) == synth.pixel_ref(v, t, x, y)


def test_partial_generation_matches_full():
    v = manifest.c1_video()
    full = synth.gen_frames(v)
    part = synth.gen_frames(v, t0=17, n=9)
    assert np.array_equal(full[17:26], part)
    e = synth.gen_emb(v)
    assert np.array_equal(e[5:9], synth.gen_emb(v, t0=5, n=4))


def test_embeddings_are_exact_dyadic():
    v = manifest.c1_video()
    e = synth.gen_emb(v)
    scaled = e.astype(np.float64) * 2.0 ** 20
    assert np.array_equal(scaled, np.round(scaled))
    assert np.abs(e).max() < 1.07


def test_frame_hash_sensitive():
    v = manifest.c1_video()
    f = synth.gen_frames(v, n=1)[0]
    h = synth.frame_hash(f)
    g = f.copy()
    g[5, 7, 1] ^= 1
    assert synth.frame_hash(g) != h
    assert synth.frame_hash(f) == h


def test_manifest_shapes():
    v2 = manifest.c2_video()
    assert (v2.W, v2.H, v2.n) == (1280, 720, 18000)
    assert 100 < len(v2.hard) < 220 and len(v2.false) > 0
    c3 = manifest.c3_videos()
    assert len(c3) == 64 and all((v.W, v.H, v.n) == (1920, 1080, 1800) for v in c3)
    c4 = manifest.c4_videos()
    assert len(c4) == 16 and all((v.W, v.H, v.n) == (3840, 2160, 3600) for v in c4)
    shapes = manifest.c5_shapes()
    assert len(shapes) == 1000
    assert all(60 <= n <= 900 for _, _, n in shapes)
    assert all((W * H) % 16 == 0 for W, H, _ in shapes)
    # deterministic
    assert manifest.c5_shapes() == shapes
    assert np.array_equal(manifest.c2_video().frames, v2.frames)
