/*
 * synth.h — the seeded synthetic-input generator shared by both sides of the
 * parity check (the CPU oracle's driver and the CUDA bench/tests).
 *
 * This module holds NONE of the method's arithmetic (no HSV, no histogram, no
 * distance, no threshold, no merge).  It only defines, as pure integer
 * functions of (seed, video, frame, y, x, d), the decoded RGB24 frames and the
 * per-frame f32 image embeddings that the paper's clipping pipeline consumes
 * (§2.1 "Clipping Pipeline": raw videos in, split by colour
 * change, merged by image-embedding similarity).  Frames and embeddings are
 * synthetic because the paper's datasets/models are out of scope; the recipe
 * (scenes, hard cuts, false cuts, flashes, fades) is DESIGN.md §"Input recipe"
 * (PROPOSED).
 *
 * Everything is integer arithmetic, so the host (oracle side) and the device
 * (CUDA side) produce bit-identical bytes; the embedding value is an exact f32
 * (|u*32+n| < 2^21 scaled by 2^-20), also bit-identical.
 *
 * Frame record (one per frame, built from the event manifest by synth/manifest.py):
 *   scene  : scene id (selects palette, texture and embedding direction)
 *   mode   : 0 normal, 1/2 palette rotated by 120/240 degrees ("false cut"),
 *            3 flash (near white), 4 uniform-noise stress frame
 *   fade_w : 256 = no fade, else channel weight w in (p*w+128)>>8
 */
#ifndef SYNTH_H_
#define SYNTH_H_

#include <stdint.h>

#if defined(__CUDACC__)
#define SYNTH_HD __host__ __device__ __forceinline__
#else
#define SYNTH_HD static inline
#endif

#define SYNTH_MODE_NORMAL 0u
#define SYNTH_MODE_ROT1 1u
#define SYNTH_MODE_ROT2 2u
#define SYNTH_MODE_FLASH 3u
#define SYNTH_MODE_NOISE 4u

#define SYNTH_TAG_TEX 0xC0FFEEull
#define SYNTH_TAG_NOISE 0x5EED0001ull
#define SYNTH_TAG_EMB 0xE3BE0001ull
#define SYNTH_TAG_EMBN 0xE3BE0002ull

typedef struct {
  uint32_t scene;
  uint16_t mode;
  uint16_t fade_w;
} synth_frame; /* 8 bytes */

/* SplitMix64 finaliser step (SPEC.md:26-28 idea: counter-based, identical on
 * every platform). */
SYNTH_HD uint64_t synth_mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* 32-bit avalanche ("lowbias32"). */
SYNTH_HD uint32_t synth_hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7FEB352Du;
  x ^= x >> 15;
  x *= 0x846CA68Bu;
  x ^= x >> 16;
  return x;
}

/* H(a, b, ...) folds left from k = 0 via k = mix64(k ^ x). */
SYNTH_HD uint64_t synth_h3(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t k = 0;
  k = synth_mix64(k ^ a);
  k = synth_mix64(k ^ b);
  k = synth_mix64(k ^ c);
  return k;
}
SYNTH_HD uint64_t synth_h4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return synth_mix64(synth_h3(a, b, c) ^ d);
}
SYNTH_HD uint64_t synth_h5(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t e) {
  return synth_mix64(synth_h4(a, b, c, d) ^ e);
}
SYNTH_HD uint64_t synth_h6(uint64_t a, uint64_t b, uint64_t c, uint64_t d, uint64_t e,
                           uint64_t f) {
  return synth_mix64(synth_h5(a, b, c, d, e) ^ f);
}

/* Texture cell edge in pixels. */
SYNTH_HD uint32_t synth_cell(uint32_t W) { return (W / 64u) > 8u ? (W / 64u) : 8u; }

/* Palette index (0..7) of texture cell (cx, cy) of a scene. */
SYNTH_HD uint32_t synth_cell_index(uint64_t seed, uint32_t video, uint32_t scene, uint32_t cx,
                                   uint32_t cy) {
  return (uint32_t)(synth_h6(seed, video, scene, SYNTH_TAG_TEX, cx, cy) & 7u);
}

/* Channel c (0=r,1=g,2=b) of palette colour k of a scene. */
SYNTH_HD uint32_t synth_palette(uint64_t seed, uint32_t video, uint32_t scene, uint32_t k,
                                uint32_t c) {
  return (uint32_t)(synth_h5(seed, video, scene, k, c) & 255u);
}

/* Per-frame key of the pixel-noise stream. */
SYNTH_HD uint32_t synth_noise_key(uint64_t seed, uint32_t video, uint32_t t) {
  return (uint32_t)synth_h3(seed ^ SYNTH_TAG_NOISE, video, t);
}

/* Raw 32-bit noise word of pixel index p (= y*W + x) of a frame. */
SYNTH_HD uint32_t synth_noise_word(uint32_t key, uint32_t p) {
  return synth_hash32(key + p * 0x9E3779B9u);
}

/* Noise in [-6, 6]. */
SYNTH_HD int32_t synth_noise(uint32_t word) {
  return (int32_t)((((word >> 16) * 13u) >> 16)) - 6;
}

SYNTH_HD uint32_t synth_clamp255(int32_t v) {
  return (uint32_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
}

/* Finish one pixel given its palette colour (b0,b1,b2) and noise word.
 * Writes r,g,b to out[0..2]. */
SYNTH_HD void synth_finish_pixel(uint32_t b0, uint32_t b1, uint32_t b2, uint32_t word,
                                 uint32_t mode, uint32_t fade_w, uint8_t* out) {
  uint32_t p0, p1, p2;
  int32_t n = synth_noise(word);
  if (mode == SYNTH_MODE_NOISE) {
    /* uniform random colour: K1 stress content (bank-conflict heavy) */
    p0 = word & 255u;
    p1 = (word >> 8) & 255u;
    p2 = (word >> 16) & 255u;
  } else if (mode == SYNTH_MODE_FLASH) {
    uint32_t f = 255u - (uint32_t)(n < 0 ? -n : n);
    p0 = f;
    p1 = f;
    p2 = f;
  } else {
    uint32_t q0 = synth_clamp255((int32_t)b0 + n);
    uint32_t q1 = synth_clamp255((int32_t)b1 + n);
    uint32_t q2 = synth_clamp255((int32_t)b2 + n);
    if (mode == SYNTH_MODE_ROT1) {
      p0 = q2; p1 = q0; p2 = q1;
    } else if (mode == SYNTH_MODE_ROT2) {
      p0 = q1; p1 = q2; p2 = q0;
    } else {
      p0 = q0; p1 = q1; p2 = q2;
    }
  }
  if (fade_w != 256u) {
    p0 = (p0 * fade_w + 128u) >> 8;
    p1 = (p1 * fade_w + 128u) >> 8;
    p2 = (p2 * fade_w + 128u) >> 8;
  }
  out[0] = (uint8_t)p0;
  out[1] = (uint8_t)p1;
  out[2] = (uint8_t)p2;
}

/* One pixel, computed from scratch (no caching).  t = frame index in video. */
SYNTH_HD void synth_pixel(uint64_t seed, uint32_t video, uint32_t t, synth_frame fr,
                          uint32_t W, uint32_t x, uint32_t y, uint8_t* out) {
  uint32_t cell = synth_cell(W);
  uint32_t cx = x / cell + t / 8u;
  uint32_t cy = y / cell;
  uint32_t k = synth_cell_index(seed, video, fr.scene, cx, cy);
  uint32_t b0 = synth_palette(seed, video, fr.scene, k, 0);
  uint32_t b1 = synth_palette(seed, video, fr.scene, k, 1);
  uint32_t b2 = synth_palette(seed, video, fr.scene, k, 2);
  uint32_t word = synth_noise_word(synth_noise_key(seed, video, t), y * W + x);
  synth_finish_pixel(b0, b1, b2, word, fr.mode, fr.fade_w, out);
}

/* ---- embeddings: e[t][d] = (u_scene[d]*32 + n_t[d]) * 2^-20, exact in f32 ---- */
SYNTH_HD int32_t synth_emb_dir(uint64_t seed, uint32_t video, uint32_t scene, uint32_t d) {
  return (int32_t)(synth_h4(seed ^ SYNTH_TAG_EMB, video, scene, d) & 0xFFFFu) - 32768;
}
SYNTH_HD uint32_t synth_emb_key(uint64_t seed, uint32_t video, uint32_t t) {
  return (uint32_t)synth_h3(seed ^ SYNTH_TAG_EMBN, video, t);
}
SYNTH_HD float synth_emb_value(int32_t dir, uint32_t key, uint32_t d) {
  int32_t nz = (int32_t)(synth_hash32(key + d * 0x9E3779B9u) & 0x1FFFFu) - 65536;
  return (float)(dir * 32 + nz) * (1.0f / 1048576.0f);
}

/* ---- frame hash: fh = sum_i mix64(w_i ^ i) mod 2^64 over little-endian u64 words ---- */
SYNTH_HD uint64_t synth_hash_word(uint64_t w, uint64_t i) { return synth_mix64(w ^ i); }


/* ---- NV12 frames (NVDEC's native 4:2:0 output): a scene model in YUV.
 * Y plane [H][W] then interleaved UV plane [H/2][W/2][2] (U then V).
 * Palette colour k of a scene: Y in [16, 235], U, V in [16, 240]; luma noise +-6
 * per pixel, chroma noise +-2 per 2x2 block.  Modes: 1 = chroma swapped (U,V) ->
 * (V,U), 2 = chroma mirrored (256-U, 256-V) (both: "false cut", same scene);
 * 3 = flash (Y = 235 - |noise|, U = V = 128); fade: Y -> 16 + w*(Y-16)/256,
 * U,V -> 128 + w*(U-128)/256 (integer, rounded). */
#define SYNTH_TAG_YUV 0x7A11E001ull

SYNTH_HD uint32_t synth_yuv_palette(uint64_t seed, uint32_t video, uint32_t scene, uint32_t k,
                                    uint32_t c) {
  uint32_t h = (uint32_t)(synth_h5(seed ^ SYNTH_TAG_YUV, video, scene, k, c) & 0xFFFFu);
  return c == 0 ? 16u + h % 220u : 16u + h % 225u;
}

SYNTH_HD uint32_t synth_fade8(uint32_t x, uint32_t center, uint32_t w) {
  /* center + round(w*(x - center)/256), computed on non-negative integers */
  int32_t d = (int32_t)x - (int32_t)center;
  int32_t r = (d * (int32_t)w + 256 * 256 + 128) >> 8;  /* >= 0 for |d| <= 255 */
  return (uint32_t)((int32_t)center + r - 256);
}

/* Luma of pixel (x, y). */
SYNTH_HD uint32_t synth_nv12_y(uint64_t seed, uint32_t video, uint32_t t, synth_frame fr,
                               uint32_t W, uint32_t x, uint32_t y) {
  uint32_t cell = synth_cell(W);
  uint32_t k = synth_cell_index(seed, video, fr.scene, x / cell + t / 8u, y / cell);
  uint32_t word = synth_noise_word(synth_noise_key(seed, video, t), y * W + x);
  int32_t n = synth_noise(word);
  uint32_t Y;
  if (fr.mode == SYNTH_MODE_NOISE) {
    Y = word & 255u;
  } else if (fr.mode == SYNTH_MODE_FLASH) {
    Y = 235u - (uint32_t)(n < 0 ? -n : n);
  } else {
    Y = synth_clamp255((int32_t)synth_yuv_palette(seed, video, fr.scene, k, 0) + n);
  }
  if (fr.fade_w != 256u) Y = synth_fade8(Y, 16u, fr.fade_w);
  return Y;
}

/* Chroma (U, V) of the 2x2 block (bx, by) = pixels (2bx.., 2by..). */
SYNTH_HD void synth_nv12_uv(uint64_t seed, uint32_t video, uint32_t t, synth_frame fr, uint32_t W,
                            uint32_t bx, uint32_t by, uint32_t* U, uint32_t* V) {
  uint32_t cell = synth_cell(W);
  uint32_t x = 2u * bx, y = 2u * by;
  uint32_t k = synth_cell_index(seed, video, fr.scene, x / cell + t / 8u, y / cell);
  uint32_t word = synth_noise_word(synth_noise_key(seed ^ SYNTH_TAG_YUV, video, t), by * W + bx);
  int32_t n = (int32_t)((((word >> 16) * 5u) >> 16)) - 2; /* [-2, 2] */
  uint32_t u = synth_clamp255((int32_t)synth_yuv_palette(seed, video, fr.scene, k, 1) + n);
  uint32_t v = synth_clamp255((int32_t)synth_yuv_palette(seed, video, fr.scene, k, 2) - n);
  if (fr.mode == SYNTH_MODE_NOISE) {
    u = word & 255u;
    v = (word >> 8) & 255u;
  } else if (fr.mode == SYNTH_MODE_FLASH) {
    u = 128u;
    v = 128u;
  } else if (fr.mode == SYNTH_MODE_ROT1) {
    uint32_t tmp = u; u = v; v = tmp;
  } else if (fr.mode == SYNTH_MODE_ROT2) {
    u = 256u - u; v = 256u - v;
  }
  if (fr.fade_w != 256u) {
    u = synth_fade8(u, 128u, fr.fade_w);
    v = synth_fade8(v, 128u, fr.fade_w);
  }
  *U = u;
  *V = v;
}

#endif /* SYNTH_H_ */
