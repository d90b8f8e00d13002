/*
 * synth_host.c — host (CPU) side of the seeded input generator (see synth.h).
 * Built into synth/libsynth.so.  Holds no method arithmetic.
 *
 * The loops memoise pure functions of synth.h (palette per frame, cell index
 * per texture cell), so the bytes are exactly synth_pixel()'s; the test
 * tests/test_synth.py checks that against the uncached synth_pixel().
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "synth.h"

/* ---------------------------------------------------------------- frames */

typedef struct {
  uint64_t seed;
  uint32_t video, W, H;
  int64_t t0, n;
  const synth_frame* frames; /* indexed by absolute frame index t */
  uint8_t* out;              /* [n][H][W][3] */
  int64_t f_begin, f_end;    /* relative frame range of this worker */
} gen_job;

static void gen_one_frame(uint64_t seed, uint32_t video, uint32_t W, uint32_t H, uint32_t t,
                          synth_frame fr, uint8_t* dst) {
  uint32_t pal[8][3];
  for (uint32_t k = 0; k < 8; ++k)
    for (uint32_t c = 0; c < 3; ++c) pal[k][c] = synth_palette(seed, video, fr.scene, k, c);
  uint32_t key = synth_noise_key(seed, video, t);
  uint32_t cell = synth_cell(W);
  uint32_t ncx = W / cell + 2;
  uint32_t* row_k = (uint32_t*)malloc(sizeof(uint32_t) * ncx);
  uint32_t last_cy = 0xFFFFFFFFu;
  for (uint32_t y = 0; y < H; ++y) {
    uint32_t cy = y / cell;
    if (cy != last_cy) {
      for (uint32_t j = 0; j < ncx; ++j)
        row_k[j] = synth_cell_index(seed, video, fr.scene, j + t / 8u, cy);
      last_cy = cy;
    }
    uint8_t* p = dst + (size_t)y * W * 3;
    for (uint32_t x = 0; x < W; ++x) {
      uint32_t k = row_k[x / cell];
      uint32_t word = synth_noise_word(key, y * W + x);
      synth_finish_pixel(pal[k][0], pal[k][1], pal[k][2], word, fr.mode, fr.fade_w, p + 3 * x);
    }
  }
  free(row_k);
}

static void* gen_worker(void* arg) {
  gen_job* j = (gen_job*)arg;
  size_t fb = (size_t)j->W * j->H * 3;
  for (int64_t f = j->f_begin; f < j->f_end; ++f) {
    int64_t t = j->t0 + f;
    gen_one_frame(j->seed, j->video, j->W, j->H, (uint32_t)t, j->frames[t], j->out + (size_t)f * fb);
  }
  return NULL;
}

/* Generate frames t0 .. t0+n-1 of one video into out ([n][H][W][3] u8). */
void synth_gen_frames(uint64_t seed, uint32_t video, uint32_t W, uint32_t H, int64_t t0, int64_t n,
                      const synth_frame* frames, uint8_t* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  gen_job jobs[256];
  if (nthreads > 256) nthreads = 256;
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].seed = seed;
    jobs[i].video = video;
    jobs[i].W = W;
    jobs[i].H = H;
    jobs[i].t0 = t0;
    jobs[i].n = n;
    jobs[i].frames = frames;
    jobs[i].out = out;
    jobs[i].f_begin = n * i / nthreads;
    jobs[i].f_end = n * (i + 1) / nthreads;
  }
  if (nthreads == 1) {
    gen_worker(&jobs[0]);
    return;
  }
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, gen_worker, &jobs[i]);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* ---------------------------------------------------------------- NV12 */

typedef struct {
  uint64_t seed;
  uint32_t video, W, H;
  int64_t t0;
  const synth_frame* frames;
  uint8_t* out;
  int64_t f_begin, f_end;
} nv12_job;

static void* nv12_worker(void* arg) {
  nv12_job* j = (nv12_job*)arg;
  const size_t fb = (size_t)j->W * j->H * 3 / 2;
  for (int64_t f = j->f_begin; f < j->f_end; ++f) {
    const uint32_t t = (uint32_t)(j->t0 + f);
    const synth_frame fr = j->frames[t];
    uint8_t* Y = j->out + (size_t)f * fb;
    uint8_t* UV = Y + (size_t)j->W * j->H;
    for (uint32_t y = 0; y < j->H; ++y)
      for (uint32_t x = 0; x < j->W; ++x)
        Y[(size_t)y * j->W + x] = (uint8_t)synth_nv12_y(j->seed, j->video, t, fr, j->W, x, y);
    for (uint32_t by = 0; by < j->H / 2; ++by)
      for (uint32_t bx = 0; bx < j->W / 2; ++bx) {
        uint32_t u, v;
        synth_nv12_uv(j->seed, j->video, t, fr, j->W, bx, by, &u, &v);
        UV[(size_t)by * j->W + 2 * bx] = (uint8_t)u;
        UV[(size_t)by * j->W + 2 * bx + 1] = (uint8_t)v;
      }
  }
  return NULL;
}

/* NV12 frames t0..t0+n-1 (each: Y [H][W] then UV [H/2][W]) into out. */
void synth_gen_nv12(uint64_t seed, uint32_t video, uint32_t W, uint32_t H, int64_t t0, int64_t n,
                    const synth_frame* frames, uint8_t* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  nv12_job jobs[256];
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].seed = seed;
    jobs[i].video = video;
    jobs[i].W = W;
    jobs[i].H = H;
    jobs[i].t0 = t0;
    jobs[i].frames = frames;
    jobs[i].out = out;
    jobs[i].f_begin = n * i / nthreads;
    jobs[i].f_end = n * (i + 1) / nthreads;
  }
  if (nthreads == 1) {
    nv12_worker(&jobs[0]);
    return;
  }
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, nv12_worker, &jobs[i]);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* Uncached single pixel (for testing the memoised loop). */
void synth_pixel_ref(uint64_t seed, uint32_t video, uint32_t t, const synth_frame* fr, uint32_t W,
                     uint32_t x, uint32_t y, uint8_t* out) {
  synth_pixel(seed, video, t, *fr, W, x, y, out);
}

/* ------------------------------------------------------------ embeddings */

/* e[f][d] for frames t0..t0+n-1 (out: [n][D] f32). */
void synth_gen_emb(uint64_t seed, uint32_t video, int64_t t0, int64_t n, uint32_t D,
                   const synth_frame* frames, float* out) {
  int32_t* dir = (int32_t*)malloc(sizeof(int32_t) * D);
  uint32_t cur_scene = 0xFFFFFFFFu;
  for (int64_t f = 0; f < n; ++f) {
    int64_t t = t0 + f;
    uint32_t s = frames[t].scene;
    if (s != cur_scene) {
      for (uint32_t d = 0; d < D; ++d) dir[d] = synth_emb_dir(seed, video, s, d);
      cur_scene = s;
    }
    uint32_t key = synth_emb_key(seed, video, (uint32_t)t);
    float* row = out + (size_t)f * D;
    for (uint32_t d = 0; d < D; ++d) row[d] = synth_emb_value(dir[d], key, d);
  }
  free(dir);
}

/* ------------------------------------------------------------ frame hash */

/* fh = sum_i mix64(w_i ^ i) mod 2^64 over the little-endian u64 words. */
uint64_t synth_frame_hash(const uint8_t* frame, int64_t bytes) {
  uint64_t acc = 0;
  int64_t nw = bytes / 8;
  for (int64_t i = 0; i < nw; ++i) {
    uint64_t w;
    memcpy(&w, frame + 8 * i, 8);
    acc += synth_hash_word(w, (uint64_t)i);
  }
  return acc;
}
