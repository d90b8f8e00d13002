/*
 * oracle.c — CPU ORACLE (test infrastructure only; see oracle.h header).
 *
 * Follows PAPER.md:35 (§2.1 "Clipping Pipeline") step by step, with the
 * readings O1..O9 of DESIGN.md §"Readings".  No blocking, no
 * fusion, no SIMD; every division is a plain integer floor division of
 * non-negative integers; sums run in ascending index order.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ O1 --
 * Pixel -> HSV bin (hexcone HSV, OpenCV max tie-break r > g > b).
 *   mx = max(r,g,b), mn = min(r,g,b), d = mx - mn
 *   hue: d == 0 -> h = 0; else
 *        mx == r: num6 = g - b (+ 6d if negative)
 *        mx == g: num6 = 2d + (b - r)
 *        else   : num6 = 4d + (r - g)
 *        h = floor(nh * num6 / (6d))           (num6 in [0, 6d))
 *   sat: s = mx == 0 ? 0 : min(ns - 1, floor(ns * d / mx))
 *   val: v = floor(nv * mx / 256)
 *   bin = (h * ns + s) * nv + v
 */
int32_t oracle_bin(int32_t r, int32_t g, int32_t b, int32_t nh, int32_t ns, int32_t nv) {
  int32_t mx = r;
  if (g > mx) mx = g;
  if (b > mx) mx = b;
  int32_t mn = r;
  if (g < mn) mn = g;
  if (b < mn) mn = b;
  int32_t d = mx - mn;

  int32_t h;
  if (d == 0) {
    h = 0;
  } else {
    int32_t num6;
    if (mx == r) {
      num6 = g - b;
      if (num6 < 0) num6 += 6 * d;
    } else if (mx == g) {
      num6 = 2 * d + (b - r);
    } else {
      num6 = 4 * d + (r - g);
    }
    h = (nh * num6) / (6 * d);
  }

  int32_t s;
  if (mx == 0) {
    s = 0;
  } else {
    s = (ns * d) / mx;
    if (s > ns - 1) s = ns - 1;
  }

  int32_t v = (nv * mx) / 256;

  return (h * ns + s) * nv + v;
}

void oracle_bin_table(int32_t nh, int32_t ns, int32_t nv, uint8_t* table) {
  for (int32_t r = 0; r < 256; ++r)
    for (int32_t g = 0; g < 256; ++g)
      for (int32_t b = 0; b < 256; ++b)
        table[(r << 16) | (g << 8) | b] = (uint8_t)oracle_bin(r, g, b, nh, ns, nv);
}

/* ------------------------------------------------------------------ O0 --
 * NV12 -> RGB (reading O0, for NVDEC-native input, §2.3):
 * BT.601 limited range, 20-bit fixed point:
 *   y' = max(0, Y - 16) * 1220542
 *   R = sat((y' + 2^19 + 1673527 (V-128)) >> 20)
 *   G = sat((y' + 2^19 - 852492 (V-128) - 409993 (U-128)) >> 20)
 *   B = sat((y' + 2^19 + 2116026 (U-128)) >> 20)
 * with sat() clamping to [0, 255] and >> an arithmetic (floor) shift; the
 * chroma of pixel (x, y) is the UV pair of block (x/2, y/2). */
static int32_t sat255(int64_t v) { return v < 0 ? 0 : (v > 255 ? 255 : (int32_t)v); }

static int64_t floor_shift20(int64_t v) {
  /* floor(v / 2^20) for any sign */
  return v >= 0 ? v / 1048576 : -((-v + 1048575) / 1048576);
}

void oracle_nv12_to_rgb(const uint8_t* nv12, int64_t H, int64_t W, uint8_t* rgb) {
  const uint8_t* Yp = nv12;
  const uint8_t* UVp = nv12 + H * W;
  for (int64_t y = 0; y < H; ++y) {
    for (int64_t x = 0; x < W; ++x) {
      int64_t Y = Yp[y * W + x];
      int64_t U = UVp[(y / 2) * W + 2 * (x / 2)];
      int64_t V = UVp[(y / 2) * W + 2 * (x / 2) + 1];
      int64_t yy = (Y - 16 > 0 ? Y - 16 : 0) * 1220542;
      int64_t r = yy + 524288 + 1673527 * (V - 128);
      int64_t g = yy + 524288 - 852492 * (V - 128) - 409993 * (U - 128);
      int64_t b = yy + 524288 + 2116026 * (U - 128);
      uint8_t* o = rgb + 3 * (y * W + x);
      o[0] = (uint8_t)sat255(floor_shift20(r));
      o[1] = (uint8_t)sat255(floor_shift20(g));
      o[2] = (uint8_t)sat255(floor_shift20(b));
    }
  }
}

/* ------------------------------------------------------------------ O2 --
 * hist_t[b] = #{pixels of frame t with bin b}; every pixel is analysed
 * (no downscaling, cropping or letterbox handling). */
void oracle_hist(const uint8_t* frame, int64_t npix, int32_t nh, int32_t ns, int32_t nv,
                 uint32_t* hist) {
  int32_t nbins = nh * ns * nv;
  for (int32_t i = 0; i < nbins; ++i) hist[i] = 0;
  for (int64_t p = 0; p < npix; ++p) {
    int32_t r = frame[3 * p + 0];
    int32_t g = frame[3 * p + 1];
    int32_t b = frame[3 * p + 2];
    hist[oracle_bin(r, g, b, nh, ns, nv)] += 1;
  }
}

typedef struct {
  const uint8_t* frames;
  int64_t f0, f1, npix;
  int32_t nh, ns, nv;
  uint32_t* hist;
} hist_job;

static void* hist_worker(void* arg) {
  hist_job* j = (hist_job*)arg;
  int32_t nbins = j->nh * j->ns * j->nv;
  for (int64_t f = j->f0; f < j->f1; ++f)
    oracle_hist(j->frames + f * j->npix * 3, j->npix, j->nh, j->ns, j->nv,
                j->hist + f * nbins);
  return NULL;
}

void oracle_hist_frames(const uint8_t* frames, int64_t n, int64_t npix, int32_t nh, int32_t ns,
                        int32_t nv, uint32_t* hist, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  hist_job jobs[256];
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].frames = frames;
    jobs[i].f0 = n * i / nthreads;
    jobs[i].f1 = n * (i + 1) / nthreads;
    jobs[i].npix = npix;
    jobs[i].nh = nh;
    jobs[i].ns = ns;
    jobs[i].nv = nv;
    jobs[i].hist = hist;
  }
  if (nthreads == 1) {
    hist_worker(&jobs[0]);
    return;
  }
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, hist_worker, &jobs[i]);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

typedef struct {
  const uint8_t* frames;
  int64_t f0, f1, H, W;
  int32_t nh, ns, nv;
  uint32_t* hist;
} nv12_job;

static void* nv12_hist_worker(void* arg) {
  nv12_job* j = (nv12_job*)arg;
  int32_t nbins = j->nh * j->ns * j->nv;
  uint8_t* rgb = (uint8_t*)malloc((size_t)(3 * j->H * j->W));
  for (int64_t f = j->f0; f < j->f1; ++f) {
    oracle_nv12_to_rgb(j->frames + f * (j->H * j->W * 3 / 2), j->H, j->W, rgb);
    oracle_hist(rgb, j->H * j->W, j->nh, j->ns, j->nv, j->hist + f * nbins);
  }
  free(rgb);
  return NULL;
}

void oracle_hist_nv12_frames(const uint8_t* frames, int64_t n, int64_t H, int64_t W, int32_t nh,
                             int32_t ns, int32_t nv, uint32_t* hist, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
  pthread_t th[256];
  nv12_job jobs[256];
  for (int i = 0; i < nthreads; ++i) {
    jobs[i].frames = frames;
    jobs[i].f0 = n * i / nthreads;
    jobs[i].f1 = n * (i + 1) / nthreads;
    jobs[i].H = H;
    jobs[i].W = W;
    jobs[i].nh = nh;
    jobs[i].ns = ns;
    jobs[i].nv = nv;
    jobs[i].hist = hist;
  }
  if (nthreads == 1) {
    nv12_hist_worker(&jobs[0]);
    return;
  }
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, nv12_hist_worker, &jobs[i]);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
}

/* ------------------------------------------------------------------ O3 --
 * L1_t = sum_b |hist_t[b] - hist_{t-1}[b]| for t >= 1, L1_0 = 0;
 * score_t = L1_t / (2N), one IEEE f64 division (total-variation distance). */
void oracle_l1(const uint32_t* hist, int64_t n, int32_t nbins, int64_t npix, uint32_t* l1,
               double* score) {
  for (int64_t t = 0; t < n; ++t) {
    uint64_t acc = 0;
    if (t >= 1) {
      for (int32_t b = 0; b < nbins; ++b) {
        int64_t a = hist[t * nbins + b];
        int64_t c = hist[(t - 1) * nbins + b];
        acc += (uint64_t)(a > c ? a - c : c - a);
      }
    }
    l1[t] = (uint32_t)acc;
    if (score) score[t] = (double)acc / (double)(2 * npix);
  }
}

/* ------------------------------------------------------------------ O4 --
 * Candidate <=> t >= 1 and L1_t * 10^6 >= tau_ppm * 2N (exact, u64). */
int64_t oracle_candidates(const uint32_t* l1, int64_t n, int64_t npix, int64_t tau_ppm,
                          int64_t* cand) {
  int64_t k = 0;
  for (int64_t t = 1; t < n; ++t) {
    uint64_t lhs = (uint64_t)l1[t] * 1000000ull;
    uint64_t rhs = (uint64_t)tau_ppm * (uint64_t)(2 * npix);
    if (lhs >= rhs) cand[k++] = t;
  }
  return k;
}

/* ------------------------------------------------------------- O5 + O6 --
 * O5: last = 0; for candidates t ascending: accept t iff t - last >= L_min.
 * O6: if any cut was accepted and n - last < L_min, drop the last accepted cut. */
int64_t oracle_min_length(const int64_t* cand, int64_t n_cand, int64_t n, int64_t l_min,
                          int64_t* cuts) {
  int64_t last = 0, k = 0;
  for (int64_t i = 0; i < n_cand; ++i) {
    int64_t t = cand[i];
    if (t - last >= l_min) {
      cuts[k++] = t;
      last = t;
    }
  }
  if (k > 0 && n - last < l_min) k -= 1;
  return k;
}

/* ------------------------------------------------------------------ O8 --
 * Clip embedding S = sum of the clip's per-frame image embeddings, f64,
 * ascending frame order (the sum is equivalent to the mean for cosine). */
void oracle_clip_sum(const float* emb, int64_t dim, int64_t f0, int64_t f1, double* S) {
  for (int64_t d = 0; d < dim; ++d) S[d] = 0.0;
  for (int64_t f = f0; f < f1; ++f)
    for (int64_t d = 0; d < dim; ++d) S[d] += (double)emb[f * dim + d];
}

double oracle_cosine(const double* a, const double* b, int64_t dim) {
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int64_t d = 0; d < dim; ++d) {
    dot += a[d] * b[d];
    na += a[d] * a[d];
    nb += b[d] * b[d];
  }
  na = sqrt(na);
  nb = sqrt(nb);
  if (na == 0.0 || nb == 0.0) return 0.0;
  return dot / (na * nb);
}

/* ------------------------------------------------------------------ O9 --
 * Round-synchronous merge to a fixed point:
 *   B = [0] ++ cuts ++ [n]; repeat: c_k = cos(S_k, S_{k+1}) for every adjacent
 *   pair; M = {k : c_k >= theta}; if M is empty stop; else remove B_{k+1} for
 *   all k in M at once and recompute the S of the merged clips from frames.
 *   Band hit <=> |c_k - theta| <= band_rel * theta (counted in every round). */
/* O8' (NEXT f4): with keyframe stride sigma >= 1 only the keyframes enter the
 * clip sums: frame f is a keyframe iff (f - b) % sigma == 0, b = the first frame
 * of the DETECTED clip containing f (embeddings are computed once per detected
 * clip, every sigma-th frame); a merged clip sums its constituents' keyframes.
 * sigma = 1 is O8. */
static void clip_sum_keyframes(const float* emb, int64_t dim, int64_t f0, int64_t f1,
                               const char* key, double* S) {
  for (int64_t d = 0; d < dim; ++d) S[d] = 0.0;
  for (int64_t f = f0; f < f1; ++f)
    if (key[f])
      for (int64_t d = 0; d < dim; ++d) S[d] += (double)emb[f * dim + d];
}

int64_t oracle_merge(const float* emb, int64_t n, int64_t dim, const int64_t* cuts,
                     int64_t n_cuts, double theta, double band_rel, int32_t max_rounds,
                     int64_t* final_cuts, double* cos_at_decision, int64_t* n_band_hits,
                     int32_t* rounds) {
  return oracle_merge_stride(emb, n, dim, cuts, n_cuts, theta, band_rel, max_rounds, 1,
                             final_cuts, cos_at_decision, n_band_hits, rounds);
}

int64_t oracle_merge_stride(const float* emb, int64_t n, int64_t dim, const int64_t* cuts,
                            int64_t n_cuts, double theta, double band_rel, int32_t max_rounds,
                            int64_t stride, int64_t* final_cuts, double* cos_at_decision,
                            int64_t* n_band_hits, int32_t* rounds) {
  char* key = (char*)malloc(n > 0 ? n : 1);
  for (int64_t j = 0, b = 0; j <= n_cuts; ++j) {
    const int64_t e = j < n_cuts ? cuts[j] : n;
    for (int64_t f = b; f < e; ++f) key[f] = ((f - b) % stride) == 0;
    b = e;
  }
  /* B holds the boundaries; idx[j] = index of B[j] among the detected cuts */
  int64_t* B = (int64_t*)malloc(sizeof(int64_t) * (n_cuts + 2));
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (n_cuts + 2));
  int64_t nb = 0;
  B[nb] = 0;
  idx[nb++] = -1;
  for (int64_t j = 0; j < n_cuts; ++j) {
    B[nb] = cuts[j];
    idx[nb++] = j;
  }
  B[nb] = n;
  idx[nb++] = -1;
  for (int64_t j = 0; j < n_cuts; ++j) cos_at_decision[j] = 0.0;

  double* S = (double*)malloc(sizeof(double) * dim * (n_cuts + 1));
  double* c = (double*)malloc(sizeof(double) * (n_cuts + 1));
  char* rm = (char*)malloc(n_cuts + 2);
  int64_t hits = 0;
  int32_t r = 0;
  for (;;) {
    int64_t K = nb - 1; /* clips */
    if (K < 2) break;
    if (max_rounds > 0 && r >= max_rounds) break;
    for (int64_t k = 0; k < K; ++k) clip_sum_keyframes(emb, dim, B[k], B[k + 1], key, S + k * dim);
    int64_t m = 0;
    for (int64_t k = 0; k + 1 < K; ++k) {
      c[k] = oracle_cosine(S + k * dim, S + (k + 1) * dim, dim);
      cos_at_decision[idx[k + 1]] = c[k];
      if (fabs(c[k] - theta) <= band_rel * theta) hits += 1;
      rm[k + 1] = (c[k] >= theta);
      m += rm[k + 1];
    }
    r += 1;
    if (m == 0) break;
    int64_t w = 0;
    for (int64_t j = 0; j < nb; ++j) {
      if (j > 0 && j < nb - 1 && rm[j]) continue;
      B[w] = B[j];
      idx[w] = idx[j];
      ++w;
    }
    nb = w;
  }
  int64_t nf = nb - 2;
  for (int64_t j = 0; j < nf; ++j) final_cuts[j] = B[j + 1];
  *n_band_hits = hits;
  *rounds = r;
  free(B);
  free(idx);
  free(S);
  free(c);
  free(rm);
  free(key);
  return nf;
}

/* ------------------------------------------------------------ the path --
 * O1-O2 histograms, O3 distance, O4 threshold, O5-O6 greedy + tail,
 * O8-O9 merge on the detected cuts. */
int oracle_video(const uint8_t* frames, int64_t n, int64_t npix, const float* emb, int64_t dim,
                 const oracle_params* p, int nthreads, uint32_t* hist, uint32_t* l1,
                 double* score, int64_t* detected, int64_t* final_cuts, double* cos,
                 oracle_result* res) {
  int32_t nbins = p->nh * p->ns * p->nv;
  oracle_hist_frames(frames, n, npix, p->nh, p->ns, p->nv, hist, nthreads);
  oracle_l1(hist, n, nbins, npix, l1, score);
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  int64_t nc = oracle_candidates(l1, n, npix, p->tau_ppm, cand);
  int64_t nd = oracle_min_length(cand, nc, n, p->l_min, detected);
  free(cand);
  res->n_candidates = nc;
  res->n_detected = nd;
  if (emb) {
    res->n_final = oracle_merge(emb, n, dim, detected, nd, p->theta, p->band_rel,
                                p->max_rounds, final_cuts, cos, &res->n_band_hits,
                                &res->rounds);
  } else {
    res->n_final = nd;
    for (int64_t j = 0; j < nd; ++j) final_cuts[j] = detected[j];
    res->n_band_hits = 0;
    res->rounds = 0;
  }
  return 0;
}

/* ------------------------------------------------------------------ O10/O11 (NEXT f3) */
/* O10: frame i (0 <= i < k) sampled from clip [s, e): the middle of the i-th of
 * k equal parts, s + floor((2i + 1)(e - s) / (2k)). */
int64_t oracle_sample_index(int64_t s, int64_t e, int64_t i, int64_t k) {
  return s + ((2 * i + 1) * (e - s)) / (2 * k);
}

/* O11 coefficients of one output coordinate d of an axis src -> dst: OpenCV's
 * 8-bit INTER_LINEAR (half-pixel centres, float32 position, 11-bit weights
 * rounded to nearest-even, clamped at the border). */
static void lin_coeff(int64_t src, int64_t dst, int64_t d, int64_t* s0, int64_t* s1, int32_t* w0,
                      int32_t* w1) {
  const double scale = 1.0 / ((double)dst / (double)src);
  float f = (float)(((double)d + 0.5) * scale - 0.5);
  int64_t s = (int64_t)floorf(f);
  f = f - (float)s;
  if (s < 0) {
    f = 0.0f;
    s = 0;
  }
  if (s >= src - 1) {
    f = 0.0f;
    s = src - 1;
  }
  *s0 = s;
  *s1 = s + 1 < src ? s + 1 : src - 1;
  *w0 = (int32_t)lrintf((1.0f - f) * 2048.0f);
  *w1 = (int32_t)lrintf(f * 2048.0f);
}

/* O11: resize one RGB24 frame [H][W][3] -> [H2][W2][3].  Horizontal pass
 * h = p0*w0 + p1*w1 (exact int), vertical pass
 * out = sat((((h0 >> 4) * v0 >> 16) + ((h1 >> 4) * v1 >> 16) + 2) >> 2)
 * (the fixed-point rounding of OpenCV's vectorised 8-bit path). */
void oracle_resize_linear(const uint8_t* src, int64_t H, int64_t W, uint8_t* dst, int64_t H2,
                          int64_t W2) {
  for (int64_t dy = 0; dy < H2; ++dy) {
    int64_t y0, y1;
    int32_t v0, v1;
    lin_coeff(H, H2, dy, &y0, &y1, &v0, &v1);
    for (int64_t dx = 0; dx < W2; ++dx) {
      int64_t x0, x1;
      int32_t w0, w1;
      lin_coeff(W, W2, dx, &x0, &x1, &w0, &w1);
      for (int c = 0; c < 3; ++c) {
        const int64_t h0 = (int64_t)src[(y0 * W + x0) * 3 + c] * w0 + (int64_t)src[(y0 * W + x1) * 3 + c] * w1;
        const int64_t h1 = (int64_t)src[(y1 * W + x0) * 3 + c] * w0 + (int64_t)src[(y1 * W + x1) * 3 + c] * w1;
        const int64_t t0 = ((h0 >> 4) * v0) >> 16, t1 = ((h1 >> 4) * v1) >> 16;
        const int64_t o = (t0 + t1 + 2) >> 2;
        dst[(dy * W2 + dx) * 3 + c] = (uint8_t)(o < 0 ? 0 : (o > 255 ? 255 : o));
      }
    }
  }
}

/* O10 + O11 for one video: clips from cuts[n_cuts] (O7), k frames per clip,
 * out [(n_cuts+1)*k][H2][W2][3] in clip order, index [(n_cuts+1)*k]. */
void oracle_sample_clips(const uint8_t* frames, int64_t n, int64_t H, int64_t W, const int64_t* cuts,
                         int64_t n_cuts, int64_t k, int64_t H2, int64_t W2, uint8_t* out,
                         int64_t* index) {
  for (int64_t c = 0; c <= n_cuts; ++c) {
    const int64_t s = c == 0 ? 0 : cuts[c - 1];
    const int64_t e = c == n_cuts ? n : cuts[c];
    for (int64_t i = 0; i < k; ++i) {
      const int64_t t = oracle_sample_index(s, e, i, k);
      index[c * k + i] = t;
      oracle_resize_linear(frames + t * H * W * 3, H, W, out + (c * k + i) * H2 * W2 * 3, H2, W2);
    }
  }
}

/* ------------------------------------------------------------------ O3'/O4' (NEXT f4) */
/* O3' distance between the histograms a (frame t-1) and b (frame t), f64,
 * bins in ascending order, N = npix pixels each:
 *   kind 1  chi-square   D = (1/2N) sum_{a+b>0} (a-b)^2 / (a+b)           in [0, 1]
 *   kind 2  Bhattacharyya D = sqrt(max(0, 1 - sum sqrt(a*b) / N))         in [0, 1]
 *   kind 3  correlation  D = 1 - r, r = (K S_ab - N^2) / sqrt((K S_aa - N^2)(K S_bb - N^2)),
 *           K = nbins, S_xy = sum x*y (exact integers); r = 1 if both
 *           denominators are 0, else 0 if one is                        in [0, 2] */
double oracle_distance(const uint32_t* a, const uint32_t* b, int32_t nbins, int64_t npix,
                       int32_t kind) {
  if (kind == 1) {
    double acc = 0.0;
    for (int32_t i = 0; i < nbins; ++i) {
      const int64_t s = (int64_t)a[i] + (int64_t)b[i];
      if (s == 0) continue;
      const int64_t d = (int64_t)a[i] - (int64_t)b[i];
      acc = acc + (double)(d * d) / (double)s;
    }
    return acc / (double)(2 * npix);
  }
  if (kind == 2) {
    double acc = 0.0;
    for (int32_t i = 0; i < nbins; ++i) acc = acc + sqrt((double)a[i] * (double)b[i]);
    const double x = 1.0 - acc / (double)npix;
    return sqrt(x > 0.0 ? x : 0.0);
  }
  if (kind == 3) {
    int64_t sab = 0, saa = 0, sbb = 0;
    for (int32_t i = 0; i < nbins; ++i) {
      sab += (int64_t)a[i] * (int64_t)b[i];
      saa += (int64_t)a[i] * (int64_t)a[i];
      sbb += (int64_t)b[i] * (int64_t)b[i];
    }
    const int64_t n2 = npix * npix;
    const int64_t num = (int64_t)nbins * sab - n2;
    const int64_t A = (int64_t)nbins * saa - n2, B = (int64_t)nbins * sbb - n2;
    double r;
    if (A == 0 && B == 0) r = 1.0;
    else if (A == 0 || B == 0) r = 0.0;
    else r = (double)num / sqrt((double)A * (double)B);
    return 1.0 - r;
  }
  return -1.0;
}

/* O3' for n frames of one video: d[0] = 0, d[t] = distance(h_{t-1}, h_t). */
void oracle_distances(const uint32_t* hist, int64_t n, int32_t nbins, int64_t npix, int32_t kind,
                      double* d) {
  if (n > 0) d[0] = 0.0;
  for (int64_t t = 1; t < n; ++t)
    d[t] = oracle_distance(hist + (t - 1) * nbins, hist + t * nbins, nbins, npix, kind);
}

/* O4' fixed threshold on an f64 distance: candidate <=> t >= 1 and d[t] >= tau_ppm / 1e6. */
int64_t oracle_candidates_f64(const double* d, int64_t n, int64_t tau_ppm, int64_t* cand) {
  const double tau = (double)tau_ppm / 1e6;
  int64_t k = 0;
  for (int64_t t = 1; t < n; ++t)
    if (d[t] >= tau) cand[k++] = t;
  return k;
}

/* O4'' adaptive threshold on L1 (exact integers): with the neighbours
 * U_t = {u : 1 <= u <= n-1, 0 < |u - t| <= w} (m = |U_t|), candidate <=>
 * t >= 1, m > 0, L1_t * m * 1e6 >= ratio_ppm * sum_{u in U_t} L1_u, and
 * L1_t * 1e6 >= tau_ppm * 2N (the fixed rule as a floor). */
int64_t oracle_candidates_adaptive(const uint32_t* l1, int64_t n, int64_t npix, int64_t tau_ppm,
                                   int64_t w, int64_t ratio_ppm, int64_t* cand) {
  int64_t k = 0;
  for (int64_t t = 1; t < n; ++t) {
    unsigned __int128 sum = 0;
    int64_t m = 0;
    for (int64_t u = t - w; u <= t + w; ++u) {
      if (u < 1 || u > n - 1 || u == t) continue;
      sum += l1[u];
      ++m;
    }
    if (m == 0) continue;
    const unsigned __int128 lhs = (unsigned __int128)l1[t] * (unsigned __int128)m * 1000000u;
    const unsigned __int128 rhs = (unsigned __int128)ratio_ppm * sum;
    const int floor_ok = (uint64_t)l1[t] * 1000000ull >= (uint64_t)tau_ppm * (uint64_t)(2 * npix);
    if (lhs >= rhs && floor_ok) cand[k++] = t;
  }
  return k;
}
