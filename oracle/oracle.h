/*
 * oracle.h — CPU ORACLE for the shot-boundary clip-splitting path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load liboracle.so.  The
 * product path (paper_2503_12964_b200/) never links, imports or calls it; it
 * shares no code, header, table or constant with the CUDA path.
 *
 * The method (§2.1 "Clipping Pipeline"): "It uses an aggressive
 * method of splitting clips, analyzing the color changes between frames,
 * which is smoothed out by computing the similarity between image embeddings
 * of adjacent clips to potentially merge them back together."  Every
 * quantitative rule below is a READING (the paper is silent), listed in
 * DESIGN.md §"Readings" under the same labels O1..O9.
 *
 * Plain, slow, obviously correct: integer divisions written out, sums in
 * ascending index order, f64 for floating point.
 */
#ifndef ORACLE_H_
#define ORACLE_H_

#include <stdint.h>

typedef struct {
  int32_t nh, ns, nv;          /* hue / saturation / value bins (18, 3, 3) */
  int64_t tau_ppm;             /* cut threshold on TV distance, parts per million (300000) */
  int64_t l_min;               /* minimum clip length in frames (8) */
  double theta;                /* merge cosine threshold (0.90) */
  double band_rel;             /* band half-width relative to theta (1e-5) */
  int32_t max_rounds;          /* 0 = merge until fixed point */
} oracle_params;

/* O0 (NV12 input, NEXT f1): one NV12 frame (Y plane [H][W], then the
 * interleaved UV plane [H/2][W/2][2]) -> RGB24 [H][W][3], BT.601 limited range
 * in 20-bit fixed point (the definition of OpenCV's COLOR_YUV2RGB_NV12). */
void oracle_nv12_to_rgb(const uint8_t* nv12, int64_t H, int64_t W, uint8_t* rgb);

/* O0 + O2: histograms of n NV12 frames ([n][H*W*3/2] bytes) -> [n][nbins]. */
void oracle_hist_nv12_frames(const uint8_t* frames, int64_t n, int64_t H, int64_t W, int32_t nh,
                             int32_t ns, int32_t nv, uint32_t* hist, int nthreads);

/* O1: pixel -> joint HSV bin in [0, nh*ns*nv). */
int32_t oracle_bin(int32_t r, int32_t g, int32_t b, int32_t nh, int32_t ns, int32_t nv);

/* O1 over all 2^24 colours; table[(r<<16)|(g<<8)|b]. */
void oracle_bin_table(int32_t nh, int32_t ns, int32_t nv, uint8_t* table);

/* O2: histogram of one frame (npix RGB24 pixels) into hist[nbins] (overwritten). */
void oracle_hist(const uint8_t* frame, int64_t npix, int32_t nh, int32_t ns, int32_t nv,
                 uint32_t* hist);

/* O2 for n frames ([n][npix*3] bytes) -> hist [n][nbins], using nthreads threads
 * (frames are independent; the arithmetic per frame is oracle_hist). */
void oracle_hist_frames(const uint8_t* frames, int64_t n, int64_t npix, int32_t nh, int32_t ns,
                        int32_t nv, uint32_t* hist, int nthreads);

/* O3: L1[t] = sum_b |h_t[b] - h_{t-1}[b]| (L1[0] = 0); score[t] = L1[t] / (2N). */
void oracle_l1(const uint32_t* hist, int64_t n, int32_t nbins, int64_t npix, uint32_t* l1,
               double* score);

/* O4: candidates t >= 1 with L1[t] * 1e6 >= tau_ppm * 2N; returns their count. */
int64_t oracle_candidates(const uint32_t* l1, int64_t n, int64_t npix, int64_t tau_ppm,
                          int64_t* cand);

/* O5 + O6: greedy minimum clip length, then the tail rule; returns #cuts. */
int64_t oracle_min_length(const int64_t* cand, int64_t n_cand, int64_t n, int64_t l_min,
                          int64_t* cuts);

/* O8: S[d] = sum_{f in [f0, f1)} emb[f][d], f64, ascending f. */
void oracle_clip_sum(const float* emb, int64_t dim, int64_t f0, int64_t f1, double* S);

/* O9 cosine: S_a.S_b / (|S_a| |S_b|), 0 if a norm is 0. */
double oracle_cosine(const double* a, const double* b, int64_t dim);

/* O8 + O9: round-synchronous merge to a fixed point.
 * In: detected cuts[n_cuts].  Out: final[] (returns count), cos_at_decision[n_cuts]
 * (the cosine of each detected boundary in the last round it was evaluated),
 * *n_band_hits (over all rounds), *rounds (rounds that evaluated cosines). */
int64_t oracle_merge(const float* emb, int64_t n, int64_t dim, const int64_t* cuts,
                     int64_t n_cuts, double theta, double band_rel, int32_t max_rounds,
                     int64_t* final_cuts, double* cos_at_decision, int64_t* n_band_hits,
                     int32_t* rounds);

/* O8' + O9 (NEXT f4): the merge with keyframe stride sigma >= 1 (O8': only every
 * sigma-th frame of each detected clip enters the clip sums); sigma = 1 is oracle_merge. */
int64_t oracle_merge_stride(const float* emb, int64_t n, int64_t dim, const int64_t* cuts,
                            int64_t n_cuts, double theta, double band_rel, int32_t max_rounds,
                            int64_t stride, int64_t* final_cuts, double* cos_at_decision,
                            int64_t* n_band_hits, int32_t* rounds);

/* The whole path for one video (O1..O9). hist [n][nbins], l1 [n], score [n],
 * detected / final [n] capacity, cos [n]. Returns 0. */
typedef struct {
  int64_t n_candidates, n_detected, n_final, n_band_hits;
  int32_t rounds;
} oracle_result;

int oracle_video(const uint8_t* frames, int64_t n, int64_t npix, const float* emb, int64_t dim,
                 const oracle_params* p, int nthreads, uint32_t* hist, uint32_t* l1,
                 double* score, int64_t* detected, int64_t* final_cuts, double* cos,
                 oracle_result* res);

/* O10 (NEXT f3): frame i of k sampled from clip [s, e): s + floor((2i+1)(e-s) / (2k)). */
int64_t oracle_sample_index(int64_t s, int64_t e, int64_t i, int64_t k);

/* O11 (NEXT f3): bilinear resize of one RGB24 frame [H][W][3] -> [H2][W2][3]
 * (OpenCV 8-bit INTER_LINEAR fixed point). */
void oracle_resize_linear(const uint8_t* src, int64_t H, int64_t W, uint8_t* dst, int64_t H2,
                          int64_t W2);

/* O10 + O11 for one video's clips (cuts as in O7): out [(n_cuts+1)*k][H2][W2][3],
 * index [(n_cuts+1)*k]. */
void oracle_sample_clips(const uint8_t* frames, int64_t n, int64_t H, int64_t W, const int64_t* cuts,
                         int64_t n_cuts, int64_t k, int64_t H2, int64_t W2, uint8_t* out,
                         int64_t* index);

/* O3' (NEXT f4): f64 distance of histograms a (t-1), b (t): kind 1 chi-square,
 * 2 Bhattacharyya, 3 one minus correlation (definitions in oracle.c). */
double oracle_distance(const uint32_t* a, const uint32_t* b, int32_t nbins, int64_t npix,
                       int32_t kind);
void oracle_distances(const uint32_t* hist, int64_t n, int32_t nbins, int64_t npix, int32_t kind,
                      double* d);

/* O4' (NEXT f4): candidates t >= 1 with d[t] >= tau_ppm / 1e6. */
int64_t oracle_candidates_f64(const double* d, int64_t n, int64_t tau_ppm, int64_t* cand);

/* O4'' (NEXT f4): adaptive candidates on L1 (window w, ratio ratio_ppm / 1e6, floor tau_ppm). */
int64_t oracle_candidates_adaptive(const uint32_t* l1, int64_t n, int64_t npix, int64_t tau_ppm,
                                   int64_t w, int64_t ratio_ppm, int64_t* cand);

#endif /* ORACLE_H_ */
