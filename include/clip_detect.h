/*
 * clip_detect.h — C ABI of libclipdetect (B200 / sm_100a), ABI version 2.
 *
 * The hot path of the NeMo Curator clipping pipeline, PAPER.md:35 (§2.1
 * "Clipping Pipeline"): "It uses an aggressive method of splitting clips,
 * analyzing the color changes between frames, which is smoothed out by
 * computing the similarity between image embeddings of adjacent clips to
 * potentially merge them back together."  The paper gives no constants; every
 * rule below is a reading listed in DESIGN.md §"Readings" (labels O1..O9, as
 * in SURVEY.md §8(c)).
 *
 * Conventions (all entry points):
 *  - Pointers documented "device" must be CUDA device pointers on the ctx's
 *    device; "host" pointers are ordinary host memory.  All buffers are
 *    caller-owned; the ctx owns only its scratch.  Nothing is freed by the
 *    library except the ctx itself (clip_detect_destroy).
 *  - Calls enqueue on the ctx stream (borrowed, never destroyed).  Only calls
 *    that return host values synchronise that stream (marked "SYNC").
 *  - Every call returns a clip_status.  CLIP_E_INVALID / CLIP_E_CAPACITY are
 *    raised by host-side validation BEFORE anything is enqueued (no side
 *    effects).  CLIP_E_CUDA is sticky: the ctx must be destroyed.
 *    clip_last_error() gives a one-line message for the last failure.
 *  - Frames are decoded RGB24, u8 [n][H][W][3] contiguous, base 16-byte
 *    aligned, H*W % 16 == 0 (every resolution of the workloads satisfies it),
 *    or (the *_nv12 entry points, clip_video.format = CLIP_FORMAT_NV12) the
 *    decoder's NV12 surfaces, u8 [n][H*3/2][W] contiguous: H rows of Y, then
 *    H/2 rows of interleaved U,V at half horizontal resolution; H and W even,
 *    base 16-byte aligned, H*W % 32 == 0.  NV12 is converted to RGB by reading
 *    O0 (BT.601 limited range, 20-bit fixed point = OpenCV COLOR_YUV2RGB_NV12)
 *    inside the histogram kernel; the RGB frame is never materialised.
 *    H*W < 2^31 (L1 <= 2 H W is a u32); with CLIP_DIST_CORREL H*W <= 2^27
 *    (its exact int64 sums reach nbins (H W)^2); larger frames are
 *    CLIP_E_INVALID.
 *  - Only compute capability 10.0 (B200, sm_100a) is supported: any other
 *    device gives CLIP_E_ARCH.  There is no CPU fallback.
 *  - Results are deterministic: histograms, L1, cuts bit-identical for any
 *    grid or GPU count; cosines bit-identical run to run (fixed reduction
 *    order, no float atomics).
 */
#ifndef CLIP_DETECT_H_
#define CLIP_DETECT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CLIP_ABI_VERSION 2u

typedef enum {
  CLIP_OK = 0,
  CLIP_E_INVALID = 1,  /* bad argument (null, misaligned, shape, params)        */
  CLIP_E_CAPACITY = 2, /* an output capacity is too small                       */
  CLIP_E_CUDA = 3,     /* CUDA runtime error (sticky)                           */
  CLIP_E_NOMEM = 4,    /* device allocation of ctx scratch failed               */
  CLIP_E_ARCH = 5,     /* device is not sm_100 (B200)                           */
  CLIP_E_STATE = 6     /* ctx unusable (earlier sticky error)                   */
} clip_status;

#define CLIP_FLAG_TIMING 1u /* record CUDA events around each kernel (clip_get_stats) */

/* Method parameters.  Defaults (clip_params_default) are the readings of
 * O1 (18,3,3) bins, O4 tau = 0.30, O5 L_min = 8, O9 theta = 0.90. */
typedef struct {
  uint32_t abi_version;       /* must equal CLIP_ABI_VERSION                         */
  uint32_t h_bins;            /* O1 hue bins (18); h*s*v <= 256                      */
  uint32_t s_bins;            /* O1 saturation bins (3)                              */
  uint32_t v_bins;            /* O1 value bins (3)                                   */
  uint64_t cut_threshold_ppm; /* O4: cut iff L1*1e6 >= ppm*2N (300000 = TV 0.30)     */
  uint32_t min_clip_frames;   /* O5/O6: L_min >= 1 (8)                               */
  uint32_t max_merge_rounds;  /* O9: 0 = until fixed point                           */
  double merge_cos_threshold; /* O9: merge iff cos >= theta (0.90)                   */
  double band_rel;            /* band hit iff |cos - theta| <= band_rel*theta (1e-5)  */
  uint32_t flags;             /* CLIP_FLAG_*                                          */
  uint32_t reserved;          /* must be 0                                            */
  /* ABI 2: the f4 variants (readings O3', O4'' in DESIGN.md).
   * Supported by clip_frame_scores (score) and clip_run_videos; clip_cuts
   * (streaming on L1 values) accepts only the defaults (CLIP_E_INVALID otherwise). */
  uint32_t distance;          /* O3': CLIP_DIST_* (default L1/TV); non-L1 distances are
                                 f64, cut iff d >= cut_threshold_ppm / 1e6               */
  uint32_t adaptive_window;   /* O4'': 0 = fixed threshold (default); w in [1, 1024]:
                                 cut iff L1_t * m >= ratio * (sum of the m neighbour L1 within
                                 +-w frames of the same video, frames >= 1) and the fixed
                                 rule holds; needs distance = CLIP_DIST_L1                 */
  uint64_t adaptive_ratio_ppm;/* O4'': ratio in ppm (3.0 = 3000000), <= 1e9              */
  uint32_t emb_stride;        /* O8': keyframe stride sigma (0 or 1 = every frame): only
                                 frames f with (f - start of their detected clip) % sigma == 0
                                 enter the clip sums; other embeddings are never read    */
  uint32_t reserved2;         /* must be 0                                            */
} clip_params;

#define CLIP_DIST_L1 0u            /* O3: L1 = 2N * total variation (exact integers) */
#define CLIP_DIST_CHI2 1u          /* O3': (1/2N) sum (a-b)^2/(a+b)                  */
#define CLIP_DIST_BHATTACHARYYA 2u /* O3': sqrt(1 - sum sqrt(a b) / N)               */
#define CLIP_DIST_CORREL 3u        /* O3': 1 - Pearson correlation of the two histograms */

typedef struct clip_ctx clip_ctx; /* opaque; one per device; not thread-safe */

/* Fill *p with the defaults above. */
void clip_params_default(clip_params* p);

/* Create a ctx on CUDA device `cuda_device`, enqueueing on `cuda_stream`
 * (a cudaStream_t cast to uintptr_t; 0 = legacy default stream).
 * Errors: CLIP_E_INVALID (null out, bad params), CLIP_E_ARCH, CLIP_E_CUDA. */
int clip_detect_init(clip_ctx** out, const clip_params* p, int cuda_device, uintptr_t cuda_stream);

/* Destroy a ctx (synchronises its stream, frees its scratch).  NULL is a no-op. */
int clip_detect_destroy(clip_ctx* ctx);

/* Last error message of this ctx ("" if none).  Valid until the next call. */
const char* clip_last_error(const clip_ctx* ctx);

/* Rows a1-a4 for n_frames frames of ONE video (a chunk of it).
 *   frames    device u8 [n_frames][height][width][3]
 *   prev_hist device u32 [nbins] = histogram of the frame just before this
 *             chunk, or NULL at video start (then l1[0] = 0, reading O3)
 *   hist      device u32 [n_frames][nbins] out (O2: per-frame bin counts)
 *   l1        device u32 [n_frames] out or NULL (O3: sum_b |h_t - h_{t-1}|)
 *   score     device f32 [n_frames] out or NULL (O3: l1 / (2*H*W), f64 division rounded to f32;
 *             with params.distance != L1 the O3' distance to the previous frame, f64 rounded to f32)
 * nbins = h_bins*s_bins*v_bins.  Async. */
int clip_frame_scores(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                      int32_t width, const uint32_t* prev_hist, uint32_t* hist, uint32_t* l1,
                      float* score);

/* Rows a1-a4 as clip_frame_scores, for NV12 frames (device u8 [n_frames][height*3/2][width]).
 * O0 conversion fused into the histogram kernel (fast path for the default
 * 18x3x3 bins and width % 16 == 0; any other case runs a generic kernel with
 * the same results).  Errors: CLIP_E_INVALID for odd height/width.  Async. */
int clip_frame_scores_nv12(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                           int32_t width, const uint32_t* prev_hist, uint32_t* hist, uint32_t* l1,
                           float* score);

/* Row a4 alone, from histograms already computed (e.g. the seam frame of a
 * frame-sharded video, whose predecessor's histogram lives on another GPU).
 *   hist      device u32 [n_frames][nbins]; prev_hist device u32 [nbins] or NULL
 *   l1, score as clip_frame_scores (either may be NULL).  Async. */
int clip_hist_scores(clip_ctx* ctx, const uint32_t* hist, int64_t n_frames, int64_t pixels_per_frame,
                     const uint32_t* prev_hist, uint32_t* l1, float* score);

/* Streaming cut state of one video; lives in DEVICE memory, zeroed by the
 * caller at video start and passed unchanged between chunks. */
typedef struct {
  int64_t frames_seen;  /* frames consumed so far                          */
  int64_t last_cut;     /* O5 "last" (0 at video start)                    */
  int64_t n_candidates; /* O4 candidates seen so far                       */
  int64_t n_cuts;       /* accepted cuts (true count, may exceed capacity) */
} clip_cut_state;

/* Rows a5-a6 for the next chunk of ONE video's L1 values.
 *   l1        device u32 [n_frames] (from clip_frame_scores)
 *   state     device clip_cut_state (in/out)
 *   cuts      device i32 [cuts_capacity]; accepted cuts (frame index of the first
 *             frame of a new clip, video-global) are appended at state->n_cuts
 *   is_final_chunk: apply the O6 tail rule (drop the last cut if the final
 *             clip would be shorter than L_min).
 * O4: candidate <=> t >= 1 and l1*1e6 >= ppm*2N; O5: accept t iff t - last >= L_min.
 * Overflow is reported through state->n_cuts > cuts_capacity (entries beyond
 * the capacity are not written).  Async. */
int clip_cuts(clip_ctx* ctx, const uint32_t* l1, int64_t n_frames, int64_t pixels_per_frame,
              clip_cut_state* state, int32_t* cuts, int64_t cuts_capacity, int is_final_chunk);

/* Rows a7-a9 for ONE video.  SYNC.
 *   emb          device f32 [n_frames][dim] per-frame image embeddings
 *   cuts         device i32 [n_cuts] detected cuts, strictly increasing in (0, n_frames)
 *   merged       device i32 [n_cuts] out: final cuts (first *n_merged entries)
 *   n_merged     host out
 *   boundary_cos device f64 [n_cuts] out or NULL: cosine of each detected cut at the
 *                last round it was evaluated (O9)
 *   n_band_hits  host out or NULL: #evaluations with |cos - theta| <= band_rel*theta
 *   rounds       host out or NULL: rounds that evaluated cosines
 * O8: clip embedding = f64 sum of its frames' embeddings; O9: round-synchronous
 * merge of every adjacent pair with cos >= theta, to a fixed point.  Every
 * round runs on the device (one cooperative kernel launch); the call
 * synchronises once, at the end. */
int clip_merge(clip_ctx* ctx, const float* emb, int64_t n_frames, int32_t dim,
               const int32_t* cuts, int64_t n_cuts, int32_t* merged, int64_t* n_merged,
               double* boundary_cos, int64_t* n_band_hits, int32_t* rounds);

/* Clip frame sampling + resize (NEXT f3, readings O10/O11) for ONE video: the
 * step after the path, producing the encoder input of every final clip
 * (the clips feed "video embeddings").
 *   frames   device u8 [n_frames][height][width][3] (RGB24, as clip_frame_scores)
 *   cuts     device i32 [n_cuts] final cuts, strictly increasing in (0, n_frames)
 *            (clips [0,c0), [c0,c1), ..., [c_last, n_frames), as O7)
 *   k        frames per clip (>= 1): frame i of clip [s, e) is
 *            s + floor((2i+1)(e-s) / 2k)  (O10: middles of k equal parts)
 *   out_h, out_w  output size (>= 1, out_w <= 4096)
 *   out      device u8 [(n_cuts+1)*k][out_h][out_w][3], clip-major (O11: OpenCV
 *            INTER_LINEAR 8-bit fixed point, computed on the device)
 *   index    device i32 [(n_cuts+1)*k] out or NULL: the sampled frame indices
 * Errors: CLIP_E_INVALID for bad sizes / NULL pointers.  Async. */
int clip_sample_frames(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                       int32_t width, const int32_t* cuts, int64_t n_cuts, int32_t k, int32_t out_h,
                       int32_t out_w, uint8_t* out, int32_t* index);

/* clip_sample_frames for NV12 frames (device u8 [n_frames][height*3/2][width]): each
 * bilinear tap is converted by O0 before O11 — identical to converting the whole frame
 * to RGB24 first.  Same outputs, errors and asynchrony as clip_sample_frames. */
int clip_sample_frames_nv12(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                            int32_t width, const int32_t* cuts, int64_t n_cuts, int32_t k,
                            int32_t out_h, int32_t out_w, uint8_t* out, int32_t* index);

/* ---------------------------------------------------------------- batch API */

#define CLIP_FORMAT_RGB24 0 /* u8 [n][H][W][3]                */
#define CLIP_FORMAT_NV12 1  /* u8 [n][H*3/2][W] (see above)    */

/* Frame source callback: fill dst (device, in the video's format) with frames
 * first_frame..first_frame+n-1 of video `video_index` on `stream`; return 0
 * on success.  Used when clip_video.frames is NULL. */
typedef int (*clip_fill_fn)(void* user, int64_t video_index, int64_t first_frame, int64_t n,
                            uint8_t* dst, uintptr_t stream);

typedef struct {
  int64_t id;             /* caller's id, copied to the result           */
  int64_t n_frames;       /* >= 1                                        */
  int32_t height, width;  /* H*W % 16 == 0 (NV12: H, W even, H*W % 32 == 0) */
  int32_t dim;            /* embedding dim (same for all videos) or 0    */
  int32_t format;         /* CLIP_FORMAT_RGB24 (0) or CLIP_FORMAT_NV12   */
  const uint8_t* frames;  /* device or host (pinned or pageable) pointer, or NULL = fill callback */
  const float* emb;       /* device [n_frames][dim] or NULL (no merge: final = detected) */
} clip_video;

typedef struct {
  int64_t id;
  int64_t n_candidates;   /* O4 candidates                                */
  int64_t n_detected;     /* O5/O6 cuts                                   */
  int64_t n_final;        /* O9 cuts                                      */
  int64_t n_band_hits;
  int64_t detected_offset; /* into cut_buf: detected cuts                 */
  int64_t final_offset;    /* into cut_buf: final cuts                    */
  int32_t rounds;
  int32_t reserved;
} clip_video_result;

/* Optional extra outputs of clip_run_videos (any field may be NULL). */
typedef struct {
  uint32_t* hist;      /* device u32 [sum n_frames][nbins]: per-frame histograms, videos in order */
  uint32_t* l1;        /* device u32 [sum n_frames]                                             */
  double* detected_cos; /* host f64 [cut_capacity], parallel to the detected cuts in cut_buf     */
} clip_run_outputs;

/* All rows a1-a9 for a batch of videos on this ctx's GPU.  SYNC.
 *   chunk_frames: frames per staging chunk for host/callback frames (0 = ~1 GiB)
 *   cut_buf      host i32 [cut_capacity]: per video its detected cuts then its final cuts
 *   results      host [n_videos]
 *   out          optional extra outputs or NULL.
 * Device-resident videos are scanned by ONE K1 launch (frame-descriptor
 * table), host/callback videos chunk by chunk through ctx staging buffers.
 * Errors: CLIP_E_CAPACITY if cut_capacity < sum over videos of 2*floor(n/L_min)+2. */
int clip_run_videos(clip_ctx* ctx, const clip_video* videos, int32_t n_videos, clip_fill_fn fill,
                    void* user, int64_t chunk_frames, int32_t* cut_buf, int64_t cut_capacity,
                    clip_video_result* results, const clip_run_outputs* out);

/* ------------------------------------------------------- stats and test hooks */

typedef struct {
  double k1_ms;        /* CUDA-event time of K1 (hist) launches since reset (CLIP_FLAG_TIMING) */
  double k2_ms;        /* L1 + threshold + compaction + greedy                           */
  double k3_ms;        /* merge                                                           */
  double total_ms;     /* first to last event of clip_run_videos calls                    */
  int64_t k1_launches; /* K1 launches since reset                                         */
  int64_t launches;    /* all kernel launches since reset                                 */
  int64_t k1_bytes;    /* frame bytes scanned by K1 since reset                           */
  int64_t memcpy_h2d;  /* bytes copied host->device by the library since reset            */
  int64_t memcpy_d2h;  /* bytes copied device->host by the library since reset            */
} clip_stats;

/* Read (SYNC) and optionally reset the ctx counters. */
int clip_get_stats(clip_ctx* ctx, clip_stats* out, int reset);

/* Test hook (K5): the device bin function of the hot path over all 2^24
 * colours into table (device u8 [2][1<<24], index (r<<16)|(g<<8)|b):
 * table[0] = the colour evaluated in lane 0 of the two-pixel code, table[1]
 * = in lane 1 (identical for the generic bins).  Async. */
int clip_debug_binmap(clip_ctx* ctx, uint8_t* table);

/* Test hook (K5, NV12): the fused conversion + bin function over every
 * (Y, U, V) into table (device u8 [2][1<<24], index (Y<<16)|(U<<8)|V):
 * table[0] = Y evaluated in lane 0 of a pixel pair sharing chroma (U, V),
 * table[1] = in lane 1 (the lane-0 pixel then has luma Y ^ 0x5A).  Async. */
int clip_debug_nv12map(clip_ctx* ctx, uint8_t* table);

/* Bench hook (K6): stream n_frames frames through K1's TMA pipeline without
 * binning (the read roofline of the same kernel skeleton).  Async. */
int clip_debug_read_roofline(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames,
                             int32_t height, int32_t width);
/* K6 for NV12 frames (the fused NV12 kernel's TMA pipeline without binning;
 * needs width % 16 == 0).  Async. */
int clip_debug_read_roofline_nv12(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames,
                                  int32_t height, int32_t width);

#ifdef __cplusplus
}
#endif

#endif /* CLIP_DETECT_H_ */
