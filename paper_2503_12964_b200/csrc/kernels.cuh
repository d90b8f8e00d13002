// kernels.cuh — host-side launchers of the libclipdetect kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace clipdetect {

enum { kModeFast = 0, kModeGeneric = 1, kModeRead = 2 };

// ---- K1 (hist.cu)
int64_t k1_stages(int64_t groups);  // K1 stages of a frame of `groups` 48-byte groups
cudaError_t k1_configure();
// The fast path's shared-memory tables, built once per context into global
// memory (kK1TableBytes each: the 64 KiB hue table, then the 8 KiB code -> bin
// map) and moved into every CTA by one TMA bulk copy at launch instead of
// being recomputed per CTA per launch.  hash: kHashRgb (K1) or kHashNv12.
constexpr int kK1TableBytes = 65536 + 8192;
cudaError_t k1_tables_build(uint8_t* d_tables, int hash, cudaStream_t stream);
// persistent grid of min(total_stages, sm_count) CTAs; tables: k1_tables_build(kHashRgb)
cudaError_t k1_launch(int mode, const HistSeg* d_segs, int32_t nseg, int64_t total_stages,
                      uint32_t nh, uint32_t ns, uint32_t nv, const uint8_t* tables,
                      uint32_t* sink, int sm_count, cudaStream_t stream);
cudaError_t k5_binmap_launch(uint8_t* out, uint32_t nh, uint32_t ns, uint32_t nv, int fast,
                             cudaStream_t stream);

// ---- K1 for NV12 input (hist_nv12.cu)
int nv12_stage_rows(int32_t width);
bool nv12_fast_ok(int32_t width, uint32_t nh, uint32_t ns, uint32_t nv);
int nv12_generic_rows();
cudaError_t k1_nv12_configure();
// mode kModeFast / kModeRead: persistent TMA kernel over `total` stages;
// kModeGeneric: generic kernel over `total` (frame, 8-block-row) items.
// tables: k1_tables_build(kHashNv12)
cudaError_t k1_nv12_launch(int mode, const Nv12Seg* d_segs, int32_t nseg, int64_t total,
                           uint32_t nh, uint32_t ns, uint32_t nv, const uint8_t* tables,
                           uint32_t* sink, int sm_count, cudaStream_t stream);
cudaError_t k5_nv12map_launch(uint8_t* out, uint32_t nh, uint32_t ns, uint32_t nv, int fast,
                              cudaStream_t stream);

// ---- K4 (sample.cu): clip frame sampling + resize (NEXT f3)
int k4_rows_per_band(int32_t W, bool nv12);
int k4_max_width();
cudaError_t k4_sample_launch(const uint8_t* frames, int64_t n, int32_t H, int32_t W,
                             const int32_t* cuts, int32_t n_cuts, int32_t k, int32_t H2, int32_t W2,
                             uint8_t* out, int32_t* index, bool nv12, cudaStream_t stream);

// ---- K2 (cuts.cu)
struct VideoDesc {
  int64_t fbase;  // first frame in the batch's flat frame space
  int64_t n;      // frames
  int64_t npix;   // H*W
};
constexpr int kCompactFrames = 128;  // frames per compaction block

// l1/score for frames [0, F) of the flat frame space (+ optional candidate
// flags compacted in order per 128-frame block).
cudaError_t k2_l1_launch(const uint32_t* hist, int64_t F, const VideoDesc* d_vids, int32_t nvid,
                         uint32_t nbins, const uint32_t* prev_hist, uint32_t* l1, float* score,
                         uint64_t tau_ppm, int32_t* cand_slots, int32_t* cand_count,
                         cudaStream_t stream);
// f4 variants: O3' distances (kind 1 chi-square, 2 Bhattacharyya, 3 1 - correlation;
// f32 scores; flags d >= tau unless adaptive) and / or O4'' adaptive flags on L1
// (adaptive_w > 0), then ordered compaction of the flags.
cudaError_t k2_variant_launch(const uint32_t* hist, const uint32_t* l1, int64_t F,
                              const VideoDesc* d_vids, int32_t nvid, uint32_t nbins,
                              const uint32_t* prev_hist, int kind, int32_t adaptive_w,
                              uint64_t ratio_ppm, uint64_t tau_ppm, float* score, uint8_t* flags,
                              int32_t* cand_slots, int32_t* cand_count, int* launches,
                              cudaStream_t stream);
// greedy min-length + tail per video (one warp per video) over the compacted candidates.
cudaError_t k2_greedy_launch(const VideoDesc* d_vids, int32_t nvid, const int32_t* cand_slots,
                             const int32_t* cand_count, int64_t l_min, int32_t* cuts,
                             int32_t* n_cuts, int32_t* n_cand, cudaStream_t stream);
// streaming clip_cuts: compaction of one l1 chunk + stateful greedy.
cudaError_t k2_stream_launch(const uint32_t* l1, int64_t n, int64_t npix, uint64_t tau_ppm,
                             int64_t l_min, void* state, int32_t* cuts, int64_t cap,
                             int is_final, int32_t* cand_slots, int32_t* cand_count,
                             cudaStream_t stream);

// ---- K3 (merge.cu)
struct MergeVideo {
  const float* emb;    // device [n][dim]
  int64_t n;           // frames
  int64_t cut_base;    // offset of this video's detected cuts in the cuts array
  int32_t clip_base;   // first global clip index
  int32_t n_clips;     // n_cuts + 1
};
constexpr int kPieceFrames = 16;  // frames per piece-sum CTA (parallelism over the frame axis)

struct MergeScratch {
  int32_t* clip_video;  // [K]
  int32_t* clip_f0;     // [K]
  int32_t* clip_f1;     // [K]
  int32_t* piece_base;  // [K+1]
  double* P;            // [pieces][dim]
  double* S;            // [K][dim]
  int32_t* alive;       // [K]  right-clip index of each alive boundary
  int32_t* alive2;      // [K]
  double* cos_b;        // [K]  per alive boundary
  double* cos_clip;     // [K]  per right-clip: cosine at its last evaluation
  double* norm2;        // [K]  |S|^2 of the range starting at clip k
  int32_t* run_dest;    // [K]  per run of merged boundaries: the range it joins
  int32_t* run_lo;      // [K]  first merged boundary of the run (alive index)
  int32_t* run_hi;      // [K]  one past the last
  int32_t* run_cbase;   // [K+1] first partial-sum chunk of each run
  int64_t* counters;    // [8]  n_alive, merges this round, runs, chunks, next n_alive
  int32_t* Kd;          // [1]  K, the total clip count (written by k3_video_table_kernel)
  int64_t* vstate;      // [nv][4] done, rounds, band hits, merges this round (+ alive via vstate2)
  int64_t* valive;      // [nv] alive boundaries of the video after the round
};

// Device-side sizing: K (the clip count) and the piece count exist only on the
// device (s.Kd, piece_base[K]); the host passes upper bounds (Kub >= K, from the
// minimum clip length) for grids and scratch.  d_ncuts: K2's per-video cut
// counts (the video table's n_clips / clip_base are filled from them), or null
// when the host filled n_clips.
cudaError_t k3_prepare_launch(MergeVideo* d_mv, int32_t nv, int32_t Kub, const int32_t* d_ncuts,
                              const int32_t* cuts, MergeScratch s, cudaStream_t stream);
// stride: O8' keyframe stride (1 = every frame)
cudaError_t k3_piece_sum_launch(const MergeVideo* d_mv, int32_t dim, int64_t pieces_bound,
                                int32_t stride, MergeScratch s, cudaStream_t stream);
cudaError_t k3_clip_sum_launch(int32_t Kub, int32_t dim, MergeScratch s, cudaStream_t stream);
// every merge round of every video on the device (one cooperative launch; the
// alive list ends in s.alive, its length in s.counters[0]); max_alive bounds
// the boundaries (grid size); max_rounds 0 = until the fixed point.
cudaError_t k3_rounds_launch(const MergeVideo* d_mv, int32_t nv, int32_t dim, int64_t max_alive,
                             double theta, double band_rel, int32_t max_rounds, int sm_count,
                             MergeScratch s, cudaStream_t stream);
// final cuts per video at cuts-array layout (offset cut_base, count n_final[v])
// and the per-detected-cut cosines (same layout), from the alive list.
cudaError_t k3_finish_launch(const MergeVideo* d_mv, int32_t nv, int32_t Kub, MergeScratch s,
                             int32_t* final_cuts, int32_t* n_final, double* detected_cos,
                             cudaStream_t stream);

}  // namespace clipdetect
