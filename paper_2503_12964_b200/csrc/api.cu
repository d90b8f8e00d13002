// api.cu — the C ABI of libclipdetect (include/clip_detect.h): validation,
// ctx scratch management, launch bookkeeping.  All arithmetic of rows a1-a9
// runs in the kernels of hist.cu (K1), cuts.cu (K2) and merge.cu (K3); the
// host code here only validates, sizes grids, uploads descriptor tables and
// copies results.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/clip_detect.h"
#include "binfn.cuh"
#include "kernels.cuh"

using namespace clipdetect;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Events {
  cudaEvent_t e[2] = {nullptr, nullptr};
};

}  // namespace

struct clip_ctx {
  clip_params p{};
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;
  int sm_count = kSMs;
  bool sticky = false;
  std::string err;
  clip_stats stats{};
  // scratch
  DevBuf segs, segs2, flags, vids, hist, l1, cand_slots, cand_count, cuts, ncuts, ncand, final_cuts, nfinal,
      detcos, pack, pack_cos, sink;
  DevBuf m_video, m_clip_video, m_f0, m_f1, m_piece_base, m_P, m_S, m_alive, m_alive2, m_cos_b,
      m_cos_clip, m_norm2, m_runs, m_counters, m_vstate, m_valive;
  DevBuf staging[2];
  cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
  // timing
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_spans;  // (kind, start/end)
  // pinned host staging for small D2H
  void* hpin = nullptr;
  size_t hpin_bytes = 0;
  // K1 / K1-NV12 shared-memory tables (k1_tables_build; RGB then NV12), built once
  DevBuf tables;
  // pinned double buffer for small H2D descriptor tables: a pageable
  // cudaMemcpyAsync would block the host until the stream drains, so every
  // streamed chunk's K1 launch would wait for the previous one
  uint8_t* dpin = nullptr;
  cudaEvent_t desc_ev[2] = {nullptr, nullptr};
  int desc_half = 0;
};
constexpr size_t kDescHalf = 128 << 10;

namespace {

int fail(clip_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) {
    c->err = buf;
    if (code == CLIP_E_CUDA) c->sticky = true;
  }
  return code;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(ctx, CLIP_E_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                               \
  } while (0)

#define CKS(call)                       \
  do {                                  \
    int s_ = (call);                    \
    if (s_ != CLIP_OK) return s_;       \
  } while (0)

// Host -> device copy of a small descriptor table on the ctx stream through the
// pinned double buffer (falls back to a plain copy above kDescHalf bytes).
int upload(clip_ctx* ctx, void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return CLIP_OK;
  if (bytes > kDescHalf) {
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return CLIP_OK;
  }
  const int h = ctx->desc_half;
  ctx->desc_half ^= 1;
  CK(cudaEventSynchronize(ctx->desc_ev[h]));  // the copy that last used this half is done
  uint8_t* stage = ctx->dpin + h * kDescHalf;
  memcpy(stage, src, bytes);
  CK(cudaMemcpyAsync(dst, stage, bytes, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaEventRecord(ctx->desc_ev[h], ctx->stream));
  return CLIP_OK;
}

int ensure(clip_ctx* ctx, DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.bytes >= bytes) return CLIP_OK;
  if (b.p) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaFree(b.p));
    b.p = nullptr;
    b.bytes = 0;
  }
  size_t want = std::max(bytes, b.bytes + b.bytes / 2);
  if (cudaMalloc(&b.p, want) != cudaSuccess) {
    cudaGetLastError();
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) {
      cudaGetLastError();
      b.p = nullptr;
      return fail(ctx, CLIP_E_NOMEM, "cudaMalloc(%zu) failed", bytes);
    }
    want = bytes;
  }
  b.bytes = want;
  return CLIP_OK;
}

template <class T>
T* P(DevBuf& b) {
  return reinterpret_cast<T*>(b.p);
}

int ensure_pinned(clip_ctx* ctx, size_t bytes) {
  if (ctx->hpin_bytes >= bytes) return CLIP_OK;
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  ctx->hpin = nullptr;
  ctx->hpin_bytes = 0;
  size_t want = std::max(bytes, (size_t)1 << 20);
  CK(cudaMallocHost(&ctx->hpin, want));
  ctx->hpin_bytes = want;
  return CLIP_OK;
}

bool timing(const clip_ctx* ctx) { return (ctx->p.flags & CLIP_FLAG_TIMING) != 0; }

cudaEvent_t next_event(clip_ctx* ctx) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->ev_used++];
}

// kind: 0 = K1, 1 = K2, 2 = K3, 3 = whole call
struct Span {
  clip_ctx* ctx;
  int kind;
  cudaEvent_t a = nullptr;
  Span(clip_ctx* c, int k) : ctx(c), kind(k) {
    if (timing(ctx)) {
      a = next_event(ctx);
      cudaEventRecord(a, ctx->stream);
    }
  }
  void end() {
    if (a) {
      cudaEvent_t b = next_event(ctx);
      cudaEventRecord(b, ctx->stream);
      ctx->ev_spans.push_back({kind, {a, b}});
      a = nullptr;
    }
  }
};

// Called after a stream sync: fold recorded spans into the stats.
void harvest(clip_ctx* ctx) {
  for (auto& s : ctx->ev_spans) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s.second.first, s.second.second);
    if (s.first == 0) ctx->stats.k1_ms += ms;
    else if (s.first == 1) ctx->stats.k2_ms += ms;
    else if (s.first == 2) ctx->stats.k3_ms += ms;
    else ctx->stats.total_ms += ms;
  }
  ctx->ev_spans.clear();
  ctx->ev_used = 0;
}

int check_ctx(clip_ctx* ctx) {
  if (!ctx) return CLIP_E_INVALID;
  if (ctx->sticky) return fail(ctx, CLIP_E_STATE, "ctx unusable after CUDA error: %s", ctx->err.c_str());
  CK(cudaSetDevice(ctx->device));
  return CLIP_OK;
}

uint32_t nbins_of(const clip_params& p) { return p.h_bins * p.s_bins * p.v_bins; }

int k1_mode(const clip_params& p) {
  return (p.h_bins == 18 && p.s_bins == 3 && p.v_bins == 3) ? kModeFast : kModeGeneric;
}

// One K1 launch over a list of segments (hist pointers already set).
int launch_k1(clip_ctx* ctx, std::vector<HistSeg>& segs, int mode) {
  int64_t total = 0;
  for (auto& s : segs) {
    s.stages = k1_stages(s.groups);
    s.stage_base = total;
    total += s.n_frames * s.stages;
  }
  if (total == 0) return CLIP_OK;
  CKS(ensure(ctx, ctx->segs, segs.size() * sizeof(HistSeg)));
  CKS(upload(ctx, ctx->segs.p, segs.data(), segs.size() * sizeof(HistSeg)));
  CKS(ensure(ctx, ctx->sink, 16));
  Span sp(ctx, 0);
  CK(k1_launch(mode, P<HistSeg>(ctx->segs), (int32_t)segs.size(), total, ctx->p.h_bins,
               ctx->p.s_bins, ctx->p.v_bins, P<uint8_t>(ctx->tables), P<uint32_t>(ctx->sink),
               ctx->sm_count, ctx->stream));
  sp.end();
  ctx->stats.k1_launches += 1;
  ctx->stats.launches += 1;
  for (auto& s : segs) ctx->stats.k1_bytes += s.n_frames * s.groups * 48;
  return CLIP_OK;
}

// One K1 launch per kernel kind over a list of NV12 segments: the fused TMA
// kernel for the segments it supports, the generic kernel for the rest.
int launch_k1_nv12(clip_ctx* ctx, const std::vector<Nv12Seg>& all, int mode) {
  const clip_params& p = ctx->p;
  std::vector<Nv12Seg> lists[2];  // 0 = fused (fast / read), 1 = generic
  for (const Nv12Seg& s0 : all) {
    Nv12Seg s = s0;
    const bool fast = mode == kModeRead || (mode == kModeFast && nv12_fast_ok(s.width, p.h_bins, p.s_bins, p.v_bins));
    s.rows = fast ? nv12_stage_rows(s.width) : nv12_generic_rows();
    s.stages = (s.height / 2 + s.rows - 1) / s.rows;
    lists[fast ? 0 : 1].push_back(s);
  }
  for (int k = 0; k < 2; ++k) {
    auto& segs = lists[k];
    if (segs.empty()) continue;
    int64_t total = 0;
    for (auto& s : segs) {
      s.stage_base = total;
      total += s.n_frames * s.stages;
    }
    CKS(ensure(ctx, k ? ctx->segs2 : ctx->segs, segs.size() * sizeof(Nv12Seg)));
    DevBuf& db = k ? ctx->segs2 : ctx->segs;
    CKS(upload(ctx, db.p, segs.data(), segs.size() * sizeof(Nv12Seg)));
    CKS(ensure(ctx, ctx->sink, 16));
    Span sp(ctx, 0);
    CK(k1_nv12_launch(k ? kModeGeneric : mode, P<Nv12Seg>(db), (int32_t)segs.size(), total,
                      p.h_bins, p.s_bins, p.v_bins, P<uint8_t>(ctx->tables) + kK1TableBytes,
                      P<uint32_t>(ctx->sink), ctx->sm_count, ctx->stream));
    sp.end();
    ctx->stats.k1_launches += 1;
    ctx->stats.launches += 1;
    for (auto& s : segs) ctx->stats.k1_bytes += s.n_frames * (int64_t)s.height * s.width * 3 / 2;
  }
  return CLIP_OK;
}

int validate_params(clip_ctx* ctx, const clip_params* p) {
  if (!p) return fail(ctx, CLIP_E_INVALID, "params is NULL");
  if (p->abi_version != CLIP_ABI_VERSION)
    return fail(ctx, CLIP_E_INVALID, "abi_version %u != %u", p->abi_version, CLIP_ABI_VERSION);
  if (p->h_bins < 1 || p->s_bins < 1 || p->v_bins < 1 || p->v_bins > 256 ||
      (uint64_t)p->h_bins * p->s_bins * p->v_bins > 256)
    return fail(ctx, CLIP_E_INVALID, "bins %u x %u x %u: need >= 1 each and product <= 256",
                p->h_bins, p->s_bins, p->v_bins);
  if (p->min_clip_frames < 1) return fail(ctx, CLIP_E_INVALID, "min_clip_frames must be >= 1");
  if (p->cut_threshold_ppm > 1000000) return fail(ctx, CLIP_E_INVALID, "cut_threshold_ppm > 1e6");
  if (!(p->merge_cos_threshold >= -1.0 && p->merge_cos_threshold <= 1.0))
    return fail(ctx, CLIP_E_INVALID, "merge_cos_threshold outside [-1, 1]");
  if (!(p->band_rel >= 0.0)) return fail(ctx, CLIP_E_INVALID, "band_rel < 0");
  if (p->reserved != 0) return fail(ctx, CLIP_E_INVALID, "reserved must be 0");
  if (p->distance > CLIP_DIST_CORREL) return fail(ctx, CLIP_E_INVALID, "unknown distance %u", p->distance);
  if (p->adaptive_window > 1024) return fail(ctx, CLIP_E_INVALID, "adaptive_window > 1024");
  if (p->adaptive_window > 0 && p->distance != CLIP_DIST_L1)
    return fail(ctx, CLIP_E_INVALID, "the adaptive threshold is defined on L1 (distance must be L1)");
  if (p->adaptive_ratio_ppm > 1000000000ull) return fail(ctx, CLIP_E_INVALID, "adaptive_ratio_ppm > 1e9");
  if (p->reserved2 != 0) return fail(ctx, CLIP_E_INVALID, "reserved2 must be 0");
  return CLIP_OK;
}

int validate_frames(clip_ctx* ctx, const void* frames, int64_t n, int32_t h, int32_t w,
                    bool allow_null, int format = CLIP_FORMAT_RGB24) {
  if (n < 1) return fail(ctx, CLIP_E_INVALID, "n_frames must be >= 1 (got %lld)", (long long)n);
  if (h < 1 || w < 1) return fail(ctx, CLIP_E_INVALID, "bad frame size %dx%d", w, h);
  if (format != CLIP_FORMAT_RGB24 && format != CLIP_FORMAT_NV12)
    return fail(ctx, CLIP_E_INVALID, "unknown frame format %d", format);
  if (format == CLIP_FORMAT_NV12 && ((h | w) & 1))
    return fail(ctx, CLIP_E_INVALID, "NV12 needs even height and width (got %dx%d)", w, h);
  if (((int64_t)h * w) % (format == CLIP_FORMAT_NV12 ? 32 : 16) != 0)
    return fail(ctx, CLIP_E_INVALID, "H*W = %lld is not a multiple of %d", (long long)h * w,
                format == CLIP_FORMAT_NV12 ? 32 : 16);
  // L1 <= 2 N is stored as u32 (O3): N < 2^31.  The correlation distance (O3')
  // sums nbins * sum(h^2) <= 256 N^2 in int64: N <= 2^27 (8K frames are 2^25).
  if ((int64_t)h * w >= (1ll << 31)) return fail(ctx, CLIP_E_INVALID, "frame too large (H*W >= 2^31)");
  if (ctx && ctx->p.distance == CLIP_DIST_CORREL && (int64_t)h * w > (1ll << 27))
    return fail(ctx, CLIP_E_INVALID, "correlation distance needs H*W <= 2^27");
  if (!frames && !allow_null) return fail(ctx, CLIP_E_INVALID, "frames is NULL");
  if (frames && ((uintptr_t)frames & 15)) return fail(ctx, CLIP_E_INVALID, "frames not 16-byte aligned");
  return CLIP_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------------ merge core
// Enqueues K3 on the detected cuts (device, per video at cut_base) of nv
// videos; nothing is read back here.  mvh: emb, n, cut_base per video, and
// n_clips when d_ncuts is null (else the device fills n_clips / clip_base from
// K2's counts).  Kub >= the clip count K (the host knows only this bound when
// the counts stay on the device).  Writes final cuts (same layout), n_final[v]
// and detected cosines (device); the per-video state [nv][4] is in ctx->m_vstate.
int run_merge(clip_ctx* ctx, const std::vector<MergeVideo>& mvh, int32_t dim, const int32_t* d_cuts,
              const int32_t* d_ncuts, int64_t Kub, int32_t* d_final, int32_t* d_nfinal,
              double* d_detcos) {
  const int32_t nv = (int32_t)mvh.size();
  int64_t pieces = Kub;  // sum over clips of ceil(len / kPieceFrames) <= n / kPieceFrames + clips
  for (auto& m : mvh) pieces += (m.n + kPieceFrames - 1) / kPieceFrames;
  if (Kub > INT32_MAX || pieces > INT32_MAX)
    return fail(ctx, CLIP_E_INVALID, "too many clips for one merge (%lld)", (long long)Kub);
  const int64_t K = Kub;
  CKS(ensure(ctx, ctx->m_video, sizeof(MergeVideo) * nv));
  CKS(ensure(ctx, ctx->m_clip_video, 4 * K));
  CKS(ensure(ctx, ctx->m_f0, 4 * K));
  CKS(ensure(ctx, ctx->m_f1, 4 * K));
  CKS(ensure(ctx, ctx->m_piece_base, 4 * (K + 1)));
  CKS(ensure(ctx, ctx->m_P, sizeof(double) * pieces * dim));
  CKS(ensure(ctx, ctx->m_S, sizeof(double) * K * dim));
  CKS(ensure(ctx, ctx->m_alive, 4 * K));
  CKS(ensure(ctx, ctx->m_alive2, 4 * K));
  CKS(ensure(ctx, ctx->m_cos_b, 8 * K));
  CKS(ensure(ctx, ctx->m_cos_clip, 8 * K));
  CKS(ensure(ctx, ctx->m_norm2, 8 * K));
  CKS(ensure(ctx, ctx->m_runs, 4 * (4 * K + 1)));
  CKS(ensure(ctx, ctx->m_counters, 8 * 9));
  CKS(ensure(ctx, ctx->m_vstate, 8 * 4 * nv));
  CKS(ensure(ctx, ctx->m_valive, 8 * nv));
  CKS(upload(ctx, ctx->m_video.p, mvh.data(), sizeof(MergeVideo) * nv));
  CK(cudaMemsetAsync(ctx->m_cos_clip.p, 0, 8 * K, ctx->stream));
  MergeScratch s;
  s.clip_video = P<int32_t>(ctx->m_clip_video);
  s.clip_f0 = P<int32_t>(ctx->m_f0);
  s.clip_f1 = P<int32_t>(ctx->m_f1);
  s.piece_base = P<int32_t>(ctx->m_piece_base);
  s.P = P<double>(ctx->m_P);
  s.S = P<double>(ctx->m_S);
  s.alive = P<int32_t>(ctx->m_alive);
  s.alive2 = P<int32_t>(ctx->m_alive2);
  s.cos_b = P<double>(ctx->m_cos_b);
  s.cos_clip = P<double>(ctx->m_cos_clip);
  s.norm2 = P<double>(ctx->m_norm2);
  s.run_dest = P<int32_t>(ctx->m_runs);
  s.run_lo = s.run_dest + K;
  s.run_hi = s.run_lo + K;
  s.run_cbase = s.run_hi + K;
  s.counters = P<int64_t>(ctx->m_counters);
  s.Kd = reinterpret_cast<int32_t*>(s.counters + 8);
  s.vstate = P<int64_t>(ctx->m_vstate);
  s.valive = P<int64_t>(ctx->m_valive);
  MergeVideo* d_mv = P<MergeVideo>(ctx->m_video);

  Span sp(ctx, 2);
  CK(k3_prepare_launch(d_mv, nv, (int32_t)K, d_ncuts, d_cuts, s, ctx->stream));
  CK(k3_piece_sum_launch(d_mv, dim, pieces, ctx->p.emb_stride > 1 ? (int32_t)ctx->p.emb_stride : 1,
                         s, ctx->stream));
  CK(k3_clip_sum_launch((int32_t)K, dim, s, ctx->stream));
  ctx->stats.launches += 5;
  if (K - nv > 0) {
    CK(k3_rounds_launch(d_mv, nv, dim, K - nv, ctx->p.merge_cos_threshold, ctx->p.band_rel,
                        (int32_t)ctx->p.max_merge_rounds, ctx->sm_count, s, ctx->stream));
    ctx->stats.launches += 1;
  }
  CK(k3_finish_launch(d_mv, nv, (int32_t)K, s, d_final, d_nfinal, d_detcos, ctx->stream));
  ctx->stats.launches += 1;
  sp.end();
  return CLIP_OK;
}

// Result summary of a clip_run_videos call, one int64 row per video (after a
// leading total): the counts and state the host reports, and the video's
// offset in the packed cut buffer (exclusive scan of 2 * n_detected).
enum { SUM_NCUTS = 0, SUM_NCAND, SUM_NFINAL, SUM_OFF, SUM_BAND, SUM_ROUNDS, SUM_W };

__global__ void __launch_bounds__(1024)
summary_kernel(int32_t nvid, const int32_t* __restrict__ ncuts, const int32_t* __restrict__ ncand,
               const int32_t* __restrict__ nfin, const int64_t* __restrict__ vstate,
               int64_t* __restrict__ sum) {
  __shared__ int64_t wsum[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t carry = 0;
  for (int32_t base = 0; base < nvid; base += 1024) {
    const int32_t v = base + threadIdx.x;
    const int64_t x = v < nvid ? 2 * (int64_t)ncuts[v] : 0;
    int64_t inc = x;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      const int64_t w = wsum[lane];
      int64_t wi = w;
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += y;
      }
      wsum[lane] = wi - w;
      if (lane == 31) wsum[32] = wi;
    }
    __syncthreads();
    if (v < nvid) {
      int64_t* r = sum + 1 + (int64_t)SUM_W * v;
      r[SUM_NCUTS] = ncuts[v];
      r[SUM_NCAND] = ncand[v];
      r[SUM_NFINAL] = nfin ? nfin[v] : ncuts[v];
      r[SUM_OFF] = carry + wsum[warp] + inc - x;
      r[SUM_BAND] = vstate ? vstate[4 * v + 2] : 0;
      r[SUM_ROUNDS] = vstate ? vstate[4 * v + 1] : 0;
    }
    carry += wsum[32];
    __syncthreads();
  }
  if (threadIdx.x == 0) sum[0] = carry;
}

// pack per-video detected / final cuts and cosines into contiguous buffers:
// video v at sum row v's offset, [detected | final (n_detected reserved)]
__global__ void pack_kernel(const VideoDesc* __restrict__ vids, int32_t nvid, int64_t F,
                            const int32_t* __restrict__ cuts, const int32_t* __restrict__ ncuts,
                            const int32_t* __restrict__ fin, const int32_t* __restrict__ nfin,
                            const double* __restrict__ detcos, const int64_t* __restrict__ sum,
                            int32_t* __restrict__ out, double* __restrict__ out_cos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= F) return;
  int32_t lo = 0, hi = nvid - 1;
  while (lo < hi) {
    const int32_t m = (lo + hi + 1) >> 1;
    if (vids[m].fbase <= i) lo = m; else hi = m - 1;
  }
  const int64_t j = i - vids[lo].fbase;
  const int64_t det_off = sum[1 + (int64_t)SUM_W * lo + SUM_OFF];
  if (j < ncuts[lo]) {
    out[det_off + j] = cuts[i];
    if (out_cos) out_cos[det_off + j] = detcos ? detcos[i] : 0.0;
  }
  if (j < nfin[lo]) out[det_off + ncuts[lo] + j] = fin[i];
}

}  // namespace

// =================================================================== C ABI
extern "C" {

void clip_params_default(clip_params* p) {
  if (!p) return;
  memset(p, 0, sizeof *p);
  p->abi_version = CLIP_ABI_VERSION;
  p->h_bins = 18;
  p->s_bins = 3;
  p->v_bins = 3;
  p->cut_threshold_ppm = 300000;
  p->min_clip_frames = 8;
  p->max_merge_rounds = 0;
  p->merge_cos_threshold = 0.90;
  p->band_rel = 1e-5;
  p->flags = 0;
  p->distance = CLIP_DIST_L1;
  p->adaptive_window = 0;
  p->adaptive_ratio_ppm = 3000000;
  p->emb_stride = 1;
}

int clip_detect_init(clip_ctx** out, const clip_params* p, int cuda_device, uintptr_t cuda_stream) {
  if (!out) return CLIP_E_INVALID;
  *out = nullptr;
  int st = validate_params(nullptr, p);
  if (st) return st;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) {
    cudaGetLastError();
    return CLIP_E_INVALID;
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, cuda_device) != cudaSuccess) return CLIP_E_CUDA;
  if (!(prop.major == 10 && prop.minor == 0)) return CLIP_E_ARCH;
  clip_ctx* ctx = new clip_ctx();
  ctx->p = *p;
  ctx->device = cuda_device;
  ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
  ctx->sm_count = prop.multiProcessorCount;
  if (cudaSetDevice(cuda_device) != cudaSuccess || k1_configure() != cudaSuccess ||
      k1_nv12_configure() != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return CLIP_E_CUDA;
  }
  for (int i = 0; i < 2; ++i) {
    cudaEventCreateWithFlags(&ctx->copied[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->consumed[i], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ctx->desc_ev[i], cudaEventDisableTiming);
  }
  // the fast paths' shared-memory tables, once per context
  if (cudaMallocHost(reinterpret_cast<void**>(&ctx->dpin), 2 * kDescHalf) != cudaSuccess ||
      ensure(ctx, ctx->tables, 2 * kK1TableBytes) != CLIP_OK ||
      k1_tables_build(P<uint8_t>(ctx->tables), kHashRgb, ctx->stream) != cudaSuccess ||
      k1_tables_build(P<uint8_t>(ctx->tables) + kK1TableBytes, kHashNv12, ctx->stream) != cudaSuccess ||
      cudaStreamSynchronize(ctx->stream) != cudaSuccess) {
    cudaGetLastError();
    clip_detect_destroy(ctx);
    return CLIP_E_CUDA;
  }
  *out = ctx;
  return CLIP_OK;
}

int clip_detect_destroy(clip_ctx* ctx) {
  if (!ctx) return CLIP_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  DevBuf* bufs[] = {&ctx->segs, &ctx->segs2, &ctx->flags, &ctx->vids, &ctx->hist, &ctx->l1, &ctx->cand_slots,
                    &ctx->cand_count, &ctx->cuts, &ctx->ncuts, &ctx->ncand, &ctx->final_cuts,
                    &ctx->nfinal, &ctx->detcos, &ctx->pack, &ctx->pack_cos, &ctx->sink,
                    &ctx->m_video, &ctx->m_clip_video, &ctx->m_f0, &ctx->m_f1,
                    &ctx->m_piece_base, &ctx->m_P, &ctx->m_S, &ctx->m_alive, &ctx->m_alive2,
                    &ctx->m_cos_b, &ctx->m_cos_clip, &ctx->m_norm2, &ctx->m_runs,
                    &ctx->m_counters, &ctx->m_vstate,
                    &ctx->m_valive, &ctx->staging[0], &ctx->staging[1], &ctx->tables};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (int i = 0; i < 2; ++i) {
    if (ctx->copied[i]) cudaEventDestroy(ctx->copied[i]);
    if (ctx->consumed[i]) cudaEventDestroy(ctx->consumed[i]);
    if (ctx->desc_ev[i]) cudaEventDestroy(ctx->desc_ev[i]);
  }
  if (ctx->dpin) cudaFreeHost(ctx->dpin);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->hpin) cudaFreeHost(ctx->hpin);
  delete ctx;
  return CLIP_OK;
}

const char* clip_last_error(const clip_ctx* ctx) { return ctx ? ctx->err.c_str() : "null ctx"; }

}  // extern "C"

namespace {
int frame_scores(clip_ctx* ctx, int format, const uint8_t* frames, int64_t n_frames,
                 int32_t height, int32_t width, const uint32_t* prev_hist, uint32_t* hist,
                 uint32_t* l1, float* score) {
  CKS(check_ctx(ctx));
  CKS(validate_frames(ctx, frames, n_frames, height, width, false, format));
  if (!hist) return fail(ctx, CLIP_E_INVALID, "hist is NULL");
  const uint32_t nbins = nbins_of(ctx->p);
  const int64_t npix = (int64_t)height * width;
  CK(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * nbins * n_frames, ctx->stream));
  if (format == CLIP_FORMAT_NV12) {
    std::vector<Nv12Seg> segs(1);
    segs[0] = Nv12Seg{frames, hist, n_frames, height, width, 0, 0, 0};
    CKS(launch_k1_nv12(ctx, segs, k1_mode(ctx->p)));
  } else {
    std::vector<HistSeg> segs(1);
    segs[0].frames = frames;
    segs[0].hist = hist;
    segs[0].n_frames = n_frames;
    segs[0].groups = npix / 16;
    CKS(launch_k1(ctx, segs, k1_mode(ctx->p)));
  }
  if (l1 || score) {
    VideoDesc vd{0, n_frames, npix};
    CKS(ensure(ctx, ctx->vids, sizeof(VideoDesc)));
    CKS(upload(ctx, ctx->vids.p, &vd, sizeof vd));
    Span sp(ctx, 1);
    const bool var = ctx->p.distance != CLIP_DIST_L1;
    CK(k2_l1_launch(hist, n_frames, P<VideoDesc>(ctx->vids), 1, nbins, prev_hist, l1,
                    var ? nullptr : score, ctx->p.cut_threshold_ppm, nullptr, nullptr, ctx->stream));
    ctx->stats.launches += 1;
    if (var && score) {
      int nl = 0;
      CK(k2_variant_launch(hist, l1, n_frames, P<VideoDesc>(ctx->vids), 1, nbins, prev_hist,
                           (int)ctx->p.distance, 0, 0, ctx->p.cut_threshold_ppm, score, nullptr,
                           nullptr, nullptr, &nl, ctx->stream));
      ctx->stats.launches += nl;
    }
    sp.end();
  }
  return CLIP_OK;
}
}  // namespace

extern "C" {

int clip_frame_scores(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                      int32_t width, const uint32_t* prev_hist, uint32_t* hist, uint32_t* l1,
                      float* score) {
  return frame_scores(ctx, CLIP_FORMAT_RGB24, frames, n_frames, height, width, prev_hist, hist,
                      l1, score);
}

int clip_frame_scores_nv12(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                           int32_t width, const uint32_t* prev_hist, uint32_t* hist, uint32_t* l1,
                           float* score) {
  return frame_scores(ctx, CLIP_FORMAT_NV12, frames, n_frames, height, width, prev_hist, hist,
                      l1, score);
}

int clip_hist_scores(clip_ctx* ctx, const uint32_t* hist, int64_t n_frames, int64_t pixels_per_frame,
                     const uint32_t* prev_hist, uint32_t* l1, float* score) {
  CKS(check_ctx(ctx));
  if (!hist || n_frames < 1 || pixels_per_frame < 1 || pixels_per_frame >= (1ll << 31) ||
      (ctx->p.distance == CLIP_DIST_CORREL && pixels_per_frame > (1ll << 27)))
    return fail(ctx, CLIP_E_INVALID, "bad histograms (n %lld, N %lld)", (long long)n_frames,
                (long long)pixels_per_frame);
  const uint32_t nbins = nbins_of(ctx->p);
  VideoDesc vd{0, n_frames, pixels_per_frame};
  CKS(ensure(ctx, ctx->vids, sizeof(VideoDesc)));
  CKS(upload(ctx, ctx->vids.p, &vd, sizeof vd));
  Span sp(ctx, 1);
  const bool var = ctx->p.distance != CLIP_DIST_L1;
  CK(k2_l1_launch(hist, n_frames, P<VideoDesc>(ctx->vids), 1, nbins, prev_hist, l1,
                  var ? nullptr : score, ctx->p.cut_threshold_ppm, nullptr, nullptr, ctx->stream));
  ctx->stats.launches += 1;
  if (var && score) {
    int nl = 0;
    CK(k2_variant_launch(hist, l1, n_frames, P<VideoDesc>(ctx->vids), 1, nbins, prev_hist,
                         (int)ctx->p.distance, 0, 0, ctx->p.cut_threshold_ppm, score, nullptr,
                         nullptr, nullptr, &nl, ctx->stream));
    ctx->stats.launches += nl;
  }
  sp.end();
  return CLIP_OK;
}

int clip_cuts(clip_ctx* ctx, const uint32_t* l1, int64_t n_frames, int64_t pixels_per_frame,
              clip_cut_state* state, int32_t* cuts, int64_t cuts_capacity, int is_final_chunk) {
  CKS(check_ctx(ctx));
  if (n_frames < 0) return fail(ctx, CLIP_E_INVALID, "n_frames < 0");
  if (n_frames > 0 && !l1) return fail(ctx, CLIP_E_INVALID, "l1 is NULL");
  if (!state) return fail(ctx, CLIP_E_INVALID, "state is NULL");
  if (pixels_per_frame < 1) return fail(ctx, CLIP_E_INVALID, "pixels_per_frame < 1");
  if (ctx->p.distance != CLIP_DIST_L1 || ctx->p.adaptive_window > 0)
    return fail(ctx, CLIP_E_INVALID, "clip_cuts streams the default L1 rule only (use clip_run_videos for variants)");
  if (cuts_capacity < 0 || (cuts_capacity > 0 && !cuts))
    return fail(ctx, CLIP_E_INVALID, "bad cuts buffer");
  const int64_t blocks = (n_frames + kCompactFrames - 1) / kCompactFrames;
  CKS(ensure(ctx, ctx->cand_slots, 4 * std::max<int64_t>(1, blocks) * kCompactFrames));
  CKS(ensure(ctx, ctx->cand_count, 4 * std::max<int64_t>(1, blocks)));
  Span sp(ctx, 1);
  CK(k2_stream_launch(l1, n_frames, pixels_per_frame, ctx->p.cut_threshold_ppm,
                      ctx->p.min_clip_frames, state, cuts, cuts_capacity, is_final_chunk,
                      P<int32_t>(ctx->cand_slots), P<int32_t>(ctx->cand_count), ctx->stream));
  sp.end();
  ctx->stats.launches += n_frames > 0 ? 2 : 1;
  return CLIP_OK;
}

int clip_merge(clip_ctx* ctx, const float* emb, int64_t n_frames, int32_t dim,
               const int32_t* cuts, int64_t n_cuts, int32_t* merged, int64_t* n_merged,
               double* boundary_cos, int64_t* n_band_hits, int32_t* rounds) {
  CKS(check_ctx(ctx));
  if (!emb || n_frames < 1 || dim < 1 || dim > 65536)
    return fail(ctx, CLIP_E_INVALID, "bad embeddings (emb %p, n %lld, dim %d)", (const void*)emb,
                (long long)n_frames, dim);
  if (n_cuts < 0 || n_cuts >= n_frames || (n_cuts > 0 && (!cuts || !merged)))
    return fail(ctx, CLIP_E_INVALID, "bad cuts (n_cuts %lld)", (long long)n_cuts);
  if (!n_merged) return fail(ctx, CLIP_E_INVALID, "n_merged is NULL");
  if (n_frames > INT32_MAX) return fail(ctx, CLIP_E_INVALID, "n_frames too large");
  if (n_cuts == 0) {
    *n_merged = 0;
    if (n_band_hits) *n_band_hits = 0;
    if (rounds) *rounds = 0;
    return CLIP_OK;
  }
  std::vector<MergeVideo> mv(1);
  mv[0].emb = emb;
  mv[0].n = n_frames;
  mv[0].cut_base = 0;
  mv[0].clip_base = 0;
  mv[0].n_clips = (int32_t)n_cuts + 1;
  CKS(ensure(ctx, ctx->nfinal, 4));
  CKS(ensure_pinned(ctx, 64));
  CKS(run_merge(ctx, mv, dim, cuts, nullptr, n_cuts + 1, merged, P<int32_t>(ctx->nfinal),
                boundary_cos));
  // one read-back: the video state [4] and n_final
  int64_t* hp = reinterpret_cast<int64_t*>(ctx->hpin);
  CK(cudaMemcpyAsync(hp, ctx->m_vstate.p, 8 * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaMemcpyAsync(hp + 4, ctx->nfinal.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stats.memcpy_d2h += 8 * 4 + 4;
  int32_t nf = 0;
  memcpy(&nf, hp + 4, 4);
  harvest(ctx);
  *n_merged = nf;
  if (n_band_hits) *n_band_hits = hp[2];
  if (rounds) *rounds = (int32_t)hp[1];
  return CLIP_OK;
}

int clip_run_videos(clip_ctx* ctx, const clip_video* videos, int32_t n_videos, clip_fill_fn fill,
                    void* user, int64_t chunk_frames, int32_t* cut_buf, int64_t cut_capacity,
                    clip_video_result* results, const clip_run_outputs* out) {
  CKS(check_ctx(ctx));
  if (!videos || n_videos < 1) return fail(ctx, CLIP_E_INVALID, "no videos");
  if (!results) return fail(ctx, CLIP_E_INVALID, "results is NULL");
  if (!cut_buf && cut_capacity > 0) return fail(ctx, CLIP_E_INVALID, "cut_buf is NULL");
  const int32_t dim = videos[0].dim;
  const bool merge = dim > 0;
  int64_t F = 0, need = 0;
  std::vector<VideoDesc> vd(n_videos);
  const int64_t L = ctx->p.min_clip_frames;
  for (int32_t i = 0; i < n_videos; ++i) {
    const clip_video& v = videos[i];
    CKS(validate_frames(ctx, v.frames, v.n_frames, v.height, v.width, fill != nullptr, v.format));
    if (v.dim != dim) return fail(ctx, CLIP_E_INVALID, "video %d: dim %d != %d", i, v.dim, dim);
    if (merge && !v.emb) return fail(ctx, CLIP_E_INVALID, "video %d: emb is NULL", i);
    if (dim < 0 || dim > 65536) return fail(ctx, CLIP_E_INVALID, "bad dim %d", dim);
    vd[i].fbase = F;
    vd[i].n = v.n_frames;
    vd[i].npix = (int64_t)v.height * v.width;
    F += v.n_frames;
    need += 2 * (v.n_frames / L + 1);
  }
  if (F > INT32_MAX) return fail(ctx, CLIP_E_INVALID, "too many frames in one call");
  if (cut_capacity < need)
    return fail(ctx, CLIP_E_CAPACITY, "cut_capacity %lld < %lld", (long long)cut_capacity,
                (long long)need);
  const uint32_t nbins = nbins_of(ctx->p);
  const int mode = k1_mode(ctx->p);
  const int64_t blocks = (F + kCompactFrames - 1) / kCompactFrames;
  uint32_t* d_hist;
  uint32_t* d_l1;
  if (out && out->hist) {
    d_hist = out->hist;
  } else {
    CKS(ensure(ctx, ctx->hist, sizeof(uint32_t) * nbins * F));
    d_hist = P<uint32_t>(ctx->hist);
  }
  if (out && out->l1) {
    d_l1 = out->l1;
  } else {
    CKS(ensure(ctx, ctx->l1, sizeof(uint32_t) * F));
    d_l1 = P<uint32_t>(ctx->l1);
  }
  CKS(ensure(ctx, ctx->vids, sizeof(VideoDesc) * n_videos));
  CKS(ensure(ctx, ctx->cand_slots, 4 * blocks * kCompactFrames));
  CKS(ensure(ctx, ctx->cand_count, 4 * blocks));
  CKS(ensure(ctx, ctx->cuts, 4 * F));
  CKS(ensure(ctx, ctx->ncuts, 4 * n_videos));
  CKS(ensure(ctx, ctx->ncand, 4 * n_videos));
  CKS(ensure(ctx, ctx->final_cuts, 4 * F));
  CKS(ensure(ctx, ctx->nfinal, 4 * n_videos));
  CKS(ensure(ctx, ctx->detcos, 8 * F));

  Span whole(ctx, 3);
  CKS(upload(ctx, ctx->vids.p, vd.data(), sizeof(VideoDesc) * n_videos));
  CK(cudaMemsetAsync(d_hist, 0, sizeof(uint32_t) * nbins * F, ctx->stream));

  // ---- K1: device-resident videos in one launch
  std::vector<HistSeg> segs;
  std::vector<Nv12Seg> nsegs;
  std::vector<int32_t> streamed;
  for (int32_t i = 0; i < n_videos; ++i) {
    const clip_video& v = videos[i];
    if (v.frames && is_device_ptr(v.frames) && v.format == CLIP_FORMAT_NV12) {
      nsegs.push_back(Nv12Seg{v.frames, d_hist + vd[i].fbase * nbins, v.n_frames, v.height,
                              v.width, 0, 0, 0});
    } else if (v.frames && is_device_ptr(v.frames)) {
      HistSeg s{};
      s.frames = v.frames;
      s.hist = d_hist + vd[i].fbase * nbins;
      s.n_frames = v.n_frames;
      s.groups = vd[i].npix / 16;
      segs.push_back(s);
    } else {
      streamed.push_back(i);
    }
  }
  CKS(launch_k1(ctx, segs, mode));
  CKS(launch_k1_nv12(ctx, nsegs, mode));

  // ---- K1: host / callback videos through two staging buffers.  Chunks of
  // consecutive videos are packed into one staging buffer (each chunk 16-B
  // aligned: frame sizes are multiples of 48 B) and histogrammed by ONE K1
  // launch over all of them (one segment per chunk), so batches of short
  // videos are not launch- and tail-bound (SURVEY 8(d) "C5 batching").
  if (!streamed.empty()) {
    int64_t max_fb = 0;
    auto frame_bytes = [&](int32_t i) {
      return videos[i].format == CLIP_FORMAT_NV12 ? 3 * vd[i].npix / 2 : 3 * vd[i].npix;
    };
    for (int32_t i : streamed) max_fb = std::max<int64_t>(max_fb, frame_bytes(i));
    int64_t cf = chunk_frames > 0 ? chunk_frames : std::max<int64_t>(1, ((int64_t)1 << 30) / max_fb);
    const int64_t cap = cf * max_fb;  // staging bytes: every single chunk fits
    CKS(ensure(ctx, ctx->staging[0], cap));
    CKS(ensure(ctx, ctx->staging[1], cap));
    struct Piece { int32_t i; int64_t t0, m; };
    std::vector<Piece> pieces;
    for (int32_t i : streamed)
      for (int64_t t0 = 0; t0 < videos[i].n_frames; t0 += cf)
        pieces.push_back(Piece{i, t0, std::min(cf, videos[i].n_frames - t0)});
    int batch_i = 0;
    for (size_t p0 = 0; p0 < pieces.size(); ++batch_i) {
      // the batch: consecutive pieces of one format within the staging capacity
      const bool nv12 = videos[pieces[p0].i].format == CLIP_FORMAT_NV12;
      size_t p1 = p0;
      int64_t used = 0;
      while (p1 < pieces.size() &&
             (videos[pieces[p1].i].format == CLIP_FORMAT_NV12) == nv12 &&
             used + pieces[p1].m * frame_bytes(pieces[p1].i) <= cap) {
        used += pieces[p1].m * frame_bytes(pieces[p1].i);
        ++p1;
      }
      const int b = batch_i & 1;
      uint8_t* base = P<uint8_t>(ctx->staging[b]);
      bool copies = false;
      CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->consumed[b], 0));
      std::vector<HistSeg> segs_b;
      std::vector<Nv12Seg> nsegs_b;
      int64_t off = 0;
      for (size_t q = p0; q < p1; ++q) {
        const Piece& pc = pieces[q];
        const clip_video& v = videos[pc.i];
        const int64_t fb = frame_bytes(pc.i);
        uint8_t* dst = base + off;
        if (v.frames) {
          CK(cudaMemcpyAsync(dst, v.frames + pc.t0 * fb, pc.m * fb, cudaMemcpyHostToDevice,
                             ctx->copy_stream));
          ctx->stats.memcpy_h2d += pc.m * fb;
          copies = true;
        } else {
          if (!copies) CK(cudaStreamWaitEvent(ctx->stream, ctx->consumed[b], 0));
          if (fill(user, pc.i, pc.t0, pc.m, dst, reinterpret_cast<uintptr_t>(ctx->stream)) != 0)
            return fail(ctx, CLIP_E_INVALID, "fill callback failed (video %d, frame %lld)", pc.i,
                        (long long)pc.t0);
        }
        if (nv12) {
          nsegs_b.push_back(Nv12Seg{dst, d_hist + (vd[pc.i].fbase + pc.t0) * nbins, pc.m, v.height,
                                    v.width, 0, 0, 0});
        } else {
          HistSeg s{};
          s.frames = dst;
          s.hist = d_hist + (vd[pc.i].fbase + pc.t0) * nbins;
          s.n_frames = pc.m;
          s.groups = vd[pc.i].npix / 16;
          segs_b.push_back(s);
        }
        off += pc.m * fb;
      }
      if (copies) {
        CK(cudaEventRecord(ctx->copied[b], ctx->copy_stream));
        CK(cudaStreamWaitEvent(ctx->stream, ctx->copied[b], 0));
      }
      if (nv12)
        CKS(launch_k1_nv12(ctx, nsegs_b, mode));
      else
        CKS(launch_k1(ctx, segs_b, mode));
      CK(cudaEventRecord(ctx->consumed[b], ctx->stream));
      p0 = p1;
    }
  }

  // ---- K2: distance, threshold, ordered compaction, greedy + tail
  {
    Span sp(ctx, 1);
    const bool var = ctx->p.distance != CLIP_DIST_L1 || ctx->p.adaptive_window > 0;
    CK(k2_l1_launch(d_hist, F, P<VideoDesc>(ctx->vids), n_videos, nbins, nullptr, d_l1, nullptr,
                    ctx->p.cut_threshold_ppm, var ? nullptr : P<int32_t>(ctx->cand_slots),
                    P<int32_t>(ctx->cand_count), ctx->stream));
    if (var) {
      CKS(ensure(ctx, ctx->flags, F));
      int nl = 0;
      CK(k2_variant_launch(d_hist, d_l1, F, P<VideoDesc>(ctx->vids), n_videos, nbins, nullptr,
                           (int)ctx->p.distance, (int32_t)ctx->p.adaptive_window,
                           ctx->p.adaptive_ratio_ppm, ctx->p.cut_threshold_ppm, nullptr,
                           P<uint8_t>(ctx->flags), P<int32_t>(ctx->cand_slots),
                           P<int32_t>(ctx->cand_count), &nl, ctx->stream));
      ctx->stats.launches += nl;
    }
    CK(k2_greedy_launch(P<VideoDesc>(ctx->vids), n_videos, P<int32_t>(ctx->cand_slots),
                        P<int32_t>(ctx->cand_count), L, P<int32_t>(ctx->cuts),
                        P<int32_t>(ctx->ncuts), P<int32_t>(ctx->ncand), ctx->stream));
    sp.end();
    ctx->stats.launches += 2;
  }
  // ---- K3: merge (the cut counts stay on the device: K3 sizes itself from
  // them, the host passes the min-clip-length bound)
  int32_t* d_final = P<int32_t>(ctx->final_cuts);
  if (merge) {
    std::vector<MergeVideo> mv(n_videos);
    int64_t Kub = 0;
    for (int32_t i = 0; i < n_videos; ++i) {
      mv[i].emb = videos[i].emb;
      mv[i].n = videos[i].n_frames;
      mv[i].cut_base = vd[i].fbase;
      mv[i].clip_base = 0;
      mv[i].n_clips = 0;
      Kub += videos[i].n_frames / L + 1;
    }
    CKS(run_merge(ctx, mv, dim, P<int32_t>(ctx->cuts), P<int32_t>(ctx->ncuts), Kub, d_final,
                  P<int32_t>(ctx->nfinal), P<double>(ctx->detcos)));
  }

  // ---- pack results: per video [detected | final (n_detected reserved)] at
  // offsets scanned on the device; ONE read-back of summary + packed cuts
  // (sized by the capacity bound `need` >= the packed total) and one sync.
  const int64_t sum_words = 1 + (int64_t)SUM_W * n_videos;
  CKS(ensure(ctx, ctx->pack, 8 * sum_words + 4 * need));
  const bool want_cos = merge && out && out->detected_cos;
  if (want_cos) CKS(ensure(ctx, ctx->pack_cos, 8 * need));
  const size_t pin_cos = (size_t)(8 * sum_words + 4 * need + 7) & ~(size_t)7;
  CKS(ensure_pinned(ctx, pin_cos + (want_cos ? 8 * need : 0)));
  int64_t* d_sum = P<int64_t>(ctx->pack);
  int32_t* d_pack = reinterpret_cast<int32_t*>(d_sum + sum_words);
  summary_kernel<<<1, 1024, 0, ctx->stream>>>(n_videos, P<int32_t>(ctx->ncuts), P<int32_t>(ctx->ncand),
                                              merge ? P<int32_t>(ctx->nfinal) : nullptr,
                                              merge ? P<int64_t>(ctx->m_vstate) : nullptr, d_sum);
  CK(cudaGetLastError());
  pack_kernel<<<(unsigned)((F + 255) / 256), 256, 0, ctx->stream>>>(
      P<VideoDesc>(ctx->vids), n_videos, F, P<int32_t>(ctx->cuts), P<int32_t>(ctx->ncuts),
      merge ? d_final : P<int32_t>(ctx->cuts), merge ? P<int32_t>(ctx->nfinal) : P<int32_t>(ctx->ncuts),
      want_cos ? P<double>(ctx->detcos) : nullptr, d_sum, d_pack,
      want_cos ? P<double>(ctx->pack_cos) : nullptr);
  CK(cudaGetLastError());
  ctx->stats.launches += 2;
  CK(cudaMemcpyAsync(ctx->hpin, ctx->pack.p, 8 * sum_words + 4 * need, cudaMemcpyDeviceToHost,
                     ctx->stream));
  if (want_cos)
    CK(cudaMemcpyAsync(static_cast<uint8_t*>(ctx->hpin) + pin_cos, ctx->pack_cos.p, 8 * need,
                       cudaMemcpyDeviceToHost, ctx->stream));
  whole.end();
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stats.memcpy_d2h += 8 * sum_words + 4 * need + (want_cos ? 8 * need : 0);
  const int64_t* hs = static_cast<const int64_t*>(ctx->hpin);
  const int64_t total = hs[0];
  if (total > need)  // K2 keeps every clip >= min_clip_frames: cannot happen
    return fail(ctx, CLIP_E_CUDA, "packed cuts %lld exceed the bound %lld", (long long)total,
                (long long)need);
  if (total > 0) {
    memcpy(cut_buf, hs + sum_words, 4 * total);
    if (want_cos) memcpy(out->detected_cos, static_cast<uint8_t*>(ctx->hpin) + pin_cos, 8 * total);
  }
  for (int32_t i = 0; i < n_videos; ++i) {
    const int64_t* r = hs + 1 + (int64_t)SUM_W * i;
    clip_video_result& res = results[i];
    memset(&res, 0, sizeof res);
    res.id = videos[i].id;
    res.n_candidates = (int32_t)r[SUM_NCAND];
    res.n_detected = (int32_t)r[SUM_NCUTS];
    res.n_final = (int32_t)r[SUM_NFINAL];
    res.n_band_hits = r[SUM_BAND];
    res.rounds = (int32_t)r[SUM_ROUNDS];
    res.detected_offset = r[SUM_OFF];
    res.final_offset = r[SUM_OFF] + r[SUM_NCUTS];
  }
  harvest(ctx);
  return CLIP_OK;
}

int clip_get_stats(clip_ctx* ctx, clip_stats* out, int reset) {
  if (!ctx || !out) return CLIP_E_INVALID;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  harvest(ctx);
  *out = ctx->stats;
  if (reset) memset(&ctx->stats, 0, sizeof ctx->stats);
  return CLIP_OK;
}

int clip_debug_binmap(clip_ctx* ctx, uint8_t* table) {
  CKS(check_ctx(ctx));
  if (!table) return fail(ctx, CLIP_E_INVALID, "table is NULL");
  CK(k5_binmap_launch(table, ctx->p.h_bins, ctx->p.s_bins, ctx->p.v_bins,
                      k1_mode(ctx->p) == kModeFast, ctx->stream));
  ctx->stats.launches += 1;
  return CLIP_OK;
}

}  // extern "C"

namespace {
int sample_frames(clip_ctx* ctx, int format, const uint8_t* frames, int64_t n_frames,
                  int32_t height, int32_t width, const int32_t* cuts, int64_t n_cuts, int32_t k,
                  int32_t out_h, int32_t out_w, uint8_t* out, int32_t* index) {
  CKS(check_ctx(ctx));
  CKS(validate_frames(ctx, frames, n_frames, height, width, false, format));
  if (n_cuts < 0 || n_cuts >= n_frames || (n_cuts > 0 && !cuts))
    return fail(ctx, CLIP_E_INVALID, "bad cuts (n_cuts %lld)", (long long)n_cuts);
  if (k < 1 || out_h < 1 || out_w < 1 || out_w > k4_max_width())
    return fail(ctx, CLIP_E_INVALID, "bad sampling (k %d, out %dx%d)", k, out_w, out_h);
  if (!out) return fail(ctx, CLIP_E_INVALID, "out is NULL");
  if ((n_cuts + 1) * (int64_t)k > INT32_MAX / 2)
    return fail(ctx, CLIP_E_INVALID, "too many output frames");
  Span sp(ctx, 2);
  CK(k4_sample_launch(frames, n_frames, height, width, cuts, (int32_t)n_cuts, k, out_h, out_w, out,
                      index, format == CLIP_FORMAT_NV12, ctx->stream));
  sp.end();
  ctx->stats.launches += 1;
  return CLIP_OK;
}
}  // namespace

extern "C" {

int clip_sample_frames(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                       int32_t width, const int32_t* cuts, int64_t n_cuts, int32_t k, int32_t out_h,
                       int32_t out_w, uint8_t* out, int32_t* index) {
  return sample_frames(ctx, CLIP_FORMAT_RGB24, frames, n_frames, height, width, cuts, n_cuts, k,
                       out_h, out_w, out, index);
}

int clip_sample_frames_nv12(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames, int32_t height,
                            int32_t width, const int32_t* cuts, int64_t n_cuts, int32_t k,
                            int32_t out_h, int32_t out_w, uint8_t* out, int32_t* index) {
  return sample_frames(ctx, CLIP_FORMAT_NV12, frames, n_frames, height, width, cuts, n_cuts, k,
                       out_h, out_w, out, index);
}

int clip_debug_nv12map(clip_ctx* ctx, uint8_t* table) {
  CKS(check_ctx(ctx));
  if (!table) return fail(ctx, CLIP_E_INVALID, "table is NULL");
  CK(k5_nv12map_launch(table, ctx->p.h_bins, ctx->p.s_bins, ctx->p.v_bins,
                       k1_mode(ctx->p) == kModeFast, ctx->stream));
  ctx->stats.launches += 1;
  return CLIP_OK;
}

int clip_debug_read_roofline_nv12(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames,
                                  int32_t height, int32_t width) {
  CKS(check_ctx(ctx));
  CKS(validate_frames(ctx, frames, n_frames, height, width, false, CLIP_FORMAT_NV12));
  if (width % 16 != 0 || nv12_stage_rows(width) < 1)
    return fail(ctx, CLIP_E_INVALID, "NV12 read roofline needs width %% 16 == 0 and <= 20480");
  std::vector<Nv12Seg> segs(1);
  segs[0] = Nv12Seg{frames, nullptr, n_frames, height, width, 0, 0, 0};
  return launch_k1_nv12(ctx, segs, kModeRead);
}

int clip_debug_read_roofline(clip_ctx* ctx, const uint8_t* frames, int64_t n_frames,
                             int32_t height, int32_t width) {
  CKS(check_ctx(ctx));
  CKS(validate_frames(ctx, frames, n_frames, height, width, false));
  std::vector<HistSeg> segs(1);
  segs[0].frames = frames;
  segs[0].hist = nullptr;
  segs[0].n_frames = n_frames;
  segs[0].groups = (int64_t)height * width / 16;
  return launch_k1(ctx, segs, kModeRead);
}

}  // extern "C"
