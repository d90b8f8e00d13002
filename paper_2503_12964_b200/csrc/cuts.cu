// cuts.cu — K2: adjacent-frame distance, integer threshold, ordered
// candidate compaction and the greedy minimum-clip-length pass (rows a4-a6).
//
//   O3  L1_t = sum_b |h_t[b] - h_{t-1}[b]| (L1_0 = 0), score_t = L1_t / 2N
//   O4  candidate <=> t >= 1 and L1_t * 1e6 >= tau_ppm * 2N (exact, u64)
//   O5  last = 0; accept candidate t iff t - last >= L_min
//   O6  drop the final cut if n - last < L_min
// (§2.1: "analyzing the color changes between frames";
//  the "aggressive" split is smoothed by the merge, merge.cu.)
//
// Layout: one warp per frame for L1 (lanes stride the bins, redux.sync add),
// candidate flags compacted IN ORDER per 128-frame block with ballot/popc,
// then one warp per video walks the blocks' compacted lists in order.
#include "common.cuh"
#include "kernels.cuh"

namespace clipdetect {

namespace {

__device__ __forceinline__ int32_t find_video(const VideoDesc* __restrict__ v, int32_t nv,
                                              int64_t f) {
  int32_t lo = 0, hi = nv - 1;
  while (lo < hi) {
    const int32_t m = (lo + hi + 1) >> 1;
    if (v[m].fbase <= f) lo = m; else hi = m - 1;
  }
  return lo;
}

constexpr int kL1Warps = 8;
constexpr int kFramesPerWarp = kCompactFrames / kL1Warps;  // 16

__device__ __forceinline__ bool is_candidate(int64_t t, uint32_t l1, uint64_t tau_ppm,
                                             int64_t npix) {
  return t >= 1 && (uint64_t)l1 * 1000000ull >= tau_ppm * (uint64_t)(2 * npix);
}

// Ordered compaction of kCompactFrames flags held in sflag (threads 0..127).
__device__ __forceinline__ void compact_block(const uint8_t* sflag, int* wcnt, int64_t block,
                                              int32_t value_base, int32_t* __restrict__ slots,
                                              int32_t* __restrict__ counts) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  bool fl = false;
  uint32_t m = 0;
  if (warp < kCompactFrames / 32) {
    fl = sflag[tid] != 0;
    m = __ballot_sync(0xffffffffu, fl);
    if (lane == 0) wcnt[warp] = __popc(m);
  }
  __syncthreads();
  if (warp < kCompactFrames / 32) {
    int off = 0;
    for (int w = 0; w < warp; ++w) off += wcnt[w];
    if (fl) slots[block * kCompactFrames + off + __popc(m & ((1u << lane) - 1u))] = value_base + tid;
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < kCompactFrames / 32; ++w) tot += wcnt[w];
      counts[block] = tot;
    }
  }
}

__global__ void __launch_bounds__(kL1Warps * 32)
k2_l1_kernel(const uint32_t* __restrict__ hist, int64_t F, const VideoDesc* __restrict__ vids,
             int32_t nvid, uint32_t nbins, const uint32_t* __restrict__ prev_hist,
             uint32_t* __restrict__ l1, float* __restrict__ score, uint64_t tau_ppm,
             int32_t* __restrict__ cand_slots, int32_t* __restrict__ cand_count) {
  __shared__ uint8_t sflag[kCompactFrames];
  __shared__ int wcnt[kCompactFrames / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f0 = (int64_t)blockIdx.x * kCompactFrames;
  for (int j = 0; j < kFramesPerWarp; ++j) {
    const int lf = warp * kFramesPerWarp + j;
    const int64_t f = f0 + lf;
    if (f >= F) {
      if (lane == 0) sflag[lf] = 0;
      continue;
    }
    const VideoDesc vd = vids[find_video(vids, nvid, f)];
    const int64_t t = f - vd.fbase;
    const uint32_t* cur = hist + f * nbins;
    const uint32_t* prev = t >= 1 ? cur - nbins : prev_hist;
    uint32_t acc = 0;
    if (prev != nullptr) {
      for (uint32_t b = lane; b < nbins; b += 32) {
        const uint32_t a = cur[b], c = prev[b];
        acc += a > c ? a - c : c - a;
      }
    }
    acc = __reduce_add_sync(0xffffffffu, acc);
    if (lane == 0) {
      if (l1) l1[f] = acc;
      if (score) score[f] = (float)((double)acc / (double)(2 * vd.npix));
      sflag[lf] = is_candidate(t, acc, tau_ppm, vd.npix);
    }
  }
  if (cand_slots == nullptr) return;
  __syncthreads();
  compact_block(sflag, wcnt, blockIdx.x, (int32_t)f0, cand_slots, cand_count);
}

// One warp per video: greedy over the video's candidates in ascending order.
__global__ void k2_greedy_kernel(const VideoDesc* __restrict__ vids, int32_t nvid,
                                 const int32_t* __restrict__ cand_slots,
                                 const int32_t* __restrict__ cand_count, int64_t l_min,
                                 int32_t* __restrict__ cuts, int32_t* __restrict__ n_cuts,
                                 int32_t* __restrict__ n_cand) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t v = blockIdx.x * (blockDim.x >> 5) + warp;
  if (v >= nvid) return;
  const int64_t fbase = vids[v].fbase, n = vids[v].n;
  const int64_t c0 = fbase / kCompactFrames, c1 = (fbase + n - 1) / kCompactFrames;
  int32_t* out = cuts + fbase;  // capacity n per video
  int64_t last = 0;
  int32_t k = 0, nc = 0;
  auto take = [&](int64_t f) {  // the greedy step for candidate frame f (ascending)
    if (f < fbase || f >= fbase + n) return;
    const int64_t t = f - fbase;
    ++nc;
    if (t - last >= l_min) {
      CD_CHECK(k < n && t > last);  // cuts strictly increasing, capacity n per video
      if (lane == 0) out[k] = (int32_t)t;
      ++k;
      last = t;
    }
  };
  constexpr int kPre = 4;  // candidates per chunk fetched up front, all chunks at once
  for (int64_t cb = c0; cb <= c1; cb += 32) {
    const int64_t c = cb + lane;
    const int32_t cnt = c <= c1 ? cand_count[c] : 0;
    CD_CHECK(cnt >= 0 && cnt <= kCompactFrames);
    // every lane loads the first kPre candidates of its chunk: one round trip
    // for the 32 chunks instead of one per non-empty chunk
    int32_t pre[kPre];
#pragma unroll
    for (int j = 0; j < kPre; ++j) pre[j] = j < cnt ? cand_slots[c * kCompactFrames + j] : -1;
    uint32_t nz = __ballot_sync(0xffffffffu, cnt > 0);
    while (nz) {
      const int src = __ffs(nz) - 1;
      nz &= nz - 1;
      const int32_t cc = __shfl_sync(0xffffffffu, cnt, src);
      const int64_t chunk = cb + src;
      if (cc <= kPre) {
#pragma unroll
        for (int j = 0; j < kPre; ++j) {
          const int32_t f = __shfl_sync(0xffffffffu, pre[j], src);
          if (j < cc) take(f);
        }
        continue;
      }
      for (int32_t e0 = 0; e0 < cc; e0 += 32) {
        const int32_t fidx = e0 + lane < cc ? cand_slots[chunk * kCompactFrames + e0 + lane] : -1;
        const int32_t m = min(32, cc - e0);
        for (int32_t i = 0; i < m; ++i) take(__shfl_sync(0xffffffffu, fidx, i));
      }
    }
  }
  if (k > 0 && n - last < l_min) --k;
  if (lane == 0) {
    n_cuts[v] = k;
    n_cand[v] = nc;
  }
}

struct CutState {
  int64_t frames_seen, last_cut, n_candidates, n_cuts;
};

__global__ void __launch_bounds__(kCompactFrames)
k2_stream_flags_kernel(const uint32_t* __restrict__ l1, int64_t n, int64_t npix,
                       uint64_t tau_ppm, const CutState* __restrict__ st,
                       int32_t* __restrict__ cand_slots, int32_t* __restrict__ cand_count) {
  __shared__ uint8_t sflag[kCompactFrames];
  __shared__ int wcnt[kCompactFrames / 32];
  const int64_t i = (int64_t)blockIdx.x * kCompactFrames + threadIdx.x;
  const int64_t t = st->frames_seen + i;
  sflag[threadIdx.x] = i < n && is_candidate(t, l1[i], tau_ppm, npix);
  __syncthreads();
  compact_block(sflag, wcnt, blockIdx.x, (int32_t)((int64_t)blockIdx.x * kCompactFrames),
                cand_slots, cand_count);
}

__global__ void k2_stream_greedy_kernel(int64_t n, int64_t l_min, CutState* __restrict__ st,
                                        const int32_t* __restrict__ cand_slots,
                                        const int32_t* __restrict__ cand_count,
                                        int32_t* __restrict__ cuts, int64_t cap, int is_final) {
  const int lane = threadIdx.x & 31;
  const int64_t base = st->frames_seen;
  int64_t last = st->last_cut, k = st->n_cuts, nc = st->n_candidates;
  const int64_t nblk = (n + kCompactFrames - 1) / kCompactFrames;
  for (int64_t cb = 0; cb < nblk; cb += 32) {
    const int64_t c = cb + lane;
    const int32_t cnt = c < nblk ? cand_count[c] : 0;
    uint32_t nz = __ballot_sync(0xffffffffu, cnt > 0);
    while (nz) {
      const int src = __ffs(nz) - 1;
      nz &= nz - 1;
      const int32_t cc = __shfl_sync(0xffffffffu, cnt, src);
      const int64_t chunk = cb + src;
      for (int32_t e0 = 0; e0 < cc; e0 += 32) {
        const int32_t li = e0 + lane < cc ? cand_slots[chunk * kCompactFrames + e0 + lane] : 0;
        const int32_t m = min(32, cc - e0);
        for (int32_t j = 0; j < m; ++j) {
          const int64_t t = base + __shfl_sync(0xffffffffu, li, j);
          ++nc;
          if (t - last >= l_min) {
            if (lane == 0 && k < cap) cuts[k] = (int32_t)t;
            ++k;
            last = t;
          }
        }
      }
    }
  }
  const int64_t seen = base + n;
  if (is_final && k > 0 && seen - last < l_min) --k;
  __syncwarp();
  if (lane == 0) {
    st->frames_seen = seen;
    st->last_cut = last;
    st->n_candidates = nc;
    st->n_cuts = k;
  }
}

// ------------------------------------------------------------ f4 variants
// O3' distances, one thread per frame, bins in ascending order, f64 with
// explicitly rounded operations (no contraction): the same IEEE operations,
// in the same order, as the oracle's plain loop, so the scores and every
// threshold decision are bit-identical to it.
__device__ double frame_distance(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                 uint32_t nbins, int64_t npix, int kind) {
  if (kind == 1) {
    double acc = 0.0;
    for (uint32_t i = 0; i < nbins; ++i) {
      const int64_t x = a[i], y = b[i];
      const int64_t s = x + y;
      if (s == 0) continue;
      const int64_t d = x - y;
      acc = __dadd_rn(acc, __ddiv_rn((double)(d * d), (double)s));
    }
    return __ddiv_rn(acc, (double)(2 * npix));
  }
  if (kind == 2) {
    double acc = 0.0;
    for (uint32_t i = 0; i < nbins; ++i)
      acc = __dadd_rn(acc, __dsqrt_rn(__dmul_rn((double)a[i], (double)b[i])));
    const double x = __dsub_rn(1.0, __ddiv_rn(acc, (double)npix));
    return __dsqrt_rn(x > 0.0 ? x : 0.0);
  }
  int64_t sab = 0, saa = 0, sbb = 0;
  for (uint32_t i = 0; i < nbins; ++i) {
    const int64_t x = a[i], y = b[i];
    sab += x * y;
    saa += x * x;
    sbb += y * y;
  }
  const int64_t n2 = npix * npix;
  const int64_t num = (int64_t)nbins * sab - n2;
  const int64_t A = (int64_t)nbins * saa - n2, B = (int64_t)nbins * sbb - n2;
  double r;
  if (A == 0 && B == 0) r = 1.0;
  else if (A == 0 || B == 0) r = 0.0;
  else r = __ddiv_rn((double)num, __dsqrt_rn(__dmul_rn((double)A, (double)B)));
  return __dsub_rn(1.0, r);
}

// O3' scores (f32 out) and, unless adaptive, O4' flags d >= tau_ppm / 1e6.
__global__ void __launch_bounds__(128)
k2_dist_kernel(const uint32_t* __restrict__ hist, int64_t F, const VideoDesc* __restrict__ vids,
               int32_t nvid, uint32_t nbins, const uint32_t* __restrict__ prev_hist, int kind,
               uint64_t tau_ppm, float* __restrict__ score, uint8_t* __restrict__ flags) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const VideoDesc vd = vids[find_video(vids, nvid, f)];
  const int64_t t = f - vd.fbase;
  const uint32_t* cur = hist + f * nbins;
  const uint32_t* prev = t >= 1 ? cur - nbins : prev_hist;
  const double d = prev ? frame_distance(prev, cur, nbins, vd.npix, kind) : 0.0;
  if (score) score[f] = __double2float_rn(d);
  if (flags) flags[f] = t >= 1 && d >= __ddiv_rn((double)tau_ppm, 1e6);
}

// O4'' adaptive flags on L1 (exact integers, 128-bit products).
__global__ void __launch_bounds__(128)
k2_adaptive_kernel(const uint32_t* __restrict__ l1, int64_t F, const VideoDesc* __restrict__ vids,
                   int32_t nvid, uint64_t tau_ppm, int32_t w, uint64_t ratio_ppm,
                   uint8_t* __restrict__ flags) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const VideoDesc vd = vids[find_video(vids, nvid, f)];
  const int64_t t = f - vd.fbase, n = vd.n;
  bool c = false;
  if (t >= 1) {
    unsigned __int128 sum = 0;
    int64_t m = 0;
    for (int64_t u = t - w; u <= t + w; ++u) {
      if (u < 1 || u > n - 1 || u == t) continue;
      sum += l1[vd.fbase + u];
      ++m;
    }
    const uint32_t x = l1[f];
    if (m > 0) {
      const unsigned __int128 lhs = (unsigned __int128)x * (unsigned __int128)m * 1000000u;
      c = lhs >= (unsigned __int128)ratio_ppm * sum &&
          (uint64_t)x * 1000000ull >= tau_ppm * (uint64_t)(2 * vd.npix);
    }
  }
  flags[f] = c;
}

__global__ void __launch_bounds__(kCompactFrames)
k2_compact_kernel(const uint8_t* __restrict__ flags, int64_t F, int32_t* __restrict__ cand_slots,
                  int32_t* __restrict__ cand_count) {
  __shared__ uint8_t sflag[kCompactFrames];
  __shared__ int wcnt[kCompactFrames / 32];
  const int64_t f = (int64_t)blockIdx.x * kCompactFrames + threadIdx.x;
  sflag[threadIdx.x] = f < F ? flags[f] : 0;
  __syncthreads();
  compact_block(sflag, wcnt, blockIdx.x, (int32_t)((int64_t)blockIdx.x * kCompactFrames),
                cand_slots, cand_count);
}

}  // namespace

cudaError_t k2_l1_launch(const uint32_t* hist, int64_t F, const VideoDesc* d_vids, int32_t nvid,
                         uint32_t nbins, const uint32_t* prev_hist, uint32_t* l1, float* score,
                         uint64_t tau_ppm, int32_t* cand_slots, int32_t* cand_count,
                         cudaStream_t stream) {
  if (F <= 0) return cudaSuccess;
  const int64_t blocks = (F + kCompactFrames - 1) / kCompactFrames;
  k2_l1_kernel<<<(unsigned)blocks, kL1Warps * 32, 0, stream>>>(
      hist, F, d_vids, nvid, nbins, prev_hist, l1, score, tau_ppm, cand_slots, cand_count);
  return cudaGetLastError();
}

cudaError_t k2_variant_launch(const uint32_t* hist, const uint32_t* l1, int64_t F,
                              const VideoDesc* d_vids, int32_t nvid, uint32_t nbins,
                              const uint32_t* prev_hist, int kind, int32_t adaptive_w,
                              uint64_t ratio_ppm, uint64_t tau_ppm, float* score, uint8_t* flags,
                              int32_t* cand_slots, int32_t* cand_count, int* launches,
                              cudaStream_t stream) {
  if (F <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((F + 127) / 128);
  *launches = 0;
  if (kind != 0) {
    k2_dist_kernel<<<blocks, 128, 0, stream>>>(hist, F, d_vids, nvid, nbins, prev_hist, kind,
                                               tau_ppm, score, adaptive_w > 0 ? nullptr : flags);
    ++*launches;
  }
  if (adaptive_w > 0 && flags) {
    k2_adaptive_kernel<<<blocks, 128, 0, stream>>>(l1, F, d_vids, nvid, tau_ppm, adaptive_w,
                                                   ratio_ppm, flags);
    ++*launches;
  }
  if (cand_slots && flags) {
    k2_compact_kernel<<<(unsigned)((F + kCompactFrames - 1) / kCompactFrames), kCompactFrames, 0,
                        stream>>>(flags, F, cand_slots, cand_count);
    ++*launches;
  }
  return cudaGetLastError();
}

cudaError_t k2_greedy_launch(const VideoDesc* d_vids, int32_t nvid, const int32_t* cand_slots,
                             const int32_t* cand_count, int64_t l_min, int32_t* cuts,
                             int32_t* n_cuts, int32_t* n_cand, cudaStream_t stream) {
  if (nvid <= 0) return cudaSuccess;
  const int wpb = 4;
  k2_greedy_kernel<<<(nvid + wpb - 1) / wpb, wpb * 32, 0, stream>>>(
      d_vids, nvid, cand_slots, cand_count, l_min, cuts, n_cuts, n_cand);
  return cudaGetLastError();
}

cudaError_t k2_stream_launch(const uint32_t* l1, int64_t n, int64_t npix, uint64_t tau_ppm,
                             int64_t l_min, void* state, int32_t* cuts, int64_t cap,
                             int is_final, int32_t* cand_slots, int32_t* cand_count,
                             cudaStream_t stream) {
  CutState* st = reinterpret_cast<CutState*>(state);
  if (n > 0) {
    const int64_t blocks = (n + kCompactFrames - 1) / kCompactFrames;
    k2_stream_flags_kernel<<<(unsigned)blocks, kCompactFrames, 0, stream>>>(
        l1, n, npix, tau_ppm, st, cand_slots, cand_count);
  }
  k2_stream_greedy_kernel<<<1, 32, 0, stream>>>(n, l_min, st, cand_slots, cand_count, cuts, cap,
                                                is_final);
  return cudaGetLastError();
}

}  // namespace clipdetect
