// merge.cu — K3: clip embeddings, adjacent cosines and the round-synchronous
// merge (rows a7-a9).
//
//   O8  S_k = sum_{f in clip k} e_f, accumulated in f64 from f32 inputs
//   O9  repeat: c_k = S_k.S_{k+1} / (|S_k| |S_{k+1}|) (0 if a norm is 0);
//       remove every boundary with c_k >= theta at once; recompute; stop when
//       no boundary of the video merges.  Band hit: |c_k - theta| <= band_rel*theta.
// (§2.1: the split "is smoothed out by computing the similarity
//  between image embeddings of adjacent clips to potentially merge them back
//  together".)
//
// Determinism: every sum runs in a fixed order (frames ascending inside a
// <=16-frame piece, pieces ascending inside a clip, clips ascending inside a
// merged range, fixed shuffle trees for the dot products); no float atomics.
// The oracle sums a merged clip frame by frame, the device piece by piece:
// same terms, different association (~1e-16 relative).
#include <math.h>

#include "kernels.cuh"

namespace clipdetect {

namespace {

constexpr int kT = 256;
enum { VS_DONE = 0, VS_ROUNDS = 1, VS_BAND = 2, VS_MERGES = 3 };

__device__ __forceinline__ int32_t find_clip_video(const MergeVideo* __restrict__ mv, int32_t nv,
                                                   int32_t k) {
  int32_t lo = 0, hi = nv - 1;
  while (lo < hi) {
    const int32_t m = (lo + hi + 1) >> 1;
    if (mv[m].clip_base <= k) lo = m; else hi = m - 1;
  }
  return lo;
}

// clip tables + per-video state reset
__global__ void k3_clip_table_kernel(const MergeVideo* __restrict__ mv, int32_t nv, int32_t K,
                                     const int32_t* __restrict__ cuts, MergeScratch s) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nv) {
    int64_t* vs = s.vstate + 4 * k;
    vs[VS_DONE] = mv[k].n_clips < 2;
    vs[VS_ROUNDS] = 0;
    vs[VS_BAND] = 0;
    vs[VS_MERGES] = 0;
    s.valive[k] = mv[k].n_clips - 1;
  }
  if (k >= K) return;
  const int32_t v = find_clip_video(mv, nv, k);
  const MergeVideo m = mv[v];
  const int32_t j = k - m.clip_base;
  s.clip_video[k] = v;
  s.clip_f0[k] = j == 0 ? 0 : cuts[m.cut_base + j - 1];
  s.clip_f1[k] = j == m.n_clips - 1 ? (int32_t)m.n : cuts[m.cut_base + j];
}

// Block-wide exclusive scan helper (1024 threads).
__device__ __forceinline__ int32_t block_excl_scan(int32_t x, int32_t* wsum, int32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t inc = x;
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int32_t w = wsum[lane];
    int32_t wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    wsum[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) wsum[32] = wi;
  }
  __syncthreads();
  const int32_t r = wsum[warp] + inc - x;
  total = wsum[32];
  __syncthreads();
  return r;
}

// piece_base = exclusive scan of ceil(len/kPieceFrames); alive = clips that
// start a boundary (clip_f0 > 0), in order.
__global__ void __launch_bounds__(1024)
k3_scan_kernel(int32_t K, MergeScratch s) {
  __shared__ int32_t wsum[33];
  int32_t carry_p = 0, carry_a = 0;
  for (int32_t base = 0; base < K; base += 1024) {
    const int32_t k = base + threadIdx.x;
    int32_t np = 0, isb = 0;
    if (k < K) {
      const int32_t len = s.clip_f1[k] - s.clip_f0[k];
      np = (len + kPieceFrames - 1) / kPieceFrames;
      isb = s.clip_f0[k] > 0;
    }
    int32_t tp, ta;
    const int32_t ep = block_excl_scan(np, wsum, tp);
    const int32_t ea = block_excl_scan(isb, wsum, ta);
    if (k < K) {
      s.piece_base[k] = carry_p + ep;
      if (isb) s.alive[carry_a + ea] = k;
    }
    carry_p += tp;
    carry_a += ta;
  }
  if (threadIdx.x == 0) {
    s.piece_base[K] = carry_p;
    s.counters[0] = carry_a;
    s.counters[1] = 0;
  }
}

__device__ __forceinline__ int32_t find_piece_clip(const int32_t* __restrict__ pb, int32_t K,
                                                   int64_t p) {
  int32_t lo = 0, hi = K - 1;
  while (lo < hi) {
    const int32_t m = (lo + hi + 1) >> 1;
    if (pb[m] <= p) lo = m; else hi = m - 1;
  }
  return lo;
}

// P[p][d] = sum of frames of piece p (f64, ascending frames); float4 loads
// when the rows allow it (D = 768: 192 threads x 4 dims)
__global__ void __launch_bounds__(kT)
k3_piece_sum_kernel(const MergeVideo* __restrict__ mv, int32_t K, int32_t dim, int32_t stride,
                    MergeScratch s) {
  const int64_t p = blockIdx.x;
  if (p >= s.piece_base[K]) return;
  const int32_t k = find_piece_clip(s.piece_base, K, p);
  const int32_t i = (int32_t)(p - s.piece_base[k]);
  const int32_t c0 = s.clip_f0[k];
  // O8' keyframes: (f - c0) % stride == 0 (every frame for stride 1); the
  // embeddings of other frames are never read
  const int32_t fp = c0 + i * kPieceFrames;
  const int32_t f0 = fp + (stride - (fp - c0) % stride) % stride;
  const int32_t f1 = min(s.clip_f1[k], fp + kPieceFrames);
  const float* __restrict__ e = mv[s.clip_video[k]].emb;
  double* __restrict__ out = s.P + p * dim;
  if ((dim & 3) == 0 && (reinterpret_cast<uintptr_t>(e) & 15) == 0) {
    const int32_t d4n = dim >> 2;
    for (int32_t d4 = threadIdx.x; d4 < d4n; d4 += kT) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      const float4* src = reinterpret_cast<const float4*>(e + (int64_t)f0 * dim) + d4;
#pragma unroll 4
      for (int32_t f = f0; f < f1; f += stride) {
        const float4 x = __ldg(src);
        src += (int64_t)d4n * stride;
        a0 += (double)x.x;
        a1 += (double)x.y;
        a2 += (double)x.z;
        a3 += (double)x.w;
      }
      double2* o = reinterpret_cast<double2*>(out + 4 * d4);
      o[0] = make_double2(a0, a1);
      o[1] = make_double2(a2, a3);
    }
    return;
  }
  for (int32_t d = threadIdx.x; d < dim; d += kT) {
    double acc = 0.0;
    for (int32_t f = f0; f < f1; f += stride) acc += (double)__ldg(e + (int64_t)f * dim + d);
    out[d] = acc;
  }
}

// S[k][d] = sum over the clip's pieces, ascending
__global__ void __launch_bounds__(kT)
k3_clip_sum_kernel(int32_t dim, MergeScratch s) {
  const int32_t k = blockIdx.x;
  const int32_t p0 = s.piece_base[k], p1 = s.piece_base[k + 1];
  for (int32_t d = threadIdx.x; d < dim; d += kT) {
    double acc = 0.0;
    for (int32_t p = p0; p < p1; ++p) acc += s.P[(int64_t)p * dim + d];
    s.S[(int64_t)k * dim + d] = acc;
  }
}

__device__ __forceinline__ double block_sum(double x, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kT / 32; ++w) t += red[w];
  __syncthreads();
  return t;  // valid in thread 0
}

// cosine of every alive boundary b (left range | right range of clips)
__global__ void __launch_bounds__(kT)
k3_cos_kernel(const MergeVideo* __restrict__ mv, int64_t n_alive, int32_t dim, MergeScratch s) {
  __shared__ double red[kT / 32];
  const int64_t b = blockIdx.x;
  const int32_t rk = s.alive[b];
  const int32_t v = s.clip_video[rk];
  if (s.vstate[4 * v + VS_DONE]) return;
  const int32_t lk0 = (b > 0 && s.clip_video[s.alive[b - 1]] == v) ? s.alive[b - 1] : mv[v].clip_base;
  const int32_t rk1 = (b + 1 < n_alive && s.clip_video[s.alive[b + 1]] == v)
                          ? s.alive[b + 1]
                          : mv[v].clip_base + mv[v].n_clips;
  double dot = 0.0, na = 0.0, nb = 0.0;
  for (int32_t d = threadIdx.x; d < dim; d += kT) {
    double L = 0.0, R = 0.0;
    for (int32_t k = lk0; k < rk; ++k) L += s.S[(int64_t)k * dim + d];
    for (int32_t k = rk; k < rk1; ++k) R += s.S[(int64_t)k * dim + d];
    dot += L * R;
    na += L * L;
    nb += R * R;
  }
  dot = block_sum(dot, red);
  na = block_sum(na, red);
  nb = block_sum(nb, red);
  if (threadIdx.x == 0) {
    const double sa = sqrt(na), sb = sqrt(nb);
    s.cos_b[b] = (sa == 0.0 || sb == 0.0) ? 0.0 : dot / (sa * sb);
  }
}

// decisions + ordered compaction alive -> alive2 + per-video round bookkeeping
__global__ void __launch_bounds__(1024)
k3_decide_kernel(int32_t nv, int64_t n_alive, double theta, double band_rel, MergeScratch s) {
  __shared__ int32_t wsum[33];
  int32_t carry = 0;
  int64_t merges = 0;
  for (int32_t v = threadIdx.x; v < nv; v += 1024) s.valive[v] = 0;
  __syncthreads();
  for (int64_t base = 0; base < n_alive; base += 1024) {
    const int64_t b = base + threadIdx.x;
    int32_t keep = 0, rk = 0;
    if (b < n_alive) {
      rk = s.alive[b];
      const int32_t v = s.clip_video[rk];
      keep = 1;
      if (!s.vstate[4 * v + VS_DONE]) {
        const double c = s.cos_b[b];
        s.cos_clip[rk] = c;
        if (fabs(c - theta) <= band_rel * theta)
          atomicAdd(reinterpret_cast<unsigned long long*>(&s.vstate[4 * v + VS_BAND]), 1ull);
        if (c >= theta) {
          keep = 0;
          atomicAdd(reinterpret_cast<unsigned long long*>(&s.vstate[4 * v + VS_MERGES]), 1ull);
        }
      }
      if (keep) atomicAdd(reinterpret_cast<unsigned long long*>(&s.valive[v]), 1ull);
    }
    int32_t tot;
    const int32_t e = block_excl_scan(keep, wsum, tot);
    if (keep) s.alive2[carry + e] = rk;
    carry += tot;
  }
  __syncthreads();
  for (int32_t v = threadIdx.x; v < nv; v += 1024) {
    int64_t* vs = s.vstate + 4 * v;
    if (vs[VS_DONE]) continue;
    vs[VS_ROUNDS] += 1;
    merges += vs[VS_MERGES];
    if (vs[VS_MERGES] == 0 || s.valive[v] == 0) vs[VS_DONE] = 1;
    vs[VS_MERGES] = 0;
  }
  // reduce merges over threads
  __shared__ unsigned long long m_tot;
  if (threadIdx.x == 0) m_tot = 0;
  __syncthreads();
  if (merges) atomicAdd(&m_tot, (unsigned long long)merges);
  __syncthreads();
  if (threadIdx.x == 0) {
    s.counters[0] = carry;
    s.counters[1] = (int64_t)m_tot;
  }
}

__global__ void k3_finish_kernel(const MergeVideo* __restrict__ mv, int32_t nv, int32_t K,
                                 int64_t n_alive, MergeScratch s, int32_t* __restrict__ final_cuts,
                                 int32_t* __restrict__ n_final, double* __restrict__ detected_cos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_alive) {
    const int32_t rk = s.alive[i];
    const int32_t v = s.clip_video[rk];
    // first alive index of video v (alive is sorted by clip index, hence by video)
    int64_t lo = 0, hi = i;
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (s.clip_video[s.alive[m]] < v) lo = m + 1; else hi = m;
    }
    const int64_t pos = i - lo;
    final_cuts[mv[v].cut_base + pos] = s.clip_f0[rk];
    if (i + 1 == n_alive || s.clip_video[s.alive[i + 1]] != v) n_final[v] = (int32_t)(pos + 1);
  }
  if (detected_cos != nullptr && i < K) {
    const int32_t v = s.clip_video[i];
    const int32_t j = (int32_t)i - mv[v].clip_base;
    if (j >= 1) detected_cos[mv[v].cut_base + j - 1] = s.cos_clip[i];
  }
}

}  // namespace

cudaError_t k3_prepare_launch(const MergeVideo* d_mv, int32_t nv, int32_t K, const int32_t* cuts,
                              MergeScratch s, cudaStream_t stream) {
  const int32_t nthreads = K > nv ? K : nv;
  k3_clip_table_kernel<<<(nthreads + 255) / 256, 256, 0, stream>>>(d_mv, nv, K, cuts, s);
  k3_scan_kernel<<<1, 1024, 0, stream>>>(K, s);
  return cudaGetLastError();
}

cudaError_t k3_piece_sum_launch(const MergeVideo* d_mv, int32_t nv, int32_t K, int32_t dim,
                                int64_t pieces_bound, int32_t stride, MergeScratch s,
                                cudaStream_t stream) {
  (void)nv;
  if (K <= 0 || pieces_bound <= 0) return cudaSuccess;
  k3_piece_sum_kernel<<<(unsigned)pieces_bound, kT, 0, stream>>>(d_mv, K, dim, stride, s);
  return cudaGetLastError();
}

cudaError_t k3_clip_sum_launch(int32_t K, int32_t dim, MergeScratch s, cudaStream_t stream) {
  if (K <= 0) return cudaSuccess;
  k3_clip_sum_kernel<<<K, kT, 0, stream>>>(dim, s);
  return cudaGetLastError();
}

cudaError_t k3_round_launch(const MergeVideo* d_mv, int32_t nv, int32_t dim, int64_t n_alive,
                            double theta, double band_rel, MergeScratch s, cudaStream_t stream) {
  if (n_alive > 0) k3_cos_kernel<<<(unsigned)n_alive, kT, 0, stream>>>(d_mv, n_alive, dim, s);
  k3_decide_kernel<<<1, 1024, 0, stream>>>(nv, n_alive, theta, band_rel, s);
  return cudaGetLastError();
}

cudaError_t k3_finish_launch(const MergeVideo* d_mv, int32_t nv, int32_t K, int64_t n_alive,
                             MergeScratch s, int32_t* final_cuts, int32_t* n_final,
                             double* detected_cos, cudaStream_t stream) {
  cudaMemsetAsync(n_final, 0, sizeof(int32_t) * nv, stream);
  const int64_t n = n_alive > K ? n_alive : K;
  if (n > 0)
    k3_finish_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(d_mv, nv, K, n_alive, s,
                                                                       final_cuts, n_final,
                                                                       detected_cos);
  return cudaGetLastError();
}

}  // namespace clipdetect
