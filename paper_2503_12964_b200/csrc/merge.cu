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
// <=16-frame piece, pieces ascending inside a clip; a merged range's sum is
// the previous round's range sums added in ascending order; fixed shuffle
// trees for the dot products and norms); no float atomics.  The oracle sums a
// merged clip frame by frame, the device piece by piece and range by range:
// same terms, different association (~1e-16 relative).
//
// The rounds run on the device (k3_rounds_kernel, one cooperative launch, grid
// syncs between the phases): no host round trip per round, and a merged
// range's sum and squared norm are kept, so a round costs O(D) per alive
// boundary plus O(D) per absorbed range — not O(clips in range x D).
#include <cooperative_groups.h>
#include <math.h>

#include "common.cuh"
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

// Block-wide exclusive scan helper (any multiple of 32 threads up to 1024).
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
    int32_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
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

// Per-video clip counts and clip bases (ncuts: the detected-cut counts K2 left
// on the device, or null when the host already filled them) and the total clip
// count K (s.Kd): nothing goes back to the host between K2 and K3.
__global__ void __launch_bounds__(1024)
k3_video_table_kernel(MergeVideo* __restrict__ mv, int32_t nv, const int32_t* __restrict__ ncuts,
                      MergeScratch s) {
  __shared__ int32_t wsum[33];
  int32_t carry = 0;
  for (int32_t base = 0; base < nv; base += 1024) {
    const int32_t v = base + threadIdx.x;
    int32_t nc = 0;
    if (v < nv) nc = ncuts ? ncuts[v] + 1 : mv[v].n_clips;
    int32_t tot;
    const int32_t e = block_excl_scan(nc, wsum, tot);
    if (v < nv) {
      mv[v].n_clips = nc;
      mv[v].clip_base = carry + e;
    }
    carry += tot;
  }
  if (threadIdx.x == 0) *s.Kd = carry;
}

// clip tables + per-video state reset (grid: an upper bound of K clips)
__global__ void k3_clip_table_kernel(const MergeVideo* __restrict__ mv, int32_t nv,
                                     const int32_t* __restrict__ cuts, MergeScratch s) {
  const int32_t K = *s.Kd;
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  CD_CHECK(K <= (int64_t)gridDim.x * blockDim.x);  // K2's cuts obey the min clip length
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


// piece_base = exclusive scan of ceil(len/kPieceFrames); alive = clips that
// start a boundary (clip_f0 > 0), in order.
__global__ void __launch_bounds__(1024)
k3_scan_kernel(MergeScratch s) {
  __shared__ int32_t wsum[33];
  const int32_t K = *s.Kd;
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
    s.counters[2] = 0;
    s.counters[3] = 0;
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
__device__ __forceinline__ void piece_sum(const MergeVideo* __restrict__ mv, int32_t dim,
                                          int32_t stride, const MergeScratch& s, int32_t K,
                                          int64_t p) {
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

// one block per piece, grid-stride (the grid is sized from an upper bound of
// the piece count: the count itself is only on the device)
__global__ void __launch_bounds__(kT)
k3_piece_sum_kernel(const MergeVideo* __restrict__ mv, int32_t dim, int32_t stride,
                    MergeScratch s) {
  const int32_t K = *s.Kd;
  const int64_t np = s.piece_base[K];
  for (int64_t p = blockIdx.x; p < np; p += gridDim.x) piece_sum(mv, dim, stride, s, K, p);
}

// S[k][d] = sum over the clip's pieces, ascending; norm2[k] = |S_k|^2 (one
// block per clip, grid-stride)
__global__ void __launch_bounds__(kT)
k3_clip_sum_kernel(int32_t dim, MergeScratch s) {
  __shared__ double red[kT / 32];
  const int32_t K = *s.Kd;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int32_t k = blockIdx.x; k < K; k += gridDim.x) {
    const int32_t p0 = s.piece_base[k], p1 = s.piece_base[k + 1];
    double n2 = 0.0;
    for (int32_t d = threadIdx.x; d < dim; d += kT) {
      double acc = 0.0;
      for (int32_t p = p0; p < p1; ++p) acc += s.P[(int64_t)p * dim + d];
      s.S[(int64_t)k * dim + d] = acc;
      n2 += acc * acc;
    }
    for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
    if (lane == 0) red[warp] = n2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kT / 32; ++w) t += red[w];
      s.norm2[k] = t;
    }
    __syncthreads();
  }
}

// Left range start of alive boundary b (the previous boundary of the same
// video, else the video's first clip).
__device__ __forceinline__ int32_t left_start(const MergeVideo* __restrict__ mv, const int32_t* alive,
                                              const int32_t* clip_video, int64_t b, int32_t v) {
  return (b > 0 && clip_video[alive[b - 1]] == v) ? alive[b - 1] : mv[v].clip_base;
}

// All merge rounds of every video in one cooperative launch.  Range sums live
// in S at the range's first clip (S[k] = clip sum before any merge), their
// squared norms in norm2.  Per round:
//   1. cosines of the alive boundaries of videos not done: one warp per
//      boundary, c = dot / (sqrt(|L|^2) sqrt(|R|^2)) (0 if a norm is 0);
//   2. block 0: decisions (c >= theta merges, band hits |c - theta| <=
//      band_rel * theta counted every evaluation), ordered compaction of the
//      kept boundaries, the runs of merged boundaries (each run joins the
//      range on its left) cut into chunks of <= kChunk absorbed ranges, and
//      per-video rounds / done flags;
//   3a. every chunk: partial = sum of its ranges, ascending (the first chunk
//      of a run starts with the run's own range), into the scratch rows of P;
//   3b. every run: S[dest] = sum of its chunks' partials, ascending; norm2.
constexpr int kChunk = 64;

__global__ void __launch_bounds__(kT)
k3_rounds_kernel(const MergeVideo* __restrict__ mv, int32_t nv, int32_t dim, double theta,
                 double band_rel, int32_t max_rounds, MergeScratch s) {
  const int32_t K = *s.Kd;
  (void)K;  // bounds of the checked build
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ int32_t wsum[33];
  __shared__ double red[kT / 32];
  __shared__ unsigned long long m_tot;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gwarp = (int64_t)blockIdx.x * (kT / 32) + warp;
  const int64_t nwarps = (int64_t)gridDim.x * (kT / 32);
  int32_t* alive = s.alive;
  int32_t* alive2 = s.alive2;
  for (int32_t r = 0; max_rounds <= 0 || r < max_rounds; ++r) {
    const int64_t n_alive = *(volatile int64_t*)&s.counters[0];
    if (n_alive == 0) break;
    CD_CHECK(n_alive < K);
    // ---- 1. cosines
    for (int64_t b = gwarp; b < n_alive; b += nwarps) {
      const int32_t rk = alive[b];
      CD_CHECK(rk > 0 && rk < K && (b == 0 || alive[b - 1] < rk));  // sorted right-clip indices
      const int32_t v = s.clip_video[rk];
      if (s.vstate[4 * v + VS_DONE]) continue;
      const int32_t lk = left_start(mv, alive, s.clip_video, b, v);
      const double* __restrict__ L = s.S + (int64_t)lk * dim;
      const double* __restrict__ R = s.S + (int64_t)rk * dim;
      double dot = 0.0;
      for (int32_t d = lane; d < dim; d += 32) dot += L[d] * R[d];
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (lane == 0) {
        const double sa = sqrt(s.norm2[lk]), sb = sqrt(s.norm2[rk]);
        s.cos_b[b] = (sa == 0.0 || sb == 0.0) ? 0.0 : dot / (sa * sb);
      }
    }
    grid.sync();
    // ---- 2. decisions, compaction, runs (block 0)
    if (blockIdx.x == 0) {
      for (int32_t v = threadIdx.x; v < nv; v += kT) s.valive[v] = 0;
      if (threadIdx.x == 0) m_tot = 0;
      __syncthreads();
      // merged(b): b evaluated this round (its video not done) and c >= theta
      auto merged_at = [&](int64_t b, int32_t v) {
        return s.clip_video[alive[b]] == v && s.cos_b[b] >= theta;
      };
      int32_t carry = 0, rcarry = 0;
      for (int64_t base = 0; base < n_alive; base += kT) {
        const int64_t b = base + threadIdx.x;
        int32_t keep = 0, rk = 0, run0 = 0, runend = 0;
        if (b < n_alive) {
          rk = alive[b];
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
              atomicAdd(&m_tot, 1ull);
              // a run of merged boundaries of video v: [first, last]
              run0 = !(b > 0 && merged_at(b - 1, v));
              runend = !(b + 1 < n_alive && merged_at(b + 1, v));
            }
          }
          if (keep) atomicAdd(reinterpret_cast<unsigned long long*>(&s.valive[v]), 1ull);
        }
        int32_t tot, rtot;
        const int32_t e = block_excl_scan(keep, wsum, tot);
        const int32_t re = block_excl_scan(run0, wsum, rtot);
        if (keep) alive2[carry + e] = rk;
        if (run0) {
          s.run_dest[rcarry + re] = left_start(mv, alive, s.clip_video, b, s.clip_video[rk]);
          s.run_lo[rcarry + re] = (int32_t)b;
        }
        if (runend) s.run_hi[rcarry + re + run0 - 1] = (int32_t)(b + 1);  // its run's number
        carry += tot;
        rcarry += rtot;
      }
      __syncthreads();
      // chunk bases of the runs: run q has ceil((hi - lo) / kChunk) chunks
      int32_t ccarry = 0;
      for (int32_t base = 0; base < rcarry; base += kT) {
        const int32_t q = base + threadIdx.x;
        const int32_t nc = q < rcarry ? (s.run_hi[q] - s.run_lo[q] + kChunk - 1) / kChunk : 0;
        int32_t tot;
        const int32_t e = block_excl_scan(nc, wsum, tot);
        if (q < rcarry) s.run_cbase[q] = ccarry + e;
        ccarry += tot;
      }
      for (int32_t v = threadIdx.x; v < nv; v += kT) {
        int64_t* vs = s.vstate + 4 * v;
        if (vs[VS_DONE]) continue;
        vs[VS_ROUNDS] += 1;
        if (vs[VS_MERGES] == 0 || s.valive[v] == 0) vs[VS_DONE] = 1;
        vs[VS_MERGES] = 0;
      }
      if (threadIdx.x == 0) {
        s.run_cbase[rcarry] = ccarry;
        s.counters[1] = (int64_t)m_tot;
        s.counters[2] = rcarry;
        s.counters[3] = ccarry;
        s.counters[4] = carry;  // next round's n_alive (published after the sums)
      }
    }
    grid.sync();
    const int64_t merges = *(volatile int64_t*)&s.counters[1];
    if (merges == 0) break;  // every block reads the same value
    const int32_t nruns = (int32_t)*(volatile int64_t*)&s.counters[2];
    const int32_t nchunks = (int32_t)*(volatile int64_t*)&s.counters[3];
    // ---- 3a. chunk partial sums (rows of P: the piece sums are no longer needed)
    for (int32_t w = blockIdx.x; w < nchunks; w += gridDim.x) {
      int32_t lo = 0, hi = nruns - 1;  // run of chunk w: last run with cbase <= w
      while (lo < hi) {
        const int32_t m = (lo + hi + 1) >> 1;
        if (s.run_cbase[m] <= w) lo = m; else hi = m - 1;
      }
      const int32_t q = lo, c = w - s.run_cbase[q];
      const int32_t t0 = s.run_lo[q] + c * kChunk;
      const int32_t t1 = min(s.run_hi[q], t0 + kChunk);
      CD_CHECK(w < K && c >= 0 && t0 < t1 && t1 <= n_alive && s.run_dest[q] < alive[t0]);
      const double* __restrict__ own = c == 0 ? s.S + (int64_t)s.run_dest[q] * dim : nullptr;
      double* __restrict__ out = s.P + (int64_t)w * dim;
      for (int32_t d = threadIdx.x; d < dim; d += kT) {
        double acc = own ? own[d] : 0.0;
        for (int32_t t = t0; t < t1; ++t) acc += s.S[(int64_t)alive[t] * dim + d];
        out[d] = acc;
      }
    }
    grid.sync();
    // ---- 3b. merged range sums and norms
    for (int32_t q = blockIdx.x; q < nruns; q += gridDim.x) {
      const int32_t dest = s.run_dest[q], c0 = s.run_cbase[q], c1 = s.run_cbase[q + 1];
      CD_CHECK(dest >= 0 && dest < K && c0 < c1 && c1 <= nchunks);
      double* __restrict__ D = s.S + (int64_t)dest * dim;
      double n2 = 0.0;
      for (int32_t d = threadIdx.x; d < dim; d += kT) {
        double acc = s.P[(int64_t)c0 * dim + d];
        for (int32_t c = c0 + 1; c < c1; ++c) acc += s.P[(int64_t)c * dim + d];
        D[d] = acc;
        n2 += acc * acc;
      }
      for (int o = 16; o > 0; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
      if (lane == 0) red[warp] = n2;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kT / 32; ++w) t += red[w];
        s.norm2[dest] = t;
      }
      __syncthreads();
    }
    int32_t* tmp = alive;
    alive = alive2;
    alive2 = tmp;
    if (blockIdx.x == 0 && threadIdx.x == 0) s.counters[0] = s.counters[4];
    grid.sync();
  }
  // the final alive list is in s.alive for k3_finish_kernel
  if (alive != s.alive) {
    const int64_t n_alive = *(volatile int64_t*)&s.counters[0];
    for (int64_t b = (int64_t)blockIdx.x * kT + threadIdx.x; b < n_alive; b += (int64_t)gridDim.x * kT)
      s.alive[b] = alive[b];
  }
}

__global__ void k3_finish_kernel(const MergeVideo* __restrict__ mv, int32_t nv,
                                 MergeScratch s, int32_t* __restrict__ final_cuts,
                                 int32_t* __restrict__ n_final, double* __restrict__ detected_cos) {
  const int32_t K = *s.Kd;
  const int64_t n_alive = s.counters[0];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < K;
       i += (int64_t)gridDim.x * blockDim.x) {
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
    if (detected_cos != nullptr) {
      const int32_t v = s.clip_video[i];
      const int32_t j = (int32_t)i - mv[v].clip_base;
      if (j >= 1) detected_cos[mv[v].cut_base + j - 1] = s.cos_clip[i];
    }
  }
}

}  // namespace

cudaError_t k3_prepare_launch(MergeVideo* d_mv, int32_t nv, int32_t Kub, const int32_t* d_ncuts,
                              const int32_t* cuts, MergeScratch s, cudaStream_t stream) {
  k3_video_table_kernel<<<1, 1024, 0, stream>>>(d_mv, nv, d_ncuts, s);
  const int32_t nthreads = Kub > nv ? Kub : nv;
  k3_clip_table_kernel<<<(nthreads + 255) / 256, 256, 0, stream>>>(d_mv, nv, cuts, s);
  k3_scan_kernel<<<1, 1024, 0, stream>>>(s);
  return cudaGetLastError();
}

cudaError_t k3_piece_sum_launch(const MergeVideo* d_mv, int32_t dim, int64_t pieces_bound,
                                int32_t stride, MergeScratch s, cudaStream_t stream) {
  if (pieces_bound <= 0) return cudaSuccess;
  const int64_t grid = pieces_bound < kSMs * 8 ? pieces_bound : kSMs * 8;
  k3_piece_sum_kernel<<<(unsigned)grid, kT, 0, stream>>>(d_mv, dim, stride, s);
  return cudaGetLastError();
}

cudaError_t k3_clip_sum_launch(int32_t Kub, int32_t dim, MergeScratch s, cudaStream_t stream) {
  if (Kub <= 0) return cudaSuccess;
  k3_clip_sum_kernel<<<Kub < kSMs * 8 ? Kub : kSMs * 8, kT, 0, stream>>>(dim, s);
  return cudaGetLastError();
}

cudaError_t k3_rounds_launch(const MergeVideo* d_mv, int32_t nv, int32_t dim, int64_t max_alive,
                             double theta, double band_rel, int32_t max_rounds, int sm_count,
                             MergeScratch s, cudaStream_t stream) {
  static int occ = 0;
  if (occ == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k3_rounds_kernel, kT, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
  }
  // enough warps for one boundary each (up to every co-resident block)
  int64_t want = (max_alive + kT / 32 - 1) / (kT / 32);
  int64_t grid = (int64_t)sm_count * occ;
  if (want < grid) grid = want < 1 ? 1 : want;
  void* args[] = {(void*)&d_mv, (void*)&nv, (void*)&dim, (void*)&theta, (void*)&band_rel,
                  (void*)&max_rounds, (void*)&s};
  return cudaLaunchCooperativeKernel((const void*)k3_rounds_kernel, dim3((unsigned)grid), dim3(kT),
                                     args, 0, stream);
}

cudaError_t k3_finish_launch(const MergeVideo* d_mv, int32_t nv, int32_t Kub, MergeScratch s,
                             int32_t* final_cuts, int32_t* n_final, double* detected_cos,
                             cudaStream_t stream) {
  cudaMemsetAsync(n_final, 0, sizeof(int32_t) * nv, stream);
  const int32_t grid = (Kub + 255) / 256 < kSMs * 4 ? (Kub + 255) / 256 : kSMs * 4;
  if (grid > 0)
    k3_finish_kernel<<<grid, 256, 0, stream>>>(d_mv, nv, s, final_cuts, n_final, detected_cos);
  return cudaGetLastError();
}

}  // namespace clipdetect
