// hist_nv12.cu — K1 for NV12 input (NEXT f1): fused NV12 -> RGB -> HSV bin ->
// per-frame histogram (rows a1-a3 on the decoder's native surface format).
//
// Reading O0: the RGB frame of the method is the BT.601
// limited-range conversion of NVDEC's NV12 output in 20-bit fixed point
// (binfn.cuh nv12_*), after which the histogram is exactly K1's (O1, O2;
// PAPER.md:35 §2.1 "analyzing the color changes between frames").  Fusing the
// conversion into the histogram pass means the RGB frame never exists in HBM:
// 1.5 bytes per pixel are read instead of 3 (+3 written and re-read by a
// separate conversion kernel).
//
// B200 design (same skeleton as hist.cu K1):
//  * persistent grid, one CTA per SM, contiguous ranges of "stages" of the
//    flattened (segment, frame, stage) space; a stage is R chroma-block rows of
//    one frame (R = floor(20480 / W)): the 2R Y rows and the R UV rows are two
//    contiguous byte ranges, moved by two 1-D TMA bulk copies completing on
//    one mbarrier into a 4-deep ring of 24 KiB slots;
//  * 16 consumer warps; a work unit is a 2 x 8 pixel tile (two LDS.64 of Y,
//    one LDS.64 of interleaved UV = 4 chroma blocks); the chroma terms are
//    computed once per 2 x 2 block, each horizontal pixel pair is converted
//    directly into u16x2 lanes (VIADDMNMX luma clamp, IMAD, PRMT pack,
//    VIMNMX.S16x2.RELU saturation) and then coded exactly like K1's LUT
//    variant (code_pair_lut_pre / post, 64 KiB hue table, ATOMS.POPC.INC into
//    a 5120-entry code histogram, code -> bin at the frame flush).
// Fast path: 18x3x3 bins, W % 16 == 0, W <= 20480.  Anything else runs the
// plain generic kernel at the bottom of this file (same conversion, direct
// global loads, bin_generic).
#include <stddef.h>

#include <algorithm>

#include "binfn.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace clipdetect {

namespace {

#ifndef CLIPDETECT_NV_STAGES  // experiment builds (tools/) may override
#define CLIPDETECT_NV_STAGES 2
#endif
constexpr int kNvStages = CLIPDETECT_NV_STAGES;
#ifndef CLIPDETECT_NV_STAGE_BYTES  // experiment builds (tools/) may override
#define CLIPDETECT_NV_STAGE_BYTES 61440
#endif
constexpr int kNvStageBytes = CLIPDETECT_NV_STAGE_BYTES;  // 3 * R * W <= 61440  <=>  R * W <= 20480
constexpr int kNvWarps = 16;
constexpr int kNvConsumers = kNvWarps * 32;
constexpr int kNvLutBytes = 65536;
constexpr int kNvSwz = 3;  // table swizzle (binfn.cuh lut_swizzle): conflict-free rows on NV12 content

// DIR > 0: direct-offset codes (binfn.cuh code_pair_dir_pre, 8192 entries):
// 1 = bank hash d & 3, table swizzle multiplier 4; 2 = hash ((d >> 5) ^ na) & 3,
// multiplier 4; 3 = that hash, multiplier 5 (CLIPDETECT_NV12_DIR selects; 4 = layout 2
// with two tiles per loop iteration; 5 = layout 2 with the lane -> unit map rotated by
// two warps per stage, see ROT below; 6 / 7 = 5 with 20 / 24 consumer warps)
__host__ __device__ constexpr int nv_hash(int dir) { return dir == 1 ? 1 : 4; }
__host__ __device__ constexpr int nv_ks(int dir) { return dir == 3 ? 5 : 4; }
template <int DIR>
struct NvSmem {
  static constexpr int kEntries = DIR ? kDirCodes : kLutCodes;
  alignas(128) uint8_t buf[kNvStages][kNvStageBytes];
  uint8_t lut[kNvLutBytes];
  uint32_t hist[kEntries];
  uint32_t binacc[256];
  uint8_t c2b[kEntries];
  uint64_t full[kNvStages];
  uint64_t empty[kNvStages];
  MadK mk;
};

// Walks the flattened (segment, frame, stage) space.
struct NvIter {
  const Nv12Seg* segs;
  int32_t seg, frame, st;
  int32_t H, W, R, stages, n_frames;
  const uint8_t* frames;
  __device__ void load() {
    const Nv12Seg& g = segs[seg];
    H = g.height;
    W = g.width;
    R = g.rows;
    stages = g.stages;
    n_frames = (int32_t)g.n_frames;
    frames = g.frames;
  }
  __device__ void seek(const Nv12Seg* s, int32_t nseg, int64_t g) {
    segs = s;
    int32_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int32_t m = (lo + hi + 1) >> 1;
      if (s[m].stage_base <= g) lo = m; else hi = m - 1;
    }
    seg = lo;
    load();
    const int64_t rel = g - s[lo].stage_base;
    frame = (int32_t)(rel / stages);
    st = (int32_t)(rel - (int64_t)frame * stages);
  }
  __device__ __forceinline__ int32_t nr() const {
    const int32_t left = (H >> 1) - st * R;
    return left < R ? left : R;
  }
  __device__ __forceinline__ const uint8_t* frame_base() const {
    return frames + (int64_t)frame * (3 * (int64_t)H * W / 2);
  }
  __device__ __forceinline__ bool next(bool more) {
    if (++st == stages) {
      st = 0;
      if (++frame == n_frames) {
        frame = 0;
        ++seg;
        if (more) load();
      }
      return true;
    }
    return false;
  }
};

// Chroma terms of block k (0..3) of a UV word pair.
__device__ __forceinline__ void block_chroma(uint32_t uv, int k, int32_t& ruv, int32_t& guv,
                                             int32_t& buv) {
  const uint32_t U = __byte_perm(uv, 0u, 0x4440u | (2 * k & 3));
  const uint32_t V = __byte_perm(uv, 0u, 0x4440u | ((2 * k + 1) & 3));
  nv12_chroma(U, V, ruv, guv, buv);
}

// Shared-window offset of dynamic shared memory (after the 1 KiB system
// reserve) for a launch without clusters, checked at kernel entry: the table
// loads become LDS [index + imm] with no per-load base add.
constexpr uint32_t kNvDynSmemBase = 0x400;

// NT 2 x 8 tiles: Y row 0 (y0), Y row 1 (y1), UV (c) of each: 8 NT pixel
// pairs, issued phase by phase (conversion + codes, table loads, atomics).
template <int DIR, int NT = 1>
__device__ __forceinline__ void nv_tiles(const uint2* y0s, const uint2* y1s, const uint2* cs,
                                         char* hb, MadK mk) {
  constexpr int P = 8 * NT;
  uint32_t pre[P], ia[P], ib[P];
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const uint2 y0 = y0s[t], y1 = y1s[t], c = cs[t];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      int32_t ruv, guv, buv;
      block_chroma(k < 2 ? c.x : c.y, k, ruv, guv, buv);
      const uint32_t w0 = k < 2 ? y0.x : y0.y, w1 = k < 2 ? y1.x : y1.y;
      const int o = 2 * (k & 1);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t w = r ? w1 : w0;
        const int j = 8 * t + 2 * k + r;
        uint32_t R, G, B;
        nv12_pair_rgb(__byte_perm(w, 0u, 0x4440u | o), __byte_perm(w, 0u, 0x4440u | (o + 1)), ruv,
                      guv, buv, R, G, B);
        if constexpr (DIR)
          pre[j] = code_pair_dir_pre<0, nv_ks(DIR)>(R, G, B, mk, ia[j], ib[j]);
        else
          pre[j] = code_pair_lut_pre<kNvSwz>(R, G, B, mk, ia[j], ib[j]);
      }
    }
  }
  uint32_t qa[P], qb[P];
  constexpr uint32_t lut_s = kNvDynSmemBase + (uint32_t)offsetof(NvSmem<DIR>, lut);
#pragma unroll
  for (int j = 0; j < P; ++j) {
    qa[j] = lds_u8(lut_s + ia[j]);
    qb[j] = lds_u8(lut_s + ib[j]);
  }
  if constexpr (DIR) {
    // ATOMS [offset + imm]: the histogram's shared-window address is a constant too
    constexpr uint32_t hist_s = kNvDynSmemBase + (uint32_t)offsetof(NvSmem<DIR>, hist);
#pragma unroll
    for (int j = 0; j < P; ++j) {
      asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(dir_off_lo(pre[j], qa[j])), "n"(hist_s) : "memory");
      asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(dir_off_hi(pre[j], qb[j])), "n"(hist_s) : "memory");
    }
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const uint32_t code = code_pair_lut_post(pre[j], qa[j], qb[j], mk);
      atomicAdd(reinterpret_cast<uint32_t*>(hb + lut_off_lo(code, mk)), 1u);
      atomicAdd(reinterpret_cast<uint32_t*>(hb + lut_off_hi(code, mk)), 1u);
    }
  }
}

// ROT = 1: a stage holds nu = R * W / 8 units (960 at 720p, 1080p and 4K) for 512
// lanes, so 448 lanes take two units and 64 take one.  Without rotation the
// one-unit lanes are always warps 14 and 15 (schedulers 2 and 3), and schedulers
// 0 and 1 carry 8 of the stage's 30 warp-units against 7.  Rotating the lane ->
// unit map by 64 lanes per stage moves the one-unit pair over warps (12, 13),
// (10, 11), ...: every scheduler carries 15 warp-units per two stages.  NW =
// consumer warps (layout 6: 20, 10 of them take two units; layout 7: 24, 6 of them).
template <int MODE, int DIR, int NT = 1, int ROT = 0, int NW = kNvWarps>
__global__ void __launch_bounds__(NW * 32 + 32, 1)
k1_nv12_kernel(const Nv12Seg* __restrict__ segs, int32_t nseg, int64_t total_stages,
               MadK mk_param, uint32_t* __restrict__ sink) {
  constexpr int kNvConsumers = NW * 32;  // this instance's consumer lanes
  extern __shared__ __align__(128) uint8_t smem_raw[];
  using Smem = NvSmem<DIR>;
  constexpr int kEntries = Smem::kEntries;
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t nbins = 162;

  const int64_t s_begin = total_stages * blockIdx.x / gridDim.x;
  const int64_t s_end = total_stages * (blockIdx.x + 1) / gridDim.x;
  if ((uint32_t)__cvta_generic_to_shared(smem_raw) != kNvDynSmemBase) __trap();  // see nv_tile

  if (MODE == kModeFast) {
    for (int i = tid; i < kEntries; i += blockDim.x) {
      sm.hist[i] = 0u;
      sm.c2b[i] = (uint8_t)(DIR ? code_to_bin_dir(i) : code_to_bin_lut(i));
    }
    for (int i = tid; i < 256; i += blockDim.x) sm.binacc[i] = 0u;
    for (int i = tid; i < kNvLutBytes; i += blockDim.x) {
      const uint32_t d = (uint32_t)i >> 8,
                     na = DIR ? lut_unswizzle_k((uint32_t)i & 255u, d, nv_ks(DIR))
                              : lut_unswizzle((uint32_t)i & 255u, d, kNvSwz);
      sm.lut[i] = (uint8_t)(na > d ? 0u : (DIR ? lut_entry_dir(na, d, nv_hash(DIR)) : lut_entry(na, d)));
    }
  }
  if (tid == 0) {
    sm.mk = mk_param;
    for (int i = 0; i < kNvStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (s_begin >= s_end) return;
  const int32_t n = (int32_t)(s_end - s_begin);

  if (warp == NW) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      NvIter it;
      it.seek(segs, nseg, s_begin);
      uint32_t slot = 0, par = 0;
      for (int32_t i = 0; i < n; ++i) {
        if (i >= kNvStages) mbar_wait(&sm.empty[slot], par ^ 1u);
        const int32_t nr = it.nr();
        const uint32_t ybytes = 2u * nr * it.W, cbytes = (uint32_t)nr * it.W;
        const uint8_t* fb = it.frame_base();
        const int64_t r0 = (int64_t)it.st * it.R;
        mbar_arrive_expect_tx(&sm.full[slot], ybytes + cbytes);
        bulk_g2s(sm.buf[slot], fb + 2 * r0 * it.W, ybytes, &sm.full[slot], pol);
        bulk_g2s(sm.buf[slot] + ybytes, fb + (int64_t)it.H * it.W + r0 * it.W, cbytes,
                 &sm.full[slot], pol);
        it.next(i + 1 < n);
        if (++slot == kNvStages) {
          slot = 0;
          par ^= 1u;
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  MadK mk;
  {
    const volatile uint32_t* v = reinterpret_cast<const volatile uint32_t*>(&sm.mk);
    uint32_t* m = reinterpret_cast<uint32_t*>(&mk);
#pragma unroll
    for (int j = 0; j < (int)(sizeof(MadK) / 4); ++j) m[j] = v[j];
  }
  char* hb = reinterpret_cast<char*>(sm.hist);
  uint32_t xacc = 0;
  NvIter it;
  it.seek(segs, nseg, s_begin);
  // this thread's first unit (block row, 8-column chunk) and the per-step increments
  int32_t cur_seg = -1, wu = 1, br0 = 0, cx0 = 0, dq = 0, dr = 0;
  uint32_t slot = 0, par = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (it.seg != cur_seg) {
      cur_seg = it.seg;
      wu = it.W >> 3;
      br0 = tid / wu;
      cx0 = tid - br0 * wu;
      dq = kNvConsumers / wu;
      dr = kNvConsumers - dq * wu;
    }
    const int32_t nr = it.nr(), W = it.W;
    mbar_wait(&sm.full[slot], par);
    const uint8_t* buf = sm.buf[slot];
    const uint8_t* uvb = buf + 2 * nr * W;
    const int32_t nu = nr * wu;
    int32_t br = br0, cx = cx0, u = tid;
    if constexpr (ROT) {
      static_assert(kNvConsumers % 64 == 0, "rotation by two warps");
      u = (tid + 64 * (i % (kNvConsumers / 64))) % kNvConsumers;  // virtual lane of this stage
      br = u / wu;
      cx = u - br * wu;
    }
    auto step = [&]() {
      cx += dr;
      br += dq;
      if (cx >= wu) {
        cx -= wu;
        ++br;
      }
    };
    if constexpr (MODE == kModeFast && NT == 2) {
      // two of this lane's tiles per iteration: 16 independent pixel-pair chains
#pragma unroll 1
      for (; u + kNvConsumers < nu; u += 2 * kNvConsumers) {
        uint2 a[2], b[2], c[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const uint8_t* yp = buf + 2 * br * W + 8 * cx;
          a[t] = *reinterpret_cast<const uint2*>(yp);
          b[t] = *reinterpret_cast<const uint2*>(yp + W);
          c[t] = *reinterpret_cast<const uint2*>(uvb + br * W + 8 * cx);
          step();
        }
        nv_tiles<DIR, 2>(a, b, c, hb, mk);
      }
    }
#pragma unroll 1
    for (; u < nu; u += kNvConsumers) {
      const uint8_t* yp = buf + 2 * br * W + 8 * cx;
      const uint2 a = *reinterpret_cast<const uint2*>(yp);
      const uint2 b = *reinterpret_cast<const uint2*>(yp + W);
      const uint2 c = *reinterpret_cast<const uint2*>(uvb + br * W + 8 * cx);
      if constexpr (MODE == kModeRead) {
        xacc ^= a.x ^ a.y ^ b.x ^ b.y ^ c.x ^ c.y;
      } else {
        nv_tiles<DIR, 1>(&a, &b, &c, hb, mk);
      }
      step();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[slot]);
    if (++slot == kNvStages) {
      slot = 0;
      par ^= 1u;
    }
    const int32_t seg_now = it.seg, frame_now = it.frame;
    const bool last = (i + 1 == n);
    const bool changed = it.next(!last);
    if (MODE == kModeFast && (last || changed)) {
      // one RED per non-zero code to the frame's global bins (as K1)
      named_bar_sync(1, kNvConsumers);
      uint32_t* gh = segs[seg_now].hist + (int64_t)frame_now * nbins;
      for (uint32_t cc = tid; cc < (uint32_t)kEntries; cc += kNvConsumers) {
        const uint32_t cnt = sm.hist[cc];
        if (cnt) {
          sm.hist[cc] = 0u;
          atomicAdd(gh + sm.c2b[cc], cnt);
        }
      }
      named_bar_sync(1, kNvConsumers);
    }
  }
  if (MODE == kModeRead && xacc == 0x9E3779B9u) sink[0] = xacc;
}

// ------------------------------------------------------------ generic kernel
// Any bins / any even W: one CTA per (frame, 8 block rows) work item,
// direct global loads, exact bin_generic per pixel, smem bin histogram.
constexpr int kGenRows = 8;

__global__ void __launch_bounds__(256)
k1_nv12_generic_kernel(const Nv12Seg* __restrict__ segs, int32_t nseg, int64_t total_items,
                       uint32_t nh, uint32_t ns, uint32_t nv) {
  __shared__ uint32_t h[256];
  const uint32_t nbins = nh * ns * nv;
  for (int64_t w = blockIdx.x; w < total_items; w += gridDim.x) {
    int32_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int32_t m = (lo + hi + 1) >> 1;
      if (segs[m].stage_base <= w) lo = m; else hi = m - 1;
    }
    const Nv12Seg& g = segs[lo];
    const int64_t rel = w - g.stage_base;
    const int64_t f = rel / g.stages;
    const int32_t c = (int32_t)(rel - f * g.stages);
    const int32_t H = g.height, W = g.width;
    const uint8_t* Y = g.frames + f * (3 * (int64_t)H * W / 2);
    const uint8_t* UV = Y + (int64_t)H * W;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0u;
    __syncthreads();
    const int32_t r0 = c * kGenRows, r1 = min(r0 + kGenRows, H >> 1);
    const int32_t bw = W >> 1;
    for (int32_t k = threadIdx.x; k < (r1 - r0) * bw; k += blockDim.x) {
      const int32_t by = r0 + k / bw, bx = k % bw;
      int32_t ruv, guv, buv;
      nv12_chroma(UV[(int64_t)by * W + 2 * bx], UV[(int64_t)by * W + 2 * bx + 1], ruv, guv, buv);
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint8_t* yr = Y + (int64_t)(2 * by + r) * W + 2 * bx;
        uint32_t R, G, B;
        nv12_pair_rgb(yr[0], yr[1], ruv, guv, buv, R, G, B);
#pragma unroll
        for (int l = 0; l < 2; ++l) {
          const uint32_t s = 16 * l;
          atomicAdd(&h[bin_generic((R >> s) & 255u, (G >> s) & 255u, (B >> s) & 255u, nh, ns, nv)], 1u);
        }
      }
    }
    __syncthreads();
    uint32_t* gh = g.hist + f * nbins;
    for (uint32_t b = threadIdx.x; b < nbins; b += blockDim.x)
      if (h[b]) atomicAdd(gh + b, h[b]);
    __syncthreads();
  }
}

// ------------------------------------------------------------ K5 for NV12 (test)
// Every (Y, U, V): lane 0 = Y, lane 1 = Y ^ 0x5A of one pixel pair sharing the
// chroma (U, V), through the fast path's conversion, codes and tables (or the
// generic path's conversion and bin_generic).  out[0][(Y<<16)|(U<<8)|V] = lane
// 0 result, out[1][...] = lane 1 result.
template <int FAST>
__global__ void __launch_bounds__(256)
k5_nv12map_kernel(uint8_t* __restrict__ out, uint32_t nh, uint32_t ns, uint32_t nv, MadK mk,
                  int dir) {
  extern __shared__ __align__(16) uint8_t lut[];
  if (FAST) {
    for (int i = threadIdx.x; i < kNvLutBytes; i += blockDim.x) {
      const uint32_t d = (uint32_t)i >> 8,
                     na = FAST == 2 ? lut_unswizzle_k((uint32_t)i & 255u, d, nv_ks(dir))
                                    : lut_unswizzle((uint32_t)i & 255u, d, kNvSwz);
      lut[i] = (uint8_t)(na > d ? 0u : (FAST == 2 ? lut_entry_dir(na, d, nv_hash(dir)) : lut_entry(na, d)));
    }
    __syncthreads();
  }
  for (uint32_t cidx = blockIdx.x * blockDim.x + threadIdx.x; cidx < (1u << 24);
       cidx += gridDim.x * blockDim.x) {
    const uint32_t Yv = cidx >> 16, U = (cidx >> 8) & 255u, V = cidx & 255u, Y2 = Yv ^ 0x5Au;
    int32_t ruv, guv, buv;
    nv12_chroma(U, V, ruv, guv, buv);
    uint32_t R, G, B;
    nv12_pair_rgb(Yv, Y2, ruv, guv, buv, R, G, B);
    uint32_t b0, b1;
    if (FAST == 2) {  // direct-offset codes (DIR kernel)
      uint32_t i0, i1;
      const uint32_t pre = nv_ks(dir) == 5 ? code_pair_dir_pre<0, 5>(R, G, B, mk, i0, i1)
                                           : code_pair_dir_pre<0, 4>(R, G, B, mk, i0, i1);
      b0 = code_to_bin_dir(dir_off_lo(pre, lut[i0]) >> 2);
      b1 = code_to_bin_dir(dir_off_hi(pre, lut[i1]) >> 2);
    } else if (FAST) {
      uint32_t i0, i1;
      const uint32_t pre = code_pair_lut_pre<kNvSwz>(R, G, B, mk, i0, i1);
      const uint32_t code = code_pair_lut_post(pre, lut[i0], lut[i1], mk);
      b0 = code_to_bin_lut(lut_off_lo(code, mk) >> 2);
      b1 = code_to_bin_lut(lut_off_hi(code, mk) >> 2);
    } else {
      b0 = bin_generic(R & 255u, G & 255u, B & 255u, nh, ns, nv);
      b1 = bin_generic(R >> 16, G >> 16, B >> 16, nh, ns, nv);
    }
    out[cidx] = (uint8_t)b0;
    out[(1u << 24) + ((Y2 << 16) | (U << 8) | V)] = (uint8_t)b1;
  }
}

}  // namespace

int nv12_stage_rows(int32_t width) { return width > 0 ? kNvStageBytes / 3 / width : 0; }

bool nv12_fast_ok(int32_t width, uint32_t nh, uint32_t ns, uint32_t nv) {
  return nh == 18 && ns == 3 && nv == 3 && width % 16 == 0 && nv12_stage_rows(width) >= 1;
}

int nv12_generic_rows() { return kGenRows; }

cudaError_t k1_nv12_configure() {
  cudaError_t e;
#define NV_CONF(M, D)                                                                          \
  e = cudaFuncSetAttribute(k1_nv12_kernel<M, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           (int)sizeof(NvSmem<D>));                                           \
  if (e != cudaSuccess) return e;
  NV_CONF(kModeFast, 0) NV_CONF(kModeFast, 1) NV_CONF(kModeFast, 2) NV_CONF(kModeFast, 3)
  NV_CONF(kModeRead, 0)
  e = cudaFuncSetAttribute(k1_nv12_kernel<kModeFast, 2, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NvSmem<2>));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k1_nv12_kernel<kModeFast, 2, 1, 1>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NvSmem<2>));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k1_nv12_kernel<kModeFast, 2, 1, 1, 20>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NvSmem<2>));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k1_nv12_kernel<kModeFast, 2, 1, 1, 24>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(NvSmem<2>));
  if (e != cudaSuccess) return e;
#undef NV_CONF
  e = cudaFuncSetAttribute(k5_nv12map_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kNvLutBytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k5_nv12map_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kNvLutBytes);
}

cudaError_t k1_nv12_launch(int mode, const Nv12Seg* d_segs, int32_t nseg, int64_t total,
                           uint32_t nh, uint32_t ns, uint32_t nv, uint32_t* sink, int sm_count,
                           int dir, cudaStream_t stream) {
  if (total <= 0) return cudaSuccess;
  if (mode == kModeGeneric) {
    const int64_t grid = std::min<int64_t>(total, (int64_t)sm_count * 8);
    k1_nv12_generic_kernel<<<(unsigned)grid, 256, 0, stream>>>(d_segs, nseg, total, nh, ns, nv);
    return cudaGetLastError();
  }
  const int grid = (int)std::min<int64_t>(total, sm_count);
  if (mode == kModeFast && dir == 1)
    k1_nv12_kernel<kModeFast, 1><<<grid, kNvConsumers + 32, sizeof(NvSmem<1>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else if (mode == kModeFast && dir == 2)
    k1_nv12_kernel<kModeFast, 2><<<grid, kNvConsumers + 32, sizeof(NvSmem<2>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else if (mode == kModeFast && dir == 4)  // layout 2, two tiles per iteration
    k1_nv12_kernel<kModeFast, 2, 2><<<grid, kNvConsumers + 32, sizeof(NvSmem<2>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else if (mode == kModeFast && dir == 5)  // layout 2, rotated lane -> unit map
    k1_nv12_kernel<kModeFast, 2, 1, 1><<<grid, kNvConsumers + 32, sizeof(NvSmem<2>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else if (mode == kModeFast && dir == 6)  // layout 5 with 20 consumer warps
    k1_nv12_kernel<kModeFast, 2, 1, 1, 20><<<grid, 20 * 32 + 32, sizeof(NvSmem<2>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else if (mode == kModeFast && dir == 7)  // layout 5 with 24 consumer warps
    k1_nv12_kernel<kModeFast, 2, 1, 1, 24><<<grid, 24 * 32 + 32, sizeof(NvSmem<2>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else if (mode == kModeFast && dir == 3)
    k1_nv12_kernel<kModeFast, 3><<<grid, kNvConsumers + 32, sizeof(NvSmem<3>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else if (mode == kModeFast)
    k1_nv12_kernel<kModeFast, 0><<<grid, kNvConsumers + 32, sizeof(NvSmem<0>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  else
    k1_nv12_kernel<kModeRead, 0><<<grid, kNvConsumers + 32, sizeof(NvSmem<0>), stream>>>(
        d_segs, nseg, total, kMadK, sink);
  return cudaGetLastError();
}

cudaError_t k5_nv12map_launch(uint8_t* out, uint32_t nh, uint32_t ns, uint32_t nv, int fast,
                              int dir, cudaStream_t stream) {
  if (fast && dir)
    k5_nv12map_kernel<2><<<kSMs, 256, kNvLutBytes, stream>>>(out, nh, ns, nv, kMadK, dir);
  else if (fast)
    k5_nv12map_kernel<1><<<kSMs, 256, kNvLutBytes, stream>>>(out, nh, ns, nv, kMadK, 0);
  else
    k5_nv12map_kernel<0><<<kSMs * 8, 256, 0, stream>>>(out, nh, ns, nv, kMadK, 0);
  return cudaGetLastError();
}

}  // namespace clipdetect
