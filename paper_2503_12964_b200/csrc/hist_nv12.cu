// hist_nv12.cu — K1 for NV12 input (NEXT f1): fused NV12 -> RGB -> HSV bin ->
// per-frame histogram (rows a1-a3 on the decoder's native surface format).
//
// Reading O0: the RGB frame of the method is the BT.601
// limited-range conversion of NVDEC's NV12 output in 20-bit fixed point
// (binfn.cuh nv12_*), after which the histogram is exactly K1's (O1, O2;
// PAPER.md:35 §2.1 "analyzing the color changes between frames"; NVDEC:
// PAPER.md:43 §2.3).  Fusing the conversion into the histogram pass means the
// RGB frame never exists in HBM: 1.5 bytes per pixel are read instead of 3
// (+3 written and re-read by a separate conversion kernel).
//
// B200 design (same skeleton as hist.cu K1; DESIGN.md §7 "K1-NV12"):
//  * persistent grid, one CTA per SM, contiguous ranges of "stages" of the
//    flattened (segment, frame, stage) space; a stage is R chroma-block rows of
//    one frame (R = floor(20480 / W): 16 at 720p, 10 at 1080p): the 2R Y rows
//    and the R UV rows are two contiguous byte ranges, moved by two 1-D TMA
//    bulk copies completing on one mbarrier into a 2-deep ring of 60 KiB
//    slots;
//  * 24 consumer warps; a work unit is a 2 x 8 pixel tile (two LDS.64 of Y,
//    one LDS.64 of interleaved UV = 4 chroma blocks); the chroma terms are
//    computed once per 2 x 2 block, each horizontal pixel pair is converted
//    directly into u16x2 lanes (VIADDMNMX luma clamp, IMAD, PRMT pack,
//    VIMNMX.S16x2.RELU saturation) and then coded exactly like K1
//    (code_pair_dir_pre, 64 KiB hue table, direct-offset codes, ATOMS into an
//    8192-entry code histogram, one RED per non-zero code at the frame flush);
//  * the lane -> tile map rotates by two warps per stage, so that the lanes
//    that get one tile fewer than the others move over the four schedulers.
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

constexpr int kNvStages = 2;
constexpr int kNvStageBytes = 61440;  // 3 * R * W <= 61440  <=>  R * W <= 20480
constexpr int kNvWarps = 24;  // B200 A/B (profiles/r02/ab/): +1.0 % over 20, 16 and 28 -2 %
constexpr int kNvConsumers = kNvWarps * 32;
constexpr int kNvThreads = kNvConsumers + 32;
constexpr int kNvLutBytes = 65536;
static_assert(kNvConsumers % 64 == 0, "rotation by two warps");
constexpr uint32_t kNvDynSmemBase = 0x400;  // see hist.cu kDynSmemBase

// The stage in a ring slot, written by the producer before it arms the slot's
// "full" barrier (see hist.cu StageMeta): the consumers run no iterator.
struct NvMeta {
  uint32_t* gh;  // the frame's global histogram, when this stage is its last; else null
  int32_t nr;    // chroma-block rows in the stage
  int32_t W;     // frame width
  int32_t seq;   // the stage's index in the CTA's range (checked builds verify the hand-off)
  int32_t pad;
};

struct NvSmem {
  alignas(128) uint8_t buf[kNvStages][kNvStageBytes];
  NvMeta meta[kNvStages];
  uint8_t lut[kNvLutBytes];  // lut[lut_index(na, d)] = lut_entry_dir(na, d, kHashNv12)
  uint32_t hist[kDirCodes];
  uint8_t c2b[kDirCodes];
  uint64_t full[kNvStages];
  uint64_t empty[kNvStages];
  uint64_t tab;  // the lut + c2b bulk copies at launch
  MadK mk;
};
constexpr uint32_t kNvLutOff = (uint32_t)offsetof(NvSmem, lut);
constexpr uint32_t kNvHistOff = (uint32_t)offsetof(NvSmem, hist);

// Walks the flattened (segment, frame, stage) space.
struct NvIter {
  const Nv12Seg* segs;
  int32_t seg, frame, st;
  int32_t H, W, R, stages, n_frames;
  const uint8_t* frames;
  uint32_t* hist;
  __device__ void load() {
    const Nv12Seg& g = segs[seg];
    hist = g.hist;
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

// hue-table load / code-histogram increment (IMM: register + immediate address)
template <bool IMM>
__device__ __forceinline__ uint32_t nv_lut_ld(uint32_t sb, uint32_t x) {
  uint32_t v;
  if constexpr (IMM)
    asm("ld.shared.u8 %0, [%1+%2];" : "=r"(v) : "r"(x), "n"(kNvDynSmemBase + kNvLutOff));
  else
    asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(sb + kNvLutOff + x));
  return v;
}
template <bool IMM>
__device__ __forceinline__ void nv_hist_inc(uint32_t sb, uint32_t x) {
  if constexpr (IMM)
    asm volatile("red.shared.add.u32 [%0+%1], 1;" ::"r"(x), "n"(kNvDynSmemBase + kNvHistOff) : "memory");
  else
    asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(sb + kNvHistOff + x) : "memory");
}

// One 2 x 8 tile: Y row 0 (y0), Y row 1 (y1), UV (c): 8 pixel pairs, issued
// phase by phase (conversion + codes, table loads, atomics).
template <bool IMM>
__device__ __forceinline__ void nv_tile(uint2 y0, uint2 y1, uint2 c, uint32_t sb, MadK mk) {
  uint32_t pre[8], ia[8], ib[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int32_t ruv, guv, buv;
    block_chroma(k < 2 ? c.x : c.y, k, ruv, guv, buv);
    const uint32_t w0 = k < 2 ? y0.x : y0.y, w1 = k < 2 ? y1.x : y1.y;
    const int o = 2 * (k & 1);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint32_t w = r ? w1 : w0;
      const int j = 2 * k + r;
      uint32_t R, G, B;
      nv12_pair_rgb(__byte_perm(w, 0u, 0x4440u | o), __byte_perm(w, 0u, 0x4440u | (o + 1)), ruv,
                    guv, buv, R, G, B);
      pre[j] = code_pair_dir_pre(R, G, B, mk, ia[j], ib[j]);
    }
  }
  uint32_t qa[8], qb[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    qa[j] = nv_lut_ld<IMM>(sb, ia[j]);
    qb[j] = nv_lut_ld<IMM>(sb, ib[j]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    CD_CHECK(dir_off_lo(pre[j], qa[j]) < 4u * kDirCodes && dir_off_hi(pre[j], qb[j]) < 4u * kDirCodes);
    nv_hist_inc<IMM>(sb, dir_off_lo(pre[j], qa[j]));
    nv_hist_inc<IMM>(sb, dir_off_hi(pre[j], qb[j]));
  }
}

// The consumer loop.  A stage holds nu = R * W / 8 tiles (2,560 at 720p, 2,400
// at 1080p and 4K) for 768 lanes: at 720p 256 lanes take four tiles and 512
// three.  The lane -> tile map is rotated by 64 lanes (two warps) per stage so
// that the lanes with the extra tile move over the four schedulers instead of
// always being the same ones.
template <int MODE, bool IMM>
__device__ __forceinline__ void nv_consume(NvSmem& sm, uint32_t sb, int32_t n, uint32_t* sink) {
  const int tid = threadIdx.x;
  MadK mk;
  {
    const volatile uint32_t* v = reinterpret_cast<const volatile uint32_t*>(&sm.mk);
    uint32_t* m = reinterpret_cast<uint32_t*>(&mk);
#pragma unroll
    for (int j = 0; j < (int)(sizeof(MadK) / 4); ++j) m[j] = v[j];
  }
  uint32_t xacc = 0;
  if constexpr (MODE == kModeFast) mbar_wait(&sm.tab, 0);  // the tables have landed
  // per-step increments of the (block row, 8-column chunk) position
  int32_t cur_w = -1, wu = 1, dq = 0, dr = 0, q64 = 0, r64 = 0, q640 = 0, r640 = 0;
  // this stage's virtual lane u0 = (tid + 64 i) mod kNvConsumers and its (block row,
  // 8-column chunk) = divmod(u0, wu), advanced incrementally (no per-stage division)
  int32_t u0 = tid, br0 = 0, cx0 = 0;
  uint32_t slot = 0, par = 0;
  for (int32_t i = 0; i < n; ++i) {
    mbar_wait(&sm.full[slot], par);
    const NvMeta meta = sm.meta[slot];
    CD_CHECK(meta.seq == i && meta.nr >= 1 && (meta.W & 15) == 0);  // the slot holds stage i
    if (meta.W != cur_w) {
      cur_w = meta.W;
      wu = meta.W >> 3;
      dq = kNvConsumers / wu;
      dr = kNvConsumers - dq * wu;
      q64 = 64 / wu;
      r64 = 64 - q64 * wu;
      q640 = dq;
      r640 = dr;
      br0 = u0 / wu;
      cx0 = u0 - br0 * wu;
    }
    const int32_t nr = meta.nr, W = meta.W;
    const uint8_t* buf = sm.buf[slot];
    const uint8_t* uvb = buf + 2 * nr * W;
    const int32_t nu = nr * wu;
    int32_t u = u0, br = br0, cx = cx0;
#pragma unroll 1
    for (; u < nu; u += kNvConsumers) {
      CD_CHECK(br < nr && cx < wu);  // the tile lies inside the stage's rows
      const uint8_t* yp = buf + 2 * br * W + 8 * cx;
      const uint2 a = *reinterpret_cast<const uint2*>(yp);
      const uint2 b = *reinterpret_cast<const uint2*>(yp + W);
      const uint2 c = *reinterpret_cast<const uint2*>(uvb + br * W + 8 * cx);
      if constexpr (MODE == kModeRead)
        xacc ^= a.x ^ a.y ^ b.x ^ b.y ^ c.x ^ c.y;
      else
        nv_tile<IMM>(a, b, c, sb, mk);
      cx += dr;
      br += dq;
      if (cx >= wu) {
        cx -= wu;
        ++br;
      }
    }
    // every consumer lane releases the slot (its reads are done; no warp sync:
    // B200 A/B +1.4 % over one release per warp, the reverse of K1)
    mbar_arrive(&sm.empty[slot]);
    if (++slot == kNvStages) {
      slot = 0;
      par ^= 1u;
    }
    // rotate the lane -> tile map by 64 lanes: u0 += 64 (mod kNvConsumers)
    u0 += 64;
    br0 += q64;
    cx0 += r64;
    if (cx0 >= wu) {
      cx0 -= wu;
      ++br0;
    }
    if (u0 >= kNvConsumers) {
      u0 -= kNvConsumers;
      br0 -= q640;
      cx0 -= r640;
      if (cx0 < 0) {
        cx0 += wu;
        --br0;
      }
    }
    if (MODE == kModeFast && meta.gh != nullptr) {
      // one RED per non-zero code to the frame's global bins (as K1)
      named_bar_sync(1, kNvConsumers);
      uint32_t* gh = meta.gh;
      for (uint32_t cc = tid; cc < (uint32_t)kDirCodes; cc += kNvConsumers) {
        const uint32_t cnt = sm.hist[cc];
        if (cnt) {
          sm.hist[cc] = 0u;
          CD_CHECK(sm.c2b[cc] < 162);  // only reachable codes counted
          atomicAdd(gh + sm.c2b[cc], cnt);
        }
      }
      named_bar_sync(1, kNvConsumers);
    }
  }
  if (MODE == kModeRead && xacc == 0x9E3779B9u) sink[0] = xacc;
}

template <int MODE>
__global__ void __launch_bounds__(kNvThreads, 1)
k1_nv12_kernel(const Nv12Seg* __restrict__ segs, int32_t nseg, int64_t total_stages,
               MadK mk_param, const uint8_t* __restrict__ tables, uint32_t* __restrict__ sink) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  NvSmem& sm = *reinterpret_cast<NvSmem*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int64_t s_begin = total_stages * blockIdx.x / gridDim.x;
  const int64_t s_end = total_stages * (blockIdx.x + 1) / gridDim.x;

  if (MODE == kModeFast) {
    for (int i = tid; i < kDirCodes; i += kNvThreads) sm.hist[i] = 0u;
  }
  if (tid == 0) {
    sm.mk = mk_param;
    for (int i = 0; i < kNvStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kNvConsumers);
    }
    mbar_init(&sm.tab, 1);
    fence_mbar_init();
    if (MODE == kModeFast) {  // hue table and code -> bin map (k1_tables_build, kHashNv12)
      CD_CHECK(tables != nullptr && (reinterpret_cast<uintptr_t>(tables) & 15) == 0);
      const uint64_t pol = policy_evict_last();
      mbar_arrive_expect_tx(&sm.tab, kNvLutBytes + kDirCodes);
      bulk_g2s(sm.lut, tables, kNvLutBytes, &sm.tab, pol);
      bulk_g2s(sm.c2b, tables + kNvLutBytes, kDirCodes, &sm.tab, pol);
    }
  }
  __syncthreads();
  if (s_begin >= s_end) {
    if (MODE == kModeFast && tid == 0) mbar_wait(&sm.tab, 0);  // no copy outlives the CTA
    return;
  }
  const int32_t n = (int32_t)(s_end - s_begin);

  if (warp == kNvWarps) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      NvIter it;
      it.seek(segs, nseg, s_begin);
      uint32_t slot = 0, par = 0;
      for (int32_t i = 0; i < n; ++i) {
        if (i >= kNvStages) mbar_wait(&sm.empty[slot], par ^ 1u);
        const int32_t nr = it.nr(), W = it.W;
        const uint32_t ybytes = 2u * nr * W, cbytes = (uint32_t)nr * W;
        const uint8_t* ysrc = it.frame_base() + 2 * (int64_t)it.st * it.R * W;
        const uint8_t* csrc = it.frame_base() + (int64_t)it.H * W + (int64_t)it.st * it.R * W;
        CD_CHECK(nr >= 1 && ybytes + cbytes <= kNvStageBytes && ((ybytes | cbytes) & 15) == 0);
        CD_CHECK(ysrc >= it.frame_base() && csrc + cbytes <= it.frame_base() + 3 * (int64_t)it.H * W / 2);
        CD_CHECK(it.frame < it.n_frames);
        uint32_t* gh = it.hist + (int64_t)it.frame * 162;
        const bool last = i + 1 == n;
        const bool changed = it.next(!last);  // the frame ends with this stage
        sm.meta[slot] = NvMeta{(last || changed) ? gh : nullptr, nr, W, i, 0};
        mbar_arrive_expect_tx(&sm.full[slot], ybytes + cbytes);  // release: orders the meta store
        bulk_g2s(sm.buf[slot], ysrc, ybytes, &sm.full[slot], pol);
        bulk_g2s(sm.buf[slot] + ybytes, csrc, cbytes, &sm.full[slot], pol);
        if (++slot == kNvStages) {
          slot = 0;
          par ^= 1u;
        }
      }
    }
    return;
  }
  // ------------------------------------------------------------ consumers
  const uint32_t sb = smem_u32(smem_raw);
  if (sb == kNvDynSmemBase)
    nv_consume<MODE, true>(sm, sb, n, sink);
  else
    nv_consume<MODE, false>(sm, sb, n, sink);
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
// chroma (U, V), through the fast path's conversion, codes and table (or the
// generic path's conversion and bin_generic).  out[0][(Y<<16)|(U<<8)|V] = lane
// 0 result, out[1][...] = lane 1 result.
__global__ void __launch_bounds__(256)
k5_nv12map_kernel(uint8_t* __restrict__ out, uint32_t nh, uint32_t ns, uint32_t nv, int fast, MadK mk) {
  extern __shared__ __align__(16) uint8_t lut[];
  if (fast) {
    for (int i = threadIdx.x; i < kNvLutBytes; i += blockDim.x) {
      const uint32_t d = (uint32_t)i >> 8, na = lut_unswizzle((uint32_t)i & 255u, d);
      lut[i] = (uint8_t)(na > d ? 0u : lut_entry_dir(na, d, kHashNv12));
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
    if (fast) {
      uint32_t i0, i1;
      const uint32_t pre = code_pair_dir_pre(R, G, B, mk, i0, i1);
      b0 = code_to_bin_dir(dir_off_lo(pre, lut[i0]) >> 2);
      b1 = code_to_bin_dir(dir_off_hi(pre, lut[i1]) >> 2);
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
  if ((e = cudaFuncSetAttribute(k1_nv12_kernel<kModeFast>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(NvSmem))) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k1_nv12_kernel<kModeRead>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)sizeof(NvSmem))) != cudaSuccess)
    return e;
  return cudaFuncSetAttribute(k5_nv12map_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kNvLutBytes);
}

cudaError_t k1_nv12_launch(int mode, const Nv12Seg* d_segs, int32_t nseg, int64_t total,
                           uint32_t nh, uint32_t ns, uint32_t nv, const uint8_t* tables,
                           uint32_t* sink, int sm_count, cudaStream_t stream) {
  if (total <= 0) return cudaSuccess;
  if (mode == kModeGeneric) {
    const int64_t grid = std::min<int64_t>(total, (int64_t)sm_count * 8);
    k1_nv12_generic_kernel<<<(unsigned)grid, 256, 0, stream>>>(d_segs, nseg, total, nh, ns, nv);
    return cudaGetLastError();
  }
  const int grid = (int)std::min<int64_t>(total, sm_count);
  if (mode == kModeFast)
    k1_nv12_kernel<kModeFast><<<grid, kNvThreads, sizeof(NvSmem), stream>>>(d_segs, nseg, total, kMadK,
                                                                          tables, sink);
  else
    k1_nv12_kernel<kModeRead><<<grid, kNvThreads, sizeof(NvSmem), stream>>>(d_segs, nseg, total, kMadK,
                                                                          tables, sink);
  return cudaGetLastError();
}

cudaError_t k5_nv12map_launch(uint8_t* out, uint32_t nh, uint32_t ns, uint32_t nv, int fast,
                              cudaStream_t stream) {
  if (fast)
    k5_nv12map_kernel<<<kSMs, 256, kNvLutBytes, stream>>>(out, nh, ns, nv, 1, kMadK);
  else
    k5_nv12map_kernel<<<kSMs * 8, 256, 0, stream>>>(out, nh, ns, nv, 0, kMadK);
  return cudaGetLastError();
}

}  // namespace clipdetect
