// sample.cu — K4: clip frame sampling + resize (NEXT f3; readings O10, O11).
//
// The step after the path (§2.1: the final clips feed "video
// embeddings" and transcoding): for every final clip [s, e) of a video, take
// k frames t_i = s + floor((2i+1)(e-s) / 2k) (O10) and resize each to the
// encoder input H2 x W2 with OpenCV's 8-bit bilinear fixed point (O11):
//   horizontal  h = p[x0]*a0 + p[x1]*a1               (11-bit weights)
//   vertical    o = sat((((h0 >> 4)*b0 >> 16) + ((h1 >> 4)*b1 >> 16) + 2) >> 2)
// with the weights of each output coordinate computed in-kernel exactly as
// OpenCV does (double position, float fraction, round-to-nearest-even).
//
// B200 design: HBM-bound gather.  One CTA per (output frame, band of RB output
// rows): one elected thread moves the band's 2*RB source rows HBM -> shared
// memory with 1-D TMA bulk copies (16-byte-aligned supersets of the rows,
// completion on one mbarrier, L2 evict-first); the x weights of the W2 output
// columns are computed once per CTA into shared memory; the 256 threads then
// produce the band's pixels from shared memory (3 channels per thread-pixel)
// and store them (the output is ~8 % of the bytes read).  Many CTAs per SM
// keep the copies of several bands in flight.
#include <math.h>
#include <stdlib.h>

#include "binfn.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace clipdetect {

namespace {

constexpr int kK4Threads = 256;
constexpr int kK4SmemRows = 24 * 1024;  // staged source rows per CTA (swept: tools/k4_micro.py)
constexpr int kK4MaxW2 = 4096;

struct LinCoeff {
  int32_t s0, s1;
  int32_t w0, w1;
};

// O11 coefficients of output coordinate d on an axis src -> dst (OpenCV
// INTER_LINEAR, 8-bit): identical IEEE operations on the device.
__device__ __forceinline__ LinCoeff lin_coeff(int32_t src, int32_t dst, int32_t d) {
  const double scale = 1.0 / ((double)dst / (double)src);
  float f = __double2float_rn(((double)d + 0.5) * scale - 0.5);
  int32_t s = (int32_t)floorf(f);
  f = __fsub_rn(f, (float)s);
  if (s < 0) {
    f = 0.0f;
    s = 0;
  }
  if (s >= src - 1) {
    f = 0.0f;
    s = src - 1;
  }
  LinCoeff c;
  c.s0 = s;
  c.s1 = s + 1 < src ? s + 1 : src - 1;
  c.w0 = __float2int_rn(__fmul_rn(__fsub_rn(1.0f, f), 2048.0f));
  c.w1 = __float2int_rn(__fmul_rn(f, 2048.0f));
  return c;
}

// One source pixel of an NV12 frame -> (r, g, b) by reading O0 (scalar).
__device__ __forceinline__ void nv12_px(const uint8_t* yrow, const uint8_t* uvrow, int32_t x,
                                        int32_t& r, int32_t& g, int32_t& b) {
  int32_t ruv, guv, buv;
  const int32_t xc = x & ~1;
  nv12_chroma(uvrow[xc], uvrow[xc + 1], ruv, guv, buv);
  const int32_t l = nv12_luma(yrow[x]);
  r = min(max((l + ruv) >> 20, 0), 255);
  g = min(max((l + guv) >> 20, 0), 255);
  b = min(max((l + buv) >> 20, 0), 255);
}

// NV12: frames are u8 [n][H*3/2][W]; the band stages, per output row, the two
// Y rows and the two UV rows (y/2) its taps use, and converts each tap (O0)
// before the resize (O11) -- identical to converting the whole frame first.
template <bool NV12>
__global__ void __launch_bounds__(kK4Threads)
k4_sample_kernel(const uint8_t* __restrict__ frames, int64_t n, int32_t H, int32_t W,
                 const int32_t* __restrict__ cuts, int32_t n_cuts, int32_t k, int32_t H2, int32_t W2,
                 int32_t rb, int32_t bands, int32_t slot_bytes, uint8_t* __restrict__ out,
                 int32_t* __restrict__ index) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ int32_t row_off[64];  // per staged row: offset of the row's first byte in its slot
  __shared__ LinCoeff ycs[32];     // y weights of the band's output rows
  LinCoeff* xc = reinterpret_cast<LinCoeff*>(sm);                    // [W2]
  uint8_t* rows = sm + ((sizeof(LinCoeff) * W2 + 127) & ~(size_t)127);  // [2*rb][slot_bytes]

  const int32_t j = blockIdx.x / bands, band = blockIdx.x - j * bands;
  const int32_t c = j / k, i = j - c * k;
  const int64_t s = c == 0 ? 0 : cuts[c - 1];
  const int64_t e = c == n_cuts ? n : cuts[c];
  int64_t t = s + ((2 * (int64_t)i + 1) * (e - s)) / (2 * (int64_t)k);  // O10
  t = t < 0 ? 0 : (t >= n ? n - 1 : t);
  if (band == 0 && threadIdx.x == 0 && index) index[j] = (int32_t)t;

  const int32_t r0 = band * rb, nr = min(rb, H2 - r0);
  constexpr int kRowsPerOut = NV12 ? 4 : 2;
  const int64_t row_bytes = NV12 ? (int64_t)W : 3 * (int64_t)W;
  const uint8_t* fb = frames + t * (NV12 ? 3 * (int64_t)H * W / 2 : (int64_t)H * row_bytes);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_first();
    for (int32_t q = 0; q < kRowsPerOut * nr; ++q) {
      const int32_t dy = q / kRowsPerOut, which = q % kRowsPerOut;
      const LinCoeff yc = lin_coeff(H, H2, r0 + dy);
      if (which == 0) ycs[dy] = yc;
      const int32_t sy = which & 1 ? yc.s1 : yc.s0;
      const uint8_t* row = which < 2 ? fb + (int64_t)sy * row_bytes                 // Y or RGB row
                                     : fb + (int64_t)H * W + (int64_t)(sy >> 1) * W;  // UV row
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(row) & ~(uintptr_t)15;
      const uintptr_t a1 = (reinterpret_cast<uintptr_t>(row) + row_bytes + 15) & ~(uintptr_t)15;
      CD_CHECK(q < 64 && a1 - a0 <= (uintptr_t)slot_bytes && (int64_t)(q + 1) * slot_bytes <= 2LL * rb * slot_bytes * (NV12 ? 2 : 1));
      CD_CHECK(a0 >= reinterpret_cast<uintptr_t>(frames) &&
               a1 <= reinterpret_cast<uintptr_t>(frames) + (uintptr_t)n * (NV12 ? 3 * (uint64_t)H * W / 2 : 3 * (uint64_t)H * W));
      row_off[q] = (int32_t)(reinterpret_cast<uintptr_t>(row) - a0);
      mbar_expect_tx(&bar, (uint32_t)(a1 - a0));
      bulk_g2s(rows + (int64_t)q * slot_bytes, reinterpret_cast<const uint8_t*>(a0),
               (uint32_t)(a1 - a0), &bar, pol);
    }
    mbar_arrive(&bar);
  }
  for (int32_t dx = threadIdx.x; dx < W2; dx += blockDim.x) xc[dx] = lin_coeff(W, W2, dx);
  __syncthreads();
  mbar_wait(&bar, 0);

  uint8_t* ob = out + ((int64_t)j * H2 + r0) * W2 * 3;
  for (int32_t p = threadIdx.x; p < nr * W2; p += blockDim.x) {
    const int32_t dy = p / W2, dx = p - dy * W2;
    const LinCoeff yc = ycs[dy];
    const LinCoeff x = xc[dx];
    const int32_t base = kRowsPerOut * dy;
    const uint8_t* q0 = rows + (int64_t)base * slot_bytes + row_off[base];
    const uint8_t* q1 = rows + (int64_t)(base + 1) * slot_bytes + row_off[base + 1];
    int32_t p00[3], p01[3], p10[3], p11[3];
    if constexpr (NV12) {
      const uint8_t* u0 = rows + (int64_t)(base + 2) * slot_bytes + row_off[base + 2];
      const uint8_t* u1 = rows + (int64_t)(base + 3) * slot_bytes + row_off[base + 3];
      nv12_px(q0, u0, x.s0, p00[0], p00[1], p00[2]);
      nv12_px(q0, u0, x.s1, p01[0], p01[1], p01[2]);
      nv12_px(q1, u1, x.s0, p10[0], p10[1], p10[2]);
      nv12_px(q1, u1, x.s1, p11[0], p11[1], p11[2]);
    } else {
      const int32_t o0 = 3 * x.s0, o1 = 3 * x.s1;
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        p00[ch] = q0[o0 + ch];
        p01[ch] = q0[o1 + ch];
        p10[ch] = q1[o0 + ch];
        p11[ch] = q1[o1 + ch];
      }
    }
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const int32_t h0 = p00[ch] * x.w0 + p01[ch] * x.w1;
      const int32_t h1 = p10[ch] * x.w0 + p11[ch] * x.w1;
      const int32_t v = ((((h0 >> 4) * yc.w0) >> 16) + (((h1 >> 4) * yc.w1) >> 16) + 2) >> 2;
      ob[(int64_t)p * 3 + ch] = (uint8_t)(v < 0 ? 0 : (v > 255 ? 255 : v));
    }
  }
}

}  // namespace

int k4_rows_per_band(int32_t W, bool nv12) {
  const int32_t slot = (((nv12 ? W : 3 * W) + 32) + 15) & ~15;
  int32_t rb = kK4SmemRows / ((nv12 ? 4 : 2) * slot);
  if (rb > (nv12 ? 16 : 32)) rb = nv12 ? 16 : 32;
  return rb < 1 ? 1 : rb;
}

int k4_max_width() { return kK4MaxW2; }

cudaError_t k4_sample_launch(const uint8_t* frames, int64_t n, int32_t H, int32_t W,
                             const int32_t* cuts, int32_t n_cuts, int32_t k, int32_t H2, int32_t W2,
                             uint8_t* out, int32_t* index, bool nv12, cudaStream_t stream) {
  const int32_t rb = k4_rows_per_band(W, nv12);
  const int32_t slot = (((nv12 ? W : 3 * W) + 32) + 15) & ~15;
  const int32_t bands = (H2 + rb - 1) / rb;
  const size_t smem = ((sizeof(LinCoeff) * W2 + 127) & ~(size_t)127) + (size_t)(nv12 ? 4 : 2) * rb * slot;
  auto kern = nv12 ? k4_sample_kernel<true> : k4_sample_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (int64_t)(n_cuts + 1) * k * bands;
  if (blocks <= 0) return cudaSuccess;
  if (blocks > 0x7FFFFFFF) return cudaErrorInvalidValue;
  kern<<<(unsigned)blocks, kK4Threads, smem, stream>>>(frames, n, H, W, cuts, n_cuts, k, H2, W2, rb,
                                                      bands, slot, out, index);
  return cudaGetLastError();
}

}  // namespace clipdetect
