/*
 * synth_dev.cu — device (CUDA) side of the seeded input generator (see
 * synth.h).  Built into synth/libsynthdev.so; used by bench.py and the GPU
 * tests to fill HBM with the same bytes the host generator produces (checked
 * by frame hashes).  Holds no method arithmetic.
 */
#include <cuda_runtime.h>
#include <stdint.h>

#include "synth.h"

namespace {

constexpr int kGenThreads = 256;
constexpr int kPxPerThread = 16;
constexpr int kBlockPx = kGenThreads * kPxPerThread;
constexpr int kMaxCells = 2048;  // texture cells one block's pixels can touch (else direct)

// 16 pixels of one thread, specialised on the frame's (uniform) mode and fade
// so that synth_finish_pixel's branches fold away.  k_of(i): palette index.
template <uint32_t MODE, bool FADE, typename KOf>
__device__ __forceinline__ void gen16(const uint32_t (*pal)[3], uint32_t key, uint32_t p0,
                                      uint32_t fade_w, KOf k_of, uint32_t* bytes) {
  uint8_t* b8 = reinterpret_cast<uint8_t*>(bytes);
#pragma unroll  // full: the 48 output bytes stay in registers
  for (int i = 0; i < kPxPerThread; ++i) {
    const uint32_t k = k_of(i);
    synth_finish_pixel(pal[k][0], pal[k][1], pal[k][2], synth_noise_word(key, p0 + i), MODE,
                       FADE ? fade_w : 256u, b8 + 3 * i);
  }
}

template <typename KOf>
__device__ __forceinline__ void gen16_any(const uint32_t (*pal)[3], uint32_t key, uint32_t p0,
                                          synth_frame fr, KOf k_of, uint32_t* bytes) {
  const bool fade = fr.fade_w != 256u;
  switch (fr.mode) {
    case SYNTH_MODE_NORMAL:
      if (fade) gen16<SYNTH_MODE_NORMAL, true>(pal, key, p0, fr.fade_w, k_of, bytes);
      else gen16<SYNTH_MODE_NORMAL, false>(pal, key, p0, fr.fade_w, k_of, bytes);
      break;
    case SYNTH_MODE_ROT1:
      gen16<SYNTH_MODE_ROT1, true>(pal, key, p0, fr.fade_w, k_of, bytes);
      break;
    case SYNTH_MODE_ROT2:
      gen16<SYNTH_MODE_ROT2, true>(pal, key, p0, fr.fade_w, k_of, bytes);
      break;
    case SYNTH_MODE_FLASH:
      gen16<SYNTH_MODE_FLASH, true>(pal, key, p0, fr.fade_w, k_of, bytes);
      break;
    default:
      gen16<SYNTH_MODE_NOISE, true>(pal, key, p0, fr.fade_w, k_of, bytes);
      break;
  }
}

// One CTA = kBlockPx consecutive pixels of one frame.  The texture-cell palette
// indices those pixels need (a 64-bit hash chain each) are computed once per
// cell by the whole CTA into shared memory; a thread's 16 pixels then need no
// division (16 < 2 * cell: at most two cell edges) and no warp-divergent hash
// chain.  Bytes identical to synth_pixel (the host generator; GPU test
// test_device_generator_matches_host).
__global__ void __launch_bounds__(kGenThreads)
gen_frames_kernel(uint64_t seed, uint32_t video, uint32_t W, uint32_t H, int64_t t0,
                  const synth_frame* __restrict__ frames, uint8_t* __restrict__ out) {
  __shared__ uint32_t pal[8][3];
  __shared__ uint8_t cellk[kMaxCells];
  __shared__ uint32_t u_key, u_cy0, u_ncx, u_ncell, u_x0, u_y0;  // CTA-uniform, computed once
  const int64_t f = blockIdx.y;
  const uint32_t t = (uint32_t)(t0 + f);
  const synth_frame fr = frames[t];
  const uint32_t npx = W * H;
  const uint32_t cell = synth_cell(W);
  const uint32_t b0 = blockIdx.x * kBlockPx;
  if (threadIdx.x == 0) {
    const uint32_t b1 = min(b0 + kBlockPx, npx) - 1;
    u_x0 = b0 % W;
    u_y0 = b0 / W;
    u_cy0 = u_y0 / cell;
    u_ncx = (W - 1) / cell + 1;
    u_ncell = ((b1 / W) / cell - u_cy0 + 1) * u_ncx;
  } else if (threadIdx.x == 32) {
    u_key = synth_noise_key(seed, video, t);
  } else if (threadIdx.x >= 64 && threadIdx.x < 64 + 24) {
    const uint32_t k = (threadIdx.x - 64) / 3, c = (threadIdx.x - 64) % 3;
    pal[k][c] = synth_palette(seed, video, fr.scene, k, c);
  }
  __syncthreads();
  const uint32_t cy0 = u_cy0, ncx = u_ncx, ncell = u_ncell, shift = t / 8u;
  const bool tab = ncell <= (uint32_t)kMaxCells;
  if (tab)
    for (uint32_t c = threadIdx.x; c < ncell; c += kGenThreads)
      cellk[c] = (uint8_t)synth_cell_index(seed, video, fr.scene, c % ncx + shift, cy0 + c / ncx);
  __syncthreads();
  const uint32_t p0 = b0 + threadIdx.x * kPxPerThread;
  if (p0 >= npx) return;  // npx is a multiple of 16
  const uint32_t key = u_key;
  uint32_t bytes[12];
  // (x, y) of p0 from the CTA's first pixel without a per-thread division
  uint32_t x = u_x0 + threadIdx.x * kPxPerThread, y = u_y0;
  if (W >= 256) {
    while (x >= W) {
      x -= W;
      ++y;
    }
  } else {
    y += x / W;
    x %= W;
  }
  const uint32_t cx = x / cell, rx = x - cx * cell, cy = y / cell;
  if (tab && x + kPxPerThread <= W) {
    // one row: pixel i is in cell cx + [rx + i >= cell] + [rx + i >= 2 cell]
    const uint8_t* row = cellk + (cy - cy0) * ncx + cx;
    const uint32_t e1 = cell - rx, e2 = 2 * cell - rx;
    gen16_any(pal, key, p0, fr,
              [&](int i) { return (uint32_t)row[((uint32_t)i >= e1) + ((uint32_t)i >= e2)]; },
              bytes);
  } else if (tab) {
    // the group wraps a row (W % 16 != 0)
    const uint32_t cyn = (y + 1) / cell;
    gen16_any(pal, key, p0, fr,
              [&](int i) {
                uint32_t xi = x + i, c = cy;
                if (xi >= W) {
                  xi -= W;
                  c = cyn;
                }
                return (uint32_t)cellk[(c - cy0) * ncx + xi / cell];
              },
              bytes);
  } else {
    // the cell table did not fit
    gen16_any(pal, key, p0, fr,
              [&](int i) {
                const uint32_t q = p0 + i, xi = q % W, yi = q / W;
                return synth_cell_index(seed, video, fr.scene, xi / cell + shift, yi / cell);
              },
              bytes);
  }
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)f * npx * 3 + (size_t)p0 * 3);
  dst[0] = make_uint4(bytes[0], bytes[1], bytes[2], bytes[3]);
  dst[1] = make_uint4(bytes[4], bytes[5], bytes[6], bytes[7]);
  dst[2] = make_uint4(bytes[8], bytes[9], bytes[10], bytes[11]);
}

__global__ void gen_emb_kernel(uint64_t seed, uint32_t video, int64_t t0, uint32_t D,
                               const synth_frame* __restrict__ frames, float* __restrict__ out) {
  const int64_t f = blockIdx.x;
  const uint32_t t = (uint32_t)(t0 + f);
  const uint32_t s = frames[t].scene;
  const uint32_t key = synth_emb_key(seed, video, t);
  for (uint32_t d = threadIdx.x; d < D; d += blockDim.x)
    out[(size_t)f * D + d] = synth_emb_value(synth_emb_dir(seed, video, s, d), key, d);
}

__global__ void frame_hash_kernel(const uint8_t* __restrict__ frames, int64_t bytes_per_frame,
                                  unsigned long long* __restrict__ out) {
  const int64_t f = blockIdx.y;
  const int64_t nw = bytes_per_frame / 8;
  const uint64_t* w = reinterpret_cast<const uint64_t*>(frames + f * bytes_per_frame);
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw;
       i += (int64_t)gridDim.x * blockDim.x)
    acc += synth_hash_word(w[i], (uint64_t)i);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out + f, acc);
}

// NV12: one thread per 2x2 block (4 luma + 1 chroma pair)
__global__ void gen_nv12_kernel(uint64_t seed, uint32_t video, uint32_t W, uint32_t H, int64_t t0,
                                const synth_frame* __restrict__ frames, uint8_t* __restrict__ out) {
  const int64_t f = blockIdx.y;
  const uint32_t t = (uint32_t)(t0 + f);
  const synth_frame fr = frames[t];
  const uint32_t nb = (W / 2) * (H / 2);
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint32_t bx = b % (W / 2), by = b / (W / 2);
  uint8_t* Y = out + (size_t)f * W * H * 3 / 2;
  uint8_t* UV = Y + (size_t)W * H;
  for (uint32_t dy = 0; dy < 2; ++dy)
    for (uint32_t dx = 0; dx < 2; ++dx) {
      const uint32_t x = 2 * bx + dx, y = 2 * by + dy;
      Y[(size_t)y * W + x] = (uint8_t)synth_nv12_y(seed, video, t, fr, W, x, y);
    }
  uint32_t u, v;
  synth_nv12_uv(seed, video, t, fr, W, bx, by, &u, &v);
  UV[(size_t)by * W + 2 * bx] = (uint8_t)u;
  UV[(size_t)by * W + 2 * bx + 1] = (uint8_t)v;
}

}  // namespace

extern "C" {

/* NV12 frames t0..t0+n-1 of one video into d_out ([n][H*W*3/2] u8, device). */
int synth_dev_gen_nv12(uint64_t seed, uint32_t video, uint32_t W, uint32_t H, int64_t t0,
                       int64_t n, const synth_frame* d_frames, uint8_t* d_out, uintptr_t stream) {
  if (n <= 0) return 0;
  if ((W % 2) || (H % 2)) return (int)cudaErrorInvalidValue;
  const uint32_t nb = (W / 2) * (H / 2);
  for (int64_t f0 = 0; f0 < n; f0 += 65535) {
    int64_t nf = n - f0 < 65535 ? n - f0 : 65535;
    dim3 grid((nb + 255) / 256, (unsigned)nf);
    gen_nv12_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(seed, video, W, H, t0 + f0, d_frames,
                                                            d_out + (size_t)f0 * W * H * 3 / 2);
  }
  return (int)cudaGetLastError();
}


/* Frames t0..t0+n-1 of one video into d_out ([n][H][W][3] u8, device).
 * d_frames: device array of synth_frame indexed by absolute frame index.
 * Returns a cudaError_t value (0 = success). */
int synth_dev_gen_frames(uint64_t seed, uint32_t video, uint32_t W, uint32_t H, int64_t t0,
                         int64_t n, const synth_frame* d_frames, uint8_t* d_out,
                         uintptr_t stream) {
  if (n <= 0) return 0;
  if ((W * H) % 16 != 0) return (int)cudaErrorInvalidValue;
  const uint32_t npx = W * H;
  for (int64_t f0 = 0; f0 < n; f0 += 65535) {
    int64_t nf = n - f0 < 65535 ? n - f0 : 65535;
    dim3 grid((npx + kBlockPx - 1) / kBlockPx, (unsigned)nf);
    gen_frames_kernel<<<grid, kGenThreads, 0, (cudaStream_t)stream>>>(
        seed, video, W, H, t0 + f0, d_frames, d_out + (size_t)f0 * W * H * 3);
  }
  return (int)cudaGetLastError();
}

/* Embeddings of frames t0..t0+n-1 into d_out ([n][D] f32, device). */
int synth_dev_gen_emb(uint64_t seed, uint32_t video, int64_t t0, int64_t n, uint32_t D,
                      const synth_frame* d_frames, float* d_out, uintptr_t stream) {
  if (n <= 0) return 0;
  gen_emb_kernel<<<(unsigned)n, 256, 0, (cudaStream_t)stream>>>(seed, video, t0, D, d_frames,
                                                                 d_out);
  return (int)cudaGetLastError();
}

/* Frame hashes (synth.h definition) of n frames; d_out [n] u64 is zeroed here. */
int synth_dev_frame_hash(const uint8_t* d_frames, int64_t n, int64_t bytes_per_frame,
                         uint64_t* d_out, uintptr_t stream) {
  if (n <= 0) return 0;
  cudaMemsetAsync(d_out, 0, sizeof(uint64_t) * n, (cudaStream_t)stream);
  for (int64_t f0 = 0; f0 < n; f0 += 65535) {
    int64_t nf = n - f0 < 65535 ? n - f0 : 65535;
    dim3 grid(16, (unsigned)nf);
    frame_hash_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        d_frames + f0 * bytes_per_frame, bytes_per_frame,
        reinterpret_cast<unsigned long long*>(d_out + f0));
  }
  return (int)cudaGetLastError();
}

}  // extern "C"
