// hist.cu — K1: fused RGB24 -> HSV bin -> per-frame histogram (rows a1-a3).
//
// hist_t[b] = #{pixels of frame t with bin b} (reading O2; §2.1).
//
// B200 design:
//  * persistent grid, 2 CTAs/SM; each CTA owns a CONTIGUOUS range of "stages"
//    of the flattened (segment, frame, stage) space, so a CTA flushes its
//    histogram only when its frame changes;
//  * one producer lane streams each stage (<= kStageGroups x 48 B of one
//    frame) HBM -> shared memory with a 1-D TMA bulk copy
//    (cp.async.bulk ... mbarrier::complete_tx, L2 evict_first) into a
//    kStages-deep ring; consumers signal "empty" per warp;
//  * 8 consumer warps; each thread takes 48-byte groups (16 pixels, three
//    conflict-free LDS.128) and bins them with the division-free sector
//    form (binfn.cuh) into a warp-private shared histogram
//    (atomicAdd(+1) -> ATOMS.POPC.INC, same-bin lanes combined in hardware);
//  * at a frame change the 8 warp histograms are summed and added to the
//    global u32 histogram (integer adds: order-free, bit-deterministic).
#include "binfn.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace clipdetect {

namespace {

constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;  // + producer warp
constexpr int kGroupsPerThread = 2;
constexpr int kStageGroups = kConsumers * kGroupsPerThread;  // 512 groups = 24 KiB
constexpr int kStageBytes = kStageGroups * 48;
constexpr int kStages = 4;
constexpr int kHistStride = 256;

struct K1Smem {
  alignas(128) uint8_t buf[kStages][kStageBytes];
  uint32_t whist[kConsumerWarps][kHistStride];
  uint64_t full[kStages];
  uint64_t empty[kStages];
};

struct StageIter {
  const HistSeg* segs;
  int32_t seg;
  int64_t frame, st;
  __device__ void seek(const HistSeg* s, int32_t nseg, int64_t g) {
    segs = s;
    int32_t lo = 0, hi = nseg - 1;
    while (lo < hi) {  // last segment with stage_base <= g
      int32_t m = (lo + hi + 1) >> 1;
      if (s[m].stage_base <= g) lo = m; else hi = m - 1;
    }
    seg = lo;
    int64_t rel = g - s[lo].stage_base;
    frame = rel / s[lo].stages;
    st = rel - frame * s[lo].stages;
  }
  __device__ void next() {
    if (++st == segs[seg].stages) {
      st = 0;
      if (++frame == segs[seg].n_frames) {
        frame = 0;
        ++seg;
      }
    }
  }
};

template <int MODE>
__device__ __forceinline__ void bin_group(const uint8_t* src, uint32_t* wh, uint32_t nh,
                                          uint32_t ns, uint32_t nv, uint32_t& xacc) {
  const uint4* p = reinterpret_cast<const uint4*>(src);
  const uint4 a = p[0], b = p[1], c = p[2];
  const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
  if (MODE == kModeRead) {
#pragma unroll
    for (int i = 0; i < 12; ++i) xacc ^= w[i];
    return;
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int o = 3 * i;
    const uint32_t r = __byte_perm(w[o >> 2], 0u, 0x4440u | (o & 3));
    const uint32_t g = __byte_perm(w[(o + 1) >> 2], 0u, 0x4440u | ((o + 1) & 3));
    const uint32_t bb = __byte_perm(w[(o + 2) >> 2], 0u, 0x4440u | ((o + 2) & 3));
    uint32_t bin;
    if (MODE == kModeFast)
      bin = bin_18_3_3(r, g, bb);
    else
      bin = bin_generic(r, g, bb, nh, ns, nv);
    atomicAdd(&wh[bin], 1u);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2)
k1_hist_kernel(const HistSeg* __restrict__ segs, int32_t nseg, int64_t total_stages,
               uint32_t nh, uint32_t ns, uint32_t nv, uint32_t* __restrict__ sink) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  K1Smem& sm = *reinterpret_cast<K1Smem*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const uint32_t nbins = nh * ns * nv;

  const int64_t s_begin = total_stages * blockIdx.x / gridDim.x;
  const int64_t s_end = total_stages * (blockIdx.x + 1) / gridDim.x;

  for (int i = tid; i < kConsumerWarps * kHistStride; i += kThreads)
    (&sm.whist[0][0])[i] = 0u;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (s_begin >= s_end) return;

  if (warp == kConsumerWarps) {
    // ---------------------------------------------------------- producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      StageIter it;
      it.seek(segs, nseg, s_begin);
      uint32_t i = 0;
      for (int64_t s = s_begin; s < s_end; ++s, ++i) {
        const uint32_t slot = i % kStages, par = (i / kStages) & 1u;
        if (i >= kStages) mbar_wait(&sm.empty[slot], par ^ 1u);
        const HistSeg& sg = segs[it.seg];
        const int64_t g0 = it.st * kStageGroups;
        const int64_t ng = min((int64_t)kStageGroups, sg.groups - g0);
        const uint32_t bytes = (uint32_t)(ng * 48);
        const uint8_t* src = sg.frames + (it.frame * sg.groups + g0) * 48;
        mbar_arrive_expect_tx(&sm.full[slot], bytes);
        bulk_g2s(sm.buf[slot], src, bytes, &sm.full[slot], pol);
        it.next();
      }
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  uint32_t* wh = sm.whist[warp];
  uint32_t xacc = 0;
  StageIter it;
  it.seek(segs, nseg, s_begin);
  uint32_t i = 0;
  for (int64_t s = s_begin; s < s_end; ++s, ++i) {
    const uint32_t slot = i % kStages, par = (i / kStages) & 1u;
    const HistSeg& sg = segs[it.seg];
    const int64_t g0 = it.st * kStageGroups;
    const int ng = (int)min((int64_t)kStageGroups, sg.groups - g0);
    mbar_wait(&sm.full[slot], par);
    const uint8_t* buf = sm.buf[slot];
#pragma unroll
    for (int j = 0; j < kGroupsPerThread; ++j) {
      const int gi = tid + j * kConsumers;
      if (gi < ng) bin_group<MODE>(buf + gi * 48, wh, nh, ns, nv, xacc);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[slot]);

    const int32_t seg_now = it.seg;
    const int64_t frame_now = it.frame;
    it.next();
    const bool last = (s + 1 == s_end);
    if (MODE != kModeRead && (last || it.frame != frame_now || it.seg != seg_now)) {
      // flush the frame's partial histogram
      named_bar_sync(1, kConsumers);
      uint32_t* gh = segs[seg_now].hist + frame_now * nbins;
      for (uint32_t bn = tid; bn < nbins; bn += kConsumers) {
        uint32_t sum = 0;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
          sum += sm.whist[w][bn];
          sm.whist[w][bn] = 0u;
        }
        if (sum) atomicAdd(gh + bn, sum);
      }
      named_bar_sync(1, kConsumers);
    }
  }
  if (MODE == kModeRead && xacc == 0x9E3779B9u) sink[0] = xacc;  // keep the loads alive
}

}  // namespace

size_t k1_smem_bytes() { return sizeof(K1Smem); }
int k1_stage_groups() { return kStageGroups; }

cudaError_t k1_configure() {
  const int bytes = (int)sizeof(K1Smem);
  cudaError_t e;
  e = cudaFuncSetAttribute(k1_hist_kernel<kModeFast>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k1_hist_kernel<kModeGeneric>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k1_hist_kernel<kModeRead>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int k1_grid(int sm_count, int64_t total_stages) {
  int64_t g = (int64_t)sm_count * 2;
  if (total_stages < g) g = total_stages;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t k1_launch(int mode, const HistSeg* d_segs, int32_t nseg, int64_t total_stages,
                      uint32_t nh, uint32_t ns, uint32_t nv, uint32_t* sink, int grid,
                      cudaStream_t stream) {
  if (total_stages <= 0) return cudaSuccess;
  const size_t bytes = sizeof(K1Smem);
  if (mode == kModeFast)
    k1_hist_kernel<kModeFast><<<grid, kThreads, bytes, stream>>>(d_segs, nseg, total_stages, nh, ns, nv, sink);
  else if (mode == kModeGeneric)
    k1_hist_kernel<kModeGeneric><<<grid, kThreads, bytes, stream>>>(d_segs, nseg, total_stages, nh, ns, nv, sink);
  else
    k1_hist_kernel<kModeRead><<<grid, kThreads, bytes, stream>>>(d_segs, nseg, total_stages, nh, ns, nv, sink);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K5 (test)
namespace {
__global__ void k5_binmap_kernel(uint8_t* __restrict__ out, uint32_t nh, uint32_t ns, uint32_t nv,
                                 int fast) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (1u << 24)) return;
  const uint32_t r = c >> 16, g = (c >> 8) & 255u, b = c & 255u;
  out[c] = (uint8_t)(fast ? bin_18_3_3(r, g, b) : bin_generic(r, g, b, nh, ns, nv));
}
}  // namespace

cudaError_t k5_binmap_launch(uint8_t* out, uint32_t nh, uint32_t ns, uint32_t nv, int fast,
                             cudaStream_t stream) {
  k5_binmap_kernel<<<(1u << 24) / 256, 256, 0, stream>>>(out, nh, ns, nv, fast);
  return cudaGetLastError();
}

}  // namespace clipdetect
