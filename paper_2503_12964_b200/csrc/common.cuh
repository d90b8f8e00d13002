// common.cuh — shared device helpers and launch descriptors of libclipdetect.
// (Product path only; nothing here is shared with oracle/.)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

namespace clipdetect {

constexpr int kSMs = 148;

// Checked build (-DCLIPDETECT_CHECKED, tools/sanitize_run.py --checked: the
// pool's compute-sanitizer is closed): CD_CHECK(c) bounds-checks a shared- or
// global-memory access, a ring hand-off or an index, prints the failing
// condition and traps (the call then fails with CLIP_E_CUDA).  The product
// build compiles every check away.
#ifdef CLIPDETECT_CHECKED
#define CD_CHECK(c)                                                                           \
  do {                                                                                        \
    if (!(c)) {                                                                               \
      printf("CD_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,            \
             (int)blockIdx.x, (int)threadIdx.x, #c);                                          \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define CD_CHECK(c) \
  do {              \
  } while (0)
#endif

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Byte load from a 32-bit shared-window address (uniform base + per-thread
// offset: lets ptxas fold the base into the LDS's uniform-register operand).
__device__ __forceinline__ uint32_t lds_u8(uint32_t saddr) {
  uint32_t v;
  asm("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(saddr));
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// The same wait with a back-off, for the producer lanes: spinning there steals
// issue slots from the consumer warps of its scheduler, which then release ring
// slots last for the whole CTA (B200 A/B with the L2 prefetch below: K1 +2.5 %,
// profiles/r02/ab/).
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
               : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  while (!done) {
    __nanosleep(256);
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}

// 1-D TMA bulk copy global -> shared, completion counted on an mbarrier.
// bytes and both addresses must be multiples of 16.  L2 evict-first: frame
// bytes are read exactly once.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gsrc, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// L2 prefetch of a global range (TMA bulk prefetch; no shared memory, no
// barrier): lets a producer run further ahead than its ring is deep.
__device__ __forceinline__ void bulk_prefetch_l2(const void* gsrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(gsrc), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- descriptors
// One "segment" = the frames of one video (or one chunk of one video) that a
// single K1 launch scans.  Frames are u8 [n][H][W][3] contiguous, H*W % 16 == 0.
struct HistSeg {
  const uint8_t* frames;  // device
  uint32_t* hist;         // device, [n][nbins] for this segment's frame 0
  int64_t n_frames;
  int64_t groups;        // 16-pixel groups per frame = H*W/16
  int64_t stages;        // stages per frame = ceil(groups / kStageGroups)
  int64_t stage_base;    // prefix of n_frames*stages over earlier segments
};

// NV12 segment (NEXT f1): frames u8 [n][H*3/2][W] (Y rows, then H/2 rows of
// interleaved UV), H and W even.  A stage = `rows` chroma-block rows of one
// frame (2*rows Y rows + rows UV rows).
struct Nv12Seg {
  const uint8_t* frames;  // device
  uint32_t* hist;         // device, [n][nbins]
  int64_t n_frames;
  int32_t height, width;
  int32_t rows;           // block rows per stage (fast kernel; 0 for the generic one)
  int32_t stages;         // stages per frame = ceil((H/2) / rows)
  int64_t stage_base;     // prefix of n_frames*stages over earlier segments
};

}  // namespace clipdetect
