// Host-side exhaustive check of the device bin code (paper_2503_12964_b200/csrc/binfn.cuh),
// compiled with g++ (the CUDA intrinsics are emulated on the host).  Writes
// 2^24-entry bin tables to the output file, which the pytest compares with the
// oracle's tables (test infrastructure):
//   e0, e1  K1's direct-offset codes (RGB hue table, (d ^ na) & 3 hash), lane 0 / lane 1
//   tg      bin_generic for the requested layout
//   m0, m1  K1-NV12: NV12 pair conversion + direct-offset codes (NV12 hash) of every (Y, U, V)
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>

#include "binfn.cuh"

using namespace clipdetect;

int main(int argc, char** argv) {
  if (argc < 5) {
    fprintf(stderr, "usage: %s out nh ns nv\n", argv[0]);
    return 2;
  }
  const uint32_t nh = atoi(argv[2]), ns = atoi(argv[3]), nv = atoi(argv[4]);
  const uint32_t N = 1u << 24;
  std::vector<uint8_t> e0(N), e1(N), tg(N), m0(N), m1(N);
  std::vector<uint8_t> lut_rgb(65536, 0), lut_nv(65536, 0);
  for (uint32_t d = 0; d < 256; ++d)
    for (uint32_t na = 0; na <= d; ++na) {
      lut_rgb[lut_index(na, d)] = (uint8_t)lut_entry_dir(na, d, kHashRgb);
      lut_nv[lut_index(na, d)] = (uint8_t)lut_entry_dir(na, d, kHashNv12);
    }
  // the kernels fill the table by unswizzling every byte: it must invert lut_index
  for (uint32_t d = 0; d < 256; ++d)
    for (uint32_t na = 0; na < 256; ++na)
      if (lut_unswizzle(lut_index(na, d) & 255u, d) != na || (lut_index(na, d) >> 8) != d) {
        fprintf(stderr, "lut_unswizzle mismatch\n");
        return 1;
      }
  for (uint32_t c = 0; c < N; ++c) {
    const uint32_t c2 = c ^ 0xA5A5A5u;
    const uint32_t R = (c >> 16) | ((c2 >> 16) << 16);
    const uint32_t G = ((c >> 8) & 255u) | (((c2 >> 8) & 255u) << 16);
    const uint32_t B = (c & 255u) | ((c2 & 255u) << 16);
    tg[c] = (uint8_t)bin_generic(c >> 16, (c >> 8) & 255u, c & 255u, nh, ns, nv);
    uint32_t i0, i1;
    const uint32_t dp = code_pair_dir_pre<true>(R, G, B, kMadK, i0, i1);
    const uint32_t o0 = dir_off_lo(dp, lut_rgb[i0]), o1 = dir_off_hi(dp, lut_rgb[i1]);
    if (o0 >= 4u * kDirCodes || o1 >= 4u * kDirCodes || (o0 & 3u) || (o1 & 3u)) {
      fprintf(stderr, "dir code offset out of range\n");
      return 1;
    }
    e0[c] = (uint8_t)code_to_bin_dir(o0 >> 2);
    e1[c2] = (uint8_t)code_to_bin_dir(o1 >> 2);
  }
  // unpack4 on pseudo-random bytes
  uint32_t x = 12345u;
  for (int it = 0; it < 100000; ++it) {
    uint8_t by[12];
    for (int i = 0; i < 12; ++i) {
      x = x * 1664525u + 1013904223u;
      by[i] = (uint8_t)(x >> 24);
    }
    uint32_t w[3];
    memcpy(w, by, 12);
    uint32_t R01, G01, B01, R23, G23, B23;
    unpack4(w[0], w[1], w[2], R01, G01, B01, R23, G23, B23);
    const uint32_t want[6] = {by[0] | (uint32_t)by[3] << 16, by[1] | (uint32_t)by[4] << 16,
                              by[2] | (uint32_t)by[5] << 16, by[6] | (uint32_t)by[9] << 16,
                              by[7] | (uint32_t)by[10] << 16, by[8] | (uint32_t)by[11] << 16};
    const uint32_t got[6] = {R01, G01, B01, R23, G23, B23};
    for (int i = 0; i < 6; ++i)
      if (got[i] != want[i]) {
        fprintf(stderr, "unpack4 mismatch %d: %08x vs %08x\n", i, got[i], want[i]);
        return 1;
      }
  }
  // NV12 pair conversion + codes for every (Y, U, V): lane 0 = Y, lane 1 = Y ^ 0x5A
  for (uint32_t c = 0; c < N; ++c) {
    const uint32_t Y = c >> 16, U = (c >> 8) & 255u, V = c & 255u, Y2 = Y ^ 0x5Au;
    int32_t ruv, guv, buv;
    nv12_chroma(U, V, ruv, guv, buv);
    uint32_t R, G, B;
    nv12_pair_rgb(Y, Y2, ruv, guv, buv, R, G, B);
    uint32_t i0, i1;
    const uint32_t dp = code_pair_dir_pre(R, G, B, kMadK, i0, i1);
    m0[c] = (uint8_t)code_to_bin_dir(dir_off_lo(dp, lut_nv[i0]) >> 2);
    m1[(Y2 << 16) | (U << 8) | V] = (uint8_t)code_to_bin_dir(dir_off_hi(dp, lut_nv[i1]) >> 2);
  }
  FILE* f = fopen(argv[1], "wb");
  fwrite(e0.data(), 1, N, f);
  fwrite(e1.data(), 1, N, f);
  fwrite(tg.data(), 1, N, f);
  fwrite(m0.data(), 1, N, f);
  fwrite(m1.data(), 1, N, f);
  fclose(f);
  return 0;
}
