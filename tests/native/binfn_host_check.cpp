// Host-side exhaustive check of the device bin code (paper_2503_12964_b200/csrc/binfn.cuh),
// compiled with g++ (the CUDA intrinsics are emulated on the host).  Writes the
// 2^24-entry bin tables of lane 0 and lane 1 of code_pair(), and of
// bin_generic() for the requested layout, to the output file; the pytest
// compares them with the oracle's table.  (Test infrastructure.)
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
  std::vector<uint8_t> t0(N), t1(N), tg(N), l0(N), l1(N), e0(N), e1(N);
  std::vector<uint8_t> lut(65536, 0);
  for (uint32_t d = 0; d < 256; ++d)
    for (uint32_t na = 0; na <= d; ++na) lut[lut_index(na, d, 1)] = (uint8_t)lut_entry(na, d);  // K1 cfg14
  std::vector<uint8_t> lut2(65536, 0);  // swizzle 3 (the NV12 kernel's table)
  std::vector<uint8_t> lut3(65536, 0);  // swizzle 3, direct-offset entries, d & 3 bank hash
  std::vector<uint8_t> lut4(65536, 0);  // swizzle multiplier 5, ((d >> 5) ^ na) & 3 bank hash
  for (uint32_t d = 0; d < 256; ++d)
    for (uint32_t na = 0; na <= d; ++na) {
      lut2[lut_index(na, d, 3)] = (uint8_t)lut_entry(na, d);
      lut3[lut_index(na, d, 3)] = (uint8_t)lut_entry_dir(na, d, 1);
      lut4[lut_index_k(na, d, 5)] = (uint8_t)lut_entry_dir(na, d, 4);
    }
  // the unswizzle used by the kernels' table initialisation inverts every swizzle
  for (int swz = 0; swz <= 3; ++swz)
    for (uint32_t d = 0; d < 256; ++d)
      for (uint32_t na = 0; na < 256; ++na)
        if (lut_unswizzle(lut_index(na, d, swz) & 255u, d, swz) != na) {
          fprintf(stderr, "lut_unswizzle mismatch swz %d\n", swz);
          return 1;
        }
  for (uint32_t c = 0; c < N; ++c) {
    const uint32_t c2 = c ^ 0xA5A5A5u;
    const uint32_t R = (c >> 16) | ((c2 >> 16) << 16);
    const uint32_t G = ((c >> 8) & 255u) | (((c2 >> 8) & 255u) << 16);
    const uint32_t B = (c & 255u) | ((c2 & 255u) << 16);
    const uint32_t code = code_pair(R, G, B);
    t0[c] = (uint8_t)code_to_bin(code_off_lo(code, kMadK) >> 2);
    t1[c2] = (uint8_t)code_to_bin(code_off_hi(code, kMadK) >> 2);
    tg[c] = (uint8_t)bin_generic(c >> 16, (c >> 8) & 255u, c & 255u, nh, ns, nv);
    uint32_t i0, i1;
    const uint32_t pre = code_pair_lut_pre<1>(R, G, B, kMadK, i0, i1);
    const uint32_t lc = code_pair_lut_post(pre, lut[i0], lut[i1], kMadK);
    l0[c] = (uint8_t)code_to_bin_lut(lut_off_lo(lc, kMadK) >> 2);
    l1[c2] = (uint8_t)code_to_bin_lut(lut_off_hi(lc, kMadK) >> 2);
    if (lut_off_lo(lc, kMadK) >= 4u * kLutCodes || lut_off_hi(lc, kMadK) >= 4u * kLutCodes) {
      fprintf(stderr, "lut code offset out of range\n");
      return 1;
    }
    // direct-offset codes: both B forms, offsets in range and multiples of 4
    const uint32_t dp = code_pair_dir_pre<0>(R, G, B, kMadK, i0, i1);
    // XU: a per-pixel offset 256 X in the high byte of every lane, taken back via kz / km
    const uint32_t off = (((c * 7u) & 255u) << 8) | (((c * 13u + 5u) & 255u) << 24);
    uint32_t x0, x1;
    const uint32_t dpx = code_pair_dir_pre<0, 4, 1>(R + off, G + off, B + off, kMadK, x0, x1,
                                                    off + 0x04000400u, off * 0xFFFFFFFDu);
    if (dpx != dp || x0 != i0 || x1 != i1) {
      fprintf(stderr, "dir pre XU mismatch\n");
      return 1;
    }
    if (code_pair_dir_pre<1>(R, G, B, kMadK, i0, i1) != dp ||
        code_pair_dir_pre<2>(R, G, B, kMadK, i0, i1) != dp) {
      fprintf(stderr, "dir pre TBF mismatch\n");
      return 1;
    }
    // odd colours: swizzle multiplier 5 and another bank hash (the bin must not depend on either)
    uint32_t k0 = i0, k1 = i1;
    const uint32_t dp5 = code_pair_dir_pre<0, 5>(R, G, B, kMadK, k0, k1);
    const bool odd = c & 1u;
    const uint32_t o0 = odd ? dir_off_lo(dp5, lut4[k0]) : dir_off_lo(dp, lut3[i0]);
    const uint32_t o1 = odd ? dir_off_hi(dp5, lut4[k1]) : dir_off_hi(dp, lut3[i1]);
    if (o0 >= 4u * kDirCodes || o1 >= 4u * kDirCodes || (o0 & 3u) || (o1 & 3u)) {
      fprintf(stderr, "dir code offset out of range\n");
      return 1;
    }
    e0[c] = (uint8_t)code_to_bin_dir(o0 >> 2);
    e1[c2] = (uint8_t)code_to_bin_dir(o1 >> 2);
  }
  // unpack4 / unpack4x on pseudo-random bytes
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
    uint32_t X[6], off;
    unpack4x(w[0], w[1], w[2], X[0], X[1], X[2], X[3], X[4], X[5], off);
    const uint32_t xo = ((uint32_t)by[4] << 8) | ((uint32_t)by[5] << 24);  // 256 X: X0 = w1.b0, X1 = w1.b1
    if (off != xo) {
      fprintf(stderr, "unpack4x offset mismatch\n");
      return 1;
    }
    for (int i = 0; i < 6; ++i)
      if (X[i] != want[i] + xo) {
        fprintf(stderr, "unpack4x mismatch %d: %08x vs %08x\n", i, X[i], want[i] + xo);
        return 1;
      }
  }
  // NV12 pair conversion + LUT codes for every (Y, U, V): lane 0 = Y, lane 1 = Y ^ 0x5A
  std::vector<uint8_t> n0(N), n1(N), m0(N), m1(N);
  for (uint32_t c = 0; c < N; ++c) {
    const uint32_t Y = c >> 16, U = (c >> 8) & 255u, V = c & 255u, Y2 = Y ^ 0x5Au;
    int32_t ruv, guv, buv;
    nv12_chroma(U, V, ruv, guv, buv);
    uint32_t R, G, B;
    nv12_pair_rgb(Y, Y2, ruv, guv, buv, R, G, B);
    uint32_t i0, i1;
    const uint32_t pre = code_pair_lut_pre<3>(R, G, B, kMadK, i0, i1);
    const uint32_t lc = code_pair_lut_post(pre, lut2[i0], lut2[i1], kMadK);
    n0[c] = (uint8_t)code_to_bin_lut(lut_off_lo(lc, kMadK) >> 2);
    n1[(Y2 << 16) | (U << 8) | V] = (uint8_t)code_to_bin_lut(lut_off_hi(lc, kMadK) >> 2);
    const uint32_t dp = code_pair_dir_pre<0>(R, G, B, kMadK, i0, i1);  // direct-offset codes
    m0[c] = (uint8_t)code_to_bin_dir(dir_off_lo(dp, lut3[i0]) >> 2);
    m1[(Y2 << 16) | (U << 8) | V] = (uint8_t)code_to_bin_dir(dir_off_hi(dp, lut3[i1]) >> 2);
  }
  FILE* f = fopen(argv[1], "wb");
  fwrite(t0.data(), 1, N, f);
  fwrite(t1.data(), 1, N, f);
  fwrite(tg.data(), 1, N, f);
  fwrite(l0.data(), 1, N, f);
  fwrite(l1.data(), 1, N, f);
  fwrite(n0.data(), 1, N, f);
  fwrite(n1.data(), 1, N, f);
  fwrite(e0.data(), 1, N, f);
  fwrite(e1.data(), 1, N, f);
  fwrite(m0.data(), 1, N, f);
  fwrite(m1.data(), 1, N, f);
  fclose(f);
  return 0;
}
