// binfn.cuh — pixel -> joint HSV bin on the device (rows a1-a2 of the hot path).
//
// Reading O1 (§2.1 "analyzing the color
// changes between frames"): exact integer hexcone HSV with floor bins,
//   bin = (h*ns + s)*nv + v,  h = floor(nh*H/360deg), s = min(ns-1, floor(ns*S)),
//   v = floor(nv*max/256).
// The device evaluates it WITHOUT division via the sector form: order the
// channels, sector k in 0..5 (60 degrees each), in-sector numerator
//   num = mid - min (k even, hue rising)   or   max - mid (k odd, falling),
// so that the exact hue numerator is num6 = k*d + num over 6d (d = max - min),
// and for nh = 18: h = 3k + floor(3*num/d).
//
// Hot path (18, 3, 3): TWO pixels per 32-bit register (u16x2 lanes).  Every
// threshold test a >= b is bit j of (a - b + 2^j) in its lane (no lane
// borrows: |a - b| < 2^j <= 2^15).  The in-sector hue offsets come from a
// 64 KiB shared-memory table indexed by (d, na = mid - min), and each lane's
// code IS the byte offset of its entry in an 8192-entry code histogram (the
// "direct-offset" layout below); codes are mapped to the 162 bins only when a
// frame is flushed.  Verified bit-exact against the oracle on all 2^24
// colours in both lanes (tests/test_binfn_host.py on the CPU, K5 on the GPU).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define CD_HD __host__ __device__ __forceinline__
#else
#define CD_HD static inline
#endif

namespace clipdetect {

// 3k for the 8 ordering codes idx = [r>=g]*4 + [g>=b]*2 + [r>=b]
// (codes 1 and 6 are infeasible):  idx 0 -> k=3, 2 -> k=2, 3 -> k=1, 4 -> k=4,
// 5 -> k=5, 7 -> k=0.  One nibble per code.
constexpr uint32_t kSector3k = (9u << 0) | (0u << 4) | (6u << 8) | (3u << 12) | (12u << 16) |
                               (15u << 20) | (0u << 24) | (0u << 28);

// ------------------------------------------------------------ SIMD primitives
CD_HD uint32_t cd_prmt(uint32_t a, uint32_t b, uint32_t sel) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
#else
  const uint64_t x = ((uint64_t)b << 32) | a;
  uint32_t r = 0;
  for (int i = 0; i < 4; ++i) {
    const uint32_t s = (sel >> (4 * i)) & 15u;
    uint32_t byte = (uint32_t)(x >> (8 * (s & 7u))) & 0xFFu;
    if (s & 8u) byte = (byte & 0x80u) ? 0xFFu : 0u;
    r |= byte << (8 * i);
  }
  return r;
#endif
}

CD_HD uint32_t cd_max3_u16x2(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  return __vimax3_u16x2(a, b, c);
#else
  uint32_t r = 0;
  for (int i = 0; i < 2; ++i) {
    uint32_t x = (a >> (16 * i)) & 0xFFFFu, y = (b >> (16 * i)) & 0xFFFFu, z = (c >> (16 * i)) & 0xFFFFu;
    uint32_t m = x > y ? x : y;
    m = m > z ? m : z;
    r |= m << (16 * i);
  }
  return r;
#endif
}

CD_HD uint32_t cd_min3_u16x2(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  return __vimin3_u16x2(a, b, c);
#else
  uint32_t r = 0;
  for (int i = 0; i < 2; ++i) {
    uint32_t x = (a >> (16 * i)) & 0xFFFFu, y = (b >> (16 * i)) & 0xFFFFu, z = (c >> (16 * i)) & 0xFFFFu;
    uint32_t m = x < y ? x : y;
    m = m < z ? m : z;
    r |= m << (16 * i);
  }
  return r;
#endif
}

// Runtime multiplier constants.  Passed in as kernel arguments (and read back
// through shared memory) so that ptxas cannot fold them and must issue IMAD:
// that arithmetic then runs on the FMA pipe and leaves the ALU pipe
// (LOP3/PRMT/VIMNMX/IADD3, the binding pipe on sm_100: DESIGN.md §7) to the
// bit work.
struct MadK {
  uint32_t one, neg1, three, neg6;
};
constexpr MadK kMadK{1u, 0xFFFFFFFFu, 3u, 0xFFFFFFFAu};

CD_HD uint32_t cd_mad(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
#else
  return a * b + c;
#endif
}

// bit select (a where m, else b) as ONE LOP3: written as inline PTX so that the
// compiler does not flatten a chain of selects into and-or terms (one more op)
template <uint32_t M>
CD_HD uint32_t cd_sel(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "n"(M));
  return r;
#else
  return (a & M) | (b & ~M);
#endif
}

// a ^ b ^ c as ONE LOP3
CD_HD uint32_t cd_xor3(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
#else
  return a ^ b ^ c;
#endif
}

// ------------------------------------------------------------ hue table
// lut_entry: qr | qf << 2 with qr = floor(3 na / d) (rising sectors) and
// qf = floor(3 (d - na) / d) (falling), both clamped to 3; 0 for grey (d = 0).
CD_HD uint32_t lut_entry(uint32_t na, uint32_t d) {
  if (d == 0) return 0u;
  const uint32_t qr = (3u * na) / d, qf = (3u * (d - na)) / d;
  return (qr > 3u ? 3u : qr) | ((qf > 3u ? 3u : qf) << 2);
}

// Table row d holds na at byte (na + 4d) mod 256: rows d and d + 1 of the same
// na land in different banks (the swizzle keeps warps on smooth content, where
// (d, na) jitter by +-1, nearly conflict-free), and the index comes straight
// from the channel sum (code_pair_dir_pre).
CD_HD uint32_t lut_index(uint32_t na, uint32_t d) { return d * 256u + ((na + 4u * d) & 255u); }
CD_HD uint32_t lut_unswizzle(uint32_t b, uint32_t d) { return (b - 4u * d) & 255u; }

// ------------------------------------------------------------ direct-offset codes
// Each lane's code IS the byte offset of its code-histogram entry, so nothing
// runs between the table lookup and the shared-memory atomic but one PRMT:
//   offset = byte1 << 8 | byte0,
//   byte0 = the table entry: q3 << 2 | hash << 5  (bits 0-1 zero),
//   byte1 = v (bits 8-9) and, in bits 10-14, an invertible XOR mix of
//           s1, s2, A = [r>=g], B = [g>=b], C = [r>=b] (code_pair_dir_pre),
//           bit 15 zero                         -> offsets < 0x8000: 8192 entries.
// q3 in [0, 8) is the compact index of the table's (qr, qf) pair (kDirQ below);
// hash (2 bits, a function of (d, na) that the bin ignores) only spreads the
// entries over the 32 shared-memory banks: the bank of an entry is offset bits
// 2-6 = (q3, hash), all from byte 0.  Without it a warp's atomics on noisy
// content would share 8 banks.
constexpr int kDirCodes = 8192;
// (qr, qf) of q3 = 0..7: grey, then na/d = 0, (0,1/3), 1/3, (1/3,2/3), 2/3, (2/3,1), 1
constexpr uint32_t kDirQ = (0u << 0) | (12u << 4) | (8u << 8) | (9u << 12) | (5u << 16) |
                           (6u << 20) | (2u << 24) | (3u << 28);  // nibble = qr | qf << 2
CD_HD uint32_t dir_q3(uint32_t q) {  // (qr | qf << 2) -> q3
  for (uint32_t i = 0; i < 8; ++i)
    if (((kDirQ >> (4 * i)) & 15u) == q) return i;
  return 0u;
}
// Bank hashes (tools/atoms_bank_sim.py): K1 (RGB24) uses (d ^ na) & 3, K1-NV12
// ((d >> 5) ^ na) & 3 — on decoded NV12 the luma noise moves r, g, b
// together, so d is nearly constant within a palette cell.
enum { kHashRgb = 0, kHashNv12 = 1 };
CD_HD uint32_t lut_entry_dir(uint32_t na, uint32_t d, int hash) {
  const uint32_t h = hash == kHashNv12 ? ((d >> 5) ^ na) : (d ^ na);
  return (dir_q3(lut_entry(na, d)) << 2) | ((h & 3u) << 5);
}

// Part 1: byte 1 of both lanes' offsets (in bytes 1 and 3 of the result) and
// the two table indices.  The table index is (na + 4d) mod 256 of row d,
// computed straight from the channel sum: na + 4d = (r + g + b) + 3 max - 6 min
// (mid = sum - max - min).  The byte-1 fields are threshold bits (a - b + 2^j)
// in u16x2 lanes (no lane borrows), merged as below.
// SUM_ALU: r + g + b by one IADD3 (ALU pipe) instead of two IMADs (FMA pipe):
// one issue slot less, one ALU instruction more — K1 gains (+3.1 %, its ALU pipe
// has room), K1-NV12 loses (−1.0 %, its conversion already loads the ALU pipe).
template <bool SUM_ALU = false>
CD_HD uint32_t code_pair_dir_pre(uint32_t R, uint32_t G, uint32_t B, MadK k, uint32_t& i0,
                                 uint32_t& i1) {
  const uint32_t mx = cd_max3_u16x2(R, G, B);
  const uint32_t mn = cd_min3_u16x2(R, G, B);
  const uint32_t d = cd_mad(mn, k.neg1, mx);
  const uint32_t t = SUM_ALU ? cd_mad(mx, k.three, R + G + B)
                             : cd_mad(B, k.one, cd_mad(G, k.one, cd_mad(mx, k.three, R)));
  const uint32_t nas = cd_mad(mn, k.neg6, t);  // na + 4d; lanes < 2^16
  i0 = cd_prmt(nas, d, 0x5540u);  // lane 0: nas.b0 | d.b0 << 8
  i1 = cd_prmt(nas, d, 0x7762u);  // lane 1: nas.b2 | d.b2 << 8
  const uint32_t tA = R + 0x10001000u - G;                                 // bit 12: r >= g
  const uint32_t tB = G + 0x20002000u - B;                                 // bit 13: g >= b
  // s flags against max itself: black (max = 0) sets both, but a grey pixel is
  // recognisable from its table entry (q3 = 0 only when d = 0) and
  // code_to_bin_dir forces s = 0 for it.
  const uint32_t z1 = cd_mad(mx, k.neg1, 0x04000400u);
  const uint32_t x1 = cd_mad(d, k.three, z1);  // 3d - mx + 2^10:  bit 10 = s1, < 2^11
  const uint32_t x2 = cd_mad(z1, k.one, x1);   // 3d - 2mx + 2^11: bit 11 = s2, < 2^12
  const uint32_t m3 = cd_mad(mx, k.three, 0u);  // bits 8-9 of 3 max = v, < 2^10
  const uint32_t tC = cd_mad(B, k.neg1, cd_mad(R, k.one, 0x40004000u));  // bit 14: r >= b
  // Above its low byte every threshold word is CLEAN: a - b + 2^j with
  // |a - b| < 256 has bit j = [a >= b], its complement in bits 8..j-1 and
  // zeros above (tA, tB, tC); x2 = 3d - 2mx + 2^11 lies in [1538, 2303], so its
  // bit 10 is ~s2 and only bits 0-9 vary otherwise, and x1 < 2^11.  Two
  // three-input XORs therefore merge the five flags into bits 10-14
  // invertibly, and one select puts v into bits 8-9 (x1 and x2 vary there):
  //   b10 = s1 ^ ~s2 ^ ~P,  b11 = s2 ^ ~P,  b12 = P = A ^ B ^ C,
  //   b13 = ~(B ^ C),  b14 = C          (decoded by code_to_bin_dir)
  // Three LOP3 instead of five bit-selects (B200 A/B: K1 +3.9 %, K1-NV12 +4.3 %).
  return cd_sel<0x03000300u>(m3, cd_xor3(x1, x2, cd_xor3(tA, tB, tC)));
}
// Part 2: the two lanes' byte offsets from the looked-up entries q0, q1 (u8).
CD_HD uint32_t dir_off_lo(uint32_t pre, uint32_t q0) { return cd_prmt(q0, pre, 0x1150u); }
CD_HD uint32_t dir_off_hi(uint32_t pre, uint32_t q1) { return cd_prmt(q1, pre, 0x1170u); }

// code index (byte offset / 4) -> bin in [0,162), or 255 for an unreachable code.
CD_HD uint32_t code_to_bin_dir(uint32_t idx) {
  const uint32_t c = idx << 2;
  const uint32_t q = (kDirQ >> (4 * ((c >> 2) & 7u))) & 15u;
  const uint32_t qr = q & 3u, qf = q >> 2, z = (c >> 7) & 1u, v = (c >> 8) & 3u;
  // undo code_pair_dir_pre's XOR mix of bits 10-14
  const uint32_t P = (c >> 12) & 1u, C = (c >> 14) & 1u, B = 1u ^ ((c >> 13) & 1u) ^ C;
  const uint32_t A = P ^ B ^ C, s2 = ((c >> 11) & 1u) ^ 1u ^ P;
  const uint32_t s1 = ((c >> 10) & 1u) ^ s2 ^ P, z2 = c >> 15;
  const uint32_t ris = A ^ B ^ C;  // odd #(>=) <=> rising sector
  const uint32_t oidx = (A << 2) | (B << 1) | C;
  if (z || z2 || oidx == 1u || oidx == 6u || v > 2u || s2 > s1) return 255u;
  if (qr == 0u && qf == 0u) return oidx == 7u ? v : 255u;  // grey (d = 0): h = 0, s = 0
  const uint32_t k3 = (kSector3k >> (oidx << 2)) & 15u;
  return (k3 + (ris ? qr : qf)) * 9u + (s1 + s2) * 3u + v;
}

// ------------------------------------------------------------ NV12 input (NEXT f1)
// Reading O0: NVDEC's NV12 (Y plane + interleaved UV at half resolution) ->
// RGB by BT.601 limited range in 20-bit fixed point (OpenCV's
// COLOR_YUV2RGB_NV12):  y' = max(0, Y-16)*1220542,  R = sat((y' + ruv) >> 20),
// G = sat((y' + guv) >> 20), B = sat((y' + buv) >> 20) with the chroma terms
// below (int32 throughout: |y' + c| < 2^30).  Two horizontally adjacent pixels
// share one chroma sample, so the pair comes out directly as u16x2 lanes.
constexpr int32_t kCY = 1220542;
CD_HD void nv12_chroma(uint32_t U, uint32_t V, int32_t& ruv, int32_t& guv, int32_t& buv) {
  ruv = 1673527 * (int32_t)V + (524288 - 128 * 1673527);
  guv = -852492 * (int32_t)V - 409993 * (int32_t)U + (524288 + 128 * 852492 + 128 * 409993);
  buv = 2116026 * (int32_t)U + (524288 - 128 * 2116026);
}
CD_HD int32_t nv12_luma(uint32_t Y) {
#if defined(__CUDA_ARCH__)
  return __viaddmax_s32((int32_t)Y, -16, 0) * kCY;  // VIADDMNMX
#else
  const int32_t y = (int32_t)Y - 16;
  return (y > 0 ? y : 0) * kCY;
#endif
}
// Per signed 16-bit lane: clamp to [0, 255].
CD_HD uint32_t cd_sat_u8_s16x2(uint32_t x) {
#if defined(__CUDA_ARCH__)
  return __vimin_s16x2_relu(x, 0x00FF00FFu);  // VIMNMX.S16x2.RELU
#else
  uint32_t out = 0;
  for (int l = 0; l < 2; ++l) {
    int32_t v = (int16_t)(x >> (16 * l));
    v = v < 0 ? 0 : (v > 255 ? 255 : v);
    out |= (uint32_t)v << (16 * l);
  }
  return out;
#endif
}
CD_HD uint32_t nv12_chan_pair(int32_t la, int32_t lb, int32_t c) {
  return cd_sat_u8_s16x2(cd_prmt((uint32_t)((la + c) >> 20), (uint32_t)((lb + c) >> 20), 0x5410u));
}
CD_HD void nv12_pair_rgb(uint32_t ya, uint32_t yb, int32_t ruv, int32_t guv, int32_t buv,
                         uint32_t& R, uint32_t& G, uint32_t& B) {
  const int32_t la = nv12_luma(ya), lb = nv12_luma(yb);
  R = nv12_chan_pair(la, lb, ruv);
  G = nv12_chan_pair(la, lb, guv);
  B = nv12_chan_pair(la, lb, buv);
}

// Pack 4 pixels (12 bytes in words w0, w1, w2) into two u16x2 pairs:
// (R01, G01, B01) = pixels 0,1 and (R23, G23, B23) = pixels 2,3.
CD_HD void unpack4(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t& R01, uint32_t& G01,
                   uint32_t& B01, uint32_t& R23, uint32_t& G23, uint32_t& B23) {
  // w0 = [r0 g0 b0 r1], w1 = [g1 b1 r2 g2], w2 = [b2 r3 g3 b3] (byte 0 first)
  const uint32_t s0 = w0 >> 8;  // [g0 b0 r1 0]
  const uint32_t s1 = w1 >> 8;  // [b1 r2 g2 0]
  R01 = cd_prmt(w0, 0u, 0x4340u);
  G01 = cd_prmt(s0, w1, 0x3430u);
  B01 = cd_prmt(s0, w1, 0x3531u);
  R23 = cd_prmt(s1, w2, 0x3531u);
  G23 = cd_prmt(s1, w2, 0x3632u);
  B23 = cd_prmt(w2, 0u, 0x4340u);
}

// ------------------------------------------------- general layouts (not the hot path)
// General (nh, ns, nv) with nh*ns*nv <= 256 (integer division).
CD_HD uint32_t bin_generic(uint32_t r, uint32_t g, uint32_t b, uint32_t nh, uint32_t ns,
                           uint32_t nv) {
  uint32_t mx = r > g ? r : g;
  mx = mx > b ? mx : b;
  uint32_t mn = r < g ? r : g;
  mn = mn < b ? mn : b;
  const uint32_t d = mx - mn;
  const uint32_t mid = r + g + b - mx - mn;
  const uint32_t idx = ((uint32_t)(r >= g) << 2) | ((uint32_t)(g >= b) << 1) | (uint32_t)(r >= b);
  const uint32_t k = ((kSector3k >> (idx << 2)) & 15u) / 3u;
  const uint32_t num = (k & 1u) ? (mx - mid) : (mid - mn);
  const uint32_t h = d == 0 ? 0u : (nh * (k * d + num)) / (6u * d);
  uint32_t s = mx == 0 ? 0u : (ns * d) / mx;
  s = s > ns - 1 ? ns - 1 : s;
  const uint32_t v = (nv * mx) >> 8;
  return (h * ns + s) * nv + v;
}

}  // namespace clipdetect
