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
// and for nh = 18: h = 3k + floor(3*num/d), an integer threshold count.
// Verified bit-exact against the oracle on all 2^24 colours (K5 test).
#pragma once

#include <stdint.h>

namespace clipdetect {

// 3k for the 8 ordering codes idx = [r>=g]*4 + [g>=b]*2 + [r>=b]
// (codes 1 and 6 are infeasible):  idx 0 -> k=3, 2 -> k=2, 3 -> k=1, 4 -> k=4,
// 5 -> k=5, 7 -> k=0.  One nibble per code.
constexpr uint32_t kSector3k = (9u << 0) | (0u << 4) | (6u << 8) | (3u << 12) | (12u << 16) |
                               (15u << 20) | (0u << 24) | (0u << 28);

// Fast path, (nh, ns, nv) = (18, 3, 3): 162 bins, branch-free, no division.
__device__ __forceinline__ uint32_t bin_18_3_3(uint32_t r, uint32_t g, uint32_t b) {
  const uint32_t mx = __vimax3_u32(r, g, b);
  const uint32_t mn = __vimin3_u32(r, g, b);
  const uint32_t d = mx - mn;
  const uint32_t mid = r + g + b - mx - mn;
  const uint32_t idx = ((r >= g) << 2) | ((g >= b) << 1) | (r >= b);
  const uint32_t k3 = (kSector3k >> (idx << 2)) & 15u;
  const uint32_t num = (k3 & 1u) ? (mx - mid) : (mid - mn);
  const uint32_t d1 = max(d, 1u);  // d = 0: grey, num = 0 -> q = 0
  const uint32_t n3 = 3u * num;
  const uint32_t q = (n3 >= d1) + (n3 >= 2u * d1) + (num >= d1);
  const uint32_t mx1 = max(mx, 1u);  // mx = 0: black, s = 0
  const uint32_t d3 = 3u * d;
  const uint32_t s = (d3 >= mx1) + (d3 >= 2u * mx1);
  const uint32_t v = (mx >= 86u) + (mx >= 171u);  // floor(3*mx/256)
  return (k3 + q) * 9u + s * 3u + v;
}

// General (nh, ns, nv) with nh*ns*nv <= 256 (integer division; not the hot path).
__device__ __forceinline__ uint32_t bin_generic(uint32_t r, uint32_t g, uint32_t b, uint32_t nh,
                                                uint32_t ns, uint32_t nv) {
  const uint32_t mx = __vimax3_u32(r, g, b);
  const uint32_t mn = __vimin3_u32(r, g, b);
  const uint32_t d = mx - mn;
  const uint32_t mid = r + g + b - mx - mn;
  const uint32_t idx = ((r >= g) << 2) | ((g >= b) << 1) | (r >= b);
  const uint32_t k = ((kSector3k >> (idx << 2)) & 15u) / 3u;
  const uint32_t num = (k & 1u) ? (mx - mid) : (mid - mn);
  const uint32_t h = d == 0 ? 0u : (nh * (k * d + num)) / (6u * d);
  uint32_t s = mx == 0 ? 0u : (ns * d) / mx;
  s = s > ns - 1 ? ns - 1 : s;
  const uint32_t v = (nv * mx) >> 8;
  return (h * ns + s) * nv + v;
}

}  // namespace clipdetect
