// sampler.cuh -- point-pair sources of the hot path.
//
// Uniform random sampling of point pairs of two bricks, PAPER.md:139-140 (§3.1):
// "One sample position corresponds to a position in a 6 dimensional space, where 3
// dimensions represent the position in one brick, and the remaining 3 ... in the
// respective other brick."  Generator = DESIGN.md reading R15 (counter-based, keyed by
// the two boxes so that shards of the region list draw identical samples):
//   mix64 = splitmix64 finaliser;  h_{t+1} = mix64(h_t ^ (uint32(c_t) + G*(t+1)))
//   u_s = mix64(h_12 + G*(s+1));  a_local = (lo32(u_s)*|A|)>>32,  b_local = (hi32(u_s)*|B|)>>32
// Exhaustive enumeration: q = a_local*|B| + b_local ("all point-to-point pairs").
#pragma once

#include "corr_internal.cuh"

namespace corr {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__host__ __device__ inline uint64_t region_key(uint64_t seed, const corr_box& A, const corr_box& B) {
  const int32_t c[12] = {A.x0, A.y0, A.z0, A.x1, A.y1, A.z1, B.x0, B.y0, B.z0, B.x1, B.y1, B.z1};
  uint64_t h = seed;
  for (int t = 0; t < 12; ++t) h = mix64(h ^ ((uint64_t)(uint32_t)c[t] + kGolden * (uint64_t)(t + 1)));
  return h;
}

// local index (x fastest inside the box) -> global point index
__device__ __forceinline__ int64_t box_to_point(const corr_box& b, int64_t local, int nx, int ny) {
  const int64_t ax = b.x1 - b.x0, ay = b.y1 - b.y0;
  const int64_t lx = local % ax;
  const int64_t t = local / ax;
  const int64_t ly = t % ay;
  const int64_t lz = t / ay;
  return ((int64_t)(b.z0 + lz) * ny + (b.y0 + ly)) * nx + (b.x0 + lx);
}

// Region of an exhaustive-mode unit: largest r with reg[r].off <= u.
__device__ __forceinline__ int64_t find_region(const RegionDev* reg, int64_t nreg, int64_t u) {
  int64_t lo = 0, hi = nreg - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (reg[mid].off <= u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Unit u -> (a, b, region r, tie-break index).  Returns false if the pair is invalid
// (out-of-range list index: err flag raised) or must be skipped (self pair, one field).
__device__ __forceinline__ bool unit_pair(const PairSrc& s, int64_t u, int64_t& a, int64_t& b,
                                          int64_t& r, uint32_t& idx) {
  if (s.mode == kList) {
    a = s.idxA[u];
    b = s.idxB[u];
    r = u;
    idx = 0;
    if (a < 0 || a >= s.P || b < 0 || b >= s.P) {
      atomicOr(s.err, 1);
      return false;
    }
    return true;
  }
  if (s.mode == kSampled) {
    r = u / s.samples;
    const int64_t smp = u - r * s.samples;
    const RegionDev& R = s.reg[r];
    const uint64_t v = mix64(s.rkey[r] + kGolden * (uint64_t)(smp + 1));
    const uint64_t al = ((v & 0xFFFFFFFFULL) * (uint64_t)R.nA) >> 32;
    const uint64_t bl = ((v >> 32) * (uint64_t)R.nB) >> 32;
    a = box_to_point(R.A, (int64_t)al, s.nx, s.ny);
    b = box_to_point(R.B, (int64_t)bl, s.nx, s.ny);
    idx = (uint32_t)smp;
  } else {
    r = find_region(s.reg, s.nreg, u);
    const RegionDev& R = s.reg[r];
    const int64_t q = u - R.off;
    const int64_t al = q / R.nB, bl = q - al * R.nB;
    a = box_to_point(R.A, al, s.nx, s.ny);
    b = box_to_point(R.B, bl, s.nx, s.ny);
    idx = (uint32_t)q;
  }
  return !(s.same_field && a == b);
}

// Order-preserving packing of (value, index): larger value wins, ties -> lowest index.
// NaN is never packed (callers skip it); -0 is canonicalised to +0 (reading R16).
__device__ __forceinline__ unsigned long long pack_key(float v, uint32_t idx) {
  v = v + 0.0f;
  uint32_t u = __float_as_uint(v);
  u ^= (u >> 31) ? 0xFFFFFFFFu : 0x80000000u;
  return ((unsigned long long)u << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
}

__device__ __forceinline__ float unpack_value(unsigned long long key) {
  uint32_t u = (uint32_t)(key >> 32);
  u ^= (u >> 31) ? 0x80000000u : 0xFFFFFFFFu;
  return __uint_as_float(u);
}

}  // namespace corr
