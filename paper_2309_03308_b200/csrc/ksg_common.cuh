// ksg_common.cuh -- device helpers shared by the KSG kernels (ksg.cu: sweep / dense / warp
// kernels, ksg_cell.cu: the column-cell kernel): packed fp32 differences, the Chebyshev distance,
// the sorted k-list merge network, immediate-offset shared loads, and the TMA-unit staging
// (cp.async.bulk + mbarrier, L2 bulk prefetch).
#pragma once

#include <math.h>

#include "sampler.cuh"

namespace corr {

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long ua = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long ub = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long ud;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ud) : "l"(ua), "l"(ub));
  return *reinterpret_cast<float2*>(&ud);
}

__device__ __forceinline__ float cheb(float2 zi, float2 zj) {
  const float2 d = sub2(zi, zj);
  return fmaxf(fabsf(d.x), fabsf(d.y));
}

template <int K>
__device__ __forceinline__ void merge2(float (&l)[K], float d0, float d1) {
  const float a = fminf(d0, d1), b = fmaxf(d0, d1);
  float nl[K];
  nl[0] = fminf(l[0], a);
  if (K >= 2) nl[1] = fminf(fminf(l[1], fmaxf(l[0], a)), b);
#pragma unroll
  for (int r = 2; r < K; ++r) nl[r] = fminf(fminf(l[r], fmaxf(l[r - 1], a)), fmaxf(l[r - 2], b));
#pragma unroll
  for (int r = 0; r < K; ++r) l[r] = nl[r];
}

template <int K>
__device__ __forceinline__ void insert1(float (&l)[K], float d) {
#pragma unroll
  for (int t = K - 1; t >= 1; --t) l[t] = fminf(l[t], fmaxf(l[t - 1], d));
  l[0] = fminf(l[0], d);
}

template <int OFF>
__device__ __forceinline__ float lds_imm(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1+%2];" : "=f"(v) : "r"(addr), "n"(OFF));
  return v;
}

// ---- a2 staging through the TMA unit: 1-D bulk copies global -> shared with an mbarrier
// (cp.async.bulk, contiguous rows: no tensor map needed) and bulk L2 prefetches of the
// next pair's rows, so a CTA's next staging finds its rows in L2.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(b))
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Side-effect-free peek at unit u's point pair (prefetch only; errors are raised when the
// unit itself is processed).
__device__ __forceinline__ bool peek_pair(const PairSrc& s, int64_t u, int64_t& a, int64_t& b) {
  if (s.mode == kList) {
    a = s.idxA[u];
    b = s.idxB[u];
    return a >= 0 && a < s.P && b >= 0 && b < s.P;
  }
  int64_t r;
  uint32_t idx;
  return unit_pair(s, u, a, b, r, idx);
}

}  // namespace corr
