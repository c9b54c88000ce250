// pearson.cu -- Pearson (PPMCC) for batches of point pairs, SURVEY.md §8(a) row a6,
// and the region-pair max/argmax finalisation, row a9.
//
// PAPER.md:169 (§3.2): "PPMCC requires merely to compute means and variances".  The
// field stores each series standardised in fp64 (field.cu), so r = <Z_a, Z_b>: one
// fp32 dot product of two contiguous rows, 8n bytes per pair -- an HBM/L2-bound gather
// (DESIGN.md).  One warp per pair, float4 loads, fp32 FMA, warp-shuffle reduction,
// clamp to [-1, 1].
#include <math.h>
#include <stdlib.h>

#include "sampler.cuh"

namespace corr {
namespace {

// LPP lanes per pair (4..32): small n packs several pairs into one warp so every lane keeps
// loads in flight (one-to-all / sampled pairs are a latency-bound gather otherwise).
template <int LPP>
__global__ void __launch_bounds__(256) pearson_pairs_kernel(const float* __restrict__ Za, const float* __restrict__ Zb,
                                                            const uint8_t* __restrict__ ca,
                                                            const uint8_t* __restrict__ cb, int n_pad, PairSrc src,
                                                            PairOut out) {
  constexpr int PPW = 32 / LPP;  // pairs per warp
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPP, sl = lane % LPP;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nq = n_pad >> 2;
  for (int64_t u0 = warp0 * PPW; u0 < src.nunits; u0 += nwarps * PPW) {
    const int64_t u = u0 + sub;
    int64_t a = 0, b = 0, r = 0;
    uint32_t idx = 0;
    const bool live = u < src.nunits;
    const bool ok = live && unit_pair(src, u, a, b, r, idx);
    const bool valid = ok && !(ca[a] | cb[b]);
    float acc = 0.f, acc1 = 0.f;
    if (valid) {
      const float4* pa = reinterpret_cast<const float4*>(Za + a * n_pad);
      const float4* pb = reinterpret_cast<const float4*>(Zb + b * n_pad);
      int q = sl;
      for (; q + LPP < nq; q += 2 * LPP) {
        const float4 x0 = __ldg(pa + q), y0 = __ldg(pb + q);
        const float4 x1 = __ldg(pa + q + LPP), y1 = __ldg(pb + q + LPP);
        acc = fmaf(x0.x, y0.x, acc); acc = fmaf(x0.y, y0.y, acc);
        acc = fmaf(x0.z, y0.z, acc); acc = fmaf(x0.w, y0.w, acc);
        acc1 = fmaf(x1.x, y1.x, acc1); acc1 = fmaf(x1.y, y1.y, acc1);
        acc1 = fmaf(x1.z, y1.z, acc1); acc1 = fmaf(x1.w, y1.w, acc1);
      }
      if (q < nq) {
        const float4 x0 = __ldg(pa + q), y0 = __ldg(pb + q);
        acc = fmaf(x0.x, y0.x, acc); acc = fmaf(x0.y, y0.y, acc);
        acc = fmaf(x0.z, y0.z, acc); acc = fmaf(x0.w, y0.w, acc);
      }
    }
    acc += acc1;
#pragma unroll
    for (int o = LPP / 2; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (sl == 0 && live) {
      const float v = valid ? fminf(1.f, fmaxf(-1.f, acc)) : NAN;
      if (src.mode == kList) {
        out.out[u] = v;
      } else if (valid) {
        atomicMax(out.keys + r, pack_key(out.absval ? fabsf(v) : v, idx));
      }
    }
  }
}

// ---- screened region max over sampled / enumerated pairs (exact) -------------------------------
// Only each region pair's maximum is kept, so pass 1 evaluates every pair on bf16(Z) rows (half the
// bytes of the fp32 rows: this gather is HBM-bound) and records the approximate value per pair and
// the approximate maximum per region pair; pass 2 recomputes in fp32 only the pairs within delta
// of their region's approximate maximum.  |fp32 dot - bf16 dot| <= (2u + u^2) + K 2^-23 per pass
// for unit rows (u = 2^-8), so with delta = 2b no pair that could be (or tie) the maximum is
// dropped -- the same argument as the screened block GEMM (pearson_gemm.cu).
__device__ __forceinline__ uint32_t ord_u32(float v) {
  uint32_t u = __float_as_uint(v + 0.0f);
  return u ^ ((u >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float unord_u32(uint32_t u) {
  return __uint_as_float(u ^ ((u >> 31) ? 0x80000000u : 0xFFFFFFFFu));
}

template <int LPP>
__global__ void __launch_bounds__(256) pearson_screen_kernel(const uint16_t* __restrict__ Za, const uint16_t* __restrict__ Zb,
                                                             const uint8_t* __restrict__ ca,
                                                             const uint8_t* __restrict__ cb, int n_pad, PairSrc src,
                                                             int absval, float* __restrict__ approx,
                                                             uint32_t* __restrict__ regkey) {
  constexpr int PPW = 32 / LPP;
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPP, sl = lane % LPP;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int n8 = n_pad >> 3;  // uint4 = 8 bf16
  for (int64_t u0 = warp0 * PPW; u0 < src.nunits; u0 += nwarps * PPW) {
    const int64_t u = u0 + sub;
    int64_t a = 0, b = 0, r = 0;
    uint32_t idx = 0;
    const bool live = u < src.nunits;
    const bool ok = live && unit_pair(src, u, a, b, r, idx);
    const bool valid = ok && !(ca[a] | cb[b]);
    float acc = 0.f;
    if (valid) {
      const uint4* pa = reinterpret_cast<const uint4*>(Za + a * n_pad);
      const uint4* pb = reinterpret_cast<const uint4*>(Zb + b * n_pad);
      for (int q = sl; q < n8; q += LPP) {
        const uint4 x = __ldg(pa + q), y = __ldg(pb + q);
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          acc = fmaf(__uint_as_float(xs[h] << 16), __uint_as_float(ys[h] << 16), acc);
          acc = fmaf(__uint_as_float(xs[h] & 0xFFFF0000u), __uint_as_float(ys[h] & 0xFFFF0000u), acc);
        }
      }
    }
#pragma unroll
    for (int o = LPP / 2; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (sl == 0 && live) {
      const float v = absval ? fabsf(acc) : acc;
      approx[u] = valid ? v : -INFINITY;
      if (valid) atomicMax(regkey + r, ord_u32(v));
    }
  }
}

// pass 2: fp32 dot products only for the pairs that can hold their region pair's maximum.  Lanes
// test 32 consecutive units at once (coalesced approx[] reads); the rare candidates are then
// evaluated one by one by the whole warp (float4 loads over 32 lanes).
__global__ void __launch_bounds__(256) pearson_exact_selected_kernel(const float* __restrict__ Za,
                                                                     const float* __restrict__ Zb, int n_pad,
                                                                     PairSrc src, PairOut out,
                                                                     const float* __restrict__ approx,
                                                                     const uint32_t* __restrict__ regkey, float delta) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nq = n_pad >> 2;
  for (int64_t g0 = warp0 * 32; g0 < src.nunits; g0 += nwarps * 32) {
    const int64_t u = g0 + lane;
    bool need = false;
    if (u < src.nunits) {
      const float v1 = approx[u];
      if (v1 > -INFINITY) {
        const int64_t r = src.mode == kSampled ? u / src.samples : find_region(src.reg, src.nreg, u);
        need = v1 >= unord_u32(regkey[r]) - delta;
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, need);
    while (mask) {
      const int srcl = __ffs(mask) - 1;
      mask &= mask - 1;
      const int64_t uu = __shfl_sync(0xffffffffu, u, srcl);
      int64_t a, b, r;
      uint32_t idx;
      unit_pair(src, uu, a, b, r, idx);
      const float4* pa = reinterpret_cast<const float4*>(Za + a * n_pad);
      const float4* pb = reinterpret_cast<const float4*>(Zb + b * n_pad);
      float acc = 0.f;
      for (int q = lane; q < nq; q += 32) {
        const float4 x0 = __ldg(pa + q), y0 = __ldg(pb + q);
        acc = fmaf(x0.x, y0.x, acc); acc = fmaf(x0.y, y0.y, acc);
        acc = fmaf(x0.z, y0.z, acc); acc = fmaf(x0.w, y0.w, acc);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        const float v = fminf(1.f, fmaxf(-1.f, acc));
        atomicMax(out.keys + r, pack_key(out.absval ? fabsf(v) : v, idx));
      }
    }
  }
}

__global__ void region_keys_kernel(const RegionDev* __restrict__ reg, int64_t nreg, uint64_t seed,
                                   uint64_t* __restrict__ rkey) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nreg) rkey[r] = region_key(seed, reg[r].A, reg[r].B);
}

__global__ void region_finalize_kernel(PairSrc src, const unsigned long long* __restrict__ keys,
                                       float* __restrict__ out_max, int64_t* __restrict__ out_arg) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= src.nreg) return;
  const unsigned long long key = keys[r];
  if (key == 0ULL) {
    out_max[r] = NAN;
    out_arg[2 * r] = -1;
    out_arg[2 * r + 1] = -1;
    return;
  }
  const uint32_t idx = 0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFULL);
  const RegionDev& R = src.reg[r];
  int64_t a, b;
  if (src.mode == kSampled) {
    const uint64_t v = mix64(src.rkey[r] + kGolden * (uint64_t)((int64_t)idx + 1));
    a = box_to_point(R.A, (int64_t)(((v & 0xFFFFFFFFULL) * (uint64_t)R.nA) >> 32), src.nx, src.ny);
    b = box_to_point(R.B, (int64_t)(((v >> 32) * (uint64_t)R.nB) >> 32), src.nx, src.ny);
  } else {
    const int64_t q = (int64_t)idx;
    a = box_to_point(R.A, q / R.nB, src.nx, src.ny);
    b = box_to_point(R.B, q % R.nB, src.nx, src.ny);
  }
  out_max[r] = unpack_value(key);
  out_arg[2 * r] = a;
  out_arg[2 * r + 1] = b;
}

}  // namespace

cudaError_t launch_region_keys(const RegionDev* dreg, int64_t nreg, uint64_t seed, uint64_t* rkey, cudaStream_t st) {
  if (nreg == 0) return cudaSuccess;
  region_keys_kernel<<<(unsigned)((nreg + 255) / 256), 256, 0, st>>>(dreg, nreg, seed, rkey);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_pearson_pairs(const corr_field* fa, const corr_field* fb, const PairSrc& src,
                                 const PairOut& out, cudaStream_t st) {
  if (src.nunits == 0) return cudaSuccess;
  const int nq = fa->n_pad / 4;
  int lpp = 4;
  // at most 8 lanes per pair (>= 4 pairs per warp, more loads in flight per lane): the Table-1
  // one-to-all PPMCC at n = 1000 1.72 -> 1.28 ms (16 lanes: 1.47 ms)
  while (lpp < 8 && lpp * 4 < nq) lpp <<= 1;
  static const int noscreen = [] {
    const char* v = getenv("CORR_PAIRS_NOSCREEN");  // A/B switch: every pair in fp32
    return (v && v[0] == '1') ? 1 : 0;
  }();
  auto grid_of = [&](auto kern, int ppw) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    if (occ < 1) occ = 1;
    int64_t blocks = (src.nunits + 8 * ppw - 1) / (8 * ppw);
    const int w = grid_waves_env() == -1 ? 64 : grid_waves_env();  // 64 waves: -2.5 % time vs 4 (A/B: CORR_WAVES)
    const int64_t cap = w > 0 ? (int64_t)kSMs * occ * w : blocks;
    if (blocks > cap) blocks = cap;
    return (unsigned)(blocks > 0x7FFFFFFF ? 0x7FFFFFFF : blocks);
  };
  if (src.mode != kList && !noscreen) {
    // screened (exact) region max: bf16 pass over every pair, fp32 pass over the candidates
    float* approx = nullptr;
    uint32_t* regkey = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&approx, (size_t)src.nunits * 4, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&regkey, (size_t)src.nreg * 4, st);
    if (e != cudaSuccess) {
      if (approx) cudaFreeAsync(approx, st);
      return e;
    }
    cudaMemsetAsync(regkey, 0, (size_t)src.nreg * 4, st);
    const double uu = 1.0 / 256.0;  // bf16 unit roundoff 2^-8
    const double b_bound = 2.0 * uu + uu * uu + 2.0 * (double)fa->n_pad / 8388608.0 + 1e-6;
    const float delta = (float)(2.0 * b_bound * 1.1);
    int l8 = 4;
    // lanes per pair for the bf16 rows (>= 4 pairs per warp): at n = 1000, 8 lanes x 16 loads of
    // 16 B per row keep more loads in flight than 16 x 8: 12.5 -> 10.6 ms for the C4 screen
    // (5.9 TB/s of assumed bytes); 4 lanes: 18.0 ms, 32 lanes: 13.0 ms
    while (l8 < 8 && l8 * 4 < fa->n_pad / 8) l8 <<= 1;
    auto scr = [&](auto kern, int ppw) {
      kern<<<grid_of(kern, ppw), 256, 0, st>>>(fa->Zb, fb->Zb, fa->cflag, fb->cflag, fa->n_pad, src, out.absval,
                                               approx, regkey);
    };
    switch (l8) {
      case 4: scr(pearson_screen_kernel<4>, 8); break;
      case 8: scr(pearson_screen_kernel<8>, 4); break;
      case 16: scr(pearson_screen_kernel<16>, 2); break;
      default: scr(pearson_screen_kernel<32>, 1); break;
    }
    {
      auto kern = pearson_exact_selected_kernel;
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
      if (occ < 1) occ = 1;
      int64_t blocks = (src.nunits + 255) / 256;
      const int64_t cap = (int64_t)kSMs * occ * 4;
      kern<<<(unsigned)(blocks > cap ? cap : blocks), 256, 0, st>>>(fa->Z, fb->Z, fa->n_pad, src, out, approx, regkey,
                                                                   delta);
    }
    note_launch(2);
    e = cudaGetLastError();
    cudaFreeAsync(approx, st);
    cudaFreeAsync(regkey, st);
    return e;
  }
  auto launch = [&](auto kern, int ppw) {
    kern<<<grid_of(kern, ppw), 256, 0, st>>>(fa->Z, fb->Z, fa->cflag, fb->cflag, fa->n_pad, src, out);
  };
  switch (lpp) {
    case 4: launch(pearson_pairs_kernel<4>, 8); break;
    case 8: launch(pearson_pairs_kernel<8>, 4); break;
    case 16: launch(pearson_pairs_kernel<16>, 2); break;
    default: launch(pearson_pairs_kernel<32>, 1); break;
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_region_finalize(const PairSrc& src, const unsigned long long* keys, float* out_max,
                                   int64_t* out_argmax, cudaStream_t st) {
  if (src.nreg == 0) return cudaSuccess;
  region_finalize_kernel<<<(unsigned)((src.nreg + 127) / 128), 128, 0, st>>>(src, keys, out_max, out_argmax);
  note_launch();
  return cudaGetLastError();
}

}  // namespace corr
