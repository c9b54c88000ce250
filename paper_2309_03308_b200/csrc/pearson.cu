// pearson.cu -- Pearson (PPMCC) for batches of point pairs, SURVEY.md §8(a) row a6,
// and the region-pair max/argmax finalisation, row a9.
//
// PAPER.md:169 (§3.2): "PPMCC requires merely to compute means and variances".  The
// field stores each series standardised in fp64 (field.cu), so r = <Z_a, Z_b>: one
// fp32 dot product of two contiguous rows, 8n bytes per pair -- an HBM/L2-bound gather
// (DESIGN.md).  One warp per pair, float4 loads, fp32 FMA, warp-shuffle reduction,
// clamp to [-1, 1].
#include <math.h>

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
    const uint64_t v = mix64(R.key + kGolden * (uint64_t)((int64_t)idx + 1));
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

cudaError_t launch_pearson_pairs(const corr_field* fa, const corr_field* fb, const PairSrc& src,
                                 const PairOut& out, cudaStream_t st) {
  if (src.nunits == 0) return cudaSuccess;
  const int nq = fa->n_pad / 4;
  int lpp = 4;
  while (lpp < 32 && lpp * 4 < nq) lpp <<= 1;
  auto launch = [&](auto kern, int ppw) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    if (occ < 1) occ = 1;
    int64_t blocks = (src.nunits + 8 * ppw - 1) / (8 * ppw);
    const int64_t cap = (int64_t)kSMs * occ * 4;
    if (blocks > cap) blocks = cap;
    kern<<<(unsigned)blocks, 256, 0, st>>>(fa->Z, fb->Z, fa->cflag, fb->cflag, fa->n_pad, src, out);
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
