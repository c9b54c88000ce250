// ksg.cu -- Kraskov (KSG) mutual information for batches of point pairs,
// SURVEY.md §8(a) rows a2-a5 (+ a8/a9 when fed by the region sampler).
//
// PAPER.md:172-174 (§3.2): for the joint samples z_i = (x_i, y_i), i = 1..n,
//   eps_i  = Chebyshev distance to the k-th nearest neighbour (j != i),
//   n_x,i  = #{ j : |x_i - x_j| < eps_i },  n_y,i likewise (strict),
//   MI     = psi(n) + psi(k) - (1/n) sum_i [ psi(n_x,i) + psi(n_y,i) ]   (reading R2)
// with fp32 distances (reading R7) so that eps and the counts are bit-identical to
// the oracle's brute force.
//
// B200 design: the paper builds one k-d tree per pair in one
// thread.  Here a team of warps owns one pair; each lane owns R = 4
// members ("register blocking": one broadcast LDS.128 of two joint samples feeds
// 8 comparisons) and keeps its k smallest distances in a sorted register list updated
// by a branch-free min/max network (2k-1 FMNMX per comparison, no divergence).  The
// self pair is excluded only on the diagonal 32-member chunks.  Marginal counts are
// two binary searches per marginal on the field's pre-sorted rows with monotone fp32
// predicates (bit-exact, O(log n) instead of the O(n) brute-force count).  psi comes
// from a shared-memory fp64 table (arguments are integers; reading R17).
#include <math.h>
#include <stdlib.h>

#include "sampler.cuh"

namespace corr {
namespace {

constexpr int R = 4;            // members per lane
constexpr int kBlockMembers = 32 * R;

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  unsigned long long ua = *reinterpret_cast<unsigned long long*>(&a);
  unsigned long long ub = *reinterpret_cast<unsigned long long*>(&b);
  unsigned long long ud;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(ud) : "l"(ua), "l"(ub));
  return *reinterpret_cast<float2*>(&ud);
}

template <int K>
__device__ __forceinline__ void knn_insert(float (&l)[K], float d) {
#pragma unroll
  for (int t = K - 1; t >= 1; --t) l[t] = fminf(l[t], fmaxf(l[t - 1], d));
  l[0] = fminf(l[0], d);
}

// strict marginal count, on the sorted row S[0..n):
//   u = first t with S[t] >= v && fl(S[t]-v) >= e ;  w = first t with S[t] >= v || fl(v-S[t]) < e
//   count = (u - w) - [e > 0]   (the self sample is inside [w, u) iff e > 0)
__device__ __forceinline__ int marginal_count(const float* __restrict__ S, int n, float v, float e) {
  int lo = 0, len = n;
  while (len > 0) {
    const int half = len >> 1;
    const float s = S[lo + half];
    const bool pred = (s >= v) && (s - v >= e);
    if (pred) len = half; else { lo += half + 1; len -= half + 1; }
  }
  const int u = lo;
  lo = 0; len = n;
  while (len > 0) {
    const int half = len >> 1;
    const float s = S[lo + half];
    const bool pred = (s >= v) || (v - s < e);
    if (pred) len = half; else { lo += half + 1; len -= half + 1; }
  }
  return (u - lo) - (e > 0.f ? 1 : 0);
}

// Team = one warp (TEAM_WARPS == 1, eight independent teams per CTA) or the whole CTA.
template <int TEAM_WARPS>
__device__ __forceinline__ void team_sync() {
  if (TEAM_WARPS == 1) __syncwarp(); else __syncthreads();
}

template <int K, int TEAM_WARPS>
__global__ void __launch_bounds__(256) ksg_kernel(const float* __restrict__ Fa, const float* __restrict__ Fb,
                                                  const float* __restrict__ Sa, const float* __restrict__ Sb,
                                                  const uint8_t* __restrict__ ca, const uint8_t* __restrict__ cb,
                                                  const double* __restrict__ psi_g, int n, int n_pad, int k,
                                                  int plus1, PairSrc src, PairOut out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kTeams = TEAM_WARPS == 1 ? 8 : 1;
  const int warps_per_team = TEAM_WARPS == 1 ? 1 : (int)(blockDim.x >> 5);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int team = TEAM_WARPS == 1 ? warp : 0;
  const int wt = TEAM_WARPS == 1 ? 0 : warp;  // warp index inside the team
  const int tt = TEAM_WARPS == 1 ? lane : (int)threadIdx.x;
  const int team_threads = 32 * warps_per_team;
  const int nblk = (n + kBlockMembers - 1) / kBlockMembers;
  const int nxy = nblk * kBlockMembers;  // joint samples staged, +inf padded

  double* psi = reinterpret_cast<double*>(smem_raw);
  const int psi_len = (n + 2 + 1) & ~1;
  unsigned char* team_base = smem_raw + psi_len * sizeof(double);
  const size_t team_bytes = (size_t)nxy * sizeof(float2) + 2 * (size_t)n_pad * sizeof(float) + 32 * sizeof(double);
  float2* xy = reinterpret_cast<float2*>(team_base + team * team_bytes);
  float* sx = reinterpret_cast<float*>(xy + nxy);
  float* sy = sx + n_pad;
  double* red = reinterpret_cast<double*>(sy + n_pad);

  for (int i = threadIdx.x; i < n + 2; i += blockDim.x) psi[i] = psi_g[i];
  __syncthreads();

  const double psi_nk = psi[n] + psi[k];
  const int off = plus1 ? 1 : 0;
  const int64_t team_id = (int64_t)blockIdx.x * kTeams + team;
  const int64_t team_stride = (int64_t)gridDim.x * kTeams;

  for (int64_t u = team_id; u < src.nunits; u += team_stride) {
    int64_t a, b, r;
    uint32_t idx;
    const bool ok = unit_pair(src, u, a, b, r, idx);
    if (!ok) {
      if (src.mode == kList && tt == 0) out.out[u] = NAN;
      continue;
    }
    const bool degenerate = (ca[a] | cb[b]) != 0;  // constant series (reading R10)
    if (degenerate && out.dbg_eps == nullptr) {
      if (src.mode == kList && tt == 0) out.out[u] = NAN;
      continue;
    }
    team_sync<TEAM_WARPS>();  // previous unit finished reading shared memory
    // ---- a2: stage the pair (rows are 32-byte aligned) ----
    {
      const float4* fa4 = reinterpret_cast<const float4*>(Fa + a * n_pad);
      const float4* fb4 = reinterpret_cast<const float4*>(Fb + b * n_pad);
      const float4* sa4 = reinterpret_cast<const float4*>(Sa + a * n_pad);
      const float4* sb4 = reinterpret_cast<const float4*>(Sb + b * n_pad);
      float4* sx4 = reinterpret_cast<float4*>(sx);
      float4* sy4 = reinterpret_cast<float4*>(sy);
      for (int q = tt; q < n_pad / 4; q += team_threads) {
        const float4 va = __ldg(fa4 + q), vb = __ldg(fb4 + q);
        const int j = 4 * q;
        float4* dst = reinterpret_cast<float4*>(xy + j);
        const float inf = INFINITY;
        dst[0] = make_float4(j + 0 < n ? va.x : inf, j + 0 < n ? vb.x : inf, j + 1 < n ? va.y : inf, j + 1 < n ? vb.y : inf);
        dst[1] = make_float4(j + 2 < n ? va.z : inf, j + 2 < n ? vb.z : inf, j + 3 < n ? va.w : inf, j + 3 < n ? vb.w : inf);
        sx4[q] = __ldg(sa4 + q);
        sy4[q] = __ldg(sb4 + q);
      }
      for (int j = n_pad + tt; j < nxy; j += team_threads) xy[j] = make_float2(INFINITY, INFINITY);
    }
    team_sync<TEAM_WARPS>();

    // ---- a3: k-NN pass; a4: counts; a5: psi terms ----
    double acc = 0.0;
    for (int mb = wt; mb < nblk; mb += warps_per_team) {
      float2 zi[R];
      float l[R][K];
      int irow[R];
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        irow[rr] = mb * kBlockMembers + 32 * rr + lane;
        zi[rr] = xy[irow[rr]];
#pragma unroll
        for (int t = 0; t < K; ++t) l[rr][t] = INFINITY;
      }
      const float4* xy4 = reinterpret_cast<const float4*>(xy);
      const int nch = (n + 31) >> 5;
      for (int c = 0; c < nch; ++c) {
        const float4* cp = xy4 + c * 16;
        if ((c >> 2) != mb) {
#pragma unroll 8
          for (int t = 0; t < 16; ++t) {
            const float4 v = cp[t];
            const float2 z0 = make_float2(v.x, v.y), z1 = make_float2(v.z, v.w);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              const float2 d0 = sub2(zi[rr], z0);
              const float2 d1 = sub2(zi[rr], z1);
              knn_insert<K>(l[rr], fmaxf(fabsf(d0.x), fabsf(d0.y)));
              knn_insert<K>(l[rr], fmaxf(fabsf(d1.x), fabsf(d1.y)));
            }
          }
        } else {  // diagonal chunk: skip j == i ("k-th nearest neighbor", reading R3)
          const int jb = c * 32;
#pragma unroll 4
          for (int t = 0; t < 16; ++t) {
            const float4 v = cp[t];
            const float2 z0 = make_float2(v.x, v.y), z1 = make_float2(v.z, v.w);
#pragma unroll
            for (int rr = 0; rr < R; ++rr) {
              const float2 d0 = sub2(zi[rr], z0);
              const float2 d1 = sub2(zi[rr], z1);
              float e0 = fmaxf(fabsf(d0.x), fabsf(d0.y));
              float e1 = fmaxf(fabsf(d1.x), fabsf(d1.y));
              if (jb + 2 * t == irow[rr]) e0 = INFINITY;
              if (jb + 2 * t + 1 == irow[rr]) e1 = INFINITY;
              knn_insert<K>(l[rr], e0);
              knn_insert<K>(l[rr], e1);
            }
          }
        }
      }
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        if (irow[rr] < n) {
          const float e = l[rr][K - 1];
          const int cx = marginal_count(sx, n, zi[rr].x, e);
          const int cy = marginal_count(sy, n, zi[rr].y, e);
          acc += psi[cx + off] + psi[cy + off];
          if (out.dbg_eps) {
            out.dbg_eps[u * n + irow[rr]] = e;
            out.dbg_nx[u * n + irow[rr]] = cx;
            out.dbg_ny[u * n + irow[rr]] = cy;
          }
        }
      }
    }
    // ---- team reduction of the psi sum (fp64, fixed order) ----
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (TEAM_WARPS != 1) {
      if (lane == 0) red[wt] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < warps_per_team; ++w) s += red[w];
        red[31] = s;
      }
      __syncthreads();
      acc = red[31];
    }
    if (tt == 0) {
      const float mi = degenerate ? NAN : (float)(psi_nk - acc / (double)n);
      if (src.mode == kList) {
        out.out[u] = mi;
      } else if (!isnan(mi)) {
        atomicMax(out.keys + r, pack_key(out.absval ? fabsf(mi) : mi, idx));
      }
    }
  }
}

template <int K>
cudaError_t launch_k(const corr_field* fa, const corr_field* fb, int k, int plus1, const PairSrc& src,
                     const PairOut& out, cudaStream_t st) {
  static const int small_sorted = [] {
    const char* s = getenv("CORR_KSG_SMALL");  // "warp" keeps the one-warp-per-pair kernel
    return (s && s[0] == 'w') ? 0 : 1;
  }();
  if (fa->n > kBlockMembers || small_sorted || k > 8) return launch_ksg_sorted(fa, fb, k, plus1, src, out, st);
  const int n = fa->n, n_pad = fa->n_pad;
  const int nblk = (n + kBlockMembers - 1) / kBlockMembers;
  const int nxy = nblk * kBlockMembers;
  const size_t psi_bytes = (size_t)((n + 2 + 1) & ~1) * sizeof(double);
  const size_t team_bytes = (size_t)nxy * sizeof(float2) + 2 * (size_t)n_pad * sizeof(float) + 32 * sizeof(double);
  int dev_sms = kSMs;
  if (n <= kBlockMembers) {
    auto kern = ksg_kernel<K, 1>;
    const size_t smem = psi_bytes + 8 * team_bytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
    if (occ < 1) occ = 1;
    int64_t blocks = (src.nunits + 7) / 8;
    const int64_t cap = (int64_t)dev_sms * occ;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, 256, smem, st>>>(fa->F, fb->F, fa->S, fb->S, fa->cflag, fb->cflag, fa->psi, n,
                                              n_pad, k, plus1 & 1, src, out);
    note_launch();
  } else {
    auto kern = ksg_kernel<K, 8>;
    const int warps = nblk < 8 ? nblk : 8;
    const size_t smem = psi_bytes + team_bytes;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem);
    if (occ < 1) occ = 1;
    int64_t blocks = src.nunits;
    const int64_t cap = (int64_t)dev_sms * occ;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, warps * 32, smem, st>>>(fa->F, fb->F, fa->S, fb->S, fa->cflag, fb->cflag, fa->psi,
                                                     n, n_pad, k, plus1 & 1, src, out);
    note_launch();
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ksg(const corr_field* fa, const corr_field* fb, int k, int plus1, const PairSrc& src,
                       const PairOut& out, cudaStream_t st) {
  if (src.nunits == 0) return cudaSuccess;
  if (k > 8) return launch_ksg_sorted(fa, fb, k, plus1, src, out, st);
  switch (k) {
    case 1: return launch_k<1>(fa, fb, k, plus1, src, out, st);
    case 2: return launch_k<2>(fa, fb, k, plus1, src, out, st);
    case 3: return launch_k<3>(fa, fb, k, plus1, src, out, st);
    case 4: return launch_k<4>(fa, fb, k, plus1, src, out, st);
    case 5: return launch_k<5>(fa, fb, k, plus1, src, out, st);
    case 6: return launch_k<6>(fa, fb, k, plus1, src, out, st);
    case 7: return launch_k<7>(fa, fb, k, plus1, src, out, st);
    case 8: return launch_k<8>(fa, fb, k, plus1, src, out, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace corr
