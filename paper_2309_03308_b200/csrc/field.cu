// field.cu -- field ingest, SURVEY.md §8(a) row a1 (§3).
//
// Input : float32 [n][P] (member-major file order), device-resident.
// Output: member-contiguous rows, one 32-byte-aligned row per grid point, so that a
//         point pair's 2n member values are two contiguous HBM reads (row a2) and a
//         region block is a dense K-major matrix for the tensor cores (row a7):
//   F  [P][n_pad]  raw values (pad 0)
//   Z  [P][n_pad]  standardised series (x - mean)/||x - mean||, fp64 -> fp32
//                  (Pearson = <Z_a, Z_b>, "means and variances")
//   Zhi, Zlo       split-TF32 planes: Zhi = tf32_rna(Z), Zlo = tf32_rna(Z - Zhi)
//   Zb             bf16_rn(Z): the screening pass of the exhaustive Pearson GEMM
//   S, perm        row sorted ascending (+inf pad) and its argsort (uint16)
//   cflag          constant series (min == max) -> NaN correlations (reading R10)
// All kernels are HBM-bound; DESIGN.md lists their algorithmic bytes.
#include <math.h>
#include <stdlib.h>

#include <cuda_bf16.h>

#include <cub/block/block_radix_sort.cuh>

#include "corr_internal.cuh"
#include "ksg_common.cuh"

namespace corr {
namespace {

// ---- 1. transpose [n][P] -> F[P][n_pad] through a 32x32 shared tile -----------
// `in` holds members [m0, m1) of the member-major input ([m1-m0][P]); the kernel writes columns
// [m0, m0 + mw) of F (mw extends to n_pad on the last slice: pad columns are written as 0), so the
// host path can stream the input in member slices and transpose each as soon as it lands.
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ in, float* __restrict__ F,
                                                        int m0, int m1, int mw, int n_pad, int64_t P, int* err) {
  __shared__ float tile[32][33];
  const int64_t p0 = (int64_t)blockIdx.x * 32;
  const int mb = m0 + blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  bool bad = false;
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int m = mb + ty + r;
    const int64_t p = p0 + tx;
    float v = 0.f;
    if (m < m1 && p < P) {
      v = in[(int64_t)(m - m0) * P + p];
      bad |= !isfinite(v);
    }
    tile[ty + r][tx] = v;
  }
  if (bad) atomicOr(err, 2);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 32; r += 8) {
    const int64_t p = p0 + ty + r;
    const int m = mb + tx;
    if (p < P && m < m0 + mw) F[p * n_pad + m] = tile[tx][ty + r];
  }
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- 2. per-point statistics, standardisation, tf32 split (one warp per row) ---
__global__ void __launch_bounds__(256) stats_kernel(const float* __restrict__ F, float* __restrict__ Z,
                                                    float* __restrict__ Zhi, float* __restrict__ Zlo,
                                                    uint16_t* __restrict__ Zb,
                                                    uint8_t* __restrict__ cflag, float* __restrict__ spread,
                                                    int n, int n_pad, int64_t P) {
  const int lane = threadIdx.x & 31;
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (p >= P) return;
  const float* row = F + p * n_pad;
  double s = 0.0;
  float mn = INFINITY, mx = -INFINITY;
  for (int e = lane; e < n; e += 32) {
    const float v = row[e];
    s += (double)v;
    mn = fminf(mn, v);
    mx = fmaxf(mx, v);
  }
  s = warp_sum(s);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const double mean = s / (double)n;
  double ss = 0.0;
  for (int e = lane; e < n; e += 32) {
    const double d = (double)row[e] - mean;
    ss += d * d;
  }
  ss = warp_sum(ss);
  const bool constant = (mn == mx);
  const double inv = constant ? 0.0 : 1.0 / sqrt(ss);
  for (int e = lane; e < n_pad; e += 32) {
    float z = 0.f;
    if (e < n && !constant) z = (float)(((double)row[e] - mean) * inv);
    const float hi = tf32_rna(z);
    const float lo = tf32_rna(z - hi);
    Z[p * n_pad + e] = z;
    Zhi[p * n_pad + e] = hi;
    Zlo[p * n_pad + e] = lo;
    Zb[p * n_pad + e] = __bfloat16_as_ushort(__float2bfloat16_rn(z));
  }
  if (lane == 0) {
    cflag[p] = constant ? 1 : 0;
    spread[p] = constant ? 0.f : (float)sqrt(ss);
  }
}

// ---- 3. per-row bitonic sort with argsort (shared memory) ----------------------
// A group of N2/2 threads sorts one row of N2 = next_pow2(n) (value, index) pairs.
__global__ void __launch_bounds__(512) sort_kernel(const float* __restrict__ F, float* __restrict__ S,
                                                   uint16_t* __restrict__ perm, int n, int n_pad,
                                                   int64_t P, int log2n2) {
  extern __shared__ unsigned char smem_raw[];
  const int N2 = 1 << log2n2;
  const int tpr = min(N2 >> 1, 512);                 // threads per row
  const int rows_per_block = blockDim.x / tpr;
  const int g = threadIdx.x / tpr, t = threadIdx.x % tpr;
  float* sv = reinterpret_cast<float*>(smem_raw) + g * N2;
  uint16_t* si = reinterpret_cast<uint16_t*>(reinterpret_cast<float*>(smem_raw) + rows_per_block * N2) + g * N2;
  const int64_t p = (int64_t)blockIdx.x * rows_per_block + g;
  const bool live = p < P;
  for (int e = t; e < N2; e += tpr) {
    sv[e] = (live && e < n) ? F[p * n_pad + e] : INFINITY;
    si[e] = (uint16_t)(e < n ? e : 0xFFFF);
  }
  __syncthreads();
  for (int size = 2; size <= N2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int c = t; c < (N2 >> 1); c += tpr) {
        const int lo = 2 * c - (c & (stride - 1));
        const int hi = lo + stride;
        const bool asc = (lo & size) == 0;
        const float a = sv[lo], b = sv[hi];
        if ((a > b) == asc) {
          sv[lo] = b; sv[hi] = a;
          const uint16_t ia = si[lo];
          si[lo] = si[hi]; si[hi] = ia;
        }
      }
      __syncthreads();
    }
  }
  if (live) {
    for (int e = t; e < n_pad; e += tpr) {
      S[p * n_pad + e] = e < n ? sv[e] : INFINITY;
      perm[p * n_pad + e] = e < n ? si[e] : (uint16_t)0xFFFF;
    }
  }
}

// ---- 3b. per-row radix sort (one CTA of T threads x I items per row, N2 = T*I) ------
// The bitonic network above costs log2(N2)(log2(N2)+1)/2 shared-memory passes with a
// barrier each (55 at n = 1000); an LSD radix sort of order-preserving u32 keys needs at
// most 8 4-bit passes.  Keys: u = bits(f); u ^= (u >> 31 ? 0xFFFFFFFF : 0x80000000) (finite
// inputs, checked at ingest), so u32 order == float order (-0 before +0; equal floats
// compare equal in every consumer, and KSG only needs SOME sorted permutation, R4).
// Only the key bits that vary within the row are sorted: all keys lie in [kmin, kmax], so
// they share every bit above the highest bit where kmin and kmax differ (ensemble rows share
// sign, exponent and leading mantissa bits: typically 5 passes instead of 8).  The row is
// loaded BLOCKED (thread t holds members t*I .. t*I+I-1), the padding slots e >= n get key kmax
// and sit at the highest blocked positions, so the stable sort leaves them last.  Values: the
// member index.  Output is written striped (coalesced).
template <int T, int I>
__global__ void __launch_bounds__(T) sort_radix_kernel(const float* __restrict__ F, float* __restrict__ S,
                                                       uint16_t* __restrict__ perm, int n, int n_pad, int64_t P) {
  using Sorter = cub::BlockRadixSort<uint32_t, T, I, uint16_t>;
  __shared__ typename Sorter::TempStorage tmp;
  __shared__ uint32_t kext[2];  // min and max key of the row
  for (int64_t p = blockIdx.x; p < P; p += gridDim.x) {
    const float* row = F + p * n_pad;
    uint32_t key[I];
    uint16_t idx[I];
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const int e = (int)threadIdx.x * I + i;
      uint32_t u = 0u;
      if (e < n) {
        u = __float_as_uint(row[e]);
        u ^= (u >> 31) ? 0xFFFFFFFFu : 0x80000000u;
        kmin = min(kmin, u);
        kmax = max(kmax, u);
      }
      key[i] = u;
      idx[i] = (uint16_t)(e < n ? e : 0xFFFF);
    }
    if (threadIdx.x == 0) {
      kext[0] = 0xFFFFFFFFu;
      kext[1] = 0u;
    }
    __syncthreads();
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&kext[0], kmin);
      atomicMax(&kext[1], kmax);
    }
    __syncthreads();
    kmin = kext[0];
    kmax = kext[1];
#pragma unroll
    for (int i = 0; i < I; ++i)
      if ((int)threadIdx.x * I + i >= n) key[i] = kmax;
    const uint32_t diff = kmin ^ kmax;
    const int end_bit = diff ? 32 - __clz(diff) : 1;  // a constant row still goes through one pass
    Sorter(tmp).SortBlockedToStriped(key, idx, 0, end_bit);
#pragma unroll
    for (int i = 0; i < I; ++i) {
      const int e = i * T + (int)threadIdx.x;
      if (e < n_pad) {
        uint32_t u = key[i];
        u ^= (u >> 31) ? 0x80000000u : 0xFFFFFFFFu;
        S[p * n_pad + e] = e < n ? __uint_as_float(u) : INFINITY;
        perm[p * n_pad + e] = e < n ? idx[i] : (uint16_t)0xFFFF;
      }
    }
    __syncthreads();  // tmp / kext are reused by the next row
  }
}

// ---- 3c. per-row bucket sort (one CTA per row at a time, persistent over rows) ---------------
// The radix sort above needs ~5 ranked passes per row; ensemble rows are smooth distributions,
// so one pass of BUCKETING plus tiny per-bucket sorts does the same job: keys u (order-preserving
// u32, as above) map to NB buckets by b = floor((u - kmin) * NB / (kmax - kmin + 1)) computed in
// fp32 -- a monotone non-decreasing map (monotone rounding), so bucket order is key order -- with
// a shared-memory histogram whose atomic return value is the slot inside the bucket; after an
// exclusive scan the row is scattered by bucket and every key's final position is its bucket
// start plus its rank inside the bucket (about n/NB <= 0.5 keys per bucket).  Equal keys may land in any order: consumers only need SOME sorted
// permutation (R4).  Rows whose largest bucket exceeds kMaxBucket (heavy outliers stretching the
// range) are sorted by a block bitonic network instead, so no row costs O(n^2).
constexpr int kMaxBucket = 48;

__device__ __forceinline__ uint32_t ord_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return u ^ ((u >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t u) {
  return __uint_as_float(u ^ ((u >> 31) ? 0x80000000u : 0xFFFFFFFFu));
}

// Persistent CTAs of TPB threads, one row at a time; the TMA unit stages the NEXT row
// (cp.async.bulk of n_pad floats on an mbarrier) while the current one is bucketed.  Keys stay
// in registers (N2 / TPB per thread); bucket counters are laid out so the scan's loads are
// conflict-free; the sorted row and argsort leave through 16-byte stores.  Measured at C4
// (n = 1000): 15.3 -> 14.5 ms per re-ingest sort with 128 threads per row; 256 threads cost more
// (the per-warp reductions and scans are duplicated per warp; ncu: 6.7k warp-instructions per
// row, issue 53 %), 64 threads starve the SM (28 KB of shared memory per CTA).
template <int NB, int N2, int TPB>
__global__ void __launch_bounds__(TPB) sort_bucket_kernel(const float* __restrict__ F, float* __restrict__ S,
                                                          uint16_t* __restrict__ perm, int n, int n_pad, int64_t P) {
  constexpr int PT = N2 / TPB;   // keys per thread
  constexpr int NWARP = TPB / 32;
  constexpr int PER = NB / TPB;  // bucket counters per thread in the scan
  // bucket b's counter lives at (b % PER) * TPB + b / PER: thread t scans buckets t*PER ..
  // t*PER + PER-1 with conflict-free loads (bucket NB -> NB, the end sentinel)
  auto cidx = [](int b) { return b >= NB ? NB : (b % PER) * TPB + b / PER; };
  __shared__ __align__(16) float buf[2][N2];  // staged rows (double buffer)
  __shared__ uint32_t key[N2];                // bucketed keys (then, on the fallback, the bitonic array)
  __shared__ uint16_t idx[N2];
  __shared__ __align__(16) float sv[N2];      // the sorted row
  __shared__ __align__(16) uint16_t si[N2];   // its argsort
  __shared__ int cnt[NB + 1];
  __shared__ uint32_t red[NWARP][2];
  __shared__ int maxb;
  __shared__ uint64_t bar[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t row_bytes = (uint32_t)n_pad * 4u;  // n_pad % 8 == 0: a multiple of 16 bytes
  if (tid == 0) {
    bar_init(bar);
    bar_init(bar + 1);
    if ((int64_t)blockIdx.x < P) {
      bar_expect(bar, row_bytes);
      bulk_g2s(buf[0], F + (int64_t)blockIdx.x * n_pad, row_bytes, bar);
    }
  }
  __syncthreads();
  uint32_t it = 0;
  for (int64_t p = blockIdx.x; p < P; p += gridDim.x, ++it) {
    const int b = it & 1;
    if (tid == 0 && p + gridDim.x < P) {  // buf[b ^ 1] was released by the previous row's last barrier
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_expect(bar + (b ^ 1), row_bytes);
      bulk_g2s(buf[b ^ 1], F + (p + gridDim.x) * n_pad, row_bytes, bar + (b ^ 1));
    }
    for (int q = tid; q <= NB; q += TPB) cnt[q] = 0;
    if (tid == 0) maxb = 0;
    bar_wait(bar + b, (it >> 1) & 1u);
    uint32_t u[PT];
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      const int e = tid + i * TPB;
      u[i] = ord_key(buf[b][e < n ? e : 0]);
      if (e < n) {
        kmin = min(kmin, u[i]);
        kmax = max(kmax, u[i]);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) {
      red[warp][0] = kmin;
      red[warp][1] = kmax;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < NWARP; ++w) {
      kmin = min(kmin, red[w][0]);
      kmax = max(kmax, red[w][1]);
    }
    const float scale = (float)NB / ((float)(kmax - kmin) + 1.0f);
    // histogram: the atomic's return value is the key's slot inside its bucket
    int slot[PT], bk[PT];
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      const int e = tid + i * TPB;
      if (e < n) {
        const int bb = min(NB - 1, (int)((float)(u[i] - kmin) * scale));
        bk[i] = bb;
        slot[i] = atomicAdd(&cnt[cidx(bb)], 1);
      }
    }
    __syncthreads();
    // exclusive scan of the NB counters (each thread NB/TPB consecutive ones), largest bucket
    int loc[PER], sum = 0, mb = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      loc[i] = cnt[i * TPB + tid];
      mb = max(mb, loc[i]);
      sum += loc[i];
    }
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
    if (lane == 31) red[warp][0] = (uint32_t)incl;
    if (lane == 0) atomicMax(&maxb, mb);
    __syncthreads();
    int base = incl - sum;
    for (int w = 0; w < warp; ++w) base += (int)red[w][0];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      cnt[i * TPB + tid] = base;
      base += loc[i];
    }
    if (tid == TPB - 1) cnt[NB] = n;
    __syncthreads();
    const bool fallback = maxb > kMaxBucket;
    if (!fallback) {
#pragma unroll
      for (int i = 0; i < PT; ++i) {
        const int e = tid + i * TPB;
        if (e < n) {
          const int q = cnt[cidx(bk[i])] + slot[i];
          key[q] = u[i];
        }
      }
      __syncthreads();
      // final position of each key: its bucket's start + its rank inside the bucket (smaller keys,
      // then equal keys at lower slots) -- independent per key, no sequential insertion
#pragma unroll
      for (int i = 0; i < PT; ++i) {
        const int e = tid + i * TPB;
        if (e < n) {
          const int lo = cnt[cidx(bk[i])], hi = cnt[cidx(bk[i] + 1)], q = lo + slot[i];
          const uint32_t kv = u[i];
          int rank = 0;
          for (int j = lo; j < hi; ++j) {
            const uint32_t kj = key[j];
            rank += (kj < kv || (kj == kv && j < q)) ? 1 : 0;
          }
          sv[lo + rank] = key_float(kv);
          si[lo + rank] = (uint16_t)e;
        }
      }
    } else {
      // a stretched row: block bitonic network over N2 slots (+inf-key padding sorts last)
#pragma unroll
      for (int i = 0; i < PT; ++i) {
        const int e = tid + i * TPB;
        key[e] = e < n ? u[i] : 0xFFFFFFFFu;
        idx[e] = (uint16_t)(e < n ? e : 0xFFFF);
      }
      __syncthreads();
      for (int size = 2; size <= N2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
          for (int c = tid; c < (N2 >> 1); c += TPB) {
            const int lo = 2 * c - (c & (stride - 1));
            const int hi = lo + stride;
            const bool asc = (lo & size) == 0;
            const uint32_t a = key[lo], bv = key[hi];
            if ((a > bv) == asc) {
              key[lo] = bv;
              key[hi] = a;
              const uint16_t t = idx[lo];
              idx[lo] = idx[hi];
              idx[hi] = t;
            }
          }
          __syncthreads();
        }
      }
      for (int e = tid; e < n; e += TPB) {
        sv[e] = key_float(key[e]);
        si[e] = idx[e];
      }
    }
    for (int e = n + tid; e < n_pad; e += TPB) {  // pad: +inf, index 0xFFFF
      sv[e] = INFINITY;
      si[e] = (uint16_t)0xFFFF;
    }
    __syncthreads();
    float4* S4 = reinterpret_cast<float4*>(S + p * n_pad);
    for (int q = tid; q < (n_pad >> 2); q += TPB) S4[q] = reinterpret_cast<const float4*>(sv)[q];
    uint4* P8 = reinterpret_cast<uint4*>(perm + p * n_pad);
    for (int q = tid; q < (n_pad >> 3); q += TPB) P8[q] = reinterpret_cast<const uint4*>(si)[q];
    __syncthreads();  // smem (and buf[b]) reused by the next rows
  }
}

template <int NB, int N2, int TPB>
cudaError_t launch_sort_bucket(corr_field* f, cudaStream_t st) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sort_bucket_kernel<NB, N2, TPB>, TPB, 0);
  if (occ < 1) occ = 1;
  int64_t blocks = (int64_t)kSMs * occ;  // persistent: one wave, each CTA streams its rows
  if (blocks > f->P) blocks = f->P;
  sort_bucket_kernel<NB, N2, TPB><<<(unsigned)blocks, TPB, 0, st>>>(f->F, f->S, f->perm, f->n, f->n_pad, f->P);
  return cudaSuccess;
}

template <int T, int I>
cudaError_t launch_sort_radix(corr_field* f, cudaStream_t st) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sort_radix_kernel<T, I>, T, 0);
  if (occ < 1) occ = 1;
  int64_t blocks = (int64_t)kSMs * occ * 8;
  if (blocks > f->P) blocks = f->P;
  sort_radix_kernel<T, I><<<(unsigned)blocks, T, 0, st>>>(f->F, f->S, f->perm, f->n, f->n_pad, f->P);
  return cudaSuccess;
}

// ---- 4. mean-tree level (§3.3): per-member block means ----------
// One warp per coarse point; lanes stride over members, so every fine row is read with
// coalesced loads and the coarse row is written contiguously.  fp64 sums, fp32 means; a
// boundary block averages the fine points that exist (SPEC.md:59 voxel-count weighting).
__global__ void __launch_bounds__(256) aggregate_kernel(const float* __restrict__ F, float* __restrict__ G,
                                                        int nx, int ny, int nz, int cx, int cy, int cz, int fx,
                                                        int fy, int fz, int n, int n_pad) {
  const int lane = threadIdx.x & 31;
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (q >= (int64_t)cx * cy * cz) return;
  const int X = (int)(q % cx), Y = (int)((q / cx) % cy), Z = (int)(q / ((int64_t)cx * cy));
  const int x0 = X * fx, y0 = Y * fy, z0 = Z * fz;
  const int x1 = min(nx, x0 + fx), y1 = min(ny, y0 + fy), z1 = min(nz, z0 + fz);
  const double cnt = (double)((x1 - x0) * (y1 - y0) * (z1 - z0));
  for (int e = lane; e < n_pad; e += 32) {
    float out = 0.f;
    if (e < n) {
      double s = 0.0;
      for (int z = z0; z < z1; ++z)
        for (int y = y0; y < y1; ++y)
          for (int x = x0; x < x1; ++x) s += (double)F[(((int64_t)z * ny + y) * nx + x) * n_pad + e];
      out = (float)(s / cnt);
    }
    G[q * n_pad + e] = out;
  }
}

}  // namespace

cudaError_t launch_field_aggregate(const corr_field* src, corr_field* dst, int fx, int fy, int fz, cudaStream_t st) {
  const int64_t threads = dst->P * 32;
  aggregate_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(src->F, dst->F, src->nx, src->ny, src->nz,
                                                                     dst->nx, dst->ny, dst->nz, fx, fy, fz, src->n,
                                                                     src->n_pad);
  note_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_field_ingest(dst, nullptr, st);
}

// Transposes members [m0, m1) of the member-major input (din = that slice, [m1-m0][P]) into F.
cudaError_t launch_transpose_slice(corr_field* f, const float* din, int m0, int m1, cudaStream_t st) {
  const int mw = (m1 >= f->n ? f->n_pad : m1) - m0;
  dim3 grid((unsigned)((f->P + 31) / 32), (unsigned)((mw + 31) / 32));
  transpose_kernel<<<grid, 256, 0, st>>>(din, f->F, m0, m1, mw, f->n_pad, f->P, f->err + 1);
  note_launch();
  return cudaGetLastError();
}

// din == nullptr: F is already filled (aggregate levels, or a streamed host upload); else
// transpose din [n][P] into F.  Then the derived buffers (stats, tf32/bf16 planes, sorted rows).
cudaError_t launch_field_ingest(corr_field* f, const float* din, cudaStream_t st) {
  const int64_t P = f->P;
  if (din) {
    const cudaError_t e = launch_transpose_slice(f, din, 0, f->n, st);
    if (e != cudaSuccess) return e;
  }
  {
    const int64_t threads = P * 32;
    stats_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(f->F, f->Z, f->Zhi, f->Zlo, f->Zb, f->cflag,
                                                                   f->spread, f->n, f->n_pad, P);
  }
  {
    int log2n2 = 1;
    while ((1 << log2n2) < f->n) ++log2n2;
    const int N2 = 1 << log2n2;
    cudaError_t er = cudaErrorInvalidValue;
    static const bool radix = [] {  // A/B switch: the round-1 CUB radix sort
      const char* v = getenv("CORR_SORT_RADIX");
      return v && v[0] == '1';
    }();
    if (radix || N2 > 1024) {  // n > 1024: the radix sort (the bucket kernel's static smem is for n <= 1024)
      switch (N2) {
        case 64: er = launch_sort_radix<32, 2>(f, st); break;
        case 128: er = launch_sort_radix<32, 4>(f, st); break;
        case 256: er = launch_sort_radix<64, 4>(f, st); break;
        case 512: er = launch_sort_radix<64, 8>(f, st); break;
        case 1024: er = launch_sort_radix<64, 16>(f, st); break;
        case 2048: er = launch_sort_radix<256, 8>(f, st); break;
        case 4096: er = launch_sort_radix<256, 16>(f, st); break;
        default: break;
      }
    } else {
      switch (N2) {  // NB = 2 N2 buckets: about 0.5 keys per bucket, so the per-bucket sorts stay short
        case 64:
        case 128:
        case 256: er = launch_sort_bucket<512, 256, 128>(f, st); break;
        case 512: er = launch_sort_bucket<1024, 512, 128>(f, st); break;
        case 1024: {
          static const int tpb = [] {  // A/B switch: threads per row
            const char* v = getenv("CORR_SORT_TPB");
            return v ? atoi(v) : 128;
          }();
          er = tpb == 256 ? launch_sort_bucket<2048, 1024, 256>(f, st)
               : tpb == 64 ? launch_sort_bucket<2048, 1024, 64>(f, st)
                           : launch_sort_bucket<2048, 1024, 128>(f, st);
          break;
        }
        default: break;
      }
    }
    if (er == cudaSuccess) {
      note_launch(2);
      return cudaGetLastError();
    }
    const int tpr = N2 / 2 < 512 ? N2 / 2 : 512;
    int threads = 512;
    if (threads < tpr) threads = tpr;
    const int rows_per_block = threads / tpr;
    const size_t smem = (size_t)rows_per_block * N2 * (sizeof(float) + sizeof(uint16_t));
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    const int64_t blocks = (P + rows_per_block - 1) / rows_per_block;
    sort_kernel<<<(unsigned)blocks, threads, smem, st>>>(f->F, f->S, f->perm, f->n, f->n_pad, P, log2n2);
  }
  note_launch(2);
  return cudaGetLastError();
}

}  // namespace corr
