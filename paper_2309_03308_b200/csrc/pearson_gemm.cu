// pearson_gemm.cu -- exhaustive Pearson region-pair maximum as a tcgen05 GEMM,
// SURVEY.md §8(a) row a7 (+ a9).
//
// PAPER.md:133 (§3): the region-pair indicator is the maximum point-pair correlation of
// two bricks; PAPER.md:45 and :498 note that all point pairs take ">2 days" / "365 days"
// on the paper's GPU.  With the series standardised in fp64 (field.cu), every Pearson
// value of a brick pair is one entry of C = Z_A . Z_B^T (|A| x |B|, K = n), a dense
// contraction that belongs on the 5th-gen tensor cores.  fp32 tolerance (1e-5) is kept
// with split-TF32: Z = Z_hi + Z_lo (both tf32) and
//     C ~= Z_hi Z_hi^T + Z_hi Z_lo^T + Z_lo Z_hi^T          (3 tcgen05.mma per k-step)
// (the dropped Z_lo Z_lo^T term is ~2^-22 relative).  C is never written to memory: the
// epilogue reduces each 128x256 accumulator tile straight out of TMEM to one packed
// (value, lowest q) key per thread and a u64 atomicMax per warp (reading R16).
//
// Kernel shape (one CTA per SM, persistent over the tiles of all region pairs):
//   warp 0      TMA producer: 4 tensor-map loads per k-block (A_hi, A_lo, B_hi, B_lo),
//               K-major, 128-byte swizzle, boxes of 32 members x (points of a brick slab)
//   warp 1      TMEM owner + single-thread MMA issuer, kind::tf32, M=128 N=256 K=8
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 -> column mask (region / constant /
//               self pair) -> per-32-column FMNMX max -> first index of the max ->
//               (value, q) key -> warp max -> atomicMax
//   TMEM: 2 accumulators x 256 columns (double-buffered so the epilogue of tile t
//   overlaps the MMAs of tile t+1); smem: 2 stages x 96 KB.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "sampler.cuh"

namespace corr {
namespace {

constexpr int BM = 128, BN = 256, BK = 32, STAGES = 2;
constexpr int A_BYTES = BM * BK * 4;  // 16 KB per plane
constexpr int B_BYTES = BN * BK * 4;  // 32 KB per plane
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 512;

struct GemmRegion {
  corr_box A, B;
  int ntA[3], ntB[3];  // tiles along x, y, z
  int64_t tile_off;    // prefix of mt*nt
  int64_t nA, nB;
  int overlap;         // one field and the boxes intersect -> self-pair mask needed
  int pad;
  int64_t pair_off;    // prefix of ceil(nta/2)*ntb tile pairs (multicast screen)
};

struct GemmGeom {
  int bxA, byA, bzA, bxB, byB, bzB;
  int nx, ny;
  int kblocks;
  int absval;
  int same_field;
  int64_t nreg;
  int64_t total_tiles;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void tc_mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// K-major operand, 128-byte swizzle atoms of 8 rows x 128 B (SBO = 1024 B), sm_100 version 1
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// instruction descriptor: D=f32, A=B=tf32, K-major both, N=256, M=128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
// D=f32, A=B=bf16 (kind::f16), K-major both, N=256, M=128 -- the screening pass
constexpr uint32_t kIdescBF16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct TileCoord {
  int64_t r;
  int tx, ty, tz, ux, uy, uz;  // A tile (tx,ty,tz), B tile (ux,uy,uz)
};

__device__ __forceinline__ TileCoord tile_coord(const GemmRegion* __restrict__ reg, int64_t nreg, int64_t t) {
  int64_t lo = 0, hi = nreg - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (reg[mid].tile_off <= t) lo = mid; else hi = mid - 1;
  }
  const GemmRegion& R = reg[lo];
  int64_t q = t - R.tile_off;
  const int64_t ntB = (int64_t)R.ntB[0] * R.ntB[1] * R.ntB[2];
  const int64_t mi = q / ntB, ni = q - mi * ntB;
  TileCoord c;
  c.r = lo;
  c.tx = (int)(mi % R.ntA[0]);
  c.ty = (int)((mi / R.ntA[0]) % R.ntA[1]);
  c.tz = (int)(mi / ((int64_t)R.ntA[0] * R.ntA[1]));
  c.ux = (int)(ni % R.ntB[0]);
  c.uy = (int)((ni / R.ntB[0]) % R.ntB[1]);
  c.uz = (int)(ni / ((int64_t)R.ntB[0] * R.ntB[1]));
  return c;
}

// Order-preserving u32 of a float (0 is reserved for "no value"; every real key is > 0).
__device__ __forceinline__ uint32_t ord32(float v) {
  uint32_t u = __float_as_uint(v + 0.0f);
  return u ^ ((u >> 31) ? 0xFFFFFFFFu : 0x80000000u);
}
__device__ __forceinline__ float unord32(uint32_t u) {
  return __uint_as_float(u ^ ((u >> 31) ? 0x80000000u : 0xFFFFFFFFu));
}

// SCREEN = true: the hi*hi product only (1 of the 3 MMAs, half the operand bytes); the epilogue
// records each tile's masked maximum (tile_keys[t]) and each region pair's (reg_keys[r]).
// SCREEN = false: the full split-TF32 product with the max/argmax epilogue, over the tile list
// tlist[0 .. *tcount) (or every tile when tlist == nullptr).
// SCREEN with BF16: the screening maps are bf16 planes (64 members per 128-byte k-block row, one
// kind::f16 MMA per 16 members) -- twice the members per k-block, half the operand bytes.
template <bool SCREEN, bool BF16 = false>
__global__ void __launch_bounds__(kThreads, 1)
    pearson_block_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                         const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                         const GemmRegion* __restrict__ reg, GemmGeom g, const uint8_t* __restrict__ ca,
                         const uint8_t* __restrict__ cb, unsigned long long* __restrict__ keys,
                         const int* __restrict__ tlist, const int* __restrict__ tcount,
                         uint32_t* __restrict__ tile_keys, uint32_t* __restrict__ reg_keys) {
  const int64_t ntiles = tlist ? (int64_t)*tcount : g.total_tiles;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-align the operand stages (128-byte swizzle atoms)
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* stage_base = base;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* colbias = reinterpret_cast<float*>(tmem_slot + 4);  // [2][BN]
  int* colpt = reinterpret_cast<int*>(colbias + 2 * BN);      // [2][BN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mAhi) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mAlo) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mBhi) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mBlo) : "memory");
      uint32_t it = 0;
      for (int64_t i = blockIdx.x; i < ntiles; i += gridDim.x) {
        const int64_t t = tlist ? (int64_t)tlist[i] : i;
        const TileCoord c = tile_coord(reg, g.nreg, t);
        const GemmRegion& R = reg[c.r];
        const int ax = R.A.x0 + c.tx * g.bxA, ay = R.A.y0 + c.ty * g.byA, az = R.A.z0 + c.tz * g.bzA;
        const int bx = R.B.x0 + c.ux * g.bxB, by = R.B.y0 + c.uy * g.byB, bz = R.B.z0 + c.uz * g.bzB;
        for (int kb = 0; kb < g.kblocks; ++kb, ++it) {
          const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
          mbar_wait(empty + s, ph ^ 1);
          unsigned char* st = stage_base + s * STAGE_BYTES;
          mbar_expect_tx(full + s, SCREEN ? A_BYTES + B_BYTES : STAGE_BYTES);
          const int k0 = kb * (BF16 ? 2 * BK : BK);  // members per k-block: 32 tf32 or 64 bf16 (128 B)
          tma_load_4d(st, &mAhi, full + s, k0, ax, ay, az);
          if (!SCREEN) tma_load_4d(st + A_BYTES, &mAlo, full + s, kb * BK, ax, ay, az);
          tma_load_4d(st + 2 * A_BYTES, &mBhi, full + s, k0, bx, by, bz);
          if (!SCREEN) tma_load_4d(st + 2 * A_BYTES + B_BYTES, &mBlo, full + s, kb * BK, bx, by, bz);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    uint32_t it = 0, tt = 0;
    for (int64_t i = blockIdx.x; i < ntiles; i += gridDim.x, ++tt) {
      const uint32_t acc = tt & 1, aph = (tt >> 1) & 1;
      mbar_wait(tempty + acc, aph ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem_base + acc * BN;
      for (int kb = 0; kb < g.kblocks; ++kb, ++it) {
        const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
        mbar_wait(full + s, ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t st = smem_u32(stage_base + s * STAGE_BYTES);
          const uint64_t dAhi = sdesc_sw128(st), dAlo = sdesc_sw128(st + A_BYTES);
          const uint64_t dBhi = sdesc_sw128(st + 2 * A_BYTES), dBlo = sdesc_sw128(st + 2 * A_BYTES + B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 tf32 = 32 bytes inside the swizzle atom
            const uint32_t first = (kb == 0 && kk == 0) ? 0u : 1u;
            if (BF16) tc_mma_bf16(dcol, dAhi + adv, dBhi + adv, kIdescBF16, first);
            else tc_mma_tf32(dcol, dAhi + adv, dBhi + adv, kIdesc, first);
            if (!SCREEN) {
              tc_mma_tf32(dcol, dAhi + adv, dBlo + adv, kIdesc, 1u);
              tc_mma_tf32(dcol, dAlo + adv, dBhi + adv, kIdesc, 1u);
            }
          }
          tc_commit(empty + s);  // smem stage free once these MMAs have read it
        }
        __syncwarp();
      }
      if (lane == 0) tc_commit(tfull + acc);  // accumulator complete
      __syncwarp();
    }
  } else {
    // ===================== epilogue (warps 2..5) =====================
    const int q4 = warp & 3;               // TMEM lane quarter this warp may access
    const int row = q4 * 32 + lane;        // accumulator row = A point of the tile
    const int et = threadIdx.x - 64;       // 0..127
    uint32_t tt = 0;
    for (int64_t i = blockIdx.x; i < ntiles; i += gridDim.x, ++tt) {
      const int64_t t = tlist ? (int64_t)tlist[i] : i;
      const uint32_t acc = tt & 1, aph = (tt >> 1) & 1;
      const TileCoord c = tile_coord(reg, g.nreg, t);
      const GemmRegion& R = reg[c.r];
      // per-tile column table (B points): bias 0 / -inf and point id (self-pair mask)
      float* cbias = colbias + acc * BN;
      int* cpt = colpt + acc * BN;
      for (int n = et; n < BN; n += 128) {
        const int lx = n % g.bxB, ly = (n / g.bxB) % g.byB, lz = n / (g.bxB * g.byB);
        const int x = R.B.x0 + c.ux * g.bxB + lx, y = R.B.y0 + c.uy * g.byB + ly, z = R.B.z0 + c.uz * g.bzB + lz;
        bool ok = x < R.B.x1 && y < R.B.y1 && z < R.B.z1;
        int p = -1;
        if (ok) {
          p = (z * g.ny + y) * g.nx + x;
          ok = cb[p] == 0;
        }
        cbias[n] = ok ? 0.f : -INFINITY;
        cpt[n] = p;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      // this thread's row (A point)
      const int lxA = row % g.bxA, lyA = (row / g.bxA) % g.byA, lzA = row / (g.bxA * g.byA);
      const int xa = R.A.x0 + c.tx * g.bxA + lxA, ya = R.A.y0 + c.ty * g.byA + lyA, za = R.A.z0 + c.tz * g.bzA + lzA;
      bool row_ok = xa < R.A.x1 && ya < R.A.y1 && za < R.A.z1;
      int pa = -1;
      if (row_ok) {
        pa = (za * g.ny + ya) * g.nx + xa;
        row_ok = ca[pa] == 0;
      }
      const bool selfmask = R.overlap != 0;
      mbar_wait(tfull + acc, aph);
      tc_fence_after();
      float best = -INFINITY;
      int bidx = 0;
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q4 * 32) << 16);
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        float v[32];
        tmem_ld32(taddr + ch * 32, v);
        const float4* b4 = reinterpret_cast<const float4*>(cbias + ch * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 bb = b4[i];
          v[4 * i + 0] = (g.absval ? fabsf(v[4 * i + 0]) : v[4 * i + 0]) + bb.x;
          v[4 * i + 1] = (g.absval ? fabsf(v[4 * i + 1]) : v[4 * i + 1]) + bb.y;
          v[4 * i + 2] = (g.absval ? fabsf(v[4 * i + 2]) : v[4 * i + 2]) + bb.z;
          v[4 * i + 3] = (g.absval ? fabsf(v[4 * i + 3]) : v[4 * i + 3]) + bb.w;
        }
        if (selfmask) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cpt[ch * 32 + i] == pa) v[i] = -INFINITY;
        }
        if (!SCREEN) {
          // clamp to [-1, 1] BEFORE the max / first-index search (masked entries stay -inf), so
          // split-TF32 values rounding above 1 tie at 1 and the lowest q wins (R16), as in the
          // sampled path
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = v[i] > -INFINITY ? fminf(1.f, fmaxf(-1.f, v[i])) : v[i];
        }
        float m = v[0];
#pragma unroll
        for (int i = 1; i < 32; ++i) m = fmaxf(m, v[i]);
        if (SCREEN) {
          best = fmaxf(best, m);
          continue;
        }
        if (m > best) {
          int j = 31;
#pragma unroll
          for (int i = 31; i >= 0; --i)
            if (v[i] == m) j = i;
          best = m;
          bidx = ch * 32 + j;
        }
      }
      // release the accumulator to the MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      if (SCREEN) {
        uint32_t k32 = (row_ok && best > -INFINITY) ? ord32(best) : 0u;
#pragma unroll
        for (int o = 16; o; o >>= 1) k32 = max(k32, __shfl_xor_sync(0xffffffffu, k32, o));
        if (lane == 0 && k32 != 0u) {
          atomicMax(tile_keys + t, k32);
          atomicMax(reg_keys + c.r, k32);
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        continue;
      }
      unsigned long long key = 0ULL;
      if (row_ok && best > -INFINITY) {
        best = fminf(1.f, fmaxf(-1.f, best));
        const int pb = cpt[bidx];
        const int xb = pb % g.nx, yb = (pb / g.nx) % g.ny, zb = pb / (g.nx * g.ny);
        const int64_t axs = R.A.x1 - R.A.x0, ays = R.A.y1 - R.A.y0;
        const int64_t bxs = R.B.x1 - R.B.x0, bys = R.B.y1 - R.B.y0;
        const int64_t al = ((int64_t)(za - R.A.z0) * ays + (ya - R.A.y0)) * axs + (xa - R.A.x0);
        const int64_t bl = ((int64_t)(zb - R.B.z0) * bys + (yb - R.B.y0)) * bxs + (xb - R.B.x0);
        key = pack_key(best, (uint32_t)(al * R.nB + bl));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
      }
      if (lane == 0 && key != 0ULL) atomicMax(keys + c.r, key);
      // the column table of this accumulator is rewritten two tiles later; all 4 warps
      // must be past it before then
      asm volatile("bar.sync 2, 128;" ::: "memory");
    }
  }
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ============================================================================
// 2-SM variant (cta_group::2): a cluster of two CTAs computes a 256 x 256 tile with one
// M=256 N=256 tcgen05.mma per k-step issued by the leader CTA.  Each CTA stages its own
// 128 A rows and its own 128 of the 256 B rows (the MMA reads the peer's halves at the same
// shared-memory offsets), so every SM moves 2/3 of the operand bytes of the 1-SM kernel for
// the same tensor work.  TMA completions of both CTAs land on the leader's full barrier
// (peer bit cleared); MMA commits multicast to both CTAs' empty / accumulator barriers; both
// epilogues release the leader's accumulator barrier.  Per CTA the epilogue is unchanged:
// its 128 TMEM lanes are its 128 A rows, the 256 columns span both CTAs' B halves.
// ============================================================================
constexpr int STAGES2 = 3;
constexpr int H_BYTES = 128 * BK * 4;            // one 128-row plane of one k-block: 16 KB
constexpr int STAGE2_BYTES = 4 * H_BYTES;        // A_hi, A_lo, B_hi, B_lo halves: 64 KB
constexpr uint32_t kIdesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);

struct Gemm2Region {
  corr_box A, B;
  int ntA[3], ntB[3];   // 128-row tiles along x, y, z
  int64_t nta, ntb;     // 128-row tiles per box
  int64_t tile_off;     // prefix of cluster tiles ceil(nta/2) * ceil(ntb/2)
  int64_t nA, nB;
  int overlap;
  int pad;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_4d_2sm(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                                int c2, int c3) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;  // peer bit cleared: the leader's barrier
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_2sm(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void tc_commit_2sm(uint64_t* bar) {
  const uint16_t mask = 0x3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tile_xyz(const int (&nt)[3], int64_t t, int& tx, int& ty, int& tz) {
  tx = (int)(t % nt[0]);
  ty = (int)((t / nt[0]) % nt[1]);
  tz = (int)(t / ((int64_t)nt[0] * nt[1]));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    pearson_block2_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                          const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo,
                          const Gemm2Region* __restrict__ reg, GemmGeom g, const uint8_t* __restrict__ ca,
                          const uint8_t* __restrict__ cb, unsigned long long* __restrict__ keys) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* stage_base = base;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES2 * STAGE2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* colbias = reinterpret_cast<float*>(tmem_slot + 4);  // [2][256]
  int* colpt = reinterpret_cast<int*>(colbias + 2 * BN);      // [2][256]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(full + s, 2);
      mbar_init(empty + s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto coord = [&](int64_t t, int64_t& r, int64_t& mi, int64_t& ni) {
    int64_t lo = 0, hi = g.nreg - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (reg[mid].tile_off <= t) lo = mid; else hi = mid - 1;
    }
    r = lo;
    const int64_t mb = (reg[lo].ntb + 1) >> 1;
    const int64_t q = t - reg[lo].tile_off;
    mi = q / mb;
    ni = q - mi * mb;
  };

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mAhi) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mAlo) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mBhi) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mBlo) : "memory");
      uint32_t it = 0;
      for (int64_t t = cid; t < g.total_tiles; t += ncl) {
        int64_t r, mi, ni;
        coord(t, r, mi, ni);
        const Gemm2Region& R = reg[r];
        int64_t ta = 2 * mi + rank, tb = 2 * ni + rank;
        if (ta >= R.nta) ta = R.nta - 1;  // odd tail: any valid tile, rows masked in the epilogue
        if (tb >= R.ntb) tb = R.ntb - 1;
        int tx, ty, tz, ux, uy, uz;
        tile_xyz(R.ntA, ta, tx, ty, tz);
        tile_xyz(R.ntB, tb, ux, uy, uz);
        const int ax = R.A.x0 + tx * g.bxA, ay = R.A.y0 + ty * g.byA, az = R.A.z0 + tz * g.bzA;
        const int bx = R.B.x0 + ux * g.bxB, by = R.B.y0 + uy * g.byB, bz = R.B.z0 + uz * g.bzB;
        for (int kb = 0; kb < g.kblocks; ++kb, ++it) {
          const uint32_t s = it % STAGES2, ph = (it / STAGES2) & 1;
          mbar_wait(empty + s, ph ^ 1);
          if (rank == 0) mbar_expect_tx(full + s, 2 * STAGE2_BYTES);
          else mbar_arrive_cluster(mapa_rank(smem_u32(full + s), 0));
          unsigned char* st = stage_base + s * STAGE2_BYTES;
          tma_load_4d_2sm(st, &mAhi, full + s, kb * BK, ax, ay, az);
          tma_load_4d_2sm(st + H_BYTES, &mAlo, full + s, kb * BK, ax, ay, az);
          tma_load_4d_2sm(st + 2 * H_BYTES, &mBhi, full + s, kb * BK, bx, by, bz);
          tma_load_4d_2sm(st + 3 * H_BYTES, &mBlo, full + s, kb * BK, bx, by, bz);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (rank == 0) {
      uint32_t it = 0, tt = 0;
      for (int64_t t = cid; t < g.total_tiles; t += ncl, ++tt) {
        const uint32_t acc = tt & 1, aph = (tt >> 1) & 1;
        mbar_wait(tempty + acc, aph ^ 1);
        tc_fence_after();
        const uint32_t dcol = tmem_base + acc * BN;
        for (int kb = 0; kb < g.kblocks; ++kb, ++it) {
          const uint32_t s = it % STAGES2, ph = (it / STAGES2) & 1;
          mbar_wait(full + s, ph);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t st = smem_u32(stage_base + s * STAGE2_BYTES);
            const uint64_t dAhi = sdesc_sw128(st), dAlo = sdesc_sw128(st + H_BYTES);
            const uint64_t dBhi = sdesc_sw128(st + 2 * H_BYTES), dBlo = sdesc_sw128(st + 3 * H_BYTES);
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t adv = (uint64_t)(kk * 32) >> 4;
              const uint32_t first = (kb == 0 && kk == 0) ? 0u : 1u;
              tc_mma_tf32_2sm(dcol, dAhi + adv, dBhi + adv, kIdesc2, first);
              tc_mma_tf32_2sm(dcol, dAhi + adv, dBlo + adv, kIdesc2, 1u);
              tc_mma_tf32_2sm(dcol, dAlo + adv, dBhi + adv, kIdesc2, 1u);
            }
            tc_commit_2sm(empty + s);
          }
          __syncwarp();
        }
        if (lane == 0) tc_commit_2sm(tfull + acc);
        __syncwarp();
      }
    }
  } else {
    // ===================== epilogue (warps 2..5 of both CTAs) =====================
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const int et = threadIdx.x - 64;
    const uint32_t tempty_leader = mapa_rank(smem_u32(tempty), 0);
    uint32_t tt = 0;
    for (int64_t t = cid; t < g.total_tiles; t += ncl, ++tt) {
      const uint32_t acc = tt & 1, aph = (tt >> 1) & 1;
      int64_t r, mi, ni;
      coord(t, r, mi, ni);
      const Gemm2Region& R = reg[r];
      float* cbias = colbias + acc * BN;
      int* cpt = colpt + acc * BN;
      for (int n = et; n < BN; n += 128) {
        const int h = n >> 7, nr = n & 127;
        const int64_t tb = 2 * ni + h;
        bool ok = tb < R.ntb;
        int p = -1;
        if (ok) {
          int ux, uy, uz;
          tile_xyz(R.ntB, tb, ux, uy, uz);
          const int lx = nr % g.bxB, ly = (nr / g.bxB) % g.byB, lz = nr / (g.bxB * g.byB);
          const int x = R.B.x0 + ux * g.bxB + lx, y = R.B.y0 + uy * g.byB + ly, z = R.B.z0 + uz * g.bzB + lz;
          ok = x < R.B.x1 && y < R.B.y1 && z < R.B.z1;
          if (ok) {
            p = (z * g.ny + y) * g.nx + x;
            ok = cb[p] == 0;
          }
        }
        cbias[n] = ok ? 0.f : -INFINITY;
        cpt[n] = p;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int64_t ta = 2 * mi + rank;
      bool row_ok = ta < R.nta;
      int xa = 0, ya = 0, za = 0, pa = -1;
      if (row_ok) {
        int tx, ty, tz;
        tile_xyz(R.ntA, ta, tx, ty, tz);
        const int lxA = row % g.bxA, lyA = (row / g.bxA) % g.byA, lzA = row / (g.bxA * g.byA);
        xa = R.A.x0 + tx * g.bxA + lxA;
        ya = R.A.y0 + ty * g.byA + lyA;
        za = R.A.z0 + tz * g.bzA + lzA;
        row_ok = xa < R.A.x1 && ya < R.A.y1 && za < R.A.z1;
        if (row_ok) {
          pa = (za * g.ny + ya) * g.nx + xa;
          row_ok = ca[pa] == 0;
        }
      }
      const bool selfmask = R.overlap != 0;
      mbar_wait(tfull + acc, aph);
      tc_fence_after();
      float best = -INFINITY;
      int bidx = 0;
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q4 * 32) << 16);
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        float v[32];
        tmem_ld32(taddr + ch * 32, v);
        const float4* b4 = reinterpret_cast<const float4*>(cbias + ch * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 bb = b4[i];
          v[4 * i + 0] = (g.absval ? fabsf(v[4 * i + 0]) : v[4 * i + 0]) + bb.x;
          v[4 * i + 1] = (g.absval ? fabsf(v[4 * i + 1]) : v[4 * i + 1]) + bb.y;
          v[4 * i + 2] = (g.absval ? fabsf(v[4 * i + 2]) : v[4 * i + 2]) + bb.z;
          v[4 * i + 3] = (g.absval ? fabsf(v[4 * i + 3]) : v[4 * i + 3]) + bb.w;
        }
        if (selfmask) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (cpt[ch * 32 + i] == pa) v[i] = -INFINITY;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = v[i] > -INFINITY ? fminf(1.f, fmaxf(-1.f, v[i])) : v[i];  // as above
        float m = v[0];
#pragma unroll
        for (int i = 1; i < 32; ++i) m = fmaxf(m, v[i]);
        if (m > best) {
          int j = 31;
#pragma unroll
          for (int i = 31; i >= 0; --i)
            if (v[i] == m) j = i;
          best = m;
          bidx = ch * 32 + j;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader + acc * 8);
      unsigned long long key = 0ULL;
      if (row_ok && best > -INFINITY) {
        best = fminf(1.f, fmaxf(-1.f, best));
        const int pb = cpt[bidx];
        const int xb = pb % g.nx, yb = (pb / g.nx) % g.ny, zb = pb / (g.nx * g.ny);
        const int64_t axs = R.A.x1 - R.A.x0, ays = R.A.y1 - R.A.y0;
        const int64_t bxs = R.B.x1 - R.B.x0, bys = R.B.y1 - R.B.y0;
        const int64_t al = ((int64_t)(za - R.A.z0) * ays + (ya - R.A.y0)) * axs + (xa - R.A.x0);
        const int64_t bl = ((int64_t)(zb - R.B.z0) * bys + (yb - R.B.y0)) * bxs + (xb - R.B.x0);
        key = pack_key(best, (uint32_t)(al * R.nB + bl));
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, key, o);
        key = other > key ? other : key;
      }
      if (lane == 0 && key != 0ULL) atomicMax(keys + r, key);
      asm volatile("bar.sync 2, 128;" ::: "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// ============================================================================
// Screening pass with B-tile multicast (cluster of 2 CTAs; session 3).  The bf16 screen moves
// 48 KB per k-block per SM (A 16 KB + B 32 KB) for 4 MMAs of 128x256x16: at the tensor pipe's
// rate that is ~170 GB/s of L2 -> SM traffic per SM, so the screen ran at ~0.5 of the bf16 peak.
// Here the two CTAs of a cluster take tiles (2i, n) and (2i+1, n) -- same B tile, adjacent A
// tiles -- and each loads HALF of the B tile with a multicast TMA into both CTAs' shared memory:
// 32 KB per k-block per SM.  Every CTA still runs the 1-SM MMA (M=128, N=256) on its own tile
// and writes the same per-tile / per-region keys as pearson_block_kernel<true, true>, so the
// tile selection and the exact pass are unchanged.  A stage is refilled only after BOTH CTAs'
// MMAs have read it (each MMA commit arrives on both CTAs' empty barriers, count 2).  An odd
// A-tile count gives the last pair's second CTA a duplicate of the first tile (max is idempotent).
// 4 stages of 48 KB.
// ============================================================================
constexpr int MC_STAGES = 4;
constexpr int MC_STAGE_BYTES = A_BYTES + B_BYTES;

__device__ __forceinline__ void tma_load_4d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                               int c3, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%2, "
      "%3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// (region, A tile, B tile) of tile pair tp; rank r takes A tile 2*mp + r (clamped)
__device__ __forceinline__ void mc_coord(const GemmRegion* __restrict__ reg, int64_t nreg, int64_t tp, uint32_t rank,
                                         int64_t& r, int64_t& t, TileCoord& c) {
  int64_t lo = 0, hi = nreg - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (reg[mid].pair_off <= tp) lo = mid; else hi = mid - 1;
  }
  const GemmRegion& R = reg[lo];
  const int64_t nta = (int64_t)R.ntA[0] * R.ntA[1] * R.ntA[2];
  const int64_t ntb = (int64_t)R.ntB[0] * R.ntB[1] * R.ntB[2];
  const int64_t q = tp - R.pair_off;
  const int64_t mp = q / ntb, ni = q - mp * ntb;
  int64_t mi = 2 * mp + rank;
  if (mi >= nta) mi = nta - 1;
  r = lo;
  t = R.tile_off + mi * ntb + ni;
  c.r = lo;
  c.tx = (int)(mi % R.ntA[0]);
  c.ty = (int)((mi / R.ntA[0]) % R.ntA[1]);
  c.tz = (int)(mi / ((int64_t)R.ntA[0] * R.ntA[1]));
  c.ux = (int)(ni % R.ntB[0]);
  c.uy = (int)((ni / R.ntB[0]) % R.ntB[1]);
  c.uz = (int)(ni / ((int64_t)R.ntB[0] * R.ntB[1]));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    pearson_screen_mc_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mBh,
                             const GemmRegion* __restrict__ reg, GemmGeom g, int64_t npairs, int bhy, int bhz,
                             const uint8_t* __restrict__ ca, const uint8_t* __restrict__ cb,
                             uint32_t* __restrict__ tile_keys, uint32_t* __restrict__ reg_keys) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  unsigned char* stage_base = base;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + MC_STAGES * MC_STAGE_BYTES);
  uint64_t* empty = full + MC_STAGES;
  uint64_t* tfull = empty + MC_STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* colbias = reinterpret_cast<float*>(tmem_slot + 4);  // [2][BN]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < MC_STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 2);  // both CTAs' MMAs must have read the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull + a, 1);
      mbar_init(tempty + a, 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mBh) : "memory");
      uint32_t it = 0;
      for (int64_t tp = cid; tp < npairs; tp += ncl) {
        int64_t r, t;
        TileCoord c;
        mc_coord(reg, g.nreg, tp, rank, r, t, c);
        const GemmRegion& R = reg[r];
        const int ax = R.A.x0 + c.tx * g.bxA, ay = R.A.y0 + c.ty * g.byA, az = R.A.z0 + c.tz * g.bzA;
        // this CTA's half of the B tile: rows [rank*128, rank*128+128) = the second half along y or z
        const int bx = R.B.x0 + c.ux * g.bxB, by = R.B.y0 + c.uy * g.byB + (int)rank * bhy,
                  bz = R.B.z0 + c.uz * g.bzB + (int)rank * bhz;
        for (int kb = 0; kb < g.kblocks; ++kb, ++it) {
          const uint32_t s = it % MC_STAGES, ph = (it / MC_STAGES) & 1;
          mbar_wait(empty + s, ph ^ 1);
          unsigned char* st = stage_base + s * MC_STAGE_BYTES;
          mbar_expect_tx(full + s, MC_STAGE_BYTES);
          const int k0 = kb * 2 * BK;  // 64 bf16 members per k-block
          tma_load_4d(st, &mA, full + s, k0, ax, ay, az);
          tma_load_4d_mc(st + A_BYTES + rank * (B_BYTES / 2), &mBh, full + s, k0, bx, by, bz, (uint16_t)0x3);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    uint32_t it = 0, tt = 0;
    for (int64_t tp = cid; tp < npairs; tp += ncl, ++tt) {
      const uint32_t acc = tt & 1, aph = (tt >> 1) & 1;
      mbar_wait(tempty + acc, aph ^ 1);
      tc_fence_after();
      const uint32_t dcol = tmem_base + acc * BN;
      for (int kb = 0; kb < g.kblocks; ++kb, ++it) {
        const uint32_t s = it % MC_STAGES, ph = (it / MC_STAGES) & 1;
        mbar_wait(full + s, ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t st = smem_u32(stage_base + s * MC_STAGE_BYTES);
          const uint64_t dA = sdesc_sw128(st), dB = sdesc_sw128(st + A_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 16 bf16 = 32 bytes inside the swizzle atom
            tc_mma_bf16(dcol, dA + adv, dB + adv, kIdescBF16, (kb == 0 && kk == 0) ? 0u : 1u);
          }
          tc_commit_mc(empty + s, (uint16_t)0x3);  // this stage is read: tell both producers
        }
        __syncwarp();
      }
      if (lane == 0) tc_commit(tfull + acc);
      __syncwarp();
    }
  } else {
    // ===================== epilogue (warps 2..5): tile and region-pair maxima =====================
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const int et = threadIdx.x - 64;
    uint32_t tt = 0;
    for (int64_t tp = cid; tp < npairs; tp += ncl, ++tt) {
      const uint32_t acc = tt & 1, aph = (tt >> 1) & 1;
      int64_t r, t;
      TileCoord c;
      mc_coord(reg, g.nreg, tp, rank, r, t, c);
      const GemmRegion& R = reg[r];
      float* cbias = colbias + acc * BN;
      for (int n = et; n < BN; n += 128) {
        const int lx = n % g.bxB, ly = (n / g.bxB) % g.byB, lz = n / (g.bxB * g.byB);
        const int x = R.B.x0 + c.ux * g.bxB + lx, y = R.B.y0 + c.uy * g.byB + ly, z = R.B.z0 + c.uz * g.bzB + lz;
        bool ok = x < R.B.x1 && y < R.B.y1 && z < R.B.z1;
        int p = -1;
        if (ok) {
          p = (z * g.ny + y) * g.nx + x;
          ok = cb[p] == 0;
        }
        // the self pair is masked through +inf bias on overlapping boxes (screen only needs the
        // max: a masked self pair never raises it)
        cbias[n] = ok ? 0.f : -INFINITY;
        if (R.overlap) colbias[2 * BN + acc * BN + n] = __int_as_float(p);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      const int lxA = row % g.bxA, lyA = (row / g.bxA) % g.byA, lzA = row / (g.bxA * g.byA);
      const int xa = R.A.x0 + c.tx * g.bxA + lxA, ya = R.A.y0 + c.ty * g.byA + lyA, za = R.A.z0 + c.tz * g.bzA + lzA;
      bool row_ok = xa < R.A.x1 && ya < R.A.y1 && za < R.A.z1;
      int pa = -1;
      if (row_ok) {
        pa = (za * g.ny + ya) * g.nx + xa;
        row_ok = ca[pa] == 0;
      }
      const bool selfmask = R.overlap != 0;
      const float* cpt = colbias + 2 * BN + acc * BN;
      mbar_wait(tfull + acc, aph);
      tc_fence_after();
      float best = -INFINITY;
      const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(q4 * 32) << 16);
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        float v[32];
        tmem_ld32(taddr + ch * 32, v);
        const float4* b4 = reinterpret_cast<const float4*>(cbias + ch * 32);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float4 bb = b4[i];
          v[4 * i + 0] = (g.absval ? fabsf(v[4 * i + 0]) : v[4 * i + 0]) + bb.x;
          v[4 * i + 1] = (g.absval ? fabsf(v[4 * i + 1]) : v[4 * i + 1]) + bb.y;
          v[4 * i + 2] = (g.absval ? fabsf(v[4 * i + 2]) : v[4 * i + 2]) + bb.z;
          v[4 * i + 3] = (g.absval ? fabsf(v[4 * i + 3]) : v[4 * i + 3]) + bb.w;
        }
        if (selfmask) {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (__float_as_int(cpt[ch * 32 + i]) == pa) v[i] = -INFINITY;
        }
        float m = v[0];
#pragma unroll
        for (int i = 1; i < 32; ++i) m = fmaxf(m, v[i]);
        best = fmaxf(best, m);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty + acc);
      uint32_t k32 = (row_ok && best > -INFINITY) ? ord32(best) : 0u;
#pragma unroll
      for (int o = 16; o; o >>= 1) k32 = max(k32, __shfl_xor_sync(0xffffffffu, k32, o));
      if (lane == 0 && k32 != 0u) {
        atomicMax(tile_keys + t, k32);
        atomicMax(reg_keys + r, k32);
      }
      asm volatile("bar.sync 2, 128;" ::: "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer may still multicast into it or signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap* m, const float* plane, const corr_field* f, int bx, int by, int bz) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)f->n_pad, (cuuint64_t)f->nx, (cuuint64_t)f->ny, (cuuint64_t)f->nz};
  cuuint64_t strides[3] = {(cuuint64_t)f->n_pad * 4, (cuuint64_t)f->n_pad * 4 * f->nx,
                           (cuuint64_t)f->n_pad * 4 * f->nx * f->ny};
  cuuint32_t box[4] = {(cuuint32_t)BK, (cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)plane, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_map_bf16(CUtensorMap* m, const uint16_t* plane, const corr_field* f, int bx, int by, int bz) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[4] = {(cuuint64_t)f->n_pad, (cuuint64_t)f->nx, (cuuint64_t)f->ny, (cuuint64_t)f->nz};
  cuuint64_t strides[3] = {(cuuint64_t)f->n_pad * 2, (cuuint64_t)f->n_pad * 2 * f->nx,
                           (cuuint64_t)f->n_pad * 2 * f->nx * f->ny};
  cuuint32_t box[4] = {(cuuint32_t)(2 * BK), (cuuint32_t)bx, (cuuint32_t)by, (cuuint32_t)bz};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)plane, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// Brick-slab box of `rows` points: x extent first (coalesced), then y, then z.
void box_shape(int rows, int ax, int ay, int& bx, int& by, int& bz) {
  bx = pow2ceil(ax) < 32 ? pow2ceil(ax) : 32;
  by = pow2ceil(ay) < rows / bx ? pow2ceil(ay) : rows / bx;
  bz = rows / (bx * by);
}

}  // namespace

cudaError_t launch_pearson_block2(const corr_field* fa, const corr_field* fb, const RegionDev* hreg, int64_t nreg,
                                  int absval, unsigned long long* keys, cudaStream_t st) {
  int maxax = 1, maxay = 1, maxbx = 1, maxby = 1;
  for (int64_t r = 0; r < nreg; ++r) {
    const RegionDev& R = hreg[r];
    maxax = std::max(maxax, R.A.x1 - R.A.x0);
    maxay = std::max(maxay, R.A.y1 - R.A.y0);
    maxbx = std::max(maxbx, R.B.x1 - R.B.x0);
    maxby = std::max(maxby, R.B.y1 - R.B.y0);
  }
  GemmGeom g;
  memset(&g, 0, sizeof(g));
  box_shape(128, maxax, maxay, g.bxA, g.byA, g.bzA);
  box_shape(128, maxbx, maxby, g.bxB, g.byB, g.bzB);
  if (g.bzA > 256 || g.bzB > 256) return cudaErrorNotSupported;
  g.nx = fa->nx;
  g.ny = fa->ny;
  g.kblocks = (fa->n_pad + BK - 1) / BK;
  g.absval = absval;
  g.same_field = fa == fb;
  g.nreg = nreg;
  std::vector<Gemm2Region> gr((size_t)nreg);
  int64_t tiles = 0;
  for (int64_t r = 0; r < nreg; ++r) {
    const RegionDev& R = hreg[r];
    Gemm2Region& G = gr[(size_t)r];
    memset(&G, 0, sizeof(G));
    G.A = R.A;
    G.B = R.B;
    G.ntA[0] = (R.A.x1 - R.A.x0 + g.bxA - 1) / g.bxA;
    G.ntA[1] = (R.A.y1 - R.A.y0 + g.byA - 1) / g.byA;
    G.ntA[2] = (R.A.z1 - R.A.z0 + g.bzA - 1) / g.bzA;
    G.ntB[0] = (R.B.x1 - R.B.x0 + g.bxB - 1) / g.bxB;
    G.ntB[1] = (R.B.y1 - R.B.y0 + g.byB - 1) / g.byB;
    G.ntB[2] = (R.B.z1 - R.B.z0 + g.bzB - 1) / g.bzB;
    G.nta = (int64_t)G.ntA[0] * G.ntA[1] * G.ntA[2];
    G.ntb = (int64_t)G.ntB[0] * G.ntB[1] * G.ntB[2];
    G.tile_off = tiles;
    G.nA = R.nA;
    G.nB = R.nB;
    G.overlap = g.same_field && R.A.x0 < R.B.x1 && R.B.x0 < R.A.x1 && R.A.y0 < R.B.y1 && R.B.y0 < R.A.y1 &&
                R.A.z0 < R.B.z1 && R.B.z0 < R.A.z1;
    tiles += ((G.nta + 1) / 2) * ((G.ntb + 1) / 2);
  }
  g.total_tiles = tiles;
  CUtensorMap mAhi, mAlo, mBhi, mBlo;
  if (!make_map(&mAhi, fa->Zhi, fa, g.bxA, g.byA, g.bzA) || !make_map(&mAlo, fa->Zlo, fa, g.bxA, g.byA, g.bzA) ||
      !make_map(&mBhi, fb->Zhi, fb, g.bxB, g.byB, g.bzB) || !make_map(&mBlo, fb->Zlo, fb, g.bxB, g.byB, g.bzB))
    return cudaErrorNotSupported;
  Gemm2Region* dgr = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dgr, gr.size() * sizeof(Gemm2Region), st);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyAsync(dgr, gr.data(), gr.size() * sizeof(Gemm2Region), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  const size_t smem = 1024 + (size_t)STAGES2 * STAGE2_BYTES + 8 * (2 * STAGES2 + 4) + 16 + 2 * BN * 4 + 2 * BN * 4;
  e = cudaFuncSetAttribute(pearson_block2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = kSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t clusters = tiles < sms / 2 ? tiles : sms / 2;
  pearson_block2_kernel<<<(unsigned)(2 * clusters), kThreads, smem, st>>>(mAhi, mAlo, mBhi, mBlo, dgr, g, fa->cflag,
                                                                         fb->cflag, keys);
  note_launch();
  e = cudaGetLastError();
  cudaFreeAsync(dgr, st);
  return e;
}

// executed tensor-core work of the block GEMMs (logical MMA flops incl. tile padding): the
// roofline numerator of bench.py's Pearson block line (corr_gemm_flops)
// [0]: bf16 flops (the screening pass), [1]: tf32 flops (the exact pass; a tf32 screen too)
__device__ unsigned long long g_gemm_flops[2];

__global__ void gemm_account_kernel(const int* __restrict__ tcount, long long tiles_screen, long long flop_per_mma_tile,
                                    int screen_bf16, long long tiles_exact_all) {
  const long long exact = tcount ? (long long)*tcount : tiles_exact_all;
  atomicAdd(&g_gemm_flops[screen_bf16 ? 0 : 1], (unsigned long long)(tiles_screen * flop_per_mma_tile));
  atomicAdd(&g_gemm_flops[1], (unsigned long long)(3 * exact * flop_per_mma_tile));
}

// screen -> tile list: keep tile t iff its approximate maximum is within delta of its region pair's
// approximate maximum (tiles with no admissible entry, key 0, are dropped)

__global__ void __launch_bounds__(256) screen_select_kernel(const GemmRegion* __restrict__ reg, int64_t nreg,
                                                            int64_t tiles, const uint32_t* __restrict__ tile_keys,
                                                            const uint32_t* __restrict__ reg_keys,
                                                            int* __restrict__ tlist, int* __restrict__ tcount,
                                                            float delta) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < tiles; t += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = tile_keys[t];
    if (k == 0u) continue;
    int64_t lo = 0, hi = nreg - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (reg[mid].tile_off <= t) lo = mid; else hi = mid - 1;
    }
    if (unord32(k) >= unord32(reg_keys[lo]) - delta) tlist[atomicAdd(tcount, 1)] = (int)t;
  }
}

cudaError_t launch_pearson_block(const corr_field* fa, const corr_field* fb, const RegionDev* hreg,
                                 const RegionDev* /*dreg*/, int64_t nreg, int absval, unsigned long long* keys,
                                 cudaStream_t st) {
  if (nreg == 0) return cudaSuccess;
  static const int two_sm = [] {
    const char* e = getenv("CORR_GEMM_2SM");  // opt-in: measured slower than the 1-SM kernel
    return (e && e[0] == '1') ? 1 : 0;
  }();
  if (two_sm) {
    const cudaError_t e2 = launch_pearson_block2(fa, fb, hreg, nreg, absval, keys, st);
    if (e2 != cudaErrorNotSupported) return e2;
  }
  int maxax = 1, maxay = 1, maxbx = 1, maxby = 1;
  for (int64_t r = 0; r < nreg; ++r) {
    const RegionDev& R = hreg[r];
    maxax = std::max(maxax, R.A.x1 - R.A.x0);
    maxay = std::max(maxay, R.A.y1 - R.A.y0);
    maxbx = std::max(maxbx, R.B.x1 - R.B.x0);
    maxby = std::max(maxby, R.B.y1 - R.B.y0);
  }
  GemmGeom g;
  memset(&g, 0, sizeof(g));
  box_shape(BM, maxax, maxay, g.bxA, g.byA, g.bzA);
  box_shape(BN, maxbx, maxby, g.bxB, g.byB, g.bzB);
  if (g.bzA > 256 || g.bzB > 256) return cudaErrorNotSupported;
  g.nx = fa->nx;
  g.ny = fa->ny;
  g.kblocks = (fa->n_pad + BK - 1) / BK;
  g.absval = absval;
  g.same_field = fa == fb;
  g.nreg = nreg;
  std::vector<GemmRegion> gr((size_t)nreg);
  int64_t tiles = 0, pairs = 0;
  for (int64_t r = 0; r < nreg; ++r) {
    const RegionDev& R = hreg[r];
    GemmRegion& G = gr[(size_t)r];
    G.A = R.A;
    G.B = R.B;
    G.ntA[0] = (R.A.x1 - R.A.x0 + g.bxA - 1) / g.bxA;
    G.ntA[1] = (R.A.y1 - R.A.y0 + g.byA - 1) / g.byA;
    G.ntA[2] = (R.A.z1 - R.A.z0 + g.bzA - 1) / g.bzA;
    G.ntB[0] = (R.B.x1 - R.B.x0 + g.bxB - 1) / g.bxB;
    G.ntB[1] = (R.B.y1 - R.B.y0 + g.byB - 1) / g.byB;
    G.ntB[2] = (R.B.z1 - R.B.z0 + g.bzB - 1) / g.bzB;
    G.tile_off = tiles;
    G.nA = R.nA;
    G.nB = R.nB;
    G.overlap = g.same_field && R.A.x0 < R.B.x1 && R.B.x0 < R.A.x1 && R.A.y0 < R.B.y1 && R.B.y0 < R.A.y1 &&
                R.A.z0 < R.B.z1 && R.B.z0 < R.A.z1;
    G.pair_off = pairs;
    const int64_t nta = (int64_t)G.ntA[0] * G.ntA[1] * G.ntA[2], ntb = (int64_t)G.ntB[0] * G.ntB[1] * G.ntB[2];
    tiles += nta * ntb;
    pairs += (nta + 1) / 2 * ntb;
  }
  g.total_tiles = tiles;
  CUtensorMap mAhi, mAlo, mBhi, mBlo;
  if (!make_map(&mAhi, fa->Zhi, fa, g.bxA, g.byA, g.bzA) || !make_map(&mAlo, fa->Zlo, fa, g.bxA, g.byA, g.bzA) ||
      !make_map(&mBhi, fb->Zhi, fb, g.bxB, g.byB, g.bzB) || !make_map(&mBlo, fb->Zlo, fb, g.bxB, g.byB, g.bzB))
    return cudaErrorNotSupported;
  // the tile table: resident device copy reused across calls with the same region pairs
  GemmRegion* dgr = const_cast<GemmRegion*>(
      static_cast<const GemmRegion*>(cached_table(fa->device, gr.data(), gr.size() * sizeof(GemmRegion), st)));
  const bool own_gr = dgr == nullptr;
  cudaError_t e = cudaSuccess;
  if (own_gr) {
    e = cudaMallocAsync((void**)&dgr, gr.size() * sizeof(GemmRegion), st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(dgr, gr.data(), gr.size() * sizeof(GemmRegion), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
  }
  const size_t smem = 1024 + (size_t)STAGES * STAGE_BYTES + 8 * (2 * STAGES + 4) + 16 + 2 * BN * 4 + 2 * BN * 4;
  e = cudaFuncSetAttribute(pearson_block_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(pearson_block_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(pearson_block_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = kSMs;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t grid = tiles < sms ? tiles : sms;
  static const int noscreen = [] {
    const char* v = getenv("CORR_GEMM_NOSCREEN");  // A/B switch: every tile through the full product
    return (v && v[0] == '1') ? 1 : 0;
  }();
  const long long flop_tile = 2LL * BM * BN * (long long)(g.kblocks * BK);
  if (noscreen || tiles >= (int64_t)INT32_MAX) {
    pearson_block_kernel<false><<<(unsigned)grid, kThreads, smem, st>>>(
        mAhi, mAlo, mBhi, mBlo, dgr, g, fa->cflag, fb->cflag, keys, nullptr, nullptr, nullptr, nullptr);
    gemm_account_kernel<<<1, 1, 0, st>>>(nullptr, 0, flop_tile, 0, (long long)tiles);
    note_launch(2);
    e = cudaGetLastError();
    if (own_gr) cudaFreeAsync(dgr, st);
    return e;
  }
  // Screened two-pass evaluation (exact): pass 1 computes every tile with the hi*hi product only
  // and records tile and region-pair maxima of that approximation; a tile can hold the region
  // pair's maximum only if its approximate maximum is within kScreenDelta of the region pair's,
  // so pass 2 runs the full split-TF32 product (and the max/argmax epilogue) on those tiles only.
  // Bound on |pass-1 value - pass-2 value| for unit-norm rows (Cauchy-Schwarz):
  //   split:        |z z' - hi hi'| summed <= (2 * 2^-11 + 2^-22) ||z|| ||z'||
  //   accumulation: each pass adds K fp32 terms, error <= K * 2^-23 * sum|terms| (any order,
  //                 truncating adds) -> 2 * K * 2^-23 for both passes together
  // A tile whose approximate maximum is below (region approx max - 2b) holds only entries whose
  // exact value is below the region's maximum, so dropping it changes neither max nor argmax.
  // The screening pass runs on bf16(Z) (unit roundoff 2^-8) unless CORR_GEMM_SCREEN_TF32=1 selects
  // tf32 Z_hi (2^-11): bf16 moves half the operand bytes and runs the MMA at twice the rate, at
  // the price of a wider margin (1.8e-2 vs 2.7e-3 at n = 1000), i.e. a few more kept tiles.
  static const int screen_tf32 = [] {
    const char* v = getenv("CORR_GEMM_SCREEN_TF32");
    return (v && v[0] == '1') ? 1 : 0;
  }();
  const double u_scr = screen_tf32 ? std::ldexp(1.0, -11) : std::ldexp(1.0, -8);
  const double b_bound = 2.0 * u_scr + u_scr * u_scr + 2.0 * (double)(g.kblocks * BK) * std::ldexp(1.0, -23) + 1e-6;
  const float delta = (float)(2.0 * b_bound * 1.1);  // 10 % margin
  GemmGeom gs = g;  // the bf16 screen covers 64 members per k-block
  CUtensorMap mAb, mBb;
  if (!screen_tf32) {
    gs.kblocks = (fa->n_pad + 2 * BK - 1) / (2 * BK);
    if (!make_map_bf16(&mAb, fa->Zb, fa, g.bxA, g.byA, g.bzA) || !make_map_bf16(&mBb, fb->Zb, fb, g.bxB, g.byB, g.bzB)) {
      if (own_gr) cudaFreeAsync(dgr, st);
      return cudaErrorNotSupported;
    }
  }
  uint32_t* tile_keys = nullptr;
  uint32_t* reg_keys = nullptr;
  int* tlist = nullptr;
  int* tcount = nullptr;
  e = cudaMallocAsync((void**)&tile_keys, (size_t)tiles * 4, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&tlist, (size_t)tiles * 4, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&reg_keys, (size_t)nreg * 4 + 16, st);
  if (e != cudaSuccess) {
    if (tile_keys) cudaFreeAsync(tile_keys, st);
    if (tlist) cudaFreeAsync(tlist, st);
    if (own_gr) cudaFreeAsync(dgr, st);
    return e;
  }
  tcount = reinterpret_cast<int*>(reg_keys + nreg);
  cudaMemsetAsync(tile_keys, 0, (size_t)tiles * 4, st);
  cudaMemsetAsync(reg_keys, 0, (size_t)nreg * 4 + 16, st);
  // bf16 screen: the B-multicast cluster kernel (pearson_screen_mc_kernel) unless
  // CORR_GEMM_SCREEN_MC=0 selects the 1-SM screen (A/B switch)
  static const int screen_mc = [] {
    const char* v = getenv("CORR_GEMM_SCREEN_MC");
    return (v && v[0] == '0') ? 0 : 1;
  }();
  bool mc_done = false;
  if (!screen_tf32 && screen_mc && sms >= 2) {
    const bool zsplit = gs.bzB >= 2;
    const int bhy = zsplit ? 0 : gs.byB / 2, bhz = zsplit ? gs.bzB / 2 : 0;
    CUtensorMap mBh;
    if (make_map_bf16(&mBh, fb->Zb, fb, gs.bxB, zsplit ? gs.byB : gs.byB / 2, zsplit ? gs.bzB / 2 : gs.bzB)) {
      const size_t smem_mc = 1024 + (size_t)MC_STAGES * MC_STAGE_BYTES + 8 * (2 * MC_STAGES + 4) + 16 + 4 * BN * 4;
      e = cudaFuncSetAttribute(pearson_screen_mc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_mc);
      if (e == cudaSuccess) {
        const int64_t clusters = pairs < sms / 2 ? pairs : sms / 2;
        pearson_screen_mc_kernel<<<(unsigned)(2 * clusters), kThreads, smem_mc, st>>>(
            mAb, mBh, dgr, gs, pairs, bhy, bhz, fa->cflag, fb->cflag, tile_keys, reg_keys);
        mc_done = true;
      } else {
        cudaGetLastError();
      }
    }
  }
  if (mc_done) {
  } else if (screen_tf32)
    pearson_block_kernel<true><<<(unsigned)grid, kThreads, smem, st>>>(
        mAhi, mAlo, mBhi, mBlo, dgr, g, fa->cflag, fb->cflag, keys, nullptr, nullptr, tile_keys, reg_keys);
  else
    pearson_block_kernel<true, true><<<(unsigned)grid, kThreads, smem, st>>>(
        mAb, mAb, mBb, mBb, dgr, gs, fa->cflag, fb->cflag, keys, nullptr, nullptr, tile_keys, reg_keys);
  screen_select_kernel<<<(unsigned)std::min<int64_t>((tiles + 255) / 256, (int64_t)sms * 16), 256, 0, st>>>(
      dgr, g.nreg, tiles, tile_keys, reg_keys, tlist, tcount, delta);
  pearson_block_kernel<false><<<(unsigned)grid, kThreads, smem, st>>>(
      mAhi, mAlo, mBhi, mBlo, dgr, g, fa->cflag, fb->cflag, keys, tlist, tcount, nullptr, nullptr);
  // executed work: the screen's MMA count per tile equals one tf32 set (same K coverage), counted
  // as one set of 2*M*N*K flops (bf16 or tf32)
  gemm_account_kernel<<<1, 1, 0, st>>>(tcount, (long long)tiles, flop_tile, screen_tf32 ? 0 : 1, 0);
  note_launch(4);
  e = cudaGetLastError();
  cudaFreeAsync(tile_keys, st);
  cudaFreeAsync(tlist, st);
  cudaFreeAsync(reg_keys, st);
  if (own_gr) cudaFreeAsync(dgr, st);
  return e;
}

cudaError_t gemm_flops(unsigned long long* value, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(value, g_gemm_flops, 2 * sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long zero[2] = {0, 0};
    e = cudaMemcpyToSymbol(g_gemm_flops, zero, sizeof(zero));
  }
  return e;
}

}  // namespace corr
