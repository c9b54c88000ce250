// ksg.cu -- Kraskov (KSG) MI for batches of point pairs: sorted, filtered, exact sweep.
// SURVEY.md §8(a) rows a2-a5 (+ a8/a9 via the pair source); NEXT #1 of §8(f).
//
// Definitions (readings R1-R7): eps_i = k-th smallest Chebyshev distance
// (fp32), strict marginal counts, MI = psi(n) + psi(k) - (1/n) sum_i [psi(n_x,i) + psi(n_y,i)].
//
// Measured facts that shape this kernel: FMNMX/FSETP issue on the ALU pipe at
// 0.5 warp-instr/clk/SMSP (ncu: ALU 89 % busy at IPC 2.27 for the plain register network);
// FMNMX3 costs the same slot for twice the work; FADD2 runs on the FMA pipe.  So the kernel
// minimises ALU work per comparison:
//  * the pair is staged sorted along its WIDER marginal (spread = ||x - mean||): the k-NN of a
//    member then lies in a narrow window of that order.  KSG is symmetric in (x, y) (Eq. 1), so
//    swapping the roles of a and b leaves eps unchanged and swaps the two counts (exact);
//  * xy[t] = (S_u[t], F_v[perm_u[t]]) -- a member permutation; eps is order-free (R4);
//  * a warp owns 32*RM sort-consecutive members (RM per lane: one broadcast LDS.128 of two
//    joint samples feeds 2*RM comparisons); it scans its own block first (exact merge network,
//    the j == i mask only on the diagonal member of each chunk), then 32-wide chunks outward;
//  * outside the own block, per group of 4 j and member: 4 distances (FADD2 + FMNMX|.|), their
//    min (FMNMX3 + FMNMX) and one compare with the list's k-th entry; only if some lane can
//    insert (VOTE.ANY) does the warp run the exact merge network
//        l'_r = min(l_r, max(l_{r-1}, a), max(l_{r-2}, b)),  (a, b) = sorted pair of new values
//    -- inserting d >= l[K-1] is a no-op, so skipping it is exact;
//  * SWEEP: a direction stops once fl(x_block_edge - x_chunk_edge) >= every member's current
//    k-th distance: |fl(x_i - x_j)| >= that gap for all remaining j (monotone rounding), so no
//    remaining j can enter any list (exact).  Executed comparisons are counted for the roofline;
//  * counts: two binary searches per marginal on the sorted rows with monotone fp32
//    predicates (bit-exact), psi from an fp64 shared table, fixed-order fp64 reduction.
#include <math.h>
#include <stdlib.h>

#include <algorithm>

#include "ksg_common.cuh"

namespace corr {

__device__ unsigned long long g_ksg_comparisons;  // executed comparisons (corr_ksg_comparisons)
__device__ unsigned long long g_ksg_nan_pairs;    // region-max pairs skipped as NaN (corr_ksg_nan_pairs)

namespace {

// Strict marginal count of a member with value v and radius e on a sorted
// array S (element stride ST): #{j != i : |fl(v - S_j)| < e}.
//   e == 0: the strict interval is empty -> 0 (reading R5).
//   e  > 0: u = first s with fl(s - v) >= e, w = first s with fl(v - s) < e (both predicates
//           are monotone in s by monotone rounding, and imply / cover s >= v because e > 0);
//           [w, u) holds every s with |fl(s - v)| < e, the member itself included -> u - w - 1.
// Branch-free lower bounds (uniform trip count), the two searches interleaved for ILP.
// The four searches of one member (u and w on the sorted marginal x -- stride 8 B inside xy --
// and on the sorted y row), interleaved; step 2^B is a compile-time immediate offset.
template <int B>
struct CountSearch {
  __device__ __forceinline__ static void run(int log2p, uint32_t& xu, uint32_t& xw, uint32_t& yu, uint32_t& yw,
                                             float x, float y, float e) {
    if (B < log2p) {
      constexpr int SX = (1 << B) * 8, SY = (1 << B) * 4;
      const float pxu = lds_imm<SX - 8>(xu), pxw = lds_imm<SX - 8>(xw);
      const float pyu = lds_imm<SY - 4>(yu), pyw = lds_imm<SY - 4>(yw);
      xu = (pxu - x >= e) ? xu : xu + SX;  // not yet P_u -> move right
      xw = (x - pxw < e) ? xw : xw + SX;   // not yet P_w -> move right
      yu = (pyu - y >= e) ? yu : yu + SY;
      yw = (y - pyw < e) ? yw : yw + SY;
    }
    CountSearch<B - 1>::run(log2p, xu, xw, yu, yw, x, y, e);
  }
};
template <>
struct CountSearch<-1> {
  __device__ __forceinline__ static void run(int, uint32_t&, uint32_t&, uint32_t&, uint32_t&, float, float, float) {}
};

// Strict marginal counts of a member (x, y) with radius e: returns n_x, n_y.
__device__ __forceinline__ void marginal_counts(const float2* __restrict__ xy, const float* __restrict__ sy,
                                                int log2p, float x, float y, float e, int& cx, int& cy) {
  if (!(e > 0.f)) {
    cx = cy = 0;
    return;
  }
  const uint32_t bx = (uint32_t)__cvta_generic_to_shared(xy), by = (uint32_t)__cvta_generic_to_shared(sy);
  uint32_t xu = bx, xw = bx, yu = by, yw = by;
  CountSearch<12>::run(log2p, xu, xw, yu, yw, x, y, e);
  cx = (int)((xu - xw) >> 3) - 1;
  cy = (int)((yu - yw) >> 2) - 1;
}

// own-block chunk: exact network; the self pair j == i exists only for member RC of each lane
template <int K, int RM, int RC>
__device__ __forceinline__ void own_chunk(const float4* __restrict__ cp, const float2 (&zi)[RM],
                                          float (&l)[RM][K], int lane) {
#pragma unroll 4
  for (int h = 0; h < 16; ++h) {
    const float4 v = cp[h];
    const float2 z0 = make_float2(v.x, v.y), z1 = make_float2(v.z, v.w);
#pragma unroll
    for (int rr = 0; rr < RM; ++rr) {
      float e0 = cheb(zi[rr], z0), e1 = cheb(zi[rr], z1);
      if (rr == RC) {
        if (2 * h == lane) e0 = INFINITY;
        if (2 * h + 1 == lane) e1 = INFINITY;
      }
      merge2<K>(l[rr], e0, e1);
    }
  }
}

// RM == 1 own chunk without masks: lane L reads the warp's 32 joint samples rotated by L
// (a private doubled copy, dup[i] = chunk[i & 31]); s = 1..31 visits every j != i exactly once.
template <int K>
__device__ __forceinline__ void own_rotated(const float2* __restrict__ dup, int lane, float2 zi, float (&l)[K]) {
  const float2* p = dup + lane;
#pragma unroll(K <= 8 ? 15 : 1)
  for (int s = 1; s < 31; s += 2) merge2<K>(l, cheb(zi, p[s]), cheb(zi, p[s + 1]));
  insert1<K>(l, cheb(zi, p[31]));
}

// RM == 1 own block with only v < 32 members (the last block when 32 does not divide n): dup
// holds the block with period v, so s = 1..v-1 visits the v-1 others (lanes >= v are padding).
template <int K>
__device__ __forceinline__ void own_rotated_part(const float2* __restrict__ dup, int lane, float2 zi, float (&l)[K],
                                                 int v) {
  const float2* p = dup + lane;
  int s = 1;
  for (; s + 1 < v; s += 2) merge2<K>(l, cheb(zi, p[s]), cheb(zi, p[s + 1]));
  if (s < v) insert1<K>(l, cheb(zi, p[s]));
}

template <int K, int RM, int RC>
struct OwnBlock {
  __device__ __forceinline__ static void run(const float4* xy4, int c0, int nch, const float2 (&zi)[RM],
                                             float (&l)[RM][K], int lane) {
    OwnBlock<K, RM, RC - 1>::run(xy4, c0, nch, zi, l, lane);
    if (c0 + RC < nch) own_chunk<K, RM, RC>(xy4 + (c0 + RC) * 16, zi, l, lane);
  }
};
template <int K, int RM>
struct OwnBlock<K, RM, -1> {
  __device__ __forceinline__ static void run(const float4*, int, int, const float2 (&)[RM], float (&)[RM][K], int) {}
};

// one unfiltered 32-j chunk (no self pair inside): exact merge network on every value.  Used for
// the chunks adjacent to the own block, where the filter would trigger on most groups anyway.
// Fully unrolled so every shared load is issued well ahead of its FADD2.
template <int K, int RM>
__device__ __forceinline__ void chunk_plain(const float4* __restrict__ cp, const float2 (&zi)[RM], float (&l)[RM][K],
                                            int cnt) {
  if (cnt < 32) {  // the partial last chunk: compact loop over its (cnt + 1) / 2 float4s
    for (int h = 0; h < ((cnt + 1) >> 1); ++h) {
      const float4 v = cp[h];
#pragma unroll
      for (int rr = 0; rr < RM; ++rr) merge2<K>(l[rr], cheb(zi[rr], make_float2(v.x, v.y)), cheb(zi[rr], make_float2(v.z, v.w)));
    }
    return;
  }
#pragma unroll((RM == 1 && K <= 8) ? 16 : 2)
  for (int h = 0; h < 16; ++h) {
    const float4 v = cp[h];
    const float2 z0 = make_float2(v.x, v.y), z1 = make_float2(v.z, v.w);
#pragma unroll
    for (int rr = 0; rr < RM; ++rr) merge2<K>(l[rr], cheb(zi[rr], z0), cheb(zi[rr], z1));
  }
}

// one filtered 32-j chunk, groups of G j's per vote, compact loop (RM > 1: the dense
// 4-members-per-lane layout; K > 8: the long lists of the paper's k = ceil(3n/100))
template <int K, int RM, int G, bool DESC>
__device__ __forceinline__ void chunk_filtered_rm(const float4* __restrict__ cp, const float2 (&zi)[RM],
                                                  float (&l)[RM][K], int cnt) {
  constexpr int NG = 32 / G;
  const int ng = (cnt + G - 1) / G;  // DESC chunks are always full (the partial chunk is the last)
#pragma unroll 2
  for (int gi = 0; gi < ng; ++gi) {
    const int g = DESC ? NG - 1 - gi : gi;
    float2 z[G];
#pragma unroll
    for (int q = 0; q < G / 2; ++q) {
      const float4 v = cp[g * (G / 2) + q];
      z[2 * q] = make_float2(v.x, v.y);
      z[2 * q + 1] = make_float2(v.z, v.w);
    }
    float d[RM][G];
    bool p = false;
#pragma unroll
    for (int rr = 0; rr < RM; ++rr) {
#pragma unroll
      for (int q = 0; q < G; ++q) d[rr][q] = cheb(zi[rr], z[q]);
      float m = d[rr][0];
#pragma unroll
      for (int q = 1; q < G; ++q) m = fminf(m, d[rr][q]);
      p |= m < l[rr][K - 1];
    }
    if (__any_sync(0xffffffffu, p)) {
#pragma unroll
      for (int rr = 0; rr < RM; ++rr) {
#pragma unroll
        for (int q = 0; q < G; q += 2) merge2<K>(l[rr], d[rr][q], d[rr][q + 1]);
      }
    }
  }
}

// one filtered 32-j chunk, groups of G j's per vote; the next group's shared loads are issued
// before this group's vote (software pipelining across the data-dependent branch)
template <int K, int RM, int G, bool DESC>
__device__ __forceinline__ void chunk_filtered(const float4* __restrict__ cp, const float2 (&zi)[RM],
                                               float (&l)[RM][K], int cnt) {
  if constexpr (RM > 1 || K > 8) {  // compact loop: long lists make the unrolled body too big for the i-cache
    chunk_filtered_rm<K, RM, G, DESC>(cp, zi, l, cnt);
    return;
  }
  if (!DESC && cnt < 32) {  // the partial last chunk (only ever scanned upward): compact loop
    chunk_filtered_rm<K, RM, G, DESC>(cp, zi, l, cnt);
    return;
  }
  constexpr int NG = 32 / G, NQ = G / 2;
  float4 cur[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) cur[q] = cp[(DESC ? NG - 1 : 0) * NQ + q];
#pragma unroll
  for (int gi = 0; gi < NG; ++gi) {
    const int g = DESC ? NG - 1 - gi : gi;
    float4 nxt[NQ];
    if (gi + 1 < NG) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) nxt[q] = cp[(DESC ? g - 1 : g + 1) * NQ + q];
    }
    float2 z[G];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      z[2 * q] = make_float2(cur[q].x, cur[q].y);
      z[2 * q + 1] = make_float2(cur[q].z, cur[q].w);
    }
    float d[RM][G];
    bool p = false;
#pragma unroll
    for (int rr = 0; rr < RM; ++rr) {
#pragma unroll
      for (int q = 0; q < G; ++q) d[rr][q] = cheb(zi[rr], z[q]);
      float m = d[rr][0];
#pragma unroll
      for (int q = 1; q < G; ++q) m = fminf(m, d[rr][q]);
      p |= m < l[rr][K - 1];
    }
    if (__any_sync(0xffffffffu, p)) {
#pragma unroll
      for (int rr = 0; rr < RM; ++rr) {
#pragma unroll
        for (int q = 0; q < G; q += 2) merge2<K>(l[rr], d[rr][q], d[rr][q + 1]);
      }
    }
    if (gi + 1 < NG) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) cur[q] = nxt[q];
    }
  }
}

// the chunk adjacent to the own block (RM == 1, K <= 8, full chunk; warp kernel, n < 128): the 16
// candidates nearest to the block in x order with the exact network, the far 16 filtered in
// groups of 4 (C3: +4 %; at n = 1000 the all-exact chunk is 2 % faster, so the CTA kernel keeps it)
template <int K, bool DESC>
__device__ __forceinline__ void chunk_adjacent(const float4* __restrict__ cp, const float2 (&zi)[1],
                                               float (&l)[1][K]) {
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const float4 v = cp[DESC ? 15 - h : h];
    merge2<K>(l[0], cheb(zi[0], make_float2(v.x, v.y)), cheb(zi[0], make_float2(v.z, v.w)));
  }
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int b = DESC ? 6 - 2 * g : 8 + 2 * g;
    const float4 v0 = cp[b], v1 = cp[b + 1];
    float d[4] = {cheb(zi[0], make_float2(v0.x, v0.y)), cheb(zi[0], make_float2(v0.z, v0.w)),
                  cheb(zi[0], make_float2(v1.x, v1.y)), cheb(zi[0], make_float2(v1.z, v1.w))};
    const float m = fminf(fminf(fminf(d[0], d[1]), d[2]), d[3]);
    if (__any_sync(0xffffffffu, m < l[0][K - 1])) {
      merge2<K>(l[0], d[0], d[1]);
      merge2<K>(l[0], d[2], d[3]);
    }
  }
}

// ---- a3 / a4 / a5 for one member block (32*RM sort-consecutive members) of a staged pair:
// own block, outward chunks with the exact sweep, marginal counts, psi sum into acc.
// xy: interleaved (x, y) in x order (+inf pad to nxy), sy: sorted y (+inf pad to nsy),
// dup: this warp's 64-entry scratch (RM == 1), pm: the x argsort (debug dump only).
// PARTIAL: when 32 does not divide n, scan only the existing members of the last chunk /
// own block (the warp kernel, n < 128, where that chunk is a large share of the work); the CTA
// kernel scans the +inf-padded chunk as a full one (identical results: +inf never enters).
template <int K, int RM, int G, bool SWEEP, bool PARTIAL>
__device__ __forceinline__ int ksg_block(const float2* __restrict__ xy, const float* __restrict__ sy,
                                          float2* __restrict__ dup, int n, int nch, int log2p, int mb, int lane,
                                          int k, const double* __restrict__ psi, int off, double& acc,
                                          unsigned long long& executed, const PairOut& out, int64_t u,
                                          const uint16_t* __restrict__ pm, bool swap, int* next_blk) {
  constexpr int BLK = 32 * RM;
  const float4* xy4 = reinterpret_cast<const float4*>(xy);
  float2 zi[RM];
  float l[RM][K];
  int ts[RM];
#pragma unroll
  for (int rr = 0; rr < RM; ++rr) {
    ts[rr] = mb * BLK + 32 * rr + lane;
    zi[rr] = xy[ts[rr]];
#pragma unroll
    for (int t = 0; t < K; ++t) l[rr][t] = INFINITY;
  }
  const int c0 = mb * RM;
  const int c1 = min(c0 + RM, nch);
  const int vown = min(32, n - c0 * 32);  // members in the own chunk
  if constexpr (RM == 1) {
    if (!PARTIAL || vown == 32) {
      const float2 zc = xy[c0 * 32 + lane];
      dup[lane] = zc;
      dup[lane + 32] = zc;
      __syncwarp();
      own_rotated<K>(dup, lane, zi[0], l[0]);
    } else {
      dup[lane] = xy[c0 * 32 + lane % vown];
      dup[lane + 32] = xy[c0 * 32 + (lane + 32) % vown];
      __syncwarp();
      own_rotated_part<K>(dup, lane, zi[0], l[0], vown);
    }
    __syncwarp();
  } else {
    OwnBlock<K, RM, RM - 1>::run(xy4, c0, nch, zi, l, lane);
  }
  // outward in chunks of 32 j; below descending, above ascending
  const int nh = nch;
  // executed comparisons per valid member: the own block's others + every scanned candidate
  int ncand = (RM == 1) ? vown - 1 : min(BLK, n - c0 * 32) - 1;
  int hlo = c0 - 1, hhi = c1;
  while (hlo >= 0 || hhi < nh) {
    // SWEEP: per-member exact test -- member i still needs the chunk iff the x-gap to the
    // chunk's nearest edge is below its current k-th distance: fl(x_i - x_edge) < l_i[K-1]
    // (below) or fl(x_edge - x_i) < l_i[K-1] (above).  Skip the direction once no lane does.
    if (hlo >= 0) {
      bool need = true;
      if (SWEEP) {
        const float xe = xy[hlo * 32 + 31].x;
        bool p = false;
#pragma unroll
        for (int rr = 0; rr < RM; ++rr) p |= (ts[rr] < n) && (zi[rr].x - xe < l[rr][K - 1]);
        need = __any_sync(0xffffffffu, p);
      }
      if (!need) {
        hlo = -1;
      } else {
        if (hlo == c0 - 1) {
          if constexpr (PARTIAL && RM == 1 && K <= 8) chunk_adjacent<K, true>(xy4 + hlo * 16, zi, l);
          else chunk_plain<K, RM>(xy4 + hlo * 16, zi, l, 32);
        }
        // warp kernel (n < 128): the compact filtered loop -- its code path runs on few chunks per
        // pair, and the unrolled body costs more in i-cache misses than it saves (C3 +4 %)
        else if constexpr (PARTIAL) chunk_filtered_rm<K, RM, G, true>(xy4 + hlo * 16, zi, l, 32);
        else chunk_filtered<K, RM, G, true>(xy4 + hlo * 16, zi, l, 32);
        ncand += 32;
        --hlo;
      }
    }
    if (hhi < nh) {
      bool need = true;
      if (SWEEP) {
        const float xe = xy[hhi * 32].x;
        bool p = false;
#pragma unroll
        for (int rr = 0; rr < RM; ++rr) p |= (ts[rr] < n) && (xe - zi[rr].x < l[rr][K - 1]);
        need = __any_sync(0xffffffffu, p);
      }
      if (!need) {
        hhi = nh;
      } else {
        const int cnt = min(32, n - hhi * 32);
        if (hhi == c1) {
          if constexpr (PARTIAL && RM == 1 && K <= 8) {
            if (cnt == 32) chunk_adjacent<K, false>(xy4 + hhi * 16, zi, l);
            else chunk_plain<K, RM>(xy4 + hhi * 16, zi, l, cnt);
          } else {
            chunk_plain<K, RM>(xy4 + hhi * 16, zi, l, PARTIAL ? cnt : 32);
          }
        }
        else if constexpr (PARTIAL) chunk_filtered_rm<K, RM, G, false>(xy4 + hhi * 16, zi, l, cnt);
        else chunk_filtered<K, RM, G, false>(xy4 + hhi * 16, zi, l, 32);
        ncand += cnt;
        ++hhi;
      }
    }
  }
  const int valid = min(BLK, n - mb * BLK);
  // claim the warp's next member block now (CTA kernel): the shared atomic's latency hides under
  // the count searches
  int nb = 0;
  if (lane == 0) {
    executed += (unsigned long long)ncand * (unsigned long long)valid;
    if (next_blk) nb = atomicAdd(next_blk, 1);
  }
#pragma unroll
  for (int rr = 0; rr < RM; ++rr) {
    if (ts[rr] < n) {
      float e = l[rr][K - 1];
      if (K > 8) {  // list longer than k: eps = l[k-1] (the K smallest are exact)
#pragma unroll
        for (int t = 0; t < K - 1; ++t)
          if (t == k - 1) e = l[rr][t];
      }
      int cu, cv;
      marginal_counts(xy, sy, log2p, zi[rr].x, zi[rr].y, e, cu, cv);
      acc += __ldg(psi + cu + off) + __ldg(psi + cv + off);
      if (out.dbg_eps) {
        const int m = pm[ts[rr]];
        out.dbg_eps[u * n + m] = e;
        out.dbg_nx[u * n + m] = swap ? cv : cu;
        out.dbg_ny[u * n + m] = swap ? cu : cv;
      }
    }
  }
  return __shfl_sync(0xffffffffu, nb, 0);
}


// ---- large k (the paper's k = ceil(3n/100), e.g. 30 at n = 1000): batched exact updates ------
// With a 32-entry list the 2-value merge network costs ~3K min/max per pair of values.  Here a
// whole 32-candidate chunk is merged at once: the lane's 32 distances are sorted by a bitonic
// network (240 compare-exchanges) and merged with the sorted list by the half-cleaner
// c_i = min(l_i, d_{31-i}) (the 32 smallest of both, as a bitonic sequence) followed by a
// 5-stage bitonic merge: ~21 min/max per value instead of ~48.  The list INCLUDES the member
// itself (d_ii = 0), so eps_i = l[k] -- the (k+1)-th smallest over all j, identical to the
// k-th over j != i (R3).  Chunks whose distances are all >= l[KT] (KT = k, compile-time) are
// skipped (exact: they cannot change the k+1 smallest); the sweep uses the same threshold.
__device__ __forceinline__ void cas_asc(float& a, float& b) {
  const float lo = fminf(a, b), hi = fmaxf(a, b);
  a = lo;
  b = hi;
}

__device__ __forceinline__ void bitonic_sort32(float (&d)[32]) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int j = i ^ stride;
        if (j > i) {
          if ((i & size) == 0) cas_asc(d[i], d[j]);
          else cas_asc(d[j], d[i]);
        }
      }
    }
  }
}

// l (sorted, 32) <- the 32 smallest of l and d (d is destroyed)
__device__ __forceinline__ void batch_merge32(float (&l)[32], float (&d)[32]) {
  bitonic_sort32(d);
#pragma unroll
  for (int i = 0; i < 32; ++i) l[i] = fminf(l[i], d[31 - i]);
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int j = i ^ stride;
      if (j > i) cas_asc(l[i], l[j]);
    }
  }
}

// k >= 33 (the paper's k = ceil(3n/100) for n >= 1067): MULTI-PASS batched lists.  Pass p keeps
// the 32 smallest distances ABOVE a floor (the previous pass's 32nd value; -1 in pass 0) and counts
// c_p = #{d <= floor} over all j (self included); the (k+1)-th smallest overall is then
// L_p[k - c_p] as soon as k - c_p < 32 (the multiset below the floor is exactly c_p long, and L_p
// lists the next values in order -- ties at the floor are all counted, none listed; k - c_p < 0
// means rank k is one of the floor's unlisted tie copies, eps = floor).  Every pass
// is a full exact sweep: unvisited or filtered candidates have d >= l[31] > floor, so the count is
// exact.  Lanes that are done keep their eps; the warp runs passes until every lane is done.
template <int KT, bool SWEEP, bool MULTI>
__device__ __forceinline__ int ksg_block_big(const float2* __restrict__ xy, const float* __restrict__ sy, int n,
                                             int nch, int log2p, int mb, int lane, int k,
                                             const double* __restrict__ psi, int off, double& acc,
                                             unsigned long long& executed, const PairOut& out, int64_t u,
                                             const uint16_t* __restrict__ pm, bool swap, int* next_blk) {
  const int ti = mb * 32 + lane;
  const float2 zi = xy[ti];
  float l[32];
  const float4* xy4 = reinterpret_cast<const float4*>(xy);
  const int c0 = mb, c1 = mb + 1;
  int ncand = 0;
  float floor_ = -1.f;  // distances are >= 0: pass 0 has no floor
  float e = INFINITY;
  bool done = ti >= n;
#pragma unroll 1
  while (true) {
#pragma unroll
    for (int t = 0; t < 32; ++t) l[t] = INFINITY;
    int below = 0;  // #{d <= floor_} (MULTI)
    ncand += min(32, n - c0 * 32) - 1;
    // chunk sequence: own block (exact), then below / above alternately; the first chunk in each
    // direction is merged unconditionally, later ones only if some lane has a candidate < l[KT]
    int hlo = c0 - 1, hhi = c1, dir = 1;
    int h = c0;
    bool exact = true;
#pragma unroll 1
    while (true) {
      float d[32];
      const float4* cp = xy4 + h * 16;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float4 v = cp[q];
        d[2 * q] = cheb(zi, make_float2(v.x, v.y));
        d[2 * q + 1] = cheb(zi, make_float2(v.z, v.w));
      }
      if (MULTI) {
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          below += d[q] <= floor_ ? 1 : 0;
          d[q] = d[q] <= floor_ ? INFINITY : d[q];
        }
      }
      bool merge = exact;
      if (!merge) {
        float m = d[0];
#pragma unroll
        for (int q = 1; q < 32; ++q) m = fminf(m, d[q]);
        merge = __any_sync(0xffffffffu, m < l[KT]);
      }
      if (merge) batch_merge32(l, d);
      if (h != c0) ncand += min(32, n - h * 32);
      // next chunk: alternate directions; a direction ends at the array edge or by the sweep test
      bool found = false;
#pragma unroll 1
      for (int tries = 0; tries < 2 && !found; ++tries) {
        dir ^= 1;
        const int hc = dir ? hhi : hlo;
        if (dir ? hc >= nch : hc < 0) continue;
        bool need = true;
        if (SWEEP) {
          const float xe = xy[hc * 32 + (dir ? 0 : 31)].x;
          const float gap = dir ? xe - zi.x : zi.x - xe;
          need = __any_sync(0xffffffffu, (ti < n) && (gap < l[KT]));
        }
        if (!need) {
          if (dir) hhi = nch; else hlo = -1;
          continue;
        }
        exact = dir ? (hc == c1) : (hc == c0 - 1);
        h = hc;
        if (dir) ++hhi; else --hlo;
        found = true;
      }
      if (!found) break;
    }
    // (k+1)-th smallest including the member itself (R3): rank k - below within this pass's list
    // r < 0: more than k values lie at or below the floor, i.e. rank k falls on the tie copies of
    // the floor value that the previous pass could not list -> eps = floor
    const int r = k - below;
    if (!done && r < 32) {
      float v = r < 0 ? floor_ : l[0];
#pragma unroll
      for (int t = 1; t < 32; ++t)
        if (t == r) v = l[t];
      e = v;
      done = true;
    }
    if (!MULTI || __all_sync(0xffffffffu, done)) break;
    floor_ = done ? INFINITY : l[31];  // finished lanes: every candidate is "below", no merges
  }
  const int valid = min(32, n - mb * 32);
  int nb = 0;
  if (lane == 0) {
    executed += (unsigned long long)ncand * (unsigned long long)valid;
    if (next_blk) nb = atomicAdd(next_blk, 1);
  }
  if (ti < n) {
    int cu, cv;
    marginal_counts(xy, sy, log2p, zi.x, zi.y, e, cu, cv);
    acc += __ldg(psi + cu + off) + __ldg(psi + cv + off);
    if (out.dbg_eps) {
      const int m = pm[ti];
      out.dbg_eps[u * n + m] = e;
      out.dbg_nx[u * n + m] = swap ? cv : cu;
      out.dbg_ny[u * n + m] = swap ? cu : cv;
    }
  }
  return __shfl_sync(0xffffffffu, nb, 0);
}

template <int K, int RM, int G, bool SWEEP>
__global__ void __launch_bounds__(RM == 1 ? 128 : 256, (K > 8 ? 4 : (RM == 1 ? (K <= 4 ? 10 : 9) : 3))) ksg_sorted_kernel(
    const float* __restrict__ Sa, const uint16_t* __restrict__ Pa, const float* __restrict__ Fa,
    const float* __restrict__ Sb, const uint16_t* __restrict__ Pb, const float* __restrict__ Fb,
    const float* __restrict__ spa, const float* __restrict__ spb, const uint8_t* __restrict__ ca,
    const uint8_t* __restrict__ cb, const double* __restrict__ psi_g, int n, int n_pad, int k, int plus1,
    PairSrc src, PairOut out) {
  constexpr int BLK = 32 * RM;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int nthreads = blockDim.x;
  const int nblk = (n + BLK - 1) / BLK;
  int log2p = 1;
  while ((1 << log2p) <= n) ++log2p;  // 2^log2p > n: +inf padded search arrays
  const int nxy = max(((n + 127) / 128) * 128, 1 << log2p);
  const int nsy = max(n_pad, 1 << log2p);
  const int nch = (n + 31) >> 5;

  // psi(m) is read through L1 from the field's fp64 table (8 KB at n = 1000, shared by all
  // CTAs of an SM): keeping it out of shared memory lets 8 CTAs fit per SM
  const double* __restrict__ psi = psi_g;
  float2* xy = reinterpret_cast<float2*>(smem_raw);
  float* sy = reinterpret_cast<float*>(xy + nxy);
  float* tb = sy + nsy;
  uint16_t* pm = reinterpret_cast<uint16_t*>(tb + n_pad);
  double* red = reinterpret_cast<double*>(pm + n_pad + 8);
  int* next_blk = reinterpret_cast<int*>(red + 32);
  uint64_t* stage_bar = reinterpret_cast<uint64_t*>(red + 33);
  float2* dupbuf = reinterpret_cast<float2*>(red + 34);  // [warps][64] (RM == 1 own chunk)

  for (int t = n_pad + threadIdx.x; t < nsy; t += nthreads) sy[t] = INFINITY;  // never overwritten
  if (threadIdx.x == 0) bar_init(stage_bar);
  __syncthreads();
  uint32_t stage_phase = 0;
  const uint32_t row_bytes = (uint32_t)n_pad * 4u;
  const double psi_nk = __ldg(psi + n) + __ldg(psi + k);
  const int off = plus1 ? 1 : 0;
  unsigned long long executed = 0, nan_pairs = 0;

  for (int64_t u = blockIdx.x; u < src.nunits; u += gridDim.x) {
    int64_t a, b, r;
    uint32_t idx;
    const bool ok = unit_pair(src, u, a, b, r, idx);
    if (!ok) {
      if (src.mode == kList && threadIdx.x == 0) out.out[u] = NAN;
      continue;
    }
    const bool degenerate = (ca[a] | cb[b]) != 0;
    if (degenerate && out.dbg_eps == nullptr) {
      if (src.mode == kList && threadIdx.x == 0) out.out[u] = NAN;
      else if (threadIdx.x == 0) ++nan_pairs;
      continue;
    }
    // sort along the wider marginal (swap roles of x and y; exact by Eq. 1 symmetry)
    const bool swap = spb[b] > spa[a];
    const float* Su = swap ? Sb + b * n_pad : Sa + a * n_pad;
    const uint16_t* Pu = swap ? Pb + b * n_pad : Pa + a * n_pad;
    const float* Fv = swap ? Fa + a * n_pad : Fb + b * n_pad;
    const float* Sv = swap ? Sa + a * n_pad : Sb + b * n_pad;
    __syncthreads();  // the previous pair is done with sy, tb, pm
    // ---- a2: stage (bulk copies by one thread; L2 prefetch of this CTA's next pair) ----
    if (threadIdx.x == 0) {
      *next_blk = nwarps;  // blocks 0..nwarps-1 are taken statically
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_expect(stage_bar, 2u * row_bytes + row_bytes / 2u);
      bulk_g2s(tb, Fv, row_bytes, stage_bar);
      bulk_g2s(sy, Sv, row_bytes, stage_bar);
      bulk_g2s(pm, Pu, row_bytes / 2u, stage_bar);
      int64_t a2, b2;
      if (u + gridDim.x < src.nunits && peek_pair(src, u + gridDim.x, a2, b2)) {
        const bool swap2 = spb[b2] > spa[a2];  // the four rows that pair will stage
        bulk_prefetch_l2(swap2 ? Sb + b2 * n_pad : Sa + a2 * n_pad, row_bytes);
        bulk_prefetch_l2(swap2 ? Pb + b2 * n_pad : Pa + a2 * n_pad, row_bytes / 2u);
        bulk_prefetch_l2(swap2 ? Fa + a2 * n_pad : Fb + b2 * n_pad, row_bytes);
        bulk_prefetch_l2(swap2 ? Sa + a2 * n_pad : Sb + b2 * n_pad, row_bytes);
      }
    }
    bar_wait(stage_bar, stage_phase);
    stage_phase ^= 1u;
    for (int q = threadIdx.x; q < nxy / 4; q += nthreads) {
      const int t = 4 * q;
      float4 xs = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
      if (t < n_pad) xs = __ldg(reinterpret_cast<const float4*>(Su) + q);
      float4* dst = reinterpret_cast<float4*>(xy + t);
      const float inf = INFINITY;
      dst[0] = make_float4(t + 0 < n ? xs.x : inf, t + 0 < n ? tb[pm[t + 0]] : inf, t + 1 < n ? xs.y : inf,
                           t + 1 < n ? tb[pm[t + 1]] : inf);
      dst[1] = make_float4(t + 2 < n ? xs.z : inf, t + 2 < n ? tb[pm[t + 2]] : inf, t + 3 < n ? xs.w : inf,
                           t + 3 < n ? tb[pm[t + 3]] : inf);
    }
    __syncthreads();

    // ---- a3 / a4 / a5 ----
    double acc = 0.0;
    // member blocks: first one static, then dynamic (sweep lengths differ per block)
    for (int mb = warp; mb < nblk;) {
      if constexpr (RM == 1 && (K == 30 || K == 31 || K == 64)) {
        // batched 32-entry lists including the member itself: K is the threshold index l[K]
        // (K = 30 for the paper's k = 30; K = 31 serves 24 < k <= 31)
        // K = 64 marks the multi-pass lists for k >= 33 (threshold index l[31])
        mb = ksg_block_big<(K < 32 ? K : 31), SWEEP, (K == 64)>(xy, sy, n, nch, log2p, mb, lane, k, psi, off, acc,
                                                                 executed, out, u, pm, swap, next_blk);
      } else {
        mb = ksg_block<K, RM, G, SWEEP, false>(xy, sy, dupbuf + warp * 64, n, nch, log2p, mb, lane, k, psi, off,
                                               acc, executed, out, u, pm, swap, next_blk);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int w = 0; w < nwarps; ++w) s += red[w];
      const float mi = degenerate ? NAN : (float)(psi_nk - s / (double)n);
      if (src.mode == kList) {
        out.out[u] = mi;
      } else if (!isnan(mi)) {
        atomicMax(out.keys + r, pack_key(out.absval ? fabsf(mi) : mi, idx));
      } else {
        ++nan_pairs;
      }
    }
  }
  if (lane == 0 && executed) atomicAdd(&g_ksg_comparisons, executed);
  if (threadIdx.x == 0 && nan_pairs) atomicAdd(&g_ksg_nan_pairs, nan_pairs);
}

template <int K, int RM, int G, bool SWEEP>
cudaError_t launch_t(const corr_field* fa, const corr_field* fb, int k, int plus1, const PairSrc& src,
                     const PairOut& out, cudaStream_t st) {
  const int n = fa->n, n_pad = fa->n_pad;
  int log2p = 1;
  while ((1 << log2p) <= n) ++log2p;
  const int nxy = std::max(((n + 127) / 128) * 128, 1 << log2p);
  const int nsy = std::max(n_pad, 1 << log2p);
  const int nblk = (n + 32 * RM - 1) / (32 * RM);
  const int wmax = RM == 1 ? 4 : 8;  // 4-warp CTAs (8/SM) for the sweep; 8-warp CTAs for the dense layout
  const int warps = nblk < wmax ? nblk : wmax;
  const size_t smem = (size_t)nxy * sizeof(float2) + (size_t)(nsy + n_pad) * sizeof(float) +
                      ((size_t)n_pad + 8) * sizeof(uint16_t) + 34 * sizeof(double) + (size_t)warps * 64 * sizeof(float2);
  auto kern = ksg_sorted_kernel<K, RM, G, SWEEP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, warps * 32, smem);
  if (occ < 1) occ = 1;
  int64_t blocks = src.nunits;
  // one pair unit per CTA (grid_waves_env): +11 % over a persistent wave for the sweep at C4
  const int waves = grid_waves_env() == -1 ? 0 : grid_waves_env();
  if (waves > 0 && blocks > (int64_t)kSMs * occ * waves) blocks = (int64_t)kSMs * occ * waves;
  if (blocks > 0x7FFFFFFF) blocks = 0x7FFFFFFF;
  kern<<<(unsigned)blocks, warps * 32, smem, st>>>(fa->S, fa->perm, fa->F, fb->S, fb->perm, fb->F, fa->spread,
                                                   fb->spread, fa->cflag, fb->cflag, fa->psi, n, n_pad, k, plus1 & 1,
                                                   src, out);
  note_launch();
  return cudaGetLastError();
}


// ---- small n (n < 128): one WARP per pair, no CTA barriers ------------------------------
// At n = 100 (the paper's usual member count) a pair is only 4 member blocks; with a CTA per
// pair the end-of-pair barrier and the staging latency dominate (ncu: 27 % barrier stalls).
// Here each warp owns its pairs end to end: two staging slots per warp, the NEXT pair's four
// rows are bulk-copied (cp.async.bulk, its own mbarrier) while the current pair is computed,
// and the psi sum is reduced with shuffles.  Same per-block code (ksg_block) as the CTA kernel.
constexpr int kWarpKernelMaxN = 127;  // 2^log2p <= 128: every per-warp array fits 4.8 KB

struct WarpSlotMeta {
  int64_t a, b, r;
  uint32_t idx;
  int flags;  // bit0 ok, bit1 degenerate, bit2 swap, bit3 rows staged
};

template <int K, bool SWEEP>
__global__ void __launch_bounds__(128, 8) ksg_warp_kernel(
    const float* __restrict__ Sa, const uint16_t* __restrict__ Pa, const float* __restrict__ Fa,
    const float* __restrict__ Sb, const uint16_t* __restrict__ Pb, const float* __restrict__ Fb,
    const float* __restrict__ spa, const float* __restrict__ spb, const uint8_t* __restrict__ ca,
    const uint8_t* __restrict__ cb, const double* __restrict__ psi, int n, int n_pad, int k, int plus1,
    PairSrc src, PairOut out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  int log2p = 1;
  while ((1 << log2p) <= n) ++log2p;
  constexpr int NXY = 128, NSY = 128;  // 2^log2p <= 128 and n_pad <= 128
  const int nblk = (n + 31) >> 5;
  const int nch = nblk;
  // per-warp layout: xy[128] float2 | dup[64] float2 | 2 slots x {sy[128], tb[n_pad], su[n_pad], pm[n_pad+8]}
  //                  | meta[2] | bar[2]
  const int slot_bytes = NSY * 4 + 2 * n_pad * 4 + (n_pad + 8) * 2;
  const int warp_bytes = NXY * 8 + 64 * 8 + 2 * slot_bytes + 2 * (int)sizeof(WarpSlotMeta) + 16;
  unsigned char* wb = smem_raw + warp * ((warp_bytes + 15) & ~15);
  float2* xy = reinterpret_cast<float2*>(wb);
  float2* dup = xy + NXY;
  unsigned char* slots = reinterpret_cast<unsigned char*>(dup + 64);
  WarpSlotMeta* meta = reinterpret_cast<WarpSlotMeta*>(slots + 2 * slot_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta + 2);
  auto slot_sy = [&](int s) { return reinterpret_cast<float*>(slots + s * slot_bytes); };
  auto slot_tb = [&](int s) { return slot_sy(s) + NSY; };
  auto slot_su = [&](int s) { return slot_tb(s) + n_pad; };
  auto slot_pm = [&](int s) { return reinterpret_cast<uint16_t*>(slot_su(s) + n_pad); };

  for (int s = 0; s < 2; ++s)
    for (int t = n_pad + lane; t < NSY; t += 32) slot_sy(s)[t] = INFINITY;  // never overwritten
  if (lane == 0) {
    bar_init(bars + 0);
    bar_init(bars + 1);
  }
  __syncwarp();
  const uint32_t row_bytes = (uint32_t)n_pad * 4u;
  const double psi_nk = __ldg(psi + n) + __ldg(psi + k);
  const int off = plus1 ? 1 : 0;
  unsigned long long executed = 0, nan_pairs = 0;
  const int64_t W = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t u0 = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;

  // lane 0: resolve unit u into slot s and start its four row copies
  auto issue = [&](int s, int64_t u) {
    WarpSlotMeta m;
    const bool ok = unit_pair(src, u, m.a, m.b, m.r, m.idx);
    m.flags = ok ? 1 : 0;
    if (ok) {
      const bool degenerate = (ca[m.a] | cb[m.b]) != 0;
      const bool swap = spb[m.b] > spa[m.a];
      m.flags |= (degenerate ? 2 : 0) | (swap ? 4 : 0);
      if (!degenerate || out.dbg_eps != nullptr) {
        m.flags |= 8;
        const float* Su = swap ? Sb + m.b * n_pad : Sa + m.a * n_pad;
        const uint16_t* Pu = swap ? Pb + m.b * n_pad : Pa + m.a * n_pad;
        const float* Fv = swap ? Fa + m.a * n_pad : Fb + m.b * n_pad;
        const float* Sv = swap ? Sa + m.a * n_pad : Sb + m.b * n_pad;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        bar_expect(bars + s, 3u * row_bytes + row_bytes / 2u);
        bulk_g2s(slot_sy(s), Sv, row_bytes, bars + s);
        bulk_g2s(slot_tb(s), Fv, row_bytes, bars + s);
        bulk_g2s(slot_su(s), Su, row_bytes, bars + s);
        bulk_g2s(slot_pm(s), Pu, row_bytes / 2u, bars + s);
      }
    }
    meta[s] = m;
  };

  if (lane == 0 && u0 < src.nunits) issue(0, u0);
  uint32_t phase = 0;  // bit s = parity of slot s's next completion
  int it = 0;
  for (int64_t u = u0; u < src.nunits; u += W, ++it) {
    const int s = it & 1;
    if (lane == 0 && u + W < src.nunits) issue(s ^ 1, u + W);
    __syncwarp();
    const WarpSlotMeta m = meta[s];
    if (!(m.flags & 1) || !(m.flags & 8)) {  // invalid / self pair, or degenerate without debug dump
      if (src.mode == kList && lane == 0) out.out[u] = NAN;
      else if (lane == 0 && (m.flags & 1)) ++nan_pairs;  // a constant series: NaN, skipped
      __syncwarp();
      continue;
    }
    bar_wait(bars + s, (phase >> s) & 1u);
    phase ^= 1u << s;
    const bool swap = (m.flags & 4) != 0;
    const float* sy = slot_sy(s);
    const float* tb = slot_tb(s);
    const float* su = slot_su(s);
    const uint16_t* pm = slot_pm(s);
    for (int t = lane; t < NXY; t += 32)
      xy[t] = t < n ? make_float2(su[t], tb[pm[t]]) : make_float2(INFINITY, INFINITY);
    __syncwarp();
    double acc = 0.0;
    for (int mb = 0; mb < nblk; ++mb)
      ksg_block<K, 1, 4, SWEEP, true>(xy, sy, dup, n, nch, log2p, mb, lane, k, psi, off, acc, executed, out, u, pm, swap,
                                      nullptr);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const float mi = (m.flags & 2) ? NAN : (float)(psi_nk - acc / (double)n);
      if (src.mode == kList) {
        out.out[u] = mi;
      } else if (!isnan(mi)) {
        atomicMax(out.keys + m.r, pack_key(out.absval ? fabsf(mi) : mi, m.idx));
      } else {
        ++nan_pairs;
      }
    }
    __syncwarp();  // slot s and xy are free: the next iteration's issue may overwrite slot s
  }
  if (lane == 0 && executed) atomicAdd(&g_ksg_comparisons, executed);
  if (lane == 0 && nan_pairs) atomicAdd(&g_ksg_nan_pairs, nan_pairs);
}

template <int K, bool SWEEP>
cudaError_t launch_warp(const corr_field* fa, const corr_field* fb, int k, int plus1, const PairSrc& src,
                        const PairOut& out, cudaStream_t st) {
  const int n = fa->n, n_pad = fa->n_pad;
  const int slot_bytes = 128 * 4 + 2 * n_pad * 4 + (n_pad + 8) * 2;
  const int warp_bytes = (128 * 8 + 64 * 8 + 2 * slot_bytes + 2 * (int)sizeof(WarpSlotMeta) + 16 + 15) & ~15;
  const size_t smem = (size_t)4 * warp_bytes;
  auto kern = ksg_warp_kernel<K, SWEEP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, smem);
  if (occ < 1) occ = 1;
  int64_t blocks = (src.nunits + 3) / 4;
  // 32 waves of warps looping over pairs (keeps each warp's two-slot staging pipeline, adds the
  // block scheduler's balancing): +13 % over one persistent wave at C3 (grid_waves_env)
  const int waves = grid_waves_env() == -1 ? 32 : grid_waves_env();
  if (waves > 0 && blocks > (int64_t)kSMs * occ * waves) blocks = (int64_t)kSMs * occ * waves;
  if (blocks > 0x7FFFFFFF) blocks = 0x7FFFFFFF;
  kern<<<(unsigned)blocks, 128, smem, st>>>(fa->S, fa->perm, fa->F, fb->S, fb->perm, fb->F, fa->spread, fb->spread,
                                            fa->cflag, fb->cflag, fa->psi, n, n_pad, k, plus1 & 1, src, out);
  note_launch();
  return cudaGetLastError();
}

template <int K>
cudaError_t launch_k(const corr_field* fa, const corr_field* fb, int k, int plus1, const PairSrc& src,
                     const PairOut& out, cudaStream_t st) {
  // Default: the exact sweep with one member per lane (RM = 1).  CORR_F_KSG_DENSE (plus1 bit 1)
  // evaluates all n(n-1) comparisons with the 4-members-per-lane layout (the faster dense form).
  if (fa->n <= kWarpKernelMaxN)
    return (plus1 & 2) ? launch_warp<K, false>(fa, fb, k, plus1, src, out, st)
                       : launch_warp<K, true>(fa, fb, k, plus1, src, out, st);
  if (plus1 & 2) return launch_t<K, 4, 4, false>(fa, fb, k, plus1, src, out, st);
  return launch_t<K, 1, 4, true>(fa, fb, k, plus1, src, out, st);
}

}  // namespace

cudaError_t launch_ksg(const corr_field* fa, const corr_field* fb, int k, bool plus1_flag, KsgPath path, bool count,
                       const PairSrc& src, const PairOut& out, cudaStream_t st) {
  if (src.nunits == 0) return cudaSuccess;
  static const bool env_sweep = [] {
    const char* v = getenv("CORR_KSG_PATH");
    return v && v[0] == 's';
  }();
  if (path == kKsgAuto && env_sweep) path = kKsgSweep;
  if (path == kKsgAuto && fa->n > kWarpKernelMaxN && k <= 8) return launch_ksg_cell(fa, fb, k, plus1_flag, count, src, out, st);
  // internal plumbing of the ksg.cu launchers: bit 0 = psi(n+1) variant, bit 1 = dense
  const int plus1 = (plus1_flag ? 1 : 0) | (path == kKsgDense ? 2 : 0);
  switch (k) {
    case 1: return launch_k<1>(fa, fb, k, plus1, src, out, st);
    case 2: return launch_k<2>(fa, fb, k, plus1, src, out, st);
    case 3: return launch_k<3>(fa, fb, k, plus1, src, out, st);
    case 4: return launch_k<4>(fa, fb, k, plus1, src, out, st);
    case 5: return launch_k<5>(fa, fb, k, plus1, src, out, st);
    case 6: return launch_k<6>(fa, fb, k, plus1, src, out, st);
    case 7: return launch_k<7>(fa, fb, k, plus1, src, out, st);
    case 8: return launch_k<8>(fa, fb, k, plus1, src, out, st);
    default: break;
  }
  // NEXT #2 (paper default k = ceil(3n/100)): register lists of 12/16/24/32;
  // inserting d >= l[KT-1] >= l[k-1] cannot change the k smallest, so the filter and the sweep
  // stay exact with the longer list, and eps = l[k-1].
  const bool sweep = !(plus1 & 2);
  if (k <= 12) return sweep ? launch_t<12, 1, 4, true>(fa, fb, k, plus1, src, out, st)
                            : launch_t<12, 1, 4, false>(fa, fb, k, plus1, src, out, st);
  if (k <= 16) return sweep ? launch_t<16, 1, 4, true>(fa, fb, k, plus1, src, out, st)
                            : launch_t<16, 1, 4, false>(fa, fb, k, plus1, src, out, st);
  if (k <= 24) return sweep ? launch_t<24, 1, 4, true>(fa, fb, k, plus1, src, out, st)
                            : launch_t<24, 1, 4, false>(fa, fb, k, plus1, src, out, st);
  // 24 < k <= 31 (k = 30 is the paper's rule ceil(3n/100) at n = 1000, Table 1): batched
  // 32-entry lists (ksg_block_big); k = 30 gets its own threshold index l[30]
  if (k == 30) return sweep ? launch_t<30, 1, 4, true>(fa, fb, k, plus1, src, out, st)
                            : launch_t<30, 1, 4, false>(fa, fb, k, plus1, src, out, st);
  if (k <= 31) return sweep ? launch_t<31, 1, 4, true>(fa, fb, k, plus1, src, out, st)
                            : launch_t<31, 1, 4, false>(fa, fb, k, plus1, src, out, st);
  if (k <= 32) return sweep ? launch_t<32, 1, 4, true>(fa, fb, k, plus1, src, out, st)
                            : launch_t<32, 1, 4, false>(fa, fb, k, plus1, src, out, st);
  // k >= 33 (up to n - 1): multi-pass 32-entry batched lists (ksg_block_big<31, SWEEP, true>)
  return sweep ? launch_t<64, 1, 4, true>(fa, fb, k, plus1, src, out, st)
               : launch_t<64, 1, 4, false>(fa, fb, k, plus1, src, out, st);
}

cudaError_t ksg_cell_comparisons(unsigned long long* value, bool reset);
cudaError_t ksg_cell_nan_pairs(unsigned long long* value, bool reset);

cudaError_t ksg_nan_pairs(unsigned long long* value, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(value, g_ksg_nan_pairs, sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long zero = 0;
    e = cudaMemcpyToSymbol(g_ksg_nan_pairs, &zero, sizeof(zero));
  }
  unsigned long long cell = 0;
  if (e == cudaSuccess) e = ksg_cell_nan_pairs(&cell, reset);
  *value += cell;
  return e;
}

cudaError_t ksg_comparisons(unsigned long long* value, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(value, g_ksg_comparisons, sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long zero = 0;
    e = cudaMemcpyToSymbol(g_ksg_comparisons, &zero, sizeof(zero));
  }
  unsigned long long cell = 0;
  if (e == cudaSuccess) e = ksg_cell_comparisons(&cell, reset);
  *value += cell;
  return e;
}

}  // namespace corr
