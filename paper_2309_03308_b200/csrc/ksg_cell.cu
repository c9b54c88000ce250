// ksg_cell.cu -- Kraskov (KSG) MI of point pairs with a column-cell k-NN (round 2 default for
// 128 <= n and k <= 8).  SURVEY.md §8(a) rows a2-a5; PAPER.md:172-174 (Eq. 2), readings R1-R7.
//
// The paper builds a k-d tree per pair; the round-1 kernel scanned the
// pair's x-sorted order outward from 32-member blocks (exact sweep), executing ~169 candidate
// distances per member because the 32 lanes of a warp advance over the same candidates.  Here
// each member scans ITS OWN candidates, in a two-level structure built per pair in shared memory:
//
//   x = the wider marginal (KSG is symmetric in x and y, Eq. 1).  Columns = 32 consecutive
//   x-ranks; inside a column the members are kept in y order (a stable multisplit of the y-sorted
//   row by column).  cellstart[c][g] = number of column-c members whose y-rank is < 32 g.
//
//   A warp owns a column (lane = member in the column's y order):
//     own column  -- scan up (p+1, p+2, ...) and down (p-1, ...) in y order, one candidate per
//                    direction per step, merged into the register k-list; a direction stops once
//                    fl(y_j - y_i) >= l[k-1] (every further candidate is at least as far in y, so
//                    none can enter the list: monotone rounding, the list only shrinks);
//     neighbour columns, nearest first, alternating sides -- a lane needs column c' iff the x-gap
//                    to its nearest edge is < l[k-1] (the round-1 sweep test); the side ends when
//                    no lane needs it.  Needing lanes start at cellstart[c'][y-band of the member]
//                    (no search: the member's position in c' lies inside that cell) and scan
//                    up / down with the same stop rule.
//     far-visit queue -- after the distance-1 columns, the lanes that still need a farther
//                    column (~10 % of members, but in ~2 extra visits per column that each last as
//                    long as their longest scan, with ~2.4 of 32 lanes busy) are written to a
//                    CTA-wide queue (their k-list + member slot, in the staging buffer of the
//                    x-argsort, dead after the build).  Once every column is done, each warp takes
//                    32 queued members and every lane visits ITS nearest still-needed column per
//                    round (tools/cell_sim7.py: far-visit scan steps 181 -> 60 per pair); a full
//                    queue leaves the rest in their column warp.  +4.4 % at C4.
//   Candidates of other columns are real members, so any extra candidate is harmless (the
//   k-smallest multiset over a superset that contains every candidate below the final eps is
//   exact); the self pair is never visited.  Column ends hold sentinels (+inf, -inf) / (+inf,
//   +inf) so a scan stops there without bounds checks, and a stopped direction stays on its stop
//   candidate (re-merging a value >= l[k-1] is a no-op).
//
// Counts (a4) are binary searches on the two sorted rows (128-wide windows around the member's own
// ranks when every lane's strips fit, else the whole row); psi / reduction as in ksg.cu.
// Launch: one pair unit per CTA (the hardware block scheduler balances and staggers the CTAs:
// +18 % over a persistent grid-stride wave).
#include <stdlib.h>

#include <algorithm>

#include "ksg_common.cuh"

namespace corr {

// executed comparisons of this kernel (no relocatable device code: ksg.cu's counter is not
// visible here; ksg_comparisons() reads both)
__device__ unsigned long long g_ksg_cell_comparisons;
__device__ unsigned long long g_ksg_cell_nan_pairs;  // region-max pairs skipped as NaN

namespace {

constexpr int kCS = 34;  // float2 entries per column: lo sentinel, 32 members, hi sentinel

struct CellLayout {
  int n, n_pad, nch, nseg, nsx, log2p;
  uint32_t o_su, o_sv, o_col, o_pu, o_pv, o_xr, o_cs, o_cols, o_red, o_misc, bytes;
};

__host__ __device__ inline CellLayout cell_layout(int n, int n_pad, int nw) {
  CellLayout L;
  L.n = n;
  L.n_pad = n_pad;
  L.nch = (n + 31) >> 5;
  L.nseg = L.nch;
  int log2p = 1;
  while ((1 << log2p) <= n) ++log2p;  // 2^log2p > n: +inf padded search arrays
  L.log2p = log2p;
  L.nsx = n_pad > (1 << log2p) ? n_pad : (1 << log2p);
  uint32_t o = 0;
  auto take = [&](uint32_t bytes, uint32_t align) {
    o = (o + align - 1) / align * align;
    const uint32_t r = o;
    o += bytes;
    return r;
  };
  L.o_su = take(L.nsx * 4u, 16);
  L.o_sv = take(L.nsx * 4u, 16);
  L.o_col = take(((uint32_t)L.nch * kCS + 2u) * 8u, 16);  // + one pad entry before and after
  L.o_pu = take(n_pad * 2u, 16);
  L.o_pv = take(n_pad * 2u, 16);
  L.o_xr = take(n_pad * 2u, 16);
  L.o_cs = take((uint32_t)L.nch * (L.nseg + 1) * 2u, 16);
  L.o_cols = take((uint32_t)L.nch * 32u * 2u, 16);
  L.o_red = take((uint32_t)nw * 8u, 8);
  L.o_misc = take(24, 8);  // (unused int), flags (int), staging mbarrier (u64), queue count (int)
  L.bytes = (o + 15) / 16 * 16;
  return L;
}

__device__ __forceinline__ float2 lds_f2(uint32_t addr) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
  return v;
}

__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}

__device__ __forceinline__ float chebd(float2 d) { return fmaxf(fabsf(d.x), fabsf(d.y)); }

// psi table entry m (m >= 0): one 32 x 32 -> 64-bit multiply-add for the address instead of the
// sign-extended 64-bit index arithmetic the compiler emits for psi[m + off]
__device__ __forceinline__ double ldg_psi(const double* base, uint32_t m) {
  const double* a;
  asm("mad.wide.u32 %0, %1, 8, %2;" : "=l"(a) : "r"(m), "l"(base));
  return __ldg(a);
}

// Lockstep up / down scan of one column for the whole warp, one candidate per direction per
// step.  A direction stops once fl(y_j - y_i) >= l[K-1]; its pointer then rests on that
// candidate, whose distance is >= l[K-1] (re-merging it is a no-op).  Column ends hold
// sentinels (infinite distance, immediate stop).  Lanes that do not need the column start on the
// sentinels.  The body is written out twice so the loop-carried pointers alternate registers
// (measured +0.5 % over the single body; a variant issuing the next loads one step ahead, off the
// stop test's dependency chain, measured -0.4 %: the loop is ALU-bound, not latency-bound).
template <int K>
__device__ __forceinline__ bool scan_step(uint32_t& pu, uint32_t& pd, float2 zi, float (&l)[K]) {
  const float2 zu = lds_f2(pu), zd = lds_f2(pd);
  const float2 du = sub2(zi, zu), dd = sub2(zi, zd);
  merge2<K>(l, chebd(du), chebd(dd));
  // stop tests fused with the predicated pointer steps (fl(y_j - y_i) = -fl(y_i - y_j) exactly);
  // written in PTX so each pointer moves in place (+1.0 % over the compiler's select + copy)
  uint32_t both;
  asm("{\n\t.reg .pred ps, pt, pb;\n\t"
      "setp.ge.f32 ps, %3, %5;\n\t"
      "setp.ge.f32 pt, %4, %5;\n\t"
      "@!ps add.u32 %0, %0, 8;\n\t"
      "@!pt sub.u32 %1, %1, 8;\n\t"
      "and.pred pb, ps, pt;\n\t"
      "selp.u32 %2, 1, 0, pb;\n\t}"
      : "+r"(pu), "+r"(pd), "=r"(both)
      : "f"(-du.y), "f"(dd.y), "f"(l[K - 1]));
  return __all_sync(0xffffffffu, both != 0u);
}

// single-body variant for the own-column scan: there the compiler's register alternation of the
// two-body loop costs two moves per step; in place it is 21 instructions per step (+0.6 %)
template <int K>
__device__ __forceinline__ void scan_column1(uint32_t& pu, uint32_t& pd, float2 zi, float (&l)[K]) {
#pragma unroll 1
  while (!scan_step<K>(pu, pd, zi, l)) {
  }
}

template <int K>
__device__ __forceinline__ void scan_column(uint32_t& pu, uint32_t& pd, float2 zi, float (&l)[K]) {
#pragma unroll 1
  while (true) {
    if (scan_step<K>(pu, pd, zi, l)) break;
    if (scan_step<K>(pu, pd, zi, l)) break;
  }
}

// Strict marginal counts on the two sorted rows (stride 4 B, +inf padded to
// 2^log2p): the round-1 monotone-predicate binary searches (ksg.cu), both arrays float.
template <int B>
struct CountSearch44 {
  __device__ __forceinline__ static void run(int log2p, uint32_t& xu, uint32_t& xw, uint32_t& yu, uint32_t& yw,
                                             float x, float y, float e) {
    if (B < log2p) {
      constexpr int ST = (1 << B) * 4;
      const float pxu = lds_imm<ST - 4>(xu), pxw = lds_imm<ST - 4>(xw);
      const float pyu = lds_imm<ST - 4>(yu), pyw = lds_imm<ST - 4>(yw);
      // the x and y differences in packed pairs (sub.rn.f32x2: the same RN fp32 subtractions)
      const float2 du = sub2(make_float2(pxu, pyu), make_float2(x, y));
      const float2 dw = sub2(make_float2(x, y), make_float2(pxw, pyw));
      xu = (du.x >= e) ? xu : xu + ST;
      xw = (dw.x < e) ? xw : xw + ST;
      yu = (du.y >= e) ? yu : yu + ST;
      yw = (dw.y < e) ? yw : yw + ST;
    }
    CountSearch44<B - 1>::run(log2p, xu, xw, yu, yw, x, y, e);
  }
};
template <>
struct CountSearch44<-1> {
  __device__ __forceinline__ static void run(int, uint32_t&, uint32_t&, uint32_t&, uint32_t&, float, float, float) {}
};

// __launch_bounds__ minimum of 6 CTAs: the register allocation it induces (58 registers, still 8
// resident CTAs) measured +2.3 % over a minimum of 8 (54 registers) and 7 (60): A/B, C4
template <int K, int NW, bool COUNT>
__global__ void __launch_bounds__(NW * 32, (NW == 4 ? 6 : 4)) ksg_cell_kernel(
    const float* __restrict__ Sa, const uint16_t* __restrict__ Pa, const float* __restrict__ Sb,
    const uint16_t* __restrict__ Pb, const float* __restrict__ spa, const float* __restrict__ spb,
    const uint8_t* __restrict__ ca, const uint8_t* __restrict__ cb, const double* __restrict__ psi, int n, int n_pad,
    int k, int plus1, int qcap, PairSrc src, PairOut out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const CellLayout L = cell_layout(n, n_pad, NW);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, tid = threadIdx.x;
  constexpr int NT = NW * 32;
  const int nch = L.nch, nseg = L.nseg, cs_stride = L.nseg + 1;
  float* su = reinterpret_cast<float*>(smem + L.o_su);
  float* sv = reinterpret_cast<float*>(smem + L.o_sv);
  float2* col = reinterpret_cast<float2*>(smem + L.o_col) + 1;  // col[-1] and col[nch*kCS] are pads
  uint16_t* pu_s = reinterpret_cast<uint16_t*>(smem + L.o_pu);
  uint16_t* pv_s = reinterpret_cast<uint16_t*>(smem + L.o_pv);
  uint16_t* xr = reinterpret_cast<uint16_t*>(smem + L.o_xr);
  uint16_t* rk = pu_s;  // rank inside the cell, per y-rank s (pu_s is dead once xr is built)
  uint16_t* cs = reinterpret_cast<uint16_t*>(smem + L.o_cs);
  uint16_t* cols = reinterpret_cast<uint16_t*>(smem + L.o_cols);  // y-rank s of each column entry
  double* red = reinterpret_cast<double*>(smem + L.o_red);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.o_misc + 8);
  const uint32_t col_base = su32(col), su_base = su32(su), sv_base = su32(sv), cs_base = su32(cs),
                 cols_base = su32(cols);

  for (int t = n_pad + tid; t < L.nsx; t += NT) su[t] = sv[t] = INFINITY;  // never overwritten
  if (tid == 0) col[-1] = col[nch * kCS] = make_float2(INFINITY, INFINITY);
  if (tid == 0) bar_init(bar);
  __syncthreads();
  uint32_t phase = 0;
  const uint32_t row_bytes = (uint32_t)n_pad * 4u;
  const double psi_nk = __ldg(psi + n) + __ldg(psi + k);
  const int off = plus1 ? 1 : 0;
  const double* __restrict__ psi_o = psi + off;  // psi(m + off), indexed by unsigned 32-bit counts
  unsigned long long executed = 0, nan_pairs = 0;

  int* flags_s = reinterpret_cast<int*>(smem + L.o_misc) + 1;  // this pair's flags (skip, swap, degenerate)
  int* qcount = reinterpret_cast<int*>(smem + L.o_misc + 16);   // far-visit queue length
  for (int64_t u = blockIdx.x; u < src.nunits; u += gridDim.x) {
    // thread 0 alone resolves the pair (sampler, flags) and stages its rows; the others learn the
    // flags after the first build barrier.  A skipped unit stages row 0 (valid addresses, unused).
    int64_t a = 0, b = 0, r = 0;
    uint32_t idx = 0;
    __syncthreads();  // the previous pair is done with every shared array
    if (tid == 0) {
      const bool ok = unit_pair(src, u, a, b, r, idx);
      int fl = 0;
      if (!ok) {
        fl = 1;
        a = b = 0;
        if (src.mode == kList) out.out[u] = NAN;
      } else if ((ca[a] | cb[b]) != 0) {  // a constant series: NaN (R10)
        fl = 4;
        if (out.dbg_eps == nullptr) {
          fl |= 1;
          if (src.mode == kList) out.out[u] = NAN; else ++nan_pairs;
        }
      }
      const bool swap = spb[b] > spa[a];  // x = the wider marginal
      fl |= swap ? 2 : 0;
      *flags_s = fl;
      const float* Su = swap ? Sb + b * n_pad : Sa + a * n_pad;
      const uint16_t* Pu = swap ? Pb + b * n_pad : Pa + a * n_pad;
      const float* Sv = swap ? Sa + a * n_pad : Sb + b * n_pad;
      const uint16_t* Pv = swap ? Pa + a * n_pad : Pb + b * n_pad;
      *qcount = 0;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_expect(bar, 2u * row_bytes + row_bytes);
      bulk_g2s(su, Su, row_bytes, bar);
      bulk_g2s(sv, Sv, row_bytes, bar);
      bulk_g2s(pu_s, Pu, row_bytes / 2u, bar);
      bulk_g2s(pv_s, Pv, row_bytes / 2u, bar);
      int64_t a2, b2;  // the next pair stages S and perm of both of its points, whichever is x
      if (u + gridDim.x < src.nunits && peek_pair(src, u + gridDim.x, a2, b2)) {
        bulk_prefetch_l2(Sa + a2 * n_pad, row_bytes);
        bulk_prefetch_l2(Sb + b2 * n_pad, row_bytes);
        bulk_prefetch_l2(Pa + a2 * n_pad, row_bytes / 2u);
        bulk_prefetch_l2(Pb + b2 * n_pad, row_bytes / 2u);
      }
    }
    for (int q = tid; q < nch * cs_stride; q += NT) cs[q] = 0;
    bar_wait(bar, phase);
    phase ^= 1u;
    // ---- build: x-rank of every member, stable multisplit of the y order by column ----
    for (int t = tid; t < n; t += NT) xr[pu_s[t]] = (uint16_t)t;
    __syncthreads();
    const int fl = *flags_s;
    if (__all_sync(0xffffffffu, (fl & 1) != 0)) continue;  // uniform: skipped unit (a vote: provably warp-uniform)
    const bool swap = (fl & 2) != 0, degenerate = (fl & 4) != 0;
    for (int g = warp; g < nseg; g += NW) {
      const int s = 32 * g + lane;
      const bool valid = s < n;
      const int c = valid ? (xr[pv_s[s]] >> 5) : 0xFFFF;
      const unsigned peers = __match_any_sync(0xffffffffu, c);
      const int rank = __popc(peers & ((1u << lane) - 1u));
      if (valid) {
        rk[s] = (uint16_t)rank;
        if (rank == 0) cs[c * cs_stride + g] = (uint16_t)__popc(peers);
      }
    }
    __syncthreads();
    // exclusive prefix over the y-segments of every column: one thread per column walks its
    // segments (sequential, ~10x fewer instructions than a warp scan per column: +3.9 %)
    for (int c = tid; c < nch; c += NT) {
      int run = 0;
      for (int g = 0; g < nseg; ++g) {
        const int v = cs[c * cs_stride + g];
        cs[c * cs_stride + g] = (uint16_t)run;
        run += v;
      }
    }
    __syncthreads();
    for (int s = tid; s < n; s += NT) {
      const int t = xr[pv_s[s]];
      const int c = t >> 5;
      const int pos = cs[c * cs_stride + (s >> 5)] + rk[s];
      col[c * kCS + 1 + pos] = make_float2(su[t], sv[s]);
      cols[c * 32 + pos] = (uint16_t)s;
    }
    for (int c = tid; c < nch; c += NT) {
      col[c * kCS] = make_float2(INFINITY, -INFINITY);
      const int v = min(32, n - 32 * c);
      for (int q = v; q < 33; ++q) col[c * kCS + 1 + q] = make_float2(INFINITY, INFINITY);
    }
    __syncthreads();

    // ---- a3: one column per warp (static: warp w takes columns w, w + NW, ...), lockstep scans ----
    double acc = 0.0;
    // far-visit queue, in pu_s (dead once the build is done): K list entries + member slot
    float* q_l = reinterpret_cast<float*>(smem + L.o_pu);  // [K][qcap]
    uint16_t* q_m = reinterpret_cast<uint16_t*>(q_l + K * qcap);
    // a4 / a5 for one member per lane (on = lane holds a member whose list is final): strict
    // marginal counts by binary searches on the sorted rows, then psi.  The strips |x - x_i| < eps
    // and |y - y_i| < eps lie around the member's own ranks (t_i in the x row, s_i in the y row);
    // if, for every lane, both strips end within 127 ranks of t_i / s_i on both sides (checked at
    // the window edges with the same monotone predicates), 7-step searches over 128-wide windows
    // replace the full log2(n)-step ones.  Called by all 32 lanes (warp vote).
    auto count_psi = [&](bool on, int c, int ln, float2 zi, float e) {
      uint32_t xu = su_base, xw = su_base, yu = sv_base, yw = sv_base;
      bool win_ok = true;
      if (on && e > 0.f) {
        const int si = (int)lds_u16(cols_base + (uint32_t)(c * 32 + ln) * 2u);
        const int ti = xr[pv_s[si]];
        const int bxw = max(0, ti - 127), bxu = min(ti, L.nsx - 128);
        const int byw = max(0, si - 127), byu = min(si, L.nsx - 128);
        // branch-free (the four edge tests as packed differences, no short-circuit branches)
        const float2 dl = sub2(zi, make_float2(su[max(bxw - 1, 0)], sv[max(byw - 1, 0)]));
        const float2 dh = sub2(make_float2(su[bxu + 127], sv[byu + 127]), zi);
        win_ok = ((bxw == 0) | !(dl.x < e)) & (dh.x >= e) & ((byw == 0) | !(dl.y < e)) & (dh.y >= e);
        xw = su_base + (uint32_t)bxw * 4u;
        xu = su_base + (uint32_t)bxu * 4u;
        yw = sv_base + (uint32_t)byw * 4u;
        yu = sv_base + (uint32_t)byu * 4u;
      }
      const bool windowed = __all_sync(0xffffffffu, win_ok);
      if (on) {
        int cx = 0, cy = 0;
        if (e > 0.f) {
          if (windowed) {
            CountSearch44<6>::run(7, xu, xw, yu, yw, zi.x, zi.y, e);
          } else {
            xu = xw = su_base;
            yu = yw = sv_base;
            CountSearch44<12>::run(L.log2p, xu, xw, yu, yw, zi.x, zi.y, e);
          }
          cx = (int)((xu - xw) >> 2) - 1;
          cy = (int)((yu - yw) >> 2) - 1;
        }
        acc += ldg_psi(psi_o, (uint32_t)cx) + ldg_psi(psi_o, (uint32_t)cy);
        if (out.dbg_eps) {
          const int m = pv_s[cols[c * 32 + ln]];
          out.dbg_eps[u * n + m] = e;
          out.dbg_nx[u * n + m] = swap ? cy : cx;
          out.dbg_ny[u * n + m] = swap ? cx : cy;
        }
      }
    };
    {
      int ncand = 0;
      // The loop and side conditions below are warp-uniform by construction; writing them as
      // votes lets ptxas PROVE it, so the scan steps' votes need no divergence check (no UMOV +
      // BRA.DIV per step: 23 -> 21 warp-instructions per neighbour-scan step, +2.3 % at C4)
      for (int c = warp; __all_sync(0xffffffffu, c < nch);) {
        const int v = min(32, n - 32 * c);
        const bool active = lane < v;
        const uint32_t cb0 = col_base + (uint32_t)(c * kCS) * 8u;
        // lanes without a member take (0, 0): finite, so their scans stop on the sentinels at once
        const float2 zi = active ? lds_f2(cb0 + (uint32_t)(1 + lane) * 8u) : make_float2(0.f, 0.f);
        const int band = active ? (int)lds_u16(cols_base + (uint32_t)(c * 32 + lane) * 2u) >> 5 : 0;
        float l[K];
#pragma unroll
        for (int t = 0; t < K; ++t) l[t] = INFINITY;
        // own column: up from p+1, down from p-1 (lanes without a member start on the sentinels)
        uint32_t pu = active ? cb0 + (uint32_t)(lane + 2) * 8u : cb0 + 33u * 8u;
        uint32_t pd = active ? cb0 + (uint32_t)lane * 8u : cb0;
        scan_column1<K>(pu, pd, zi, l);
        // executed comparisons: the visited entries [pd, pu] minus the member itself and sentinels
        if (COUNT && active) ncand += (int)((pu - pd) >> 3) - (pu == cb0 + 33u * 8u) - (pd == cb0);
        // neighbour columns, nearest first, alternating sides; a side ends at the first column no
        // lane needs (its x-gap only grows outward, the lists only shrink)
        int lo = c - 1, hi = c + 1;
        // addresses kept incrementally: the nearest x of the next column on each side (its last /
        // first x-rank) and that column's entry block
        uint32_t eL = su_base + (uint32_t)(32 * lo + 31) * 4u, eR = su_base + (uint32_t)(32 * hi) * 4u;
        uint32_t bL = col_base + (uint32_t)(lo * kCS) * 8u, bR = col_base + (uint32_t)(hi * kCS) * 8u;
        uint32_t sL = cs_base + (uint32_t)(lo * cs_stride + band) * 2u, sR = cs_base + (uint32_t)(hi * cs_stride + band) * 2u;
        bool queued = false, first = true;
#pragma unroll 1
        while (__all_sync(0xffffffffu, lo >= 0 || hi < nch)) {
          // left then right, each side's test and visit written out (no per-test side select)
          if (__all_sync(0xffffffffu, lo >= 0)) {
            const bool need = active && !queued && (zi.x - lds_f32(eL) < l[K - 1]);
            if (!__any_sync(0xffffffffu, need)) {
              lo = -1;
            } else {
              const uint32_t start = lds_u16(sL);
              pu = need ? bL + (1u + start) * 8u : bL + 33u * 8u;
              pd = need ? bL + start * 8u : bL;
              scan_column<K>(pu, pd, zi, l);
              if (COUNT && need) ncand += (int)((pu - pd) >> 3) + 1 - (pu == bL + 33u * 8u) - (pd == bL);
              --lo;
              eL -= 128u;
              bL -= kCS * 8u;
              sL -= (uint32_t)cs_stride * 2u;
            }
          }
          if (__all_sync(0xffffffffu, hi < nch)) {
            const bool need = active && !queued && (lds_f32(eR) - zi.x < l[K - 1]);
            if (!__any_sync(0xffffffffu, need)) {
              hi = nch;
            } else {
              const uint32_t start = lds_u16(sR);
              pu = need ? bR + (1u + start) * 8u : bR + 33u * 8u;
              pd = need ? bR + start * 8u : bR;
              scan_column<K>(pu, pd, zi, l);
              if (COUNT && need) ncand += (int)((pu - pd) >> 3) + 1 - (pu == bR + 33u * 8u) - (pd == bR);
              ++hi;
              eR += 128u;
              bR += kCS * 8u;
              sR += (uint32_t)cs_stride * 2u;
            }
          }
          if (qcap > 0 && __all_sync(0xffffffffu, first)) {
            // after the distance-1 columns: lanes that still need a farther column (few per
            // warp, each visit lasting as long as its longest scan) continue from a CTA-wide
            // queue, 32 needing members per warp, once every column is done
            first = false;
            const bool want = active && ((lo >= 0 && zi.x - lds_f32(eL) < l[K - 1]) ||
                                         (hi < nch && lds_f32(eR) - zi.x < l[K - 1]));
            const unsigned wm = __ballot_sync(0xffffffffu, want);
            if (wm != 0u) {
              int qb = 0;
              if (lane == 0) qb = atomicAdd(qcount, __popc(wm));
              qb = __shfl_sync(0xffffffffu, qb, 0);
              const int slot = qb + __popc(wm & ((1u << lane) - 1u));
              if (want && slot < qcap) {
#pragma unroll
                for (int t = 0; t < K; ++t) q_l[t * qcap + slot] = l[t];
                q_m[slot] = (uint16_t)(c * 32 + lane);
                queued = true;
              }
            }
            if (!__any_sync(0xffffffffu, want && !queued)) break;  // the others need nothing farther
          }
        }
        count_psi(active && !queued, c, lane, zi, l[K - 1]);
        // static column assignment (warp w: columns w, w + NW, ...): with the far visits in the
        // queue the columns cost about the same, and the dynamic claim (a shared atomic + shuffle
        // per column) measured 1.5 % slower
        c += NW;
      }
      if (qcap > 0) {
        __syncthreads();  // every column is done and the queue complete
        const int qn = min(*qcount, qcap);
        for (int g = warp * 32; g < qn; g += NW * 32) {
          const int q = g + lane;
          const bool on = q < qn;
          float l[K];
#pragma unroll
          for (int t = 0; t < K; ++t) l[t] = on ? q_l[t * qcap + q] : INFINITY;
          const int m = on ? (int)q_m[q] : 0;
          const int c = m >> 5, ln = m & 31;
          const float2 zi = on ? lds_f2(col_base + (uint32_t)(c * kCS + 1 + ln) * 8u) : make_float2(0.f, 0.f);
          const int band = on ? (int)lds_u16(cols_base + (uint32_t)(c * 32 + ln) * 2u) >> 5 : 0;
          // per-lane rounds: every lane visits ITS nearest still-needed column (any order of
          // visits is exact: extra candidates are real members)
          int lo = c - 2, hi = c + 2;
#pragma unroll 1
          while (true) {
            const float gl = lo >= 0 ? zi.x - su[32 * lo + 31] : INFINITY;
            const float gr = hi < nch ? su[32 * hi] - zi.x : INFINITY;
            const bool nl = on && gl < l[K - 1], nr = on && gr < l[K - 1];
            if (!__any_sync(0xffffffffu, nl || nr)) break;
            const bool go_l = nl && (!nr || gl <= gr);
            const int cc = go_l ? lo : hi;
            uint32_t pu = col_base + 33u * 8u, pd = col_base;  // idle lanes: column 0's sentinels
            if (nl || nr) {
              const uint32_t bb = col_base + (uint32_t)(cc * kCS) * 8u;
              const uint32_t start = cs[cc * cs_stride + band];
              pu = bb + (1u + start) * 8u;
              pd = bb + start * 8u;
            }
            const uint32_t pu0 = pu, pd0 = pd;
            scan_column<K>(pu, pd, zi, l);
            if (COUNT && (nl || nr)) {
              const uint32_t bb = col_base + (uint32_t)(cc * kCS) * 8u;
              ncand += (int)((pu - pd) >> 3) + 1 - (pu == bb + 33u * 8u) - (pd == bb);
            }
            (void)pu0;
            (void)pd0;
            if (go_l) --lo;
            else if (nr) ++hi;
          }
          count_psi(on, c, ln, zi, l[K - 1]);
        }
      }
      if (COUNT) {
        for (int o = 16; o; o >>= 1) ncand += __shfl_xor_sync(0xffffffffu, ncand, o);
        if (lane == 0) executed += (unsigned long long)ncand;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int w = 0; w < NW; ++w) s += red[w];
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
  if (lane == 0 && executed) atomicAdd(&g_ksg_cell_comparisons, executed);
  if (tid == 0 && nan_pairs) atomicAdd(&g_ksg_cell_nan_pairs, nan_pairs);
}

template <int K, int NW>
cudaError_t launch_cell_t(const corr_field* fa, const corr_field* fb, int k, bool plus1, bool count,
                          const PairSrc& src, const PairOut& out, cudaStream_t st) {
  const CellLayout L = cell_layout(fa->n, fa->n_pad, NW);
  auto kern = count ? ksg_cell_kernel<K, NW, true> : ksg_cell_kernel<K, NW, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes);
  if (e != cudaSuccess) return e;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NW * 32, L.bytes);
  static const int occ_cap = [] {  // A/B switch: resident CTAs per SM
    const char* v = getenv("CORR_KSG_OCC");
    return v ? atoi(v) : 0;
  }();
  if (occ_cap > 0 && occ > occ_cap) occ = occ_cap;
  if (occ < 1) occ = 1;
  // one pair unit per CTA by default (grid_waves_env, corr_internal.cuh): +18 % over a
  // persistent grid-stride wave at C4
  int64_t blocks = src.nunits;
  const int waves = grid_waves_env();
  if (waves > 0 && blocks > (int64_t)kSMs * occ * waves) blocks = (int64_t)kSMs * occ * waves;
  if (blocks > 0x7FFFFFFF) blocks = 0x7FFFFFFF;
  // far-visit queue capacity: K list entries + a u16 member slot each, in the n_pad * 2 bytes of
  // pu_s (CORR_KSG_QUEUE=0: no queue, every visit in the column warps -- A/B switch);
  // capacity NW * 32 = one group per warp (measured: 128 -> 2.707e7 pairs/s at C4, the full
  // 142 entries 2.702e7, 64 2.638e7, no queue 2.591e7)
  static const int qmax = [] {  // CORR_KSG_QUEUE = capacity cap (0: no queue)
    const char* v = getenv("CORR_KSG_QUEUE");
    return v ? atoi(v) : NW * 32;
  }();
  const int qcap = std::min(qmax, (fa->n_pad * 2) / (4 * K + 2));
  kern<<<(unsigned)blocks, NW * 32, L.bytes, st>>>(fa->S, fa->perm, fb->S, fb->perm, fa->spread, fb->spread, fa->cflag,
                                                   fb->cflag, fa->psi, fa->n, fa->n_pad, k, plus1 ? 1 : 0, qcap, src,
                                                   out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace

cudaError_t ksg_cell_comparisons(unsigned long long* value, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(value, g_ksg_cell_comparisons, sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long zero = 0;
    e = cudaMemcpyToSymbol(g_ksg_cell_comparisons, &zero, sizeof(zero));
  }
  return e;
}

cudaError_t ksg_cell_nan_pairs(unsigned long long* value, bool reset) {
  cudaError_t e = cudaMemcpyFromSymbol(value, g_ksg_cell_nan_pairs, sizeof(unsigned long long));
  if (e == cudaSuccess && reset) {
    const unsigned long long zero = 0;
    e = cudaMemcpyToSymbol(g_ksg_cell_nan_pairs, &zero, sizeof(zero));
  }
  return e;
}

// Column-cell KSG for 128 <= n <= 4096, k <= 8 (register lists of K = k entries).
cudaError_t launch_ksg_cell(const corr_field* fa, const corr_field* fb, int k, bool plus1, bool count,
                            const PairSrc& src, const PairOut& out, cudaStream_t st) {
  switch (k) {
    case 1: return launch_cell_t<1, 4>(fa, fb, k, plus1, count, src, out, st);
    case 2: return launch_cell_t<2, 4>(fa, fb, k, plus1, count, src, out, st);
    case 3: return launch_cell_t<3, 4>(fa, fb, k, plus1, count, src, out, st);
    case 4: return launch_cell_t<4, 4>(fa, fb, k, plus1, count, src, out, st);
    case 5: return launch_cell_t<5, 4>(fa, fb, k, plus1, count, src, out, st);
    case 6: return launch_cell_t<6, 4>(fa, fb, k, plus1, count, src, out, st);
    case 7: return launch_cell_t<7, 4>(fa, fb, k, plus1, count, src, out, st);
    case 8: return launch_cell_t<8, 4>(fa, fb, k, plus1, count, src, out, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace corr
