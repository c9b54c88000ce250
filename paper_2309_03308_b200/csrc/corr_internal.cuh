// corr_internal.cuh -- internal types of libcorr.so (B200 / sm_100a).
// The field layout and pair-source abstraction shared by every kernel of the hot
// path.  Nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "corr.h"

struct corr_field {
  int device;
  int nx, ny, nz;
  int n;          // members
  int n_pad;      // ceil(n/8)*8: rows are 32-byte aligned, tf32 K multiple of 8
  int64_t P;      // points
  float* F;       // [P][n_pad] member-contiguous raw values, pad = 0
  float* Z;       // [P][n_pad] (x - mean)/||x - mean|| (fp64 -> fp32), pad = 0
  float* Zhi;     // [P][n_pad] tf32(Z)               (split-TF32 high part)
  float* Zlo;     // [P][n_pad] tf32(Z - Zhi)         (split-TF32 low part)
  uint16_t* Zb;   // [P][n_pad] bf16(Z)  (screening pass of the exhaustive Pearson GEMM)
  float* S;       // [P][n_pad] row sorted ascending, pad = +inf
  uint16_t* perm; // [P][n_pad] argsort of the row (S[p][t] = F[p][perm[p][t]])
  uint8_t* cflag; // [P] 1 = constant series (min == max)
  float* spread;  // [P] ||x - mean|| (picks the sort marginal of a KSG pair)
  double* psi;    // [n + 2] digamma at integers, psi[0] = NaN
  int* err;       // device status words: err[0] bit0 = index out of range, err[1] bit1 = non-finite input
  void* tmaps;    // lazily built TMA descriptors (pearson_gemm.cu)
  // host-input streaming (api.cu ingest_values): two device slices of kStageMembers members,
  // a copy stream and the events that order copies against the transposes (lazily created)
  float* stage[2];
  cudaStream_t copy_st;
  cudaEvent_t ev_copied[2], ev_used[2];
};

#include <atomic>

namespace corr {

constexpr int kSMs = 148;

// Grid size of the pair kernels: `waves` CTAs per resident CTA slot, each CTA looping over its
// pair units with a grid stride.  Measured (round 2, ksg_cell_kernel, C4): one persistent wave
// 2.14e7 pairs/s, 16 waves 2.48e7, one unit per CTA 2.52e7 -- the hardware block scheduler's
// dynamic assignment and staggered CTA phases beat a static grid-stride split.  The environment
// variable CORR_WAVES overrides (A/B); <= 0 means one unit per CTA.
int grid_waves_env();
extern std::atomic<long long> g_launch_count;  // kernels launched (corr_launch_count)
inline void note_launch(int k = 1) { g_launch_count.fetch_add(k, std::memory_order_relaxed); }

// A region pair on the device (boxes, sizes, exhaustive offsets).  Seed-free, so the resident
// table (cached_table) is reused by calls with any seed; the seed-dependent sampler keys live in
// a per-call device array (PairSrc::rkey, filled by launch_region_keys).
struct RegionDev {
  corr_box A, B;
  int64_t nA, nB;
  int64_t off;   // exhaustive mode: prefix sum of nA*nB
};

enum PairMode { kList = 0, kSampled = 1, kExhaustive = 2 };

struct PairSrc {
  int mode;
  const int64_t* idxA;
  const int64_t* idxB;
  const RegionDev* reg;
  const uint64_t* rkey;  // kSampled: sampler key h_12 per region pair (reading R15)
  int64_t nreg;
  int64_t samples;
  int64_t nunits;
  int nx, ny;
  int64_t P;
  int same_field;
  int* err;
};

struct PairOut {
  float* out;                // kList: [npairs]
  unsigned long long* keys;  // kSampled / kExhaustive: [nreg] packed (value, index)
  int absval;
  float* dbg_eps;            // optional debug dumps [npairs][n]
  int32_t* dbg_nx;
  int32_t* dbg_ny;
};

// ---- launchers (defined in the .cu files) ----
cudaError_t launch_field_ingest(corr_field* f, const float* dvalues_member_major, cudaStream_t st);
cudaError_t launch_transpose_slice(corr_field* f, const float* dslice, int m0, int m1, cudaStream_t st);
constexpr int kStageMembers = 32;  // members per host-upload slice (one transpose tile row)
cudaError_t launch_field_aggregate(const corr_field* src, corr_field* dst, int fx, int fy, int fz, cudaStream_t st);
// Which k-NN formulation launch_ksg runs (all give bit-identical eps / counts / MI):
//   kKsgAuto  -- column-cell kernel for 128 <= n, k <= 8 (ksg_cell.cu), else the sweep / warp /
//                batched kernels of ksg.cu;
//   kKsgDense -- every n(n-1) comparison (CORR_F_KSG_DENSE);
//   kKsgSweep -- the round-1 x-sorted exact sweep (A/B reference; env CORR_KSG_PATH=sweep).
enum KsgPath { kKsgAuto = 0, kKsgDense = 1, kKsgSweep = 2 };
// count: tally executed comparisons (corr_ksg_comparisons) -- the column-cell kernel does so only
// when asked (CORR_F_KSG_COUNT), the ksg.cu kernels always.
cudaError_t launch_ksg(const corr_field* fa, const corr_field* fb, int k, bool plus1, KsgPath path, bool count,
                       const PairSrc& src, const PairOut& out, cudaStream_t st);
cudaError_t launch_ksg_cell(const corr_field* fa, const corr_field* fb, int k, bool plus1, bool count,
                            const PairSrc& src, const PairOut& out, cudaStream_t st);
cudaError_t ksg_comparisons(unsigned long long* value, bool reset);
cudaError_t ksg_nan_pairs(unsigned long long* value, bool reset);
// Device copy of a small host table (region lists) that stays resident and is reused when the
// same bytes come again: no host->device copy on the call path of repeated calls.  (A small copy
// queued behind a large pinned upload on the same copy engine would otherwise stall the stream
// for the whole upload.)  Returns nullptr on failure.
const void* cached_table(int device, const void* host, size_t bytes, cudaStream_t st);
cudaError_t gemm_flops(unsigned long long* value /* [2]: bf16, tf32 */, bool reset);
cudaError_t launch_pearson_pairs(const corr_field* fa, const corr_field* fb, const PairSrc& src,
                                 const PairOut& out, cudaStream_t st);
// rkey[r] = the sampler key of region pair r for `seed` (R15), computed on the device.
cudaError_t launch_region_keys(const RegionDev* dreg, int64_t nreg, uint64_t seed, uint64_t* rkey, cudaStream_t st);
cudaError_t launch_region_finalize(const PairSrc& src, const unsigned long long* keys,
                                   float* out_max, int64_t* out_argmax, cudaStream_t st);
// tcgen05 split-TF32 block GEMM with fused max/argmax epilogue (pearson_gemm.cu).
// Returns cudaErrorNotSupported if a region shape is not tileable (caller falls back).
cudaError_t launch_pearson_block(const corr_field* fa, const corr_field* fb, const RegionDev* hreg,
                                 const RegionDev* dreg, int64_t nreg, int absval,
                                 unsigned long long* keys, cudaStream_t st);

}  // namespace corr
