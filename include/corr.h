/*
 * corr.h -- C ABI of libcorr.so, the B200 (sm_100a) hot path of arXiv 2309.03308
 * ("Adaptive Sampling of 3D Spatial Correlations for Focus+Context Visualization").
 *
 * The three calls follow the paper's problem statement:
 *   - an ensemble of E members on an X x Y x Z grid           (§3)
 *   - point-to-point correlation of two grid points' member series, Pearson
 *     (§3.2) or the Kraskov k-NN MI estimator (Eq. 2)
 *   - the region-pair indicator = maximum of the point-pair correlations of two
 *     bricks (§3), sampled uniformly at random (§3.1)
 *     or exhaustively (§5.4, "all point-to-point pairs").
 * Readings of ambiguous passages are DESIGN.md's ledger R1..R17.
 *
 * Conventions (all calls):
 *   - plain C types only; no exceptions cross the ABI; every call returns a status
 *     (CORR_OK or a negative CORR_E_*) and sets a thread-local message readable
 *     with corr_last_error().
 *   - `cuda_stream` is a cudaStream_t (NULL = legacy default stream).  Compute calls
 *     are asynchronous on that stream; device buffers passed in must stay valid
 *     until the stream reaches the call.
 *   - point index p = (z*ny + y)*nx + x (x fastest), int64.
 *   - the library never falls back to the CPU: with no usable CUDA device every call
 *     returns CORR_E_CUDA.
 */
#ifndef CORR_H_
#define CORR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque ensemble field, immutable after creation (so concurrent calls on different
 * streams are safe).  Owns all derived device buffers (member-contiguous rows,
 * standardised rows, tf32 split planes, sorted rows, constant-series flags). */
typedef struct corr_field corr_field;

/* Half-open grid-index box [x0,x1) x [y0,y1) x [z0,z1): a brick. */
typedef struct {
  int32_t x0, y0, z0, x1, y1, z1;
} corr_box;

/* `measure` = kind in the low byte, OR-ed with flags. */
enum { CORR_PEARSON = 0, CORR_KSG = 1 };
enum {
  CORR_F_KSG_PLUS1 = 1 << 8, /* KSG with psi(n_x+1), psi(n_y+1) (Kraskov alg. 1; reading R1) */
  CORR_F_ABS = 1 << 9,       /* region max of |value| (reading R11)           */
  CORR_F_KSG_DENSE = 1 << 10, /* KSG: evaluate all n(n-1) comparisons (no pruning); same results  */
  CORR_F_KSG_COUNT = 1 << 11, /* KSG: tally executed comparisons for corr_ksg_comparisons (slower; */
                              /* same results) -- a diagnostic for the roofline report          */
  CORR_F_KSG_SWEEP = 1 << 12  /* KSG: the round-1 x-sorted block sweep instead of the column-cell */
                              /* k-NN (same results) -- the bench's reference formulation        */
};
enum { CORR_OK = 0, CORR_E_INVAL = -1, CORR_E_RANGE = -2, CORR_E_NOMEM = -3, CORR_E_CUDA = -4 };

/* corr_field_create -- ingest one variable of an ensemble.
 *   values   : float32 [members][nz][ny][nx] (the paper's/SPEC's file order),
 *              host or device pointer (detected); copied, caller keeps ownership.  A host
 *              pointer is streamed in 32-member slices as in corr_field_update.
 *   nx,ny,nz : grid dims >= 1;  2 <= members (n) <= 4096 (a pair is staged in shared memory).
 *   device   : CUDA ordinal the field lives on; the call makes it current.
 * Builds, on `device`: member-contiguous rows F[P][n_pad] (n_pad = ceil(n/8)*8),
 * fp64-standardised rows Z, their tf32 split (Z_hi, Z_lo), per-row sorted copies and
 * argsort, constant-series flags.  Synchronises `cuda_stream` (it validates input).
 * Errors: CORR_E_INVAL (bad dims, non-finite value), CORR_E_NOMEM, CORR_E_CUDA.
 * On success *out owns the field; release with corr_field_destroy. */
int corr_field_create(const float* values, int32_t nx, int32_t ny, int32_t nz, int32_t members,
                      int32_t device, void* cuda_stream, corr_field** out);

/* corr_field_aggregate -- one level of the paper's mean-tree (§3.3: "for each
 * brick and each ensemble member ... the means ... of all variables at the grid points represented
 * by this brick"): a new field on the grid ceil(nx/fx) x ceil(ny/fy) x ceil(nz/fz) whose series at
 * coarse point (X,Y,Z) is, per member, the mean of the fine series over the block
 * [fx*X, fx*X+fx) x [fy*Y, ...) x [fz*Z, ...) (boundary blocks average the points that exist;
 * fp64 sums, fp32 result).  Same members and device as `f`; all derived buffers are rebuilt, so
 * every call above works on the aggregate ("BOS ... using the mean values at the highest
 * resolution tree-level that just fits into GPU memory").  Synchronises the stream.
 * Errors: CORR_E_INVAL (factor < 1), CORR_E_NOMEM, CORR_E_CUDA.  Release with corr_field_destroy. */
int corr_field_aggregate(const corr_field* f, int32_t fx, int32_t fy, int32_t fz, void* cuda_stream,
                         corr_field** out);

/* corr_field_update -- replace the member values of an existing field (same dims and members;
 * e.g. the next forecast time of the ensemble) and rebuild every derived buffer in place, with no
 * device allocation.  values: float32 [members][nz][ny][nx], host or device.
 * Asynchronous on `cuda_stream` (no host synchronisation).  A HOST pointer is streamed by the
 * library: slices of 32 member rows (contiguous in the input) are copied with one
 * cudaMemcpyAsync each on the field's own copy stream into two persistent device slices (allocated
 * on the first host update, 2 x 32 x P x 4 bytes) and each slice is transposed on `cuda_stream` as
 * soon as it has landed; page-locked (pinned) memory makes the copies overlap device work.  The
 * host buffer must stay unchanged until `cuda_stream` has passed this call's work.  To overlap an
 * update with compute on another stream, pass a HIGH-priority stream here: the pair kernels launch
 * one pair per CTA, and a normal-priority stream's transposes would wait behind all of them.  Calls on
 * other streams that still read the field must be ordered before it by the caller (events).
 * A non-finite value is detected on the device: the next corr_check() returns CORR_E_INVAL (the
 * field content is undefined until the next clean update).
 * Errors (immediate): CORR_E_INVAL (NULL arguments), CORR_E_NOMEM (staging), CORR_E_CUDA. */
int corr_field_update(corr_field* f, const float* values, void* cuda_stream);

/* Frees the field's device memory (device-synchronising).  NULL is a no-op. */
int corr_field_destroy(corr_field* f);

/* Field geometry: any output pointer may be NULL. */
int corr_field_info(const corr_field* f, int32_t* nx, int32_t* ny, int32_t* nz,
                    int32_t* members, int32_t* device);

/* corr_eval_pairs -- batched point-pair correlation ("compute
 * correlations for multiple feature vectors simultaneously").
 *   fa, fb   : fields; fb == NULL means fb = fa (one variable).  fb must match fa's
 *              dims, members and device.
 *   measure  : CORR_PEARSON or CORR_KSG, | flags.
 *   k        : KSG neighbour order, 1 <= k <= n-1 (every k is supported: register lists for
 *              k <= 32, multi-pass batched lists above); k == 0 selects the paper's
 *              ceil(3n/100) clamped to [1, n-1].  Ignored for Pearson.
 *              KSG needs n >= 4.
 *   idxA,idxB: DEVICE int64 [npairs] point indices into fa / fb.
 *   out      : DEVICE float32 [npairs]; out[i] = corr(fa[idxA[i]], fb[idxB[i]]).
 * Degenerate pairs are not errors: a constant series, or psi(0) in the
 * verbatim KSG form, gives NaN (reading R10).  Pearson is clamped to [-1, 1].
 * Out-of-range indices are detected on the device: the pair gets NaN and the next
 * corr_check() on the stream returns CORR_E_RANGE.
 * Errors (immediate): CORR_E_INVAL, CORR_E_CUDA. */
int corr_eval_pairs(const corr_field* fa, const corr_field* fb, int32_t measure, int32_t k,
                    const int64_t* idxA, const int64_t* idxB, int64_t npairs, float* out,
                    void* cuda_stream);

/* corr_region_max -- per region pair, the maximum point-pair correlation between
 * the two bricks and its argmax.
 *   regionA, regionB : HOST arrays [nregion_pairs] of boxes (A in fa, B in fb).
 *   samples > 0      : evaluate `samples` uniformly random point pairs per region pair
 *                       drawn by the counter-based sampler of reading
 *                      R15, keyed by (seed, box A, box B) -- independent of the region
 *                      pair's position in the list, so any sharding gives identical
 *                      results.  Ties -> lowest sample index s.
 *   samples == 0     : every one of the |A|*|B| pairs (exhaustive).  Ties ->
 *                      lowest q = a_local*|B| + b_local (local index x fastest in a box).
 *                      Pearson uses the tcgen05 split-TF32 block GEMM with a fused max; boxes
 *                      the GEMM's TMA tiling cannot map (deeper than 256 grid layers in z) run
 *                      on the CUDA-core pair path instead (same results, slower; such calls
 *                      add nothing to corr_gemm_flops).
 *   out_max          : DEVICE float32 [R]; NaN if every evaluated value was NaN.
 *   out_argmax       : DEVICE int64 [R][2] = (point in A, point in B), (-1,-1) if none.
 * NaN values are skipped.  With one field (fb == NULL) the self pair (a, a) is skipped
 * (PAPER.md:299).  CORR_F_ABS maximises |value|.  Requires samples < 2^32 and
 * |A|*|B| < 2^32 for the exhaustive mode.
 * Errors: CORR_E_INVAL (empty box, bad measure/k), CORR_E_RANGE (box outside the grid),
 * CORR_E_NOMEM, CORR_E_CUDA. */
int corr_region_max(const corr_field* fa, const corr_field* fb, int32_t measure, int32_t k,
                    const corr_box* regionA, const corr_box* regionB, int64_t nregion_pairs,
                    int64_t samples, uint64_t seed, float* out_max, int64_t* out_argmax,
                    void* cuda_stream);

/* corr_ksg_debug -- diagnostic dump of the KSG intermediates for the bit-exact parity
 * checks: for pair i and member e (original member order),
 *   eps[i*n + e] = Chebyshev distance to the k-th nearest neighbour (fp32),
 *   nx[i*n + e], ny[i*n + e] = strict marginal counts (int32).
 * idxA/idxB/eps/nx/ny are DEVICE pointers.  Same errors as corr_eval_pairs. */
int corr_ksg_debug(const corr_field* fa, const corr_field* fb, int32_t k, const int64_t* idxA,
                   const int64_t* idxB, int64_t npairs, float* eps, int32_t* nx, int32_t* ny,
                   void* cuda_stream);

/* corr_check -- synchronises `cuda_stream`; returns CORR_E_INVAL if an earlier
 * corr_field_update of `f` saw a non-finite input value, CORR_E_RANGE if an earlier call on
 * `f`'s device saw an out-of-range point index (either flag is cleared when reported),
 * CORR_E_CUDA on a CUDA error, else CORR_OK. */
int corr_check(const corr_field* f, void* cuda_stream);

/* corr_ksg_comparisons -- KSG member-comparisons (d_ij evaluations) executed on
 * `device` since the last reset; the pruned k-NN passes skip comparisons that provably cannot
 * change any eps_i, so this is <= n(n-1) per pair.  The default column-cell kernel (n >= 128,
 * k <= 8) counts only in calls with CORR_F_KSG_COUNT.  Synchronises the device; reset != 0 zeroes
 * the counter after reading.  Diagnostic for the roofline report (bench.py). */
int corr_ksg_comparisons(int32_t device, int64_t* count, int32_t reset);

/* corr_ksg_nan_pairs -- KSG point pairs that corr_region_max skipped on `device` since the last
 * reset because their value was NaN: a constant series (reading R10), or psi(0) in the verbatim
 * form when a member's joint sample is duplicated (eps = 0, reading R5; e.g. zero-inflated
 * fields).  Such pairs never win a region maximum; this count makes their number visible.
 * Synchronises the device; reset != 0 zeroes the counter after reading. */
int corr_ksg_nan_pairs(int32_t device, int64_t* count, int32_t reset);

/* corr_gemm_flops -- tensor-core work executed on `device` by the exhaustive Pearson block path
 * (corr_region_max with samples == 0) since the last reset, as logical MMA flops 2*128*256*K per
 * 128x256 tile and MMA set: *bf16_flops for the screening pass (one bf16 product per tile),
 * *tf32_flops for the exact pass (three tf32 products on the tiles that can hold a region pair's
 * maximum).  Synchronises the device; reset != 0 zeroes both.  Diagnostic for bench.py's roofline. */
int corr_gemm_flops(int32_t device, int64_t* bf16_flops, int64_t* tf32_flops, int32_t reset);

/* Number of CUDA kernels this library has launched in this process (diagnostic; bench.py
 * reports the launches inside its timed region as `gpu_launches`). */
int64_t corr_launch_count(void);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char* corr_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CORR_H_ */
