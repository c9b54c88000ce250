/*
 * corr_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the hot path of
 * arXiv 2309.03308 ("Adaptive Sampling of 3D Spatial Correlations for
 * Focus+Context Visualization").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2309_03308_b200/, libcorr.so) never links, imports or executes it.  It
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * Every function follows the plain definition in the paper (PAPER.md line
 * numbers below) written out step by step: brute force, no blocking, no fusion,
 * no reordering.  Readings of ambiguous passages are the DESIGN.md ledger
 * entries R1..R16.
 *
 * Compile WITHOUT -ffast-math and with -ffp-contract=off: the KSG distances are
 * IEEE fp32 round-to-nearest subtractions (reading R7), nothing is fused.
 *
 * Parity pins (tests/test_oracle_*.py, "-m 'not gpu'"): SPEC worked examples,
 * closed forms (self-pair MI, Gaussian MI, affine PPMCC), scipy/numpy library
 * routines (digamma, corrcoef, cKDTree), an independent sorted/binary-search
 * count algorithm, bit-exact invariances, and the splitmix64 published test
 * vector.  No function here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <omp.h>

#define ORACLE_NAN ((double)NAN)

/* ------------------------------------------------------------------------- */
/* PPMCC -- PAPER.md:169 (§3.2, "PPMCC requires merely to compute means and    */
/* variances"), PAPER.md:45 (§1); SPEC.md:155-159 (clamp to [-1,1], zero       */
/* variance is undefined -> NaN per reading R10).                               */
/* r = sum (x-xm)(y-ym) / sqrt( sum (x-xm)^2 * sum (y-ym)^2 ), in fp64.         */
/* ------------------------------------------------------------------------- */
double oracle_ppmcc(const float* x, const float* y, int n) {
  double xm = 0.0, ym = 0.0;
  for (int i = 0; i < n; ++i) { xm += (double)x[i]; ym += (double)y[i]; }
  xm /= (double)n;
  ym /= (double)n;
  double sxy = 0.0, sxx = 0.0, syy = 0.0;
  for (int i = 0; i < n; ++i) {
    double dx = (double)x[i] - xm, dy = (double)y[i] - ym;
    sxy += dx * dy;
    sxx += dx * dx;
    syy += dy * dy;
  }
  if (sxx == 0.0 || syy == 0.0) return ORACLE_NAN;
  double r = sxy / sqrt(sxx * syy);
  if (r > 1.0) r = 1.0;
  if (r < -1.0) r = -1.0;
  return r;
}

/* ------------------------------------------------------------------------- */
/* Digamma at a positive integer -- PAPER.md:174-178 (Eq. 2).  The KSG          */
/* arguments n, k, n_x,i, n_y,i are integers, so psi(m) = -gamma + sum_{t<m}1/t */
/* exactly (reading R17: the paper's Lanczos approximation is irrelevant).      */
/* psi(m <= 0) is a pole: NaN.                                                   */
/* ------------------------------------------------------------------------- */
static const double EULER_GAMMA = 0.57721566490153286060651209008240243;

double oracle_digamma_int(int m) {
  if (m <= 0) return ORACLE_NAN;
  double h = 0.0;
  for (int t = 1; t < m; ++t) h += 1.0 / (double)t;
  return h - EULER_GAMMA;
}

/* ------------------------------------------------------------------------- */
/* k-th nearest neighbour in the joint space, Chebyshev (max) norm --          */
/* PAPER.md:172-173 (§3.2): "its distance eps_i to the k-th nearest neighbor   */
/* ... d(z_i,z_j) = max{|x_i-x_j|, |y_i-y_j|}".                                 */
/*   d_ij  = fmaxf(fabsf(x_i - x_j), fabsf(y_i - y_j))  in fp32   (R7)          */
/*   eps_i = k-th smallest of the multiset {d_ij : j != i}          (R3, R4)    */
/* Marginal counts -- PAPER.md:174: "the numbers n_x,i and n_y,i of joint       */
/* samples fulfilling respectively |x_i-x_j| < eps_i and |y_i-y_j| < eps_i"     */
/*   n_x,i = #{ j != i : fabsf(x_i - x_j) < eps_i }   (strict, fp32; R1, R6)     */
/* ------------------------------------------------------------------------- */
static int cmp_float(const void* a, const void* b) {
  float fa = *(const float*)a, fb = *(const float*)b;
  return (fa > fb) - (fa < fb);
}

void oracle_knn(const float* x, const float* y, int n, int k, float* eps, int32_t* nx,
                int32_t* ny) {
  float* d = (float*)malloc(sizeof(float) * (size_t)(n > 1 ? n - 1 : 1));
  for (int i = 0; i < n; ++i) {
    int m = 0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      float dx = fabsf(x[i] - x[j]);
      float dy = fabsf(y[i] - y[j]);
      d[m++] = fmaxf(dx, dy);
    }
    qsort(d, (size_t)m, sizeof(float), cmp_float);
    float e = d[k - 1]; /* k-th smallest, with multiplicity */
    int cx = 0, cy = 0;
    for (int j = 0; j < n; ++j) {
      if (j == i) continue;
      if (fabsf(x[i] - x[j]) < e) ++cx;
      if (fabsf(y[i] - y[j]) < e) ++cy;
    }
    eps[i] = e;
    nx[i] = cx;
    ny[i] = cy;
  }
  free(d);
}

/* A series is "constant" when every member value is equal (min == max).       */
static int is_constant(const float* v, int n) {
  for (int i = 1; i < n; ++i)
    if (v[i] != v[0]) return 0;
  return 1;
}

/* ------------------------------------------------------------------------- */
/* Kraskov (KSG) MI estimate -- PAPER.md:174 (§3.2):                             */
/*   MI = psi(n) + psi(k) - (1/n) * sum_i [ psi(n_x,i) + psi(n_y,i) ]           */
/* (bracket placement: reading R2).  plus1 != 0 selects psi(n_x,i + 1)          */
/* (Kraskov's algorithm 1; reading R1).  Degenerate -> NaN (R10): a constant    */
/* x or y series, or any psi(0) in the verbatim form.  The sum is formed         */
/* order-free from the histogram of counts, sum_m h[m] * psi(m), in fp64.        */
/* ------------------------------------------------------------------------- */
double oracle_ksg(const float* x, const float* y, int n, int k, int plus1) {
  if (is_constant(x, n) || is_constant(y, n)) return ORACLE_NAN;
  float* eps = (float*)malloc(sizeof(float) * (size_t)n);
  int32_t* cx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* cy = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t* hist = (int64_t*)calloc((size_t)n + 2, sizeof(int64_t));
  oracle_knn(x, y, n, k, eps, cx, cy);
  int off = plus1 ? 1 : 0;
  for (int i = 0; i < n; ++i) {
    hist[cx[i] + off] += 1;
    hist[cy[i] + off] += 1;
  }
  double result;
  if (hist[0] > 0) {
    result = ORACLE_NAN; /* psi(0): pole */
  } else {
    double s = 0.0;
    for (int m = 1; m <= n; ++m)
      if (hist[m]) s += (double)hist[m] * oracle_digamma_int(m);
    result = oracle_digamma_int(n) + oracle_digamma_int(k) - s / (double)n;
  }
  free(eps);
  free(cx);
  free(cy);
  free(hist);
  return result;
}

/* ------------------------------------------------------------------------- */
/* Pair evaluation over a field stored as the paper's/SPEC's file order        */
/* values[member][p], p = (z*ny + y)*nx + x.  */
/* measure: 0 = PPMCC, 1 = KSG; flags bit 8 = KSG "+1" variant (R1).           */
/* fb == NULL -> single variable (fb = fa).  Results are fp64.                 */
/* ------------------------------------------------------------------------- */
static void gather(const float* field, int64_t P, int n, int64_t p, float* out) {
  for (int e = 0; e < n; ++e) out[e] = field[(int64_t)e * P + p];
}

double oracle_pair(const float* fa, const float* fb, int64_t P, int n, int measure, int k,
                   int64_t a, int64_t b) {
  float* x = (float*)malloc(sizeof(float) * (size_t)n);
  float* y = (float*)malloc(sizeof(float) * (size_t)n);
  gather(fa, P, n, a, x);
  gather(fb ? fb : fa, P, n, b, y);
  int kind = measure & 0xFF;
  double r;
  if (kind == 0)
    r = oracle_ppmcc(x, y, n);
  else
    r = oracle_ksg(x, y, n, k, (measure & (1 << 8)) != 0);
  free(x);
  free(y);
  return r;
}

void oracle_eval_pairs(const float* fa, const float* fb, int64_t P, int n, int measure, int k,
                       const int64_t* idxA, const int64_t* idxB, int64_t npairs, double* out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < npairs; ++q)
    out[q] = oracle_pair(fa, fb, P, n, measure, k, idxA[q], idxB[q]);
}

/* Per-member eps / counts for the bit-exact parity checks. out arrays [npairs][n]. */
void oracle_knn_pairs(const float* fa, const float* fb, int64_t P, int n, int k,
                      const int64_t* idxA, const int64_t* idxB, int64_t npairs, float* eps,
                      int32_t* nx, int32_t* ny) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < npairs; ++q) {
    float* x = (float*)malloc(sizeof(float) * (size_t)n);
    float* y = (float*)malloc(sizeof(float) * (size_t)n);
    gather(fa, P, n, idxA[q], x);
    gather(fb ? fb : fa, P, n, idxB[q], y);
    oracle_knn(x, y, n, k, eps + q * n, nx + q * n, ny + q * n);
    free(x);
    free(y);
  }
}

/* ------------------------------------------------------------------------- */
/* Uniform random sampling of point pairs -- PAPER.md:139-140 (§3.1): "random   */
/* sampling of correlations at grid points in each pair of bricks.  One sample  */
/* position corresponds to a position in a 6 dimensional space".  The paper     */
/* names no generator; reading R15 fixes a counter-based one keyed by the two   */
/* boxes so that any shard of the region-pair list draws the same samples:      */
/*   mix64(z)   = splitmix64 finaliser (Steele/Lea/Vigna)                       */
/*   h_0 = seed;  h_{t+1} = mix64(h_t XOR (uint32(c_t) + G*(t+1)))  t = 0..11   */
/*   c = (A.x0,A.y0,A.z0,A.x1,A.y1,A.z1, B.x0,...,B.z1),  G = 0x9E3779B97F4A7C15 */
/*   u_s = mix64(h_12 + G*(s+1))                                                 */
/*   a_local = (lo32(u_s) * |A|) >> 32,  b_local = (hi32(u_s) * |B|) >> 32      */
/* local index -> (lx, ly, lz) with x fastest inside the box, then global       */
/* p = ((z0+lz)*ny + (y0+ly))*nx + (x0+lx).                                     */
/* ------------------------------------------------------------------------- */
typedef struct {
  int32_t x0, y0, z0, x1, y1, z1;
} oracle_box;

#define GOLDEN64 0x9E3779B97F4A7C15ULL

uint64_t oracle_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t oracle_pair_key(uint64_t seed, const oracle_box* A, const oracle_box* B) {
  int32_t c[12] = {A->x0, A->y0, A->z0, A->x1, A->y1, A->z1,
                   B->x0, B->y0, B->z0, B->x1, B->y1, B->z1};
  uint64_t h = seed;
  for (int t = 0; t < 12; ++t)
    h = oracle_mix64(h ^ ((uint64_t)(uint32_t)c[t] + GOLDEN64 * (uint64_t)(t + 1)));
  return h;
}

static int64_t box_size(const oracle_box* b) {
  return (int64_t)(b->x1 - b->x0) * (int64_t)(b->y1 - b->y0) * (int64_t)(b->z1 - b->z0);
}

static int64_t box_point(const oracle_box* b, int64_t local, int nx, int ny) {
  int64_t ax = b->x1 - b->x0, ay = b->y1 - b->y0;
  int64_t lx = local % ax;
  int64_t ly = (local / ax) % ay;
  int64_t lz = local / (ax * ay);
  return ((int64_t)(b->z0 + lz) * ny + (b->y0 + ly)) * nx + (b->x0 + lx);
}

void oracle_sample(uint64_t seed, const oracle_box* A, const oracle_box* B, int64_t s, int nx,
                   int ny, int64_t* a, int64_t* b) {
  uint64_t key = oracle_pair_key(seed, A, B);
  uint64_t u = oracle_mix64(key + GOLDEN64 * (uint64_t)(s + 1));
  uint64_t na = (uint64_t)box_size(A), nb = (uint64_t)box_size(B);
  uint64_t al = ((u & 0xFFFFFFFFULL) * na) >> 32;
  uint64_t bl = ((u >> 32) * nb) >> 32;
  *a = box_point(A, (int64_t)al, nx, ny);
  *b = box_point(B, (int64_t)bl, nx, ny);
}

/* ------------------------------------------------------------------------- */
/* Region-pair maximum -- PAPER.md:133 (§3): "point-to-point correlations       */
/* between pairs of grid points in either brick are computed, and the maximum   */
/* of these correlations is used".  samples > 0: the sampled pairs s = 0..S-1;  */
/* samples == 0: all |A|*|B| pairs, q = a_local*|B| + b_local.  NaN values are  */
/* skipped; ties go to the lowest s (or q) (R16).  With one field, (a, a)       */
/* self-pairs are skipped ("self-correlations excluded").         */
/* flags bit 9 (ABS): maximise |r| (R11).  All-NaN -> NaN, argmax (-1,-1).       */
/* ------------------------------------------------------------------------- */
void oracle_region_max(const float* fa, const float* fb, int nx, int ny, int nz, int n,
                       int measure, int k, const oracle_box* regA, const oracle_box* regB,
                       int64_t nregion, int64_t samples, uint64_t seed, double* out_max,
                       int64_t* out_argmax) {
  int64_t P = (int64_t)nx * ny * nz;
  int use_abs = (measure & (1 << 9)) != 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t r = 0; r < nregion; ++r) {
    const oracle_box* A = &regA[r];
    const oracle_box* B = &regB[r];
    int64_t na = box_size(A), nb = box_size(B);
    int64_t total = samples > 0 ? samples : na * nb;
    double best = ORACLE_NAN;
    int64_t ba = -1, bb = -1;
    for (int64_t s = 0; s < total; ++s) {
      int64_t a, b;
      if (samples > 0) {
        oracle_sample(seed, A, B, s, nx, ny, &a, &b);
      } else {
        a = box_point(A, s / nb, nx, ny);
        b = box_point(B, s % nb, nx, ny);
      }
      if (fb == NULL && a == b) continue;
      double v = oracle_pair(fa, fb, P, n, measure, k, a, b);
      if (isnan(v)) continue;
      if (use_abs) v = fabs(v);
      /* values compared after rounding to the fp32 the library returns */
      v = (double)(float)v;
      if (isnan(best) || v > best) {
        best = v;
        ba = a;
        bb = b;
      }
    }
    out_max[r] = best;
    out_argmax[2 * r] = ba;
    out_argmax[2 * r + 1] = bb;
  }
}

/* Every value behind oracle_region_max, for the argmax-margin checks (the parity bar: the
 * region argmax must be bit-exact whenever the winning margin exceeds the tolerance, so the
 * tests need the runner-up).  Same enumeration, skips and fp32 rounding as oracle_region_max
 * (R11, R16); out[r * total + s] = value of sample s (or exhaustive index q) of
 * region pair r, NaN where oracle_region_max skips it (self pair, NaN value).  Pair indices
 * go to out_a / out_b (same layout) when not NULL.  Enumeration only -- no new arithmetic. */
void oracle_region_values(const float* fa, const float* fb, int nx, int ny, int nz, int n,
                          int measure, int k, const oracle_box* regA, const oracle_box* regB,
                          int64_t nregion, int64_t samples, uint64_t seed, double* out,
                          int64_t* out_a, int64_t* out_b) {
  int64_t P = (int64_t)nx * ny * nz;
  int use_abs = (measure & (1 << 9)) != 0;
  int64_t total = samples > 0 ? samples : box_size(&regA[0]) * box_size(&regB[0]);
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t r = 0; r < nregion; ++r) {
    for (int64_t s = 0; s < total; ++s) {
      const oracle_box* A = &regA[r];
      const oracle_box* B = &regB[r];
      int64_t nb = box_size(B);
      int64_t a, b;
      if (samples > 0) {
        oracle_sample(seed, A, B, s, nx, ny, &a, &b);
      } else {
        a = box_point(A, s / nb, nx, ny);
        b = box_point(B, s % nb, nx, ny);
      }
      double v = ORACLE_NAN;
      if (!(fb == NULL && a == b)) {
        v = oracle_pair(fa, fb, P, n, measure, k, a, b);
        if (!isnan(v)) {
          if (use_abs) v = fabs(v);
          v = (double)(float)v;
        }
      }
      out[r * total + s] = v;
      if (out_a) out_a[r * total + s] = a;
      if (out_b) out_b[r * total + s] = b;
    }
  }
}

/* The sampled point pairs s = s0 .. s0+count-1 of each region pair (oracle_sample in a loop),
 * out_a / out_b [nregion][count].  Enumeration only. */
void oracle_sample_many(uint64_t seed, const oracle_box* regA, const oracle_box* regB,
                        int64_t nregion, int64_t s0, int64_t count, int nx, int ny,
                        int64_t* out_a, int64_t* out_b) {
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nregion; ++r)
    for (int64_t s = 0; s < count; ++s)
      oracle_sample(seed, &regA[r], &regB[r], s0 + s, nx, ny, &out_a[r * count + s],
                    &out_b[r * count + s]);
}

/* Host threads used by the OpenMP loops above (not arithmetic: every pair is computed by one
 * thread, so results do not depend on it).  n <= 0 leaves the setting alone.  Returns the
 * thread count the next parallel region will use.  bench.py sets it explicitly because
 * torchrun exports OMP_NUM_THREADS=1. */
int oracle_set_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}
