/* ASan/UBSan driver for the CPU oracle (test infrastructure; SURVEY.md §4 item 4, §5 "sanitizers").
 * Compiled together with oracle/corr_oracle.c under -fsanitize=address,undefined by
 * tests/test_sanitizers.py; exercises every exported oracle function on small synthetic inputs
 * with ties, constant series, k = n-1, sampled and exhaustive region maxima.  Exit 0 = clean. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t x0, y0, z0, x1, y1, z1;
} box_t;

double oracle_ppmcc(const float* x, const float* y, int n);
double oracle_digamma_int(int m);
void oracle_knn(const float* x, const float* y, int n, int k, float* eps, int32_t* nx, int32_t* ny);
double oracle_ksg(const float* x, const float* y, int n, int k, int plus1);
void oracle_eval_pairs(const float* fa, const float* fb, int64_t P, int n, int measure, int k, const int64_t* idxA,
                       const int64_t* idxB, int64_t npairs, double* out);
void oracle_knn_pairs(const float* fa, const float* fb, int64_t P, int n, int k, const int64_t* idxA,
                      const int64_t* idxB, int64_t npairs, float* eps, int32_t* nx, int32_t* ny);
uint64_t oracle_mix64(uint64_t z);
void oracle_sample(uint64_t seed, const box_t* A, const box_t* B, int64_t s, int nx, int ny, int64_t* a, int64_t* b);
void oracle_region_max(const float* fa, const float* fb, int nx, int ny, int nz, int n, int measure, int k,
                       const box_t* regA, const box_t* regB, int64_t nregion, int64_t samples, uint64_t seed,
                       double* out_max, int64_t* out_argmax);
void oracle_region_values(const float* fa, const float* fb, int nx, int ny, int nz, int n, int measure, int k,
                          const box_t* regA, const box_t* regB, int64_t nregion, int64_t samples, uint64_t seed,
                          double* out, int64_t* out_a, int64_t* out_b);
void oracle_sample_many(uint64_t seed, const box_t* regA, const box_t* regB, int64_t nregion, int64_t s0,
                        int64_t count, int nx, int ny, int64_t* out_a, int64_t* out_b);
int oracle_set_threads(int n);

int main(void) {
  const int nx = 6, ny = 5, nz = 2, n = 37, P = nx * ny * nz;
  float* f = (float*)malloc(sizeof(float) * (size_t)n * P);
  float* g = (float*)malloc(sizeof(float) * (size_t)n * P);
  uint64_t st = 12345;
  for (int i = 0; i < n * P; ++i) {
    st = oracle_mix64(st + 0x9E3779B97F4A7C15ULL);
    f[i] = (float)((st >> 40) % 7) * 0.5f;          /* heavy ties */
    g[i] = (float)((double)(st & 0xFFFFFF) / 16777216.0);
  }
  for (int e = 0; e < n; ++e) f[e * P + 3] = 2.0f;   /* a constant series */
  oracle_set_threads(2);
  double acc = 0.0;
  for (int m = 1; m <= n + 1; ++m) acc += oracle_digamma_int(m);
  float x[64], y[64], eps[64];
  int32_t cx[64], cy[64];
  for (int i = 0; i < 64; ++i) {
    x[i] = g[i];
    y[i] = f[i * 3 % (n * P)];
  }
  for (int k = 1; k < 40; k += 7) {
    oracle_knn(x, y, 40, k, eps, cx, cy);
    acc += oracle_ksg(x, y, 40, k, 0) + oracle_ksg(x, y, 40, k, 1);
  }
  oracle_knn(x, y, 40, 39, eps, cx, cy);           /* k = n - 1 */
  acc += oracle_ppmcc(x, y, 40);
  int64_t ia[50], ib[50];
  for (int i = 0; i < 50; ++i) {
    ia[i] = (i * 7) % P;
    ib[i] = (i * 13 + 1) % P;
  }
  double out[50];
  for (int meas = 0; meas < 2; ++meas) {
    oracle_eval_pairs(f, NULL, P, n, meas, 3, ia, ib, 50, out);
    oracle_eval_pairs(f, g, P, n, meas | (1 << 8), 5, ia, ib, 50, out);
  }
  float* de = (float*)malloc(sizeof(float) * 50 * n);
  int32_t* dx = (int32_t*)malloc(sizeof(int32_t) * 50 * n);
  int32_t* dy = (int32_t*)malloc(sizeof(int32_t) * 50 * n);
  oracle_knn_pairs(f, g, P, n, 4, ia, ib, 50, de, dx, dy);
  box_t A[3] = {{0, 0, 0, 3, 5, 1}, {3, 0, 0, 6, 5, 2}, {0, 0, 1, 6, 2, 2}};
  box_t B[3] = {{3, 0, 0, 6, 5, 1}, {0, 0, 0, 3, 3, 2}, {0, 0, 0, 6, 5, 2}};
  double mx[3];
  int64_t arg[6];
  oracle_region_max(f, NULL, nx, ny, nz, n, 1, 3, A, B, 3, 25, 7, mx, arg);
  oracle_region_max(f, g, nx, ny, nz, n, 0 | (1 << 9), 0, A, B, 3, 0, 7, mx, arg);
  oracle_region_max(f, NULL, nx, ny, nz, n, 0, 0, A + 2, B + 2, 1, 0, 7, mx, arg); /* overlapping boxes */
  double* vals = (double*)malloc(sizeof(double) * 3 * 25);
  int64_t* va = (int64_t*)malloc(sizeof(int64_t) * 3 * 25);
  int64_t* vb = (int64_t*)malloc(sizeof(int64_t) * 3 * 25);
  oracle_region_values(f, NULL, nx, ny, nz, n, 1, 3, A, B, 3, 25, 7, vals, va, vb);
  oracle_sample_many(9, A, B, 3, 5, 25, nx, ny, va, vb);
  int64_t a1, b1;
  oracle_sample(9, A, B, 0, nx, ny, &a1, &b1);
  printf("ok %g\n", acc + mx[0]);
  free(f); free(g); free(de); free(dx); free(dy); free(vals); free(va); free(vb);
  return 0;
}
