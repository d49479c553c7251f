/*
 * A plain C caller of the drop-in boundary: no Python, no torch — the CUDA runtime for device memory
 * and libsketch_b200.so through include/sketch_b200.h, each result checked against a direct C
 * computation of the reference's arithmetic (float64 on the host).
 *
 *   1. SRTT with the Walsh-Hadamard transform (reference SparseRttTM.apply_right, rtt.py:129-140):
 *      float32 A, +-1 diagonal, xi = 2 signed samples per output column.
 *   2. A dense float64 apply, Y = A * Omega (the Gaussian / materialised families, base.py:75-79),
 *      through sk_kr_right_cc with one block (W = NULL), and its adjoint X = Omega^T * B in place.
 *   3. The sparse-sign right apply of config 1 (reference _SparseTM.apply_right, sparse.py:63-66): Omega
 *      with zeta distinct +-1 columns per row, encoded once by sk_sparse_right_cols_encode (two calls:
 *      the positions needed, then the schedule), applied to float64 A by sk_sparse_right_cols.
 *   4. The error contract: a bad shape returns SK_EINVAL with a message from sk_last_error().
 *
 * Build (tests/test_c_abi.py does this):
 *   gcc -O2 -std=c11 tests/c/abi_demo.c -Iinclude -I<cuda>/include -L<lib dir> -lsketch_b200
 *       -L<cuda>/lib64 -lcudart -lm -Wl,-rpath,<lib dir> -o abi_demo
 * Exit status 0 when every check passes.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "sketch_b200.h"

static uint64_t rng_state = 0x9E3779B97F4A7C15ull;
static uint64_t next_u64(void) { /* xorshift64* */
  rng_state ^= rng_state >> 12;
  rng_state ^= rng_state << 25;
  rng_state ^= rng_state >> 27;
  return rng_state * 2685821657736338717ull;
}
static double uniform(void) { return (double)(next_u64() >> 11) * (1.0 / 9007199254740992.0); }
static double normal(void) { /* Box-Muller */
  double u = uniform(), v = uniform();
  if (u < 1e-300) u = 1e-300;
  return sqrt(-2.0 * log(u)) * cos(6.283185307179586 * v);
}

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess) {                                                                   \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));       \
      exit(2);                                                                                 \
    }                                                                                          \
  } while (0)
#define SK(x)                                                                                  \
  do {                                                                                         \
    int s_ = (x);                                                                              \
    if (s_ != SK_OK) {                                                                         \
      fprintf(stderr, "%s:%d %s -> %d: %s\n", __FILE__, __LINE__, #x, s_, sk_last_error());  \
      exit(3);                                                                                 \
    }                                                                                          \
  } while (0)

static double rel_err(const double* a, const double* b, size_t n) {
  double num = 0, den = 0;
  for (size_t i = 0; i < n; ++i) {
    num += (a[i] - b[i]) * (a[i] - b[i]);
    den += b[i] * b[i];
  }
  return sqrt(num / (den > 0 ? den : 1));
}

/* in-place unnormalised Walsh-Hadamard transform of x[0..d) (d a power of two) */
static void fwht(double* x, int d) {
  for (int h = 1; h < d; h *= 2)
    for (int i = 0; i < d; i += 2 * h)
      for (int j = i; j < i + h; ++j) {
        const double a = x[j], b = x[j + h];
        x[j] = a + b;
        x[j + h] = a - b;
      }
}

static int check_srtt(void) {
  const int n = 300, d = 1024, k = 40, xi = 2;
  float* a = malloc(sizeof(float) * n * d);
  float* dv = malloc(sizeof(float) * d);
  int32_t* samp = malloc(sizeof(int32_t) * k * xi);
  for (int i = 0; i < n * d; ++i) a[i] = (float)normal();
  for (int j = 0; j < d; ++j) dv[j] = (next_u64() & 1) ? -1.0f : 1.0f;
  for (int c = 0; c < k * xi; ++c) {
    const uint32_t row = (uint32_t)(next_u64() % d), neg = (uint32_t)(next_u64() & 1);
    samp[c] = (int32_t)(row | (neg << 31));
  }
  const double scale = 1.0 / sqrt((double)d) * sqrt((double)d / xi) / sqrt((double)k);

  float *da, *ddv, *dy;
  int32_t* dsamp;
  CK(cudaMalloc((void**)&da, sizeof(float) * n * d));
  CK(cudaMalloc((void**)&ddv, sizeof(float) * d));
  CK(cudaMalloc((void**)&dsamp, sizeof(int32_t) * k * xi));
  CK(cudaMalloc((void**)&dy, sizeof(float) * n * k));
  CK(cudaMemcpy(da, a, sizeof(float) * n * d, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(ddv, dv, sizeof(float) * d, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsamp, samp, sizeof(int32_t) * k * xi, cudaMemcpyHostToDevice));
  SK(sk_srtt_right(SK_F32, da, n, d, d, ddv, SK_WHT | SK_DIAG_PM1, dsamp, xi, k, scale, dy, k, NULL));
  CK(cudaDeviceSynchronize());
  float* y = malloc(sizeof(float) * n * k);
  CK(cudaMemcpy(y, dy, sizeof(float) * n * k, cudaMemcpyDeviceToHost));

  double* got = malloc(sizeof(double) * n * k);
  double* ref = malloc(sizeof(double) * n * k);
  double* row = malloc(sizeof(double) * d);
  for (int r = 0; r < n; ++r) {
    for (int j = 0; j < d; ++j) row[j] = (double)a[(size_t)r * d + j] * dv[j];
    fwht(row, d);
    for (int c = 0; c < k; ++c) {
      double s = 0;
      for (int x = 0; x < xi; ++x) {
        const uint32_t e = (uint32_t)samp[c * xi + x];
        s += (e >> 31) ? -row[e & 0x7fffffffu] : row[e & 0x7fffffffu];
      }
      ref[(size_t)r * k + c] = s * scale;
      got[(size_t)r * k + c] = y[(size_t)r * k + c];
    }
  }
  const double err = rel_err(got, ref, (size_t)n * k);
  printf("srtt wht f32: rel err %.3e\n", err);
  cudaFree(da);
  cudaFree(ddv);
  cudaFree(dsamp);
  cudaFree(dy);
  free(a);
  free(dv);
  free(samp);
  free(y);
  free(got);
  free(ref);
  free(row);
  return err <= 1e-5 ? 0 : 1;
}

static int check_dense64(void) {
  const int n = 500, d = 300, k = 70, m = 90;
  double* a = malloc(sizeof(double) * n * d);
  double* om = malloc(sizeof(double) * d * k);
  double* b = malloc(sizeof(double) * d * m);
  for (int i = 0; i < n * d; ++i) a[i] = normal();
  for (int i = 0; i < d * k; ++i) om[i] = normal() / sqrt((double)k);
  for (int i = 0; i < d * m; ++i) b[i] = normal();
  double *da, *dom, *db, *dy, *dx;
  CK(cudaMalloc((void**)&da, sizeof(double) * n * d));
  CK(cudaMalloc((void**)&dom, sizeof(double) * d * k));
  CK(cudaMalloc((void**)&db, sizeof(double) * d * m));
  CK(cudaMalloc((void**)&dy, sizeof(double) * n * k));
  CK(cudaMalloc((void**)&dx, sizeof(double) * k * m));
  CK(cudaMemcpy(da, a, sizeof(double) * n * d, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dom, om, sizeof(double) * d * k, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db, b, sizeof(double) * d * m, cudaMemcpyHostToDevice));
  SK(sk_kr_right_cc(SK_F64, da, n, 1, d, d, dom, k, NULL, 0, k, 1.0, dy, k, NULL));
  SK(sk_kr_adjoint_cc(SK_F64, db, m, 1, d, m, dom, k, NULL, 0, k, 1.0, dx, m, NULL));
  CK(cudaDeviceSynchronize());
  double* y = malloc(sizeof(double) * n * k);
  double* x = malloc(sizeof(double) * k * m);
  CK(cudaMemcpy(y, dy, sizeof(double) * n * k, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(x, dx, sizeof(double) * k * m, cudaMemcpyDeviceToHost));
  double* ry = calloc((size_t)n * k, sizeof(double));
  double* rx = calloc((size_t)k * m, sizeof(double));
  for (int i = 0; i < n; ++i)
    for (int r = 0; r < d; ++r)
      for (int c = 0; c < k; ++c) ry[(size_t)i * k + c] += a[(size_t)i * d + r] * om[(size_t)r * k + c];
  for (int r = 0; r < d; ++r)
    for (int c = 0; c < k; ++c)
      for (int j = 0; j < m; ++j) rx[(size_t)c * m + j] += om[(size_t)r * k + c] * b[(size_t)r * m + j];
  const double ey = rel_err(y, ry, (size_t)n * k), ex = rel_err(x, rx, (size_t)k * m);
  printf("dense f64: right rel err %.3e, adjoint rel err %.3e\n", ey, ex);
  cudaFree(da);
  cudaFree(dom);
  cudaFree(db);
  cudaFree(dy);
  cudaFree(dx);
  free(a);
  free(om);
  free(b);
  free(y);
  free(x);
  free(ry);
  free(rx);
  return (ey <= 1e-12 && ex <= 1e-12) ? 0 : 1;
}

static int check_sparse_cols(void) {
  const int n = 700, d = 2048, k = 300, zeta = 4;
  const double mag = 1.0 / sqrt((double)zeta);
  int64_t* rows = malloc(sizeof(int64_t) * d * zeta);
  int64_t* cols = malloc(sizeof(int64_t) * d * zeta);
  uint8_t* neg = malloc((size_t)d * zeta);
  for (int r = 0; r < d; ++r)
    for (int z = 0; z < zeta; ++z) {
      int c, dup;
      do { /* zeta distinct columns per row */
        c = (int)(next_u64() % k);
        dup = 0;
        for (int q = 0; q < z; ++q) dup |= cols[r * zeta + q] == c;
      } while (dup);
      rows[r * zeta + z] = r;
      cols[r * zeta + z] = c;
      neg[r * zeta + z] = (uint8_t)(next_u64() & 1);
    }
  const int groups = sk_sparse_right_cols_groups(k);
  int32_t* colmap = malloc(sizeof(int32_t) * groups * 256);
  int32_t* tw = malloc(sizeof(int32_t) * groups * 8);
  int32_t need = 0;
  SK(sk_sparse_right_cols_encode(SK_F64, d, k, (int64_t)d * zeta, rows, cols, neg, 0, NULL, colmap, tw, &need));
  const int32_t maxp = need <= 32 ? 32 : need <= 64 ? 64 : need <= 96 ? 96 : 128;
  if (need > 128 || !sk_sparse_right_cols_supported(SK_F64, d, k, maxp)) {
    fprintf(stderr, "sparse cols: unexpected plan (need %d)\n", need);
    return 1;
  }
  uint32_t* ent = malloc(sizeof(uint32_t) * groups * 8 * maxp * 32);
  SK(sk_sparse_right_cols_encode(SK_F64, d, k, (int64_t)d * zeta, rows, cols, neg, maxp, ent, colmap, tw, &need));
  double* a = malloc(sizeof(double) * n * d);
  for (int i = 0; i < n * d; ++i) a[i] = normal();
  double *da, *dy;
  uint32_t* dent;
  int32_t *dcolmap, *dtw;
  CK(cudaMalloc((void**)&da, sizeof(double) * n * d));
  CK(cudaMalloc((void**)&dy, sizeof(double) * n * k));
  CK(cudaMalloc((void**)&dent, sizeof(uint32_t) * groups * 8 * maxp * 32));
  CK(cudaMalloc((void**)&dcolmap, sizeof(int32_t) * groups * 256));
  CK(cudaMalloc((void**)&dtw, sizeof(int32_t) * groups * 8));
  CK(cudaMemcpy(da, a, sizeof(double) * n * d, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dent, ent, sizeof(uint32_t) * groups * 8 * maxp * 32, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dcolmap, colmap, sizeof(int32_t) * groups * 256, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dtw, tw, sizeof(int32_t) * groups * 8, cudaMemcpyHostToDevice));
  SK(sk_sparse_right_cols(SK_F64, da, n, d, d, dent, dcolmap, dtw, k, maxp, mag, dy, k, 0, NULL));
  CK(cudaDeviceSynchronize());
  double* y = malloc(sizeof(double) * n * k);
  CK(cudaMemcpy(y, dy, sizeof(double) * n * k, cudaMemcpyDeviceToHost));
  double* ref = calloc((size_t)n * k, sizeof(double));
  for (int i = 0; i < n; ++i)
    for (int e = 0; e < d * zeta; ++e) {
      const double v = a[(size_t)i * d + rows[e]] * mag;
      ref[(size_t)i * k + cols[e]] += neg[e] ? -v : v;
    }
  const double err = rel_err(y, ref, (size_t)n * k);
  printf("sparse sign f64 (K1c, maxp %d): rel err %.3e\n", maxp, err);
  cudaFree(da);
  cudaFree(dy);
  cudaFree(dent);
  cudaFree(dcolmap);
  cudaFree(dtw);
  free(rows);
  free(cols);
  free(neg);
  free(colmap);
  free(tw);
  free(ent);
  free(a);
  free(y);
  free(ref);
  return err <= 1e-12 ? 0 : 1;
}

static int check_errors(void) {
  const int st = sk_srtt_right(SK_F32, NULL, 10, 1000 /* not a power of two */, 1000, NULL, SK_WHT, NULL, 1, 4, 1.0,
                               NULL, 4, NULL);
  printf("bad shape -> %d (%s)\n", st, sk_last_error());
  return (st < 0 && strlen(sk_last_error()) > 0) ? 0 : 1;
}

int main(void) {
  if (sk_abi_version() != SK_ABI_VERSION) {
    fprintf(stderr, "ABI version %d, header %d\n", sk_abi_version(), SK_ABI_VERSION);
    return 4;
  }
  printf("libsketch_b200 ABI %d, %d SMs on device 0\n", sk_abi_version(), sk_device_sm_count(0));
  const int fails = check_srtt() + check_dense64() + check_sparse_cols() + check_errors();
  printf(fails ? "FAILED\n" : "ok\n");
  return fails ? 1 : 0;
}
