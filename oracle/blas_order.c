/* TEST INFRASTRUCTURE ONLY -- restatement of the float64 operation order of the BLAS
 * call behind the reference's similarity scan, VectorStore.search
 * (/root/reference/pkg/src/servesim/predictor.py:158: sims = self._vecs[:size] @ vector).
 *
 * Third-party dependency (absent from /root/reference): numpy 2.3.5 ->
 * cblas_dgemv(RowMajor, NoTrans) of scipy-openblas 0.3.30 (DYNAMIC_ARCH, x86-64
 * Haswell/SkylakeX/Zen cores) -> the column-major transposed kernel dgemv_t
 * (kernel/x86_64/dgemv_t_4.c + the Haswell micro-kernel), whose summation order was
 * recovered by differential testing against numpy in this container (the test
 * tests/test_oracle_pred.py::test_blas_order_matches_numpy pins it):
 *   * the n rows are split over T threads when n*d >= 460800 (T = OpenBLAS threads):
 *     widths ceil(remaining / remaining threads), at least 4;
 *   * within a thread's range of w rows, rows [0, w & ~3) use the 4x4 kernel (four
 *     FMA accumulators, element i -> accumulator i % 4, reduced (a0 + a2) + (a1 + a3)),
 *     then two rows the 4x2 kernel if w & 2 (two accumulators, multiply then add,
 *     a0 + a1), then one row the 4x1 kernel if w & 1 (four accumulators, multiply then
 *     add, (a0 + a2) + (a1 + a3));
 *   * the dot dimension is cut into blocks of 2048 (the last block the remainder of
 *     d & ~3); block sums are added to y (y = 0 first);
 *   * the last d & 3 elements: 1: y = fma(a0, x0, y); 2: y + fma(a0, x0, a1 x1);
 *     3: y + fma(a2, x2, fma(a0, x0, a1 x1)).
 * Compiled with -ffp-contract=off: fma() is the only fused operation. */
#include <math.h>
#include <stdint.h>

#define NBMAX 2048
#define MT_THRESHOLD 460800L

static double blk44(const double *a, const double *x, int64_t lo, int64_t hi) {
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (int64_t i = lo; i < hi; i += 4) {
    c0 = fma(a[i], x[i], c0);
    c1 = fma(a[i + 1], x[i + 1], c1);
    c2 = fma(a[i + 2], x[i + 2], c2);
    c3 = fma(a[i + 3], x[i + 3], c3);
  }
  return (c0 + c2) + (c1 + c3);
}
static double blk42(const double *a, const double *x, int64_t lo, int64_t hi) {
  double c0 = 0, c1 = 0;
  for (int64_t i = lo; i < hi; i += 2) {
    c0 = c0 + a[i] * x[i];
    c1 = c1 + a[i + 1] * x[i + 1];
  }
  return c0 + c1;
}
static double blk41(const double *a, const double *x, int64_t lo, int64_t hi) {
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (int64_t i = lo; i < hi; i += 4) {
    c0 = c0 + a[i] * x[i];
    c1 = c1 + a[i + 1] * x[i + 1];
    c2 = c2 + a[i + 2] * x[i + 2];
    c3 = c3 + a[i + 3] * x[i + 3];
  }
  return (c0 + c2) + (c1 + c3);
}

/* one row's dot in the order of kernel `kind` (0: 4x4, 1: 4x2, 2: 4x1) */
double oracle_blas_dot(const double *a, const double *x, int64_t d, int kind) {
  const int64_t m3 = d & 3, m1 = d - m3;
  double y = 0.0;
  for (int64_t b = 0; b < m1; b += NBMAX) {
    const int64_t h = b + NBMAX < m1 ? b + NBMAX : m1;
    y = y + (kind == 0 ? blk44(a, x, b, h) : kind == 1 ? blk42(a, x, b, h) : blk41(a, x, b, h));
  }
  const double *t = a + m1, *u = x + m1;
  if (m3 == 1) {
    y = fma(t[0], u[0], y);
  } else if (m3 == 2) {
    y = y + fma(t[0], u[0], t[1] * u[1]);
  } else if (m3 == 3) {
    y = y + fma(t[2], u[2], fma(t[0], u[0], t[1] * u[1]));
  }
  return y;
}

/* kernel used for row r of an n-row product with dot length d on `threads` threads */
int oracle_blas_kind(int64_t r, int64_t n, int64_t d, int threads) {
  const int T = (n * d < MT_THRESHOLD) ? 1 : (threads < 1 ? 1 : threads);
  int64_t start = 0, left = n;
  for (int t = 0; left > 0; ++t) {
    int64_t w = (left + (T - t) - 1) / (T - t > 0 ? T - t : 1);
    if (w < 4) w = 4;
    if (left < w) w = left;
    if (r < start + w) {
      const int64_t j = r - start, w4 = w & ~(int64_t)3;
      if (j < w4) return 0;
      if ((w & 2) && j < w4 + 2) return 1;
      return 2;
    }
    start += w;
    left -= w;
  }
  return 2;
}

/* y[r] = V[r, :] . x for r < n (V row-major n x d), in the reference's BLAS order */
void oracle_blas_gemv(const double *V, int64_t n, int64_t d, const double *x, double *y, int threads) {
  for (int64_t r = 0; r < n; ++r) y[r] = oracle_blas_dot(V + r * d, x, d, oracle_blas_kind(r, n, d, threads));
}
