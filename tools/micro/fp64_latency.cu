// Dependent-chain latency of float64 add / mul and fp32 add on one warp (clock64).
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x, float xf, int n) {
  double a = x, m = x;
  float f = xf;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, x);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) m = __dmul_rn(m, x);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, xf);
  long long t3 = clock64();
  out[threadIdx.x] = a + m + f;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 32 * 8); cudaMallocManaged(&c, 3 * 8);
  const int n = 4096;
  k<<<1, 32>>>(o, c, 1.0000001, 1.0f, n);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 1.0000001, 1.0f, n);
  cudaDeviceSynchronize();
  printf("{\"dadd_cycles\": %.2f, \"dmul_cycles\": %.2f, \"fadd_cycles\": %.2f}\n", (double)c[0] / n, (double)c[1] / n,
         (double)c[2] / n);
  return 0;
}
