// Batched hashing embedder (the step before the predictor).
//
// Reference: /root/reference/pkg/src/servesim/predictor.py:22-31, 66-100
//   features "u:<t_i>" for every token and "b:<t_{i-1}>:<t_i>" for every adjacent pair,
//   h = FNV-1a-64(feature bytes), bucket h % d, sign + if bit 63 else -, then v / |v|.
// Counts are integers, so the sum of squares is exact in any order and the float64
// sqrt and division are correctly rounded: the output is bit-identical to the
// reference's numpy computation.
#pragma once
#include <stdint.h>

namespace alise {
namespace emb {

constexpr uint64_t FNV_OFFSET = 0xCBF29CE484222325ull;
constexpr uint64_t FNV_PRIME = 0x100000001B3ull;

__device__ __forceinline__ uint64_t fnv_byte(uint64_t h, uint32_t b) { return (h ^ b) * FNV_PRIME; }

// FNV-1a over the decimal representation of v (Python str(int)).
__device__ __forceinline__ uint64_t fnv_int(uint64_t h, int64_t v) {
  if (v < 0) h = fnv_byte(h, '-');
  uint64_t u = v < 0 ? (uint64_t)(-(v + 1)) + 1 : (uint64_t)v;
  char dig[20];
  int n = 0;
  do {
    dig[n++] = (char)('0' + (u % 10));
    u /= 10;
  } while (u);
  while (n) h = fnv_byte(h, (uint32_t)dig[--n]);
  return h;
}

// One block per prompt; counts in shared memory (dim <= 8192).
__global__ void k_embed(const int64_t* __restrict__ tokens, const int64_t* __restrict__ offsets, int64_t dim,
                        double* __restrict__ out64, float* __restrict__ out32) {
  extern __shared__ int cnt[];
  const int64_t b = blockIdx.x;
  const int64_t t0 = offsets[b], t1 = offsets[b + 1];
  for (int64_t i = threadIdx.x; i < dim; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const int64_t t = tokens[i];
    uint64_t h = fnv_byte(fnv_byte(FNV_OFFSET, 'u'), ':');
    h = fnv_int(h, t);
    atomicAdd(&cnt[h % (uint64_t)dim], (h >> 63) ? 1 : -1);
    if (i > t0) {
      uint64_t g = fnv_byte(fnv_byte(FNV_OFFSET, 'b'), ':');
      g = fnv_int(g, tokens[i - 1]);
      g = fnv_byte(g, ':');
      g = fnv_int(g, t);
      atomicAdd(&cnt[g % (uint64_t)dim], (g >> 63) ? 1 : -1);
    }
  }
  __syncthreads();
  __shared__ unsigned long long ss;
  if (threadIdx.x == 0) ss = 0;
  __syncthreads();
  unsigned long long part = 0;
  for (int64_t i = threadIdx.x; i < dim; i += blockDim.x) part += (unsigned long long)((int64_t)cnt[i] * cnt[i]);
  atomicAdd(&ss, part);
  __syncthreads();
  double norm = sqrt((double)ss);  // exact integer, correctly rounded sqrt
  const bool zero = ss == 0;       // cannot happen with >= 1 token; kept like the reference
  if (zero) norm = 1.0;
  for (int64_t i = threadIdx.x; i < dim; i += blockDim.x) {
    double v = (double)cnt[i];
    if (zero && i == 0) v = 1.0;
    const double r = __ddiv_rn(v, norm);
    if (out64) out64[b * dim + i] = r;
    if (out32) out32[b * dim + i] = (float)r;
  }
}

}  // namespace emb
}  // namespace alise
