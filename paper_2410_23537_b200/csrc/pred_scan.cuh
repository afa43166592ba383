// Predictor kernels (sm_100a): DB ring append, query prep, the tcgen05 coarse scan
// with a fused candidate filter, exact float64 rescoring + (-sim, seq) top-k, the
// cross-shard merge and the aggregate / all-MLP finish.
//
// Reference: /root/reference/pkg/src/servesim/predictor.py
//   VectorStore.add / search   :135-163   (ring slot = seq % capacity; sims = V @ q;
//                                          order (-sim, seq))
//   LengthPredictor.predict_vector :311-325, FallbackRegressor._forward/predict_len :209-219
//
// Exactness argument: the coarse score s~ = fp16(q).fp16(v) with
// fp32 accumulation differs from the exact dot product s by at most
//   delta_q = |q| * Vmax * (2^-10 + D*2^-21) + (|q| + Vmax) * sqrt(D) * 2^-24,
// so every row of the exact top-k has s~ >= (k-th largest s~) - 2*delta_q.  Each scan
// CTA keeps, per query, its running top-k of s~ and appends every row that reaches
// (running k-th) - 2*delta_q; since the running k-th never exceeds the final one the
// appended set is a superset of the needed candidates.  Candidates are rescored with a
// double-double float64 dot product whose correct rounding is verified per candidate.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "sm100.cuh"

namespace alise {
namespace pred {

constexpr int BM = 128;        // queries per CTA (TMEM lanes)
constexpr int BN = 256;        // DB rows per tile (UMMA N)
constexpr int BK = 64;         // K per pipeline stage (128-byte rows, SW128)
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int KMAX = 16;       // largest supported k
constexpr int CAP = 128;       // candidate slots per (split, query)
constexpr int SCAN_SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int MAXC = 512;      // candidates rescored per query

// ------------------------------------------------------------------ DB maintenance
// The master copy is fp32 or float64 (T): float64 keeps the reference's float64 vectors
// (HashingEmbedder output, predictor.py:66-100) exactly, so sims, newest() and the refit
// data are those of the reference store (predictor.py:126).
__device__ __forceinline__ __half to_half(float v) { return __float2half_rn(v); }
__device__ __forceinline__ __half to_half(double v) { return __double2half(v); }
constexpr float HALF_MAX = 65504.f;

// Append n rows at ring slots seq % capacity: master (T), fp16 coarse copy (zero padded
// to dp), lengths, seqs; track an upper bound of the row L2 norms.  A component beyond
// the fp16 range (or a non-finite one) makes the coarse copy meaningless: Vmax becomes
// +inf, which routes every later query through the exhaustive exact path.
template <typename T>
__global__ void k_db_append(const T* __restrict__ vecs, const int32_t* __restrict__ lens,
                            const int64_t* __restrict__ seqs, int64_t n, int64_t dim, int64_t dp,
                            int64_t capacity, int64_t stride, T* __restrict__ vm, __half* __restrict__ v16,
                            int32_t* __restrict__ dlens, int64_t* __restrict__ dseqs,
                            unsigned int* __restrict__ vmax_bits) {
  const int64_t i = blockIdx.x;
  if (i >= n) return;
  const int64_t slot = (seqs[i] / stride) % capacity;
  double ss = 0.0;
  bool huge = false;
  for (int64_t d = threadIdx.x; d < dp; d += blockDim.x) {
    const T v = d < dim ? vecs[i * dim + d] : T(0);
    if (d < dim) vm[slot * dim + d] = v;
    v16[slot * dp + d] = to_half(v);
    huge |= !(fabs((double)v) <= (double)HALF_MAX);
    ss += (double)v * (double)v;
  }
  __shared__ double red[32];
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  huge = __syncthreads_or(huge);
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    dlens[slot] = lens[i];
    dseqs[slot] = seqs[i];
    // round the norm up so Vmax stays an upper bound (float64 sum of squares: relative
    // error below (dim + 8) * 2^-53)
    const float nrm = huge ? __int_as_float(0x7f800000)
                           : __double2float_ru(sqrt(t) * (1.0 + (double)(dim + 64) * 0x1p-52));
    atomicMax(vmax_bits, __float_as_uint(nrm));
  }
}

// Queries: T [B][dim] -> fp16 [Bp][dp] (zero padded) and 2*delta per query (+inf when
// the query or the DB leaves the fp16 range: the rescoring then takes the exhaustive path).
// delta bounds |coarse - sim| for the sims the rescoring ranks by (correctly rounded, or
// in the reference's BLAS order).
// (gkth / need may be NULL; when given, the query's shared k-th, rank slots and
// exhaustive flag are cleared here instead of by separate memsets)
template <typename T>
__global__ void k_query_prep(const T* __restrict__ q, int64_t B, int64_t dim, int64_t dp,
                             const unsigned int* __restrict__ vmax_bits, __half* __restrict__ q16,
                             float* __restrict__ two_delta, int blas_order, uint32_t* __restrict__ gkth,
                             int32_t* __restrict__ need) {
  const int64_t i = blockIdx.x;
  if (gkth) {  // [Bp] shared k-th, then [Bp][KMAX] rank slots
    if (threadIdx.x == 0) gkth[i] = 0u;
    if (threadIdx.x < KMAX) gkth[(int64_t)gridDim.x + i * KMAX + threadIdx.x] = 0u;
  }
  if (need && threadIdx.x == 0) need[i] = 0;
  double ss = 0.0;
  bool huge = false;
  for (int64_t d = threadIdx.x; d < dp; d += blockDim.x) {
    const T v = (i < B && d < dim) ? q[i * dim + d] : T(0);
    q16[i * dp + d] = to_half(v);
    huge |= !(fabs((double)v) <= (double)HALF_MAX);
    ss += (double)v * (double)v;
  }
  __shared__ double red[32];
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  huge = __syncthreads_or(huge);
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    const double qn = sqrt(t) * (1.0 + (double)(dim + 64) * 0x1p-52);
    const double V = (double)__uint_as_float(*vmax_bits);
    const double D = (double)dim;
    // (+ the reference-BLAS-order sims' own error: at most (dim / 2 + 32) 2^-52 sum|p|,
    // sum|p| <= |q| Vmax, when the rescoring ranks by them)
    const double delta = qn * V * (0x1p-10 + D * 0x1p-21 + (blas_order ? (D * 0.5 + 32.0) * 0x1p-52 : 0.0)) +
                         (qn + V) * sqrt(D) * 0x1p-24;
    two_delta[i] = (huge || !(V <= 1e30)) ? __int_as_float(0x7f800000) : __double2float_ru(2.0 * delta);
  }
}

// ------------------------------------------------------------------ tcgen05 scan
struct ScanArgs {
  int n_kb;          // padded dim / 64
  int64_t n_rows;    // valid DB rows (slots [0, n_rows))
  int n_tiles;       // ceil(n_rows / BN)
  int n_qb;          // query blocks of 128
  int n_splits;      // max splits per query block (candidate-list slots, see next_seg)
  int G;             // tile groups per query block: group g scans tiles g, g + G, ...
  int units;         // persistent CTAs (1-SM) or CTA pairs (2-SM)
  int E;             // excess groups (see next_seg)
  int nc;            // chunks per excess group
  int C;             // tiles per chunk
  int B;             // real query count
  int Bp;            // padded query count
  int k;
  const float* two_delta;
  float* cand_s;     // [n_splits][Bp][CAP]
  int32_t* cand_r;   // [n_splits][Bp][CAP]
  int32_t* cand_n;   // [n_splits][Bp]   (-1 = overflow)
  float* topc;       // [n_splits][Bp][KMAX]
  uint32_t* gkth;    // [Bp] shared running k-th per query (ord_key; 0 = none yet)
  int warm;          // warm-start bound from each group's first tile (QueryScan)
  uint32_t* gslot;   // [Bp][KMAX] rank slots per query (ord_key; 0 = empty)
  int slot_m;        // ranks each group publishes into the slots
  int sync_tile;     // exchange the shared bounds once per tile instead of per 64 scores
};

__device__ __forceinline__ uint4 ld_relaxed_v4(const uint32_t* p) {
  uint4 r;
  asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p) : "memory");
  return r;
}

// Order-preserving float <-> uint32 (atomicMax on the key = max on the float).
__device__ __forceinline__ uint32_t ord_key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord_val(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// Running top-k of one query in registers, right-aligned: slots [0, KT-k) hold +inf
// (never displaced), the k live values are top[KT-k..KT-1] sorted descending, so the
// k-th is always top[KT-1] (a static register: a runtime index would move the list to
// local memory).  p[i] = s > top[i] is monotone in i, so every slot is computed in
// parallel from the old list (depth 3 instead of a KT-long chain).
template <int KT>
__device__ __forceinline__ void topk_init(float (&top)[KT], int k) {
#pragma unroll
  for (int x = 0; x < KT; ++x) top[x] = x < KT - k ? __int_as_float(0x7f800000) : -__int_as_float(0x7f800000);
}

template <int KT>
__device__ __forceinline__ float topk_insert(float (&top)[KT], float s) {
  bool p[KT];
#pragma unroll
  for (int i = 0; i < KT; ++i) p[i] = s > top[i];
#pragma unroll
  for (int i = KT - 1; i > 0; --i) top[i] = p[i] ? (p[i - 1] ? top[i - 1] : s) : top[i];
  top[0] = p[0] ? s : top[0];
  return top[KT - 1];
}

template <int KT>
__device__ __forceinline__ void topk_store(const float (&top)[KT], int k, float* __restrict__ out) {
#pragma unroll
  for (int x = 0; x < KT; ++x)
    if (x >= KT - k) out[x - (KT - k)] = top[x];
}

// Compaction of a full candidate buffer against the risen threshold (rare).
__device__ __forceinline__ int compact_candidates(float* __restrict__ cs, int32_t* __restrict__ cr, float thr) {
  int w = 0;
  for (int u = 0; u < CAP; ++u) {
    const float sv = cs[u];
    if (sv >= thr) {
      cs[w] = sv;
      cr[w] = cr[u];
      ++w;
    }
  }
  return w;
}

// ---------------------------------------------------------------- work split
// Every query block has G tile groups (group g = tiles g, g+G, ...), G = ceil(units /
// n_qb), so n_qb*G - E = units for E < n_qb excess groups: group G-1 of the last E
// query blocks.  Unit p first scans one whole non-excess group (all units sweep the DB
// in near lock step: L2 reuse across query blocks), then chunks of the excess groups
// (nc chunks of C tiles per excess group; chunk c of every excess group covers the same
// tile positions, so those run in lock step too).  Every unit does about the same number
// of tiles: with whole groups only, the units of the blocks that get one group fewer
// would run 1/G longer than the rest.  Each group or chunk is a split (its own candidate
// list): splits 0..G-1 are the groups, chunk c of a block's excess group is split G-1+c.
struct WorkSeg {
  int qb, split, g, pos, count;  // tiles g + (pos + i) * G, i < count
};

__device__ __forceinline__ int grp_len(int n_tiles, int G, int g) { return n_tiles / G + (g < n_tiles % G ? 1 : 0); }

__device__ __forceinline__ int splits_of_block(const ScanArgs& a, int qb) {
  if (qb < a.n_qb - a.E) return a.G;
  const int len = grp_len(a.n_tiles, a.G, a.G - 1);
  return a.G - 1 + (len + a.C - 1) / a.C;
}

// next segment of unit p (state starts at 0)
__device__ __forceinline__ bool next_seg(const ScanArgs& a, int p, int& state, WorkSeg& s) {
  if (state == 0) {
    state = 1;
    const int full = (a.n_qb - a.E) * a.G;
    if (p < full) {
      s.qb = p / a.G;
      s.g = p % a.G;
    } else {
      const int p2 = p - full;
      s.qb = a.n_qb - a.E + p2 / (a.G - 1);
      s.g = p2 % (a.G - 1);
    }
    s.split = s.g;
    s.pos = 0;
    s.count = grp_len(a.n_tiles, a.G, s.g);
    return true;
  }
  const int len = grp_len(a.n_tiles, a.G, a.G - 1);
  for (;;) {
    const int cid = p + a.units * (state - 1);
    if (cid >= a.E * a.nc) return false;
    ++state;
    const int e = cid / a.nc, c = cid % a.nc;
    const int pos0 = c * a.C;
    if (pos0 >= len) continue;
    s.qb = a.n_qb - a.E + e;
    s.g = a.G - 1;
    s.split = a.G - 1 + c;
    s.pos = pos0;
    s.count = min(a.C, len - pos0);
    return true;
  }
}

// Per-(query, tile group) state of the scan epilogue (one thread): running top-k of the
// coarse scores, candidate threshold thr = (lower bound g of the final k-th) - 2*delta,
// and the candidate buffer.  Any g <= the final k-th keeps the candidate set a superset
// (rows below g - 2*delta cannot be in the exact top-k).  Each group sees only 1/G of
// the DB, so g is raised faster than by the group's own k-th:
//  * warm start: on its first full tile a split takes the k-th largest of the tile's
//    32 maxima of 8 consecutive rows (k distinct rows reach it; k <= 32);
//  * gkth: the largest bound any group of the query has published, exchanged once per
//    64 scores, or per tile when groups are long (loads issued one exchange ahead);
//  * rank slots: group g publishes its m best values (m = ceil(k / G)) into slots
//    (g*m + i) % k with atomic max.  A slot's value is at most the current i-th best of
//    the group that wrote it and distinct slots come from distinct (group, rank) pairs,
//    i.e. distinct rows, so once all k slots are filled their minimum is a bound of the
//    k-th over the union of the groups (much tighter than the best group's own k-th).
// Values <= kfloor (the best shared bound) are not inserted into top[]: the union of
// the groups' lists already holds k values >= it (correctness does not depend on it:
// the rescoring k-th is taken from the union of the lists, a subset of all rows).
template <int KT>
struct QueryScan {
  float top[KT];
  float thr, kth, kfloor, td;
  uint32_t pub, gk;
  uint32_t* gkp;  // this query's shared bound (nullptr for padding queries)
  int cnt;
  bool ovf;
  float* cs;
  int32_t* cr;
  uint32_t* sl;  // this query's rank slots
  int m, sbase;
  bool dirty;    // top[] changed since the last slot publish
  uint4 sv[KT / 4];

  __device__ __forceinline__ void init(const ScanArgs& a, int q, size_t base, int k, int g) {
    topk_init<KT>(top, k);
    td = a.two_delta[q];
    // padding queries (q >= B) never pass
    thr = q < a.B ? -__int_as_float(0x7f800000) : __int_as_float(0x7f800000);
    kth = -__int_as_float(0x7f800000);
    kfloor = -__int_as_float(0x7f800000);
    pub = 0;
    gk = 0;
    gkp = q < a.B ? a.gkth + q : nullptr;
    cnt = 0;
    ovf = false;
    cs = a.cand_s + base * CAP;
    cr = a.cand_r + base * CAP;
    sl = a.gslot + (size_t)q * KMAX;
    m = a.slot_m;
    sbase = g * m;
    dirty = false;
    pref();
    // a split that starts mid-run (an excess chunk) takes the query's shared bounds now
    if (gkp) {
      if (gk) raise(ord_val(gk));
      uint32_t mn = 0xffffffffu;
#pragma unroll
      for (int x = 0; x < KT / 4; ++x) {
        if (4 * x + 0 < k) mn = min(mn, sv[x].x);
        if (4 * x + 1 < k) mn = min(mn, sv[x].y);
        if (4 * x + 2 < k) mn = min(mn, sv[x].z);
        if (4 * x + 3 < k) mn = min(mn, sv[x].w);
      }
      if (mn) raise(ord_val(mn));
    }
  }

  __device__ __forceinline__ void raise(float g) {
    const float t = __fsub_rn(g, td);
    if (t > thr) thr = t;
    if (g > kfloor) kfloor = g;
  }

  __device__ __forceinline__ void publish(float g) {
    const uint32_t key = ord_key(g);
    if (key > pub) {
      atomicMax(gkp, key);
      pub = key;
    }
  }

  // warm start: a bound from the split's first full tile (warm_from_tile)
  __device__ __forceinline__ void warm(float g) {
    if (!gkp || !(g > -__int_as_float(0x7f800000))) return;
    raise(g);
    publish(g);
  }

  // issue the shared-bound loads for the next block (consumed by the next sync, a whole
  // block of scores later, so the L2 latency is hidden)
  __device__ __forceinline__ void pref() {
    if (!gkp) return;
    gk = *reinterpret_cast<volatile uint32_t*>(gkp);
#pragma unroll
    for (int x = 0; x < KT / 4; ++x) sv[x] = ld_relaxed_v4(sl + 4 * x);
  }

  // after the block: publish the own k-th and best values, take the loaded bounds
  __device__ __forceinline__ void sync(int k) {
    if (!gkp) return;
    if (kth > -__int_as_float(0x7f800000)) publish(kth);
    if (gk) raise(ord_val(gk));
    if (dirty) {
      dirty = false;
#pragma unroll
      for (int x = 0; x < KT; ++x) {
        const int r = x - (KT - k);  // rank of slot x in the right-aligned list
        if (r >= 0 && r < m && top[x] > -__int_as_float(0x7f800000))
          atomicMax(sl + (sbase + r) % k, ord_key(top[x]));
      }
    }
    uint32_t mn = 0xffffffffu;
#pragma unroll
    for (int x = 0; x < KT / 4; ++x) {
      if (4 * x + 0 < k) mn = min(mn, sv[x].x);
      if (4 * x + 1 < k) mn = min(mn, sv[x].y);
      if (4 * x + 2 < k) mn = min(mn, sv[x].z);
      if (4 * x + 3 < k) mn = min(mn, sv[x].w);
    }
    if (mn) raise(ord_val(mn));
    pref();
  }

  // one coarse score sc of DB row `row` (a real row)
  __device__ __forceinline__ void hit(float sc, int row) {
    if (!(sc >= thr)) return;
    if (sc > kth && sc > kfloor) {
      kth = topk_insert<KT>(top, sc);
      thr = fmaxf(thr, __fsub_rn(kth, td));
      dirty = true;
    }
    if (ovf) return;
    if (cnt == CAP) {
      cnt = compact_candidates(cs, cr, thr);
      if (cnt == CAP) {
        ovf = true;
        return;
      }
    }
    cs[cnt] = sc;
    cr[cnt] = row;
    ++cnt;
  }

  __device__ __forceinline__ void finish(const ScanArgs& a, size_t base, int k) {
    a.cand_n[base] = ovf ? -1 : cnt;
    topk_store<KT>(top, k, a.topc + base * KMAX);
  }
};

// max of 32 scores as a tree of 3-input maxes (FMNMX3: 16 instructions)
__device__ __forceinline__ float max32(const float (&v)[32]) {
  float t[11];
#pragma unroll
  for (int x = 0; x < 10; ++x) t[x] = fmaxf(fmaxf(v[3 * x], v[3 * x + 1]), v[3 * x + 2]);
  t[10] = fmaxf(v[30], v[31]);
  const float u0 = fmaxf(fmaxf(t[0], t[1]), t[2]), u1 = fmaxf(fmaxf(t[3], t[4]), t[5]);
  const float u2 = fmaxf(fmaxf(t[6], t[7]), t[8]), u3 = fmaxf(t[9], t[10]);
  return fmaxf(fmaxf(u0, u1), fmaxf(u2, u3));
}

// First full tile of a split: the k-th largest of the 32 maxima of 8 consecutive
// columns over the whole 256-column tile of this thread's query (TMEM lane; both
// epilogue halves of a lane quarter may read all columns) is the warm-start bound:
// k distinct rows reach it (k <= 32).
template <int KT>
__device__ __forceinline__ void warm_from_tile(QueryScan<KT>& qs, uint32_t tile_addr, int k) {
  float tk[KT];
  topk_init<KT>(tk, k);
#pragma unroll 1
  for (int c2 = 0; c2 < BN / 64; ++c2) {
    uint32_t r0[32], r1[32];
    sm100::tmem_ld32_async(tile_addr + c2 * 64, r0);
    sm100::tmem_ld32_async(tile_addr + c2 * 64 + 32, r1);
    sm100::tmem_wait_ld();
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const uint32_t* r = x < 4 ? r0 : r1;
      const int o = (x & 3) * 8;
      float m = __uint_as_float(r[o]);
#pragma unroll
      for (int y = 1; y < 8; ++y) m = fmaxf(m, __uint_as_float(r[o + y]));
      if (m > tk[KT - 1]) topk_insert<KT>(tk, m);
    }
  }
  qs.warm(tk[KT - 1]);
}

// Scores of one 32-row chunk (v[x] = row rbase + x): one max-reduction and one
// compare per 32 scores on the hot path; the warp then walks the union of the 4-value
// groups its lanes hit, the group's values picked by a warp-uniform switch so each
// lane tests them by static register.
template <int KT>
__device__ __forceinline__ void scan_chunk(QueryScan<KT>& qs, const float (&v)[32], int rbase, int64_t n_rows) {
  if (!__any_sync(0xffffffffu, max32(v) >= qs.thr)) return;
  // rare path: which 4-value groups hit
  float m8[8];
#pragma unroll
  for (int x = 0; x < 8; ++x) m8[x] = fmaxf(fmaxf(v[4 * x], v[4 * x + 1]), fmaxf(v[4 * x + 2], v[4 * x + 3]));
  uint32_t gm = 0;
#pragma unroll
  for (int x = 0; x < 8; ++x) gm |= (m8[x] >= qs.thr ? 1u : 0u) << x;
  uint32_t gu = __reduce_or_sync(0xffffffffu, gm);
  const int64_t rlim = n_rows - rbase;  // value x is a real row iff x < rlim
  while (gu) {
    const int g8 = __ffs(gu) - 1;
    gu &= gu - 1;
    float w[4];
    switch (g8) {
#define ALISE_PICK(G) case G: w[0] = v[4 * G]; w[1] = v[4 * G + 1]; w[2] = v[4 * G + 2]; w[3] = v[4 * G + 3]; break;
      ALISE_PICK(0) ALISE_PICK(1) ALISE_PICK(2) ALISE_PICK(3)
      ALISE_PICK(4) ALISE_PICK(5) ALISE_PICK(6) default: ALISE_PICK(7)
#undef ALISE_PICK
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
      if (4 * g8 + x < rlim) qs.hit(w[x], rbase + 4 * g8 + x);
  }
}

// Persistent CTAs.  Work item w = (query block qb, tile group g): the CTA keeps one
// running top-k per query across all tiles t = g, g+G, g+2G, ... (so the threshold
// warms up once), and the n_qb CTAs of a group walk the same tile sequence in lock
// step, so each DB tile is read from HBM once and from L2 by the other query blocks.
template <int KT>
__global__ void __launch_bounds__(192, 1)
k_scan(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmD, const ScanArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tmQ);
    sm100::prefetch_tmap(&tmD);
    for (int s = 0; s < STAGES; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&tfull[s], 1);
      sm100::mbar_init(&tempty[s], 4);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc<512>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      int st = 0;
      WorkSeg sg;
      while (next_seg(a, blockIdx.x, st, sg)) {
        const int qb = sg.qb;
        for (int u = 0; u < sg.count; ++u) {
          const int t = sg.g + (sg.pos + u) * a.G;
          for (int kb = 0; kb < a.n_kb; ++kb) {
            sm100::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * STAGE_BYTES;
            sm100::mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
            sm100::tma_load_2d(&tmQ, sa, &full[stage], kb * BK, qb * BM);
            sm100::tma_load_2d(&tmD, sa + A_BYTES, &full[stage], kb * BK, t * BN);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer (one thread)
      constexpr uint32_t idesc = sm100::idesc_f16_f32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      int st = 0;
      WorkSeg sg;
      while (next_seg(a, blockIdx.x, st, sg)) {
        for (int u = 0; u < sg.count; ++u, ++i) {
          const int acc = i & 1;
          const uint32_t aph = (i >> 1) & 1;
          sm100::mbar_wait(&tempty[acc], aph ^ 1);
          sm100::tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < a.n_kb; ++kb) {
            sm100::mbar_wait(&full[stage], phase);
            sm100::tc_fence_after();
            const uint32_t a0 = sm100::smem_u32(smem + stage * STAGE_BYTES);
            const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              sm100::umma_f16(d_tmem, sm100::umma_desc_sw128(a0 + kk * 32),
                              sm100::umma_desc_sw128(b0 + kk * 32), idesc, (kb | kk) != 0);
            }
            sm100::umma_commit(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          sm100::umma_commit(&tfull[acc]);
        }
      }
    }
  } else {  // ---------------- epilogue: warps 2..5, thread = query
    const int quarter = warp & 3;
    const int tq = quarter * 32 + lane;
    const int k = a.k;
    int i = 0;
    int st = 0;
    WorkSeg sg;
    while (next_seg(a, blockIdx.x, st, sg)) {
      const int q = sg.qb * BM + tq;
      const size_t base = ((size_t)sg.split * a.Bp + q);
      QueryScan<KT> qs;
      qs.init(a, q, base, k, sg.split);
      for (int u = 0; u < sg.count; ++u, ++i) {
        const int t = sg.g + (sg.pos + u) * a.G;
        const int acc = i & 1;
        const uint32_t aph = (i >> 1) & 1;
        sm100::mbar_wait(&tfull[acc], aph);
        sm100::tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN;
        if (a.warm && u == 0 && (int64_t)(t + 1) * BN <= a.n_rows) warm_from_tile<KT>(qs, taddr, k);
#pragma unroll 1
        for (int c2 = 0; c2 < BN / 64; ++c2) {
          // two TMEM loads in flight per wait
          uint32_t r0[32], r1[32];
          const uint32_t ta = taddr + c2 * 64;
          sm100::tmem_ld32_async(ta, r0);
          sm100::tmem_ld32_async(ta + 32, r1);
          sm100::tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float v[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) v[x] = __uint_as_float(h ? r1[x] : r0[x]);
            scan_chunk<KT>(qs, v, t * BN + (2 * c2 + h) * 32, a.n_rows);
          }
          if (!a.sync_tile || c2 == BN / 64 - 1) qs.sync(k);
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&tempty[acc]);
      }
      qs.finish(a, base, k);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem_base);
  }
}

// ------------------------------------------------------------------ 2-SM scan
// cta_group::2 variant: a CTA pair (cluster of 2 on one TPC) computes 256 queries x
// 256 DB rows per tile with one UMMA M=256 stream issued by the leader; each CTA
// stages its own 128 queries (A) and its half of the 256 DB rows (B), so shared-memory
// and L2 traffic per MMA drop by a third versus the 1-SM kernel.  TMA of both CTAs
// completes on the leader's full barrier; the leader's commits are multicast to both
// CTAs (stage-free and accumulator-full); both CTAs' epilogues release the TMEM
// accumulator to the leader.  Epilogue logic is the same as k_scan.
constexpr int STAGES2 = 7;  // 7 x 32 KB: the hit path needs no smem staging
constexpr int A2_BYTES = BM * BK * 2;         // 16 KB: this CTA's 128 queries
constexpr int B2_BYTES = (BN / 2) * BK * 2;   // 16 KB: this CTA's 128 DB rows
constexpr int STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr int SCAN2_SMEM = STAGES2 * STAGE2_BYTES + 1024 + 256;

template <int KT, int NH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 128 * NH, 1)
k_scan2(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmD, const ScanArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);


  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const int pair = blockIdx.x >> 1;

  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tmQ);
    sm100::prefetch_tmap(&tmD);
    for (int s = 0; s < STAGES2; ++s) {
      sm100::mbar_init(&full[s], 1);
      sm100::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&tfull[s], 1);
      sm100::mbar_init(&tempty[s], 8 * NH);  // 4*NH epilogue warps x 2 CTAs (leader's copy used)
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc_2sm<512>(tmem_slot);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      int st = 0;
      WorkSeg sg;
      while (next_seg(a, pair, st, sg)) {
        const int qp = sg.qb;
        for (int u = 0; u < sg.count; ++u) {
          const int t = sg.g + (sg.pos + u) * a.G;
          for (int kb = 0; kb < a.n_kb; ++kb) {
            sm100::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * STAGE2_BYTES;
            if (rank == 0) sm100::mbar_arrive_expect_tx(&full[stage], 2 * STAGE2_BYTES);
            const uint32_t fb = sm100::mapa(sm100::smem_u32(&full[stage]), 0);
            sm100::tma_load_2d_2sm(&tmQ, sa, fb, kb * BK, qp * 2 * BM + (int)rank * BM);
            sm100::tma_load_2d_2sm(&tmD, sa + A2_BYTES, fb, kb * BK, t * BN + (int)rank * (BN / 2));
            if (++stage == STAGES2) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (leader CTA, one thread)
      constexpr uint32_t idesc = sm100::idesc_f16_f32(2 * BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int i = 0;
      int st = 0;
      WorkSeg sg;
      while (next_seg(a, pair, st, sg)) {
        for (int u = 0; u < sg.count; ++u, ++i) {
          const int acc = i & 1;
          const uint32_t aph = (i >> 1) & 1;
          sm100::mbar_wait(&tempty[acc], aph ^ 1);
          sm100::tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = 0; kb < a.n_kb; ++kb) {
            sm100::mbar_wait(&full[stage], phase);
            sm100::tc_fence_after();
            const uint32_t a0 = sm100::smem_u32(smem + stage * STAGE2_BYTES);
            const uint32_t b0 = a0 + A2_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              sm100::umma_f16_2sm(d_tmem, sm100::umma_desc_sw128(a0 + kk * 32),
                                  sm100::umma_desc_sw128(b0 + kk * 32), idesc, (kb | kk) != 0);
            }
            sm100::umma_commit_2sm(&empty[stage], 0x3);
            if (++stage == STAGES2) { stage = 0; phase ^= 1; }
          }
          sm100::umma_commit_2sm(&tfull[acc], 0x3);
        }
      }
    }
  } else {  // ---------------- epilogue: warps 2..(1 + 4*NH) of both CTAs, thread = query
    // NH = 2: two warps per TMEM lane quarter, each owning 128 of the tile's 256
    // columns as its own split (g*NH + half): half the epilogue work per warp and tile
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    const int tq = quarter * 32 + lane;
    const int k = a.k;
    constexpr int NC2 = BN / 64 / NH;
    const uint32_t tempty_leader0 = sm100::mapa(sm100::smem_u32(&tempty[0]), 0);
    const uint32_t tempty_leader1 = sm100::mapa(sm100::smem_u32(&tempty[1]), 0);
    int i = 0;
    int st = 0;
    WorkSeg sg;
    while (next_seg(a, pair, st, sg)) {
      const int q = sg.qb * 2 * BM + (int)rank * BM + tq;
      const int gs = sg.split * NH + half;
      const size_t base = ((size_t)gs * a.Bp + q);
      QueryScan<KT> qs;
      qs.init(a, q, base, k, gs);
      for (int u = 0; u < sg.count; ++u, ++i) {
        const int t = sg.g + (sg.pos + u) * a.G;
        const int acc = i & 1;
        const uint32_t aph = (i >> 1) & 1;
        sm100::mbar_wait(&tfull[acc], aph);
        sm100::tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * (BN / NH);
        const int cbase = t * BN + half * (BN / NH);
        if (a.warm && u == 0 && (int64_t)(t + 1) * BN <= a.n_rows)
          warm_from_tile<KT>(qs, taddr - half * (BN / NH), k);
#pragma unroll 1
        for (int c2 = 0; c2 < NC2; ++c2) {
          // two TMEM loads in flight per wait
          uint32_t r0[32], r1[32];
          const uint32_t ta = taddr + c2 * 64;
          sm100::tmem_ld32_async(ta, r0);
          sm100::tmem_ld32_async(ta + 32, r1);
          sm100::tmem_wait_ld();
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float v[32];
#pragma unroll
            for (int x = 0; x < 32; ++x) v[x] = __uint_as_float(h ? r1[x] : r0[x]);
            scan_chunk<KT>(qs, v, cbase + (2 * c2 + h) * 32, a.n_rows);
          }
          if (!a.sync_tile || c2 == NC2 - 1) qs.sync(k);
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_cluster(acc ? tempty_leader1 : tempty_leader0);
      }
      qs.finish(a, base, k);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  sm100::cluster_sync();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_2sm<512>(tmem_base);
  }
}

// ------------------------------------------------------------------ exact rescoring
struct DD {
  double hi, lo, ab;
};

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}


// Bound on |exact sum - (hi + lo)| of warp_exact_dot, as a multiple of sum|p| (ab):
// with n = ceil(dim / 32) terms per lane, lo collects the two_sum errors (and, for
// float64 inputs, the fma product residuals), so |lo| <= (n + 6) 2^-53 ab along the way,
// and its n (2n) per-lane and 10 butterfly roundings each err by <= 2^-53 |lo|:
//   fp32:    (n^2 + 10 n + 64) 2^-106 ab      (products exact in float64)
//   float64: (2 n^2 + 12 n + 64) 2^-106 ab    (plus dim * 2^-1074 for underflowing residuals)
// The fp32 factor keeps the older (dim + 64) 2^-104 where that is larger.
__device__ __forceinline__ double dot_err_bound(double ab, int64_t dim, bool f64) {
  const double n = (double)((dim + 31) / 32);
  const double c = f64 ? (2.0 * n * n + 12.0 * n + 64.0) : fmax(n * n + 10.0 * n + 64.0, 4.0 * (double)(dim + 64));
  return ab * c * 0x1p-106 * (1.0 + 0x1p-40) + (f64 ? (double)dim * 0x1p-1074 : 0.0) + 0x1p-1070;
}

// product a*b as p + r: exact for fp32 inputs (r = 0), two_prod (fma residual) for float64
__device__ __forceinline__ double prod_split(float a, float b, double& r) {
  r = 0.0;
  return __dmul_rn((double)a, (double)b);
}
__device__ __forceinline__ double prod_split(double a, double b, double& r) {
  const double p = __dmul_rn(a, b);
  r = __fma_rn(a, b, -p);
  return p;
}

// Warp-cooperative exact dot of two fp32 or two float64 vectors.  Returns the float64
// value and sets `ok` when it is provably the correctly rounded exact sum (fp32*fp32
// products are exact in float64; float64 products are split exactly by fma; the
// double-double accumulation error is bounded by dot_err_bound).
// U elements per lane in flight per step: 24 = one DRAM round trip per 768 dims (latency
// bound small batches), 8 = fewer registers (throughput bound large batches).
template <int U, typename T>
__device__ double warp_exact_dot(const T* __restrict__ a, const T* __restrict__ b, int64_t dim, bool& ok) {
  constexpr bool F64 = sizeof(T) == 8;
  const int lane = threadIdx.x & 31;
  double hi = 0.0, lo = 0.0, ab = 0.0;
  // rows are random DB rows (DRAM latency); out-of-range elements are 0, which leaves
  // hi, lo and ab unchanged
  for (int64_t d0 = lane; d0 < dim; d0 += 32 * U) {
    T av[U], bv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t d = d0 + 32 * u;
      av[u] = d < dim ? __ldg(a + d) : T(0);
      bv[u] = d < dim ? __ldg(b + d) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double r;
      const double p = prod_split(av[u], bv[u], r);
      double s, e;
      two_sum(hi, p, s, e);
      hi = s;
      lo = __dadd_rn(lo, e);
      if (F64) lo = __dadd_rn(lo, r);
      ab = __dadd_rn(ab, fabs(p));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    const double l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const double a2 = __shfl_xor_sync(0xffffffffu, ab, o);
    double s, e;
    two_sum(hi, h2, s, e);
    hi = s;
    lo = __dadd_rn(__dadd_rn(lo, l2), e);
    ab = __dadd_rn(ab, a2);
  }
  double r, t;
  two_sum(hi, lo, r, t);
  // r = RN(hi + lo); exact sum S = r + t + e with |e| <= bound.  RN(S) == r iff S stays
  // strictly inside r's rounding interval: half an ulp above/below, except that just
  // below a power of two the ulp halves.
  const double bound = dot_err_bound(ab, dim, F64);
  const double ar = fabs(r);
  bool exact_sum = (ab == 0.0);
  if (!exact_sum && ar > 0.0 && ar < 0x1p1020) {
    const int e2 = ilogb(ar);
    double half = ldexp(1.0, (e2 < -1022 ? -1022 : e2) - 53);
    const bool pow2 = ar == ldexp(1.0, e2) && e2 > -1022;
    const bool toward_zero = (t != 0.0) && ((t < 0.0) != (r < 0.0));
    if (pow2 && toward_zero) half *= 0.5;
    exact_sum = fabs(t) + bound < half;
  }
  ok = exact_sum;
  return r;
}

// Exact correctly rounded float64 dot product of two fp32 vectors with a 640-bit
// fixed-point accumulator (LSB weight 2^-320; fp32 x fp32 products have integer
// significands < 2^48 at weights >= 2^-298).  Single thread; used only when the
// double-double certificate cannot decide the rounding (exact ties at a float64
// midpoint are common for fp32 inputs).
constexpr int SUPER_L = 10;
constexpr int SUPER_BASE = -320;

// Add the exact product a*b (fp32 x fp32) into a 640-bit two's complement accumulator:
// the product is spread over the ten limbs with static selects and added (or
// subtracted) with one carry chain, so the accumulator stays in registers.
__device__ __forceinline__ void add640(uint64_t (&a)[SUPER_L], const uint64_t (&b)[SUPER_L]) {
  asm("add.cc.u64 %0, %0, %10;\n\t"
      "addc.cc.u64 %1, %1, %11;\n\t"
      "addc.cc.u64 %2, %2, %12;\n\t"
      "addc.cc.u64 %3, %3, %13;\n\t"
      "addc.cc.u64 %4, %4, %14;\n\t"
      "addc.cc.u64 %5, %5, %15;\n\t"
      "addc.cc.u64 %6, %6, %16;\n\t"
      "addc.cc.u64 %7, %7, %17;\n\t"
      "addc.cc.u64 %8, %8, %18;\n\t"
      "addc.u64 %9, %9, %19;"
      : "+l"(a[0]), "+l"(a[1]), "+l"(a[2]), "+l"(a[3]), "+l"(a[4]), "+l"(a[5]), "+l"(a[6]), "+l"(a[7]),
        "+l"(a[8]), "+l"(a[9])
      : "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]), "l"(b[4]), "l"(b[5]), "l"(b[6]), "l"(b[7]), "l"(b[8]),
        "l"(b[9]));
}
__device__ __forceinline__ void sub640(uint64_t (&a)[SUPER_L], const uint64_t (&b)[SUPER_L]) {
  asm("sub.cc.u64 %0, %0, %10;\n\t"
      "subc.cc.u64 %1, %1, %11;\n\t"
      "subc.cc.u64 %2, %2, %12;\n\t"
      "subc.cc.u64 %3, %3, %13;\n\t"
      "subc.cc.u64 %4, %4, %14;\n\t"
      "subc.cc.u64 %5, %5, %15;\n\t"
      "subc.cc.u64 %6, %6, %16;\n\t"
      "subc.cc.u64 %7, %7, %17;\n\t"
      "subc.cc.u64 %8, %8, %18;\n\t"
      "subc.u64 %9, %9, %19;"
      : "+l"(a[0]), "+l"(a[1]), "+l"(a[2]), "+l"(a[3]), "+l"(a[4]), "+l"(a[5]), "+l"(a[6]), "+l"(a[7]),
        "+l"(a[8]), "+l"(a[9])
      : "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]), "l"(b[4]), "l"(b[5]), "l"(b[6]), "l"(b[7]), "l"(b[8]),
        "l"(b[9]));
}
__device__ __forceinline__ void super_add(uint64_t (&acc)[SUPER_L], float fa, float fb) {
  const uint32_t bx = __float_as_uint(fa), by = __float_as_uint(fb);
  uint32_t mx = bx & 0x7fffffu, my = by & 0x7fffffu;
  int ex = (bx >> 23) & 255, ey = (by >> 23) & 255;
  if ((!ex && !mx) || (!ey && !my)) return;  // a zero factor
  if (ex) mx |= 0x800000u; else ex = 1;
  if (ey) my |= 0x800000u; else ey = 1;
  const uint64_t m = (uint64_t)mx * my;                // < 2^48
  const int e = (ex - 150) + (ey - 150) - SUPER_BASE;  // >= 22, li <= 8 for finite inputs
  const int li = e >> 6, sh = e & 63;
  const uint64_t lo = m << sh;
  const uint64_t hi = sh ? (m >> (64 - sh)) : 0;
  uint64_t b[SUPER_L];
#pragma unroll
  for (int j = 0; j < SUPER_L; ++j) b[j] = j == li ? lo : (j == li + 1 ? hi : 0ull);
  if (((bx ^ by) >> 31) == 0) add640(acc, b);
  else sub640(acc, b);
}

// Round a 640-bit two's complement fixed-point value (LSB 2^-320) to float64 (RN-even).
__device__ double super_round(uint64_t (&acc)[SUPER_L]) {
  constexpr int L = SUPER_L;
  const bool neg = (acc[L - 1] >> 63) != 0;
  if (neg) {  // two's complement magnitude
    uint64_t c = 1;
    for (int i = 0; i < L; ++i) {
      acc[i] = ~acc[i] + c;
      c = (c && acc[i] == 0) ? 1 : 0;
    }
  }
  int top = L - 1;
  while (top >= 0 && acc[top] == 0) --top;
  if (top < 0) return 0.0;
  const int msb = top * 64 + (63 - __clzll(acc[top]));
  auto bit = [&](int p) -> uint64_t { return p < 0 ? 0ull : (acc[p >> 6] >> (p & 63)) & 1ull; };
  // the 53 bits [msb-52, msb] span at most two limbs
  uint64_t mant;
  const int w = msb - 52;
  if (w < 0) {
    mant = acc[0] << (-w);
  } else {
    const int li = w >> 6, sh = w & 63;
    mant = acc[li] >> sh;
    if (sh && li + 1 < L) mant |= acc[li + 1] << (64 - sh);
  }
  mant &= (1ull << 53) - 1;
  const uint64_t guard = bit(msb - 53);
  bool sticky = false;
  const int sp = msb - 54;  // bits [0, sp] are sticky
  if (sp >= 0) {
    for (int i = 0; i < (sp >> 6); ++i) sticky |= acc[i] != 0;
    const int r = sp & 63;
    const uint64_t maskp = (r == 63) ? ~0ull : ((1ull << (r + 1)) - 1);
    sticky |= (acc[sp >> 6] & maskp) != 0;
  }
  int exp2 = msb - 52 + SUPER_BASE;
  if (guard && (sticky || (mant & 1))) {
    ++mant;
    if (mant == (1ull << 53)) { mant >>= 1; ++exp2; }
  }
  const double v = ldexp((double)mant, exp2);
  return neg ? -v : v;
}

// Warp-cooperative: each lane accumulates dim/32 products, the 640-bit partial sums are
// added across lanes (mod 2^640, carries propagated limb by limb), every lane rounds.
// Called by all 32 lanes (warp-uniform branch).
__device__ __noinline__ double warp_exact_dot_super(const float* __restrict__ a, const float* __restrict__ b,
                                                    int64_t dim) {
  const int lane = threadIdx.x & 31;
  uint64_t acc[SUPER_L];
#pragma unroll
  for (int i = 0; i < SUPER_L; ++i) acc[i] = 0;
  for (int64_t d0 = lane; d0 < dim; d0 += 256) {
    float av[8], bv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t d = d0 + 32 * u;
      av[u] = d < dim ? __ldg(a + d) : 0.f;
      bv[u] = d < dim ? __ldg(b + d) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) super_add(acc, av[u], bv[u]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    uint64_t other[SUPER_L];
#pragma unroll
    for (int i = 0; i < SUPER_L; ++i) other[i] = __shfl_xor_sync(0xffffffffu, acc[i], o);
    add640(acc, other);
  }
  return super_round(acc);
}

// Exact correctly rounded dot product of two float64 vectors (the rare fallback when
// the double-double certificate fails): every product m_a m_b 2^(e_a + e_b) (106-bit
// integer significand) is added into a 4480-bit two's complement fixed-point
// accumulator with LSB 2^-2240, which holds any sum of products of finite doubles
// (exponents of products >= -2148, magnitudes < 2^2048 * dim).  Lane 0 of the warp
// computes it (local memory); the result is broadcast.
constexpr int BIG_L = 70;
constexpr int BIG_BASE = -2240;

__device__ __forceinline__ void big_add_at(uint64_t* acc, int li, uint64_t w0, uint64_t w1, uint64_t w2, bool neg) {
  // acc += (w2:w1:w0) << (64 li), or -= when neg (two's complement; carries ripple up)
  const uint64_t w[3] = {w0, w1, w2};
  if (!neg) {
    uint64_t c = 0;
    for (int j = 0; j < 3; ++j) {
      const uint64_t x = acc[li + j];
      const uint64_t y = x + w[j];
      const uint64_t c1 = y < x;
      const uint64_t z = y + c;
      c = c1 | (z < y);
      acc[li + j] = z;
    }
    for (int i = li + 3; c && i < BIG_L; ++i) c = (++acc[i] == 0);
  } else {
    uint64_t bw = 0;
    for (int j = 0; j < 3; ++j) {
      const uint64_t x = acc[li + j];
      const uint64_t y = x - w[j];
      const uint64_t b1 = x < w[j];
      const uint64_t z = y - bw;
      bw = b1 | (y < bw);
      acc[li + j] = z;
    }
    for (int i = li + 3; bw && i < BIG_L; ++i) bw = (acc[i]-- == 0);
  }
}

__device__ __forceinline__ void dbl_parts(double v, uint64_t& m, int& e) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  const int ex = (int)((b >> 52) & 2047);
  m = b & ((1ull << 52) - 1);
  if (ex) { m |= 1ull << 52; e = ex - 1075; } else { e = -1074; }
}

// Round an L-limb two's complement fixed-point value (LSB 2^base) to float64, RN-even,
// with gradual underflow and overflow to inf.
template <int L>
__device__ double fixed_round(uint64_t* acc, int base) {
  const bool neg = (acc[L - 1] >> 63) != 0;
  if (neg) {
    uint64_t c = 1;
    for (int i = 0; i < L; ++i) {
      acc[i] = ~acc[i] + c;
      c = (c && acc[i] == 0) ? 1 : 0;
    }
  }
  int top = L - 1;
  while (top >= 0 && acc[top] == 0) --top;
  if (top < 0) return 0.0;
  const int msb = top * 64 + (63 - __clzll(acc[top]));
  // lowest kept bit: 53 significant bits, but not below 2^-1074
  int w = msb - 52;
  if (w + base < -1074) w = -1074 - base;
  auto bit = [&](int p) -> uint64_t { return p < 0 ? 0ull : (acc[p >> 6] >> (p & 63)) & 1ull; };
  uint64_t mant;
  if (w < 0) {
    mant = acc[0] << (-w);
  } else {
    const int li = w >> 6, sh = w & 63;
    mant = acc[li] >> sh;
    if (sh && li + 1 < L) mant |= acc[li + 1] << (64 - sh);
  }
  const int nbits = msb - w + 1;  // <= 53
  mant = nbits <= 0 ? 0ull : (mant & ((1ull << nbits) - 1));
  const uint64_t guard = bit(w - 1);
  bool sticky = false;
  const int sp = w - 2;  // bits [0, sp] are sticky
  if (sp >= 0) {
    for (int i = 0; i < (sp >> 6); ++i) sticky |= acc[i] != 0;
    const int r = sp & 63;
    const uint64_t maskp = (r == 63) ? ~0ull : ((1ull << (r + 1)) - 1);
    sticky |= (acc[sp >> 6] & maskp) != 0;
  }
  if (guard && (sticky || (mant & 1))) ++mant;  // a carry to 2^53 stays exact in ldexp
  const double v = ldexp((double)mant, w + base);
  return neg ? -v : v;
}

__device__ __noinline__ double exact_dot_f64_big(const double* __restrict__ a, const double* __restrict__ b,
                                                 int64_t dim) {
  uint64_t acc[BIG_L];
  for (int i = 0; i < BIG_L; ++i) acc[i] = 0;
  for (int64_t d = 0; d < dim; ++d) {
    const double x = a[d], y = b[d];
    if (x == 0.0 || y == 0.0) continue;
    uint64_t mx, my;
    int ex, ey;
    dbl_parts(x, mx, ex);
    dbl_parts(y, my, ey);
    const uint64_t lo = mx * my, hi = __umul64hi(mx, my);  // < 2^106
    const int pos = ex + ey - BIG_BASE;                     // >= 92
    const int li = pos >> 6, sh = pos & 63;
    const uint64_t w0 = lo << sh;
    const uint64_t w1 = sh ? ((lo >> (64 - sh)) | (hi << sh)) : hi;
    const uint64_t w2 = sh ? (hi >> (64 - sh)) : 0ull;
    big_add_at(acc, li, w0, w1, w2, (x < 0) != (y < 0));
  }
  return fixed_round<BIG_L>(acc, BIG_BASE);
}

// Warp-uniform fallback dispatch: fp32 rows use the warp-parallel 640-bit accumulator,
// float64 rows the lane-0 4480-bit one.
__device__ __forceinline__ double warp_exact_dot_fallback(const float* a, const float* b, int64_t dim) {
  return warp_exact_dot_super(a, b, dim);
}
__device__ __forceinline__ double warp_exact_dot_fallback(const double* a, const double* b, int64_t dim) {
  double v = 0.0;
  if ((threadIdx.x & 31) == 0) v = exact_dot_f64_big(a, b, dim);
  return __shfl_sync(0xffffffffu, v, 0);
}

// ------------------------------------------------------------------ reference BLAS order
// Optional "blas" similarity order: the float64 sims are computed with the exact
// operation sequence of the BLAS call behind the reference's scan (predictor.py:158,
// numpy -> OpenBLAS 0.3.30 dgemv_t on x86-64; restated and pinned against numpy in
// oracle/blas_order.c), so ties that are exact in real arithmetic (common for the
// reference's hashed prompt embeddings) break exactly as in the reference.  Row r of
// the reference's array is ring slot seq % ref_cap of a store holding ref_n rows.
struct BlasRef {
  int on;          // 0: correctly rounded sims (default); 1: reference BLAS order
  int threads;     // OpenBLAS threads of the reference host (used when ref_n * dim >= 460800)
  int64_t ref_cap; // capacity of the reference (global) ring
  int64_t ref_n;   // rows of the reference array (global store size)
};

__device__ __forceinline__ int blas_kind(int64_t r, int64_t n, int64_t d, int threads) {
  const int T = (n * d < 460800) ? 1 : (threads < 1 ? 1 : threads);
  int64_t start = 0, left = n;
  for (int t = 0; left > 0; ++t) {
    int64_t w = (left + (T - t) - 1) / (T - t > 0 ? T - t : 1);
    if (w < 4) w = 4;
    if (left < w) w = left;
    if (r < start + w) {
      const int64_t j = r - start, w4 = w & ~(int64_t)3;
      return j < w4 ? 0 : (((w & 2) && j < w4 + 2) ? 1 : 2);
    }
    start += w;
    left -= w;
  }
  return 2;
}

// One thread: row . x in the order of OpenBLAS kernel `kind` (0: 4x4, FMA accumulators;
// 1: 4x2; 2: 4x1), 2048-element blocks, then the d & 3 tail (oracle_blas_dot).
template <typename T>
__device__ double blas_dot(const T* __restrict__ a, const T* __restrict__ x, int64_t d, int kind) {
  const int64_t m3 = d & 3, m1 = d - m3;
  double y = 0.0;
  for (int64_t b = 0; b < m1; b += 2048) {
    const int64_t h = b + 2048 < m1 ? b + 2048 : m1;
    double bs;
    if (kind == 0) {
      double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
      for (int64_t i = b; i < h; i += 4) {
        c0 = __fma_rn((double)a[i], (double)x[i], c0);
        c1 = __fma_rn((double)a[i + 1], (double)x[i + 1], c1);
        c2 = __fma_rn((double)a[i + 2], (double)x[i + 2], c2);
        c3 = __fma_rn((double)a[i + 3], (double)x[i + 3], c3);
      }
      bs = __dadd_rn(__dadd_rn(c0, c2), __dadd_rn(c1, c3));
    } else if (kind == 1) {
      double c0 = 0, c1 = 0;
      for (int64_t i = b; i < h; i += 2) {
        c0 = __dadd_rn(c0, __dmul_rn((double)a[i], (double)x[i]));
        c1 = __dadd_rn(c1, __dmul_rn((double)a[i + 1], (double)x[i + 1]));
      }
      bs = __dadd_rn(c0, c1);
    } else {
      double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
      for (int64_t i = b; i < h; i += 4) {
        c0 = __dadd_rn(c0, __dmul_rn((double)a[i], (double)x[i]));
        c1 = __dadd_rn(c1, __dmul_rn((double)a[i + 1], (double)x[i + 1]));
        c2 = __dadd_rn(c2, __dmul_rn((double)a[i + 2], (double)x[i + 2]));
        c3 = __dadd_rn(c3, __dmul_rn((double)a[i + 3], (double)x[i + 3]));
      }
      bs = __dadd_rn(__dadd_rn(c0, c2), __dadd_rn(c1, c3));
    }
    y = __dadd_rn(y, bs);
  }
  const T* t = a + m1;
  const T* u = x + m1;
  if (m3 == 1) {
    y = __fma_rn((double)t[0], (double)u[0], y);
  } else if (m3 == 2) {
    y = __dadd_rn(y, __fma_rn((double)t[0], (double)u[0], __dmul_rn((double)t[1], (double)u[1])));
  } else if (m3 == 3) {
    y = __dadd_rn(y, __fma_rn((double)t[2], (double)u[2],
                               __fma_rn((double)t[0], (double)u[0], __dmul_rn((double)t[1], (double)u[1]))));
  }
  return y;
}

// Per-query lower bound of the global EXACT k-th score left by a shard's scan: the scan
// leaves L (shared k-th, rank slots) such that k rows of this shard have coarse score >=
// L, hence exact score >= L - delta_self, so the global exact k-th is >= L - delta_self.
// -inf when none (an empty shard: gkth == nullptr; or a query on the exhaustive path).
// After an all-reduce (max) E over the shards, a row of shard t can enter the global
// top-k only if its coarse score is >= E - delta_t (k_rescore), whatever the other
// shards' row norms are.
__global__ void k_bounds(int64_t B, int k, const uint32_t* __restrict__ gkth, const uint32_t* __restrict__ gslot,
                         const float* __restrict__ two_delta, float* __restrict__ out) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= B) return;
  const float NEG = -__int_as_float(0x7f800000);
  float L = NEG;
  if (gkth) {
    const uint32_t g0 = gkth[q];
    if (g0) L = ord_val(g0);
    uint32_t mn = 0xffffffffu;
    for (int x = 0; x < k; ++x) mn = min(mn, gslot[(size_t)q * KMAX + x]);
    if (mn) L = fmaxf(L, ord_val(mn));
    const float td = two_delta[q];
    L = (td <= 3.0e38f && L > NEG) ? __fsub_rd(L, 0.5f * td) : NEG;
  }
  out[q] = L;
}

__device__ __forceinline__ int nw_last(unsigned bd) { return (int)(bd >> 5) - 1; }

// Per query: global coarse k-th from the splits' top lists, candidate compaction,
// exact rescoring, (-sim, seq) order.  Block = 256 threads.
template <typename T>
__device__ __noinline__ void exhaustive_query(int64_t q, int k, int64_t n_rows, int64_t dim, const T* __restrict__ qx,
                                              const T* __restrict__ vm, const int32_t* __restrict__ lens,
                                              const int64_t* __restrict__ seqs, int32_t* __restrict__ need,
                                              double* __restrict__ out_sim, int64_t* __restrict__ out_seq,
                                              int32_t* __restrict__ out_len, int32_t* __restrict__ out_count,
                                              unsigned int* __restrict__ inexact_count, const BlasRef blas);

// Block = 256 threads (small batches, U = 24) or 128 (large batches, U < 24, at most 64
// registers so 8 blocks share an SM: the kernel is latency bound).  s_top is dynamic
// shared memory, top_cap floats = min(4096, the scan's largest splits x k).
template <int U, typename T>
__global__ void __launch_bounds__(U < 24 ? 128 : 256, U < 24 ? 8 : 1)
k_rescore(int qblk, int smul, const ScanArgs wa, int Bp, int64_t B, int k, int64_t n_rows, int64_t dim, const T* __restrict__ qx,
          const T* __restrict__ vm, const int32_t* __restrict__ lens, const int64_t* __restrict__ seqs,
          const float* __restrict__ two_delta, const float* __restrict__ cand_s, const int32_t* __restrict__ cand_r,
          const int32_t* __restrict__ cand_n, const float* __restrict__ topc, const float* __restrict__ ext,
          double* __restrict__ out_sim, int64_t* __restrict__ out_seq, int32_t* __restrict__ out_len,
          int32_t* __restrict__ out_count, int32_t* __restrict__ need_exhaustive,
          unsigned int* __restrict__ inexact_count, const BlasRef blas, int top_cap) {
  const int64_t q = blockIdx.x;
  if (q >= B) return;
  extern __shared__ float s_top[];  // list values >= the bound (more than top_cap: exhaustive path)
  __shared__ int s_off[513];     // n_splits <= 512 (host)
  __shared__ int s_rows[MAXC];
  __shared__ double s_sim[MAXC];
  __shared__ int64_t s_seq[MAXC];
  __shared__ float s_wk[8 * KMAX];
  __shared__ float s_kth;
  __shared__ int s_n;
  __shared__ int s_flag;
  __shared__ int s_nt;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n_splits = smul * splits_of_block(wa, (int)(q / qblk));
  const int64_t kk = k < n_rows ? k : n_rows;
  const float NEG = -__int_as_float(0x7f800000);
  // queries the candidate filter cannot serve (block-uniform conditions): small batches
  // score them exhaustively in this block (no k_exhaustive launch); large batches flag
  // them for k_exhaustive
  auto exhaustive = [&]() {
    if constexpr (U == 24) {
      exhaustive_query<T>(q, k, n_rows, dim, qx, vm, lens, seqs, need_exhaustive, out_sim, out_seq, out_len,
                          out_count, inexact_count, blas);
    } else {
      if (tid == 0) need_exhaustive[q] = 1;
    }
  };
  if (!(two_delta[q] <= 3.0e38f)) {  // outside the fp16 range: no coarse bound holds
    exhaustive();
    return;
  }
#ifdef ALISE_RESCORE_TIMING
  const long long T0 = clock64();
#endif
  // 1) stage the splits' top lists and candidate counts (all loads in flight at once).
  //    The scan leaves a lower bound L of the final coarse k-th (shared k-th, rank
  //    slots) such that the union of the lists holds k values >= L, so only list values
  //    >= L can decide the k-th: they are compacted (usually about k of the n_splits*k)
  const int m = n_splits * k;
  // per-query scalars the later phases need, loaded now so they arrive with the lists
  const float td = two_delta[q];
  const float ext_q = ext ? ext[q] : NEG;
  // With an all-reduced bound from the shards (ext, an exact-score lower bound of the
  // global k-th), rows below ext - delta cannot enter the global top-k and the shard's
  // own coarse k-th is not needed (ext is at least this shard's own bound): the list
  // staging and selection are skipped.
  const bool use_ext = ext_q > NEG;
  float L = NEG;
  if (!use_ext) {
    const uint32_t g0 = wa.gkth[q];
    if (g0) L = ord_val(g0);
    uint32_t mn = 0xffffffffu;
    for (int x = 0; x < k; ++x) mn = min(mn, wa.gslot[(size_t)q * KMAX + x]);
    if (mn) L = fmaxf(L, ord_val(mn));
  }
  if (tid == 0) { s_n = 0; s_flag = 0; s_nt = 0; }
  __syncthreads();
  for (int i0 = tid; i0 < (use_ext ? 0 : m); i0 += 8 * blockDim.x) {
    float tv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // 8 loads in flight per thread
      const int i = i0 + u * (int)blockDim.x;
      const int sp = i / k, j = i - sp * k;
      tv[u] = i < m ? __ldg(topc + ((size_t)sp * Bp + q) * KMAX + j) : NEG;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u * (int)blockDim.x < m && tv[u] >= L) {
        const int at = atomicAdd(&s_nt, 1);
        if (at < top_cap) s_top[at] = tv[u];
      }
  }
  for (int sp = tid; sp < n_splits; sp += blockDim.x) {
    const int cnt = cand_n[(size_t)sp * Bp + q];
    s_off[sp + 1] = cnt < 0 ? 0 : cnt;
    if (cnt < 0) s_flag = 1;
  }
  __syncthreads();
  if (s_nt > top_cap) {  // thousands of list values tie at the bound: exhaustive path
    exhaustive();
    return;
  }
  // 2) kk-th largest coarse score over the lists: each warp takes the kk largest of its
  //    slice (kk rounds of warp argmax, the winner's slot cleared), warp 0 repeats that
  //    over the warps' results; warp 7 meanwhile scans the counts into offsets
  const int mt = s_nt;             // compacted list values
  const bool one_warp = mt <= 256;  // few values: warp 0 selects directly
  if (!one_warp) {
    const int nw = blockDim.x >> 5;
    const int per = (mt + nw - 1) / nw;
    const int lo = warp * per, hi = min(mt, lo + per);
    for (int round = 0; round < (int)kk; ++round) {
      float bv = NEG;
      int bi = -1;
      for (int i = lo + lane; i < hi; i += 32) {
        const float v = s_top[i];
        if (v > bv) { bv = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        if (v2 > bv || (v2 == bv && i2 > bi)) { bv = v2; bi = i2; }
      }
      __syncwarp();  // every lane's reads of this round precede the clear (racecheck)
      if (lane == 0) {
        s_wk[warp * (int)kk + round] = bv;
        if (bi >= 0) s_top[bi] = NEG;
      }
      __syncwarp();
    }
  }
  if (warp == nw_last(blockDim.x)) {
    int carry = 0;
    for (int base = 1; base <= n_splits; base += 32) {
      const int i = base + lane;
      int v = i <= n_splits ? s_off[i] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
      }
      if (i <= n_splits) s_off[i] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
    if (lane == 0) s_off[0] = 0;
  }
  __syncthreads();
  if (warp == 0 && mt <= 32) {
    // up to 32 values (the common case: about k of them reach the bound): one bitonic
    // sort across the lanes (15 shuffle stages instead of kk argmax rounds)
    float v = lane < mt ? s_top[lane] : NEG;
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        const float o = __shfl_xor_sync(0xffffffffu, v, stride);
        const bool desc = (lane & size) == 0 || size == 32;  // this run sorts descending
        const bool low = (lane & stride) == 0;
        v = (low == desc) ? fmaxf(v, o) : fminf(v, o);
      }
    }
    const float kth = __shfl_sync(0xffffffffu, v, (int)kk - 1);
    if (lane == 0) s_kth = kth;
  } else if (warp == 0) {
    float* src = one_warp ? s_top : s_wk;
    const int mw = one_warp ? mt : (int)(blockDim.x >> 5) * (int)kk;
    float kth = NEG;
    for (int round = 0; round < (int)kk; ++round) {
      float bv = NEG;
      int bi = -1;
      for (int i = lane; i < mw; i += 32) {
        const float v = src[i];
        if (v > bv) { bv = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
        if (v2 > bv || (v2 == bv && i2 > bi)) { bv = v2; bi = i2; }
      }
      __syncwarp();  // every lane's reads of this round precede the clear (racecheck)
      if (lane == 0 && bi >= 0) src[bi] = NEG;
      __syncwarp();
      kth = bv;
    }
    if (lane == 0) s_kth = kth;
  }
  __syncthreads();
#ifdef ALISE_RESCORE_TIMING
  const long long T1 = clock64();
#endif
  // (a bound from other shards can only raise the threshold: ext is an exact-score
  // lower bound of the global k-th, so rows with coarse score below ext - delta cannot
  // enter the global top-k)
  const float thr = fmaxf(__fsub_rd(s_kth, td), ext ? __fsub_rd(ext_q, 0.5f * td) : NEG);
  // 3) gather candidates above the final threshold: the (split, slot) entries are
  //    flattened over the whole block through the prefix sum of the counts, so every
  //    candidate load is in flight at once (candidate order is irrelevant: step 5 ranks)
  const int total = s_off[n_splits];
  for (int i0 = tid; i0 < total; i0 += 8 * blockDim.x) {
    int rv[8];
    float sv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {  // 8 candidate (score, row) loads in flight per thread;
      const int i = i0 + u * (int)blockDim.x;  // the row is loaded with the score, not after the test
      sv[u] = __int_as_float(0x7fffffff);  // NaN: past the end never passes, even thr = -inf
      rv[u] = 0;
      if (i < total) {
        int lo = 0, hi = n_splits;  // largest sp with s_off[sp] <= i
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_off[mid] <= i) lo = mid; else hi = mid;
        }
        const size_t ev = ((size_t)lo * Bp + q) * CAP + (i - s_off[lo]);
        sv[u] = __ldg(cand_s + ev);
        rv[u] = __ldg(cand_r + ev);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (sv[u] >= thr) {
        const int slot = atomicAdd(&s_n, 1);
        if (slot < MAXC) {
          s_rows[slot] = rv[u];
          // start the candidate row's DRAM fetch now (random DB row; the dots read it
          // after the block barrier)
          const char* rp = reinterpret_cast<const char*>(vm + (size_t)rv[u] * dim);
          for (int64_t off = 0; off < dim * (int64_t)sizeof(T); off += 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + off));
        }
      }
    }
  }
  __syncthreads();
#ifdef ALISE_RESCORE_TIMING
  const long long T2 = clock64();
#endif
  const int n = s_n;
  if (n > MAXC || s_flag) {
    exhaustive();
    return;
  }
  if (blas.on) {
    // 4') reference BLAS-order float64 scores, one thread per candidate
    for (int c = tid; c < n; c += blockDim.x) {
      const int row = s_rows[c];
      const int64_t sq = seqs[row];
      const int kind = blas_kind(sq % blas.ref_cap, blas.ref_n, dim, blas.threads);
      s_sim[c] = blas_dot<T>(vm + (size_t)row * dim, qx + q * dim, dim, kind);
      s_seq[c] = sq;
    }
    __syncthreads();
  } else {
    // 4) exact float64 scores, one warp per candidate.  The warp first prefetches all of
    //    its candidate rows into L2 (random DB rows: one DRAM round trip for all of them
    //    instead of one per candidate)
    for (int c = warp; c < n; c += blockDim.x >> 5) {
      const char* rp = reinterpret_cast<const char*>(vm + (size_t)s_rows[c] * dim);
      for (int64_t off = (int64_t)lane * 128; off < dim * (int64_t)sizeof(T); off += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(rp + off));
    }
    for (int c = warp; c < n; c += blockDim.x >> 5) {
      const int row = s_rows[c];
      bool ok;
      double sim = warp_exact_dot<U, T>(vm + (size_t)row * dim, qx + q * dim, dim, ok);
      if (!ok) {  // warp-uniform: the certificate is computed from butterfly-reduced sums
        sim = warp_exact_dot_fallback(vm + (size_t)row * dim, qx + q * dim, dim);
        if (lane == 0) atomicAdd(inexact_count, 1u);
      }
      if (lane == 0) {
        s_sim[c] = sim;
        s_seq[c] = seqs[row];
      }
    }
    __syncthreads();
  }
#ifdef ALISE_RESCORE_TIMING
  const long long T3 = clock64();
#endif
  // 5) rank by (-sim, seq); seqs are unique
  for (int c = tid; c < n; c += blockDim.x) {
    const double sv = s_sim[c];
    const int64_t qv = s_seq[c];
    int rank = 0;
    for (int j = 0; j < n; ++j) rank += (s_sim[j] > sv) || (s_sim[j] == sv && s_seq[j] < qv);
    if (rank < k) {
      out_sim[q * k + rank] = sv;
      out_seq[q * k + rank] = qv;
      out_len[q * k + rank] = lens[s_rows[c]];
    }
  }
  if (tid == 0) out_count[q] = (int32_t)(n < kk ? n : kk);
#ifdef ALISE_RESCORE_DEBUG
  __syncthreads();
  if (tid == 0) {
    printf("[rescore q=%lld] n=%d kk=%lld s_kth=%.9g thr=%.9g total=%d splits=%d\n", (long long)q, n, (long long)kk,
           s_kth, thr, total, n_splits);
    for (int c = 0; c < n && c < 12; ++c) printf("  cand row=%d seq=%lld sim=%.17g\n", s_rows[c], (long long)s_seq[c], s_sim[c]);
    for (int sp = 0; sp < n_splits; ++sp) {
      const int cn = cand_n[(size_t)sp * Bp + q];
      printf("  split %d cand_n=%d off=%d:", sp, cn, s_off[sp]);
      for (int u = 0; u < cn && u < 40; ++u) printf(" %d", cand_r[((size_t)sp * Bp + q) * CAP + u]);
      printf("\n");
    }
  }
#endif
#ifdef ALISE_RESCORE_TIMING
  if (tid == 0 && (q < 4 || T3 - T2 > 40000))
    printf("[rescore q=%lld] splits=%d total=%d n=%d cycles: select+counts %lld gather %lld dots %lld rank %lld\n",
           (long long)q, n_splits, total, n, T1 - T0, T2 - T1, T3 - T2, clock64() - T3);
#endif
}

// Exhaustive exact top-k for queries flagged by k_rescore (candidate overflow from
// heavy ties).  One block per 256 queries reads their flags at once (flagged queries
// are rare; one block per query cost ~9 us of empty blocks at B = 4096).  Slow but exact.
template <typename T>
__device__ __noinline__ void exhaustive_query(int64_t q, int k, int64_t n_rows, int64_t dim, const T* __restrict__ qx,
                                              const T* __restrict__ vm, const int32_t* __restrict__ lens,
                                              const int64_t* __restrict__ seqs, int32_t* __restrict__ need,
                                              double* __restrict__ out_sim, int64_t* __restrict__ out_seq,
                                              int32_t* __restrict__ out_len, int32_t* __restrict__ out_count,
                                              unsigned int* __restrict__ inexact_count, const BlasRef blas) {
  __shared__ double s_sim[8 * KMAX];
  __shared__ int64_t s_seq[8 * KMAX];
  __shared__ int s_row[8 * KMAX];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // each warp keeps its own sorted top-k list (lane 0 owns it)
  double tsim[KMAX];
  int64_t tseq[KMAX];
  int trow[KMAX];
  for (int i = 0; i < KMAX; ++i) { tsim[i] = -__longlong_as_double(0x7ff0000000000000ll); tseq[i] = INT64_MAX; trow[i] = -1; }
  const int64_t nw = blockDim.x >> 5;
  const int64_t row_end = blas.on ? (n_rows + 32 * nw - 1) / (32 * nw) * (32 * nw) : n_rows;
  for (int64_t row0 = blas.on ? warp * 32 : warp; row0 < row_end; row0 += blas.on ? 32 * nw : nw) {
    // blas order: each lane scores one row of the warp's 32 (reference BLAS order), lane
    // 0 then inserts them in row order; exact order: the warp scores one row together
    double bsim = 0.0;
    if (blas.on && row0 + lane < n_rows) {
      const int64_t r = row0 + lane;
      bsim = blas_dot<T>(vm + r * dim, qx + q * dim, dim, blas_kind(seqs[r] % blas.ref_cap, blas.ref_n, dim, blas.threads));
    }
    const int n_here = blas.on ? (int)min((int64_t)32, n_rows - row0) : 1;
    for (int u = 0; u < n_here; ++u) {
    const int64_t row = blas.on ? row0 + u : row0;
    double sim;
    if (blas.on) {
      sim = __shfl_sync(0xffffffffu, bsim, u);
    } else {
      bool ok;
      sim = warp_exact_dot<8, T>(vm + row * dim, qx + q * dim, dim, ok);
      if (!ok) {
        sim = warp_exact_dot_fallback(vm + row * dim, qx + q * dim, dim);
        if (lane == 0) atomicAdd(inexact_count, 1u);
      }
    }
    if (lane == 0) {
      double cs = sim;
      int64_t cq = seqs[row];
      int cr = (int)row;
      for (int i = 0; i < k; ++i) {
        if (cs > tsim[i] || (cs == tsim[i] && cq < tseq[i])) {
          double a = tsim[i]; int64_t b = tseq[i]; int c = trow[i];
          tsim[i] = cs; tseq[i] = cq; trow[i] = cr;
          cs = a; cq = b; cr = c;
        }
      }
    }
    }
  }
  if (lane == 0)
    for (int i = 0; i < k; ++i) { s_sim[warp * KMAX + i] = tsim[i]; s_seq[warp * KMAX + i] = tseq[i]; s_row[warp * KMAX + i] = trow[i]; }
  __syncthreads();
  const int m = (blockDim.x >> 5) * KMAX;
  for (int c = threadIdx.x; c < m; c += blockDim.x) {
    if ((c % KMAX) >= k || s_row[c] < 0) continue;
    int rank = 0;
    for (int j = 0; j < m; ++j) {
      if ((j % KMAX) >= k || s_row[j] < 0) continue;
      rank += (s_sim[j] > s_sim[c]) || (s_sim[j] == s_sim[c] && s_seq[j] < s_seq[c]);
    }
    if (rank < k) { out_sim[q * k + rank] = s_sim[c]; out_seq[q * k + rank] = s_seq[c]; out_len[q * k + rank] = lens[s_row[c]]; }
  }
  if (threadIdx.x == 0) { out_count[q] = (int32_t)(n_rows < k ? n_rows : k); need[q] = 0; }
  __syncthreads();  // the block's shared lists are reused by its next flagged query
}

template <typename T>
__global__ void __launch_bounds__(256)
k_exhaustive(int64_t B, int k, int64_t n_rows, int64_t dim, const T* __restrict__ qx,
             const T* __restrict__ vm, const int32_t* __restrict__ lens, const int64_t* __restrict__ seqs,
             int32_t* __restrict__ need, double* __restrict__ out_sim, int64_t* __restrict__ out_seq,
             int32_t* __restrict__ out_len, int32_t* __restrict__ out_count, unsigned int* __restrict__ inexact_count,
             const BlasRef blas) {
  // each block owns blockDim.x consecutive queries: one parallel read of their flags
  __shared__ int s_need[256];
  const int64_t q0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t myq = q0 + threadIdx.x;
  s_need[threadIdx.x] = myq < B ? need[myq] : 0;
  const int any = __syncthreads_or(s_need[threadIdx.x]);
  if (!any) return;
  for (int i = 0; i < (int)blockDim.x && q0 + i < B; ++i)
    if (s_need[i]) exhaustive_query(q0 + i, k, n_rows, dim, qx, vm, lens, seqs, need, out_sim, out_seq, out_len,
                                    out_count, inexact_count, blas);
}

// ------------------------------------------------------------------ large k (> KMAX)
// top_k above the scan's register lists (KMAX) takes a CUDA-core path with the same
// coarse operands and bound: stage 1 (k_bigk_scan, block = (row split, query)) forms
// s~ = fp16(q).fp16(v) with one mixed-precision FMA per element (exact fp16 products,
// fp32 sums: |s~ - s| <= delta_q, k_query_prep's bound, holds for any summation order)
// and keeps, in a shared-memory buffer, every row with s~ >= (the block's running k-th
// s~) - 2 delta (a bitonic sort compacts the buffer when it fills); stage 2
// (k_bigk_select, block per query) takes the largest of the splits' k-th values as the
// filter (each is <= the global coarse k-th), gathers the surviving rows, narrows to
// the global coarse k-th, rescores them exactly (the same certified dots / reference
// BLAS order as k_rescore) and sorts by (-sim, seq).  Heavier than the tcgen05 path
// (every row's coarse dot on CUDA cores) but exact for any k <= BIGK_MAX.
constexpr int BIGK_MAX = 1024;
constexpr int BIGK_BUF = 4096;  // candidates per block (power of two, >= 2 x BIGK_MAX + one round)

// descending bitonic sort of n2 (power of two) keyed entries in shared memory
template <typename K, typename V, typename Less>
__device__ void bitonic_desc(K* key, V* val, int n2, Less less) {
  for (int size = 2; size <= n2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = (lo & size) == 0;  // this run sorts descending when up
        const bool swap = up ? less(key[lo], val[lo], key[hi], val[hi]) : less(key[hi], val[hi], key[lo], val[lo]);
        if (swap) {
          const K tk = key[lo];
          key[lo] = key[hi];
          key[hi] = tk;
          const V tv = val[lo];
          val[lo] = val[hi];
          val[hi] = tv;
        }
      }
      __syncthreads();
    }
  }
}

struct CoarseLess {  // a before b when a's score is larger (ties: smaller row)
  __device__ bool operator()(float ka, int va, float kb, int vb) const { return ka < kb || (ka == kb && va > vb); }
};

__global__ void __launch_bounds__(256)
k_bigk_scan(int64_t n_rows, int64_t dp, int k, int splits, const __half* __restrict__ v16,
            const __half* __restrict__ q16, const float* __restrict__ two_delta, float* __restrict__ out_s,
            int32_t* __restrict__ out_r, int32_t* __restrict__ out_n, float* __restrict__ out_kth) {
  extern __shared__ uint8_t smem_bk[];
  float* s_key = reinterpret_cast<float*>(smem_bk);
  int* s_row = reinterpret_cast<int*>(s_key + BIGK_BUF);
  __shared__ int s_cnt;
  __shared__ float s_tau, s_kth;
  const int split = blockIdx.x;
  const int64_t q = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 3, sub = lane & 7;  // 4 rows per warp step, 8 lanes per row
  const float NEG = -__int_as_float(0x7f800000);
  const float td = two_delta[q];
  const int64_t per = (n_rows + splits - 1) / splits;
  const int64_t lo = split * per, hi = min(n_rows, lo + per);
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_tau = NEG;
    s_kth = NEG;
  }
  __syncthreads();
  const uint4* qv = reinterpret_cast<const uint4*>(q16 + q * dp);
  const int nv = (int)(dp / 8);  // 16-byte vectors per row
  // compaction: sort, k-th coarse, keep the entries >= k-th - 2 delta
  auto compact = [&]() {
    const int n = s_cnt;
    int n2 = 2;
    while (n2 < n) n2 <<= 1;
    for (int i = n + threadIdx.x; i < n2; i += blockDim.x) {
      s_key[i] = NEG;
      s_row[i] = INT32_MAX;
    }
    __syncthreads();
    bitonic_desc(s_key, s_row, n2, CoarseLess());
    if (threadIdx.x == 0) {
      if (n >= k) {
        s_kth = s_key[k - 1];
        s_tau = fmaxf(s_tau, __fsub_rd(s_kth, td));
      }
      int a = 0, b = n;  // sorted descending: first index below tau
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (s_key[mid] >= s_tau) a = mid + 1; else b = mid;
      }
      s_cnt = a;
    }
    __syncthreads();
  };
  constexpr int ROUND = 8 * 4 * 32;  // rows per round: 8 warps x 4 rows x 32 steps
  for (int64_t r0 = lo; r0 < hi; r0 += ROUND) {
    const float tau = s_tau;
    for (int st = 0; st < 32; ++st) {
      const int64_t r = r0 + (int64_t)st * 32 + warp * 4 + grp;
      float acc = 0.f;
      if (r < hi) {
        const uint4* rv = reinterpret_cast<const uint4*>(v16 + r * dp);
        constexpr int U = 6;  // 16-byte row chunks in flight per lane (a 768-dim row: 2 batches)
        for (int j0 = sub; j0 < nv; j0 += 8 * U) {
          uint4 a[U], b[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = j0 + 8 * u;
            a[u] = j < nv ? __ldg(rv + j) : make_uint4(0, 0, 0, 0);
            b[u] = j < nv ? __ldg(qv + j) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const uint32_t* aw = reinterpret_cast<const uint32_t*>(&a[u]);
            const uint32_t* bw = reinterpret_cast<const uint32_t*>(&b[u]);
#pragma unroll
            for (int w = 0; w < 4; ++w) {
              const unsigned short a0 = (unsigned short)(aw[w] & 0xffffu), a1 = (unsigned short)(aw[w] >> 16);
              const unsigned short b0 = (unsigned short)(bw[w] & 0xffffu), b1 = (unsigned short)(bw[w] >> 16);
              asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a0), "h"(b0));
              asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc) : "h"(a1), "h"(b1));
            }
          }
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      if (sub == 0 && r < hi && acc >= tau) {
        const int at = atomicAdd(&s_cnt, 1);
        s_key[at] = acc;  // at < BIGK_BUF: compaction leaves room for a round
        s_row[at] = (int)r;
      }
    }
    __syncthreads();
    if (s_cnt > BIGK_BUF - ROUND) compact();
    if (s_cnt > BIGK_BUF - ROUND) break;  // near-ties fill the buffer: reported below
  }
  compact();
  const int n = s_cnt;
  const bool over = n > BIGK_BUF - ROUND;
  const size_t base = ((size_t)q * splits + split) * BIGK_BUF;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    out_s[base + i] = s_key[i];
    out_r[base + i] = s_row[i];
  }
  if (threadIdx.x == 0) {
    out_n[(size_t)q * splits + split] = over ? -1 : n;
    out_kth[(size_t)q * splits + split] = s_kth;
  }
}

// Batched form of k_bigk_scan: a block serves QB queries over its row split, so each DB
// row is read from HBM once per QB queries (the single-query kernel re-reads the whole
// DB per query).  Per-query buffers of BIGK_BUF_MQ entries; same filter, compaction and
// outputs (the select stage is shared).  BIGK_BUF_MQ is a power of two (the compaction
// sorts the whole buffer) and holds k plus one round of rows.
template <int QB, int BIGK_BUF_MQ>
__global__ void __launch_bounds__(256)
k_bigk_scan_mq(int64_t n_rows, int64_t dp, int k, int splits, int64_t B, const __half* __restrict__ v16,
               const __half* __restrict__ q16, const float* __restrict__ two_delta, float* __restrict__ out_s,
               int32_t* __restrict__ out_r, int32_t* __restrict__ out_n, float* __restrict__ out_kth) {
  static_assert((BIGK_BUF_MQ & (BIGK_BUF_MQ - 1)) == 0 && BIGK_BUF_MQ <= BIGK_BUF, "power-of-two buffer");
  extern __shared__ __align__(16) uint8_t smem_mq[];
  float* s_key = reinterpret_cast<float*>(smem_mq);                  // [QB][BIGK_BUF_MQ]
  int* s_row = reinterpret_cast<int*>(s_key + QB * BIGK_BUF_MQ);      // [QB][BIGK_BUF_MQ]
  uint4* s_q = reinterpret_cast<uint4*>(s_row + QB * BIGK_BUF_MQ);    // [QB][dp / 8]
  __shared__ int s_cnt[QB];
  __shared__ float s_tau[QB], s_kth[QB], s_td[QB];
  __shared__ int s_over;
  const int split = blockIdx.x;
  const int64_t q0 = (int64_t)blockIdx.y * QB;
  const int nq = (int)(B - q0 < QB ? B - q0 : QB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int grp = lane >> 3, sub = lane & 7;
  const float NEG = -__int_as_float(0x7f800000);
  const int64_t per = (n_rows + splits - 1) / splits;
  const int64_t lo = split * per, hi = min(n_rows, lo + per);
  const int nv = (int)(dp / 8);
  for (int i = threadIdx.x; i < QB * nv; i += blockDim.x) {
    const int qi = i / nv, j = i - qi * nv;
    s_q[i] = qi < nq ? reinterpret_cast<const uint4*>(q16 + (q0 + qi) * dp)[j] : make_uint4(0, 0, 0, 0);
  }
  if (threadIdx.x < QB) {
    s_cnt[threadIdx.x] = 0;
    s_tau[threadIdx.x] = NEG;
    s_kth[threadIdx.x] = NEG;
    s_td[threadIdx.x] = threadIdx.x < nq ? two_delta[q0 + threadIdx.x] : 0.f;
  }
  if (threadIdx.x == 0) s_over = 0;
  __syncthreads();
  auto compact = [&](int qi) {
    float* key = s_key + qi * BIGK_BUF_MQ;
    int* row = s_row + qi * BIGK_BUF_MQ;
    const int n = s_cnt[qi];
    int n2 = 2;
    while (n2 < n) n2 <<= 1;
    for (int i = n + threadIdx.x; i < n2; i += blockDim.x) {
      key[i] = NEG;
      row[i] = INT32_MAX;
    }
    __syncthreads();
    bitonic_desc(key, row, n2, CoarseLess());
    if (threadIdx.x == 0) {
      if (n >= k) {
        s_kth[qi] = key[k - 1];
        s_tau[qi] = fmaxf(s_tau[qi], __fsub_rd(s_kth[qi], s_td[qi]));
      }
      int a = 0, b = n;
      while (a < b) {
        const int mid = (a + b) >> 1;
        if (key[mid] >= s_tau[qi]) a = mid + 1; else b = mid;
      }
      s_cnt[qi] = a;
    }
    __syncthreads();
  };
  constexpr int STEPS = 8;
  constexpr int ROUND = 8 * 4 * STEPS;  // rows per round: 8 warps x 4 rows x STEPS
  for (int64_t r0 = lo; r0 < hi; r0 += ROUND) {
    float tau[QB];
#pragma unroll
    for (int qi = 0; qi < QB; ++qi) tau[qi] = s_tau[qi];
    for (int st = 0; st < STEPS; ++st) {
      const int64_t r = r0 + (int64_t)st * 32 + warp * 4 + grp;
      float acc[QB];
#pragma unroll
      for (int qi = 0; qi < QB; ++qi) acc[qi] = 0.f;
      if (r < hi) {
        const uint4* rv = reinterpret_cast<const uint4*>(v16 + r * dp);
        constexpr int U = 6;
        for (int j0 = sub; j0 < nv; j0 += 8 * U) {
          uint4 a[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = j0 + 8 * u;
            a[u] = j < nv ? __ldg(rv + j) : make_uint4(0, 0, 0, 0);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = j0 + 8 * u;
            if (j >= nv) continue;
            const uint32_t* aw = reinterpret_cast<const uint32_t*>(&a[u]);
#pragma unroll
            for (int qi = 0; qi < QB; ++qi) {
              const uint4 bq = s_q[qi * nv + j];
              const uint32_t* bw = reinterpret_cast<const uint32_t*>(&bq);
#pragma unroll
              for (int w = 0; w < 4; ++w) {
                const unsigned short a0 = (unsigned short)(aw[w] & 0xffffu), a1 = (unsigned short)(aw[w] >> 16);
                const unsigned short b0 = (unsigned short)(bw[w] & 0xffffu), b1 = (unsigned short)(bw[w] >> 16);
                asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[qi]) : "h"(a0), "h"(b0));
                asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(acc[qi]) : "h"(a1), "h"(b1));
              }
            }
          }
        }
      }
#pragma unroll
      for (int qi = 0; qi < QB; ++qi) {
        float v = acc[qi];
        v += __shfl_xor_sync(0xffffffffu, v, 1);
        v += __shfl_xor_sync(0xffffffffu, v, 2);
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        if (sub == 0 && r < hi && qi < nq && v >= tau[qi]) {
          const int at = atomicAdd(&s_cnt[qi], 1);  // < BIGK_BUF_MQ: compaction leaves a round of room
          s_key[qi * BIGK_BUF_MQ + at] = v;
          s_row[qi * BIGK_BUF_MQ + at] = (int)r;
        }
      }
    }
    __syncthreads();
    for (int qi = 0; qi < nq; ++qi) {
      if (s_cnt[qi] > BIGK_BUF_MQ - ROUND) {
        compact(qi);
        if (s_cnt[qi] > BIGK_BUF_MQ - ROUND && threadIdx.x == 0) s_over = 1;
      }
    }
    __syncthreads();
    if (s_over) break;  // near-ties fill a buffer: reported below
  }
  for (int qi = 0; qi < nq; ++qi) {
    compact(qi);
    const int n = s_cnt[qi];
    const size_t base = ((size_t)(q0 + qi) * splits + split) * BIGK_BUF;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      out_s[base + i] = s_key[qi * BIGK_BUF_MQ + i];
      out_r[base + i] = s_row[qi * BIGK_BUF_MQ + i];
    }
    if (threadIdx.x == 0) {
      out_n[(size_t)(q0 + qi) * splits + split] = (s_over || n > BIGK_BUF_MQ - ROUND) ? -1 : n;
      out_kth[(size_t)(q0 + qi) * splits + split] = s_kth[qi];
    }
  }
}

struct SimLess {  // a before b when (-sim, seq) is smaller
  __device__ bool operator()(double ka, int64_t va, double kb, int64_t vb) const {
    return ka < kb || (ka == kb && va > vb);
  }
};

template <typename T>
__global__ void __launch_bounds__(256)
k_bigk_select(int64_t n_rows, int64_t dim, int k, int splits, const T* __restrict__ qx, const T* __restrict__ vm,
              const int32_t* __restrict__ lens, const int64_t* __restrict__ seqs,
              const float* __restrict__ two_delta, const float* __restrict__ in_s, const int32_t* __restrict__ in_r,
              const int32_t* __restrict__ in_n, const float* __restrict__ in_kth, double* __restrict__ out_sim,
              int64_t* __restrict__ out_seq, int32_t* __restrict__ out_len, int32_t* __restrict__ out_count,
              int32_t* __restrict__ overflow, unsigned int* __restrict__ inexact_count, const BlasRef blas) {
  extern __shared__ uint8_t smem_bs[];
  float* s_key = reinterpret_cast<float*>(smem_bs);
  int* s_row = reinterpret_cast<int*>(s_key + BIGK_BUF);
  double* s_sim = reinterpret_cast<double*>(s_row + BIGK_BUF);
  int64_t* s_seq = reinterpret_cast<int64_t*>(s_sim + BIGK_BUF);
  __shared__ float s_tau;
  __shared__ int s_cnt, s_bad;
  const int64_t q = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float NEG = -__int_as_float(0x7f800000);
  const float td = two_delta[q];
  const int kk = (int)(k < n_rows ? k : n_rows);
  if (threadIdx.x == 0) {
    float t = NEG;
    int bad = 0;
    for (int sp = 0; sp < splits; ++sp) {
      t = fmaxf(t, in_kth[(size_t)q * splits + sp]);
      bad |= in_n[(size_t)q * splits + sp] < 0;
    }
    s_tau = t > NEG ? __fsub_rd(t, td) : NEG;
    s_cnt = 0;
    s_bad = bad || !(td <= 3.0e38f);
  }
  __syncthreads();
  if (s_bad) {  // near-ties overflowed a split's buffer, or rows outside the fp16 range
    if (threadIdx.x == 0) {
      out_count[q] = 0;
      atomicOr(overflow, 1);
    }
    return;
  }
  // the global coarse kk-th over the splits' entries (each split's k-th is only a lower
  // bound of it: with many small splits the union above it holds ~k x splits entries):
  // radix select, 8 bits per pass, on the order-preserving key
  {
    __shared__ int s_hist[256];
    __shared__ uint32_t s_prefix, s_mask;
    __shared__ int s_rem, s_total;
    if (threadIdx.x == 0) {
      s_prefix = 0;
      s_mask = 0;
      s_rem = kk;
      s_total = 0;
    }
    for (int shift = 24; shift >= 0; shift -= 8) {
      s_hist[threadIdx.x] = 0;  // blockDim.x == 256
      __syncthreads();
      const uint32_t pre = s_prefix, msk = s_mask;
      for (int sp = warp; sp < splits; sp += blockDim.x >> 5) {  // a warp per split
        const int n = in_n[(size_t)q * splits + sp];
        const size_t base = ((size_t)q * splits + sp) * BIGK_BUF;
        for (int i = lane; i < n; i += 32) {
          const float v = in_s[base + i];
          const uint32_t key = ord_key(v);
          if (v >= s_tau && (key & msk) == pre) atomicAdd(&s_hist[(key >> shift) & 255], 1);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (shift == 24)
          for (int d = 0; d < 256; ++d) s_total += s_hist[d];  // entries >= the filter
        int cum = 0, dgt = 255;
        for (; dgt > 0; --dgt) {
          if (cum + s_hist[dgt] >= s_rem) break;
          cum += s_hist[dgt];
        }
        s_prefix = pre | ((uint32_t)dgt << shift);
        s_mask = msk | (255u << shift);
        s_rem -= cum;
      }
      __syncthreads();
    }
    // fewer than kk entries above the filter: every one is a candidate (tau unchanged)
    if (threadIdx.x == 0 && s_total >= kk) s_tau = fmaxf(s_tau, __fsub_rd(ord_val(s_prefix), td));
    __syncthreads();
  }
  // gather the splits' entries above the filter
  for (int sp = warp; sp < splits; sp += blockDim.x >> 5) {  // a warp per split
    const int n = in_n[(size_t)q * splits + sp];
    const size_t base = ((size_t)q * splits + sp) * BIGK_BUF;
    for (int i = lane; i < n; i += 32) {
      const float v = in_s[base + i];
      if (v >= s_tau) {
        const int at = atomicAdd(&s_cnt, 1);
        if (at < BIGK_BUF) {
          s_key[at] = v;
          s_row[at] = in_r[base + i];
        }
      }
    }
  }
  __syncthreads();
  int n = s_cnt;
  if (n > BIGK_BUF) {
    if (threadIdx.x == 0) {
      out_count[q] = 0;
      atomicOr(overflow, 1);
    }
    return;
  }

  // exact float64 scores (as k_rescore), then (-sim, seq) order
  if (blas.on) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      const int row = s_row[c];
      const int64_t sq = seqs[row];
      s_sim[c] = blas_dot<T>(vm + (size_t)row * dim, qx + q * dim, dim,
                             blas_kind(sq % blas.ref_cap, blas.ref_n, dim, blas.threads));
      s_seq[c] = sq;
    }
  } else {
    for (int c = warp; c < n; c += blockDim.x >> 5) {
      const int row = s_row[c];
      bool ok;
      double sim = warp_exact_dot<8, T>(vm + (size_t)row * dim, qx + q * dim, dim, ok);
      if (!ok) {
        sim = warp_exact_dot_fallback(vm + (size_t)row * dim, qx + q * dim, dim);
        if (lane == 0) atomicAdd(inexact_count, 1u);
      }
      if (lane == 0) {
        s_sim[c] = sim;
        s_seq[c] = seqs[row];
      }
    }
  }
  for (int i = n + threadIdx.x; i < BIGK_BUF; i += blockDim.x) {
    s_sim[i] = -__longlong_as_double(0x7ff0000000000000ll);
    s_seq[i] = INT64_MAX;
  }
  __syncthreads();
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  // s_row travels with the order through the seq -> row map: sort (sim, seq), then find
  // each output's row by its (unique) seq among the candidates
  bitonic_desc(s_sim, s_seq, n2 < 2 ? 2 : n2, SimLess());
  const int outn = n < kk ? n : kk;
  for (int i = threadIdx.x; i < outn; i += blockDim.x) {
    out_sim[q * k + i] = s_sim[i];
    out_seq[q * k + i] = s_seq[i];
  }
  // lengths: rows are looked up by seq (slot = the candidate whose seq matches)
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    const int row = s_row[c];
    const int64_t sq = seqs[row];
    for (int i = 0; i < outn; ++i)
      if (s_seq[i] == sq) out_len[q * k + i] = lens[row];
  }
  if (threadIdx.x == 0) out_count[q] = outn;
}

// ------------------------------------------------------------------ shard merge
// G per-shard sorted lists [G][B][k] -> global top-k by (-sim, seq).  Thread per query.
__global__ void k_topk_merge(int G, int64_t B, int k, const double* __restrict__ sims, const int64_t* __restrict__ seqs,
                             const int32_t* __restrict__ lens, const int32_t* __restrict__ counts,
                             double* __restrict__ o_sim, int64_t* __restrict__ o_seq, int32_t* __restrict__ o_len,
                             int32_t* __restrict__ o_cnt) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= B) return;
  int pos[64];
  for (int g = 0; g < G; ++g) pos[g] = 0;
  int n = 0;
  while (n < k) {
    int best = -1;
    double bs = 0;
    int64_t bq = 0;
    for (int g = 0; g < G; ++g) {
      const int c = counts[(size_t)g * B + q];
      if (pos[g] >= c) continue;
      const size_t idx = ((size_t)g * B + q) * k + pos[g];
      const double s = sims[idx];
      const int64_t sq = seqs[idx];
      if (best < 0 || s > bs || (s == bs && sq < bq)) { best = g; bs = s; bq = sq; }
    }
    if (best < 0) break;
    const size_t idx = ((size_t)best * B + q) * k + pos[best];
    o_sim[q * k + n] = bs;
    o_seq[q * k + n] = bq;
    o_len[q * k + n] = lens[idx];
    ++pos[best];
    ++n;
  }
  o_cnt[q] = n;
}

// ------------------------------------------------------------------ finish
// numpy's pairwise summation of a contiguous float64 array (pairwise_sum_DOUBLE): n < 8
// sequential from 0.0; n <= 128: 8 accumulators, ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
// then the remainder; above 128 the halves (split at n/2 rounded down to a multiple of 8)
// are summed recursively.  v(i) returns element i.
template <typename F>
__device__ double np_sum_f(const F& v, int lo, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, v(lo + i));
    return r;
  }
  if (n > 128) {
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(np_sum_f(v, lo, n2), np_sum_f(v, lo + n2, n - n2));
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = v(lo + j);
  int i = 8;
  for (; i + 8 <= n; i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v(lo + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, v(lo + i));
  return res;
}

// Warp per query.  Retrieval branch (predictor.py:314-324) when any neighbour has sim
// >= s0, else the float64 MLP (predictor.py:209-219): h_j = tanh(b1_j + sum_d x_d W1[d,j])
// with the sum in index order, out = b2 + sum_j h_j w2_j in index order.
template <typename X>
__global__ void k_finish(int64_t B, int k, const double* __restrict__ sims, const int32_t* __restrict__ lens,
                         const int32_t* __restrict__ counts, double s0, const X* __restrict__ x, int64_t dim,
                         const double* __restrict__ W1, const double* __restrict__ b1, const double* __restrict__ w2,
                         double b2, int64_t hidden, int64_t max_len, double log_cap, int32_t* __restrict__ out_len,
                         uint8_t* __restrict__ out_ret, bool stage) {
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
#ifdef ALISE_FINISH_TIMING
  const long long F0 = clock64();
  long long F1 = 0, F2 = 0;
#endif
  // stage W1 (and each warp's query) in shared memory when some query of the block
  // takes the MLP branch and the launch provided the space
  extern __shared__ double smem_fin[];
  const double* smem_w1 = nullptr;
  if (stage) {
    bool mlp = false;
    if (q < B && lane == 0) {
      mlp = true;
      for (int i = 0; i < counts[q]; ++i)
        if (sims[q * k + i] >= s0) mlp = false;
    }
    if (__syncthreads_or(mlp)) {
      const int64_t nw = dim * hidden;
      X* xs0 = reinterpret_cast<X*>(smem_fin + nw);
      const int64_t q0 = (int64_t)blockIdx.x * (blockDim.x >> 5);
      const int64_t nq = B - q0 < (int64_t)(blockDim.x >> 5) ? B - q0 : (int64_t)(blockDim.x >> 5);
      // one bulk (TMA) copy of W1 and of the block's query rows when the addresses allow
      // it; a plain load/store loop has one L2 round trip in flight per thread
      const bool bulk = ((reinterpret_cast<uintptr_t>(W1) | reinterpret_cast<uintptr_t>(x + q0 * dim)) & 15) == 0 &&
                        (dim & 3) == 0 && (nw & 1) == 0;
      if (bulk) {
        __shared__ uint64_t fin_bar;
        if (threadIdx.x == 0) {
          sm100::mbar_init(&fin_bar, 1);
          sm100::fence_barrier_init();
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const uint32_t wb = (uint32_t)(nw * 8), xb = (uint32_t)(nq * dim * sizeof(X));
          sm100::mbar_arrive_expect_tx(&fin_bar, wb + xb);
          for (uint32_t o = 0; o < wb; o += 32768)
            sm100::bulk_g2s(reinterpret_cast<uint8_t*>(smem_fin) + o, reinterpret_cast<const uint8_t*>(W1) + o,
                            wb - o < 32768 ? wb - o : 32768, &fin_bar);
          sm100::bulk_g2s(xs0, x + q0 * dim, xb, &fin_bar);
        }
        sm100::mbar_wait(&fin_bar, 0);
      } else {
        for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) smem_fin[i] = W1[i];
        X* xs = xs0 + (threadIdx.x >> 5) * dim;
        if (q < B)
          for (int64_t i = lane; i < dim; i += 32) xs[i] = x[q * dim + i];
        __syncthreads();
      }
      smem_w1 = smem_fin;
    }
  }
  if (q >= B) return;
#ifdef ALISE_FINISH_TIMING
  F1 = clock64();
#endif
  // retrieval branch: the list is sorted by (-sim, seq), so the qualifying neighbours
  // (sim >= s0) are a prefix of it; sums over them in numpy's order
  const int c = counts[q];
  const double* sq = sims + q * k;
  const int32_t* lq = lens + q * k;
  int nq = 0;
  while (nq < c && sq[nq] >= s0) ++nq;
  if (nq > 0) {
    if (lane == 0) {
      auto w = [&](int i) { const double v = sq[i]; return v < 0.0 ? 0.0 : v; };  // np.clip(.., 0, None)
      auto val = [&](int i) { return (double)lq[i]; };
      auto prod = [&](int i) { return __dmul_rn(w(i), val(i)); };
      const double ws = np_sum_f(w, 0, nq);
      double pred;
      if (ws > 0.0) pred = __ddiv_rn(np_sum_f(prod, 0, nq), ws);
      else pred = __ddiv_rn(np_sum_f(val, 0, nq), (double)nq);
      double r = rint(pred);
      r = fmin(fmax(r, 1.0), (double)max_len);
      out_len[q] = (int32_t)r;
      out_ret[q] = 1;
    }
    return;
  }
  // fallback MLP: lane j computes hidden units j, j+32, ... in chunks of 128 units.
  // The dependent index-order chain reads W1 and x from shared memory when the block
  // staged them (one L2 round trip per block instead of one per term).
  // hidden unit j's pre-activation in index order; instantiated once on the staged
  // shared-memory copies (32-bit shared addressing, LDS) and once on global memory
  auto pre_act = [&](const double* Wm, const X* xq, int64_t j) {
    double acc = 0.0;
    int64_t d0 = 0;
    // products of 32 terms first (independent: loads, converts and multiplies pipeline),
    // then their index-order adds: the chain runs at the add latency; two chunks per
    // iteration let the next chunk's loads fill this chunk's chain
#pragma unroll 2
    for (; d0 + 32 <= dim; d0 += 32) {
      double pr[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) pr[u] = __dmul_rn((double)xq[d0 + u], Wm[(d0 + u) * hidden + j]);
#pragma unroll
      for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, pr[u]);
    }
    for (int64_t d = d0; d < dim; ++d) acc = __dadd_rn(acc, __dmul_rn((double)xq[d], Wm[d * hidden + j]));
    return acc;
  };
  double out = 0.0;
  for (int64_t j0 = 0; j0 < hidden; j0 += 128) {
    double hv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t j = j0 + lane + 32 * t;
      double acc = 0.0;
      if (j < hidden) {
        if (smem_w1)
          acc = pre_act(smem_fin, reinterpret_cast<const X*>(smem_fin + dim * hidden) + (threadIdx.x >> 5) * dim, j);
        else
          acc = pre_act(W1, x + q * dim, j);
        hv[t] = tanh(__dadd_rn(acc, b1[j]));
      } else {
        hv[t] = 0.0;
      }
    }
#ifdef ALISE_FINISH_TIMING
    F2 = clock64();
#endif
    // sequential sum over the chunk's hidden units in index order (every lane)
    const int jn = (int)(hidden - j0 < 128 ? hidden - j0 : 128);
#pragma unroll
    for (int t = 0; t < 4; ++t) {  // hv[t] stays a static register: one shuffle per unit
      const int cnt = jn - 32 * t < 32 ? jn - 32 * t : 32;
      if (cnt <= 0) break;
      // each lane forms its own product h_j * w2_j (the same rounding as forming it after
      // the shuffle); the 32 shuffles are independent, only the adds are chained
      const int64_t jl = j0 + 32 * t + lane;
      const double pj = jl < hidden ? __dmul_rn(hv[t], w2[jl]) : 0.0;
      if (cnt == 32) {
        double ps[32];
#pragma unroll
        for (int src = 0; src < 32; ++src) ps[src] = __shfl_sync(0xffffffffu, pj, src);
#pragma unroll
        for (int src = 0; src < 32; ++src) out = __dadd_rn(out, ps[src]);
      } else {
        for (int src = 0; src < cnt; ++src) out = __dadd_rn(out, __shfl_sync(0xffffffffu, pj, src));
      }
    }
  }
  if (lane == 0) {
    out = __dadd_rn(out, b2);
    const double raw = exp(fmin(out, log_cap));
    double r = rint(raw);
    r = fmin(fmax(r, 1.0), (double)max_len);
    out_len[q] = (int32_t)r;
    out_ret[q] = 0;
#ifdef ALISE_FINISH_TIMING
    if (q < 2) printf("[finish q=%lld] stage %lld hidden %lld out %lld\n", (long long)q, F1 - F0, F2 - F1, clock64() - F2);
#endif
  }
}

}  // namespace pred
}  // namespace alise
