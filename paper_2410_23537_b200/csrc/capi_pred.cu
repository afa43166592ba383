// C ABI for the retrieval length predictor: device DB ring (VectorStore), exact
// batched top-k (tcgen05 coarse scan + exact rescoring), shard merge, finish.
// Declarations and reference citations: include/alise_b200.h.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/alise_b200.h"

// NVTX ranges around the C ABI calls (header-only NVTX v3: no cost unless a profiler
// such as nsys is attached), so host-side call spans line up with the kernel/copy
// timeline.
namespace {
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace
#include "pred_scan.cuh"
#include "embed.cuh"

namespace alise {
int fail(int code, const char* fmt, ...);
}
using namespace alise;
using namespace alise::pred;

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail(ALISE_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define CKL()                                                                                 \
  do {                                                                                        \
    cudaError_t e_ = cudaGetLastError();                                                      \
    if (e_ != cudaSuccess) return fail(ALISE_ECUDA, "launch: %s", cudaGetErrorString(e_));    \
  } while (0)

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D fp16 K-major tile map: rows x cols(=dp), box rows_box x 64, 128-byte swizzle.
static int make_map(CUtensorMap* m, void* base, uint64_t rows, uint64_t dp, uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(ALISE_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {dp, rows};
  cuuint64_t strides[1] = {dp * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ALISE_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ALISE_OK;
}

struct alise_db {
  int device = 0;
  int64_t capacity = 0, cap_p = 0, dim = 0, dp = 0;
  int64_t size = 0, next_seq = 0;
  int64_t seq_stride = 1;  // sharded stores hold every G-th sequence: slot = (seq / G) % capacity
  int f64 = 0;              // master dtype: 0 fp32, 1 float64 (ALISE_DB_F32 / ALISE_DB_F64)
  size_t esz = 4;           // bytes per master element
  void* vm = nullptr;       // master vectors [capacity][dim]
  __half* v16 = nullptr;
  int32_t* lens = nullptr;
  int64_t* seqs = nullptr;
  BlasRef blas{0, 1, 0, -1};         // sims order (ref_cap 0 / ref_n -1: this store's own)
  unsigned int* vmax = nullptr;     // float bits of the max row norm
  unsigned int* inexact = nullptr;  // candidates whose rounding could not be certified
  CUtensorMap tmD;
  CUtensorMap tmD2;  // 128-row boxes for the 2-SM scan
  // query scratch
  int64_t bp_cap = 0;
  int splits_cap = 0;
  __half* q16 = nullptr;
  float* two_delta = nullptr;
  float* cand_s = nullptr;
  int32_t* cand_r = nullptr;
  int32_t* cand_n = nullptr;
  float* topc = nullptr;
  int32_t* need = nullptr;
  // state of the last scan (alise_db_topk_scan -> alise_db_topk_rescore)
  ScanArgs last{};
  int64_t last_B = -1;
  int last_k = 0, last_qblk = 0, last_nh = 1;
  const void* last_q = nullptr;
  uint32_t* gkth = nullptr;  // shared lower bound of the k-th per query, then [bp][KMAX] rank slots
  CUtensorMap tmQ;
  // optional kernel timing (bench roofline): event pairs around each scan launch
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  double scan_flops = 0.0;
};

extern "C" int alise_db_create(int device, int64_t capacity, int64_t dim, alise_db** out) {
  return alise_db_create_ex(device, capacity, dim, ALISE_DB_F32, out);
}

extern "C" int alise_db_create_ex(int device, int64_t capacity, int64_t dim, int master_dtype, alise_db** out) {
  if (capacity <= 0 || dim <= 0) return fail(ALISE_EINVAL, "capacity and dim must be positive");
  if (master_dtype != ALISE_DB_F32 && master_dtype != ALISE_DB_F64) return fail(ALISE_EINVAL, "bad master dtype");
  if (capacity > ((int64_t)1 << 31) - 512) return fail(ALISE_EINVAL, "capacity too large");
  CK(cudaSetDevice(device));
  alise_db* db = new alise_db();
  db->device = device;
  db->capacity = capacity;
  db->cap_p = (capacity + BN - 1) / BN * BN;
  db->dim = dim;
  db->dp = (dim + 63) / 64 * 64;
  db->f64 = master_dtype == ALISE_DB_F64;
  db->esz = db->f64 ? 8 : 4;
  CK(cudaMalloc(&db->vm, db->esz * capacity * dim));
  CK(cudaMalloc(&db->v16, sizeof(__half) * db->cap_p * db->dp));
  CK(cudaMemset(db->v16, 0, sizeof(__half) * db->cap_p * db->dp));
  CK(cudaMalloc(&db->lens, sizeof(int32_t) * capacity));
  CK(cudaMalloc(&db->seqs, sizeof(int64_t) * capacity));
  CK(cudaMalloc(&db->vmax, 2 * sizeof(unsigned int)));
  CK(cudaMemset(db->vmax, 0, 2 * sizeof(unsigned int)));
  db->inexact = db->vmax + 1;
  int s = make_map(&db->tmD, db->v16, db->cap_p, db->dp, BN);
  if (s) return s;
  s = make_map(&db->tmD2, db->v16, db->cap_p, db->dp, BN / 2);
  if (s) return s;
  *out = db;
  return ALISE_OK;
}

static void free_scratch(alise_db* db) {
  cudaFree(db->q16);
  cudaFree(db->two_delta);
  cudaFree(db->cand_s);
  cudaFree(db->cand_r);
  cudaFree(db->cand_n);
  cudaFree(db->topc);
  cudaFree(db->need);
  cudaFree(db->gkth);
  db->gkth = nullptr;
  db->q16 = nullptr;
  db->bp_cap = 0;
  db->splits_cap = 0;
}

extern "C" int alise_db_destroy(alise_db* db) {
  if (!db) return ALISE_OK;
  cudaDeviceSynchronize();
  cudaFree(db->vm);
  cudaFree(db->v16);
  cudaFree(db->lens);
  cudaFree(db->seqs);
  cudaFree(db->vmax);
  free_scratch(db);
  delete db;
  return ALISE_OK;
}

extern "C" int alise_db_set_order(alise_db* db, int order, int blas_threads, int64_t ref_capacity, int64_t ref_size) {
  if (!db || (order != ALISE_ORDER_EXACT && order != ALISE_ORDER_BLAS)) return fail(ALISE_EINVAL, "bad order");
  if (ref_capacity < 0 || (ref_capacity > 0 && ref_size > ref_capacity))
    return fail(ALISE_EINVAL, "bad reference ring geometry");
  db->blas.on = order == ALISE_ORDER_BLAS;
  db->blas.threads = blas_threads < 1 ? 1 : blas_threads;
  db->blas.ref_cap = ref_capacity;
  db->blas.ref_n = ref_size;
  return ALISE_OK;
}

extern "C" int alise_db_dtype(alise_db* db, int* master_dtype) {
  if (!db || !master_dtype) return fail(ALISE_EINVAL, "null argument");
  *master_dtype = db->f64 ? ALISE_DB_F64 : ALISE_DB_F32;
  return ALISE_OK;
}

extern "C" int alise_db_append(alise_db* db, const void* vecs, const int32_t* lens, const int64_t* seqs,
                               int64_t n, void* stream) {
  NvtxRange nvtx_range("alise_db_append");
  if (!db || n < 0) return fail(ALISE_EINVAL, "bad append");
  if (n == 0) return ALISE_OK;
  // rows with equal slot in one batch would race; the host splits batches larger than capacity
  if (n > db->capacity) return fail(ALISE_EINVAL, "append batch larger than capacity");
  if (db->f64)
    k_db_append<double><<<(unsigned)n, 128, 0, S(stream)>>>(static_cast<const double*>(vecs), lens, seqs, n, db->dim,
                                                            db->dp, db->capacity, db->seq_stride,
                                                            static_cast<double*>(db->vm), db->v16, db->lens,
                                                            db->seqs, db->vmax);
  else
    k_db_append<float><<<(unsigned)n, 128, 0, S(stream)>>>(static_cast<const float*>(vecs), lens, seqs, n, db->dim,
                                                           db->dp, db->capacity, db->seq_stride,
                                                           static_cast<float*>(db->vm), db->v16, db->lens, db->seqs,
                                                           db->vmax);
  CKL();
  db->next_seq += n;
  db->size = std::min(db->capacity, db->size + n);
  return ALISE_OK;
}

extern "C" int alise_db_set_seq_stride(alise_db* db, int64_t stride) {
  if (!db || stride < 1) return fail(ALISE_EINVAL, "stride must be >= 1");
  if (db->next_seq) return fail(ALISE_EINVAL, "set the stride before the first append");
  db->seq_stride = stride;
  return ALISE_OK;
}

extern "C" int alise_db_size(alise_db* db, int64_t* size, int64_t* next_seq) {
  if (!db) return fail(ALISE_EINVAL, "null db");
  if (size) *size = db->size;
  if (next_seq) *next_seq = db->next_seq;
  return ALISE_OK;
}

extern "C" int alise_db_export(alise_db* db, void* vecs, int32_t* lens, int64_t* seqs, int64_t n, void* stream) {
  if (!db || n < 0 || n > db->size) return fail(ALISE_EINVAL, "bad export count");
  if (n == 0) return ALISE_OK;
  CK(cudaMemcpyAsync(vecs, db->vm, db->esz * n * db->dim, cudaMemcpyDeviceToDevice, S(stream)));
  CK(cudaMemcpyAsync(lens, db->lens, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, S(stream)));
  CK(cudaMemcpyAsync(seqs, db->seqs, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, S(stream)));
  return ALISE_OK;
}

extern "C" int alise_db_inexact(alise_db* db, unsigned int* count) {
  CK(cudaMemcpy(count, db->inexact, sizeof(unsigned int), cudaMemcpyDeviceToHost));
  return ALISE_OK;
}


static int ensure_scratch(alise_db* db, int64_t Bp, int splits, cudaStream_t st) {
  if (Bp <= db->bp_cap && splits <= db->splits_cap) return ALISE_OK;
  CK(cudaStreamSynchronize(st));
  free_scratch(db);
  const int64_t bp = std::max(Bp, (int64_t)128);
  const int sp = std::max(splits, 1);
  CK(cudaMalloc(&db->q16, sizeof(__half) * bp * db->dp));
  CK(cudaMalloc(&db->two_delta, sizeof(float) * bp));
  CK(cudaMalloc(&db->cand_s, sizeof(float) * sp * bp * CAP));
  CK(cudaMalloc(&db->cand_r, sizeof(int32_t) * sp * bp * CAP));
  CK(cudaMalloc(&db->cand_n, sizeof(int32_t) * sp * bp));
  CK(cudaMalloc(&db->topc, sizeof(float) * sp * bp * KMAX));
  CK(cudaMalloc(&db->need, sizeof(int32_t) * bp));
  CK(cudaMalloc(&db->gkth, sizeof(uint32_t) * bp * (1 + KMAX)));
  db->bp_cap = bp;
  db->splits_cap = sp;
  return make_map(&db->tmQ, db->q16, bp, db->dp, BM);
}

static int sm_count_pred() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Coarse scan of a search (db->size > 0, B > 0): query prep, the tcgen05 scan with the
// fused candidate filter; leaves the candidates and bounds in the DB scratch.
static int topk_scan(alise_db* db, const void* queries, int64_t B, int k, cudaStream_t st) {
  // 2-SM (cta_group::2) scan for batches above one query block; 1-SM otherwise
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("ALISE_SCAN_2SM");
    force = e ? atoi(e) : -1;
  }
  const bool two_sm = force == -1 ? (B > BM) : (force != 0);
  const int qblk = two_sm ? 2 * BM : BM;
  const int64_t Bp = (B + qblk - 1) / qblk * qblk;
  const int n_qb = (int)(Bp / qblk);
  const int n_tiles = (int)((db->size + BN - 1) / BN);
  const int units = two_sm ? sm_count_pred() / 2 : sm_count_pred();
  // work split (pred_scan.cuh next_seg): G groups per query block, E excess groups cut
  // into nc chunks of C tiles so every unit scans about the same number of tiles
  const int G = std::max(1, std::min(n_tiles, (units + n_qb - 1) / n_qb));
  const int E = std::max(0, n_qb * G - units);
  const int n_units = std::min(units, n_qb * G);
  const int glen = n_tiles / G;  // length of group G-1 (the excess groups)
  const int nc = E ? std::max(1, n_units / E) : 0;
  const int C = E ? (glen + nc - 1) / nc : 0;
  const int groups = E ? std::max(G, G - 1 + (glen + C - 1) / C) : G;
  // 2-SM scan with k <= 8: two epilogue warps per TMEM lane quarter, each its own split
  static int halves = -1;
  if (halves < 0) {
    const char* e = getenv("ALISE_SCAN2_HALVES");
    halves = e ? std::max(1, std::min(2, atoi(e))) : 2;
  }
  const int nh = (two_sm && k <= 8) ? halves : 1;
  const int splits = groups * nh;
  int s = ensure_scratch(db, Bp, splits, st);
  if (s) return s;
  if (db->f64)
    k_query_prep<double><<<(unsigned)Bp, 128, 0, st>>>(static_cast<const double*>(queries), B, db->dim, db->dp,
                                                       db->vmax, db->q16, db->two_delta, db->blas.on, db->gkth,
                                                       db->need);
  else
    k_query_prep<float><<<(unsigned)Bp, 128, 0, st>>>(static_cast<const float*>(queries), B, db->dim, db->dp,
                                                      db->vmax, db->q16, db->two_delta, db->blas.on, db->gkth,
                                                      db->need);
  CKL();
  ScanArgs a;
  a.n_kb = (int)(db->dp / BK);
  a.n_rows = db->size;
  a.n_tiles = n_tiles;
  a.n_qb = n_qb;
  a.n_splits = splits;
  a.G = G;
  a.units = n_units;
  a.E = E;
  a.nc = nc;
  a.C = C;
  a.B = (int)B;
  a.Bp = (int)Bp;
  a.k = k;
  a.two_delta = db->two_delta;
  a.cand_s = db->cand_s;
  a.cand_r = db->cand_r;
  a.cand_n = db->cand_n;
  a.topc = db->topc;
  a.gkth = db->gkth;
  static int warm = -1;
  if (warm < 0) {
    const char* e = getenv("ALISE_SCAN_WARM");
    warm = e ? atoi(e) : 1;
  }
  a.warm = warm;
  // [Bp] shared k-th, then [Bp][KMAX] rank slots (16-byte aligned: Bp % 128 == 0): one memset
  a.gslot = db->gkth + Bp;
  a.slot_m = (k + G * nh - 1) / (G * nh);
  // long groups warm up early in their run: one exchange per tile is enough
  a.sync_tile = n_tiles / G >= 256 ? 1 : 0;
  // (gkth, the rank slots and the exhaustive flags were cleared by k_query_prep)
  static bool attr_set[5] = {false, false, false, false, false};
  const int kt = two_sm ? (k <= 8 ? (nh == 2 ? 4 : 2) : 3) : (k <= 8 ? 0 : 1);
  if (!attr_set[kt]) {
    switch (kt) {
      case 0: CK(cudaFuncSetAttribute(k_scan<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN_SMEM)); break;
      case 1: CK(cudaFuncSetAttribute(k_scan<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN_SMEM)); break;
      case 2: CK(cudaFuncSetAttribute(k_scan2<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN2_SMEM)); break;
      case 3: CK(cudaFuncSetAttribute(k_scan2<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN2_SMEM)); break;
      default: CK(cudaFuncSetAttribute(k_scan2<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SCAN2_SMEM)); break;
    }
    attr_set[kt] = true;
  }
  const unsigned grid = two_sm ? (unsigned)(2 * n_units) : (unsigned)n_units;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (db->timing) {
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    db->scan_flops += 2.0 * (double)B * (double)db->size * (double)db->dim;
  }
  switch (kt) {
    case 0: k_scan<8><<<grid, 192, SCAN_SMEM, st>>>(db->tmQ, db->tmD, a); break;
    case 1: k_scan<16><<<grid, 192, SCAN_SMEM, st>>>(db->tmQ, db->tmD, a); break;
    case 2: k_scan2<8, 1><<<grid, 192, SCAN2_SMEM, st>>>(db->tmQ, db->tmD2, a); break;
    case 3: k_scan2<16, 1><<<grid, 192, SCAN2_SMEM, st>>>(db->tmQ, db->tmD2, a); break;
    default: k_scan2<8, 2><<<grid, 320, SCAN2_SMEM, st>>>(db->tmQ, db->tmD2, a); break;
  }
  CKL();
  if (db->timing) {
    CK(cudaEventRecord(e1, st));
    db->ev.push_back(e0);
    db->ev.push_back(e1);
  }
  static int stats = -1;
  if (stats < 0) {
    const char* e = getenv("ALISE_SCAN_STATS");
    stats = e ? atoi(e) : 0;
  }
  if (stats) {  // diagnostics: candidate counts after the scan
    CK(cudaStreamSynchronize(st));
    std::vector<int32_t> cn((size_t)splits * Bp);
    CK(cudaMemcpy(cn.data(), db->cand_n, cn.size() * 4, cudaMemcpyDeviceToHost));
    double tot = 0;
    int ovf = 0;
    for (int sp = 0; sp < splits; ++sp)
      for (int64_t q = 0; q < B; ++q) {
        const int c = cn[(size_t)sp * Bp + q];
        if (c < 0) ++ovf; else tot += c;
      }
    fprintf(stderr, "[scan stats] B=%lld splits=%d cand/query=%.1f ovf=%d\n", (long long)B, splits, tot / B, ovf);
  }
  db->last = a;
  db->last_B = B;
  db->last_k = k;
  db->last_qblk = qblk;
  db->last_nh = nh;
  db->last_q = queries;
  return ALISE_OK;
}

// Exact rescoring of the last scan.  ext (may be NULL): per-query exact-score lower
// bounds of the global k-th from the shards (all-reduced max of alise_db_topk_scan's
// bounds): candidates with coarse score below ext - delta cannot enter the global top-k
// and are not rescored.
static BlasRef blas_ref(const alise_db* db) {
  BlasRef b = db->blas;
  if (b.ref_cap <= 0) b.ref_cap = db->capacity;
  if (b.ref_n < 0) b.ref_n = db->size;
  return b;
}

static int grp_len_host(int n_tiles, int G, int g) { return n_tiles / G + (g < n_tiles % G ? 1 : 0); }

template <typename T>
static int topk_rescore_t(alise_db* db, const T* queries, int64_t B, int k, const float* ext, double* out_sim,
                          int64_t* out_seq, int32_t* out_len, int32_t* out_count, cudaStream_t st) {
  const ScanArgs& a = db->last;
  const int qblk = db->last_qblk, nh = db->last_nh;
  const int64_t Bp = a.Bp;
  const T* vm = static_cast<const T*>(db->vm);

  // small batches are latency bound (one DRAM round trip per candidate row), large ones
  // throughput bound (registers / occupancy)
  // (large batches: 128-thread blocks capped at 64 registers keep 8 queries in flight
  // per SM; k_rescore's launch bounds fix the block sizes)
#ifndef ALISE_RESCORE_SMALL_B
#define ALISE_RESCORE_SMALL_B 512
#endif
  const bool small_b = B <= ALISE_RESCORE_SMALL_B;
  auto rescore = small_b ? k_rescore<24, T> : k_rescore<8, T>;
  const int rthreads = small_b ? 256 : 128;
  const BlasRef br = blas_ref(db);
  // the longest top-list union a query can have: nh x (largest split count) x k
  const int max_splits = std::max(a.G, a.E > 0 ? a.G - 1 + (grp_len_host(a.n_tiles, a.G, a.G - 1) + a.C - 1) / a.C : 0);
  const int top_cap = (int)std::min<int64_t>(4096, (int64_t)nh * max_splits * k);
  rescore<<<(unsigned)B, rthreads, top_cap * sizeof(float), st>>>(
      qblk, nh, a, (int)Bp, B, k, db->size, db->dim, queries, vm, db->lens, db->seqs, db->two_delta, db->cand_s,
      db->cand_r, db->cand_n, db->topc, ext, out_sim, out_seq, out_len, out_count, db->need, db->inexact, br, top_cap);
  CKL();
  if (!small_b) {  // (small batches ran the exhaustive path inside k_rescore)
    k_exhaustive<T><<<(unsigned)((B + 255) / 256), 256, 0, st>>>(B, k, db->size, db->dim, queries, vm, db->lens,
                                                                 db->seqs, db->need, out_sim, out_seq, out_len,
                                                                 out_count, db->inexact, br);
    CKL();
  }
  return ALISE_OK;
}

static int topk_rescore(alise_db* db, const void* queries, int64_t B, int k, const float* ext, double* out_sim,
                        int64_t* out_seq, int32_t* out_len, int32_t* out_count, cudaStream_t st) {
  if (db->f64)
    return topk_rescore_t(db, static_cast<const double*>(queries), B, k, ext, out_sim, out_seq, out_len, out_count,
                          st);
  return topk_rescore_t(db, static_cast<const float*>(queries), B, k, ext, out_sim, out_seq, out_len, out_count, st);
}


// top_k above KMAX (k <= BIGK_MAX): k_bigk_scan over row splits, then k_bigk_select
// per query (pred_scan.cuh).  Exact like the tcgen05 path; near-ties that overflow a
// buffer fail with ECAPACITY instead of returning a wrong list.
template <typename T>
static int topk_bigk_t(alise_db* db, const T* queries, int64_t B, int k, double* out_sim, int64_t* out_seq,
                       int32_t* out_len, int32_t* out_count, cudaStream_t st) {
  const int64_t Bp = (B + BM - 1) / BM * BM;
  int s = ensure_scratch(db, Bp, 1, st);
  if (s) return s;
  k_query_prep<T><<<(unsigned)Bp, 128, 0, st>>>(queries, B, db->dim, db->dp, db->vmax, db->q16, db->two_delta,
                                                db->blas.on, nullptr, nullptr);
  CKL();
  // enough (split, query) blocks for 4 per SM; splits of >= 2048 rows
  // batches: blocks of 8 queries (k <= 640: 1024-entry buffers) or 4 (2048-entry
  // buffers) read each DB row once per block; the buffers hold k + a round of rows
  const bool mq8 = B >= 8 && k <= 640;
  const bool mq = mq8 || B >= 4;
  const int QB = mq8 ? 8 : 4;
  const int64_t qblocks = mq ? (B + QB - 1) / QB : B;
  // enough (split, query block) blocks for 4 per SM; splits of >= 2048 rows
  const int splits = (int)std::max<int64_t>(1, std::min<int64_t>((4 * sm_count_pred() + qblocks - 1) / qblocks,
                                                                  (db->size + 2047) / 2048));
  const size_t ent = (size_t)B * splits * BIGK_BUF;
  char* ws = nullptr;
  const size_t wbytes = ent * 8 + (size_t)B * splits * 8 + 256;
  static bool pool_kept = false;  // keep freed workspace reserved in the pool (no re-map per call)
  if (!pool_kept) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    pool_kept = true;
  }
  CK(cudaMallocAsync(reinterpret_cast<void**>(&ws), wbytes, st));
  float* es = reinterpret_cast<float*>(ws);
  int32_t* er = reinterpret_cast<int32_t*>(ws + ent * 4);
  int32_t* en = reinterpret_cast<int32_t*>(ws + ent * 8);
  float* ek = reinterpret_cast<float*>(ws + ent * 8 + (size_t)B * splits * 4);
  int32_t* ovf = reinterpret_cast<int32_t*>(ws + ent * 8 + (size_t)B * splits * 8);
  CK(cudaMemsetAsync(ovf, 0, sizeof(int32_t), st));
  const int mq_smem = (int)(QB * (mq8 ? 1024 : 2048) * 8 + QB * db->dp * 2);
  static int mq_set8 = 0, mq_set4 = 0;
  if (mq8 && mq_smem > mq_set8) {
    CK(cudaFuncSetAttribute(k_bigk_scan_mq<8, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, mq_smem));
    mq_set8 = mq_smem;
  } else if (mq && !mq8 && mq_smem > mq_set4) {
    CK(cudaFuncSetAttribute(k_bigk_scan_mq<4, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, mq_smem));
    mq_set4 = mq_smem;
  }
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(k_bigk_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, BIGK_BUF * 8));
    CK(cudaFuncSetAttribute(k_bigk_select<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, BIGK_BUF * 24));
    CK(cudaFuncSetAttribute(k_bigk_select<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, BIGK_BUF * 24));
    attr = true;
  }
  if (mq8)
    k_bigk_scan_mq<8, 1024><<<dim3((unsigned)splits, (unsigned)qblocks), 256, mq_smem, st>>>(
        db->size, db->dp, k, splits, B, db->v16, db->q16, db->two_delta, es, er, en, ek);
  else if (mq)
    k_bigk_scan_mq<4, 2048><<<dim3((unsigned)splits, (unsigned)qblocks), 256, mq_smem, st>>>(
        db->size, db->dp, k, splits, B, db->v16, db->q16, db->two_delta, es, er, en, ek);
  else
    k_bigk_scan<<<dim3((unsigned)splits, (unsigned)B), 256, BIGK_BUF * 8, st>>>(db->size, db->dp, k, splits, db->v16,
                                                                                db->q16, db->two_delta, es, er, en, ek);
  CKL();
  const BlasRef br = blas_ref(db);
  k_bigk_select<T><<<(unsigned)B, 256, BIGK_BUF * 24, st>>>(
      db->size, db->dim, k, splits, queries, static_cast<const T*>(db->vm), db->lens, db->seqs, db->two_delta, es, er,
      en, ek, out_sim, out_seq, out_len, out_count, ovf, db->inexact, br);
  CKL();
  int32_t h_ovf = 0;
  CK(cudaMemcpyAsync(&h_ovf, ovf, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaFreeAsync(ws, st));
  CK(cudaStreamSynchronize(st));
  if (h_ovf) return fail(ALISE_ECAPACITY, "top-%d search: more than %d near-tied candidates for a query", k, BIGK_BUF);
  return ALISE_OK;
}

static int topk_bigk(alise_db* db, const void* queries, int64_t B, int k, double* out_sim, int64_t* out_seq,
                     int32_t* out_len, int32_t* out_count, cudaStream_t st) {
  if (db->f64)
    return topk_bigk_t(db, static_cast<const double*>(queries), B, k, out_sim, out_seq, out_len, out_count, st);
  return topk_bigk_t(db, static_cast<const float*>(queries), B, k, out_sim, out_seq, out_len, out_count, st);
}

extern "C" int alise_db_topk(alise_db* db, const void* queries, int64_t B, int k, double* out_sim,
                             int64_t* out_seq, int32_t* out_len, int32_t* out_count, void* stream) {
  NvtxRange nvtx_range("alise_db_topk");
  if (!db || B < 0) return fail(ALISE_EINVAL, "bad topk call");
  if (k < 1 || k > BIGK_MAX) return fail(ALISE_EINVAL, "k must be in [1, %d]", BIGK_MAX);
  cudaStream_t st = S(stream);
  if (B == 0) return ALISE_OK;
  if (db->size == 0) {
    CK(cudaMemsetAsync(out_count, 0, sizeof(int32_t) * B, st));
    return ALISE_OK;
  }
  if (k > KMAX) return topk_bigk(db, queries, B, k, out_sim, out_seq, out_len, out_count, st);
  int s = topk_scan(db, queries, B, k, st);
  if (s) return s;
  return topk_rescore(db, queries, B, k, nullptr, out_sim, out_seq, out_len, out_count, st);
}

extern "C" int alise_db_topk_scan(alise_db* db, const void* queries, int64_t B, int k, float* out_bound,
                                  void* stream) {
  NvtxRange nvtx_range("alise_db_topk_scan");
  if (!db || B < 0 || (B > 0 && !out_bound)) return fail(ALISE_EINVAL, "bad topk scan call");
  if (k < 1 || k > BIGK_MAX) return fail(ALISE_EINVAL, "k must be in [1, %d]", BIGK_MAX);
  cudaStream_t st = S(stream);
  if (B == 0) return ALISE_OK;
  if (db->size == 0 || k > KMAX) {  // large k: no bound exchange (the rescore runs the exact big-k search)
    db->last_B = B;
    db->last_k = k;
    db->last_q = queries;
    k_bounds<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(B, k, nullptr, nullptr, nullptr, out_bound);
    CKL();
    return ALISE_OK;
  }
  int s = topk_scan(db, queries, B, k, st);
  if (s) return s;
  k_bounds<<<(unsigned)((B + 255) / 256), 256, 0, st>>>(B, k, db->last.gkth, db->last.gslot, db->two_delta,
                                                        out_bound);
  CKL();
  return ALISE_OK;
}

extern "C" int alise_db_topk_rescore(alise_db* db, const void* queries, int64_t B, int k, const float* ext_bound,
                                     double* out_sim, int64_t* out_seq, int32_t* out_len, int32_t* out_count,
                                     void* stream) {
  NvtxRange nvtx_range("alise_db_topk_rescore");
  if (!db || B < 0) return fail(ALISE_EINVAL, "bad topk rescore call");
  if (B == 0) return ALISE_OK;  // an empty scan records nothing
  if (B != db->last_B || k != db->last_k || queries != db->last_q)
    return fail(ALISE_EINVAL, "alise_db_topk_rescore must follow alise_db_topk_scan of the same queries");
  cudaStream_t st = S(stream);
  if (db->size == 0) {
    CK(cudaMemsetAsync(out_count, 0, sizeof(int32_t) * B, st));
    return ALISE_OK;
  }
  if (k > KMAX) return topk_bigk(db, queries, B, k, out_sim, out_seq, out_len, out_count, st);
  return topk_rescore(db, queries, B, k, ext_bound, out_sim, out_seq, out_len, out_count, st);
}

extern "C" int alise_db_timing(alise_db* db, int enable) {
  db->timing = enable != 0;
  return ALISE_OK;
}

// Sums the scan kernel time (ms) and algorithmic flops since the last call (synchronises).
extern "C" int alise_db_kernel_stats(alise_db* db, double* scan_ms, int64_t* launches, double* flops) {
  CK(cudaDeviceSynchronize());
  double tot = 0;
  for (size_t i = 0; i + 1 < db->ev.size(); i += 2) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, db->ev[i], db->ev[i + 1]));
    tot += ms;
  }
  *scan_ms = tot;
  *launches = (int64_t)(db->ev.size() / 2);
  *flops = db->scan_flops;
  for (auto e : db->ev) cudaEventDestroy(e);
  db->ev.clear();
  db->scan_flops = 0.0;
  return ALISE_OK;
}

extern "C" int alise_topk_merge(int G, int64_t B, int k, const double* sims, const int64_t* seqs,
                                const int32_t* lens, const int32_t* counts, double* out_sim, int64_t* out_seq,
                                int32_t* out_len, int32_t* out_count, void* stream) {
  NvtxRange nvtx_range("alise_topk_merge");
  if (G < 1 || G > 64 || k < 1 || k > BIGK_MAX) return fail(ALISE_EINVAL, "bad merge arguments");
  if (B == 0) return ALISE_OK;
  k_topk_merge<<<(unsigned)((B + 127) / 128), 128, 0, S(stream)>>>(G, B, k, sims, seqs, lens, counts, out_sim,
                                                                     out_seq, out_len, out_count);
  CKL();
  return ALISE_OK;
}

template <typename X>
static int predict_finish_t(int64_t B, int k, const double* sims, const int32_t* lens, const int32_t* counts, double s0,
                            const X* queries, int64_t dim, const double* W1, const double* b1, const double* w2,
                            double b2, int64_t hidden, int64_t max_len, double log_cap, int32_t* out_len,
                            uint8_t* out_retrieved, cudaStream_t st) {
  const int64_t threads = B * 32;
  // shared-memory staging of W1 + the block's 8 queries (fits for the C4 shape 768 x 32)
  const int64_t smem = dim * hidden * 8 + 8 * dim * (int64_t)sizeof(X);
  const bool stage = smem <= 220 * 1024;
  static int64_t smem_set = 0;
  if (stage && smem > smem_set) {
    CK(cudaFuncSetAttribute(k_finish<X>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    smem_set = smem;
  }
  k_finish<X><<<(unsigned)((threads + 255) / 256), 256, stage ? (size_t)smem : 0, st>>>(
      B, k, sims, lens, counts, s0, queries, dim, W1, b1, w2, b2, hidden, max_len, log_cap, out_len, out_retrieved,
      stage);
  CKL();
  return ALISE_OK;
}

extern "C" int alise_predict_finish_ex(int64_t B, int k, const double* sims, const int32_t* lens,
                                       const int32_t* counts, double s0, const void* queries, int queries_dtype,
                                       int64_t dim, const double* W1, const double* b1, const double* w2, double b2,
                                       int64_t hidden, int64_t max_len, double log_cap, int32_t* out_len,
                                       uint8_t* out_retrieved, void* stream) {
  NvtxRange nvtx_range("alise_predict_finish_ex");
  if (k < 1 || k > BIGK_MAX) return fail(ALISE_EINVAL, "k must be in [1, %d]", BIGK_MAX);
  if (hidden < 1) return fail(ALISE_EINVAL, "hidden must be >= 1");
  if (queries_dtype != ALISE_DB_F32 && queries_dtype != ALISE_DB_F64) return fail(ALISE_EINVAL, "bad query dtype");
  if (B == 0) return ALISE_OK;
  if (queries_dtype == ALISE_DB_F64)
    return predict_finish_t(B, k, sims, lens, counts, s0, static_cast<const double*>(queries), dim, W1, b1, w2, b2,
                            hidden, max_len, log_cap, out_len, out_retrieved, S(stream));
  return predict_finish_t(B, k, sims, lens, counts, s0, static_cast<const float*>(queries), dim, W1, b1, w2, b2,
                          hidden, max_len, log_cap, out_len, out_retrieved, S(stream));
}

extern "C" int alise_predict_finish(int64_t B, int k, const double* sims, const int32_t* lens,
                                    const int32_t* counts, double s0, const float* queries, int64_t dim,
                                    const double* W1, const double* b1, const double* w2, double b2,
                                    int64_t hidden, int64_t max_len, double log_cap, int32_t* out_len,
                                    uint8_t* out_retrieved, void* stream) {
  return alise_predict_finish_ex(B, k, sims, lens, counts, s0, queries, ALISE_DB_F32, dim, W1, b1, w2, b2, hidden,
                                 max_len, log_cap, out_len, out_retrieved, stream);
}

extern "C" int alise_embed_batch(const int64_t* tokens, const int64_t* offsets, int64_t B, int64_t dim,
                                 double* out_f64, float* out_f32, void* stream) {
  if (dim < 1 || dim > 8192) return fail(ALISE_EINVAL, "dimension must be in [1, 8192]");
  if (B == 0) return ALISE_OK;
  alise::emb::k_embed<<<(unsigned)B, 256, dim * sizeof(int), S(stream)>>>(tokens, offsets, dim, out_f64, out_f32);
  CKL();
  return ALISE_OK;
}
