// C ABI for the KV data plane: drop-in quantize/dequantize, whole-job KV
// quantize/dequantize, and the swapper that fuses them with host-link transfers.
// Declarations and reference citations: include/alise_b200.h.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <ctype.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <map>
#include <mutex>
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
#include "kv_quant.cuh"

namespace alise {
thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}
}  // namespace alise

using namespace alise;

#define CK(call)                                                                        \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) return fail(ALISE_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define CKL()                                                                           \
  do {                                                                                  \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess) return fail(ALISE_ECUDA, "launch: %s", cudaGetErrorString(e_)); \
  } while (0)

static inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t(255); }
static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int g_sm_count = 0;
static int sm_count() {
  if (!g_sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  return g_sm_count;
}
static inline int grid_for(int64_t work, int block, int waves = 8) {
  int64_t g = (work + block - 1) / block;
  int64_t cap = (int64_t)sm_count() * waves;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

// Segs for `per` work units per segment (per < 2^32): m = ceil(2^64 / per)
static Segs make_segs(int64_t per, int64_t stride) {
  Segs g{0, per, stride};
  if (per > 1) g.m = (uint64_t)(((unsigned __int128)1 << 64) / (uint64_t)per) + 1;
  return g;
}

extern "C" const char* alise_last_error(void) { return g_last_error.c_str(); }
extern "C" int alise_version(void) { return 1; }
extern "C" int alise_sm_count(int device, int* out) {
  CK(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device));
  return ALISE_OK;
}

__global__ void k_selftest_qdiv(const double* __restrict__ x, int64_t n, double b,
                                unsigned long long* __restrict__ bad) {
  const QDiv dq = qdiv_make(b);
  unsigned long long cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double f = qdiv(x[i], dq), r = __ddiv_rn(x[i], b);
    cnt += (__double_as_longlong(f) != __double_as_longlong(r)) ? 1 : 0;
  }
  if (cnt) atomicAdd(bad, cnt);
}

extern "C" int alise_selftest_qdiv(const double* x, int64_t n, int bits, int64_t* mismatches, void* stream) {
  if (bits != 4 && bits != 8) return fail(ALISE_EINVAL, "bits must be 4 or 8");
  if (n <= 0) return ALISE_OK;
  k_selftest_qdiv<<<grid_for(n, 256), 256, 0, S(stream)>>>(x, n, (double)((1 << bits) - 1),
                                                         reinterpret_cast<unsigned long long*>(mismatches));
  CKL();
  return ALISE_OK;
}

// ------------------------------------------------------------------ fast tile launch
template <int BITS, bool PACK, bool ZF32, int V, int TP, int WPB, int MINB = 1, int NBUF = 2>
static int launch_tile_v(const uint16_t* x, int64_t rows, int row_len, uint8_t* codes, double* scale,
                         void* zero, uint32_t* mm, int* flag, cudaStream_t st, int64_t seg_rows,
                         int64_t seg_stride, int sym) {
  constexpr int block = 32 * WPB;
  Segs seg{0, 0, 0};
  if (seg_rows) {
    // segmented sources (token-range transfers): full-width rows, whole rows per segment,
    // and every tile full (a partial tile takes the contiguous path)
    if (rows % seg_rows != 0) return fail(ALISE_EINVAL, "segmented quantize: rows must be whole segments");
    seg = make_segs(seg_rows, seg_stride);
  }
  constexpr int smem = WPB * NBUF * (8 * TP) * (64 * V + 16);
  auto kern = k_quant_tile<BITS, PACK, V, ZF32, TP, WPB, MINB, NBUF>;
  static int per_sm = 0;
  if (!per_sm) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, smem));
    per_sm = std::max(1, per_sm);
  }
  const int64_t warps = (rows + 8 * TP - 1) / (8 * TP);
  const int grid = grid_for(warps * 32, block, per_sm);
  kern<<<grid, block, smem, st>>>(x, rows, row_len, codes, scale, zero, mm, flag, seg, sym);
  CKL();
  return ALISE_OK;
}

// Tile shape per row length (V = 16-byte vectors per lane per row; TP passes of 8 rows
// per warp tile; WPB warps per CTA; MINB = register cap via min CTAs per SM; QT1 = one
// smem slot per warp).  Measured: 32-row single-buffered tiles (every lane busy in the
// float64 solve, 24 warps/SM) beat 16-row double-buffered ones by 10-13%.
// ALISE_QTILE selects tuning variants (tools/kv_kernel_bench.py sweeps them).
static int qtile_variant() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ALISE_QTILE");
    v = e ? atoi(e) : 0;
  }
  return v;
}

template <int BITS, bool PACK, bool ZF32>
static int launch_tile_bits(const uint16_t* x, int64_t rows, int row_len, uint8_t* codes,
                            double* scale, void* zero, uint32_t* mm, int* flag, cudaStream_t st,
                            int64_t seg_rows, int64_t seg_stride, int sym) {
  const int vpl = (row_len / 8 + 3) / 4;  // 16-byte vectors per lane per row
  const int var = qtile_variant();
#define QT(V, TP, WPB, MINB) return launch_tile_v<BITS, PACK, ZF32, V, TP, WPB, MINB>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym)
#define QT1(V, TP, WPB, MINB) return launch_tile_v<BITS, PACK, ZF32, V, TP, WPB, MINB, 1>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym)
  if (vpl <= 1) QT(1, 4, 8, 3);
  if (vpl <= 2) {
    if (var == 1) QT(2, 2, 8, 4);
    if (var == 2) QT(2, 4, 4, 6);
    if (var == 3) QT(2, 2, 8, 3);
    if (var == 4) QT1(2, 4, 8, 3);
    if (var == 5) QT(2, 4, 8, 3);
    QT1(2, 4, 8, 4);
  }
  if (vpl <= 4) {
    if (var == 1) QT(4, 2, 8, 4);
    if (var == 2) QT(4, 2, 8, 3);
    if (var == 3) QT(4, 1, 8, 4);
    if (var == 4) QT1(4, 4, 8, 3);
    if (var == 5) QT(4, 2, 4, 6);
    QT1(4, 4, 4, 6);
  }
  if (vpl <= 8) QT(8, 2, 4, 3);
#undef QT
#undef QT1
  return fail(ALISE_EINVAL, "row_len %d too long for the tile kernel", row_len);
}

static int launch_tile(int bits, bool pack, bool zf32, const uint16_t* x, int64_t rows,
                       int row_len, uint8_t* codes, double* scale, void* zero, int* flag,
                       cudaStream_t st, int64_t seg_rows = 0, int64_t seg_stride = 0, uint32_t* mm = nullptr,
                       int sym = 0) {
  if (bits == 8) {
    return zf32 ? launch_tile_bits<8, false, true>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym)
                : launch_tile_bits<8, false, false>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym);
  }
  if (pack)
    return zf32 ? launch_tile_bits<4, true, true>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym)
                : launch_tile_bits<4, true, false>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym);
  return zf32 ? launch_tile_bits<4, false, true>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym)
              : launch_tile_bits<4, false, false>(x, rows, row_len, codes, scale, zero, mm, flag, st, seg_rows, seg_stride, sym);
}

static bool tile_ok(int dtype, int64_t row_len, int64_t row_stride, const void* src,
                    const void* codes, bool pack) {
  if (dtype != ALISE_DT_F16 || row_len % 8 || row_len > 256 || row_stride != row_len) return false;
  if (((uintptr_t)src & 15) || ((uintptr_t)codes & (pack ? 3 : 7))) return false;
  return true;
}

// ------------------------------------------------------------------ generic rows path
static int64_t rows_chunk(int64_t row_len) { return row_len <= 16384 ? row_len : 16384; }

extern "C" int alise_quantize_rows_workspace(int64_t rows, int64_t row_len, int src_dtype,
                                             int64_t* bytes) {
  if (rows <= 0 || row_len <= 0) return fail(ALISE_EINVAL, "expected a non-empty channel-major 2D tensor");
  const int64_t ch = rows_chunk(row_len);
  const int64_t nch = (row_len + ch - 1) / ch;
  *bytes = align256(rows * nch * 8) * 2 + align256(rows * 16);
  (void)src_dtype;
  return ALISE_OK;
}

template <typename T>
static int rows_generic(const T* x, int64_t rows, int64_t row_len, int64_t row_stride, int bits,
                        bool pack, uint8_t* codes, double* scale, void* zero, bool zf32,
                        int* flag, void* ws, cudaStream_t st, int sym) {
  const int64_t ch = rows_chunk(row_len);
  const int nch = (int)((row_len + ch - 1) / ch);
  char* w = reinterpret_cast<char*>(ws);
  double* pmn = reinterpret_cast<double*>(w);
  double* pmx = reinterpret_cast<double*>(w + align256(rows * nch * 8));
  float4* fastp = reinterpret_cast<float4*>(w + 2 * align256(rows * nch * 8));
  const int64_t blocks = rows * nch;
  if (blocks > 0x7fffffff) return fail(ALISE_EINVAL, "too many rows");
  const int bt = row_len >= 4096 ? 256 : (row_len >= 1024 ? 128 : 32);
  k_minmax_rows<T><<<(unsigned)blocks, bt, 0, st>>>(x, rows, row_len, row_stride, ch, nch, pmn, pmx, flag);
  CKL();
  k_params<false><<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(
      KIND_ROWS, rows, nch, pmn, pmx, nullptr, nullptr, 0, 1, bits, InTraits<T>::wide, scale,
      zero, fastp, nullptr, sym);
  CKL();
  (void)zf32;
  const int64_t n = rows * row_len;
  const int grid = grid_for(pack ? (n + 1) / 2 : n, 256, 16);
  if (bits == 8)
    k_codes_rows<T, 8, false><<<grid, 256, 0, st>>>(x, rows, row_len, row_stride, fastp, scale, zero, false, codes);
  else if (pack)
    k_codes_rows<T, 4, true><<<grid, 256, 0, st>>>(x, rows, row_len, row_stride, fastp, scale, zero, false, codes);
  else
    k_codes_rows<T, 4, false><<<grid, 256, 0, st>>>(x, rows, row_len, row_stride, fastp, scale, zero, false, codes);
  CKL();
  return ALISE_OK;
}

extern "C" int alise_quantize_rows_ex(const void* src, int src_dtype, int64_t rows, int64_t row_len,
                                      int64_t row_stride, int bits, int mode, uint8_t* codes, double* scale,
                                      double* zero, int* flag, void* workspace, void* stream) {
  if (bits != 4 && bits != 8) return fail(ALISE_EINVAL, "bits must be 4 or 8");
  if (mode != ALISE_QMODE_ASYM && mode != ALISE_QMODE_ABSMAX) return fail(ALISE_EINVAL, "unknown quantization mode");
  if (rows <= 0 || row_len <= 0) return fail(ALISE_EINVAL, "expected a non-empty channel-major 2D tensor");
  if (row_stride < row_len) return fail(ALISE_EINVAL, "row_stride < row_len");
  cudaStream_t st = S(stream);
  if (tile_ok(src_dtype, row_len, row_stride, src, codes, false))
    return launch_tile(bits, false, false, reinterpret_cast<const uint16_t*>(src), rows,
                       (int)row_len, codes, scale, zero, flag, st, 0, 0, nullptr, mode);
  if (!workspace) return fail(ALISE_EINVAL, "workspace required for this shape");
  switch (src_dtype) {
    case ALISE_DT_F16:
      return rows_generic(reinterpret_cast<const uint16_t*>(src), rows, row_len, row_stride, bits,
                          false, codes, scale, zero, false, flag, workspace, st, mode);
    case ALISE_DT_F32:
      return rows_generic(reinterpret_cast<const float*>(src), rows, row_len, row_stride, bits,
                          false, codes, scale, zero, false, flag, workspace, st, mode);
    case ALISE_DT_F64:
      return rows_generic(reinterpret_cast<const double*>(src), rows, row_len, row_stride, bits,
                          false, codes, scale, zero, false, flag, workspace, st, mode);
  }
  return fail(ALISE_EINVAL, "unknown dtype %d", src_dtype);
}

extern "C" int alise_quantize_rows(const void* src, int src_dtype, int64_t rows, int64_t row_len,
                                   int64_t row_stride, int bits, uint8_t* codes, double* scale,
                                   double* zero, int* flag, void* workspace, void* stream) {
  return alise_quantize_rows_ex(src, src_dtype, rows, row_len, row_stride, bits, ALISE_QMODE_ASYM, codes, scale,
                                zero, flag, workspace, stream);
}

template <int BITS, bool PACK, bool ZF32>
static int launch_dequant_tile(const uint8_t* codes, const double* scale, const void* zero,
                               int64_t n, int row_len, uint16_t* out, cudaStream_t st, int64_t seg_vals,
                               int64_t seg_stride) {
  constexpr int VALS = PACK ? 32 : 16;
  const int64_t cpr = row_len / VALS;
  const bool wide = row_len % VALS == 0 && !((uintptr_t)codes & 15) && n / VALS < (int64_t(1) << 31) &&
                    cpr < 512 && getenv("ALISE_DQ_NARROW") == nullptr;
  Segs seg{0, 0, 0};
  if (seg_vals) {
    // segmented destination (token-range upload): whole 16-byte code words per segment
    if (!wide || seg_vals % VALS || seg_stride % 8 || n % seg_vals)
      return fail(ALISE_EINVAL, "segmented dequantize needs whole %d-value code words per segment", VALS);
    seg = make_segs(seg_vals / VALS, seg_stride / 8);
  }
  if (wide) {
    const uint32_t nchunks = (uint32_t)(n / VALS);
    const int shift = (cpr & (cpr - 1)) ? -1 : __builtin_ctzll((unsigned long long)cpr);
    const uint64_t recip = ((uint64_t(1) << 40) + cpr - 1) / cpr;
    // one 16-byte code word per thread, no grid-stride loop: CTAs retire continuously, so a
    // concurrent higher-priority quantize launch gets SMs as soon as it is queued
    const int grid = (int)((nchunks + 255) / 256);
    k_dequant_wide<BITS, PACK, ZF32><<<grid, 256, 0, st>>>(reinterpret_cast<const uint4*>(codes), scale, zero,
                                                           nchunks, shift, recip, reinterpret_cast<uint4*>(out), seg);
    CKL();
    return ALISE_OK;
  }
  const int grid = grid_for(n / 8, 256, 8);
  k_dequant_tile<BITS, PACK, ZF32><<<grid, 256, 0, st>>>(codes, scale, zero, n, row_len, out);
  CKL();
  return ALISE_OK;
}

template <typename OUT>
static int dequant_launch(int kind, const uint8_t* codes, const double* scale, const void* zero,
                          bool zf32, int64_t n, int64_t row_len, int64_t T, int64_t Hd, int64_t D,
                          int bits, bool pack, OUT* out, cudaStream_t st, int64_t seg_vals = 0,
                          int64_t seg_stride = 0) {
  const int64_t nv = n / 8;
  if constexpr (sizeof(OUT) == 2) {
    if (kind == KIND_ROWS && row_len % 8 == 0 && row_len <= (1 << 30) && !((uintptr_t)out & 15)) {
#define DQT(B, P, Z) launch_dequant_tile<B, P, Z>(codes, scale, zero, n, (int)row_len, out, st, seg_vals, seg_stride)
      if (bits == 8) return zf32 ? DQT(8, false, true) : DQT(8, false, false);
      if (pack) return zf32 ? DQT(4, true, true) : DQT(4, true, false);
      return zf32 ? DQT(4, false, true) : DQT(4, false, false);
#undef DQT
    }
  }
  if (seg_vals) return fail(ALISE_EINVAL, "segmented dequantize: rows kind, fp16, 16-byte aligned only");
  if (nv > 0) {
    const int grid = grid_for(nv, 256, 16);
#define DQ(B, P) k_dequant<OUT, B, P><<<grid, 256, 0, st>>>(kind, codes, scale, zero, zf32, nv * 8, row_len, T, Hd, D, out)
    if (bits == 8) DQ(8, false);
    else if (pack) DQ(4, true);
    else DQ(4, false);
#undef DQ
    CKL();
  }
  if (n % 8) {
    if (kind != KIND_ROWS) return fail(ALISE_EINVAL, "element count must be a multiple of 8");
    const int64_t e0 = nv * 8;
    if (bits == 8) k_dequant_tail<OUT, 8, false><<<1, 8, 0, st>>>(codes, scale, zero, zf32, e0, n, row_len, out);
    else if (pack) k_dequant_tail<OUT, 4, true><<<1, 8, 0, st>>>(codes, scale, zero, zf32, e0, n, row_len, out);
    else k_dequant_tail<OUT, 4, false><<<1, 8, 0, st>>>(codes, scale, zero, zf32, e0, n, row_len, out);
    CKL();
  }
  return ALISE_OK;
}

extern "C" int alise_dequantize_rows(const uint8_t* codes, const double* scale, const double* zero,
                                     int64_t rows, int64_t row_len, int out_dtype, void* out,
                                     void* stream) {
  if (rows <= 0 || row_len <= 0) return fail(ALISE_EINVAL, "empty tensor");
  // the vector kernel reads codes 8 at a time; unaligned tails go through the scalar kernel
  const int64_t n = rows * row_len;
  if ((uintptr_t)codes & 7) return fail(ALISE_EINVAL, "codes must be 8-byte aligned");
  if (out_dtype == ALISE_DT_F64)
    return dequant_launch<double>(KIND_ROWS, codes, scale, zero, false, n, row_len, 0, 1, 1, 8,
                                  false, reinterpret_cast<double*>(out), S(stream));
  if (out_dtype == ALISE_DT_F16)
    return dequant_launch<uint16_t>(KIND_ROWS, codes, scale, zero, false, n, row_len, 0, 1, 1, 8,
                                    false, reinterpret_cast<uint16_t*>(out), S(stream));
  return fail(ALISE_EINVAL, "out dtype must be f16 or f64");
}
// note: bits only matters for packed codes; the drop-in API never packs.

// ------------------------------------------------------------------ KV job layout
struct KvGeom {
  int64_t planes, plane_elems, rows_pp, code_bytes_pp, ppc, n_chunks, rec_bytes, slab_bytes;
  // chunk record: [codes][fp16 (min, -max) per group]; (scale, zero) are recomputed
  // from (min, max) on upload (k_expand_params), 4 bytes per group instead of 12
  int64_t codes_sec(int64_t np) const { return align256(np * code_bytes_pp); }
  int64_t mm_sec(int64_t np) const { return align256(np * rows_pp * 4); }
  int64_t rec(int64_t np) const { return codes_sec(np) + mm_sec(np); }
  // device scratch for a chunk's expanded (scale f64, zero f32)
  int64_t pws_bytes() const { return align256(ppc * rows_pp * 8) + align256(ppc * rows_pp * 4); }
  int64_t np_of(int64_t c) const { return std::min(ppc, planes - c * ppc); }
};


// Default transfer chunk in MiB of codes (ALISE_CHUNK_MIB, default 512: a whole 1 GiB
// fp16 C2 job at INT8).
static int64_t chunk_mib() {
  static int64_t mib = -1;
  if (mib < 0) {
    const char* e = getenv("ALISE_CHUNK_MIB");
    mib = e ? std::max(1, atoi(e)) : 512;
  }
  return mib;
}

static int geom(const alise_kv_desc* d, KvGeom* g) {
  if (!d || d->layers <= 0 || d->tokens <= 0 || d->hidden <= 0)
    return fail(ALISE_EINVAL, "kv desc: layers/tokens/hidden must be positive");
  if (d->bits != 4 && d->bits != 8) return fail(ALISE_EINVAL, "bits must be 4 or 8");
  if (d->packed && d->bits != 4) return fail(ALISE_EINVAL, "packing is INT4 only");
  if (d->mode != ALISE_QMODE_ASYM && d->mode != ALISE_QMODE_ABSMAX)
    return fail(ALISE_EINVAL, "unknown quantization mode %d", d->mode);
  if (d->hidden % 8) return fail(ALISE_EINVAL, "hidden must be a multiple of 8");
  g->planes = d->layers * 2;
  g->plane_elems = d->tokens * d->hidden;
  switch (d->kind) {
    case ALISE_KIND_ROWS:
      if (d->group <= 0 || d->group % 8 || d->hidden % d->group || d->group > 256)
        return fail(ALISE_EINVAL, "group must be a multiple of 8, <= 256, dividing hidden");
      g->rows_pp = d->tokens * (d->hidden / d->group);
      break;
    case ALISE_KIND_CHANNEL:
      g->rows_pp = d->hidden;
      break;
    case ALISE_KIND_HEAD:
      if (d->head_dim <= 0 || d->hidden % d->head_dim || d->head_dim % 8)
        return fail(ALISE_EINVAL, "head_dim must be a multiple of 8 dividing hidden");
      g->rows_pp = d->hidden / d->head_dim;
      break;
    default:
      return fail(ALISE_EINVAL, "unknown group kind %d", d->kind);
  }
  g->code_bytes_pp = d->packed ? g->plane_elems / 2 : g->plane_elems;
  int64_t ppc = d->planes_per_chunk;
  // default transfer chunk: 512 MiB of codes (a whole 1 GiB fp16 C2 job at INT8).  The
  // host link gates every chunk launch, and a larger launch amortises its ramp on an
  // idle GPU (C2 in-step quantize: 3.2 / 4.2 / 4.8 TB/s at 128 / 256 / 512 MiB); the
  // staging ring holds kSlots chunks per direction
  if (ppc <= 0) ppc = std::max<int64_t>(1, (chunk_mib() << 20) / g->code_bytes_pp);
  g->ppc = std::min(ppc, g->planes);
  g->n_chunks = (g->planes + g->ppc - 1) / g->ppc;
  g->rec_bytes = g->rec(g->ppc);
  g->slab_bytes = (g->n_chunks - 1) * g->rec_bytes + g->rec(g->np_of(g->n_chunks - 1));
  return ALISE_OK;
}

extern "C" int alise_kv_layout(const alise_kv_desc* d, int64_t* slab_bytes, int64_t* rows,
                               int64_t* chunk_bytes, int64_t* n_chunks) {
  KvGeom g{};
  int st = geom(d, &g);
  if (st) return st;
  if (slab_bytes) *slab_bytes = g.slab_bytes;
  if (rows) *rows = g.rows_pp * g.planes;
  if (chunk_bytes) *chunk_bytes = g.rec_bytes;
  if (n_chunks) *n_chunks = g.n_chunks;
  return ALISE_OK;
}

static bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && *e && strcmp(e, "0") != 0;
}

template <int BITS, bool PACK, int CW>
static int launch_cols_cl(dim3 grid, int smem, const uint16_t* kv, const alise_kv_desc* d, int cpr, int64_t rows_pp,
                          int tt, uint8_t* codes, uint32_t* mm, int* flag, cudaStream_t st) {
  auto kern = k_quant_cols_cl<BITS, PACK, CW>;
  static int set = 0;
  if (smem > set) {
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    set = smem;
  }
  kern<<<grid, 2 * CW, smem, st>>>(kv, d->tokens, d->hidden, cpr, rows_pp, tt, codes, mm, flag, d->mode);
  CKL();
  return ALISE_OK;
}

// Quantize path of the column kinds: the strip width of the single-pass cluster kernel
// (64 or 128 columns), 1 for the two-pass k_quant_cols, 0 for the generic three-phase
// path (the only one that needs a workspace).
static int cols_path(const alise_kv_desc* d) {
  const int64_t cpr = d->kind == ALISE_KIND_CHANNEL ? 1 : d->head_dim;
  const int64_t tt = (d->tokens + kColsCL - 1) / kColsCL;
  const int cw = cpr <= 64 && 64 % cpr == 0 ? 64 : 128;  // 128 B token rows unless a head is wider
  if (d->hidden % cw == 0 && cw % cpr == 0 && tt * 2 * cw <= (200 << 10) && !getenv_flag("ALISE_COLS_TWOPASS"))
    return cw;
  if (d->hidden % 128 == 0 && cpr <= 128 && 128 % cpr == 0) return 1;
  return 0;
}

static int64_t cols_workspace(const alise_kv_desc* d, const KvGeom& g, int* nch_out, int64_t* tchunk_out) {
  if (d->kind == ALISE_KIND_ROWS || cols_path(d) != 0) return 0;
  // enough (plane, token-chunk, column-block) blocks for ~4 waves
  const int64_t colblocks = (d->hidden / 8 + 127) / 128;
  int64_t nch = std::max<int64_t>(1, (4 * sm_count() + colblocks * g.ppc - 1) / (colblocks * g.ppc));
  nch = std::min<int64_t>(nch, d->tokens);
  const int64_t tchunk = (d->tokens + nch - 1) / nch;
  nch = (d->tokens + tchunk - 1) / tchunk;
  *nch_out = (int)nch;
  *tchunk_out = tchunk;
  return 2 * align256(g.ppc * nch * d->hidden * 4) + align256(g.ppc * g.rows_pp * 16) + g.pws_bytes();
}

// Quantize np planes starting at kv into one chunk record at rec ([codes][min/max]).
static int quant_chunk(const alise_kv_desc* d, const KvGeom& g, int64_t np, const uint16_t* kv,
                       uint8_t* rec, int* flag, void* ws, cudaStream_t st) {
  uint8_t* codes = rec;
  uint32_t* mm = reinterpret_cast<uint32_t*>(rec + g.codes_sec(np));
  const int64_t rows = np * g.rows_pp;
  if (d->kind == ALISE_KIND_ROWS)
    return launch_tile(d->bits, d->packed != 0, true, kv, rows, d->group, codes, nullptr, nullptr, flag, st,
                       0, 0, mm, d->mode);
  const int cpr = d->kind == ALISE_KIND_CHANNEL ? 1 : (int)d->head_dim;
  const int64_t tt = (d->tokens + kColsCL - 1) / kColsCL;
  const int cw = cols_path(d);
  if (cw > 1 && np <= 65535) {
    // one HBM pass: a cluster of kColsCL CTAs per (plane, cw-column strip)
    dim3 grid((unsigned)(d->hidden / cw), kColsCL, (unsigned)np);
    const int smem = (int)(tt * 2 * cw);
#define QCL(B, P, W) return launch_cols_cl<B, P, W>(grid, smem, kv, d, cpr, g.rows_pp, (int)tt, codes, mm, flag, st)
    if (cw == 64) {
      if (d->bits == 8) QCL(8, false, 64);
      if (d->packed) QCL(4, true, 64);
      QCL(4, false, 64);
    }
    if (d->bits == 8) QCL(8, false, 128);
    if (d->packed) QCL(4, true, 128);
    QCL(4, false, 128);
#undef QCL
  }
  if (d->hidden % 128 == 0 && cpr <= 128 && 128 % cpr == 0) {
    dim3 grid((unsigned)(d->hidden / 128), (unsigned)np);
    if (d->bits == 8) k_quant_cols<8, false><<<grid, 256, 0, st>>>(kv, d->tokens, d->hidden, cpr, g.rows_pp, codes, mm, flag, d->mode);
    else if (d->packed) k_quant_cols<4, true><<<grid, 256, 0, st>>>(kv, d->tokens, d->hidden, cpr, g.rows_pp, codes, mm, flag, d->mode);
    else k_quant_cols<4, false><<<grid, 256, 0, st>>>(kv, d->tokens, d->hidden, cpr, g.rows_pp, codes, mm, flag, d->mode);
    CKL();
    return ALISE_OK;
  }
  int nch;
  int64_t tchunk;
  cols_workspace(d, g, &nch, &tchunk);
  char* w = reinterpret_cast<char*>(ws);
  float* pmn = reinterpret_cast<float*>(w);
  float* pmx = reinterpret_cast<float*>(w + align256(g.ppc * nch * d->hidden * 4));
  float4* fastp = reinterpret_cast<float4*>(w + 2 * align256(g.ppc * nch * d->hidden * 4));
  char* pw = w + 2 * align256(g.ppc * nch * d->hidden * 4) + align256(g.ppc * g.rows_pp * 16);
  double* scale = reinterpret_cast<double*>(pw);
  float* zero = reinterpret_cast<float*>(pw + align256(g.ppc * g.rows_pp * 8));
  dim3 grid((unsigned)((d->hidden / 8 + 127) / 128), (unsigned)nch, (unsigned)np);
  k_minmax_cols<<<grid, 128, 0, st>>>(kv, d->tokens, d->hidden, tchunk, pmn, pmx, flag);
  CKL();
  k_params<true><<<(unsigned)((rows + 127) / 128), 128, 0, st>>>(
      d->kind, rows, nch, nullptr, nullptr, pmn, pmx, d->hidden, d->head_dim > 0 ? d->head_dim : 1,
      d->bits, false, scale, zero, fastp, mm, d->mode);
  CKL();
  const int64_t nvec = np * g.plane_elems / 8;
  const int gr = grid_for(nvec, 256, 16);
  const int64_t D = d->head_dim > 0 ? d->head_dim : 1;
  if (d->bits == 8)
    k_codes_cols<8, false><<<gr, 256, 0, st>>>(kv, d->kind, np, d->tokens, d->hidden, D, fastp, scale, zero, true, codes);
  else if (d->packed)
    k_codes_cols<4, true><<<gr, 256, 0, st>>>(kv, d->kind, np, d->tokens, d->hidden, D, fastp, scale, zero, true, codes);
  else
    k_codes_cols<4, false><<<gr, 256, 0, st>>>(kv, d->kind, np, d->tokens, d->hidden, D, fastp, scale, zero, true, codes);
  CKL();
  return ALISE_OK;
}

// (min, max) of `groups` groups -> (scale, zero) into the scratch pws
static int expand_params(int bits, const uint32_t* mm, int64_t groups, void* pws, int64_t cap_groups,
                         double** scale, float** zero, cudaStream_t st, int sym) {
  char* w = reinterpret_cast<char*>(pws);
  *scale = reinterpret_cast<double*>(w);
  *zero = reinterpret_cast<float*>(w + align256(cap_groups * 8));
  if (groups <= 0) return ALISE_OK;
  const unsigned grid = (unsigned)((groups + 255) / 256);
  if (bits == 8) k_expand_params<8><<<grid, 256, 0, st>>>(mm, groups, *scale, *zero, sym);
  else k_expand_params<4><<<grid, 256, 0, st>>>(mm, groups, *scale, *zero, sym);
  CKL();
  return ALISE_OK;
}

// Dequantize np planes from codes with expanded (scale, zero).
static int dequant_chunk_sz(const alise_kv_desc* d, const KvGeom& g, int64_t np, const uint8_t* codes,
                            const double* scale, const float* zero, uint16_t* kv, cudaStream_t st) {
  const int64_t D = d->head_dim > 0 ? d->head_dim : 1;
  const int cpr = d->kind == ALISE_KIND_CHANNEL ? 1 : (int)D;
  if (d->kind != ALISE_KIND_ROWS && d->hidden % 128 == 0 && cpr <= 128 && 128 % cpr == 0) {
    dim3 grid((unsigned)(d->hidden / 128), (unsigned)np);
    if (d->bits == 8) k_dequant_cols<8, false><<<grid, 256, 0, st>>>(codes, scale, zero, d->tokens, d->hidden, cpr, g.rows_pp, kv);
    else if (d->packed) k_dequant_cols<4, true><<<grid, 256, 0, st>>>(codes, scale, zero, d->tokens, d->hidden, cpr, g.rows_pp, kv);
    else k_dequant_cols<4, false><<<grid, 256, 0, st>>>(codes, scale, zero, d->tokens, d->hidden, cpr, g.rows_pp, kv);
    CKL();
    return ALISE_OK;
  }
  return dequant_launch<uint16_t>(d->kind, codes, scale, zero, true, np * g.plane_elems,
                                  d->kind == ALISE_KIND_ROWS ? d->group : 1, d->tokens, d->hidden,
                                  D, d->bits, d->packed != 0, kv, st);
}

// Expand a chunk record's (min, max) into pws, then dequantize it.
static int dequant_chunk(const alise_kv_desc* d, const KvGeom& g, int64_t np, const uint8_t* rec,
                         uint16_t* kv, void* pws, cudaStream_t st) {
  double* scale;
  float* zero;
  int s = expand_params(d->bits, reinterpret_cast<const uint32_t*>(rec + g.codes_sec(np)), np * g.rows_pp, pws,
                        g.ppc * g.rows_pp, &scale, &zero, st, d->mode);
  if (s) return s;
  return dequant_chunk_sz(d, g, np, rec, scale, zero, kv, st);
}

// Stream-ordered workspace of the one-shot quantize / dequantize calls.  The device's
// default memory pool keeps freed blocks reserved (release threshold = max) so a call
// after a synchronize does not re-map its workspace (100+ MB for a 1 GiB job: ~1 ms).
static int ws_alloc(void** p, int64_t bytes, cudaStream_t st) {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
  CK(cudaMallocAsync(p, bytes, st));
  return ALISE_OK;
}

extern "C" int alise_kv_quantize(const alise_kv_desc* d, const uint16_t* kv, uint8_t* slab,
                                 int* flag, void* stream) {
  NvtxRange nvtx_range("alise_kv_quantize");
  KvGeom g{};
  int s = geom(d, &g);
  if (s) return s;
  cudaStream_t st = S(stream);
  int nch;
  int64_t tchunk;
  const int64_t wsb = cols_workspace(d, g, &nch, &tchunk);
  void* ws = nullptr;
  if (wsb) {
    s = ws_alloc(&ws, wsb, st);
    if (s) return s;
  }
  for (int64_t c = 0; c < g.n_chunks; ++c) {
    s = quant_chunk(d, g, g.np_of(c), kv + c * g.ppc * g.plane_elems, slab + c * g.rec_bytes, flag, ws, st);
    if (s) break;
  }
  if (ws) CK(cudaFreeAsync(ws, st));
  return s;
}

extern "C" int alise_kv_dequantize(const alise_kv_desc* d, const uint8_t* slab, uint16_t* kv,
                                   void* stream) {
  NvtxRange nvtx_range("alise_kv_dequantize");
  KvGeom g{};
  int s = geom(d, &g);
  if (s) return s;
  cudaStream_t st = S(stream);
  void* pws = nullptr;
  s = ws_alloc(&pws, g.pws_bytes(), st);
  if (s) return s;
  for (int64_t c = 0; c < g.n_chunks && !s; ++c)
    s = dequant_chunk(d, g, g.np_of(c), slab + c * g.rec_bytes, kv + c * g.ppc * g.plane_elems, pws, st);
  CK(cudaFreeAsync(pws, st));
  return s;
}

// ------------------------------------------------------------------ swapper
static constexpr int kSlots = 3;
struct alise_swapper {
  int device = 0;
  int mode = ALISE_SWAP_STAGED;
  cudaStream_t s_out = nullptr, s_in = nullptr;
  int64_t slot_bytes = 0;
  uint8_t* ring_out[kSlots] = {};
  uint8_t* ring_in[kSlots] = {};
  cudaEvent_t out_ready[kSlots] = {}, out_free[kSlots] = {}, in_ready[kSlots] = {}, in_free[kSlots] = {};
  int next_out = 0, next_in = 0;
  void* ws = nullptr;
  int64_t ws_bytes = 0;
  uint8_t* pws[kSlots] = {};  // per upload slot: the chunk's expanded (scale, zero)
  int64_t pws_bytes = 0;
  // optional per-chunk kernel timing (bench roofline): event pairs around each
  // quantize / dequantize chunk on the compute stream
  bool timing = false;
  std::vector<cudaEvent_t> t_q, t_d, pool;
  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
};

static int sw_release_rings(alise_swapper* sw) {
  for (int i = 0; i < kSlots; ++i) {
    if (sw->ring_out[i]) CK(cudaFree(sw->ring_out[i]));
    if (sw->ring_in[i]) CK(cudaFree(sw->ring_in[i]));
    sw->ring_out[i] = sw->ring_in[i] = nullptr;
  }
  sw->slot_bytes = 0;
  return ALISE_OK;
}

// Staging buffers grow geometrically (at least doubling, 2 MiB granularity): a growth
// synchronises the device, so a stream of jobs of increasing size (C5 replay) must not
// trigger one per job.  The doubling stops at 1.5x the default chunk's codes (a chunk
// record is its codes plus at most half as many parameter bytes), so the staged rings
// (2 directions x kSlots) stay within 2 x 3 x 768 MiB of HBM at the 512 MiB default
// unless a single (layer, k|v) plane needs more.
static int64_t grow_to(int64_t need, int64_t have) {
  const int64_t cap = (chunk_mib() << 20) * 3 / 2;
  const int64_t g = std::max(need, std::min(2 * have, cap));
  return (g + (2 << 20) - 1) / (2 << 20) * (2 << 20);
}

static int sw_ensure(alise_swapper* sw, int64_t slot_bytes, int64_t ws_bytes) {
  if (sw->mode == ALISE_SWAP_STAGED && slot_bytes > sw->slot_bytes) {
    slot_bytes = grow_to(slot_bytes, sw->slot_bytes);
    CK(cudaStreamSynchronize(sw->s_out));
    CK(cudaStreamSynchronize(sw->s_in));
    CK(cudaDeviceSynchronize());
    int s = sw_release_rings(sw);
    if (s) return s;
    for (int i = 0; i < kSlots; ++i) {
      CK(cudaMalloc(&sw->ring_out[i], slot_bytes));
      CK(cudaMalloc(&sw->ring_in[i], slot_bytes));
    }
    sw->slot_bytes = slot_bytes;
  }
  if (ws_bytes > sw->ws_bytes) {
    ws_bytes = grow_to(ws_bytes, sw->ws_bytes);
    CK(cudaDeviceSynchronize());
    if (sw->ws) CK(cudaFree(sw->ws));
    CK(cudaMalloc(&sw->ws, ws_bytes));
    sw->ws_bytes = ws_bytes;
  }
  return ALISE_OK;
}

static int sw_ensure_pws(alise_swapper* sw, int64_t bytes) {
  if (bytes <= sw->pws_bytes) return ALISE_OK;
  bytes = grow_to(bytes, sw->pws_bytes);
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < kSlots; ++i) {
    if (sw->pws[i]) CK(cudaFree(sw->pws[i]));
    CK(cudaMalloc(&sw->pws[i], bytes));
  }
  sw->pws_bytes = bytes;
  return ALISE_OK;
}

extern "C" int alise_swapper_create(int device, int mode, int64_t ring_bytes, alise_swapper** out) {
  if (mode != ALISE_SWAP_STAGED && mode != ALISE_SWAP_ZEROCOPY) return fail(ALISE_EINVAL, "bad swap mode");
  CK(cudaSetDevice(device));
  alise_swapper* sw = new alise_swapper();
  sw->device = device;
  sw->mode = mode;
  CK(cudaStreamCreateWithFlags(&sw->s_out, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sw->s_in, cudaStreamNonBlocking));
  for (int i = 0; i < kSlots; ++i) {
    CK(cudaEventCreateWithFlags(&sw->out_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sw->out_free[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sw->in_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sw->in_free[i], cudaEventDisableTiming));
  }
  if (ring_bytes > 0) {
    int s = sw_ensure(sw, ring_bytes / kSlots, 0);
    if (s) return s;
  }
  *out = sw;
  return ALISE_OK;
}

extern "C" int alise_swapper_destroy(alise_swapper* sw) {
  if (!sw) return ALISE_OK;
  CK(cudaDeviceSynchronize());
  sw_release_rings(sw);
  if (sw->ws) cudaFree(sw->ws);
  for (int i = 0; i < kSlots; ++i)
    if (sw->pws[i]) cudaFree(sw->pws[i]);
  for (int i = 0; i < kSlots; ++i) {
    cudaEventDestroy(sw->out_ready[i]);
    cudaEventDestroy(sw->out_free[i]);
    cudaEventDestroy(sw->in_ready[i]);
    cudaEventDestroy(sw->in_free[i]);
  }
  cudaStreamDestroy(sw->s_out);
  cudaStreamDestroy(sw->s_in);
  delete sw;
  return ALISE_OK;
}

#define TSTART(v)                                   \
  if (sw->timing) {                                 \
    cudaEvent_t ev_ = sw->take();                   \
    CK(cudaEventRecord(ev_, st));                   \
    sw->v.push_back(ev_);                           \
  }
#define TSTOP(v) TSTART(v)

// Make both side (copy) streams wait for `event` before any later transfer, e.g. an
// upload that reads a host slab written by an earlier offload.
extern "C" int alise_swapper_depend(alise_swapper* sw, void* event) {
  CK(cudaStreamWaitEvent(sw->s_out, reinterpret_cast<cudaEvent_t>(event), 0));
  CK(cudaStreamWaitEvent(sw->s_in, reinterpret_cast<cudaEvent_t>(event), 0));
  return ALISE_OK;
}

extern "C" int alise_swapper_timing(alise_swapper* sw, int enable) {
  sw->timing = enable != 0;
  return ALISE_OK;
}

// Sums kernel time of the instrumented chunks since the last call (synchronises).
extern "C" int alise_swapper_kernel_stats(alise_swapper* sw, double* quant_ms, int64_t* n_quant,
                                          double* deq_ms, int64_t* n_deq) {
  CK(cudaDeviceSynchronize());
  std::vector<cudaEvent_t>* lists[2] = {&sw->t_q, &sw->t_d};
  double* outs[2] = {quant_ms, deq_ms};
  int64_t* cnts[2] = {n_quant, n_deq};
  for (int k = 0; k < 2; ++k) {
    double tot = 0;
    auto& v = *lists[k];
    for (size_t i = 0; i + 1 < v.size(); i += 2) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, v[i], v[i + 1]));
      tot += ms;
    }
    *outs[k] = tot;
    *cnts[k] = (int64_t)(v.size() / 2);
    for (auto e : v) sw->pool.push_back(e);
    v.clear();
  }
  return ALISE_OK;
}

static int host_dev_ptr(const void* host, void** dev) {
  cudaError_t e = cudaHostGetDevicePointer(dev, const_cast<void*>(host), 0);
  if (e != cudaSuccess) return fail(ALISE_EINVAL, "host slab is not pinned/mapped: %s", cudaGetErrorString(e));
  return ALISE_OK;
}

extern "C" int alise_kv_offload(alise_swapper* sw, const alise_kv_desc* d, const uint16_t* kv,
                                void* host_slab, int* flag, void* stream, void* done_event) {
  NvtxRange nvtx_range("alise_kv_offload");
  if (!sw || !kv || !host_slab) return fail(ALISE_EINVAL, "null argument");
  KvGeom g{};
  int s = geom(d, &g);
  if (s) return s;
  int nch;
  int64_t tchunk;
  const int64_t wsb = cols_workspace(d, g, &nch, &tchunk);
  s = sw_ensure(sw, g.rec_bytes, wsb);
  if (s) return s;
  cudaStream_t st = S(stream);
  uint8_t* host = reinterpret_cast<uint8_t*>(host_slab);
  if (sw->mode == ALISE_SWAP_ZEROCOPY) {
    void* dptr;
    s = host_dev_ptr(host_slab, &dptr);
    if (s) return s;
    for (int64_t c = 0; c < g.n_chunks; ++c) {
      TSTART(t_q);
      s = quant_chunk(d, g, g.np_of(c), kv + c * g.ppc * g.plane_elems,
                      reinterpret_cast<uint8_t*>(dptr) + c * g.rec_bytes, flag, sw->ws, st);
      TSTOP(t_q);
      if (s) return s;
    }
    if (done_event) CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), st));
    return ALISE_OK;
  }
  for (int64_t c = 0; c < g.n_chunks; ++c) {
    const int slot = sw->next_out;
    sw->next_out = (slot + 1) % kSlots;
    const int64_t np = g.np_of(c);
    CK(cudaStreamWaitEvent(st, sw->out_free[slot], 0));
    TSTART(t_q);
    s = quant_chunk(d, g, np, kv + c * g.ppc * g.plane_elems, sw->ring_out[slot], flag, sw->ws, st);
    TSTOP(t_q);
    if (s) return s;
    CK(cudaEventRecord(sw->out_ready[slot], st));
    CK(cudaStreamWaitEvent(sw->s_out, sw->out_ready[slot], 0));
    CK(cudaMemcpyAsync(host + c * g.rec_bytes, sw->ring_out[slot], g.rec(np),
                       cudaMemcpyDeviceToHost, sw->s_out));
    CK(cudaEventRecord(sw->out_free[slot], sw->s_out));
  }
  if (done_event) CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), sw->s_out));
  return ALISE_OK;
}

extern "C" int alise_kv_upload(alise_swapper* sw, const alise_kv_desc* d, const void* host_slab,
                               uint16_t* kv, void* stream, void* done_event) {
  NvtxRange nvtx_range("alise_kv_upload");
  if (!sw || !kv || !host_slab) return fail(ALISE_EINVAL, "null argument");
  KvGeom g{};
  int s = geom(d, &g);
  if (s) return s;
  s = sw_ensure(sw, g.rec_bytes, 0);
  if (s) return s;
  cudaStream_t st = S(stream);
  const uint8_t* host = reinterpret_cast<const uint8_t*>(host_slab);
  if (sw->mode == ALISE_SWAP_ZEROCOPY) {
    void* dptr;
    s = host_dev_ptr(host_slab, &dptr);
    if (s) return s;
    void* pws = nullptr;  // stream-ordered scratch: concurrent zero-copy uploads never share it
    s = ws_alloc(&pws, g.pws_bytes(), st);
    if (s) return s;
    for (int64_t c = 0; c < g.n_chunks && !s; ++c) {
      const uint8_t* rec = reinterpret_cast<const uint8_t*>(dptr) + c * g.rec_bytes;
      double* scale;
      float* zero;
      s = expand_params(d->bits, reinterpret_cast<const uint32_t*>(rec + g.codes_sec(g.np_of(c))),
                        g.np_of(c) * g.rows_pp, pws, g.ppc * g.rows_pp, &scale, &zero, st, d->mode);
      if (s) break;
      TSTART(t_d);
      s = dequant_chunk_sz(d, g, g.np_of(c), rec, scale, zero, kv + c * g.ppc * g.plane_elems, st);
      TSTOP(t_d);
    }
    CK(cudaFreeAsync(pws, st));
    if (s) return s;
    if (done_event) CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), st));
    return ALISE_OK;
  }
  s = sw_ensure_pws(sw, g.pws_bytes());
  if (s) return s;
  for (int64_t c = 0; c < g.n_chunks; ++c) {
    const int slot = sw->next_in;
    sw->next_in = (slot + 1) % kSlots;
    const int64_t np = g.np_of(c);
    CK(cudaStreamWaitEvent(sw->s_in, sw->in_free[slot], 0));
    CK(cudaMemcpyAsync(sw->ring_in[slot], host + c * g.rec_bytes, g.rec(np),
                       cudaMemcpyHostToDevice, sw->s_in));
    CK(cudaEventRecord(sw->in_ready[slot], sw->s_in));
    CK(cudaStreamWaitEvent(st, sw->in_ready[slot], 0));
    double* scale;
    float* zero;
    s = expand_params(d->bits, reinterpret_cast<const uint32_t*>(sw->ring_in[slot] + g.codes_sec(np)),
                      np * g.rows_pp, sw->pws[slot], g.ppc * g.rows_pp, &scale, &zero, st, d->mode);
    if (s) return s;
    TSTART(t_d);
    s = dequant_chunk_sz(d, g, np, sw->ring_in[slot], scale, zero, kv + c * g.ppc * g.plane_elems, st);
    TSTOP(t_d);
    if (s) return s;
    CK(cudaEventRecord(sw->in_free[slot], st));
  }
  if (done_event) CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), st));
  return ALISE_OK;
}

// ------------------------------------------------------------------ token-range transfers
// ROWS kind only (a quantization group never spans tokens, so the codes / params of a
// token range equal that part of a full offload: a re-offload of a job that grew from t0
// to t1 tokens moves only [t0, t1) -- incremental block-wise offload).  The desc's
// `tokens` is the job's token capacity T_cap: HBM kv[L][2][T_cap][hidden] and the host
// slab laid out for T_cap.  Per chunk of planes the range is quantized compactly into a
// ring slot and scattered into the slab with 2D copies (one row per plane).
struct RangeGeom {
  int64_t R;          // quantization rows per plane in the range
  int64_t run_vals;   // values per plane in the range
  int64_t run_codes;  // code bytes per plane in the range
  int64_t c_off, m_off;  // slab offsets of the range inside a plane's codes / (min, max)
  int64_t ring_m(int64_t np) const { return align256(np * run_codes); }
};

static int range_geom(const alise_kv_desc* d, const KvGeom& g, int64_t t0, int64_t t1, RangeGeom* r) {
  if (d->kind != ALISE_KIND_ROWS) return fail(ALISE_EINVAL, "token-range transfers need the rows group kind");
  if (t0 < 0 || t1 > d->tokens || t0 >= t1) return fail(ALISE_EINVAL, "token range [%lld, %lld) outside [0, %lld)",
                                                        (long long)t0, (long long)t1, (long long)d->tokens);
  const int64_t pk = d->packed ? 2 : 1;
  const int64_t rpt = d->hidden / d->group;
  r->R = (t1 - t0) * rpt;
  r->run_vals = (t1 - t0) * d->hidden;
  r->run_codes = r->run_vals / pk;
  r->c_off = t0 * d->hidden / pk;
  r->m_off = t0 * rpt * 4;
  (void)g;
  return ALISE_OK;
}

extern "C" int alise_kv_offload_range(alise_swapper* sw, const alise_kv_desc* d, const uint16_t* kv,
                                      void* host_slab, int64_t t0, int64_t t1, int* flag, void* stream,
                                      void* done_event) {
  NvtxRange nvtx_range("alise_kv_offload_range");
  if (!sw || !kv || !host_slab) return fail(ALISE_EINVAL, "null argument");
  if (sw->mode != ALISE_SWAP_STAGED) return fail(ALISE_EINVAL, "token-range transfers use the staged mode");
  KvGeom g{};
  int s = geom(d, &g);
  if (s) return s;
  RangeGeom rg{};
  s = range_geom(d, g, t0, t1, &rg);
  if (s) return s;
  s = sw_ensure(sw, g.rec_bytes, 0);
  if (s) return s;
  cudaStream_t st = S(stream);
  uint8_t* host = reinterpret_cast<uint8_t*>(host_slab);
  for (int64_t c = 0; c < g.n_chunks; ++c) {
    const int slot = sw->next_out;
    sw->next_out = (slot + 1) % kSlots;
    const int64_t np = g.np_of(c);
    uint8_t* ring = sw->ring_out[slot];
    CK(cudaStreamWaitEvent(st, sw->out_free[slot], 0));
    TSTART(t_q);
    s = launch_tile(d->bits, d->packed != 0, true, kv + c * g.ppc * g.plane_elems + t0 * d->hidden, np * rg.R,
                    d->group, ring, nullptr, nullptr, flag, st, rg.R, g.plane_elems,
                    reinterpret_cast<uint32_t*>(ring + rg.ring_m(np)), d->mode);
    TSTOP(t_q);
    if (s) return s;
    CK(cudaEventRecord(sw->out_ready[slot], st));
    CK(cudaStreamWaitEvent(sw->s_out, sw->out_ready[slot], 0));
    uint8_t* rec = host + c * g.rec_bytes;
    CK(cudaMemcpy2DAsync(rec + rg.c_off, g.code_bytes_pp, ring, rg.run_codes, rg.run_codes, np,
                         cudaMemcpyDeviceToHost, sw->s_out));
    CK(cudaMemcpy2DAsync(rec + g.codes_sec(np) + rg.m_off, g.rows_pp * 4, ring + rg.ring_m(np), rg.R * 4,
                         rg.R * 4, np, cudaMemcpyDeviceToHost, sw->s_out));
    CK(cudaEventRecord(sw->out_free[slot], sw->s_out));
  }
  if (done_event) CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), sw->s_out));
  return ALISE_OK;
}

extern "C" int alise_kv_upload_range(alise_swapper* sw, const alise_kv_desc* d, const void* host_slab,
                                     uint16_t* kv, int64_t t0, int64_t t1, void* stream, void* done_event) {
  NvtxRange nvtx_range("alise_kv_upload_range");
  if (!sw || !kv || !host_slab) return fail(ALISE_EINVAL, "null argument");
  if (sw->mode != ALISE_SWAP_STAGED) return fail(ALISE_EINVAL, "token-range transfers use the staged mode");
  KvGeom g{};
  int s = geom(d, &g);
  if (s) return s;
  RangeGeom rg{};
  s = range_geom(d, g, t0, t1, &rg);
  if (s) return s;
  s = sw_ensure(sw, g.rec_bytes, 0);
  if (s) return s;
  s = sw_ensure_pws(sw, g.pws_bytes());
  if (s) return s;
  cudaStream_t st = S(stream);
  const uint8_t* host = reinterpret_cast<const uint8_t*>(host_slab);
  for (int64_t c = 0; c < g.n_chunks; ++c) {
    const int slot = sw->next_in;
    sw->next_in = (slot + 1) % kSlots;
    const int64_t np = g.np_of(c);
    uint8_t* ring = sw->ring_in[slot];
    const uint8_t* rec = host + c * g.rec_bytes;
    CK(cudaStreamWaitEvent(sw->s_in, sw->in_free[slot], 0));
    CK(cudaMemcpy2DAsync(ring, rg.run_codes, rec + rg.c_off, g.code_bytes_pp, rg.run_codes, np,
                         cudaMemcpyHostToDevice, sw->s_in));
    CK(cudaMemcpy2DAsync(ring + rg.ring_m(np), rg.R * 4, rec + g.codes_sec(np) + rg.m_off, g.rows_pp * 4,
                         rg.R * 4, np, cudaMemcpyHostToDevice, sw->s_in));
    CK(cudaEventRecord(sw->in_ready[slot], sw->s_in));
    CK(cudaStreamWaitEvent(st, sw->in_ready[slot], 0));
    double* rs;
    float* rz;
    s = expand_params(d->bits, reinterpret_cast<const uint32_t*>(ring + rg.ring_m(np)), np * rg.R, sw->pws[slot],
                      g.ppc * g.rows_pp, &rs, &rz, st, d->mode);
    if (s) return s;
    TSTART(t_d);
    uint16_t* dst = kv + c * g.ppc * g.plane_elems + t0 * d->hidden;
    if (rg.run_vals % (d->packed ? 32 : 16) == 0 && rg.run_codes % 16 == 0) {
      s = dequant_launch<uint16_t>(KIND_ROWS, ring, rs, rz, true, np * rg.run_vals, d->group, d->tokens,
                                   d->hidden, 1, d->bits, d->packed != 0, dst, st, rg.run_vals, g.plane_elems);
    } else {  // runs not made of whole 16-byte code words: one launch per plane
      for (int64_t p = 0; p < np && !s; ++p)
        s = dequant_launch<uint16_t>(KIND_ROWS, ring + p * rg.run_codes, rs + p * rg.R, rz + p * rg.R, true,
                                     rg.run_vals, d->group, d->tokens, d->hidden, 1, d->bits, d->packed != 0,
                                     dst + p * g.plane_elems, st);
    }
    TSTOP(t_d);
    if (s) return s;
    CK(cudaEventRecord(sw->in_free[slot], st));
  }
  if (done_event) CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(done_event), st));
  return ALISE_OK;
}

// ------------------------------------------------------------------ host memory, events
extern "C" int alise_host_alloc(int64_t bytes, void** out) {
  CK(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable | cudaHostAllocMapped));
  return ALISE_OK;
}

// NUMA-local pinned slabs: anonymous pages with a preferred-node memory policy
// (mbind(2), no libnuma) and transparent huge pages, then page-locked and mapped for
// the GPU with cudaHostRegister, which faults every page in under that policy.  Where
// the GPU's node is unknown or mbind is refused the slab is plain cudaHostAlloc memory
// (registered 4 KB anonymous pages measured ~7% below it on the host link).
namespace {
std::mutex g_numa_mu;
std::map<void*, size_t> g_numa_allocs;  // registered region -> mapped length
}

extern "C" int alise_gpu_numa_node(int device, int* node) {
  char bus[32] = {0};
  CK(cudaDeviceGetPCIBusId(bus, sizeof bus, device));
  for (char* c = bus; *c; ++c) *c = (char)tolower(*c);
  char path[128];
  snprintf(path, sizeof path, "/sys/bus/pci/devices/%s/numa_node", bus);
  *node = -1;
  if (FILE* f = fopen(path, "r")) {
    if (fscanf(f, "%d", node) != 1) *node = -1;
    fclose(f);
  }
  return ALISE_OK;
}

extern "C" int alise_host_alloc_numa(int64_t bytes, int numa_node, void** out, int* bound) {
  if (bytes <= 0) return fail(ALISE_EINVAL, "bytes must be positive");
  if (numa_node == ALISE_NUMA_CURRENT_GPU) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    int s = alise_gpu_numa_node(dev, &numa_node);
    if (s) return s;
  }
  if (bound) *bound = 0;
  // single-node hosts (no node1) and unknown nodes: nothing to place
  const bool force = getenv_flag("ALISE_HOST_MMAP");  // A/B measurements of the two page kinds
  if (!force && (numa_node < 0 || numa_node >= 1024 || access("/sys/devices/system/node/node1", F_OK) != 0))
    return alise_host_alloc(bytes, out);
  const size_t huge = 2u << 20;
  const size_t len = ((size_t)bytes + huge - 1) & ~(huge - 1);
  void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  if (p == MAP_FAILED) return fail(ALISE_ECAPACITY, "mmap of %zu bytes failed", len);
  unsigned long mask[1024 / (8 * sizeof(unsigned long))] = {0};
  if (numa_node >= 0 && numa_node < 1024)
    mask[numa_node / (8 * sizeof(unsigned long))] |= 1ul << (numa_node % (8 * sizeof(unsigned long)));
  const long MPOL_PREFERRED_ = 1;
  const int ok = numa_node >= 0 && numa_node < 1024 &&
                 syscall(SYS_mbind, p, len, MPOL_PREFERRED_, mask, 1024ul, 0u) == 0;
  if (!ok && !force) {
    munmap(p, len);
    return alise_host_alloc(bytes, out);
  }
  madvise(p, len, MADV_HUGEPAGE);
  const cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterPortable | cudaHostRegisterMapped);
  if (e != cudaSuccess) {
    munmap(p, len);
    return fail(ALISE_ECUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
  }
  {
    std::lock_guard<std::mutex> lk(g_numa_mu);
    g_numa_allocs[p] = len;
  }
  *out = p;
  if (bound) *bound = ok;
  return ALISE_OK;
}

extern "C" int alise_host_free(void* p) {
  size_t len = 0;
  {
    std::lock_guard<std::mutex> lk(g_numa_mu);
    auto it = g_numa_allocs.find(p);
    if (it != g_numa_allocs.end()) {
      len = it->second;
      g_numa_allocs.erase(it);
    }
  }
  if (len) {  // alise_host_alloc_numa region
    CK(cudaHostUnregister(p));
    munmap(p, len);
    return ALISE_OK;
  }
  CK(cudaFreeHost(p));
  return ALISE_OK;
}
extern "C" int alise_event_create(void** ev) {
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  *ev = e;
  return ALISE_OK;
}
extern "C" int alise_event_destroy(void* ev) {
  CK(cudaEventDestroy(reinterpret_cast<cudaEvent_t>(ev)));
  return ALISE_OK;
}
extern "C" int alise_event_record(void* ev, void* stream) {
  CK(cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev), S(stream)));
  return ALISE_OK;
}
extern "C" int alise_event_query(void* ev, int* done) {
  cudaError_t e = cudaEventQuery(reinterpret_cast<cudaEvent_t>(ev));
  if (e == cudaErrorNotReady) { *done = 0; return ALISE_OK; }
  CK(e);
  *done = 1;
  return ALISE_OK;
}
extern "C" int alise_event_sync(void* ev) {
  CK(cudaEventSynchronize(reinterpret_cast<cudaEvent_t>(ev)));
  return ALISE_OK;
}
extern "C" int alise_stream_wait(void* stream, void* ev) {
  CK(cudaStreamWaitEvent(S(stream), reinterpret_cast<cudaEvent_t>(ev), 0));
  return ALISE_OK;
}
extern "C" int alise_event_elapsed_ms(void* a, void* b, float* ms) {
  CK(cudaEventElapsedTime(ms, reinterpret_cast<cudaEvent_t>(a), reinterpret_cast<cudaEvent_t>(b)));
  return ALISE_OK;
}
