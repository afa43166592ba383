// KV quantize / dequantize kernels (sm_100a).
//
// Reference: /root/reference/pkg/src/servesim/kvmanager.py:108-154 (quantize, dequantize).
// The reference quantizes the rows of a 2D "channel-major" float64 view; here
// the same rows are addressed in place inside a job's KV tensor
// kv[layer][k|v][token][hidden] (fp16, HBM), so nothing is transposed.
//
//   kind ROWS    : rows are runs of `row_len` contiguous values (group-wise g along
//                  head_dim / per (token, head); also the drop-in 2D API)
//   kind CHANNEL : rows are (layer, k|v, hidden column) along tokens — the
//                  reference's accounting channel (kvmanager.py:72-75)
//   kind HEAD    : rows are (layer, k|v, head) over tokens x head_dim
//
// Hot path (ROWS, fp16, row_len <= 256): one fused single-pass kernel
// (k_quant_tile) — cp.async double-buffered warp tiles in shared memory,
// half2 min/max + warp shuffles, lane-per-row float64 parameter solve, fp32x2
// codes with a proven exactness window, 64/32-bit coalesced stores.  HBM traffic =
// 2 B read + b/8 B written per element + 4 B per row (transfer slabs: fp16 min/max) or
// 12-16 B per row (drop-in API: float64 scale + zero).
// CHANNEL / HEAD kinds: k_quant_cols_cl, one HBM pass through a thread-block cluster
// (DSMEM combine of per-CTA column min/max); k_quant_cols (two passes) beyond its
// shared-memory reach.
// Other shapes use a three-phase path: partial min/max -> per-row params -> codes.
#include <cuda_fp16.h>
#include <stdint.h>

#include <type_traits>

#include "qmath.cuh"

namespace alise {

enum { KIND_ROWS = 0, KIND_CHANNEL = 1, KIND_HEAD = 2 };
enum { DT_F16 = 0, DT_F32 = 1, DT_F64 = 2 };

template <typename T> struct InTraits;
template <> struct InTraits<uint16_t> {
  static __device__ __forceinline__ double d(uint16_t v) { return (double)h2f(v); }
  static __device__ __forceinline__ bool bad(uint16_t v) { return h_nonfinite(v); }
  static constexpr bool wide = false;
};
template <> struct InTraits<float> {
  static __device__ __forceinline__ double d(float v) { return (double)v; }
  static __device__ __forceinline__ bool bad(float v) { return !isfinite(v); }
  static constexpr bool wide = false;
};
template <> struct InTraits<double> {
  static __device__ __forceinline__ double d(double v) { return v; }
  static __device__ __forceinline__ bool bad(double v) { return !isfinite(v); }
  static constexpr bool wide = true;
};

__device__ __forceinline__ void raise_flag(int* flag, bool bad) {
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Segmented addressing of the full-precision side of a transfer: `per` work units
// (rows / code words) per segment, segment starts `stride` elements apart; per == 0
// means one contiguous run.  A token range [t0, t1) of a layer-major job
// kv[layer][k|v][T_cap][hidden] is one segment per (layer, k|v) plane; the codes and
// parameters stay compact.  m = ceil(2^64 / per): q = umulhi(n, m) is exact for
// n, per < 2^32.
struct Segs {
  uint64_t m;
  int64_t per;
  int64_t stride;
};
__device__ __forceinline__ int64_t seg_of(int64_t n, const Segs& s) {
  return s.per == 1 ? n : (int64_t)__umul64hi((uint64_t)n, s.m);
}

// ---------------------------------------------------------------------------------
// Fused tile kernel: fp16 rows, row_len % 8 == 0, row_len <= 8 * 4 * VPL.
// A warp owns a 32-row tile.  4 lanes per row, 8 rows per pass, 4 passes; lane l
// of a row holds 16-byte vectors l, l+4, l+8, ... (VPL of them) so every load
// instruction covers 8 rows x 64 contiguous bytes.
//   A: NaN-propagating half2 min/max, 2 shuffles per row, gathered so that lane j
//      owns tile row j;
//   B: lane-per-row float64 parameter solve (scale, zero, snap loop) + fast-path
//      constants (qmath.cuh TileParams);
//   C: reload (L1/L2 hit), codes via one fp32x2 FMA + integer decision per value,
//      warp-uniform float64 re-run of the rare values near a rounding boundary.
// HBM traffic: 2 B read + b/8 B written per value + 4 B (slab) / 12-16 B (API) per row.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t f2bits(float f) { return __float_as_uint(f); }

// Pack the low bytes of eight fast-path words (bits = 1.5*2^23 + code, code < 2^BITS)
// into codes: INT8 -> 8 bytes, INT4 -> 4 bytes (low nibble = even element).  Byte
// permutes gather the low bytes; INT4 merges odd codes into the high nibbles.
__device__ __forceinline__ uint32_t gather4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}
// Two codes per byte (low nibble = even element).  The fast path's provisional code
// byte can be 0xFF (rint(t32) = -1 just below a group's minimum, flagged and rewritten
// by the fix-up pass), so each code is masked to its nibble: an unmasked 0xFF in an odd
// element would spill 0xF into the next byte's even element, which the fix-up of the
// flagged byte does not rewrite.
__device__ __forceinline__ uint32_t pack_int4x8(const uint32_t (&c)[8]) {
  const uint32_t even = gather4(c[0], c[2], c[4], c[6]) & 0x0F0F0F0Fu;
  const uint32_t odd = gather4(c[1], c[3], c[5], c[7]) & 0x0F0F0F0Fu;
  return even | (odd << 4);
}

// Each warp double-buffers its tiles in shared memory with cp.async (16-byte LDGSTS,
// rows padded by 16 B so the 4 lanes x 8 rows of a load phase hit distinct banks):
// tile i+1 streams in while tile i is reduced, solved and coded.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 16 : 0;  // zero-fill when out of range
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int BITS, bool PACK, int VPL, bool ZF32, int TP, int WPB, int MINB, int NBUF>
__global__ void __launch_bounds__(32 * WPB, MINB)
k_quant_tile(const uint16_t* __restrict__ x, int64_t rows, int row_len,
                uint8_t* __restrict__ codes, double* __restrict__ scale, void* __restrict__ zero,
                uint32_t* __restrict__ mmx, int* __restrict__ flag, const Segs seg, int sym) {
  // TP = passes of 8 rows per warp tile (TILE = 8 * TP rows; 32 keeps every lane busy
  // in the parameter solve).  A lane stages TP x VPL 16-byte vectors per tile.
  constexpr int PASSES = TP;
  constexpr int TILE = 8 * PASSES;
  constexpr int RL = 32 * VPL;         // row length of a full tile (elements)
  constexpr int ROWB = 64 * VPL + 16;  // padded smem row (bytes): 4 lanes x VPL x 16 B + 16
  constexpr float QMAXF = (float)((1 << BITS) - 1);
  extern __shared__ uint8_t smem_pf[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  // NBUF = 2: each warp double-buffers its tiles; NBUF = 1: one slot per warp, the next
  // tile is loaded after this one is coded (latency hidden by the other warps)
  uint8_t* wbuf = smem_pf + wib * (NBUF * TILE * ROWB);
  const int sub = lane >> 2;
  const int q4 = lane & 3;
  const int nvec = row_len >> 3;
  const bool wide_rows = nvec == 4 * VPL;  // every lane's vectors are in range
  const int64_t warp_global = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ntiles = (rows + TILE - 1) / TILE;
  const QDiv dq = qdiv_make((double)((1 << BITS) - 1));

  auto prefetch = [&](int64_t tile, int slot) {
    if (tile >= ntiles) {  // past the end: an empty group keeps the wait counts uniform
      cp_async_commit();
      return;
    }
    uint8_t* b = wbuf + slot * (TILE * ROWB) + sub * ROWB + q4 * 16;
    if (wide_rows && (tile + 1) * TILE <= rows) {
      // full tile: unpredicated, compile-time offsets (segmented sources: whole tiles
      // per segment, so a tile never straddles two segments)
      if (seg.per) {
        // segmented sources: segments of seg.per rows, seg.stride elements apart
#pragma unroll
        for (int p = 0; p < PASSES; ++p) {
          const int64_t r = tile * TILE + p * 8 + sub;
          const int64_t sg = seg_of(r, seg);
          const uint16_t* g = x + sg * seg.stride + (r - sg * seg.per) * (int64_t)RL + q4 * 8;
#pragma unroll
          for (int i = 0; i < VPL; ++i) cp_async16(b + p * 8 * ROWB + i * 64, g + i * 32, true);
        }
      } else {
        const uint16_t* g = x + (tile * TILE + sub) * (int64_t)RL + q4 * 8;
#pragma unroll
        for (int p = 0; p < PASSES; ++p)
#pragma unroll
          for (int i = 0; i < VPL; ++i) cp_async16(b + p * 8 * ROWB + i * 64, g + p * 8 * RL + i * 32, true);
      }
    } else {
#pragma unroll
      for (int p = 0; p < PASSES; ++p) {
        const int64_t r = tile * TILE + p * 8 + sub;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          const int vv = q4 + 4 * i;
          const bool ok = tile < ntiles && r < rows && vv < nvec;
          int64_t off = r * row_len;
          if (seg.per && ok) {
            const int64_t sg = seg_of(r, seg);
            off = sg * seg.stride + (r - sg * seg.per) * row_len;
          }
          cp_async16(b + p * 8 * ROWB + i * 64, x + (ok ? off + vv * 8 : 0), ok);
        }
      }
    }
    cp_async_commit();
  };

  int slot = 0;
  prefetch(warp_global, 0);
  for (int64_t tile = warp_global; tile < ntiles; tile += nwarps, slot ^= (NBUF - 1)) {
    if (NBUF == 2) {
      prefetch(tile + nwarps, slot ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncwarp();
    const uint8_t* b = wbuf + slot * (TILE * ROWB);
    const int64_t row0 = tile * TILE;
    // full tiles (every row live, every lane's vectors in range) skip all range checks:
    // phases A and C are instantiated twice (FULL: no predicates, compile-time offsets)
    const bool full = wide_rows && (row0 + TILE <= rows);
    // ---------------- A: per-row min / max from shared memory (zero-filled vectors
    // of a partial tile are skipped)
    auto phase_a = [&](auto full_c) -> uint32_t {
      constexpr bool FULL = decltype(full_c)::value;
      uint32_t mine = 0;
#pragma unroll
      for (int p = 0; p < PASSES; ++p) {
        const int rl = p * 8 + sub;
        __half2 lo2 = __half2half2(__ushort_as_half(0x7c00)), hi2 = __half2half2(__ushort_as_half(0xfc00));
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          if (FULL || (row0 + rl < rows && q4 + 4 * i < nvec)) {
            const uint4 d = *reinterpret_cast<const uint4*>(b + rl * ROWB + (q4 + 4 * i) * 16);
            const __half2* h = reinterpret_cast<const __half2*>(&d);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              lo2 = __hmin2_nan(lo2, h[k]);
              hi2 = __hmax2_nan(hi2, h[k]);
            }
          }
        }
        const __half mn = __hmin_nan(__low2half(lo2), __high2half(lo2));
        const __half mx = __hmax_nan(__low2half(hi2), __high2half(hi2));
        __half2 pk = __halves2half2(mn, __hneg(mx));
        uint32_t u = *reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
          uint32_t w = __shfl_xor_sync(0xffffffffu, u, o);
          __half2 c = __hmin2_nan(*reinterpret_cast<__half2*>(&u), *reinterpret_cast<__half2*>(&w));
          u = *reinterpret_cast<uint32_t*>(&c);
        }
        const uint32_t g = __shfl_sync(0xffffffffu, u, (lane & 7) << 2);
        if ((lane >> 3) == p) mine = g;
      }
      return mine;
    };
    const uint32_t mine = full ? phase_a(std::true_type{}) : phase_a(std::false_type{});
    // ---------------- B: lane-per-row parameters (lanes < TILE)
    const int64_t my_row = row0 + lane;
    const bool own = lane < TILE && my_row < rows;
    const __half2 mm = *reinterpret_cast<const __half2*>(&mine);
    float fmn = __low2float(mm), fmx = -__high2float(mm);
    const bool bad = own && !(isfinite(fmn) && isfinite(fmx));
    raise_flag(flag, bad);
    if (!own || bad) { fmn = 0.f; fmx = 0.f; }
    double s_row, z_row;
    const TileParams tp = tile_params_f16(fmn, fmx, dq, s_row, z_row, sym);
    if (own) {
      if (mmx) {  // transfer slabs carry the row's fp16 (min, -max): (scale, zero) follow exactly
        mmx[my_row] = mine;
      } else {
        scale[my_row] = s_row;
        if (ZF32) reinterpret_cast<float*>(zero)[my_row] = (float)z_row;
        else reinterpret_cast<double*>(zero)[my_row] = z_row;
      }
    }
    // ---------------- C: codes from shared memory
    // full tiles (every row live, every lane's vectors in range) take an unpredicated
    // path with compile-time offsets; the code is the low byte / nibble of
    // y = fma(x, inv_s, z + 1.5*2^23), e = fma(x, inv_s, K - y) proves it (qmath.cuh)
    auto phase_c = [&](auto full_c) -> uint32_t {
      constexpr bool FULL = decltype(full_c)::value;
      uint32_t pm = 0;  // flagged passes of this lane: bit p
      // full tiles: one base pointer per tile, compile-time offsets per pass / vector
      uint8_t* cfull = codes + ((uint64_t)((row0 + sub) * (int64_t)RL + q4 * 8) >> (PACK ? 1 : 0));
#pragma unroll
      for (int p = 0; p < PASSES; ++p) {
        const int rl = p * 8 + sub;
        const float inv_s = __shfl_sync(0xffffffffu, tp.inv_s, rl);
        const float zc = __shfl_sync(0xffffffffu, tp.zc, rl);
        const float thr = __shfl_sync(0xffffffffu, tp.thr, rl);
        const int64_t r = row0 + rl;
        const bool live_row = r < rows;
        const float2 inv2 = make_float2(inv_s, inv_s), zc2 = make_float2(zc, zc);
        const float2 nzc2 = make_float2(-zc, -zc);
        const uint8_t* srow = b + rl * ROWB + q4 * 16;
        uint8_t* crow = FULL ? cfull + ((p * 8 * RL) >> (PACK ? 1 : 0))
                             : codes + ((uint64_t)(r * (int64_t)row_len + q4 * 8) >> (PACK ? 1 : 0));
        float dmax = 0.f;  // largest |e| of this lane's values in the pass
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
          if (!FULL && !(live_row && q4 + 4 * i < nvec)) continue;
          const uint4 d = *reinterpret_cast<const uint4*>(srow + i * 64);
          const __half2* h = reinterpret_cast<const __half2*>(&d);
          uint32_t c[8];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __half22float2(h[k]);
            const float2 y = __ffma2_rn(f, inv2, zc2);                    // 1.5*2^23 + code
            const float2 cc = __fadd2_rn(y, nzc2);                        // code - z, exact
            const float2 e = __ffma2_rn(f, inv2, make_float2(-cc.x, -cc.y));  // RN(t32 - code)
            dmax = fmaxf(dmax, fmaxf(fabsf(e.x), fabsf(e.y)));
            c[2 * k] = f2bits(y.x);
            c[2 * k + 1] = f2bits(y.y);
          }
          if (PACK) {
            __stcs(reinterpret_cast<uint32_t*>(crow + i * 16), pack_int4x8(c));
          } else {
            __stcs(reinterpret_cast<uint2*>(crow + i * 32),
                   make_uint2(gather4(c[0], c[1], c[2], c[3]), gather4(c[4], c[5], c[6], c[7])));
          }
        }
        pm |= (dmax >= thr ? 1u : 0u) << p;  // a value of the pass is near a rounding boundary
      }
      return pm;
    };
    const uint32_t pmask = full ? phase_c(std::true_type{}) : phase_c(std::false_type{});
    // ---------------- D: rare fix-up of flagged (lane, pass) pairs (a value near a
    // rounding boundary), all lanes together: the pair's 8*VPL values are spread one code
    // byte per lane (INT8: one value; packed INT4: values 2j, 2j+1); each lane re-checks
    // its value(s) and runs the reference float64 ops where the check fails
    __syncwarp();  // the vector stores above are visible to the whole warp
    uint32_t pending = __ballot_sync(0xffffffffu, pmask != 0);
#pragma unroll 1
    while (pending) {
      const int src = __ffs(pending) - 1;
      pending &= pending - 1;
      uint32_t m = __shfl_sync(0xffffffffu, pmask, src);
#pragma unroll 1
      while (m) {
        const int p = __ffs(m) - 1;
        m &= m - 1;
        const int rl = p * 8 + (src >> 2);
        const float inv_s = __shfl_sync(0xffffffffu, tp.inv_s, rl);
        const float zc = __shfl_sync(0xffffffffu, tp.zc, rl);
        const float thr = __shfl_sync(0xffffffffu, tp.thr, rl);
        const double sd = __shfl_sync(0xffffffffu, s_row, rl);
        const double zd = __shfl_sync(0xffffffffu, z_row, rl);
        constexpr int PER = PACK ? 2 : 1;        // values per code byte
        constexpr int NB = 8 * VPL / PER;        // code bytes of the pair
        const int64_t r = row0 + rl;
#pragma unroll 1
        for (int bi = lane; bi < NB; bi += 32) {
          const int i = (bi * PER) >> 3, j0 = (bi * PER) & 7;
          const int vv = (src & 3) + 4 * i;
          if (r >= rows || vv >= nvec) continue;
          const uint16_t* hv = reinterpret_cast<const uint16_t*>(b + rl * ROWB + vv * 16) + j0;
          uint32_t byte = 0;
          bool fix = false;
#pragma unroll
          for (int u = 0; u < PER; ++u) {
            const float xf = h2f(hv[u]);
            const float y = fmaf(xf, inv_s, zc);
            uint32_t cc = f2bits(y) & ((1u << BITS) - 1);
            if (!(fabsf(fmaf(xf, inv_s, -__fadd_rn(y, -zc))) < thr)) {
              const float rc = (float)rint(__dadd_rn(__ddiv_rn((double)xf, sd), zd));
              cc = (uint32_t)fminf(fmaxf(rc, 0.f), QMAXF);
              fix = true;
            }
            byte |= cc << (4 * u);
          }
          if (fix) codes[(r * row_len + vv * 8 + j0) / PER] = (uint8_t)byte;
        }
      }
    }
    __syncwarp();  // all lanes are done with this slot before it is refilled
    if (NBUF == 1) prefetch(tile + nwarps, 0);
  }
  cp_async_wait<0>();
}

// Fast dequantize of ROWS-kind codes (row_len % 8 == 0) to fp16.  Each thread owns 8
// values of one row.  y = fp32(s) * ((2^23+q) - (2^23+z)) is exact up to two fp32
// roundings; fp16(y) equals fp16(float64 s*(q-z)) unless y is within 4 fp32 ulps of an
// fp16 rounding midpoint or below the fp16 normal range, where the thread re-runs the
// reference float64 product (warp-uniform branch).
template <int BITS, bool PACK, bool ZF32>
__global__ void __launch_bounds__(256)
k_dequant_tile(const uint8_t* __restrict__ codes, const double* __restrict__ scale,
               const void* __restrict__ zero, int64_t n, int row_len, uint16_t* __restrict__ out) {
  const int64_t nvec = n >> 3;
  const int vpr = row_len >> 3;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nvec;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = k / vpr;
    const double s = __ldg(scale + r);
    const double z = ZF32 ? (double)__ldg(reinterpret_cast<const float*>(zero) + r)
                          : __ldg(reinterpret_cast<const double*>(zero) + r);
    const float s32 = (float)s;
    // rows whose products may leave the fp16 normal range take the exact path
    // fast rows: integer zero (so 2^23 + z is exact in fp32) and products in the
    // fp16 normal range; constant rows (real-valued zero) take the exact path
    const bool row_fast = z == rint(z) && fabs(z) < 4194304.0 && s >= 0x1p-14 && s < 60000.0;
    const float zm = (float)(z + 8388608.0);
    uint32_t q[8];
    if (PACK) {
      const uint32_t wd = __ldcs(reinterpret_cast<const uint32_t*>(codes) + k);
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = (wd >> (4 * j)) & 15u;
    } else {
      const uint2 wd = __ldcs(reinterpret_cast<const uint2*>(codes) + k);
#pragma unroll
      for (int j = 0; j < 4; ++j) { q[j] = (wd.x >> (8 * j)) & 255u; q[4 + j] = (wd.y >> (8 * j)) & 255u; }
    }
    uint32_t o[4];
    bool unsafe = !row_fast;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 qf = make_float2(__uint_as_float(0x4B000000u | q[2 * j]), __uint_as_float(0x4B000000u | q[2 * j + 1]));
      const float2 d = __fadd2_rn(qf, make_float2(-zm, -zm));
      const float2 y = __fmul2_rn(d, make_float2(s32, s32));
      const uint32_t b0 = __float_as_uint(y.x), b1 = __float_as_uint(y.y);
      unsafe |= ((b0 + (4u - 0x1000u)) & 0x1fffu) <= 8u;
      unsafe |= ((b1 + (4u - 0x1000u)) & 0x1fffu) <= 8u;
      const __half2 hv = __floats2half2_rn(y.x, y.y);
      o[j] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    if (__any_sync(__activemask(), unsafe) && unsafe) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double v = __dmul_rn(s, __dsub_rn((double)q[j], z));
        const uint32_t hb = __half_as_ushort(__double2half(v));
        const int wi = j >> 1, sh = 16 * (j & 1);
        o[wi] = (o[wi] & ~(0xffffu << sh)) | (hb << sh);
      }
    }
    __stcs(reinterpret_cast<uint4*>(out) + k, make_uint4(o[0], o[1], o[2], o[3]));
  }
}

// Wide dequantize of ROWS-kind codes to fp16: each thread owns one 16-byte word of
// codes (16 INT8 or 32 packed INT4 values, inside one row), so a warp keeps 512 B of
// reads in flight per instruction and the row's (scale, zero) are loaded and checked
// once per 16/32 values.  Row index = chunk / chunks_per_row via shift or a 2^40
// reciprocal (exact for chunk < 2^31, chunks_per_row < 2^9).  Values: y = fp32(s) *
// ((2^23+q) - (2^23+z)) (one product rounding after an exact difference), fp16(y)
// equals fp16(float64 s*(q-z)) unless y's 13 discarded bits are within 4 of the
// fp16 rounding midpoint (checked two values at a time on 16-bit lanes, window 9
// so a carry between the lanes can only widen it) or the row's products may leave
// the fp16 normal range; those vectors re-run the reference float64 product.
template <int BITS, bool PACK, bool ZF32>
__global__ void __launch_bounds__(256)
k_dequant_wide(const uint4* __restrict__ codes, const double* __restrict__ scale,
               const void* __restrict__ zero, uint32_t nchunks, int cpr_shift, uint64_t cpr_recip,
               uint4* __restrict__ out, const Segs seg) {
  constexpr int VALS = PACK ? 32 : 16;  // values per 16-byte chunk
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nchunks; k += gridDim.x * blockDim.x) {
    const uint32_t r = cpr_shift >= 0 ? (k >> cpr_shift) : (uint32_t)(((uint64_t)k * cpr_recip) >> 40);
    const uint4 w = __ldcs(codes + k);
    const double s = __ldg(scale + r);
    float zf;
    double z;
    if (ZF32) {
      zf = __ldg(reinterpret_cast<const float*>(zero) + r);
      z = (double)zf;
    } else {
      z = __ldg(reinterpret_cast<const double*>(zero) + r);
      zf = (float)z;
    }
    const float s32 = (float)s;
    // fast rows: integer zero (2^23 + z exact in fp32) and products in the fp16 normal
    // range (s32 > 2^-14 implies s > 2^-14); constant rows (real-valued zero) go exact
    const bool row_fast = (double)zf == z && zf == rintf(zf) && fabsf(zf) < 4194304.0f &&
                          s32 > 0x1p-14f && s32 < 60000.0f;
    const float zm = zf + 8388608.0f;
    const float2 nz2 = make_float2(-zm, -zm), s2 = make_float2(s32, s32);
    const uint32_t wd[4] = {w.x, w.y, w.z, w.w};
    uint32_t o[VALS / 2];
    uint32_t acc = 0xffffffffu;
#pragma unroll
    for (int p = 0; p < VALS / 2; ++p) {
      // code -> float 2^23 + q with one byte permute: bytes (q, 0, 0, 0x4B)
      uint32_t f0, f1;
      if (PACK) {
        const uint32_t wv = wd[p >> 2];
        const int j = p & 3;
        f0 = __byte_perm(wv & 0x0F0F0F0Fu, 0x4Bu, 0x4550 + j);
        f1 = __byte_perm((wv >> 4) & 0x0F0F0F0Fu, 0x4Bu, 0x4550 + j);
      } else {
        const uint32_t wv = wd[p >> 1];
        const int j = 2 * (p & 1);
        f0 = __byte_perm(wv, 0x4Bu, 0x4550 + j);
        f1 = __byte_perm(wv, 0x4Bu, 0x4551 + j);
      }
      const float2 qf = make_float2(__uint_as_float(f0), __uint_as_float(f1));
      const float2 y = __fmul2_rn(__fadd2_rn(qf, nz2), s2);
      const __half2 hv = __floats2half2_rn(y.x, y.y);
      o[p] = *reinterpret_cast<const uint32_t*>(&hv);
      const uint32_t lo = __byte_perm(__float_as_uint(y.x), __float_as_uint(y.y), 0x5410);
      acc = __vminu2(acc, (lo + 0x10041004u) & 0x1fff1fffu);
    }
    const bool unsafe = !row_fast || (acc & 0xffffu) <= 9u || (acc >> 16) <= 9u;
    if (unsafe) {
#pragma unroll
      for (int j = 0; j < VALS; ++j) {
        const uint32_t q = PACK ? (wd[j >> 3] >> (4 * (j & 7))) & 15u : (wd[j >> 2] >> (8 * (j & 3))) & 255u;
        const double v = __dmul_rn(s, __dsub_rn((double)q, z));
        const uint32_t hb = __half_as_ushort(__double2half(v));
        const int wi = j >> 1, sh = 16 * (j & 1);
        o[wi] = (o[wi] & ~(0xffffu << sh)) | (hb << sh);
      }
    }
    uint4* dst = out + (size_t)k * (VALS / 8);
    if (seg.per) {  // segmented destination (token-range upload); stride in uint4 units
      const int64_t sg = seg_of(k, seg);
      dst = out + sg * seg.stride + (k - sg * seg.per) * (VALS / 8);
    }
#pragma unroll
    for (int c = 0; c < VALS / 8; ++c)
      __stcs(dst + c, make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]));
  }
}

// ---------------------------------------------------------------------------------
// Fused column kernel for the CHANNEL / HEAD kinds (rows run along tokens).
// Block = 256 threads = 16 column vectors (128 columns) x 16 token lanes over one
// plane [T][Hd].  Pass 1: NaN-propagating half2 min/max down the tokens, reduced
// across token lanes in shared memory, then one thread per group (column, or head
// of `cpr` columns) solves the float64 parameters.  Pass 2: the strip is re-read
// (L2) and each thread quantizes its 8 columns with per-column fp32 constants held
// in registers.  Codes stay in native [T][Hd] order.
// ---------------------------------------------------------------------------------
template <int BITS, bool PACK>
__global__ void __launch_bounds__(256, 3)
k_quant_cols(const uint16_t* __restrict__ x, int64_t T, int64_t Hd, int cpr, int64_t rows_per_plane,
             uint8_t* __restrict__ codes, uint32_t* __restrict__ mm, int* __restrict__ flag, int sym) {
  constexpr float QMAXF = (float)((1 << BITS) - 1);
  __shared__ __half2 s_mm[16][128];      // (min, -max) per token lane and column
  __shared__ float s_inv[128], s_zc[128], s_thr[128], s_zd[128];
  __shared__ double s_sd[128];
  const int tid = threadIdx.x;
  const int cv = tid & 15, tl = tid >> 4;
  const int64_t plane = blockIdx.y;
  const int64_t col0 = (int64_t)blockIdx.x * 128;
  const uint16_t* base = x + plane * T * Hd + col0 + cv * 8;
  // ---- pass 1
  __half2 lo[4], hi[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    lo[j] = __half2half2(__ushort_as_half(0x7c00));
    hi[j] = __half2half2(__ushort_as_half(0xfc00));
  }
  auto mm_vec = [&](const uint4 d) {
    const __half2* h = reinterpret_cast<const __half2*>(&d);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      lo[j] = __hmin2_nan(lo[j], h[j]);
      hi[j] = __hmax2_nan(hi[j], h[j]);
    }
  };
  int64_t t1 = tl;
  for (; t1 + 48 < T; t1 += 64) {
    uint4 d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) d[u] = __ldg(reinterpret_cast<const uint4*>(base + (t1 + 16 * u) * Hd));
#pragma unroll
    for (int u = 0; u < 4; ++u) mm_vec(d[u]);
  }
  for (; t1 < T; t1 += 16) mm_vec(__ldg(reinterpret_cast<const uint4*>(base + t1 * Hd)));
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    s_mm[tl][cv * 8 + 2 * j] = __halves2half2(__low2half(lo[j]), __hneg(__low2half(hi[j])));
    s_mm[tl][cv * 8 + 2 * j + 1] = __halves2half2(__high2half(lo[j]), __hneg(__high2half(hi[j])));
  }
  __syncthreads();
  if (tid < 128) {
    __half2 m = s_mm[0][tid];
    for (int u = 1; u < 16; ++u) m = __hmin2_nan(m, s_mm[u][tid]);
    s_mm[0][tid] = m;
  }
  __syncthreads();
  // one thread per group of cpr columns
  const int groups = 128 / cpr;
  if (tid < groups) {
    __half2 m = s_mm[0][tid * cpr];
    for (int u = 1; u < cpr; ++u) m = __hmin2_nan(m, s_mm[0][tid * cpr + u]);
    float fmn = __low2float(m), fmx = -__high2float(m);
    const bool bad = !(isfinite(fmn) && isfinite(fmx));
    if (bad) { atomicOr(flag, 1); fmn = 0.f; fmx = 0.f; }
    double sd, zd;
    const TileParams tp = tile_params_f16(fmn, fmx, qdiv_make((double)((1 << BITS) - 1)), sd, zd, sym);
    const int64_t r = plane * rows_per_plane + (col0 / cpr) + tid;
    mm[r] = *reinterpret_cast<const uint32_t*>(&m);  // the group's fp16 (min, -max)
    for (int u = 0; u < cpr; ++u) {
      s_inv[tid * cpr + u] = tp.inv_s;
      s_zc[tid * cpr + u] = tp.zc;
      s_thr[tid * cpr + u] = tp.thr;
      s_sd[tid * cpr + u] = sd;
      s_zd[tid * cpr + u] = (float)zd;
    }
  }
  __syncthreads();
  // ---- pass 2
  float inv[8], zc[8], thr[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    inv[j] = s_inv[cv * 8 + j];
    zc[j] = s_zc[cv * 8 + j];
    thr[j] = s_thr[cv * 8 + j];
  }
  uint8_t* cbase = codes + (plane * T * Hd + col0 + cv * 8) / (PACK ? 2 : 1);
  auto code_vec = [&](const uint4 d, int64_t t) {
    const __half2* h = reinterpret_cast<const __half2*>(&d);
    uint32_t c[8];
    bool unsafe = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(h[j]);
      const float2 i2 = make_float2(inv[2 * j], inv[2 * j + 1]);
      const float2 y = __ffma2_rn(f, i2, make_float2(zc[2 * j], zc[2 * j + 1]));
      const float2 cc = __fadd2_rn(y, make_float2(-zc[2 * j], -zc[2 * j + 1]));
      const float2 e = __ffma2_rn(f, i2, make_float2(-cc.x, -cc.y));
      unsafe |= !(fabsf(e.x) < thr[2 * j]) || !(fabsf(e.y) < thr[2 * j + 1]);
      c[2 * j] = f2bits(y.x) & ((1u << BITS) - 1);
      c[2 * j + 1] = f2bits(y.y) & ((1u << BITS) - 1);
    }
    if (unsafe) {  // rare: the reference float64 ops for the values near a boundary
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float f = __half2float(reinterpret_cast<const __half*>(&d)[j]);
        const float y = fmaf(f, inv[j], zc[j]);
        if (!(fabsf(fmaf(f, inv[j], -__fadd_rn(y, -zc[j]))) < thr[j])) {
          const double sd = s_sd[cv * 8 + j], zd = (double)s_zd[cv * 8 + j];
          float rr = (float)rint(__dadd_rn(__ddiv_rn((double)f, sd), zd));
          c[j] = (uint32_t)fminf(fmaxf(rr, 0.f), QMAXF);
        }
      }
    }
    if (PACK) {
      __stcs(reinterpret_cast<uint32_t*>(cbase + t * Hd / 2), pack_int4x8(c));
    } else {
      __stcs(reinterpret_cast<uint2*>(cbase + t * Hd),
             make_uint2(gather4(c[0], c[1], c[2], c[3]), gather4(c[4], c[5], c[6], c[7])));
    }
  };
  // four token rows in flight per thread (the loop is load-latency bound otherwise)
  int64_t t = tl;
  for (; t + 48 < T; t += 64) {
    uint4 d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) d[u] = __ldg(reinterpret_cast<const uint4*>(base + (t + 16 * u) * Hd));
#pragma unroll
    for (int u = 0; u < 4; ++u) code_vec(d[u], t + 16 * u);
  }
  for (; t < T; t += 16) code_vec(__ldg(reinterpret_cast<const uint4*>(base + t * Hd)), t);
}

// ---------------------------------------------------------------------------------
// Single-pass column kernel for the CHANNEL / HEAD kinds (k_quant_cols reads every
// strip twice, and its resident 512 KB strips overflow L2, so the second pass comes
// back from HBM).  A cluster of kColsCL CTAs splits one plane's CW-column strip along
// tokens; each CTA stages its TT token rows (2*CW bytes each) in shared memory with
// cp.async, reduces per-column (min, -max) locally, and the cluster combines the
// partials through distributed shared memory (every CTA reads the kColsCL partials of
// its columns, so no second barrier round precedes the float64 solve).  Codes are then
// produced from shared memory: HBM traffic is one read of the fp16 values + the codes +
// 4 B per group.  CW = 64 (channel kind: 128 B token rows, 4 warps) or 128 (head kind,
// one 128-column head per strip).
// ---------------------------------------------------------------------------------
constexpr int kColsCL = 8;

__device__ __forceinline__ uint32_t dsmem_ld_u32(uint32_t cluster_addr) {
  uint32_t v;
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(cluster_addr) : "memory");
  return v;
}

template <int BITS, bool PACK, int CW>
__global__ void __cluster_dims__(1, kColsCL, 1) __launch_bounds__(CW * 2, 768 / (CW * 2))
k_quant_cols_cl(const uint16_t* __restrict__ x, int64_t T, int64_t Hd, int cpr, int64_t rows_per_plane, int TT,
                uint8_t* __restrict__ codes, uint32_t* __restrict__ mm, int* __restrict__ flag, int sym) {
  constexpr int NCV = CW / 8;            // 16-byte column vectors per token row
  constexpr int NW = CW / 16;            // warps (16 token lanes x NCV column vectors)
  constexpr int TPW = 32 / NCV;          // token lanes per warp
  constexpr float QMAXF = (float)((1 << BITS) - 1);
  extern __shared__ uint4 s_tile[];      // [TT][NCV]: TT token rows x CW columns
  __shared__ __half2 s_mm[NW][CW];       // (min, -max) per warp and column
  __shared__ __half2 s_part[CW];         // this CTA's partial per column (read by the cluster)
  __shared__ float s_inv[CW], s_zc[CW], s_thr[CW];
  __shared__ double s_sd[CW], s_zd[CW];
  const int tid = threadIdx.x;
  const int cv = tid % NCV, tl = tid / NCV;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int64_t plane = blockIdx.z;
  const int64_t col0 = (int64_t)blockIdx.x * CW;
  const int64_t t0 = (int64_t)rank * TT;
  const int nt = (int)(T - t0 < TT ? (T - t0 > 0 ? T - t0 : 0) : TT);
  const uint16_t* base = x + (plane * T + t0) * Hd + col0 + cv * 8;
  // ---- stage the token rows: two cp.async groups so the min/max of the first half
  // overlaps the second half's loads
  const int half = min(((nt + 31) / 32) * 16, nt);
#pragma unroll 4
  for (int r = tl; r < half; r += 16) cp_async16(&s_tile[r * NCV + cv], base + (int64_t)r * Hd, true);
  cp_async_commit();
#pragma unroll 4
  for (int r = half + tl; r < nt; r += 16) cp_async16(&s_tile[r * NCV + cv], base + (int64_t)r * Hd, true);
  cp_async_commit();
  __half2 lo[4], hi[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    lo[j] = __half2half2(__ushort_as_half(0x7c00));
    hi[j] = __half2half2(__ushort_as_half(0xfc00));
  }
  auto mm_rows = [&](int r0, int r1) {
#pragma unroll 4
    for (int r = r0 + tl; r < r1; r += 16) {
      const uint4 d = s_tile[r * NCV + cv];
      const __half2* h = reinterpret_cast<const __half2*>(&d);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        lo[j] = __hmin2_nan(lo[j], h[j]);
        hi[j] = __hmax2_nan(hi[j], h[j]);
      }
    }
  };
  cp_async_wait<1>();  // a thread reads back only the vectors it staged itself
  mm_rows(0, half);
  cp_async_wait<0>();
  mm_rows(half, nt);
  // the token lanes of a warp first (shuffles), then the warps (shared memory)
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    __half2 a = __halves2half2(__low2half(lo[j]), __hneg(__low2half(hi[j])));
    __half2 b = __halves2half2(__high2half(lo[j]), __hneg(__high2half(hi[j])));
#pragma unroll
    for (int o = NCV; o < 32; o <<= 1) {
      uint32_t ua = *reinterpret_cast<uint32_t*>(&a), ub = *reinterpret_cast<uint32_t*>(&b);
      uint32_t wa = __shfl_xor_sync(0xffffffffu, ua, o), wb = __shfl_xor_sync(0xffffffffu, ub, o);
      a = __hmin2_nan(a, *reinterpret_cast<__half2*>(&wa));
      b = __hmin2_nan(b, *reinterpret_cast<__half2*>(&wb));
    }
    if (tl % TPW == 0) {
      s_mm[tl / TPW][cv * 8 + 2 * j] = a;
      s_mm[tl / TPW][cv * 8 + 2 * j + 1] = b;
    }
  }
  __syncthreads();
  if (tid < CW) {
    __half2 m = s_mm[0][tid];
#pragma unroll
    for (int u = 1; u < NW; ++u) m = __hmin2_nan(m, s_mm[u][tid]);
    s_part[tid] = m;
  }
  // ---- cluster-wide combine through distributed shared memory
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (tid < CW) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&s_part[tid]));
    uint32_t w[kColsCL];
#pragma unroll
    for (int q = 0; q < kColsCL; ++q) {
      uint32_t ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(q));
      w[q] = dsmem_ld_u32(ra);
    }
    __half2 m = *reinterpret_cast<__half2*>(&w[0]);
#pragma unroll
    for (int q = 1; q < kColsCL; ++q) m = __hmin2_nan(m, *reinterpret_cast<__half2*>(&w[q]));
    s_mm[0][tid] = m;
  }
  // the peers' partials have been read: this CTA may leave once every CTA got here
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  __syncthreads();
  // one thread per group of cpr columns (every CTA solves its strip's groups; rank 0
  // writes them to the slab)
  const int groups = CW / cpr;
  if (tid < groups) {
    __half2 m = s_mm[0][tid * cpr];
    for (int u = 1; u < cpr; ++u) m = __hmin2_nan(m, s_mm[0][tid * cpr + u]);
    float fmn = __low2float(m), fmx = -__high2float(m);
    const bool bad = !(isfinite(fmn) && isfinite(fmx));
    if (bad) { fmn = 0.f; fmx = 0.f; }
    if (bad && rank == 0) atomicOr(flag, 1);
    double sd, zd;
    const TileParams tp = tile_params_f16(fmn, fmx, qdiv_make((double)((1 << BITS) - 1)), sd, zd, sym);
    if (rank == 0) mm[plane * rows_per_plane + (col0 / cpr) + tid] = *reinterpret_cast<const uint32_t*>(&m);
    s_inv[tid] = tp.inv_s;  // per group (column / cpr)
    s_zc[tid] = tp.zc;
    s_thr[tid] = tp.thr;
    s_sd[tid] = sd;
    s_zd[tid] = zd;
  }
  __syncthreads();
  // ---- codes from shared memory.  One threshold per thread (the smallest of its 8
  // columns'): a vector whose largest |e| reaches it re-checks each value against its
  // own column's threshold.
  float inv[8], zc[8], thr[8];
  float thr_min = 1.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int gi = (cv * 8 + j) / cpr;
    inv[j] = s_inv[gi];
    zc[j] = s_zc[gi];
    thr[j] = s_thr[gi];
    thr_min = fminf(thr_min, thr[j]);
  }
  uint8_t* cbase = codes + ((plane * T + t0) * Hd + col0 + cv * 8) / (PACK ? 2 : 1);
  const float2 i2[4] = {make_float2(inv[0], inv[1]), make_float2(inv[2], inv[3]), make_float2(inv[4], inv[5]),
                        make_float2(inv[6], inv[7])};
  const float2 z2[4] = {make_float2(zc[0], zc[1]), make_float2(zc[2], zc[3]), make_float2(zc[4], zc[5]),
                        make_float2(zc[6], zc[7])};
  const float2 nz2[4] = {make_float2(-zc[0], -zc[1]), make_float2(-zc[2], -zc[3]), make_float2(-zc[4], -zc[5]),
                         make_float2(-zc[6], -zc[7])};
#pragma unroll 4
  for (int r = tl; r < nt; r += 16) {
    const uint4 d = s_tile[r * NCV + cv];
    const __half2* h = reinterpret_cast<const __half2*>(&d);
    uint32_t c[8];
    float dmax = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __half22float2(h[j]);
      const float2 y = __ffma2_rn(f, i2[j], z2[j]);
      const float2 cc = __fadd2_rn(y, nz2[j]);
      const float2 e = __ffma2_rn(f, i2[j], make_float2(-cc.x, -cc.y));
      dmax = fmaxf(dmax, fmaxf(fabsf(e.x), fabsf(e.y)));
      c[2 * j] = f2bits(y.x);
      c[2 * j + 1] = f2bits(y.y);
    }
    if (!(dmax < thr_min)) {  // rare: the reference float64 ops for the values near a boundary
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float f = __half2float(reinterpret_cast<const __half*>(&d)[j]);
        const float y = fmaf(f, inv[j], zc[j]);
        if (!(fabsf(fmaf(f, inv[j], -__fadd_rn(y, -zc[j]))) < thr[j])) {
          const int gi = (cv * 8 + j) / cpr;
          const float rr = (float)rint(__dadd_rn(__ddiv_rn((double)f, s_sd[gi]), s_zd[gi]));
          c[j] = (uint32_t)fminf(fmaxf(rr, 0.f), QMAXF);
        }
      }
    }
    if (PACK) {
      __stcs(reinterpret_cast<uint32_t*>(cbase + (int64_t)r * Hd / 2), pack_int4x8(c));
    } else {
      __stcs(reinterpret_cast<uint2*>(cbase + (int64_t)r * Hd),
             make_uint2(gather4(c[0], c[1], c[2], c[3]), gather4(c[4], c[5], c[6], c[7])));
    }
  }
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// Transfer-slab parameters -> (scale, zero): a group's fp16 (min, -max) determines its
// float64 scale and zero through exactly the quantizer's solve (kvmanager.py:130-146),
// so the slab carries 4 bytes per group instead of 12.  One group per thread (NG groups
// in sequence); the snap loop's cycle shortcut (qmath.cuh snap_scale) keeps the rare
// non-settling groups from holding their warp for 32 passes.
__device__ __forceinline__ void load_minmax(const uint32_t* mm, int64_t r, double& mn, double& mx) {
  uint32_t w = mm[r];
  const __half2 h = *reinterpret_cast<const __half2*>(&w);
  float fmn = __low2float(h), fmx = -__high2float(h);
  if (!(isfinite(fmn) && isfinite(fmx))) { fmn = 0.f; fmx = 0.f; }  // flagged at quantize time
  mn = (double)fmn;
  mx = (double)fmx;
}

// One group per thread.  The snap loop's cycle shortcut (qmath.cuh snap_scale) keeps
// the rare non-settling groups from holding their warp for 32 passes (expand 95 -> 73 us
// for a 1 GiB INT4 g=64 job; deferring unsettled groups to a dense second kernel measured
// slower, 81 + 7 us).
template <int BITS>
__global__ void __launch_bounds__(256)
k_expand_params(const uint32_t* __restrict__ mm, int64_t groups, double* __restrict__ scale,
                float* __restrict__ zero, int sym) {
  const QDiv dq = qdiv_make((double)((1 << BITS) - 1));
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= groups) return;
  double mn, mx, s, z;
  load_minmax(mm, r, mn, mx);
  if (sym) {
    solve_absmax(mn, mx, dq.b, s, z);  // no snap loop
  } else if (mx == mn) {
    s = 1.0;                           // constant group: (1, -min)
    z = -mn;
  } else {
    solve_scale_zero(mn, mx, dq, s, z);
  }
  scale[r] = s;
  zero[r] = (float)z;
}

// Column dequantize for CHANNEL / HEAD kinds: each thread owns 8 columns of a strip
// and walks the tokens with per-column constants in registers (fast path + exact
// re-run as in k_dequant_tile).
template <int BITS, bool PACK>
__global__ void __launch_bounds__(256)
k_dequant_cols(const uint8_t* __restrict__ codes, const double* __restrict__ scale, const float* __restrict__ zero,
               int64_t T, int64_t Hd, int cpr, int64_t rows_per_plane, uint16_t* __restrict__ out) {
  const int tid = threadIdx.x;
  const int cv = tid & 15, tl = tid >> 4;
  const int64_t plane = blockIdx.y;
  const int64_t col0 = (int64_t)blockIdx.x * 128 + cv * 8;
  double sd[8], zd[8];
  float s32[8], zm[8];
  bool fast = true;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t r = plane * rows_per_plane + (col0 + j) / cpr;
    sd[j] = scale[r];
    zd[j] = (double)zero[r];
    s32[j] = (float)sd[j];
    zm[j] = (float)(zd[j] + 8388608.0);
    fast &= zd[j] == rint(zd[j]) && fabs(zd[j]) < 4194304.0 && sd[j] >= 0x1p-14 && sd[j] < 60000.0;
  }
  const uint8_t* cb = codes + (plane * T * Hd + col0) / (PACK ? 2 : 1);
  uint16_t* ob = out + plane * T * Hd + col0;
  using CodeWord = typename std::conditional<PACK, uint32_t, uint2>::type;
  auto dq_vec = [&](const CodeWord wd, int64_t t) {
    uint32_t q[8];
    if constexpr (PACK) {
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = (wd >> (4 * j)) & 15u;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) { q[j] = (wd.x >> (8 * j)) & 255u; q[4 + j] = (wd.y >> (8 * j)) & 255u; }
    }
    uint32_t o[4];
    bool unsafe = !fast;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 qf = make_float2(__uint_as_float(0x4B000000u | q[2 * j]), __uint_as_float(0x4B000000u | q[2 * j + 1]));
      const float2 d = __fadd2_rn(qf, make_float2(-zm[2 * j], -zm[2 * j + 1]));
      const float2 y = __fmul2_rn(d, make_float2(s32[2 * j], s32[2 * j + 1]));
      const uint32_t b0 = __float_as_uint(y.x), b1 = __float_as_uint(y.y);
      unsafe |= ((b0 + (4u - 0x1000u)) & 0x1fffu) <= 8u;
      unsafe |= ((b1 + (4u - 0x1000u)) & 0x1fffu) <= 8u;
      const __half2 hv = __floats2half2_rn(y.x, y.y);
      o[j] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    if (unsafe) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double v = __dmul_rn(sd[j], __dsub_rn((double)q[j], zd[j]));
        const uint32_t hb = __half_as_ushort(__double2half(v));
        const int wi = j >> 1, sh = 16 * (j & 1);
        o[wi] = (o[wi] & ~(0xffffu << sh)) | (hb << sh);
      }
    }
    __stcs(reinterpret_cast<uint4*>(ob + t * Hd), make_uint4(o[0], o[1], o[2], o[3]));
  };
  auto load = [&](int64_t t) -> CodeWord {
    if constexpr (PACK) return __ldcs(reinterpret_cast<const uint32_t*>(cb + t * Hd / 2));
    else return __ldcs(reinterpret_cast<const uint2*>(cb + t * Hd));
  };
  // sixteen token rows of codes in flight per thread
  int64_t t = tl;
  for (; t + 240 < T; t += 256) {
    CodeWord w[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) w[u] = load(t + 16 * u);
#pragma unroll
    for (int u = 0; u < 16; ++u) dq_vec(w[u], t + 16 * u);
  }
  for (; t < T; t += 16) dq_vec(load(t), t);
}

// ---------------------------------------------------------------------------------
// Generic path, phase 1a: partial min/max of strided rows (any dtype), block per
// (row, chunk).  partials are float64 [rows][nch].
// ---------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
k_minmax_rows(const T* __restrict__ x, int64_t rows, int64_t row_len, int64_t row_stride,
              int64_t chunk, int nch, double* __restrict__ pmn, double* __restrict__ pmx,
              int* __restrict__ flag) {
  const int64_t r = blockIdx.x / nch;
  const int ch = blockIdx.x % nch;
  const int64_t i0 = (int64_t)ch * chunk;
  const int64_t i1 = min(row_len, i0 + chunk);
  double a = __longlong_as_double(0x7ff0000000000000ll), b = -a;
  bool bad = false;
  const T* row = x + r * row_stride;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const T v = row[i];
    bad |= InTraits<T>::bad(v);
    const double d = InTraits<T>::d(v);
    a = fmin(a, d);
    b = fmax(b, d);
  }
  raise_flag(flag, bad);
  __shared__ double sa[32], sb[32];
  for (int o = 16; o > 0; o >>= 1) {
    a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sa[w] = a; sb[w] = b; }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    a = l < nw ? sa[l] : __longlong_as_double(0x7ff0000000000000ll);
    b = l < nw ? sb[l] : -__longlong_as_double(0x7ff0000000000000ll);
    for (int o = 16; o > 0; o >>= 1) {
      a = fmin(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = fmax(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (l == 0) { pmn[r * nch + ch] = a; pmx[r * nch + ch] = b; }
  }
}

// Phase 1b: column partials for CHANNEL / HEAD kinds.  Planes of [T][Hd] fp16.
// grid: (Hd/8 / blockDim.x column-vector blocks, nch token chunks, planes).
// partials float [plane][nch][Hd].
__global__ void __launch_bounds__(128)
k_minmax_cols(const uint16_t* __restrict__ x, int64_t T, int64_t Hd, int64_t tchunk,
              float* __restrict__ pmn, float* __restrict__ pmx, int* __restrict__ flag) {
  const int64_t c8 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // column vector
  const int ch = blockIdx.y;
  const int64_t plane = blockIdx.z;
  const int nch = gridDim.y;
  const bool live = c8 * 8 < Hd;
  float a[8], b[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { a[j] = __int_as_float(0x7f800000); b[j] = -a[j]; }
  bool bad = false;
  if (live) {
    const int64_t t0 = ch * tchunk, t1 = min(T, t0 + tchunk);
    const uint16_t* base = x + plane * T * Hd + c8 * 8;
#pragma unroll 4
    for (int64_t t = t0; t < t1; ++t) {
      const uint4 v = __ldcs(reinterpret_cast<const uint4*>(base + t * Hd));
      const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        bad |= h_nonfinite(h[j]);
        const float f = h2f(h[j]);
        a[j] = fminf(a[j], f);
        b[j] = fmaxf(b[j], f);
      }
    }
    float* om = pmn + (plane * nch + ch) * Hd + c8 * 8;
    float* oM = pmx + (plane * nch + ch) * Hd + c8 * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) { om[j] = a[j]; oM[j] = b[j]; }
  }
  raise_flag(flag, bad);
}

// Phase 2: per-row params.  Writes scale (f64), zero (f64 or f32) and fast params.
template <bool ZF32>
__global__ void k_params(int kind, int64_t rows, int nch, const double* __restrict__ pmn_rows,
                         const double* __restrict__ pmx_rows, const float* __restrict__ pmn_cols,
                         const float* __restrict__ pmx_cols, int64_t Hd, int64_t D, int bits,
                         bool wide, double* __restrict__ scale, void* __restrict__ zero,
                         float4* __restrict__ fastp, uint32_t* __restrict__ mm, int sym) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  if (kind == KIND_ROWS) {
    for (int c = 0; c < nch; ++c) {
      mn = fmin(mn, pmn_rows[r * nch + c]);
      mx = fmax(mx, pmx_rows[r * nch + c]);
    }
  } else {
    const int64_t per_plane = (kind == KIND_CHANNEL) ? Hd : Hd / D;
    const int64_t plane = r / per_plane, idx = r % per_plane;
    const int64_t c0 = (kind == KIND_CHANNEL) ? idx : idx * D;
    const int64_t cn = (kind == KIND_CHANNEL) ? 1 : D;
    for (int c = 0; c < nch; ++c) {
      const float* m0 = pmn_cols + (plane * nch + c) * Hd + c0;
      const float* m1 = pmx_cols + (plane * nch + c) * Hd + c0;
      for (int64_t j = 0; j < cn; ++j) {
        mn = fmin(mn, (double)m0[j]);
        mx = fmax(mx, (double)m1[j]);
      }
    }
  }
  if (mm) {  // fp16 inputs: mn / mx are fp16 values, exact as halves
    const __half2 h = __halves2half2(__double2half(mn), __double2half(-mx));
    mm[r] = *reinterpret_cast<const uint32_t*>(&h);
  }
  const QParams q = make_params(mn, mx, bits, wide, qdiv_make((double)((1 << bits) - 1)), sym);
  scale[r] = q.s;
  if (ZF32) reinterpret_cast<float*>(zero)[r] = (float)q.z;
  else reinterpret_cast<double*>(zero)[r] = q.z;
  fastp[r] = make_float4(q.inv_s, q.zf, q.err, 0.f);
}

__device__ __forceinline__ QParams load_params(const float4* fastp, const double* scale,
                                               const void* zero, bool zf32, int64_t r) {
  const float4 f = fastp[r];
  QParams q;
  q.inv_s = f.x; q.zf = f.y; q.err = f.z;
  q.s = scale[r];
  q.z = zf32 ? (double)reinterpret_cast<const float*>(zero)[r]
             : reinterpret_cast<const double*>(zero)[r];
  return q;
}

// Phase 3a: codes for strided ROWS (any dtype); output row-major codes.
template <typename T, int BITS, bool PACK>
__global__ void __launch_bounds__(256)
k_codes_rows(const T* __restrict__ x, int64_t rows, int64_t row_len, int64_t row_stride,
             const float4* __restrict__ fastp, const double* __restrict__ scale,
             const void* __restrict__ zero, bool zf32, uint8_t* __restrict__ codes) {
  constexpr float QMAXF = (float)((1 << BITS) - 1);
  const int64_t npairs = (rows * row_len + (PACK ? 1 : 0)) / (PACK ? 2 : 1);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < npairs;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t out = 0;
#pragma unroll
    for (int j = 0; j < (PACK ? 2 : 1); ++j) {
      const int64_t e = PACK ? 2 * k + j : k;
      if (e >= rows * row_len) break;
      const int64_t r = e / row_len, i = e - r * row_len;
      const QParams q = load_params(fastp, scale, zero, zf32, r);
      const T v = x[r * row_stride + i];
      const double d = InTraits<T>::d(v);
      out |= quant_code((float)d, d, q, QMAXF) << (4 * j);
    }
    codes[k] = (uint8_t)out;
  }
}

// Phase 3b: codes for CHANNEL / HEAD planes, walking native memory 8 values at a time.
template <int BITS, bool PACK>
__global__ void __launch_bounds__(256)
k_codes_cols(const uint16_t* __restrict__ x, int kind, int64_t planes, int64_t T, int64_t Hd,
             int64_t D, const float4* __restrict__ fastp, const double* __restrict__ scale,
             const void* __restrict__ zero, bool zf32, uint8_t* __restrict__ codes) {
  constexpr float QMAXF = (float)((1 << BITS) - 1);
  const int64_t vecs_per_line = Hd / 8;
  const int64_t total = planes * T * vecs_per_line;
  const int64_t per_plane_rows = (kind == KIND_CHANNEL) ? Hd : Hd / D;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = k / vecs_per_line;
    const int64_t c = (k - line * vecs_per_line) * 8;
    const int64_t plane = line / T;
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(x + k * 8));
    const uint16_t* h = reinterpret_cast<const uint16_t*>(&v);
    uint32_t cc[8];
    if (kind == KIND_HEAD) {
      const QParams q = load_params(fastp, scale, zero, zf32, plane * per_plane_rows + c / D);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float f = h2f(h[j]);
        cc[j] = quant_code(f, (double)f, q, QMAXF);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const QParams q = load_params(fastp, scale, zero, zf32, plane * per_plane_rows + c + j);
        const float f = h2f(h[j]);
        cc[j] = quant_code(f, (double)f, q, QMAXF);
      }
    }
    if (PACK) {
      const uint32_t w = cc[0] | (cc[1] << 4) | (cc[2] << 8) | (cc[3] << 12) | (cc[4] << 16) |
                         (cc[5] << 20) | (cc[6] << 24) | (cc[7] << 28);
      reinterpret_cast<uint32_t*>(codes)[k] = w;
    } else {
      reinterpret_cast<uint2*>(codes)[k] =
          make_uint2(cc[0] | (cc[1] << 8) | (cc[2] << 16) | (cc[3] << 24),
                     cc[4] | (cc[5] << 8) | (cc[6] << 16) | (cc[7] << 24));
    }
  }
}

// ---------------------------------------------------------------------------------
// Dequantize.  value = fp(s * (q - z)) (kvmanager.py:154).  8 values per thread.
//   ROWS: row = element / row_len; CHANNEL/HEAD: native planes as above.
// OUT: uint16_t (fp16, rounded once from the float64 product) or double (exact reference).
// ---------------------------------------------------------------------------------
template <typename OUT, int BITS, bool PACK>
__global__ void __launch_bounds__(256)
k_dequant(int kind, const uint8_t* __restrict__ codes, const double* __restrict__ scale,
          const void* __restrict__ zero, bool zf32, int64_t n, int64_t row_len, int64_t T,
          int64_t Hd, int64_t D, OUT* __restrict__ out) {
  const int64_t nvec = n / 8;  // host guarantees n % 8 == 0
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nvec;
       k += (int64_t)gridDim.x * blockDim.x) {
    uint32_t q[8];
    if (PACK) {
      const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(codes) + k);
#pragma unroll
      for (int j = 0; j < 8; ++j) q[j] = (w >> (4 * j)) & 15u;
    } else {
      const uint2 w = __ldcs(reinterpret_cast<const uint2*>(codes) + k);
#pragma unroll
      for (int j = 0; j < 4; ++j) { q[j] = (w.x >> (8 * j)) & 255u; q[4 + j] = (w.y >> (8 * j)) & 255u; }
    }
    const int64_t e0 = k * 8;
    int64_t r0;
    bool uniform;
    if (kind == KIND_ROWS) {
      r0 = e0 / row_len;
      uniform = (row_len % 8) == 0;
    } else {
      const int64_t line = e0 / Hd, c = e0 - line * Hd, plane = line / T;
      if (kind == KIND_HEAD) { r0 = plane * (Hd / D) + c / D; uniform = (D % 8) == 0; }
      else { r0 = plane * Hd + c; uniform = false; }
    }
    OUT o[8];
    if (uniform) {
      const double s = scale[r0];
      const double z = zf32 ? (double)reinterpret_cast<const float*>(zero)[r0]
                            : reinterpret_cast<const double*>(zero)[r0];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double v = __dmul_rn(s, __dsub_rn((double)q[j], z));
        if constexpr (sizeof(OUT) == 2) o[j] = __half_as_ushort(__double2half(v));
        else o[j] = v;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int64_t r;
        if (kind == KIND_ROWS) r = (e0 + j) / row_len;
        else if (kind == KIND_CHANNEL) r = r0 + j;
        else { const int64_t line = (e0 + j) / Hd, c = e0 + j - line * Hd; r = (line / T) * (Hd / D) + c / D; }
        const double s = scale[r];
        const double z = zf32 ? (double)reinterpret_cast<const float*>(zero)[r]
                              : reinterpret_cast<const double*>(zero)[r];
        const double v = __dmul_rn(s, __dsub_rn((double)q[j], z));
        if constexpr (sizeof(OUT) == 2) o[j] = __half_as_ushort(__double2half(v));
        else o[j] = v;
      }
    }
    if constexpr (sizeof(OUT) == 2) {
      uint4 w;
      w.x = (uint32_t)o[0] | ((uint32_t)o[1] << 16);
      w.y = (uint32_t)o[2] | ((uint32_t)o[3] << 16);
      w.z = (uint32_t)o[4] | ((uint32_t)o[5] << 16);
      w.w = (uint32_t)o[6] | ((uint32_t)o[7] << 16);
      __stcs(reinterpret_cast<uint4*>(out) + k, w);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) out[e0 + j] = o[j];
    }
  }
}

// Dequantize for arbitrary n (tail-safe scalar version), ROWS kind only.
template <typename OUT, int BITS, bool PACK>
__global__ void k_dequant_tail(const uint8_t* __restrict__ codes, const double* __restrict__ scale,
                               const void* __restrict__ zero, bool zf32, int64_t e_begin, int64_t n,
                               int64_t row_len, OUT* __restrict__ out) {
  const int64_t e = e_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const uint32_t q = PACK ? ((codes[e >> 1] >> (4 * (e & 1))) & 15u) : codes[e];
  const int64_t r = e / row_len;
  const double s = scale[r];
  const double z = zf32 ? (double)reinterpret_cast<const float*>(zero)[r]
                        : reinterpret_cast<const double*>(zero)[r];
  const double v = __dmul_rn(s, __dsub_rn((double)q, z));
  if constexpr (sizeof(OUT) == 2) out[e] = __half_as_ushort(__double2half(v));
  else out[e] = v;
}

}  // namespace alise
