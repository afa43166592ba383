/* alise_b200.h — C ABI of libalise_b200.so, the B200 data plane behind the
 * reference servesim package's quantizer / swap / predictor API.
 *
 * Conventions (all entry points):
 *   - return int status: ALISE_OK, or an ALISE_E* code; alise_last_error()
 *     returns a thread-local message for the last failure.
 *   - every device pointer is caller-owned (torch tensors or alise_* allocations);
 *     calls are stream-ordered on the `stream` argument (a cudaStream_t, NULL =
 *     legacy default stream) and never synchronise the host unless stated.
 *   - non-finite inputs are reported through a caller-provided device int flag
 *     (set to non-zero), read by the host after the work completes; the Python
 *     layer turns it into ValueError("tensor contains non-finite values"),
 *     exactly as kvmanager.py:127-128 does.
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   alise_quantize_rows      <- servesim.kvmanager.quantize     pkg/src/servesim/kvmanager.py:108
 *   alise_dequantize_rows    <- servesim.kvmanager.dequantize   pkg/src/servesim/kvmanager.py:152
 *   alise_kv_*  / swapper    <- servesim.kvmanager.MemoryState.start_offload / start_upload /
 *                               complete (kvmanager.py:241-268) — the reference only does the
 *                               byte accounting; these move and (de)quantize the bytes
 *   alise_db_* / alise_pred* <- servesim.predictor.VectorStore.add/search (predictor.py:135-163),
 *                               LengthPredictor.predict_vector (predictor.py:311-325),
 *                               FallbackRegressor.predict_len (predictor.py:209-219)
 */
#ifndef ALISE_B200_H
#define ALISE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ALISE_OK 0
#define ALISE_EINVAL 1      /* bad argument -> ValueError                      */
#define ALISE_ENONFINITE 2  /* non-finite input -> ValueError                  */
#define ALISE_ECAPACITY 3   /* capacity / accounting violation                 */
#define ALISE_ECUDA 4       /* CUDA runtime error -> RuntimeError              */

#define ALISE_DT_F16 0
#define ALISE_DT_F32 1
#define ALISE_DT_F64 2

#define ALISE_KIND_ROWS 0     /* rows of row_len contiguous values (group-wise g)       */
#define ALISE_KIND_CHANNEL 1  /* (layer, k|v, hidden column) along tokens (reference)   */
#define ALISE_KIND_HEAD 2     /* (layer, k|v, head) over tokens x head_dim              */

/* How a group's (scale, zero) follow from its (min, max):
 *  ASYM   the reference's asymmetric min/max scheme (kvmanager.py:130-146: scale =
 *         (max-min)/qmax, zero = rint(-min/scale), snap loop);
 *  ABSMAX symmetric absmax scheme named by the north star (parity UNPINNED by the
 *         reference, which has no such mode; restated in oracle/kv_oracle.py
 *         quantize_rows_absmax): scale = max|x| / (2^(b-1)-1) (1 if 0), zero = 2^(b-1).
 * Codes and values use the reference formulas in both modes: clip(rint(x/scale +
 * zero), 0, qmax) and scale*(code - zero). */
#define ALISE_QMODE_ASYM 0
#define ALISE_QMODE_ABSMAX 1

#define ALISE_SWAP_STAGED 0   /* quantize to an HBM ring, copy engine D2H/H2D (default) */
#define ALISE_SWAP_ZEROCOPY 1 /* kernels read/write mapped pinned host memory directly  */

const char *alise_last_error(void);
int alise_version(void);
int alise_sm_count(int device, int *out);
/* Self-test of the quantizer's constant-divisor division (qmath.cuh qdiv) against
 * __ddiv_rn on n device doubles x: adds the count of bit mismatches of x/(2^bits-1)
 * to *mismatches (device int64).  Test support, not part of the reference interface. */
int alise_selftest_qdiv(const double *x, int64_t n, int bits, int64_t *mismatches, void *stream);

/* ------------------------------------------------------- host control plane ---- */
/* Residency codes (kvmanager.py:18-22: "gpu", "cpu", "none", "uploading", "offloading"). */
#define ALISE_RES_GPU 0
#define ALISE_RES_CPU 1
#define ALISE_RES_NONE 2
#define ALISE_RES_UPLOADING 3
#define ALISE_RES_OFFLOADING 4
/* Replaces kvmanager.py:276-294 ewt_ms: per job in global rank order, min(sum of the
 * remaining ms of the jobs ahead, max(level*aging_ms - waited_ms, 0)); aging_ms = +inf
 * disables the promote arm.  Host-only, float64 exactly as the reference computes it. */
int alise_ewt_ms(int64_t n, const int32_t *level, const int64_t *last_promotion_us,
                 const double *remaining_ms, double aging_ms, int64_t now_us, double *out_ewt_ms);
/* Replaces kvmanager.py:297-322 plan_swaps over n entries in plan order, budget =
 * gpu_capacity - in-flight gpu bytes.  out_action per entry: 0 denied, 1 granted,
 * 2 granted + upload (entry on CPU), 3 denied + offload (entry on GPU). */
int alise_plan_swaps(int64_t n, const int32_t *residency, const int64_t *need_gpu_bytes,
                     int64_t budget_bytes, int8_t *out_action);
/* Replaces simcore.py:439-462 _ranked_with_grants: EWT over the n jobs of the global
 * rank, plan order = level ascending then (EWT, rank position), in-flight jobs
 * (uploading/offloading) skipped, then plan_swaps.  out_order[0..*out_count) = rank
 * positions of the planned entries, out_action as alise_plan_swaps. */
int alise_rank_and_plan(int64_t n, const int32_t *level, const int64_t *last_promotion_us,
                        const double *remaining_ms, const int32_t *residency,
                        const int64_t *need_gpu_bytes, double aging_ms, int64_t now_us,
                        int64_t budget_bytes, double *out_ewt_ms, int32_t *out_order,
                        int64_t *out_count, int8_t *out_action);

/* ---------------------------------------------------------------- quantizer ---- */
/* Drop-in for kvmanager.quantize: rows x row_len values (row i at src + i*row_stride
 * elements, dtype ALISE_DT_*), bits in {4,8}.  codes: rows*row_len bytes (one code
 * per byte, the reference's uint8 layout, kvmanager.py:94).  scale, zero: float64[rows].
 * nonfinite_flag: device int (OR-ed with 1 on a non-finite value).  workspace:
 * device scratch of alise_quantize_rows_workspace() bytes (may be NULL if 0). */
int alise_quantize_rows_workspace(int64_t rows, int64_t row_len, int src_dtype, int64_t *bytes);
int alise_quantize_rows(const void *src, int src_dtype, int64_t rows, int64_t row_len,
                        int64_t row_stride, int bits, uint8_t *codes, double *scale,
                        double *zero, int *nonfinite_flag, void *workspace, void *stream);
/* alise_quantize_rows with a quantization mode (ALISE_QMODE_*). */
int alise_quantize_rows_ex(const void *src, int src_dtype, int64_t rows, int64_t row_len,
                           int64_t row_stride, int bits, int mode, uint8_t *codes, double *scale,
                           double *zero, int *nonfinite_flag, void *workspace, void *stream);
/* Drop-in for kvmanager.dequantize: out = scale*(code - zero), out_dtype F64 (reference
 * bit-exact) or F16 (one rounding of the float64 value). */
int alise_dequantize_rows(const uint8_t *codes, const double *scale, const double *zero,
                          int64_t rows, int64_t row_len, int out_dtype, void *out, void *stream);

/* ------------------------------------------------------------ KV data plane ---- */
/* One job's KV cache in HBM: kv[layers][2][tokens][hidden] fp16 (hidden = heads*head_dim). */
typedef struct {
  int64_t layers;
  int64_t tokens;
  int64_t hidden;
  int64_t head_dim;
  int32_t kind;       /* ALISE_KIND_* */
  int32_t group;      /* KIND_ROWS: values per group (multiple of 8, divides hidden) */
  int32_t bits;       /* 4 or 8 */
  int32_t packed;     /* 1: two INT4 codes per byte (low nibble = even element) */
  int32_t planes_per_chunk; /* transfer granularity in (layer, k|v) planes; 0 = auto */
  int32_t mode;       /* ALISE_QMODE_*: how a group's (scale, zero) follow from its (min, max) */
} alise_kv_desc;

/* Host slab layout: ceil(planes/planes_per_chunk) chunk records, each
 *   [codes of its planes, native element order][fp16 (min, -max) per group]
 * with every section 256-byte aligned.  A group's float64 (scale, zero) are a function
 * of its (min, max) (kvmanager.py:130-146) and are recomputed bit-exactly on upload, so
 * the slab carries 4 bytes per group instead of 12.  rows = groups; link bytes = slab
 * bytes. */
int alise_kv_layout(const alise_kv_desc *d, int64_t *slab_bytes, int64_t *rows,
                    int64_t *chunk_bytes, int64_t *n_chunks);
/* Device-to-device quantize of a whole job into a device slab (same layout). */
int alise_kv_quantize(const alise_kv_desc *d, const uint16_t *kv, uint8_t *slab,
                      int *nonfinite_flag, void *stream);
/* Device slab -> fp16 KV. */
int alise_kv_dequantize(const alise_kv_desc *d, const uint8_t *slab, uint16_t *kv, void *stream);

typedef struct alise_swapper alise_swapper;
/* ring_bytes: HBM staging per direction (0 = 3 chunks of the largest desc seen). */
int alise_swapper_create(int device, int mode, int64_t ring_bytes, alise_swapper **out);
int alise_swapper_destroy(alise_swapper *sw);
/* Quantize kv (HBM) chunk by chunk and stream the slab to host_slab (pinned host),
 * overlapping kernel and D2H copy engine.  Kernels run on `stream`, copies on the
 * swapper's side stream.  done_event (cudaEvent_t, may be NULL) fires when the
 * last byte has landed in host memory.  The kv buffer may be reused once
 * `stream` passes this point (all reads are ordered on it). */
int alise_kv_offload(alise_swapper *sw, const alise_kv_desc *d, const uint16_t *kv,
                     void *host_slab, int *nonfinite_flag, void *stream, void *done_event);
/* Stream host_slab to HBM chunk by chunk (H2D copy engine) and dequantize into kv.
 * done_event fires (on `stream`) when kv is complete. */
int alise_kv_upload(alise_swapper *sw, const alise_kv_desc *d, const void *host_slab,
                    uint16_t *kv, void *stream, void *done_event);
/* Token-range transfers (ROWS kind, staged mode): d->tokens is the job's token capacity
 * T_cap (HBM kv[L][2][T_cap][hidden], slab laid out for T_cap); only tokens [t0, t1) are
 * quantized+offloaded into / uploaded+dequantized from their places in the slab.  A
 * group never spans tokens, so the bytes equal that part of a full offload: re-offloading
 * a job that grew from t0 to t1 tokens moves only the new tokens (incremental block-wise
 * offload; the reference re-sends quantized_kv_bytes(kv_tokens) on every
 * offload, simcore.py:338-339). */
int alise_kv_offload_range(alise_swapper *sw, const alise_kv_desc *d, const uint16_t *kv,
                           void *host_slab, int64_t t0, int64_t t1, int *nonfinite_flag, void *stream,
                           void *done_event);
int alise_kv_upload_range(alise_swapper *sw, const alise_kv_desc *d, const void *host_slab,
                          uint16_t *kv, int64_t t0, int64_t t1, void *stream, void *done_event);

/* Order every later transfer of this swapper after `event` (cudaEvent_t), e.g. an
 * upload that reads a host slab an earlier offload wrote. */
int alise_swapper_depend(alise_swapper *sw, void *event);

/* Bench instrumentation: record CUDA events around every quantize / dequantize chunk
 * on the compute stream; kernel_stats sums their durations (and synchronises). */
int alise_swapper_timing(alise_swapper *sw, int enable);
int alise_swapper_kernel_stats(alise_swapper *sw, double *quant_ms, int64_t *n_quant,
                               double *deq_ms, int64_t *n_deq);

/* Pinned host memory and events (thin wrappers so non-torch hosts can drive the ABI). */
int alise_host_alloc(int64_t bytes, void **out);
/* NUMA-local pinned host memory for a GPU's slabs (each rank swaps over its
 * own host link into memory on the GPU's socket): anonymous pages with a preferred-node
 * policy (mbind), then page-locked + device-mapped (cudaHostRegister).  numa_node >= 0,
 * or ALISE_NUMA_CURRENT_GPU for the current device's node (sysfs).  *bound (may be NULL)
 * = 1 if the node policy was applied (0 on single-node hosts or where mbind is not
 * permitted: plain pinned pages).  Free with alise_host_free. */
#define ALISE_NUMA_CURRENT_GPU (-2)
int alise_host_alloc_numa(int64_t bytes, int numa_node, void **out, int *bound);
/* NUMA node of a GPU's PCI device (-1 if unknown / single node). */
int alise_gpu_numa_node(int device, int *node);
int alise_host_free(void *p);
int alise_event_create(void **ev);
int alise_event_destroy(void *ev);
int alise_event_record(void *ev, void *stream);
int alise_event_query(void *ev, int *done);
int alise_event_sync(void *ev);
int alise_stream_wait(void *stream, void *ev);
int alise_event_elapsed_ms(void *start, void *stop, float *ms);

/* ---------------------------------------------------------------- predictor ---- */
typedef struct alise_db alise_db;
/* Master dtype of a store's vectors (and of the queries searched against it). */
#define ALISE_DB_F32 0
#define ALISE_DB_F64 1
/* FIFO ring of `capacity` vectors of `dim` (master copy in fp32, or float64 like the
 * reference's np.float64 store, predictor.py:126; plus an fp16 copy for the coarse
 * tensor-core scan), observed lengths (int32) and insert sequence numbers (int64).
 * Mirrors VectorStore (predictor.py:120-152): slot = seq % capacity.
 * alise_db_create = alise_db_create_ex(..., ALISE_DB_F32, ...). */
int alise_db_create(int device, int64_t capacity, int64_t dim, alise_db **out);
int alise_db_create_ex(int device, int64_t capacity, int64_t dim, int master_dtype, alise_db **out);
int alise_db_dtype(alise_db *db, int *master_dtype);
/* Order of the float64 similarities a search ranks by and returns:
 *  ALISE_ORDER_EXACT (default): the correctly rounded exact dot product;
 *  ALISE_ORDER_BLAS: the exact operation sequence of the reference's scan
 *    (predictor.py:158 `self._vecs[:size] @ vector` -> numpy 2.3 -> OpenBLAS 0.3.30
 *    dgemv_t on x86-64, restated in oracle/blas_order.c), i.e. the reference's own
 *    float64 sims bit for bit, so ties that are exact in real arithmetic break as in
 *    the reference.  blas_threads = the reference host's OpenBLAS thread count (it
 *    splits the rows when size * dim >= 460800); row r of the reference's array is ring
 *    slot seq % ref_capacity of ref_size live rows (0 / -1: this store's own capacity
 *    and size; a sharded store passes the global ring). */
#define ALISE_ORDER_EXACT 0
#define ALISE_ORDER_BLAS 1
int alise_db_set_order(alise_db *db, int order, int blas_threads, int64_t ref_capacity, int64_t ref_size);
int alise_db_destroy(alise_db *db);
/* Append n rows (device pointers): vecs [n][dim] in the master dtype, lens int32 [n],
 * seqs int64 [n] (the store's next sequence numbers, in order; slot = (seq / stride) %
 * capacity).  VectorStore.add (predictor.py:135-152). */
int alise_db_append(alise_db *db, const void *vecs, const int32_t *lens, const int64_t *seqs,
                    int64_t n, void *stream);
int alise_db_size(alise_db *db, int64_t *size, int64_t *next_seq);
/* Shard of a G-way sequence-sharded store: this db receives every G-th sequence number
 * (seq % G == rank) and places it at slot (seq / G) % capacity, so per-shard FIFO
 * eviction equals the global FIFO when the global capacity is G * capacity. */
int alise_db_set_seq_stride(alise_db *db, int64_t stride);
/* Copy the first n live slots (master-dtype vectors, lens, seqs) to device buffers. */
int alise_db_export(alise_db *db, void *vecs, int32_t *lens, int64_t *seqs, int64_t n, void *stream);
/* Number of rescored candidates whose double-double sum could not certify the float64
 * rounding and were recomputed with the exact 640-bit accumulator (synchronous). */
int alise_db_inexact(alise_db *db, unsigned int *count);
/* Exact top-k of B queries ([B][dim] in the db's master dtype, device) against the db:
 * sims are the correctly rounded float64 dot products, ordered by (-sim, seq) (ties ->
 * older first).  Outputs [B][k]; count[b] = min(k, size).  VectorStore.search
 * (predictor.py:154-163).  k <= 16 takes the tcgen05 scan + fused filter; 16 < k <= 1024
 * a CUDA-core coarse pass over row splits with the same bound (ALISE_ECAPACITY if more
 * than 4096 rows of one query tie within the coarse error). */
int alise_db_topk(alise_db *db, const void *queries, int64_t B, int k, double *out_sim,
                  int64_t *out_seq, int32_t *out_len, int32_t *out_count, void *stream);
/* alise_db_topk in two steps for a sharded DB: the scan leaves per-query lower bounds
 * of the global EXACT k-th score in out_bound (float [B], -inf if none; a shard's coarse
 * k-th bound minus its own coarse error); after an all-reduce (max) of the bounds over
 * the shards, alise_db_topk_rescore returns the exact shard top-k restricted to rows
 * that can still enter the global top-k (counts may be < k).  ext_bound may be NULL
 * (= alise_db_topk).  The two calls must use the same queries.  For k > 16 the bound is
 * -inf and the rescore returns the shard's exact top-k. */
int alise_db_topk_scan(alise_db *db, const void *queries, int64_t B, int k, float *out_bound,
                       void *stream);
int alise_db_topk_rescore(alise_db *db, const void *queries, int64_t B, int k,
                          const float *ext_bound, double *out_sim, int64_t *out_seq,
                          int32_t *out_len, int32_t *out_count, void *stream);
/* Bench instrumentation: CUDA events around every coarse-scan launch; kernel_stats
 * returns the summed scan time, launch count and algorithmic flops (2*B*size*dim). */
int alise_db_timing(alise_db *db, int enable);
int alise_db_kernel_stats(alise_db *db, double *scan_ms, int64_t *launches, double *flops);
/* Merge G per-shard top-k lists ([G][B][k] each) into a global top-k by (-sim, seq). */
int alise_topk_merge(int G, int64_t B, int k, const double *sims, const int64_t *seqs,
                     const int32_t *lens, const int32_t *counts, double *out_sim,
                     int64_t *out_seq, int32_t *out_len, int32_t *out_count, void *stream);
/* Aggregate + all-MLP fallback (predictor.py:311-325, 209-219): per query, if any of
 * its count neighbours has sim >= s0, the similarity-weighted mean length (numpy
 * summation order), else the float64 MLP tanh(x.W1+b1).w2+b2 -> exp -> round.
 * W1 [dim][hidden] f64, b1 [hidden], w2 [hidden], b2 scalar; queries fp32 [B][dim].
 * out_len int32 [B]; out_retrieved uint8 [B] (1 = "retrieved", 0 = "fallback"). */
int alise_predict_finish(int64_t B, int k, const double *sims, const int32_t *lens,
                         const int32_t *counts, double s0, const float *queries, int64_t dim,
                         const double *W1, const double *b1, const double *w2, double b2,
                         int64_t hidden, int64_t max_len, double log_cap, int32_t *out_len,
                         uint8_t *out_retrieved, void *stream);
/* alise_predict_finish with the queries in fp32 or float64 (queries_dtype ALISE_DB_F32 /
 * ALISE_DB_F64): the MLP input is the reference's float64 vector when the caller has it. */
int alise_predict_finish_ex(int64_t B, int k, const double *sims, const int32_t *lens,
                            const int32_t *counts, double s0, const void *queries, int queries_dtype,
                            int64_t dim, const double *W1, const double *b1, const double *w2,
                            double b2, int64_t hidden, int64_t max_len, double log_cap,
                            int32_t *out_len, uint8_t *out_retrieved, void *stream);

/* Batched HashingEmbedder.embed (predictor.py:66-100): prompts are tokens[offsets[b] ..
 * offsets[b+1]) (int64, device); writes float64 [B][dim] (bit-identical to the
 * reference) and/or fp32 [B][dim] (either may be NULL).  Empty prompts are the
 * caller's error (the reference raises PredictorError). */
int alise_embed_batch(const int64_t *tokens, const int64_t *offsets, int64_t B, int64_t dim,
                      double *out_f64, float *out_f32, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ALISE_B200_H */
