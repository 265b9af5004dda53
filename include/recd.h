/*
 * librecd -- C ABI of the B200-native IKJT training hot path.
 *
 * Every entry point replaces one function of the reference's Python API
 * (`/root/reference/pkg/src/sessiondedup/`), batched over all feature keys of a
 * step so that one call launches one kernel per phase for every key:
 *
 *   recd_dedup                 <- tensors.build_ikjt            (tensors.py:269-308)
 *                                 (one IKJT per dedup group, reader.convert, reader.py:160-175)
 *   recd_pool_fwd              <- trainer_sim.embedding_lookup + pool + b[inv]
 *                                 (trainer_sim.py:308-344, 539-561), fused: the
 *                                 [N_u, D] activations are never materialised
 *   recd_expand                <- the expansion b[inv] alone     (trainer_sim.py:558-561)
 *   recd_embedding_lookup      <- trainer_sim.embedding_lookup  (trainer_sim.py:308-321)
 *   recd_pool_dense            <- trainer_sim.pool              (trainer_sim.py:324-344)
 *   recd_pool_bwd              <- (absent in the reference) segment-reduce
 *                                 onto unique rows + deterministic sorted scatter-add
 *                                 (+ fused SGD) into the tables
 *   recd_grad_unique /         the two halves of recd_pool_bwd, used by the row-sharded
 *   recd_sparse_sgd            multi-GPU step (grad onto unique rows at the source,
 *                              sorted scatter-add + SGD at the table owner)
 *   recd_shard_* /             row-sharded tables over R ranks: deduplicated IDs per
 *   recd_peer_*                (table, shard) pair to its owner (over NVLink peer
 *                              memory), shard-order sum of partially pooled rows
 *                              (the reference only simulates ranks,
 *                              trainer_sim.py:281-305)
 *   recd_jagged_index_select_* <- tensors.jagged_index_select   (tensors.py:363-390)
 *                                 and ikjt_to_kjt (tensors.py:393-399)
 *   recd_slice_renumber        <- trainer_sim.slice_ikjt_rows   (trainer_sim.py:394-413)
 *   recd_partial_ikjt          <- tensors.build_partial_ikjt    (tensors.py:311-360)
 *
 * Conventions
 *   - Jagged features use the reference layout: int64 values[N] and one int64
 *     offset per row (no trailing total; the last row runs to N).
 *   - Pointer arguments documented "device" point to GPU memory owned by the
 *     caller; "host [K]" arrays are read during the call only.
 *   - Calls are asynchronous on `stream` (a cudaStream_t); they never allocate
 *     and never synchronise, so a whole step can be captured in a CUDA graph.
 *   - Counts only known after a kernel ran (U unique rows, N_u unique values)
 *     stay on the device: `counts` arrays are int64[2F] with counts[f] = rows of
 *     feature f (U of its group) and counts[F+f] = values of feature f.
 *   - Return value: RECD_OK or an RECD_ERR_* code (argument / launch errors).
 *     Data-dependent errors the reference raises (out-of-range IDs/indices) are
 *     reported through a device int64 slot holding the first offending
 *     position, which the Python shim turns into the reference's exception.
 */
#ifndef RECD_H_
#define RECD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* recd_stream_t; /* cudaStream_t */

enum {
  RECD_OK = 0,
  RECD_ERR_ARG = 1,
  RECD_ERR_CUDA = 2,
  RECD_ERR_SCRATCH = 3,
  RECD_ERR_UNSUPPORTED = 4
};

enum { RECD_POOL_SUM = 0, RECD_POOL_AVG = 1, RECD_POOL_MAX = 2 };
/* recd_pool_fwd mode flag: the lookup runs beside a kernel on another stream
 * (e.g. recd_pool_bwd_prepare); its persistent grid leaves one CTA slot per SM. */
#define RECD_POOL_SHARE 0x100
enum { RECD_XF_IDENTITY = 0, RECD_XF_MOD_HASH = 1, RECD_XF_CLAMP = 2 };

/* Value of an error slot when no error occurred. */
#define RECD_NO_ERROR ((int64_t)0x7f7f7f7f7f7f7f7fLL)

int recd_version(void);
/* Human-readable description of the last non-OK return on this thread. */
const char* recd_last_error(void);
/* Kernels enqueued by this library since load (host counter). */
int64_t recd_launch_count(void);
/* Test hook: AND-mask applied to the 64-bit row hash (forces collisions so
 * the exact fallback path is exercised).  ~0 restores the default. */
void recd_debug_set_hash_mask(uint64_t mask);

/* Timing hook: record the given cudaEvents right before / after every launch
 * of the named kernel ("k_pool_fwd", "k_scatter"); NULL name disables. */
void recd_debug_kernel_events(const char* name, void* before, void* after);

/* ---------------------------------------------------------------- dedup --
 * KJT -> IKJT for `num_groups` feature groups of one batch of B rows.
 * Rows i, j of a group merge iff every feature list in the group is equal
 * (lengths included); unique rows are numbered in first-occurrence order and
 * the unique lists are copied in that order -- bit-identical to build_ikjt.
 *   group_sizes  host [G]       features per group (sum = F, F <= 64 per call)
 *   values       host [F]       device int64[num_values[f]]
 *   offsets      host [F]       device int64[B]
 *   num_values   host [F]
 *   inverse_out  host [G]       device int64[B]
 *   uoffsets_out host [F]       device int64[B]           (first U valid)
 *   uvalues_out  host [F]       device int64[num_values[f]] (first N_u valid)
 *   counts_out   device int64[2F]
 */
size_t recd_dedup_scratch_bytes(int32_t num_groups, int32_t num_features, int64_t batch_size);
int recd_dedup(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
               const int64_t* const* values, const int64_t* const* offsets,
               const int64_t* num_values, int64_t* const* inverse_out,
               int64_t* const* uoffsets_out, int64_t* const* uvalues_out, int64_t* counts_out,
               void* scratch, size_t scratch_bytes, recd_stream_t stream);

/* ------------------------------------------------------------- pool fwd --
 * For every feature f: pooled[u] = pool_{v in row u} tables[f][v] over the
 * unique rows (sum / avg / max, empty row -> 0; the sum follows numpy's
 * reduceat order a[0] + pairwise(a[1:]) so it is bit-identical to `pool`),
 * then out[i] = pooled[inverse[f][i]] for i < B (skipped where out[f] or
 * inverse[f] is NULL; with inverse[f] NULL and out[f] set, out = pooled).
 *   tables      host [F] device float[table_rows[f] x dim]
 *   uvalues/uoffsets host [F] device (jagged rows of feature f)
 *   counts      device int64[2F]
 *   pooled_out  host [F] device float[U_cap x dim]  (may alias out[f] when inverse[f] is NULL)
 *   err         device int64[2]: [0] first bad ID as (f << 40) | position, or RECD_NO_ERROR;
 *               [1] scratch (work counter of the launch)
 *   mode        RECD_POOL_SUM / AVG / MAX, optionally | RECD_POOL_SHARE
 */
int recd_pool_fwd(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                  const float* const* tables, const int64_t* table_rows,
                  const int64_t* const* uvalues, const int64_t* const* uoffsets,
                  const int64_t* counts, const int64_t* const* inverse,
                  float* const* pooled_out, float* const* out, int64_t* err,
                  recd_stream_t stream);

/* recd_pool_fwd with the expansion fused through the inverse CSR of
 * recd_pool_bwd_csr (batch rows of every unique row): each pooled row is
 * stored straight to out[f][i] for its batch rows i, so the [U x dim] pooled
 * buffer is neither written nor re-read (pooled_out: NULL, or per feature NULL
 * or a buffer that also receives the pooled rows).  Needs the backward's
 * RECD_BWD_INVERSE stage to have run on the same IKJT first.  A feature whose
 * csr_start and csr_rows are both NULL is an identity (plain KJT) feature --
 * recd_pool_bwd_csr reports it so -- pooled straight into out[f]. */
int recd_pool_fwd_csr(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                      const float* const* tables, const int64_t* table_rows,
                      const int64_t* const* uvalues, const int64_t* const* uoffsets,
                      const int64_t* counts, const int32_t* const* csr_start,
                      const uint32_t* const* csr_rows, float* const* pooled_out,
                      float* const* out, int64_t* err, recd_stream_t stream);

/* ------------------------------------------------------- row-coded H2D --
 * Device decode of row-delta coded KJT rows (recd_host.h encodes them on the
 * host): per feature, codes[f] uint8[B], offsets[f] int64[B] (row starts),
 * num_values device int64[F], value_caps host int64[F] (the grid), lits[f]
 * the literals; writes values_out[f][0 .. num_values[f]).  Exact. */
size_t recd_rowcode_scratch_bytes(int32_t num_features, int64_t batch_size);
int recd_rowcode_decode(int32_t num_features, int64_t batch_size, const uint8_t* const* codes,
                        const int64_t* const* offsets, const int64_t* num_values,
                        const int64_t* value_caps, const int64_t* const* lits,
                        int64_t* const* values_out, void* scratch, size_t scratch_bytes,
                        recd_stream_t stream);

/* Owner-side pooled lookup whose output rows go straight to the sources'
 * receive buffers (the all-to-all of partial rows fused into the pooling):
 * feature f's row u is stored at seg_dst[f * num_segs + s] + (u - seg_row0[f][s]) * dim
 * for the segment s with seg_row0[f][s] <= u < seg_row0[f][s + 1] (seg_row0:
 * device, ascending; num_segs <= 8; seg_dst may be peer / NVLink memory). */
int recd_pool_fwd_scatter(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                          const float* const* tables, const int64_t* table_rows,
                          const int64_t* const* uvalues, const int64_t* const* uoffsets,
                          const int64_t* counts, int32_t num_segs, const int64_t* const* seg_row0,
                          float* const* seg_dst, int64_t* err, recd_stream_t stream);

/* Expansion only: out[f][i] = pooled[f][inverse[f][i]] (inverse[f] NULL =
 * identity).  recd_pool_fwd with out = NULL followed by recd_expand equals one
 * recd_pool_fwd with out set (the split lets callers time the two kernels). */
int recd_expand(int32_t num_features, int64_t batch_size, int32_t dim,
                const int64_t* const* inverse, const float* const* pooled, float* const* out,
                recd_stream_t stream);

/* weights[values[j]] for j < n (materialised lookup, reference API). */
int recd_embedding_lookup(const float* table, int64_t table_rows, int32_t dim,
                          const int64_t* values, int64_t n, float* out, int64_t* err,
                          recd_stream_t stream);

/* pool(activations, offsets, op) over materialised activations [n_values x dim]. */
int recd_pool_dense(const float* acts, int64_t n_values, int32_t dim, const int64_t* offsets,
                    int64_t n_rows, int32_t mode, float* out, recd_stream_t stream);

/* recd_dedup in two halves (same arguments, same scratch): _number computes
 * inverse_out, uoffsets_out and counts_out; _copy gathers the unique values into
 * uvalues_out and, for features with remote_values[f] != NULL, also into
 * remote_values[f] + *remote_base[f] (device base; e.g. the owner's list in
 * peer memory -- the row-sharded step's ID dispatch fused into the gather). */
int recd_dedup_number(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                      const int64_t* const* values, const int64_t* const* offsets,
                      const int64_t* num_values, int64_t* const* inverse_out,
                      int64_t* const* uoffsets_out, int64_t* const* uvalues_out,
                      int64_t* counts_out, void* scratch, size_t scratch_bytes,
                      recd_stream_t stream);
int recd_dedup_copy(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                    const int64_t* const* values, const int64_t* const* offsets,
                    const int64_t* num_values, int64_t* const* inverse_out,
                    int64_t* const* uoffsets_out, int64_t* const* uvalues_out, int64_t* counts_out,
                    int64_t* const* remote_values, const int64_t* const* remote_base,
                    void* scratch, size_t scratch_bytes, recd_stream_t stream);
/* recd_dedup with the input value counts on the DEVICE (num_values_dev, int64[F],
 * written with the batch) and host capacities (value_caps >= every batch's
 * counts) for the launch geometry, so one captured CUDA graph serves every
 * batch: the reference's convert takes any batch (reader.py:160-175).
 *   phase  1 = number only (recd_dedup_number), 2 = copy only (recd_dedup_copy,
 *          remote_values / remote_base optional), 3 = both (recd_dedup) */
int recd_dedup_ex(int32_t num_groups, const int32_t* group_sizes, int64_t batch_size,
                  const int64_t* const* values, const int64_t* const* offsets,
                  const int64_t* value_caps, const int64_t* num_values_dev, int32_t phase,
                  int64_t* const* inverse_out, int64_t* const* uoffsets_out,
                  int64_t* const* uvalues_out, int64_t* counts_out,
                  int64_t* const* remote_values, const int64_t* const* remote_base,
                  void* scratch, size_t scratch_bytes, recd_stream_t stream);

/* ------------------------------------------------------------- pool bwd --
 * grad_u[u] = sum_{i: inverse[i]=u} grad_out[i]  (ascending i; /len for avg),
 * then for every distinct ID v of the feature, in ascending v:
 *   g[v] = sum over occurrences (u, p) with uvalues[u][p] == v, ascending
 *          (u, p), of grad_u[u];
 * apply_sgd = 1: tables[f][v] -= fp32(lr * g[v]) in place (no FMA);
 * apply_sgd = 0: grad_ids_out[f][k], grad_rows_out[f][k] = k-th distinct ID
 *                and its gradient, grad_counts_out[f] = number of IDs.
 * Features sharing an inverse pointer share one inverse CSR.  Only sum/avg.
 * An ID outside [0, table_rows[f]) anywhere in the call (negative, or >= rows:
 * the lookup reports it, trainer_sim.py:312-320) suppresses every table update
 * and gradient output of the call -- nothing is written out of bounds.
 *   value_caps  host [F] capacity of uvalues[f] (worst-case N_u)
 */
size_t recd_pool_bwd_scratch_bytes(int32_t num_features, int64_t batch_size, int32_t dim,
                                   const int64_t* value_caps);
int recd_pool_bwd(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                  float* const* tables, const int64_t* table_rows,
                  const int64_t* const* uvalues, const int64_t* const* uoffsets,
                  const int64_t* value_caps, const int64_t* counts,
                  const int64_t* const* inverse, const float* const* grad_out, float lr,
                  int32_t apply_sgd, int64_t* const* grad_ids_out, float* const* grad_rows_out,
                  int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                  recd_stream_t stream);

/* recd_pool_bwd in two halves, called with identical arguments and the same
 * scratch: _prepare enqueues the gradient-independent work (inverse CSR,
 * occurrence pairs and their sort by ID; grad_out is not read) and can run on
 * a side stream right after recd_dedup, overlapping the forward; _finish
 * enqueues the gradient reduction and the sorted scatter-add / SGD. */
int recd_pool_bwd_prepare(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                          float* const* tables, const int64_t* table_rows,
                          const int64_t* const* uvalues, const int64_t* const* uoffsets,
                          const int64_t* value_caps, const int64_t* counts,
                          const int64_t* const* inverse, const float* const* grad_out, float lr,
                          int32_t apply_sgd, int64_t* const* grad_ids_out,
                          float* const* grad_rows_out, int64_t* grad_counts_out, void* scratch,
                          size_t scratch_bytes, recd_stream_t stream);
int recd_pool_bwd_finish(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                         float* const* tables, const int64_t* table_rows,
                         const int64_t* const* uvalues, const int64_t* const* uoffsets,
                         const int64_t* value_caps, const int64_t* counts,
                         const int64_t* const* inverse, const float* const* grad_out, float lr,
                         int32_t apply_sgd, int64_t* const* grad_ids_out,
                         float* const* grad_rows_out, int64_t* grad_counts_out, void* scratch,
                         size_t scratch_bytes, recd_stream_t stream);

/* recd_pool_bwd in up to four stages (same arguments and scratch; enqueue the
 * selected stages in this order, each stage after the previous ones): INVERSE
 * (setup + inverse CSR), OCCURRENCES (occurrence pairs + their sort by ID),
 * GRAD (unique-row gradients; reads grad_out), SCATTER (sorted scatter-add /
 * SGD).  _prepare = INVERSE | OCCURRENCES, _finish = GRAD | SCATTER.  With
 * OCCURRENCES on a side stream, GRAD only waits for INVERSE and runs while the
 * sort finishes. */
/* Where recd_pool_bwd's scratch holds the inverse CSR (valid once the
 * RECD_BWD_INVERSE stage ran; same arguments as the stages): per feature,
 * csr_start_out[f] -> int32[B + 1] row starts, csr_rows_out[f] -> uint32[B]
 * batch rows grouped by unique row (NULL for identity features).  Launches
 * nothing. */
int recd_pool_bwd_csr(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                      float* const* tables, const int64_t* table_rows,
                      const int64_t* const* uvalues, const int64_t* const* uoffsets,
                      const int64_t* value_caps, const int64_t* counts,
                      const int64_t* const* inverse, const float* const* grad_out, float lr,
                      int32_t apply_sgd, int64_t* const* grad_ids_out, float* const* grad_rows_out,
                      int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                      const int32_t** csr_start_out, const uint32_t** csr_rows_out);
#define RECD_BWD_INVERSE 1
#define RECD_BWD_OCCURRENCES 2
#define RECD_BWD_GRAD 4
#define RECD_BWD_SCATTER 8
/* The step's backward bookkeeping (bad-ID flag, per-table segment counts)
 * runs with RECD_BWD_INVERSE; RECD_BWD_SETUP runs it alone, and
 * RECD_BWD_SETUP_DONE makes RECD_BWD_INVERSE skip it -- so after a SETUP call
 * the INVERSE and OCCURRENCES stages may run concurrently on two streams
 * (they use separate scratch). */
#define RECD_BWD_SETUP 16
#define RECD_BWD_SETUP_DONE 32
int recd_pool_bwd_stages(int32_t stages, int32_t num_features, int64_t batch_size, int32_t dim,
                         int32_t mode, float* const* tables, const int64_t* table_rows,
                         const int64_t* const* uvalues, const int64_t* const* uoffsets,
                         const int64_t* value_caps, const int64_t* counts,
                         const int64_t* const* inverse, const float* const* grad_out, float lr,
                         int32_t apply_sgd, int64_t* const* grad_ids_out,
                         float* const* grad_rows_out, int64_t* grad_counts_out, void* scratch,
                         size_t scratch_bytes, recd_stream_t stream);

/* ------------------------------------------------------- transforms --
 * <- reader.apply_transform (reader.py:69-83) as used by reader.process
 * (reader.py:178-217) on IKJT unique values: per feature f,
 *   out[f][j] = identity | splitmix64(in[f][j]) mod params[f] | clamp(in, 0, params[f])
 * for j < min(*device_counts[f], num_values[f]) (device_counts may be NULL or
 * hold NULL entries: num_values[f] elements).  In-place allowed (out == in). */
int recd_transform(int32_t num_features, const int64_t* const* values_in,
                   int64_t* const* values_out, const int64_t* num_values,
                   const int64_t* const* device_counts, const int32_t* ops, const int64_t* params,
                   recd_stream_t stream);

/* ------------------------------------------------------- wire format --
 * <- tensors._serialize / serialize_kjt / serialize_ikjt (tensors.py:463-505):
 * the canonical little-endian byte stream written into a device buffer
 * (8-byte aligned).  inverse = NULL for a KJT (flag 0).  Element counts of
 * each key's offsets / values come from device_counts when given (IKJT: U and
 * N_u live on the device), else from the host caps.  *total_out (device) =
 * bytes written, or -1 when out_cap is too small (nothing written).
 * recd_wire_bound gives a host upper bound; scratch >= 2 KB. */
int64_t recd_wire_bound(int32_t num_keys, const char* const* key_names, int64_t batch_size,
                        int32_t has_inverse, const int64_t* offsets_caps, const int64_t* values_caps);
int recd_wire_serialize(int32_t num_keys, const char* const* key_names, int64_t batch_size,
                        const int64_t* inverse, const int64_t* const* offsets,
                        const int64_t* const* values, const int64_t* const* offsets_counts,
                        const int64_t* const* values_counts, const int64_t* offsets_caps,
                        const int64_t* values_caps, void* out, int64_t out_cap, int64_t* total_out,
                        void* scratch, size_t scratch_bytes, recd_stream_t stream);

/* ------------------------------------------------- sequence encoder --
 * <- trainer_sim.attention_pool (trainer_sim.py:347-391), config 4, over the
 * unique rows of one dedup group: per unique row u the tokens are the rows'
 * lists of every feature concatenated (embedding rows of tables[f]);
 *   out[u] = mean_i softmax(q k^T / sqrt(dim))_i v @ w_o,  q|k|v = x W_{q|k|v},
 * empty rows -> 0.  QKV on the tcgen05 tensor cores (BF16 in, FP32 accumulate).
 *   w_qkv_t  device bf16 [3*dim][dim] = [W_q | W_k | W_v]^T (K-major)
 *   w_o      device fp32 [dim][dim]
 *   counts   device [2F]: U (all equal) then N_u per feature
 *   out      device fp32 [>= U][dim];  err as in recd_pool_fwd.  dim: 64 or 128. */
size_t recd_attention_pool_scratch_bytes(int32_t num_features, int32_t dim,
                                         const int64_t* value_caps);
int recd_attention_pool(int32_t num_features, int64_t batch_size, int32_t dim,
                        const float* const* tables, const int64_t* table_rows,
                        const int64_t* const* uvalues, const int64_t* const* uoffsets,
                        const int64_t* value_caps, const int64_t* counts, const void* w_qkv_t,
                        const float* w_o, float* out, int64_t* err, void* scratch,
                        size_t scratch_bytes, recd_stream_t stream);
/* C[m][:] = A[m][:] B^T (bf16 row-major, FP32 accumulate in TMEM), M = *m_count
 * rows (device), (n, k) in {(192, 64), (384, 128), (128, 128)}. */
int recd_gemm_bf16_tn(int32_t n, int32_t k, const void* a, const void* b, void* c,
                      const int64_t* m_count, recd_stream_t stream);

/* Segmented stable LSD radix sort (one-sweep, 8-bit digits) of (uint32 key,
 * uint32 value) pairs by the low `bits` bits of the key: segment s occupies
 * [bases[s], bases[s] + caps[s]), *device_counts[s] elements valid.  The sorted
 * pairs end in keys/vals (*in_alt_out = 0) or keys_alt/vals_alt (1). */
size_t recd_sort_pairs_scratch_bytes(int32_t num_segments, const int64_t* bases, const int64_t* caps);
int recd_sort_pairs(int32_t num_segments, const int64_t* bases, const int64_t* caps,
                    const int64_t* const* device_counts, int32_t bits, uint32_t* keys, uint32_t* vals,
                    uint32_t* keys_alt, uint32_t* vals_alt, int32_t* in_alt_out, void* scratch,
                    size_t scratch_bytes, recd_stream_t stream);

/* Source half: grad_u_out[f] ([U x dim]) = grad_u of recd_pool_bwd (avg scaled). */
size_t recd_grad_unique_scratch_bytes(int32_t num_features, int64_t batch_size);
int recd_grad_unique(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                     const int64_t* const* uoffsets, const int64_t* counts,
                     const int64_t* const* inverse, const float* const* grad_out,
                     float* const* grad_u_out, void* scratch, size_t scratch_bytes,
                     recd_stream_t stream);

/* recd_grad_unique whose rows go straight to the owners' receive buffers (the
 * push of unique-row gradients fused into the segment reduce): feature f's row
 * u is stored at seg_dst[f * num_segs + j] + (*seg_row0[f * num_segs + j] + u) * dim
 * for every j < num_segs (<= 8; seg_row0 on the device; seg_dst may be peer memory). */
int recd_grad_unique_scatter(int32_t num_features, int64_t batch_size, int32_t dim, int32_t mode,
                             const int64_t* const* uoffsets, const int64_t* counts,
                             const int64_t* const* inverse, const float* const* grad_out,
                             int32_t num_segs, const int64_t* const* seg_row0,
                             float* const* seg_dst, void* scratch, size_t scratch_bytes,
                             recd_stream_t stream);

/* Owner half: grad_rows[f] holds one gradient row per unique row of feature f
 * (max_rows >= its row count, < 2^24); occurrences are reduced per ID in
 * ascending (feature, row, position) order and applied like recd_pool_bwd. */
size_t recd_sparse_sgd_scratch_bytes(int32_t num_features, const int64_t* value_caps);
int recd_sparse_sgd(int32_t num_features, int64_t max_rows, int32_t dim, float* const* tables,
                    const int64_t* table_rows, const int64_t* const* uvalues,
                    const int64_t* const* uoffsets, const int64_t* value_caps,
                    const int64_t* counts, const float* const* grad_rows, float lr,
                    int32_t apply_sgd, int64_t* const* grad_ids_out, float* const* grad_rows_out,
                    int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                    recd_stream_t stream);
/* recd_sparse_sgd in two halves (same arguments, same scratch): _prepare sorts
 * the occurrences by ID (needs only uvalues/uoffsets/counts), _finish reduces
 * grad_rows and applies the update. */
int recd_sparse_sgd_prepare(int32_t num_features, int64_t max_rows, int32_t dim, float* const* tables,
                            const int64_t* table_rows, const int64_t* const* uvalues,
                            const int64_t* const* uoffsets, const int64_t* value_caps,
                            const int64_t* counts, const float* const* grad_rows, float lr,
                            int32_t apply_sgd, int64_t* const* grad_ids_out, float* const* grad_rows_out,
                            int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                            recd_stream_t stream);
int recd_sparse_sgd_finish(int32_t num_features, int64_t max_rows, int32_t dim, float* const* tables,
                           const int64_t* table_rows, const int64_t* const* uvalues,
                           const int64_t* const* uoffsets, const int64_t* value_caps,
                           const int64_t* counts, const float* const* grad_rows, float lr,
                           int32_t apply_sgd, int64_t* const* grad_ids_out, float* const* grad_rows_out,
                           int64_t* grad_counts_out, void* scratch, size_t scratch_bytes,
                           recd_stream_t stream);

/* ------------------------------------------------------- row sharding --
 * Every table is split into S row shards: shard(id) = id mod S, local row =
 * id div S; pair p = f * S + j is (table f, shard j), F * S <= 256, S <= 64.
 * count:    rowoff_out[f][j * batch_size + u] = exclusive offset of row u's
 *   shard-j values among all shard-j values of f (rows in order, values in
 *   row order); totals_out[p] (device) = values of f in shard j.
 * dispatch: every value v of unique row u goes to
 *   dst_ids[p][id_base[p] + rowoff[f][j][u] + k] = v div S (k = its rank
 *   among the row's shard-j values), and dst_rowoffs[p][row_base[p] + u] =
 *   id_base[p] + rowoff[f][j][u] when dst_rowoffs (and dst_rowoffs[p]) is
 *   set.  id_base / row_base: device int64[P]; id_base NULL = prefix of
 *   totals over the shards of f, row_base NULL = 0.  Destinations may be peer
 *   memory (recd_peer_import).
 * bucketize: count + dispatch into ids_out[f] (shard-major, then unique row,
 *   then position) and rowcnt_out[f][j * batch_size + u] = values of row u in
 *   shard j.
 * combine:   pooled_out[f][u] = sum over j = 0..num_blocks-1 (in that order) of
 *   blocks[f * num_blocks + j][u * dim ...] (the partial rows of shard j of
 *   feature f, F * num_blocks <= 256); avg divides by the row length;
 *   batch_size bounds the unique rows (launch geometry). */
size_t recd_shard_count_scratch_bytes(int32_t num_features, int32_t num_shards,
                                      int64_t batch_size);
int recd_shard_count(int32_t num_features, int32_t num_shards, int64_t batch_size,
                     const int64_t* const* uvalues, const int64_t* const* uoffsets,
                     const int64_t* counts, int64_t* const* rowoff_out, int64_t* totals_out,
                     void* scratch, size_t scratch_bytes, recd_stream_t stream);
int recd_shard_dispatch(int32_t num_features, int32_t num_shards, int64_t batch_size,
                        const int64_t* const* uvalues, const int64_t* const* uoffsets,
                        const int64_t* counts, const int64_t* const* rowoff,
                        const int64_t* totals, const int64_t* id_base, const int64_t* row_base,
                        int64_t* const* dst_ids, int64_t* const* dst_rowoffs,
                        recd_stream_t stream);
size_t recd_shard_scratch_bytes(int32_t num_features, int32_t num_shards, int64_t batch_size);
int recd_shard_bucketize(int32_t num_features, int32_t num_shards, int64_t batch_size,
                         const int64_t* const* uvalues, const int64_t* const* uoffsets,
                         const int64_t* counts, int64_t* const* ids_out, int64_t* const* rowcnt_out,
                         int64_t* totals_out, void* scratch, size_t scratch_bytes,
                         recd_stream_t stream);
int recd_shard_combine(int32_t num_features, int32_t num_blocks, int64_t batch_size, int32_t dim,
                       int32_t mode, const float* const* blocks, const int64_t* const* uoffsets,
                       const int64_t* counts, float* const* pooled_out, recd_stream_t stream);

/* ------------------------------------------- peer (NVLink) transport --
 * The sharded step without host synchronisation: every rank exports one
 * zeroed device allocation (recd_peer_alloc / _export), the others map it
 * (recd_peer_import), and kernels store straight into peer buffers.
 * Control block = int64 words at the start of every rank's allocation:
 *   [0, 64)          arrival flags: word s = last epoch rank s signalled here
 *   [64]             epoch of this rank's last exchange
 *   [65]             error: 1 = some peer did not arrive within timeout_ns
 *   [128, 128+2RP)   meta[s][p] = IDs source s sends to pair p,
 *                    meta[s][P + p] = unique rows of f(p) at source s
 *   then this rank's plan, at 128 + 2RP:
 *     [0, P)           src_id_base[p]  = sum_{s < rank} meta[s][p]
 *     [P, 2P)          src_row_base[p] = sum_{s < rank} meta[s][P + p]
 *     [2P, 2P+2Q)      owned-pair counts: rows of owned[q] (all sources), then IDs
 *     [2P+2Q, +Q*R)    owner_row_base[q * R + s] = sum_{s' < s} meta[s'][P + owned[q]]
 * exchange: with totals (device int64[P]) stores meta[rank] = (totals,
 *   counts[p / S] of every pair) into every rank's block, then barriers, then
 *   writes the plan; with totals NULL it is a bare barrier.  peer_ctl host
 *   [R]: every rank's control block as mapped here (own included); owned
 *   host [Q] pair ids.  Never waits longer than timeout_ns; on timeout it sets
 *   the error word and every later exchange returns at once.
 * copy_rows: segment i copies ctl[count_idx] rows of row_bytes (multiple of
 *   16) from src + ctl[src_off_idx] rows to dst + ctl[dst_off_idx] rows (an
 *   index < 0 reads as 0); segs is a DEVICE array; max_rows bounds every
 *   count (launch geometry). */
#define RECD_PEER_HANDLE_BYTES 64
#define RECD_CTL_META 128
typedef struct recd_row_seg {
  const void* src;
  void* dst;
  int64_t count_idx;
  int64_t src_off_idx;
  int64_t dst_off_idx;
} recd_row_seg;
int64_t recd_peer_ctl_words(int32_t num_ranks, int32_t num_pairs, int32_t num_owned);
int recd_peer_alloc(size_t bytes, void** ptr_out);
int recd_peer_free(void* ptr);
int recd_peer_export(const void* ptr, void* handle_out);
int recd_peer_import(const void* handle, void** ptr_out);
int recd_peer_close(void* ptr);
int recd_peer_exchange(int32_t num_ranks, int32_t rank, int32_t num_pairs, int32_t num_shards,
                       int32_t num_owned, const int32_t* owned, void* const* peer_ctl,
                       const int64_t* totals, const int64_t* counts, int64_t timeout_ns,
                       recd_stream_t stream);
int recd_peer_copy_rows(int32_t num_segments, const recd_row_seg* segs, const int64_t* ctl,
                        int32_t row_bytes, int64_t max_rows, recd_stream_t stream);

/* Batched copy of num_segments (src, dst, bytes) device segments in one
 * launch (packing of exchange buffers).  host_staging / descs: a host and a
 * device buffer of recd_batched_copy_desc_bytes(num_segments) bytes; the
 * segment table goes host_staging -> descs with one async copy, so
 * host_staging must stay untouched until the stream reaches this call. */
size_t recd_batched_copy_desc_bytes(int32_t num_segments);
int recd_batched_copy(int32_t num_segments, const void* const* src, void* const* dst,
                      const int64_t* bytes, void* host_staging, void* descs, recd_stream_t stream);

/* Segmented exclusive scan of int64 (segment s: caps[s] entries, or
 * device_counts[s] when device_counts is not NULL); totals_out nullable. */
size_t recd_exclusive_scan_scratch_bytes(int32_t num_segments, const int64_t* caps);
int recd_exclusive_scan(int32_t num_segments, const int64_t* const* in, int64_t* const* out,
                        const int64_t* caps, const int64_t* device_counts, int64_t* totals_out,
                        void* scratch, size_t scratch_bytes, recd_stream_t stream);

/* --------------------------------------------------- jagged index select --
 * Output row k of feature f = input row indices[k] (same indices for every
 * feature, as ikjt_to_kjt does with inverse_lookup).
 * plan: out_offsets[f] (int64[n_idx]) and totals_out[f] (device) = output
 *       value counts; err (device int64[1]) = first position p with
 *       indices[p] outside [0, num_rows), else RECD_NO_ERROR.
 * copy: out_values[f] (int64[total_f]).
 */
size_t recd_jagged_scratch_bytes(int32_t num_features, int64_t num_indices);
int recd_jagged_index_select_plan(int32_t num_features, const int64_t* const* offsets,
                                  int64_t num_rows, const int64_t* num_values,
                                  const int64_t* indices, int64_t num_indices,
                                  int64_t* const* out_offsets, int64_t* totals_out, int64_t* err,
                                  void* scratch, size_t scratch_bytes, recd_stream_t stream);
int recd_jagged_index_select_copy(int32_t num_features, const int64_t* const* values,
                                  const int64_t* const* offsets, int64_t num_rows,
                                  const int64_t* num_values, const int64_t* indices,
                                  int64_t num_indices, const int64_t* const* out_offsets,
                                  int64_t* const* out_values, recd_stream_t stream);

/* ------------------------------------------------------- slice renumber --
 * DP slice of an IKJT without re-hashing: for rows [start, stop) of
 * `inverse` (values in [0, num_unique)), new_inverse = first-occurrence
 * renumbering and order_out[k] = old unique row of new unique row k;
 * count_out (device int64[1]) = number of surviving unique rows.
 */
size_t recd_slice_scratch_bytes(int64_t num_unique, int64_t num_rows);
int recd_slice_renumber(const int64_t* inverse, int64_t start, int64_t stop, int64_t num_unique,
                        int64_t* new_inverse_out, int64_t* order_out, int64_t* count_out,
                        void* scratch, size_t scratch_bytes, recd_stream_t stream);

/* ------------------------------------------------------- partial IKJT ---
 * build_partial_ikjt (tensors.py:311-360) of one key, from recd_dedup's
 * unique rows (uvalues / uoffsets = row starts, num_uvalues values) and its
 * inverse lookup: values_out[0 .. *num_values_out) is the shared value buffer
 * (capacity num_uvalues), windows_out[2 i], [2 i + 1] = (offset, length) of
 * batch row i, bit-exact with the reference's greedy batch-order encoder.
 * Synchronises `stream` once per speculation round (*rounds_out, nullable).
 */
size_t recd_partial_ikjt_scratch_bytes(int64_t num_unique, int64_t num_uvalues);
int recd_partial_ikjt(int64_t batch_size, int64_t num_unique, const int64_t* uvalues,
                      const int64_t* uoffsets, int64_t num_uvalues, const int64_t* inverse,
                      int64_t* values_out, int64_t* windows_out, int64_t* num_values_out,
                      int64_t* rounds_out, void* scratch, size_t scratch_bytes, recd_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* RECD_H_ */
