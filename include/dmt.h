/*
 * dmt.h -- C ABI of libdmt.so, the sm_100a kernels of the DMT / SPTT hot path
 * (arXiv 2403.00877).  Plain pointers, sizes and a cudaStream_t; no torch
 * types.  Every entry point is stream-ordered, never allocates device memory
 * and never synchronises the host; callers own all buffers (workspace sizes
 * are queried with the *_workspace_size functions).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/towersim):
 *   dmt_lengths_to_offsets   -- offsets of SparseBatch bags           embedding.py:215-226
 *   dmt_kjt_bucketize        -- step a bundling per shard owner       exchange.py:162-178
 *   dmt_pooled_lookup_fwd    -- lookup / _shard_lookup (+ fused step-c
 *                               permute and step-d stacking)          embedding.py:64-85,
 *                                                                      exchange.py:130-146,324-365
 *   dmt_assemble             -- _combine_pieces, step-e regroup,
 *                               step-f concat, realign                exchange.py:112-127,397-437,
 *                                                                      448-449,465-486
 *   dmt_batched_copy         -- in-process all_to_all delivery         simnet.py:117-146
 *   dmt_pooled_lookup_bwd    -- (absent in the reference: backward of
 *                               lookup with fused SGD / row-wise Adagrad)
 *   dmt_gemm                 -- tm_dlrm_forward / crossnet_layer /
 *                               tm_dcn_forward matmuls + epilogues    towermod.py:110-158
 *
 * Status codes map onto the reference exception classes (errors.py):
 */
#ifndef DMT_H_
#define DMT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dmt_stream_t; /* == cudaStream_t */

enum dmt_status {
  DMT_OK = 0,
  DMT_ERR_DOMAIN = -1,      /* DomainError        errors.py:11  */
  DMT_ERR_SHAPE = -2,       /* ShapeError         errors.py:23  */
  DMT_ERR_PLAN = -3,        /* PlanError          errors.py:27  */
  DMT_ERR_LOOKUP = -4,      /* TableLookupError   errors.py:35  */
  DMT_ERR_PROTOCOL = -5,    /* ProtocolError      errors.py:19  */
  DMT_ERR_UNSUPPORTED = -6, /* DomainError (unsupported dtype / shape) */
  DMT_ERR_CUDA = -10        /* CUDA launch / runtime failure */
};

enum dmt_dtype { DMT_F32 = 0, DMT_BF16 = 1, DMT_F64 = 2, DMT_F16 = 3 };

enum dmt_pooling { DMT_POOL_NONE = 0, DMT_POOL_SUM = 1, DMT_POOL_MEAN = 2 };

/* device-side error flag bits (dmt_pooled_lookup_* `err`) */
enum dmt_err_bits { DMT_EBIT_INDEX = 1, DMT_EBIT_BAGLEN = 2 };

/* ---------------------------------------------------------------- KJT ---- */

/* offsets[0] = 0, offsets[i+1] = offsets[i] + lengths[i]  (n lengths).
 * `scratch` must hold dmt_lengths_to_offsets_workspace_size(n) bytes. */
size_t dmt_lengths_to_offsets_workspace_size(int64_t n);
int dmt_lengths_to_offsets(const int32_t* lengths, int64_t n, int64_t* offsets,
                           void* scratch, dmt_stream_t stream);

/* Step a bundling.  Input: one rank's KJT, keys (features) major:
 * lengths[F*B], offsets[F*B+1], values[offsets[F*B]].
 * slot_feature[num_slots]: feature position shipped by each send slot (slots
 * ordered owner-major, shard-id order inside an owner -- exchange.py:172-178).
 * slot_value_offset[num_slots+1]: where each slot's values start in
 * out_values (exclusive prefix of the slots' nnz; all device arrays).
 * Output: out_lengths[num_slots*B], out_values. */
int dmt_kjt_bucketize(const int32_t* lengths, const int64_t* offsets, const int32_t* values,
                      int32_t B, int32_t num_slots, const int32_t* slot_feature,
                      const int64_t* slot_value_offset, int32_t* out_lengths,
                      int32_t* out_values, dmt_stream_t stream);

/* Device-side slot offsets (when per-feature nnz is not known on the host):
 * slot_value_offset[s+1] - slot_value_offset[s] = nnz(slot_feature[s]). */
/* Step a over NVLink peer stores: slot s's lengths / values are written to
 * slot_dst[s] = {int32* len, int32* val, int64 room} (device array; peer-mapped
 * pointers for remote owners), values bounded by room (else empty bags). */
typedef struct dmt_slot_dst {
  int32_t* len;
  int32_t* val;
  int64_t room;
} dmt_slot_dst;
int dmt_kjt_bucketize_peer(const int32_t* lengths, const int64_t* offsets, const int32_t* values, int32_t B,
                           int32_t num_slots, const int32_t* slot_feature, const void* slot_dst,
                           dmt_stream_t stream);

/* Capacity-padded step a (ragged batches under CUDA graphs; no count
 * exchange): slots are bucketized at fixed capacity offsets, the owner packs
 * region seg (= src-major, shard order; bags seg*B .. seg*B+B-1) from
 * src + seg_src_start[seg] to dst + offsets[seg*B], count from the packed
 * offsets of the received lengths.  check_capacity sets *flag |= 1 when a
 * feature's nnz exceeds its capacity (values past it would be dropped). */
int dmt_kjt_compact(const int32_t* src, const int64_t* offsets, int32_t B, int32_t num_segments,
                    const int64_t* seg_src_start, int32_t* dst, dmt_stream_t stream);
int dmt_kjt_check_capacity(const int64_t* offsets, int32_t B, int32_t F, const int64_t* capacity, int32_t* flag,
                           dmt_stream_t stream);
int dmt_kjt_slot_offsets(const int64_t* offsets, int32_t B, int32_t num_slots,
                         const int32_t* slot_feature, int64_t* slot_value_offset,
                         dmt_stream_t stream);

/* ------------------------------------------------------- pooled lookup ---- */

/* One segment = `nbags` consecutive bags of one table shard whose pooled rows
 * go to out + b*out_ld (b = 0..nbags-1).  Bag i of the segment is global bag
 * bag_begin + i of the (offsets, indices) arrays.  Indices are table-global;
 * rows outside [row_begin, row_begin+rows) are skipped when `row_filter` (row-
 * wise shards, exchange.py:138-144) and flagged DMT_EBIT_INDEX otherwise. */
typedef struct dmt_lookup_segment {
  const void* weights; /* shard rows, row-major, row r at weights + (r-row_begin)*ld */
  void* out;           /* fwd: pooled output; bwd: gradient of the pooled output */
  void* state;         /* bwd row-wise Adagrad accumulator (float per row) or NULL */
  int64_t ld;          /* weights row stride (elements) */
  int64_t out_ld;      /* out row stride (elements) */
  int64_t bag_begin;   /* first global bag */
  int64_t row_begin;   /* first table row held by the shard */
  int64_t key_base;    /* bwd: base of this shard's rows in the sort key space */
  int32_t rows;        /* rows held by the shard */
  int32_t width;       /* columns of the shard */
  int32_t nbags;       /* bags in this segment */
  int32_t pooling;     /* dmt_pooling */
  int32_t row_filter;  /* 1 = row-wise shard: filter + rebase */
  int32_t table_rows;  /* row-wise shards: rows of the whole table (> 0: indices
                        * outside [0, table_rows) flag DMT_EBIT_INDEX even though
                        * every shard filters them); 0 = no global check */
} dmt_lookup_segment;

/* Forward.  All segments share dtype.  Accumulation is fp32 (f32/bf16/f16) or
 * fp64 (f64) in bag order -- bit-exact against the reference's sequential sum.
 * err (device int32, may be NULL) receives dmt_err_bits.  segs is the device
 * copy of the segment table, segs_host the identical host copy (used only for
 * launch shaping: widths, alignment, bag counts). */
int dmt_pooled_lookup_fwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host,
                          int32_t num_segs, const int64_t* offsets, const int32_t* indices,
                          int32_t dtype, int32_t* err, dmt_stream_t stream);

/* Backward with fused optimizer (absent in the reference).
 * segs[i].out is the gradient of the pooled rows, segs[i].weights is updated
 * in place (const is cast away), key_base/rows define a disjoint key range per
 * shard (segments of the same shard share it).  The segments must tile bags
 * [0, num_bags) in order (offsets[0] == 0), as the owner's received KJT does.  Duplicate rows are reduced
 * after a stable radix sort, so the update is deterministic.
 * optimizer: 0 = SGD (w -= lr*g), 1 = row-wise Adagrad
 * (s += mean(g^2); w -= lr*g/(sqrt(s)+eps)). */
enum dmt_optimizer { DMT_OPT_SGD = 0, DMT_OPT_ROWWISE_ADAGRAD = 1 };
size_t dmt_pooled_lookup_bwd_workspace_size(int64_t nnz, int64_t key_space, int64_t num_bags);
int dmt_pooled_lookup_bwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host,
                          int32_t num_segs, const int64_t* offsets, const int32_t* indices,
                          int64_t nnz, int64_t key_space, int32_t dtype, int32_t optimizer,
                          float lr, float eps, void* workspace, size_t workspace_bytes,
                          dmt_stream_t stream);

/* The same in two halves: _prepare (sort keys, per-bag records, radix sort)
 * needs only the indices and can run while the tower module computes; _apply
 * (segment reduce + optimizer) then consumes the gradients.  Both must use the
 * same workspace, segment table and sizes. */
int dmt_pooled_lookup_bwd_prepare(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host,
                                  int32_t num_segs, const int64_t* offsets, const int32_t* indices,
                                  int64_t nnz, int64_t key_space, int32_t dtype, void* workspace,
                                  size_t workspace_bytes, dmt_stream_t stream);
int dmt_pooled_lookup_bwd_apply(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host,
                                int32_t num_segs, int64_t nnz, int64_t key_space, int32_t dtype,
                                int32_t optimizer, float lr, float eps, void* workspace,
                                size_t workspace_bytes, dmt_stream_t stream);

/* ------------------------------------------------------------ assemble ---- */

/* dst[r, col0 + j] = sum_{s < nsrc} src_s[r*ld_s + j]   for r < rows, j < width.
 * Sums run in source order in fp64 (f32/f64/bf16) and round once: column
 * shards (nsrc = 1) are copies, row-wise partials (nsrc > 1) are summed in
 * row-range order like exchange.py:118-123. */
typedef struct dmt_assemble_block {
  int64_t dst_col;
  int32_t width;
  int32_t nsrc;
  int32_t first_src; /* index into the src table */
  /* multi-source (summed) blocks: bit s set = source s starts a new inner
   * partial sum; the result is ((s0 + s1 + ..) + (sk + ..) + ..) in fp64 --
   * the row-wise reduce-scatter order (per-owner partial, then group order,
   * towersim/exchange.py:380-395 + simnet.py:173-192).  0 = one flat sum in
   * source order (exchange.py:112-127). */
  uint32_t groups;
} dmt_assemble_block;

typedef struct dmt_src {
  const void* ptr;
  int64_t ld;
} dmt_src;

int dmt_assemble(const dmt_assemble_block* blocks, int32_t num_blocks, int32_t max_width,
                 const dmt_src* srcs, int64_t rows, void* dst, int64_t dst_ld, int32_t dtype,
                 dmt_stream_t stream);

/* n byte copies in one launch (in-process collective delivery). */
typedef struct dmt_copy {
  const void* src;
  void* dst;
  int64_t bytes;
} dmt_copy;
int dmt_batched_copy(const dmt_copy* copies, int32_t n, int64_t max_bytes, dmt_stream_t stream);

/* Batched 2-D strided copies: rows x width elements of elem_bytes each,
 * dst[r*dst_ld + j] = src[r*src_ld + j] (pack/unpack of exchange blocks in the
 * backward: f^-1 and d^-1 send buffers). */
typedef struct dmt_copy2d {
  const void* src;
  void* dst;
  int64_t src_ld;
  int64_t dst_ld;
  int64_t rows;
  int64_t width;
} dmt_copy2d;
/* elem_bytes < 0: the caller guarantees every copy is 16-byte granular
 * (pointers, strides, widths) -> 16-byte vector moves. */
int dmt_batched_copy2d(const dmt_copy2d* copies, int32_t n, int32_t elem_bytes, int64_t max_elems,
                       dmt_stream_t stream);

/* ---------------------------------------------------------------- GEMM ---- */

/* D[m, n] = epilogue( sum_k A[m, k] * B[n, k] )   (both operands K-major)
 *   bf16 / f16 operands: tcgen05.mma kind::f16, fp32 accumulate in TMEM
 *   f32 operands:        tcgen05.mma kind::tf32, 3xTF32 split (fp32 accuracy)
 * Epilogues (fp32 math on the TMEM accumulator):
 *   DMT_EPI_BIAS : v = acc + bias[n]
 *   DMT_EPI_CROSS: v = x0[m, n] * (acc + bias[n]) + xl[m, n]   (crossnet_layer,
 *                  towermod.py:132-139); optionally u = acc + bias stored to aux
 *   DMT_EPI_ACC  : v = acc + beta*C[m, n] (C = d)
 * Output row m goes to d + (m / rows_per_group)*ld_group + (m % rows_per_group)*ld_d,
 * so the per-feature DLRM projection can write straight into the tower output. */
enum dmt_epilogue {
  DMT_EPI_NONE = 0,
  DMT_EPI_BIAS = 1,
  DMT_EPI_CROSS = 2,
  DMT_EPI_ACC = 3,
  /* DCN backward, one layer (towermod.py:132-139 differentiated):
   *   g  = acc + beta*C            -> d      (dL/dx_{l+1})
   *   gu = g * x0                  -> aux    (dL/du_l, A operand of the next GEMMs)
   *   dx0 (+)= g * u_l             -> aux2   (fp32, accumulated if FLAG_AUX2_ACCUM)
   * with x0 = args.x0 and u_l = args.xl. */
  DMT_EPI_DCN_BWD = 4,
  /* last DCN layer: d = acc + beta*C + aux2 (fp32 dx0)  ->  dX of the tower,
   * or, with npairs > 0, d = acc + beta*C + sum_j pair_g[j] * pair_u[j]
   * (dx0 = sum_l g_{l+1} * u_l read straight from the saved layer tensors, so
   * the per-layer DCN_BWD epilogues need no fp32 dx0 read-modify-write:
   * DCN_BWD with aux2 = NULL only writes g and gu). */
  DMT_EPI_DCN_FINAL = 5,
  /* MLP layers (the DLRM dense / over arch): d = max(acc + bias, 0) */
  DMT_EPI_BIAS_RELU = 6,
  /* MLP backward: d = acc * (x0 > 0) -- dX of layer l masked by the saved
   * ReLU output of layer l-1 (x0, in_dtype, row stride ld_x) */
  DMT_EPI_RELU_BWD = 7
};

#define DMT_GEMM_MAX_PAIRS 4
#define DMT_GEMM_MAX_OUT_GROUPS 8
#define DMT_GEMM_MAX_COL_GROUPS 32

/* dmt_gemm_args.flags: operand stored transposed (MN-major).  TRANS_A: `a`
 * holds A^T as a [k, m] matrix with row stride lda (m contiguous); TRANS_B:
 * `b` holds B^T as [k, n] with row stride ldb.  Read straight by TMA, no
 * transpose pass (dW = G^T X, dX = G W). */
enum dmt_gemm_flags {
  DMT_GEMM_TRANS_A = 1,
  DMT_GEMM_TRANS_B = 2,
  DMT_GEMM_AUX2_ACCUM = 4,
  /* acc is scaled by args.alpha before the epilogue: with DMT_EPI_ACC,
   * beta = 1 and c = d = W this is a fused SGD step W -= lr * dW (alpha = -lr) */
  DMT_GEMM_SCALE_ACC = 8,
  /* tuning overrides (benchmarks): no L2 prefetch of the epilogue operands;
   * force the tile width BN = 64 * ((flags & BN_MASK) >> BN_SHIFT) */
  DMT_GEMM_NO_PREFETCH = 16,
  /* force / forbid cta_group::2 pairs (256 x BN tiles, B split across the
   * pair); default: pairs for BN 256 tiles of wide outputs (n >= 2048) */
  DMT_GEMM_CLUSTER = 32,
  DMT_GEMM_SINGLE_CTA = 64,
  DMT_GEMM_BN_SHIFT = 8,
  DMT_GEMM_BN_MASK = 0xF00,
  /* tuning override: keep the output stores of the register-direct epilogue
   * per-thread instead of TMA bulk stores */
  DMT_GEMM_NO_TMA_STORE = 0x1000
};

typedef struct dmt_gemm_args {
  const void* a;   /* [m, k] row stride lda */
  const void* b;   /* [n, k] row stride ldb */
  void* d;         /* output */
  const float* bias;
  const void* x0;  /* CROSS: [m, n] row stride ld_x */
  const void* xl;
  void* aux;       /* CROSS: u = acc + bias, row stride ld_x (may be NULL); DCN_BWD: gu */
  const void* c;   /* ACC / DCN_*: accumulate source C[m, n] (row stride ld_d; NULL = d) */
  float* aux2;     /* DCN_*: fp32 dx0, row stride ld_x */
  int64_t m, n, k;
  int64_t lda, ldb, ld_d, ld_x;
  int64_t rows_per_group, ld_group;
  float beta;
  float alpha;       /* with DMT_GEMM_SCALE_ACC */
  int32_t in_dtype;  /* dmt_dtype of a, b (and x0/xl/aux for CROSS) */
  int32_t out_dtype; /* dmt_dtype of d */
  int32_t epilogue;
  int32_t flags;     /* dmt_gemm_flags */
  /* DCN_FINAL pair sum (16-bit operands, row stride ld_x) */
  int32_t npairs;
  int32_t pad_;
  const void* pair_g[DMT_GEMM_MAX_PAIRS];
  const void* pair_u[DMT_GEMM_MAX_PAIRS];
  /* DCN_BWD, optional: fused bias gradient.  Column sums of the stored gu per
   * (128-row tile, 32-row quarter): fp32 [dmt_gemm_colsum_rows(m), n]; finish
   * with dmt_column_sum_parts.  Needs n % 32 == 0 and 16-byte aligned rows. */
  float* colsum_part;
  /* split-K (few output tiles, long K: the dW GEMMs of the DLRM tower module
   * and MLPs): ksplit > 1 partitions K into ksplit ranges computed by
   * separate CTAs into splitk_ws (fp32, ksplit * m * n), then summed in split
   * order (deterministic) with the NONE / ACC epilogue applied.  0/1 = off. */
  int32_t ksplit;
  /* scattered output rows (a GEMM fused with the exchange that follows it):
   * with n_out_groups > 0, row m goes to out_group[m / rows_per_group] +
   * (m % rows_per_group) * ld_d -- e.g. the tower module's projection writes
   * each destination tower's block straight into that rank's step-f receive
   * buffer over NVLink (peer-mapped pointers). */
  int32_t n_out_groups;
  float* splitk_ws;
  void* out_group[DMT_GEMM_MAX_OUT_GROUPS];
  /* scattered output column blocks: with n_col_groups > 0, column n goes to
   * col_group[n / col_group_width] + m * col_group_ld[g] + n % width -- e.g.
   * the DCN backward's final dX GEMM stores each shard's columns straight into
   * its owner's gradient buffer over NVLink (step d^-1 fused); width a
   * multiple of 32 covering n exactly. */
  int32_t n_col_groups;
  int32_t col_group_width;
  void* col_group[DMT_GEMM_MAX_COL_GROUPS];
  int64_t col_group_ld[DMT_GEMM_MAX_COL_GROUPS];
} dmt_gemm_args;

/* rows of the colsum_part buffer for an m-row GEMM */
int64_t dmt_gemm_colsum_rows(int64_t m);
/* out[c] = sum_r part[r, c]  (fp64 accumulation in row order, deterministic) */
int dmt_column_sum_parts(const float* part, int64_t rows, int64_t cols, float* out, dmt_stream_t stream);

int dmt_gemm(const dmt_gemm_args* args, dmt_stream_t stream);

/* fp32 operands: `args->a` / `args->b` hold the tf32 "hi" parts and a_lo /
 * b_lo the residuals (see dmt_split_tf32); bf16/f16 ignore a_lo / b_lo. */
int dmt_gemm_ex(const dmt_gemm_args* args, const void* a_lo, const void* b_lo,
                dmt_stream_t stream);

/* hi = tf32(x) (round to nearest), lo = tf32(x - hi): the 3xTF32 operand split. */
int dmt_split_tf32(const float* x, float* hi, float* lo, int64_t n, dmt_stream_t stream);

/* out[j, i] = in[i, j]  (rows x cols, row strides ld_in / ld_out) */
int dmt_transpose(const void* in, int64_t rows, int64_t cols, int64_t ld_in, void* out,
                  int64_t ld_out, int32_t dtype, dmt_stream_t stream);

/* out[c] = sum_r in[r, c] (fp32 out, fp64 accumulation, deterministic). */
size_t dmt_column_sum_workspace_size(int64_t rows, int64_t cols);
int dmt_column_sum(const void* in, int64_t rows, int64_t cols, int64_t ld, float* out,
                   int32_t dtype, void* workspace, size_t workspace_bytes, dmt_stream_t stream);

/* Element-wise helpers of the DCN backward:
 *   gu = g * x0 ; dx0 += g * u         (dmt_cross_bwd_pointwise)
 * all [rows, cols] contiguous; gu/g in in_dtype, dx0 fp32. */
int dmt_cross_bwd_pointwise(const void* g, const void* x0, const void* u, void* gu, float* dx0,
                            int64_t n, int32_t dtype, dmt_stream_t stream);

/* dx0 = (accumulate ? dx0 : 0) + g * u  (g, u in dtype; dx0 fp32; n elements,
 * 16-byte aligned): one term of the crossnet's dx0 = sum_l g_{l+1} * u_l
 * (derivative of towermod.py:132-139), run on a side stream beside the dW
 * GEMMs so the dX GEMM epilogues stay light. */
int dmt_dcn_dx0_term(const void* g, const void* u, float* dx0, int64_t n, int32_t dtype, int32_t accumulate,
                     dmt_stream_t stream);

/* Element-wise tail of the crossnet backward after the last per-layer dX
 * GEMM: dx0 in one streaming pass over the saved layer tensors (instead of
 * nlayers fp32 read-modify-write passes), then the bias column sums
 * (16-bit dtype, all [rows, cols] contiguous, cols % 8 == 0,
 * 1 <= nlayers <= 4):
 *   dx0 = sum_{l = nlayers-1 .. 0} g[l] * u[l]        (fp32; the order of
 *         dmt_dcn_dx0_term's sequence: bit-identical)
 *   colsums[l][c] = sum_r gu[l][r, c]                  (= dmt_column_sum;
 *                                                        colsums == NULL: dx0 only)
 * Replaces nlayers dx0 terms plus nlayers column sums (derivative of
 * towermod.py:132-139; the reference has no backward). */
size_t dmt_dcn_side_fused_workspace_size(int64_t rows, int64_t cols, int32_t nlayers);
int dmt_dcn_side_fused(const void* const* g, const void* const* u, const void* const* gu, int32_t nlayers,
                       int64_t rows, int64_t cols, float* dx0, float* const* colsums, int32_t dtype,
                       void* workspace, size_t workspace_bytes, dmt_stream_t stream);

/* w -= lr * g  (w in dtype, g fp32), n elements */
/* Loss head of the full DCN + SPTT training step (the reference has no
 * training): binary cross-entropy on logits z[n],
 * dz = scale * (sigmoid(z) - y), *loss = scale * sum BCE (one block, fixed
 * reduction order; loss may be NULL). */
int dmt_bce_with_logits(const void* z, const float* y, int64_t n, int32_t dtype, float scale, void* dz,
                        float* loss, dmt_stream_t stream);

int dmt_sgd_dense(void* w, const float* g, int64_t n, float lr, int32_t dtype,
                  dmt_stream_t stream);

/* DLRM pairwise dot interaction around SPTT (the C3 model; PAPER.md:359-361,
 * TorchRec InteractionArch): V = [dense (B, dim) | sparse (B, num_sparse*dim)];
 * out (B, dim + P), P = (num_sparse+1) num_sparse / 2: out[:, :dim] = dense,
 * out[:, dim + i(i-1)/2 + j] = <V_i, V_j> for i > j.  fp32 accumulation.
 * The backward writes d_dense (B, dim) and d_sparse (B, num_sparse*dim).
 * dtype: DMT_F32 or DMT_BF16 (all operands). */
/* dz = dy * (y > 0) (ReLU backward where no GEMM epilogue can take it) */
int dmt_relu_bwd(const void* dy, const void* y, void* dz, int64_t n, int32_t dtype, dmt_stream_t stream);
int dmt_dot_interaction_fwd(const void* dense, int64_t ld_dense, const void* sparse, int64_t ld_sparse,
                            int32_t num_sparse, int32_t dim, int64_t batch, void* out, int64_t ld_out,
                            int32_t dtype, dmt_stream_t stream);
int dmt_dot_interaction_bwd(const void* grad_out, int64_t ld_grad_out, const void* dense, int64_t ld_dense,
                            const void* sparse, int64_t ld_sparse, int32_t num_sparse, int32_t dim,
                            int64_t batch, void* d_dense, int64_t ld_d_dense, void* d_sparse,
                            int64_t ld_d_sparse, int32_t dtype, dmt_stream_t stream);

/* Tower gradient all-reduce fused with SGD over NVLink peer memory (replaces
 * the NCCL all-reduce of TM gradients over the tower comm, SURVEY §8e "bwd",
 * + dmt_sgd_dense): w -= lr * (g[0] + g[1] + ... + g[nsrc-1]), summed in that
 * order in fp32.  g is a HOST array of nsrc device pointers (this rank's own
 * buffer and IPC-mapped peer buffers, 16-byte aligned), nsrc <=
 * DMT_MAX_PEER_SRCS; every member passing the same order gets bit-identical
 * replicas.  The caller orders it after a barrier on the peers' writes. */
#define DMT_MAX_PEER_SRCS 8
/* Completion barrier of a peer group over NVLink (see peer_barrier_kernel):
 * epoch = this rank's device counter for the group kind; remote_slots[i] =
 * other member i's (peer-mapped) flag for this rank, local_slots[i] = this
 * rank's flag for member i (HOST arrays of n <= DMT_MAX_PEER_SRCS device
 * pointers).  *err |= 1 if a member does not arrive within ~2^26 polls. */
int dmt_peer_barrier(int32_t* epoch, int32_t* const* remote_slots, int32_t* const* local_slots, int32_t n,
                     int32_t* err, dmt_stream_t stream);
int dmt_peer_sum_sgd(void* w, const float* const* g, int32_t nsrc, int64_t n, float lr, int32_t dtype,
                     dmt_stream_t stream);

/* dst (dtype_out) = src (dtype_in), n elements */
int dmt_convert(const void* src, int32_t dtype_in, void* dst, int32_t dtype_out, int64_t n,
                dmt_stream_t stream);

/* Library identification: returns a static string ("libdmt <version> sm_100a"). */
const char* dmt_version(void);

/* Enable NVLink peer access from the current device to `peer_device` (needed
 * before kernels store into another GPU's IPC-mapped exchange buffers). */
int dmt_enable_peer_access(int peer_device);

/* CUDA IPC for the NVLink peer exchange.  dmt_ipc_export writes the 64-byte
 * handle of the allocation holding `ptr` and ptr's byte offset inside it;
 * dmt_ipc_open maps a peer's handle into the CURRENT device's context (peer
 * access enabled lazily) and returns the allocation base; dmt_ipc_close
 * unmaps it.  Replaces nothing in the reference (its fabric is simulated,
 * towersim/simnet.py); it is the B200 transport under step d / step f. */
int dmt_ipc_export(const void* ptr, void* handle64, int64_t* offset);
int dmt_ipc_open(const void* handle64, void** base);
int dmt_ipc_close(void* base);

/* Text of the last CUDA error behind a DMT_ERR_CUDA status (this thread). */
const char* dmt_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* DMT_H_ */
