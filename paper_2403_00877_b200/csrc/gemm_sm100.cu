// Tower-module GEMMs on the 5th-generation tensor cores.
//
//   D[m, n] = epilogue( sum_k A[m, k] * B[n, k] )       A, B K-major
//
// Reference math: tm_dlrm_forward (towersim/towermod.py:110-129: x W^T + b),
// crossnet_layer (towermod.py:132-139: x0 * (xl W^T + b) + xl) and the DCN
// projection (towermod.py:158).  Weights are (out, in) row-major exactly like
// the reference, i.e. already K-major for the B operand.
//
// Kernel anatomy (one CTA per SM, persistent over output tiles):
//   warp 0      : TMA producer  -- cp.async.bulk.tensor 2D, SWIZZLE_128B, an
//                 mbarrier full/empty ring of STAGES operand slots
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer; commits
//                 free smem slots and publish finished accumulators
//   warps 2..9  : epilogue -- tcgen05.ld TMEM -> registers, bias / crossnet
//                 gate / DCN-backward / accumulate, convert, store; warp w owns TMEM lanes
//                 32*(w%4) .. +31 (one output row per thread) and half the columns
// Two TMEM accumulators (2 x BN fp32 columns) let the epilogue of tile i
// overlap the MMAs of tile i+1.
//
// Precision: bf16/f16 operands use kind::f16 (fp32 accumulate).  fp32
// operands use kind::tf32 with the 3xTF32 split (a = a_hi + a_lo, products
// hi*hi + hi*lo + lo*hi accumulate in TMEM), which restores ~fp32 accuracy
// (rtol 1e-5 parity bar of the north star).
// The kernel and its launch / dispatch templates live in gemm_sm100.cuh; this
// file holds the C ABI and routes to the per-majorness instantiation units.
#include "gemm_sm100.cuh"

namespace dmt {
namespace gemm {

static int dispatch_major(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s) {
  const bool amn = (a->flags & DMT_GEMM_TRANS_A) != 0, bmn = (a->flags & DMT_GEMM_TRANS_B) != 0;
  if (!amn && !bmn) return gemm_major_kk(a, alo, blo, s);
  if (amn && bmn) return gemm_major_mm(a, alo, blo, s);
  if (bmn) return gemm_major_km(a, alo, blo, s);
  return gemm_major_mk(a, alo, blo, s);
}


__global__ void split_tf32_kernel(const float* __restrict__ x, float* __restrict__ hi, float* __restrict__ lo,
                                  int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    // round-to-nearest split: hi = tf32(v), lo = tf32(v - hi) (exact residual,
    // then rounded, so the MMA's tf32 read of lo drops nothing)
    const float v = x[i];
    uint32_t h, l;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
    const float r = v - __uint_as_float(h);
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(r));
    hi[i] = __uint_as_float(h);
    lo[i] = __uint_as_float(l);
  }
}

// out[c] = sum_r part[r, c] (fp64), the last step of the bias gradients the
// DCN backward epilogues fold per (tile, quarter).  Block = 32 columns x 8 row
// groups; group g sums rows g, g+8, ... in order, then the 8 group sums are
// added in group order: a fixed reduction tree, so the result is
// deterministic, with 8 x 32 independent load streams per block.
__global__ void colsum_parts_kernel(const float* __restrict__ part, int64_t rows, int64_t cols,
                                    float* __restrict__ out) {
  __shared__ double red[8][33];
  const int cx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + cx;
  double acc = 0.0;
  if (c < cols) {
#pragma unroll 4
    for (int64_t r = g; r < rows; r += 8) acc += (double)__ldg(part + r * cols + c);
  }
  red[g][cx] = acc;
  __syncthreads();
  if (g == 0 && c < cols) {
    double t = red[0][cx];
#pragma unroll
    for (int i = 1; i < 8; ++i) t += red[i][cx];
    out[c] = (float)t;
  }
}

}  // namespace gemm
}  // namespace dmt

namespace dmt {
namespace gemm {
// d = epi(sum_s ws[s]) over the split-K partials, s ascending (the first copied)
template <typename TO>
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int S, int64_t m, int64_t n, TO* __restrict__ d,
                                     int64_t ld_d, const TO* __restrict__ c, float alpha, float beta, int scale_acc,
                                     int acc) {
  const int64_t total = m * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, col = i - r * n;
    float v = ws[i];
    for (int s = 1; s < S; ++s) v += ws[(int64_t)s * total + i];
    if (scale_acc) v *= alpha;
    if (acc && beta != 0.f) v += beta * to_f<TO>(c[r * ld_d + col]);
    d[r * ld_d + col] = from_f<TO>(v);
  }
}
}  // namespace gemm
}  // namespace dmt

static int gemm_splitk(const dmt_gemm_args* a, const void* a_lo, const void* b_lo, cudaStream_t s) {
  using namespace dmt;
  const size_t es = dtype_size(a->in_dtype);
  const int64_t num_kb = ceil_div(a->k * (int64_t)es, 128);
  const int64_t kbs = ceil_div(num_kb, (int64_t)a->ksplit);
  dmt_gemm_args w = *a;  // the partial products: plain fp32 GEMMs into the workspace
  w.d = a->splitk_ws;
  w.c = nullptr;
  w.ld_d = a->n;
  w.out_dtype = DMT_F32;
  w.epilogue = DMT_EPI_NONE;
  w.flags = a->flags & (DMT_GEMM_TRANS_A | DMT_GEMM_TRANS_B | DMT_GEMM_BN_MASK | DMT_GEMM_NO_PREFETCH);
  w.flags |= DMT_GEMM_SINGLE_CTA;
  w.beta = 0.f;
  w.ksplit = (int32_t)ceil_div(num_kb, kbs);
  int rc = gemm::dispatch_major(&w, a_lo, b_lo, s);
  if (rc != DMT_OK) return rc;
  const int64_t total = a->m * a->n;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), DMT_NUM_SMS * 8));
  const int scale = (a->flags & DMT_GEMM_SCALE_ACC) != 0, acc = a->epilogue == DMT_EPI_ACC;
  const void* c = a->c ? a->c : a->d;
  switch (a->out_dtype) {
    case DMT_F32:
      gemm::splitk_reduce_kernel<float><<<grid, 256, 0, s>>>(a->splitk_ws, w.ksplit, a->m, a->n, (float*)a->d, a->ld_d,
                                                            (const float*)c, a->alpha, a->beta, scale, acc);
      break;
    case DMT_BF16:
      gemm::splitk_reduce_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
          a->splitk_ws, w.ksplit, a->m, a->n, (__nv_bfloat16*)a->d, a->ld_d, (const __nv_bfloat16*)c, a->alpha,
          a->beta, scale, acc);
      break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

extern "C" {

int64_t dmt_gemm_colsum_rows(int64_t m) { return 4 * dmt::ceil_div(m, (int64_t)dmt::gemm::kBlockM); }

int dmt_column_sum_parts(const float* part, int64_t rows, int64_t cols, float* out, dmt_stream_t stream) {
  if (rows < 0 || cols < 0) return DMT_ERR_SHAPE;
  if (cols == 0) return DMT_OK;
  dmt::gemm::colsum_parts_kernel<<<(unsigned)dmt::ceil_div(cols, (int64_t)32), 256, 0, (cudaStream_t)stream>>>(
      part, rows, cols, out);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_gemm_ex(const dmt_gemm_args* args, const void* a_lo, const void* b_lo, dmt_stream_t stream) {
  using namespace dmt;
  if (!args) return DMT_ERR_DOMAIN;
  const dmt_gemm_args* a = args;
  if (a->m < 0 || a->n < 0 || a->k < 0) return DMT_ERR_SHAPE;
  if (a->m == 0 || a->n == 0) return DMT_OK;
  if (a->k == 0) return DMT_ERR_SHAPE;  // caller handles the bias-only case
  if (a->m > INT32_MAX || a->n > INT32_MAX || a->k > INT32_MAX) return DMT_ERR_UNSUPPORTED;
  size_t es = dtype_size(a->in_dtype);
  if (es == 0 || a->in_dtype == DMT_F64) return DMT_ERR_UNSUPPORTED;
  // TMA: 16-byte aligned base and row strides
  if (((uintptr_t)a->a & 15) || ((uintptr_t)a->b & 15) || (a->lda * es) % 16 || (a->ldb * es) % 16)
    return DMT_ERR_UNSUPPORTED;
  if ((a->epilogue == DMT_EPI_BIAS || a->epilogue == DMT_EPI_CROSS || a->epilogue == DMT_EPI_BIAS_RELU) && !a->bias)
    return DMT_ERR_DOMAIN;
  if (a->epilogue == DMT_EPI_RELU_BWD && !a->x0) return DMT_ERR_DOMAIN;
  if (a->epilogue == DMT_EPI_CROSS && (!a->x0 || !a->xl)) return DMT_ERR_DOMAIN;
  if (a->epilogue == DMT_EPI_DCN_BWD && (!a->x0 || !a->aux || (a->aux2 && !a->xl))) return DMT_ERR_DOMAIN;
  if (a->npairs < 0 || a->npairs > DMT_GEMM_MAX_PAIRS) return DMT_ERR_DOMAIN;
  if (a->npairs && a->epilogue != DMT_EPI_DCN_FINAL) return DMT_ERR_DOMAIN;
  for (int j = 0; j < a->npairs; ++j)
    if (!a->pair_g[j] || !a->pair_u[j]) return DMT_ERR_DOMAIN;
  if (a->npairs && a->ld_x <= 0) return DMT_ERR_UNSUPPORTED;
  if (a->epilogue == DMT_EPI_DCN_FINAL && !a->aux2 && !a->npairs) return DMT_ERR_DOMAIN;
  if ((a->epilogue == DMT_EPI_DCN_BWD || a->epilogue == DMT_EPI_DCN_FINAL) && a->out_dtype != a->in_dtype)
    return DMT_ERR_UNSUPPORTED;
  if (a->epilogue > DMT_EPI_RELU_BWD || a->epilogue < 0) return DMT_ERR_DOMAIN;
  if (a->n_out_groups < 0 || a->n_out_groups > DMT_GEMM_MAX_OUT_GROUPS) return DMT_ERR_DOMAIN;
  if (a->n_col_groups < 0 || a->n_col_groups > DMT_GEMM_MAX_COL_GROUPS) return DMT_ERR_DOMAIN;
  if (a->n_col_groups) {
    if (a->n_out_groups || a->ksplit > 1 || a->col_group_width <= 0 || a->col_group_width % 32 ||
        (int64_t)a->n_col_groups * a->col_group_width != a->n || a->rows_per_group > 0)
      return DMT_ERR_DOMAIN;
    for (int j = 0; j < a->n_col_groups; ++j)
      if (!a->col_group[j] || a->col_group_ld[j] < a->col_group_width) return DMT_ERR_DOMAIN;
  }
  if (a->n_out_groups) {
    if (a->rows_per_group <= 0 || (a->m + a->rows_per_group - 1) / a->rows_per_group > a->n_out_groups ||
        a->ksplit > 1 || a->colsum_part)
      return DMT_ERR_DOMAIN;
    for (int j = 0; j < a->n_out_groups; ++j)
      if (!a->out_group[j]) return DMT_ERR_DOMAIN;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (a->ksplit > 1) {
    if (!a->splitk_ws || (a->epilogue != DMT_EPI_NONE && a->epilogue != DMT_EPI_ACC) ||
        a->rows_per_group > 0 || a->colsum_part)
      return DMT_ERR_DOMAIN;
    if (a->in_dtype == DMT_F32 && (!a_lo || !b_lo)) return DMT_ERR_DOMAIN;
    return gemm_splitk(a, a_lo, b_lo, s);
  }
  switch (a->in_dtype) {
    case DMT_BF16: return gemm::dispatch_major(a, nullptr, nullptr, s);
    case DMT_F16: return gemm::dispatch_major(a, nullptr, nullptr, s);
    case DMT_F32:
      if (!a_lo || !b_lo) return DMT_ERR_DOMAIN;
      if (((uintptr_t)a_lo & 15) || ((uintptr_t)b_lo & 15)) return DMT_ERR_UNSUPPORTED;
      return gemm::dispatch_major(a, a_lo, b_lo, s);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

int dmt_gemm(const dmt_gemm_args* args, dmt_stream_t stream) { return dmt_gemm_ex(args, nullptr, nullptr, stream); }

int dmt_split_tf32(const float* x, float* hi, float* lo, int64_t n, dmt_stream_t stream) {
  if (n == 0) return DMT_OK;
  unsigned grid = (unsigned)std::min<int64_t>(dmt::ceil_div(n, 256), DMT_NUM_SMS * 16);
  dmt::gemm::split_tf32_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(x, hi, lo, n);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

}  // extern "C"
