// DLRM pairwise dot-product feature interaction (the C3 model's interaction
// arch around SPTT; TorchRec InteractionArch semantics):
//
//   V = [dense (B, D) | sparse (B, F*D) viewed as (B, F, D)]   -> (B, F+1, D)
//   out[:, :D]         = dense
//   out[:, D + p(i,j)] = <V_i, V_j>,  i > j, p = i(i-1)/2 + j  (row-major strict
//                                      lower triangle, torch.tril_indices(-1))
//
// Memory-bound (a sample's F+1 vectors are read once, (F+1)F/2 dots are
// written), so it runs on the CUDA cores: one warp per sample, the vectors
// staged in shared memory as fp32 with a padded row stride (bank-conflict-free
// column reads), fp32 accumulation in k order.  The backward forms
//   dV_i = [i == 0] dout[:, :D] + sum_{j != i} g(max(i,j), min(i,j)) V_j
// in the same layout (j ascending, fp32).
#include "common.cuh"

namespace dmt {

constexpr int kIaWarps = 8;

__device__ __forceinline__ void pair_of(int p, int& i, int& j) {
  // i = largest with i(i-1)/2 <= p
  int ii = (int)((1.0f + sqrtf(1.0f + 8.0f * (float)p)) * 0.5f);
  while (ii * (ii - 1) / 2 > p) --ii;
  while ((ii + 1) * ii / 2 <= p) ++ii;
  i = ii;
  j = p - ii * (ii - 1) / 2;
}

template <typename T>
__device__ __forceinline__ void stage_sample(float* v, const T* dense, const T* sparse, int nf, int D, int lane) {
  const int ld = D + 1;
  for (int k = lane; k < D; k += 32) v[k] = to_f<T>(dense[k]);
  for (int f = 0; f < nf; ++f)
    for (int k = lane; k < D; k += 32) v[(f + 1) * ld + k] = to_f<T>(sparse[(int64_t)f * D + k]);
}

template <typename T>
__global__ void __launch_bounds__(kIaWarps * 32)
interact_fwd_kernel(const T* __restrict__ dense, int64_t ld_dense, const T* __restrict__ sparse, int64_t ld_sparse,
                    int nf, int D, int64_t B, T* __restrict__ out, int64_t ld_out) {
  extern __shared__ float ia_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = nf + 1, ld = D + 1;
  float* v = ia_smem + (size_t)warp * nv * ld;
  const int P = nv * nf / 2;
  for (int64_t b = (int64_t)blockIdx.x * kIaWarps + warp; b < B; b += (int64_t)gridDim.x * kIaWarps) {
    const T* dr = dense + b * ld_dense;
    T* o = out + b * ld_out;
    stage_sample<T>(v, dr, sparse + b * ld_sparse, nf, D, lane);
    __syncwarp();
    for (int k = lane; k < D; k += 32) o[k] = dr[k];
    for (int p = lane; p < P; p += 32) {
      int i, j;
      pair_of(p, i, j);
      const float* vi = v + i * ld;
      const float* vj = v + j * ld;
      float acc = 0.f;
      for (int k = 0; k < D; ++k) acc = fmaf(vi[k], vj[k], acc);
      o[D + p] = from_f<T>(acc);
    }
    __syncwarp();
  }
}

template <typename T>
__global__ void __launch_bounds__(kIaWarps * 32)
interact_bwd_kernel(const T* __restrict__ gout, int64_t ld_gout, const T* __restrict__ dense, int64_t ld_dense,
                    const T* __restrict__ sparse, int64_t ld_sparse, int nf, int D, int64_t B,
                    T* __restrict__ d_dense, int64_t ld_dd, T* __restrict__ d_sparse, int64_t ld_ds) {
  extern __shared__ float ia_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = nf + 1, ld = D + 1;
  const int P = nv * nf / 2;
  float* v = ia_smem + (size_t)warp * (nv * ld + P);
  float* g = v + nv * ld;
  for (int64_t b = (int64_t)blockIdx.x * kIaWarps + warp; b < B; b += (int64_t)gridDim.x * kIaWarps) {
    const T* go = gout + b * ld_gout;
    stage_sample<T>(v, dense + b * ld_dense, sparse + b * ld_sparse, nf, D, lane);
    for (int p = lane; p < P; p += 32) g[p] = to_f<T>(go[D + p]);
    __syncwarp();
    for (int i = 0; i < nv; ++i) {
      T* dst = i == 0 ? d_dense + b * ld_dd : d_sparse + b * ld_ds + (int64_t)(i - 1) * D;
      for (int k = lane; k < D; k += 32) {
        float acc = i == 0 ? to_f<T>(go[k]) : 0.f;
        for (int j = 0; j < nv; ++j) {
          if (j == i) continue;
          const int p = i > j ? i * (i - 1) / 2 + j : j * (j - 1) / 2 + i;
          acc = fmaf(g[p], v[j * ld + k], acc);
        }
        dst[k] = from_f<T>(acc);
      }
    }
    __syncwarp();
  }
}

template <typename T>
int launch_interact(bool bwd, const void* gout, int64_t ld_gout, const void* dense, int64_t ld_dense,
                    const void* sparse, int64_t ld_sparse, int nf, int D, int64_t B, void* out, int64_t ld_out,
                    void* d_sparse, int64_t ld_ds, cudaStream_t s) {
  const int nv = nf + 1;
  const size_t per_warp = ((size_t)nv * (D + 1) + (bwd ? (size_t)nv * nf / 2 : 0)) * sizeof(float);
  const size_t smem = per_warp * kIaWarps;
  if (smem > 200 * 1024) return DMT_ERR_UNSUPPORTED;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(B, kIaWarps), DMT_NUM_SMS * 16));
  if (!bwd) {
    auto k = interact_fwd_kernel<T>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return DMT_ERR_CUDA;
    k<<<grid, kIaWarps * 32, smem, s>>>((const T*)dense, ld_dense, (const T*)sparse, ld_sparse, nf, D, B, (T*)out,
                                        ld_out);
  } else {
    auto k = interact_bwd_kernel<T>;
    if (smem > 48 * 1024 && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return DMT_ERR_CUDA;
    k<<<grid, kIaWarps * 32, smem, s>>>((const T*)gout, ld_gout, (const T*)dense, ld_dense, (const T*)sparse,
                                        ld_sparse, nf, D, B, (T*)out, ld_out, (T*)d_sparse, ld_ds);
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

template <typename T>
__global__ void relu_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ y, T* __restrict__ dz, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dz[i] = to_f<T>(y[i]) > 0.f ? dy[i] : from_f<T>(0.f);
}

}  // namespace dmt

extern "C" {

int dmt_relu_bwd(const void* dy, const void* y, void* dz, int64_t n, int32_t dtype, dmt_stream_t stream) {
  if (n < 0) return DMT_ERR_SHAPE;
  if (n == 0) return DMT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(dmt::ceil_div(n, 256), DMT_NUM_SMS * 8));
  switch (dtype) {
    case DMT_F32: dmt::relu_bwd_kernel<float><<<grid, 256, 0, s>>>((const float*)dy, (const float*)y, (float*)dz, n); break;
    case DMT_BF16:
      dmt::relu_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)y,
                                                              (__nv_bfloat16*)dz, n);
      break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_dot_interaction_fwd(const void* dense, int64_t ld_dense, const void* sparse, int64_t ld_sparse,
                            int32_t num_sparse, int32_t dim, int64_t batch, void* out, int64_t ld_out, int32_t dtype,
                            dmt_stream_t stream) {
  if (num_sparse < 0 || dim <= 0 || batch < 0) return DMT_ERR_SHAPE;
  if (batch == 0) return DMT_OK;
  if (!dense || !out || (num_sparse > 0 && !sparse)) return DMT_ERR_DOMAIN;
  const int64_t width = dim + (int64_t)(num_sparse + 1) * num_sparse / 2;
  if (ld_out < width || ld_dense < dim || (num_sparse && ld_sparse < (int64_t)num_sparse * dim)) return DMT_ERR_SHAPE;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32:
      return dmt::launch_interact<float>(false, nullptr, 0, dense, ld_dense, sparse, ld_sparse, num_sparse, dim, batch,
                                         out, ld_out, nullptr, 0, s);
    case DMT_BF16:
      return dmt::launch_interact<__nv_bfloat16>(false, nullptr, 0, dense, ld_dense, sparse, ld_sparse, num_sparse,
                                                 dim, batch, out, ld_out, nullptr, 0, s);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

int dmt_dot_interaction_bwd(const void* grad_out, int64_t ld_grad_out, const void* dense, int64_t ld_dense,
                            const void* sparse, int64_t ld_sparse, int32_t num_sparse, int32_t dim, int64_t batch,
                            void* d_dense, int64_t ld_d_dense, void* d_sparse, int64_t ld_d_sparse, int32_t dtype,
                            dmt_stream_t stream) {
  if (num_sparse < 0 || dim <= 0 || batch < 0) return DMT_ERR_SHAPE;
  if (batch == 0) return DMT_OK;
  if (!grad_out || !dense || !d_dense || (num_sparse > 0 && (!sparse || !d_sparse))) return DMT_ERR_DOMAIN;
  const int64_t width = dim + (int64_t)(num_sparse + 1) * num_sparse / 2;
  if (ld_grad_out < width) return DMT_ERR_SHAPE;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32:
      return dmt::launch_interact<float>(true, grad_out, ld_grad_out, dense, ld_dense, sparse, ld_sparse, num_sparse,
                                         dim, batch, d_dense, ld_d_dense, d_sparse, ld_d_sparse, s);
    case DMT_BF16:
      return dmt::launch_interact<__nv_bfloat16>(true, grad_out, ld_grad_out, dense, ld_dense, sparse, ld_sparse,
                                                 num_sparse, dim, batch, d_dense, ld_d_dense, d_sparse, ld_d_sparse,
                                                 s);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

}  // extern "C"
