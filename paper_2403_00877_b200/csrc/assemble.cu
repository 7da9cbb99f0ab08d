// Data movement kernels of the exchange plus small
// dense helpers used by the tower-module backward.
//
// dmt_assemble is the single gather kernel behind
//   * _combine_pieces  (towersim/exchange.py:112-127): column shards land side
//     by side, row-wise partials are summed in row-range order (fp64, once
//     rounded -- matches the reference's float64 `total += mat`);
//   * step-e regroup   (exchange.py:417-437): (feature, dest) -> (dest, feature);
//   * step-f concat    (exchange.py:448-449) and realign (exchange.py:465-486).
// Blocks are described by (dst column, width, source list); one CTA row-tile
// covers all blocks of a few rows so the destination row is written
// contiguously.
#include "common.cuh"

namespace dmt {

constexpr int kAsmThreads = 256;

template <typename T, int VEC>
__global__ void __launch_bounds__(kAsmThreads)
assemble_kernel(const dmt_assemble_block* __restrict__ blocks, const dmt_src* __restrict__ srcs, int64_t rows,
                T* __restrict__ dst, int64_t dst_ld) {
  const dmt_assemble_block blk = blocks[blockIdx.y];
  const int nvec = blk.width / VEC;
  // grid.x covers rows x vectors of this block
  const int64_t total = rows * (int64_t)nvec;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / nvec;
    const int c = (int)(i - r * nvec) * VEC;
    T* o = dst + r * dst_ld + blk.dst_col + c;
    if (blk.nsrc == 1) {
      const dmt_src s0 = srcs[blk.first_src];
      const T* p = reinterpret_cast<const T*>(s0.ptr) + r * s0.ld + c;
      if constexpr (VEC == 1) {
        *o = *p;
      } else {
        using V = typename std::conditional<sizeof(T) * VEC == 16, uint4,
                  typename std::conditional<sizeof(T) * VEC == 8, uint2, uint32_t>::type>::type;
        *reinterpret_cast<V*>(o) = *reinterpret_cast<const V*>(p);
      }
    } else {
      // fp64 sums; the first term of each (inner / outer) sum is copied, not
      // added to 0 (numpy's `total = first.copy(); total += ...`), so the
      // bits -- a -0.0 partial included -- match the reference
      double acc[VEC], grp[VEC];
      bool have_acc = false;
      for (int s = 0; s < blk.nsrc; ++s) {
        const dmt_src sx = srcs[blk.first_src + s];
        const T* p = reinterpret_cast<const T*>(sx.ptr) + r * sx.ld + c;
        const bool new_group = s > 0 && ((blk.groups >> s) & 1u);
        if (new_group) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[e] = have_acc ? acc[e] + grp[e] : grp[e];
          have_acc = true;
        }
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const double v = to_d<T>(p[e]);
          grp[e] = (s == 0 || new_group) ? v : grp[e] + v;
        }
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) o[e] = from_d<T>(have_acc ? acc[e] + grp[e] : grp[e]);
    }
  }
}

template <typename T>
int launch_assemble(const dmt_assemble_block* blocks, int32_t nb, int32_t max_width, const dmt_src* srcs,
                    int64_t rows, void* dst, int64_t dst_ld, cudaStream_t s, bool vec_ok) {
  if (rows == 0 || nb == 0 || max_width == 0) return DMT_OK;
  if (nb > 65535) return DMT_ERR_UNSUPPORTED;
  constexpr int VEC = 16 / sizeof(T);
  int64_t work = rows * (int64_t)max_width;
  if (vec_ok) work /= VEC;
  unsigned gx = (unsigned)std::min<int64_t>(ceil_div(work, kAsmThreads), 4096);
  dim3 grid(gx, nb);
  if (vec_ok)
    assemble_kernel<T, VEC><<<grid, kAsmThreads, 0, s>>>(blocks, srcs, rows, (T*)dst, dst_ld);
  else
    assemble_kernel<T, 1><<<grid, kAsmThreads, 0, s>>>(blocks, srcs, rows, (T*)dst, dst_ld);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

// ---------------------------------------------------------------- copies ----
__global__ void batched_copy_kernel(const dmt_copy* __restrict__ copies) {
  const dmt_copy c = copies[blockIdx.y];
  const int64_t n16 = ((((uintptr_t)c.src | (uintptr_t)c.dst) & 15) == 0) ? c.bytes / 16 : 0;
  const uint4* s4 = reinterpret_cast<const uint4*>(c.src);
  uint4* d4 = reinterpret_cast<uint4*>(c.dst);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) d4[i] = s4[i];
  const char* s1 = reinterpret_cast<const char*>(c.src);
  char* d1 = reinterpret_cast<char*>(c.dst);
  for (int64_t i = n16 * 16 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < c.bytes; i += stride)
    d1[i] = s1[i];
}

// E = element type; when VB > 1 every copy is moved in 16-byte vectors (the
// host checks that widths, strides and pointers are 16-byte granular).
template <typename E, int VB>
__global__ void batched_copy2d_kernel(const dmt_copy2d* __restrict__ copies) {
  const dmt_copy2d c = copies[blockIdx.y];
  if constexpr (VB == 1) {
    const int64_t total = c.rows * c.width;
    const E* s = reinterpret_cast<const E*>(c.src);
    E* d = reinterpret_cast<E*>(c.dst);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      int64_t r = i / c.width, j = i - r * c.width;
      d[r * c.dst_ld + j] = s[r * c.src_ld + j];
    }
  } else {
    constexpr int EV = 16 / sizeof(E);  // elements per vector
    const int64_t wv = c.width / EV, sld = c.src_ld / EV, dld = c.dst_ld / EV;
    const int64_t total = c.rows * wv;
    const uint4* s = reinterpret_cast<const uint4*>(c.src);
    uint4* d = reinterpret_cast<uint4*>(c.dst);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
      int64_t r = i / wv, j = i - r * wv;
      d[r * dld + j] = s[r * sld + j];
    }
  }
}

// ------------------------------------------------------------ transpose ----
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                                 T* __restrict__ out, int64_t ld_out) {
  __shared__ T tile[32][33];
  int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * ld_in + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * ld_out + r] = tile[threadIdx.x][i];
  }
}

// --------------------------------------------------------- column sum ----
// one thread per column, rows split over grid.y; partials combined in a fixed
// order by a second pass (deterministic).
template <typename T>
__global__ void colsum_partial(const T* __restrict__ in, int64_t rows, int64_t cols, int64_t ld,
                               int64_t rows_per, double* __restrict__ part) {
  int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
  double acc = 0.0;
  for (int64_t r = r0; r < r1; ++r) acc += to_d<T>(in[r * ld + c]);
  part[(int64_t)blockIdx.y * cols + c] = acc;
}

// 16-byte vector loads: a warp reads 512 contiguous bytes of a row per step.
template <typename T>
__global__ void colsum_partial_vec(const T* __restrict__ in, int64_t rows, int64_t cols, int64_t ld,
                                   int64_t rows_per, double* __restrict__ part) {
  constexpr int V = 16 / sizeof(T);
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V;
  if (c >= cols) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(rows, r0 + rows_per);
  float acc[V];
#pragma unroll
  for (int e = 0; e < V; ++e) acc[e] = 0.f;
  double dacc[V];
#pragma unroll
  for (int e = 0; e < V; ++e) dacc[e] = 0.0;
  int cnt = 0;
  auto add = [&](const uint4& x) {
    const T* h = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int e = 0; e < V; ++e) acc[e] += to_f<T>(h[e]);
    if (++cnt == 32) {  // fold fp32 partial sums into fp64 every 32 rows
#pragma unroll
      for (int e = 0; e < V; ++e) { dacc[e] += acc[e]; acc[e] = 0.f; }
      cnt = 0;
    }
  };
  // 16 row loads in flight per thread (the loop was latency bound at one),
  // folded in row order: same arithmetic as the one-row loop
  constexpr int kBatch = 16;
  int64_t r = r0;
  for (; r + kBatch <= r1; r += kBatch) {
    uint4 x[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) x[u] = __ldg(reinterpret_cast<const uint4*>(in + (r + u) * ld + c));
#pragma unroll
    for (int u = 0; u < kBatch; ++u) add(x[u]);
  }
  for (; r < r1; ++r) add(__ldg(reinterpret_cast<const uint4*>(in + r * ld + c)));
#pragma unroll
  for (int e = 0; e < V; ++e) part[(int64_t)blockIdx.y * cols + c + e] = dacc[e] + acc[e];
}

// 32 columns x 8 partial-slices per block; fixed-order tree over the 8 slices
// (deterministic) after each thread folds nparts/8 partials.
__global__ void colsum_final(const double* __restrict__ part, int64_t cols, int nparts, float* __restrict__ out) {
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + tx;
  double acc = 0.0;
  if (c < cols) {
    int p = ty;
    for (; p + 24 < nparts; p += 32) {  // 4 independent loads in flight, summed in slice order
      const double a0 = part[(int64_t)p * cols + c], a1 = part[(int64_t)(p + 8) * cols + c];
      const double a2 = part[(int64_t)(p + 16) * cols + c], a3 = part[(int64_t)(p + 24) * cols + c];
      acc += a0; acc += a1; acc += a2; acc += a3;
    }
    for (; p < nparts; p += 8) acc += part[(int64_t)p * cols + c];
  }
  red[ty][tx] = acc;
  __syncthreads();
  if (ty == 0 && c < cols) {
    double t = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += red[i][tx];
    out[c] = (float)t;
  }
}

template <typename T>
__global__ void cross_bwd_pointwise_kernel(const T* __restrict__ g, const T* __restrict__ x0,
                                           const T* __restrict__ u, T* __restrict__ gu, float* __restrict__ dx0,
                                           int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float gv = to_f<T>(g[i]);
    gu[i] = from_f<T>(gv * to_f<T>(x0[i]));
    dx0[i] += gv * to_f<T>(u[i]);
  }
}
template <>
__global__ void cross_bwd_pointwise_kernel<double>(const double* __restrict__ g, const double* __restrict__ x0,
                                                   const double* __restrict__ u, double* __restrict__ gu,
                                                   float* __restrict__ dx0, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    gu[i] = g[i] * x0[i];
    dx0[i] += (float)(g[i] * u[i]);
  }
}

// dx0 (+)= g * u: one term of the crossnet's dx0 = sum_l g_{l+1} * u_l, on a
// side stream beside the (compute-bound) dW GEMMs instead of in the dX GEMM
// epilogues.  V elements (16 bytes of g / u) per thread and step.
template <typename T, int V>
__global__ void dcn_dx0_term_kernel(const T* __restrict__ g, const T* __restrict__ u, float* __restrict__ dx0,
                                    int64_t n, int accumulate) {
  const int64_t nv = n / V;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    float gv[V], uv[V], d[V];
    if constexpr (V == 8) {  // 16-bit types: one 16-byte load per operand
      const uint4 gr = __ldg(reinterpret_cast<const uint4*>(g + i * 8));
      const uint4 ur = __ldg(reinterpret_cast<const uint4*>(u + i * 8));
      const T* gh = reinterpret_cast<const T*>(&gr);
      const T* uh = reinterpret_cast<const T*>(&ur);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        gv[e] = to_f<T>(gh[e]);
        uv[e] = to_f<T>(uh[e]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        gv[e] = (float)to_d<T>(g[i * V + e]);
        uv[e] = (float)to_d<T>(u[i * V + e]);
      }
    }
    if (accumulate) {
#pragma unroll
      for (int e = 0; e < V; e += 4) {
        const float4 x = *reinterpret_cast<const float4*>(dx0 + i * V + e);
        d[e] = x.x; d[e + 1] = x.y; d[e + 2] = x.z; d[e + 3] = x.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) d[e] = 0.f;
    }
#pragma unroll
    for (int e = 0; e < V; ++e) d[e] += gv[e] * uv[e];
#pragma unroll
    for (int e = 0; e < V; e += 4)
      *reinterpret_cast<float4*>(dx0 + i * V + e) = make_float4(d[e], d[e + 1], d[e + 2], d[e + 3]);
  }
  // tail (n % V elements) by the first threads
  const int64_t t0 = nv * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t0 < n) {
    const float t = (float)to_d<T>(g[t0]) * (float)to_d<T>(u[t0]);
    dx0[t0] = accumulate ? dx0[t0] + t : t;
  }
}

// Element-wise tail of the crossnet backward in one streaming pass:
//   dx0 = sum_{l = L-1..0} g_l * u_l   (fp32, the dx0-term order: bit-identical)
// reading each g_l / u_l once and writing dx0 once (2 L x 54.5 MB + 109 MB at
// C2) instead of L read-modify-write passes over the fp32 dx0.  A single pass
// that also column-summed gu_l (thread = 8 columns x a 64-row slice, the
// column-sum partial layout) measured latency bound at 3.3 TB/s (181 us);
// this flat grid-stride form streams like dmt_dcn_dx0_term.
struct SidePtrs {
  const void* g[4];
  const void* u[4];
};

template <typename T, int NL>
__global__ void __launch_bounds__(256) dcn_dx0_sum_kernel(const SidePtrs P, int64_t n, float* __restrict__ dx0) {
  const int64_t nv = n / 8;
  const T* g[NL];
  const T* u[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    g[l] = reinterpret_cast<const T*>(P.g[l]);
    u[l] = reinterpret_cast<const T*>(P.u[l]);
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 gr[NL], ur[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      gr[l] = __ldg(reinterpret_cast<const uint4*>(g[l] + i * 8));
      ur[l] = __ldg(reinterpret_cast<const uint4*>(u[l] + i * 8));
    }
    float d[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) d[e] = 0.f;
#pragma unroll
    for (int l = NL - 1; l >= 0; --l) {
      const T* gh = reinterpret_cast<const T*>(&gr[l]);
      const T* uh = reinterpret_cast<const T*>(&ur[l]);
#pragma unroll
      for (int e = 0; e < 8; ++e) d[e] += to_f<T>(gh[e]) * to_f<T>(uh[e]);
    }
    *reinterpret_cast<float4*>(dx0 + i * 8) = make_float4(d[0], d[1], d[2], d[3]);
    *reinterpret_cast<float4*>(dx0 + i * 8 + 4) = make_float4(d[4], d[5], d[6], d[7]);
  }
}

template <typename T>
__global__ void sgd_dense_kernel(T* __restrict__ w, const float* __restrict__ g, int64_t n, float lr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    w[i] = from_d<T>(to_d<T>(w[i]) - (double)lr * (double)g[i]);
}

// Tower gradient all-reduce + SGD over NVLink peer memory: every member sums
// the members' fp32 gradients in tower-rank order (identical on all members)
// and applies w -= lr * sum to its own replica.  16-byte peer loads.
struct PeerSrcs {
  const float* g[DMT_MAX_PEER_SRCS];
};

// Device barrier over NVLink peer memory (replaces the 1-float NCCL
// all-reduce the peer fabric used as a completion barrier): each member bumps
// its epoch for this group kind, release-stores it into every other member's
// flag slot for it (system scope, over NVLink), then acquire-spins until every
// other member's epoch arrived in its own slots.  The preceding kernels in
// stream order happen-before the release; the acquire orders the following
// kernels' reads of the peers' stores after it.  Epochs live on the device, so
// the same launch replays correctly from a CUDA graph.
struct BarrierSlots {
  int32_t* remote[DMT_MAX_PEER_SRCS];  // member i's flag slot for this rank (peer-mapped)
  int32_t* local[DMT_MAX_PEER_SRCS];   // this rank's flag slot for member i
};

__global__ void peer_barrier_kernel(int32_t* epoch, const __grid_constant__ BarrierSlots s, int n, int32_t* err) {
  __shared__ int32_t e;
  if (threadIdx.x == 0) {
    e = *epoch + 1;
    *epoch = e;
  }
  __syncthreads();
  const int i = threadIdx.x;
  if (i < n) {
    __threadfence_system();
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(s.remote[i]), "r"(e) : "memory");
    int32_t v = 0;
    long long spins = 0;
    do {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(s.local[i]) : "memory");
      if (++spins > (1ll << 26)) {  // a peer never arrived: flag it instead of hanging the GPU
        if (err) atomicOr(err, 1);
        break;
      }
    } while (v < e);
  }
  __syncthreads();
}

template <typename T>
__global__ void peer_sum_sgd_kernel(T* __restrict__ w, const __grid_constant__ PeerSrcs src, int nsrc, int64_t n,
                                    float lr) {
  const int64_t n4 = n >> 2;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 s = reinterpret_cast<const float4*>(src.g[0])[i];
    for (int m = 1; m < nsrc; ++m) {
      const float4 x = reinterpret_cast<const float4*>(src.g[m])[i];
      s.x += x.x; s.y += x.y; s.z += x.z; s.w += x.w;
    }
    const float v[4] = {s.x, s.y, s.z, s.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) w[4 * i + e] = from_d<T>(to_d<T>(w[4 * i + e]) - (double)lr * (double)v[e]);
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float s = src.g[0][i];
    for (int m = 1; m < nsrc; ++m) s += src.g[m][i];
    w[i] = from_d<T>(to_d<T>(w[i]) - (double)lr * (double)s);
  }
}

template <typename A, typename B>
__global__ void convert_kernel(const A* __restrict__ a, B* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = from_d<B>(to_d<A>(a[i]));
}

template <typename A>
int convert_to(const void* src, void* dst, int32_t dto, int64_t n, cudaStream_t s) {
  unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), DMT_NUM_SMS * 16);
  switch (dto) {
    case DMT_F32: convert_kernel<A, float><<<grid, 256, 0, s>>>((const A*)src, (float*)dst, n); break;
    case DMT_BF16: convert_kernel<A, __nv_bfloat16><<<grid, 256, 0, s>>>((const A*)src, (__nv_bfloat16*)dst, n); break;
    case DMT_F64: convert_kernel<A, double><<<grid, 256, 0, s>>>((const A*)src, (double*)dst, n); break;
    case DMT_F16: convert_kernel<A, __half><<<grid, 256, 0, s>>>((const A*)src, (__half*)dst, n); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

// Binary cross-entropy on logits, one block (deterministic loss sum):
//   dz[i] = scale * (sigmoid(z[i]) - y[i]),   loss = scale * sum_i bce(z[i], y[i])
// bce(z, y) = max(z, 0) - z y + log1p(exp(-|z|))  (stable form).
template <typename T>
__global__ void bce_logits_kernel(const T* __restrict__ z, const float* __restrict__ y, int64_t n, float scale,
                                  T* __restrict__ dz, float* __restrict__ loss) {
  __shared__ double part[256];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double zi = to_d<T>(z[i]), yi = y[i];
    const double sg = 1.0 / (1.0 + exp(-zi));
    dz[i] = from_d<T>(scale * (sg - yi));
    acc += fmax(zi, 0.0) - zi * yi + log1p(exp(-fabs(zi)));
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0 && loss) *loss = (float)(scale * part[0]);
}

}  // namespace dmt

extern "C" {

int dmt_assemble(const dmt_assemble_block* blocks, int32_t num_blocks, int32_t max_width, const dmt_src* srcs,
                 int64_t rows, void* dst, int64_t dst_ld, int32_t dtype, dmt_stream_t stream) {
  // The vector path is only taken when the caller guarantees 16-byte
  // alignment of every block (flagged via a negative max_width).
  bool vec_ok = max_width < 0;
  if (vec_ok) max_width = -max_width;
  if (num_blocks < 0 || rows < 0) return DMT_ERR_DOMAIN;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32: return dmt::launch_assemble<float>(blocks, num_blocks, max_width, srcs, rows, dst, dst_ld, s, vec_ok);
    case DMT_BF16:
      return dmt::launch_assemble<__nv_bfloat16>(blocks, num_blocks, max_width, srcs, rows, dst, dst_ld, s, vec_ok);
    case DMT_F64: return dmt::launch_assemble<double>(blocks, num_blocks, max_width, srcs, rows, dst, dst_ld, s, vec_ok);
    case DMT_F16: return dmt::launch_assemble<__half>(blocks, num_blocks, max_width, srcs, rows, dst, dst_ld, s, vec_ok);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

int dmt_batched_copy(const dmt_copy* copies, int32_t n, int64_t max_bytes, dmt_stream_t stream) {
  if (n < 0) return DMT_ERR_DOMAIN;
  if (n == 0 || max_bytes <= 0) return DMT_OK;
  if (n > 65535) return DMT_ERR_UNSUPPORTED;
  unsigned gx = (unsigned)std::min<int64_t>(dmt::ceil_div(max_bytes, 16 * 256), 1024);
  dmt::batched_copy_kernel<<<dim3(gx, n), 256, 0, (cudaStream_t)stream>>>(copies);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_batched_copy2d(const dmt_copy2d* copies, int32_t n, int32_t elem_bytes, int64_t max_elems,
                       dmt_stream_t stream) {
  // a negative elem_bytes promises 16-byte granularity of every copy (vector path)
  const bool vec = elem_bytes < 0;
  if (vec) elem_bytes = -elem_bytes;
  if (n < 0) return DMT_ERR_DOMAIN;
  if (n == 0 || max_elems <= 0) return DMT_OK;
  if (n > 65535) return DMT_ERR_UNSUPPORTED;
  const int64_t work = vec ? max_elems * elem_bytes / 16 : max_elems;
  unsigned gx = (unsigned)std::min<int64_t>(dmt::ceil_div(work, 256), 2048);
  dim3 grid(gx, n);
  cudaStream_t s = (cudaStream_t)stream;
  switch (elem_bytes * (vec ? -1 : 1)) {
    case 2: dmt::batched_copy2d_kernel<uint16_t, 1><<<grid, 256, 0, s>>>(copies); break;
    case 4: dmt::batched_copy2d_kernel<uint32_t, 1><<<grid, 256, 0, s>>>(copies); break;
    case 8: dmt::batched_copy2d_kernel<uint64_t, 1><<<grid, 256, 0, s>>>(copies); break;
    case -2: dmt::batched_copy2d_kernel<uint16_t, 16><<<grid, 256, 0, s>>>(copies); break;
    case -4: dmt::batched_copy2d_kernel<uint32_t, 16><<<grid, 256, 0, s>>>(copies); break;
    case -8: dmt::batched_copy2d_kernel<uint64_t, 16><<<grid, 256, 0, s>>>(copies); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_transpose(const void* in, int64_t rows, int64_t cols, int64_t ld_in, void* out, int64_t ld_out,
                  int32_t dtype, dmt_stream_t stream) {
  if (rows == 0 || cols == 0) return DMT_OK;
  dim3 grid((unsigned)dmt::ceil_div(cols, 32), (unsigned)dmt::ceil_div(rows, 32));
  dim3 block(32, 8);
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32: dmt::transpose_kernel<float><<<grid, block, 0, s>>>((const float*)in, rows, cols, ld_in, (float*)out, ld_out); break;
    case DMT_BF16:
    case DMT_F16:
      dmt::transpose_kernel<uint16_t><<<grid, block, 0, s>>>((const uint16_t*)in, rows, cols, ld_in, (uint16_t*)out, ld_out);
      break;
    case DMT_F64: dmt::transpose_kernel<double><<<grid, block, 0, s>>>((const double*)in, rows, cols, ld_in, (double*)out, ld_out); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

static inline int colsum_parts(int64_t rows) {
  return (int)std::min<int64_t>(std::max<int64_t>(1, rows / 64), 256);
}

size_t dmt_column_sum_workspace_size(int64_t rows, int64_t cols) {
  return sizeof(double) * (size_t)colsum_parts(rows) * (size_t)(cols > 0 ? cols : 1);
}

int dmt_column_sum(const void* in, int64_t rows, int64_t cols, int64_t ld, float* out, int32_t dtype,
                   void* workspace, size_t workspace_bytes, dmt_stream_t stream) {
  if (cols == 0) return DMT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int nparts = colsum_parts(rows);
  int64_t rows_per = dmt::ceil_div(std::max<int64_t>(rows, 1), nparts);
  if (workspace_bytes < dmt_column_sum_workspace_size(rows, cols)) return DMT_ERR_DOMAIN;
  double* g_colsum_scratch = (double*)workspace;
  const size_t es = dmt::dtype_size(dtype);
  const bool vec = es && es <= 4 && dtype != DMT_F64 && ((uintptr_t)in % 16 == 0) && ((ld * es) % 16 == 0) &&
                   ((cols * es) % 16 == 0);
  if (vec) {
    const int V = 16 / (int)es;
    dim3 vg((unsigned)dmt::ceil_div(cols / V, 128), nparts);
    if (dtype == DMT_F32)
      dmt::colsum_partial_vec<float><<<vg, 128, 0, s>>>((const float*)in, rows, cols, ld, rows_per, g_colsum_scratch);
    else if (dtype == DMT_BF16)
      dmt::colsum_partial_vec<__nv_bfloat16><<<vg, 128, 0, s>>>((const __nv_bfloat16*)in, rows, cols, ld, rows_per,
                                                                g_colsum_scratch);
    else
      dmt::colsum_partial_vec<__half><<<vg, 128, 0, s>>>((const __half*)in, rows, cols, ld, rows_per, g_colsum_scratch);
    dmt::colsum_final<<<(unsigned)dmt::ceil_div(cols, 32), 256, 0, s>>>(g_colsum_scratch, cols, nparts, out);
    DMT_CHECK_LAUNCH();
    return DMT_OK;
  }
  dim3 grid((unsigned)dmt::ceil_div(cols, 256), nparts);
  switch (dtype) {
    case DMT_F32: dmt::colsum_partial<float><<<grid, 256, 0, s>>>((const float*)in, rows, cols, ld, rows_per, g_colsum_scratch); break;
    case DMT_BF16: dmt::colsum_partial<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)in, rows, cols, ld, rows_per, g_colsum_scratch); break;
    case DMT_F64: dmt::colsum_partial<double><<<grid, 256, 0, s>>>((const double*)in, rows, cols, ld, rows_per, g_colsum_scratch); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  dmt::colsum_final<<<(unsigned)dmt::ceil_div(cols, 32), 256, 0, s>>>(g_colsum_scratch, cols, nparts, out);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_cross_bwd_pointwise(const void* g, const void* x0, const void* u, void* gu, float* dx0, int64_t n,
                            int32_t dtype, dmt_stream_t stream) {
  if (n == 0) return DMT_OK;
  unsigned grid = (unsigned)std::min<int64_t>(dmt::ceil_div(n, 256), DMT_NUM_SMS * 16);
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32: dmt::cross_bwd_pointwise_kernel<float><<<grid, 256, 0, s>>>((const float*)g, (const float*)x0, (const float*)u, (float*)gu, dx0, n); break;
    case DMT_BF16: dmt::cross_bwd_pointwise_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((const __nv_bfloat16*)g, (const __nv_bfloat16*)x0, (const __nv_bfloat16*)u, (__nv_bfloat16*)gu, dx0, n); break;
    case DMT_F64: dmt::cross_bwd_pointwise_kernel<double><<<grid, 256, 0, s>>>((const double*)g, (const double*)x0, (const double*)u, (double*)gu, dx0, n); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

size_t dmt_dcn_side_fused_workspace_size(int64_t rows, int64_t cols, int32_t nlayers) {
  return sizeof(double) * (size_t)colsum_parts(rows) * (size_t)(cols > 0 ? cols : 1) * (size_t)(nlayers > 0 ? nlayers : 1);
}

int dmt_dcn_side_fused(const void* const* g, const void* const* u, const void* const* gu, int32_t nlayers,
                       int64_t rows, int64_t cols, float* dx0, float* const* colsums, int32_t dtype, void* workspace,
                       size_t workspace_bytes, dmt_stream_t stream) {
  if (nlayers < 1 || nlayers > 4 || rows < 0 || cols < 0) return DMT_ERR_DOMAIN;
  if (rows == 0 || cols == 0) return DMT_OK;
  if (dtype != DMT_BF16 && dtype != DMT_F16) return DMT_ERR_UNSUPPORTED;
  if (cols % 8 || ((uintptr_t)dx0 & 15)) return DMT_ERR_DOMAIN;
  for (int l = 0; l < nlayers; ++l) {
    if (((uintptr_t)g[l] | (uintptr_t)u[l]) & 15) return DMT_ERR_DOMAIN;
    if (colsums && (!gu || ((uintptr_t)gu[l] & 15) || !colsums[l])) return DMT_ERR_DOMAIN;
  }
  if (workspace_bytes < dmt_dcn_side_fused_workspace_size(rows, cols, nlayers)) return DMT_ERR_DOMAIN;
  cudaStream_t s = (cudaStream_t)stream;
  dmt::SidePtrs P = {};
  for (int l = 0; l < nlayers; ++l) { P.g[l] = g[l]; P.u[l] = u[l]; }
  const int64_t n = rows * cols;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(dmt::ceil_div(n / 8, 256), DMT_NUM_SMS * 8));
#define DMT_SIDE(T, NL) dmt::dcn_dx0_sum_kernel<T, NL><<<grid, 256, 0, s>>>(P, n, dx0)
  if (dtype == DMT_BF16) {
    switch (nlayers) {
      case 1: DMT_SIDE(__nv_bfloat16, 1); break;
      case 2: DMT_SIDE(__nv_bfloat16, 2); break;
      case 3: DMT_SIDE(__nv_bfloat16, 3); break;
      default: DMT_SIDE(__nv_bfloat16, 4); break;
    }
  } else {
    switch (nlayers) {
      case 1: DMT_SIDE(__half, 1); break;
      case 2: DMT_SIDE(__half, 2); break;
      case 3: DMT_SIDE(__half, 3); break;
      default: DMT_SIDE(__half, 4); break;
    }
  }
#undef DMT_SIDE
  // bias gradients: the dmt_column_sum kernels (same partials, same order);
  // colsums == NULL: dx0 only
  const size_t per = sizeof(double) * (size_t)colsum_parts(rows) * (size_t)cols;
  for (int l = 0; colsums && l < nlayers; ++l) {
    const int rc = dmt_column_sum(gu[l], rows, cols, cols, colsums[l], dtype, (char*)workspace + l * per, per, stream);
    if (rc != DMT_OK) return rc;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_dcn_dx0_term(const void* g, const void* u, float* dx0, int64_t n, int32_t dtype, int32_t accumulate,
                     dmt_stream_t stream) {
  if (n == 0) return DMT_OK;
  if (((uintptr_t)g | (uintptr_t)u | (uintptr_t)dx0) & 15) return DMT_ERR_DOMAIN;
  cudaStream_t s = (cudaStream_t)stream;
  auto grid = [&](int V) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(dmt::ceil_div(n / V + 1, 256), DMT_NUM_SMS * 8));
  };
  switch (dtype) {
    case DMT_F32: dmt::dcn_dx0_term_kernel<float, 4><<<grid(4), 256, 0, s>>>((const float*)g, (const float*)u, dx0, n, accumulate); break;
    case DMT_BF16: dmt::dcn_dx0_term_kernel<__nv_bfloat16, 8><<<grid(8), 256, 0, s>>>((const __nv_bfloat16*)g, (const __nv_bfloat16*)u, dx0, n, accumulate); break;
    case DMT_F16: dmt::dcn_dx0_term_kernel<__half, 8><<<grid(8), 256, 0, s>>>((const __half*)g, (const __half*)u, dx0, n, accumulate); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_sgd_dense(void* w, const float* g, int64_t n, float lr, int32_t dtype, dmt_stream_t stream) {
  if (n == 0) return DMT_OK;
  unsigned grid = (unsigned)std::min<int64_t>(dmt::ceil_div(n, 256), DMT_NUM_SMS * 16);
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32: dmt::sgd_dense_kernel<float><<<grid, 256, 0, s>>>((float*)w, g, n, lr); break;
    case DMT_BF16: dmt::sgd_dense_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((__nv_bfloat16*)w, g, n, lr); break;
    case DMT_F64: dmt::sgd_dense_kernel<double><<<grid, 256, 0, s>>>((double*)w, g, n, lr); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_peer_barrier(int32_t* epoch, int32_t* const* remote_slots, int32_t* const* local_slots, int32_t n,
                     int32_t* err, dmt_stream_t stream) {
  if (n < 0 || n > DMT_MAX_PEER_SRCS || !epoch) return DMT_ERR_SHAPE;
  dmt::BarrierSlots s{};
  for (int i = 0; i < n; ++i) {
    if (!remote_slots[i] || !local_slots[i]) return DMT_ERR_DOMAIN;
    s.remote[i] = remote_slots[i];
    s.local[i] = local_slots[i];
  }
  dmt::peer_barrier_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(epoch, s, n, err);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_peer_sum_sgd(void* w, const float* const* g, int32_t nsrc, int64_t n, float lr, int32_t dtype,
                     dmt_stream_t stream) {
  if (n < 0 || nsrc < 1 || nsrc > DMT_MAX_PEER_SRCS || !g) return DMT_ERR_SHAPE;
  if (n == 0) return DMT_OK;
  dmt::PeerSrcs src{};
  for (int m = 0; m < nsrc; ++m) {
    if (!g[m] || (reinterpret_cast<uintptr_t>(g[m]) & 15)) return DMT_ERR_SHAPE;
    src.g[m] = g[m];
  }
  // a small grid: runs beside the embedding-backward apply kernel
  unsigned grid = (unsigned)std::min<int64_t>(dmt::ceil_div(dmt::ceil_div(n, 4), 256), DMT_NUM_SMS);
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32: dmt::peer_sum_sgd_kernel<float><<<grid, 256, 0, s>>>((float*)w, src, nsrc, n, lr); break;
    case DMT_BF16: dmt::peer_sum_sgd_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>((__nv_bfloat16*)w, src, nsrc, n, lr); break;
    case DMT_F64: dmt::peer_sum_sgd_kernel<double><<<grid, 256, 0, s>>>((double*)w, src, nsrc, n, lr); break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_bce_with_logits(const void* z, const float* y, int64_t n, int32_t dtype, float scale, void* dz,
                        float* loss, dmt_stream_t stream) {
  if (n < 0) return DMT_ERR_SHAPE;
  if (n == 0) return DMT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32: dmt::bce_logits_kernel<float><<<1, 256, 0, s>>>((const float*)z, y, n, scale, (float*)dz, loss); break;
    case DMT_BF16:
      dmt::bce_logits_kernel<__nv_bfloat16><<<1, 256, 0, s>>>((const __nv_bfloat16*)z, y, n, scale,
                                                              (__nv_bfloat16*)dz, loss);
      break;
    default: return DMT_ERR_UNSUPPORTED;
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_convert(const void* src, int32_t dtype_in, void* dst, int32_t dtype_out, int64_t n, dmt_stream_t stream) {
  if (n == 0) return DMT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype_in) {
    case DMT_F32: return dmt::convert_to<float>(src, dst, dtype_out, n, s);
    case DMT_BF16: return dmt::convert_to<__nv_bfloat16>(src, dst, dtype_out, n, s);
    case DMT_F64: return dmt::convert_to<double>(src, dst, dtype_out, n, s);
    case DMT_F16: return dmt::convert_to<__half>(src, dst, dtype_out, n, s);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

}  // extern "C"
