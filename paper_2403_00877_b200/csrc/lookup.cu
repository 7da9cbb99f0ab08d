// Pooled EmbeddingBag forward (fused K3) and its backward with
// fused SGD / row-wise Adagrad (K10).
//
// Forward reference: lookup() pools each bag by a sequential bag-order sum
// (towersim/embedding.py:64-85; `values[list(bag)].sum(axis=0)`), pooling
// "none" selects the single row, empty bags give zeros; row-wise shards filter
// and rebase indices (exchange.py:138-144).  Here a group of G threads owns one
// bag; every thread owns NV 16-byte column vectors of the row, issues U row
// gathers back to back (memory-level parallelism) and then folds them into the
// accumulator strictly in bag order, so fp32 results are bit-identical to the
// reference's sequential sum.  Each segment's output pointer/stride encodes the
// destination layout, which is how the step-c permute and step-d stacking are
// fused into the lookup epilogue (zero extra bytes).
#include <cstdlib>
#include <string>

#include <cub/cub.cuh>

#include "common.cuh"

namespace dmt {

template <typename T> struct Vec16;  // 16-byte vector of T
template <> struct Vec16<float> { using type = float4; static constexpr int N = 4; };
template <> struct Vec16<double> { using type = double2; static constexpr int N = 2; };
template <> struct Vec16<__nv_bfloat16> { using type = uint4; static constexpr int N = 8; };
template <> struct Vec16<__half> { using type = uint4; static constexpr int N = 8; };

template <typename T, int VEC>
struct Loader {
  // Load VEC consecutive T at p (aligned to VEC*sizeof(T) when VEC > 1).
  static __device__ __forceinline__ void load(const T* __restrict__ p, typename Acc<T>::type* v) {
    if constexpr (VEC == 1) {
      v[0] = (typename Acc<T>::type)to_d<T>(__ldg(p));
    } else if constexpr (sizeof(T) == 4) {  // float4
      float4 x = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else if constexpr (sizeof(T) == 8) {  // double2
      double2 x = __ldg(reinterpret_cast<const double2*>(p));
      v[0] = x.x; v[1] = x.y;
    } else {  // 8 x 16-bit
      uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
      const T* h = reinterpret_cast<const T*>(&x);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = to_f<T>(h[i]);
    }
  }
  static __device__ __forceinline__ void store(T* __restrict__ p, const typename Acc<T>::type* v) {
    if constexpr (VEC == 1) {
      p[0] = from_d<T>((double)v[0]);
    } else if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    } else if constexpr (sizeof(T) == 8) {
      *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    } else {
      uint4 x;
      T* h = reinterpret_cast<T*>(&x);
#pragma unroll
      for (int i = 0; i < 8; ++i) h[i] = from_f<T>(v[i]);
      *reinterpret_cast<uint4*>(p) = x;
    }
  }
};

// Raw (unconverted) row fragment kept in registers between issue and fold.
template <typename T, int VEC>
struct Frag {
  using Raw = typename std::conditional<VEC == 1, T, typename Vec16<T>::type>::type;
  Raw r;
  __device__ __forceinline__ void load(const T* __restrict__ p) {
    r = __ldg(reinterpret_cast<const Raw*>(p));
  }
  __device__ __forceinline__ void zero() { r = Raw{}; }
  __device__ __forceinline__ void add_to(typename Acc<T>::type* acc) const {
    if constexpr (VEC == 1) {
      acc[0] += (typename Acc<T>::type)to_d<T>(r);
    } else if constexpr (sizeof(T) == 4) {
      acc[0] += r.x; acc[1] += r.y; acc[2] += r.z; acc[3] += r.w;
    } else if constexpr (sizeof(T) == 8) {
      acc[0] += r.x; acc[1] += r.y;
    } else {
      const T* h = reinterpret_cast<const T*>(&r);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += to_f<T>(h[i]);
    }
  }
};

constexpr int kLookupThreads = 256;
constexpr int kUnroll = 8;  // default rows in flight per thread (see UN below)

// G threads per bag (power of two <= 32), NV vectors of VEC elements per thread.
template <typename T, int VEC, int NV, int UN = kUnroll>
__global__ void __launch_bounds__(kLookupThreads)
pooled_fwd_kernel(const dmt_lookup_segment* __restrict__ segs, const int64_t* __restrict__ offsets,
                  const int32_t* __restrict__ indices, int log2g, int32_t* __restrict__ err) {
  using A = typename Acc<T>::type;
  const dmt_lookup_segment& sg = segs[blockIdx.y];
  const int G = 1 << log2g;
  const int gid = threadIdx.x >> log2g;            // bag slot in block
  const int t = threadIdx.x & (G - 1);             // thread in group
  const int bags_per_block = kLookupThreads >> log2g;
  const int64_t b = (int64_t)blockIdx.x * bags_per_block + gid;
  if (b >= sg.nbags) return;
  const int64_t gb = sg.bag_begin + b;
  const int64_t beg = offsets[gb], end = offsets[gb + 1];
  const int len = (int)(end - beg);
  const T* __restrict__ W = reinterpret_cast<const T*>(sg.weights);
  const int width = sg.width;
  const int64_t ld = sg.ld;
  const int64_t row_begin = sg.row_begin;
  const int64_t rows = sg.rows;
  const bool filt = sg.row_filter != 0;

  A acc[NV][VEC];
#pragma unroll
  for (int v = 0; v < NV; ++v)
#pragma unroll
    for (int e = 0; e < VEC; ++e) acc[v][e] = A(0);

  int col0[NV];
  bool colok[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    col0[v] = (v * G + t) * VEC;
    colok[v] = col0[v] < width;
  }

  if (sg.pooling == DMT_POOL_NONE && len != 1 && err) atomicOr(err, DMT_EBIT_BAGLEN);

  int bad = 0;
  // the next batch's indices are loaded while this batch's rows are in
  // flight, so only a bag's first batch waits on an index load before its
  // row loads (a bag of 20 at UN = 8 paid three index -> row chains)
  int32_t nidx[UN];
#pragma unroll
  for (int u = 0; u < UN; ++u) nidx[u] = (beg + u < end) ? __ldg(indices + beg + u) : 0;
  for (int64_t k0 = beg; k0 < end; k0 += UN) {
    Frag<T, VEC> fr[UN][NV];
    bool use[UN];
    int32_t idx[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      idx[u] = nidx[u];
      nidx[u] = (k0 + UN + u < end) ? __ldg(indices + k0 + UN + u) : 0;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      use[u] = false;
      if (k0 + u < end) {
        const int64_t gi = (int64_t)idx[u];
        int64_t r = gi - row_begin;
        bool in = r >= 0 && r < rows;
        if (!in && (!filt || (sg.table_rows > 0 && (gi < 0 || gi >= sg.table_rows)))) bad = 1;
        use[u] = in;
        const T* rp = W + (in ? r : 0) * ld;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          if (in && colok[v]) fr[u][v].load(rp + col0[v]);
          else fr[u][v].zero();
        }
      }
    }
    // fold strictly in bag order (bit-exact sequential sum)
#pragma unroll
    for (int u = 0; u < UN; ++u)
      if (use[u])
#pragma unroll
        for (int v = 0; v < NV; ++v) fr[u][v].add_to(acc[v]);
  }
  if (bad && err) atomicOr(err, DMT_EBIT_INDEX);

  if (sg.pooling == DMT_POOL_MEAN && len > 0) {
    const A l = (A)len;
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[v][e] = acc[v][e] / l;
  }
  T* __restrict__ out = reinterpret_cast<T*>(sg.out) + b * sg.out_ld;
#pragma unroll
  for (int v = 0; v < NV; ++v)
    if (colok[v]) Loader<T, VEC>::store(out + col0[v], acc[v]);
}

// Generic fallback: any width, scalar columns, one group of 32 threads per bag.
template <typename T>
__global__ void __launch_bounds__(kLookupThreads)
pooled_fwd_scalar_kernel(const dmt_lookup_segment* __restrict__ segs, const int64_t* __restrict__ offsets,
                         const int32_t* __restrict__ indices, int32_t* __restrict__ err) {
  using A = typename Acc<T>::type;
  const dmt_lookup_segment& sg = segs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (kLookupThreads / 32) + warp;
  if (b >= sg.nbags) return;
  const int64_t gb = sg.bag_begin + b;
  const int64_t beg = offsets[gb], end = offsets[gb + 1];
  const int len = (int)(end - beg);
  const T* W = reinterpret_cast<const T*>(sg.weights);
  T* out = reinterpret_cast<T*>(sg.out) + b * sg.out_ld;
  if (sg.pooling == DMT_POOL_NONE && len != 1 && err && lane == 0) atomicOr(err, DMT_EBIT_BAGLEN);
  int bad = 0;
  for (int c = lane; c < sg.width; c += 32) {
    A acc = A(0);
    for (int64_t k = beg; k < end; ++k) {
      const int64_t gi = (int64_t)__ldg(indices + k);
      int64_t r = gi - sg.row_begin;
      if (r < 0 || r >= sg.rows) {
        if (!sg.row_filter || (sg.table_rows > 0 && (gi < 0 || gi >= sg.table_rows))) bad = 1;
        continue;
      }
      acc += (A)to_d<T>(W[r * sg.ld + c]);
    }
    if (sg.pooling == DMT_POOL_MEAN && len > 0) acc = acc / (A)len;
    out[c] = from_d<T>((double)acc);
  }
  if (bad && err) atomicOr(err, DMT_EBIT_INDEX);
}

template <typename T>
int launch_fwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* hs, int32_t n,
               const int64_t* offsets, const int32_t* indices, int32_t* err, cudaStream_t s) {
  constexpr int VEC = Vec16<T>::N;
  int max_w = 0, max_b = 0;
  bool vec_ok = true;
  for (int i = 0; i < n; ++i) {
    const dmt_lookup_segment& g = hs[i];
    if (g.width > max_w) max_w = g.width;
    if (g.nbags > max_b) max_b = g.nbags;
    if (g.width % VEC || g.ld % VEC || g.out_ld % VEC || ((uintptr_t)g.weights & 15) ||
        ((uintptr_t)g.out & 15))
      vec_ok = false;
  }
  if (max_b == 0 || max_w == 0) return DMT_OK;
  if (n > 65535) return DMT_ERR_UNSUPPORTED;
  int nvec = (max_w + VEC - 1) / VEC;  // vectors per row
  if (vec_ok && nvec <= 32 * 4) {
    int G = 1, log2g = 0;
    while (G < nvec && G < 32) { G <<= 1; ++log2g; }
    int NV = (nvec + G - 1) / G;
    int bags_per_block = kLookupThreads / G;
    dim3 grid((unsigned)ceil_div(max_b, bags_per_block), n);
    static int un = [] {
      // rows in flight per thread (DMT_LOOKUP_UNROLL overrides).  With the
      // next batch's indices prefetched, fewer rows per batch at higher
      // occupancy win: C2 bf16 (L = 20) 219 us at 8 (round 1 kernel) ->
      // 218.7 / 210.7 / 213.0 us at 4 / 5 / 6 (tools/lookup_bench.py, one box)
      const char* e = getenv("DMT_LOOKUP_UNROLL");
      return e ? atoi(e) : 5;
    }();
    if (NV == 1 && un == 4)
      pooled_fwd_kernel<T, VEC, 1, 4><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
    else if (NV == 1 && un == 6)
      pooled_fwd_kernel<T, VEC, 1, 6><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
    else if (NV == 1 && un == 12)
      pooled_fwd_kernel<T, VEC, 1, 12><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
    else if (NV == 1 && un == 5)
      pooled_fwd_kernel<T, VEC, 1, 5><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
    else if (NV == 1 && un == 10)
      pooled_fwd_kernel<T, VEC, 1, 10><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
    else if (NV == 1)
      pooled_fwd_kernel<T, VEC, 1><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
    else if (NV == 2)
      pooled_fwd_kernel<T, VEC, 2><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
    else
      pooled_fwd_kernel<T, VEC, 4><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
  } else if (max_w <= 32) {
    int G = 1, log2g = 0;
    while (G < max_w) { G <<= 1; ++log2g; }
    int bags_per_block = kLookupThreads / G;
    dim3 grid((unsigned)ceil_div(max_b, bags_per_block), n);
    pooled_fwd_kernel<T, 1, 1><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, log2g, err);
  } else {
    dim3 grid((unsigned)ceil_div(max_b, kLookupThreads / 32), n);
    pooled_fwd_scalar_kernel<T><<<grid, kLookupThreads, 0, s>>>(segs, offsets, indices, err);
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

// ----------------------------------------------------------------------------
// Backward: (1) per-occurrence sort keys (shard key base + local row) and per-
// bag metadata (gradient row pointer, 1/len for mean, segment id); (2) stable
// radix sort of (key, bag) pairs; (3) one pass over the sorted occurrences:
// the thread group whose chunk holds a run's first occurrence reduces the run
// in sorted (= original occurrence) order and applies SGD / row-wise Adagrad to
// that row once -- deterministic, no atomics.  Each group owns kChunk
// consecutive occurrences and issues the loads of all its run heads together
// (memory-level parallelism; runs are 1-2 long for uniform indices).
// ----------------------------------------------------------------------------
constexpr int kChunk = 4;

// Everything the update needs about a bag, in one 32-byte record (two 16-byte
// loads from the same sector): gradient row, "virtual" weight / state bases
// (already offset by -key_base, so row = base + key * ld), 1/len for mean.
struct __align__(16) BagRec {
  const void* grad;
  const char* wvbase;
  float* svbase;
  float scale;
  uint16_t ld;
  uint16_t width;
};

// group of 8 threads per bag: coalesced key/value writes
__global__ void bwd_keys_kernel(const dmt_lookup_segment* __restrict__ segs, const int64_t* __restrict__ offsets,
                                const int32_t* __restrict__ indices, uint32_t invalid, uint32_t* __restrict__ keys,
                                int32_t* __restrict__ vals, BagRec* __restrict__ recs, int es) {
  const dmt_lookup_segment& sg = segs[blockIdx.y];
  const int sub = threadIdx.x & 7;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  if (b >= sg.nbags) return;
  const int64_t gb = sg.bag_begin + b;
  const int64_t beg = offsets[gb], end = offsets[gb + 1];
  for (int64_t k = beg + sub; k < end; k += 8) {
    int64_t r = (int64_t)__ldg(indices + k) - sg.row_begin;
    bool in = r >= 0 && r < sg.rows;
    keys[k] = in ? (uint32_t)(sg.key_base + r) : invalid;
    vals[k] = (int32_t)gb;
  }
  if (sub == 0) {
    BagRec rec;
    rec.grad = reinterpret_cast<const char*>(sg.out) + (size_t)(b * sg.out_ld) * es;
    rec.wvbase = reinterpret_cast<const char*>(sg.weights) - (ptrdiff_t)(sg.key_base * sg.ld) * es;
    rec.svbase = sg.state ? reinterpret_cast<float*>(sg.state) - sg.key_base : nullptr;
    rec.scale = (sg.pooling == DMT_POOL_MEAN && end > beg) ? 1.f / (float)(end - beg) : 1.f;
    rec.ld = (uint16_t)sg.ld;
    rec.width = (uint16_t)sg.width;
    recs[gb] = rec;
  }
}

template <typename T, int VEC, int NV, int CH>
__global__ void __launch_bounds__(kLookupThreads, 2)
bwd_update_kernel(const uint32_t* __restrict__ skeys, const int32_t* __restrict__ sbags, int64_t nnz,
                  const BagRec* __restrict__ recs, uint32_t invalid, int log2g, int opt, float lr, float eps) {
  using A = typename Acc<T>::type;
  const int G = 1 << log2g;
  const int t = threadIdx.x & (G - 1);
  const int gpw = 32 >> log2g;                      // groups per warp
  const int gin = (threadIdx.x & 31) >> log2g;      // group index inside the warp
  const int64_t warp_global = (int64_t)blockIdx.x * (kLookupThreads / 32) + (threadIdx.x >> 5);
  const int64_t stride = (int64_t)gridDim.x * (kLookupThreads / 32) * gpw * CH;
  // warp-uniform trip count: the Adagrad shuffles below never diverge
  for (int64_t base = warp_global * gpw * CH; base < nnz; base += stride) {
    const int64_t c0 = base + (int64_t)gin * CH;
    uint32_t k[CH + 1];
    const uint32_t prev = (c0 > 0 && c0 <= nnz) ? __ldg(skeys + c0 - 1) : 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u <= CH; ++u) k[u] = (c0 + u < nnz) ? __ldg(skeys + c0 + u) : 0xFFFFFFFEu;
    bool head[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) head[u] = (c0 + u < nnz) && k[u] != invalid && k[u] != (u ? k[u - 1] : prev);
    // level 1: bag records of the run heads
    BagRec rec[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u)
      if (head[u]) rec[u] = recs[__ldg(sbags + c0 + u)];
    // level 2: first gradient row and the weight row of every head, issued
    // together and kept raw until the update
    Frag<T, VEC> g0[CH][NV], w[CH][NV];
#pragma unroll
    for (int u = 0; u < CH; ++u)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int c = (v * G + t) * VEC;
        if (head[u] && c < rec[u].width) {
          g0[u][v].load(reinterpret_cast<const T*>(rec[u].grad) + c);
          w[u][v].load(reinterpret_cast<const T*>(rec[u].wvbase) + (int64_t)k[u] * rec[u].ld + c);
        } else {
          g0[u][v].zero();
          w[u][v].zero();
        }
      }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      A acc[NV][VEC];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[v][e] = A(0);
        g0[u][v].add_to(acc[v]);
        const A sc = head[u] ? (A)rec[u].scale : A(0);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[v][e] *= sc;
      }
      // further occurrences of this row (rare for uniform indices), sorted order
      if (head[u] && k[u + 1] == k[u]) {
        for (int64_t j = c0 + u + 1; j < nnz && __ldg(skeys + j) == k[u]; ++j) {
          const BagRec r2 = recs[__ldg(sbags + j)];
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int c = (v * G + t) * VEC;
            if (c < rec[u].width) {
              A x[VEC];
              Loader<T, VEC>::load(reinterpret_cast<const T*>(r2.grad) + c, x);
#pragma unroll
              for (int e = 0; e < VEC; ++e) acc[v][e] += (A)r2.scale * x[e];
            }
          }
        }
      }
      A step = (A)lr;
      if (opt == DMT_OPT_ROWWISE_ADAGRAD) {
        float sq = 0.f;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < VEC; ++e) sq += (float)(acc[v][e] * acc[v][e]);
        for (int o = G >> 1; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o, G);
        if (head[u]) {
          float* st = rec[u].svbase + k[u];
          const float s_new = *st + sq / (float)rec[u].width;
          step = (A)(lr / (sqrtf(s_new) + eps));
          __syncwarp(__activemask());
          if (t == 0) *st = s_new;
        }
      }
      if (!head[u]) continue;
      T* W = const_cast<T*>(reinterpret_cast<const T*>(rec[u].wvbase)) + (int64_t)k[u] * rec[u].ld;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int c = (v * G + t) * VEC;
        if (c < rec[u].width) {
          A nw[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) nw[e] = A(0);
          w[u][v].add_to(nw);
#pragma unroll
          for (int e = 0; e < VEC; ++e) nw[e] = nw[e] - step * acc[v][e];
          Loader<T, VEC>::store(W + c, nw);
        }
      }
    }
  }
}

// ---- fast path: no mean pooling, all gradient rows in one buffer ----------
// The sort value is the gradient row's 16-byte offset from that buffer, and
// the owning shard of a key is found in a small shard table copied to shared
// memory, so a run head needs exactly two dependent levels of loads (sorted
// key/value -> gradient row + weight row) instead of three.
constexpr int kMaxShards = 96;
struct ShardTab {
  int n;
  uint32_t key_base[kMaxShards];
  uint16_t ld[kMaxShards];
  uint16_t width[kMaxShards];
  const char* weights[kMaxShards];
  float* state[kMaxShards];
};

__global__ void bwd_keys_fast_kernel(const dmt_lookup_segment* __restrict__ segs,
                                     const int64_t* __restrict__ offsets, const int32_t* __restrict__ indices,
                                     uint32_t invalid, uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                     const char* __restrict__ gbase, int es) {
  const dmt_lookup_segment& sg = segs[blockIdx.y];
  const int sub = threadIdx.x & 7;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  if (b >= sg.nbags) return;
  const int64_t gb = sg.bag_begin + b;
  const int64_t beg = offsets[gb], end = offsets[gb + 1];
  const int32_t goff = (int32_t)((reinterpret_cast<const char*>(sg.out) + (size_t)(b * sg.out_ld) * es - gbase) >> 4);
  for (int64_t k = beg + sub; k < end; k += 8) {
    int64_t r = (int64_t)__ldg(indices + k) - sg.row_begin;
    bool in = r >= 0 && r < sg.rows;
    keys[k] = in ? (uint32_t)(sg.key_base + r) : invalid;
    vals[k] = goff;
  }
}

// PF2: the key two positions past each occurrence and the gradient row of the
// next one are prefetched with the chunk, so a run of length 2 (the common
// duplicate: ~8 % of unique rows at C2) issues its second gradient row with
// the head's loads instead of through a dependent key -> value -> row chain.
template <typename T, int VEC, int NV, int CH, int MINB = 2, bool PF2 = false>
__global__ void __launch_bounds__(kLookupThreads, MINB)
bwd_update_fast_kernel(const uint32_t* __restrict__ skeys, const int32_t* __restrict__ svals, int64_t nnz,
                       const char* __restrict__ gbase, const __grid_constant__ ShardTab tab, uint32_t invalid,
                       int log2g, int opt, float lr, float eps) {
  using A = typename Acc<T>::type;
  __shared__ uint32_t s_kb[kMaxShards];
  __shared__ uint16_t s_ld[kMaxShards], s_w[kMaxShards];
  __shared__ const char* s_wp[kMaxShards];
  __shared__ float* s_st[kMaxShards];
  for (int i = threadIdx.x; i < tab.n; i += blockDim.x) {
    s_kb[i] = tab.key_base[i];
    s_ld[i] = tab.ld[i];
    s_w[i] = tab.width[i];
    s_wp[i] = tab.weights[i];
    s_st[i] = tab.state[i];
  }
  // shard of a key: a 1024-bucket table over the key space gives the shard of
  // each bucket's first key, then a short forward walk (usually none) --
  // instead of a ~log2(shards)-deep chain of dependent shared-memory loads
  __shared__ uint8_t s_bk[1024];
  const int bsh = max(0, 32 - __clz(invalid | 1u) - 10);
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    const uint32_t key = (uint32_t)i << bsh;
    int lo = 0, hi = tab.n - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (s_kb[mid] <= key) lo = mid; else hi = mid - 1;
    }
    s_bk[i] = (uint8_t)lo;
  }
  __syncthreads();
  const int nsh = tab.n;
  const int G = 1 << log2g;
  const int t = threadIdx.x & (G - 1);
  const int gpw = 32 >> log2g;
  const int gin = (threadIdx.x & 31) >> log2g;
  const int64_t warp_global = (int64_t)blockIdx.x * (kLookupThreads / 32) + (threadIdx.x >> 5);
  const int64_t stride = (int64_t)gridDim.x * (kLookupThreads / 32) * gpw * CH;
  // software pipeline: the sorted keys / values of the next chunk are loaded
  // while the current chunk's rows are in flight
  constexpr int XK = PF2 ? 1 : 0;  // extra keys / values fetched past the chunk
  uint32_t nk[CH + 2 + XK];
  int32_t ngv[CH + XK];
  auto fetch = [&](int64_t c0) {
#pragma unroll
    for (int u = 0; u <= CH + XK; ++u) nk[u + 1] = (c0 + u < nnz) ? __ldg(skeys + c0 + u) : 0xFFFFFFFEu;
    nk[0] = (c0 > 0 && c0 <= nnz) ? __ldg(skeys + c0 - 1) : 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < CH + XK; ++u) ngv[u] = (c0 + u < nnz) ? __ldg(svals + c0 + u) : 0;
  };
  fetch(warp_global * gpw * CH + (int64_t)gin * CH);
  for (int64_t base = warp_global * gpw * CH; base < nnz; base += stride) {
    const int64_t c0 = base + (int64_t)gin * CH;
    uint32_t k[CH + 1 + XK];
    int32_t gv[CH + XK];
    const uint32_t prev = nk[0];
#pragma unroll
    for (int u = 0; u <= CH + XK; ++u) k[u] = nk[u + 1];
#pragma unroll
    for (int u = 0; u < CH + XK; ++u) gv[u] = ngv[u];
    fetch(c0 + stride);
    bool head[CH];
    int sh[CH];
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      head[u] = (c0 + u < nnz) && k[u] != invalid && k[u] != (u ? k[u - 1] : prev);
      int lo = s_bk[min(k[u] >> bsh, 1023u)];  // last shard with key_base <= key
      while (lo + 1 < nsh && s_kb[lo + 1] <= k[u]) ++lo;
      sh[u] = lo;
    }
    Frag<T, VEC> g0[CH][NV], w[CH][NV];
#pragma unroll
    for (int u = 0; u < CH; ++u)
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int c = (v * G + t) * VEC;
        if (head[u] && c < s_w[sh[u]]) {
          g0[u][v].load(reinterpret_cast<const T*>(gbase + ((int64_t)gv[u] << 4)) + c);
          w[u][v].load(reinterpret_cast<const T*>(s_wp[sh[u]]) + (int64_t)(k[u] - s_kb[sh[u]]) * s_ld[sh[u]] + c);
        } else {
          g0[u][v].zero();
          w[u][v].zero();
        }
      }
    bool dup2[CH];
    Frag<T, VEC> g1[PF2 ? CH : 1][NV];
    if constexpr (PF2) {
#pragma unroll
      for (int u = 0; u < CH; ++u) {
        dup2[u] = head[u] && k[u + 1] == k[u];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int c = (v * G + t) * VEC;
          if (dup2[u] && c < s_w[sh[u]])
            g1[u][v].load(reinterpret_cast<const T*>(gbase + ((int64_t)gv[u + 1] << 4)) + c);
          else
            g1[u][v].zero();
        }
      }
    }
#pragma unroll
    for (int u = 0; u < CH; ++u) {
      const int width = s_w[sh[u]];
      A acc[NV][VEC];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[v][e] = A(0);
        g0[u][v].add_to(acc[v]);
        if constexpr (PF2) g1[u][v].add_to(acc[v]);
      }
      if (PF2 ? (dup2[u] && k[u + 2] == k[u]) : (head[u] && k[u + 1] == k[u])) {
        for (int64_t j = c0 + u + 1 + XK; j < nnz && __ldg(skeys + j) == k[u]; ++j) {
          const T* gp = reinterpret_cast<const T*>(gbase + ((int64_t)__ldg(svals + j) << 4));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int c = (v * G + t) * VEC;
            if (c < width) {
              A x[VEC];
              Loader<T, VEC>::load(gp + c, x);
#pragma unroll
              for (int e = 0; e < VEC; ++e) acc[v][e] += x[e];
            }
          }
        }
      }
      A step = (A)lr;
      if (opt == DMT_OPT_ROWWISE_ADAGRAD) {
        float sq = 0.f;
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
          for (int e = 0; e < VEC; ++e) sq += (float)(acc[v][e] * acc[v][e]);
        for (int o = G >> 1; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o, G);
        if (head[u]) {
          float* st = s_st[sh[u]] + (k[u] - s_kb[sh[u]]);
          const float s_new = *st + sq / (float)width;
          step = (A)(lr / (sqrtf(s_new) + eps));
          __syncwarp(__activemask());
          if (t == 0) *st = s_new;
        }
      }
      if (!head[u]) continue;
      T* W = const_cast<T*>(reinterpret_cast<const T*>(s_wp[sh[u]])) + (int64_t)(k[u] - s_kb[sh[u]]) * s_ld[sh[u]];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const int c = (v * G + t) * VEC;
        if (c < width) {
          A nw[VEC];
#pragma unroll
          for (int e = 0; e < VEC; ++e) nw[e] = A(0);
          w[u][v].add_to(nw);
#pragma unroll
          for (int e = 0; e < VEC; ++e) nw[e] = nw[e] - step * acc[v][e];
          Loader<T, VEC>::store(W + c, nw);
        }
      }
    }
  }
}

// ---- asynchronous-copy variant of the fast path ----------------------------
// Each warp owns chunks of R = 256 / NVEC sorted occurrences.  For a chunk it
// resolves keys, run heads and row addresses (lane = occurrence), then streams
// the gradient rows of all its occurrences and the weight rows of its run
// heads into a 3-deep shared-memory ring with cp.async (16 B per request, no
// registers held while in flight), so ~2 chunks per warp stay in flight.  The
// update reads both from shared memory; a run that continues past the chunk
// end is finished with direct loads (rare for uniform indices).
constexpr int kAsyncWarps = 8;
constexpr int kAsyncStages = 3;
constexpr int kAsyncVecs = 256;  // 16-byte vectors per array per chunk (4 KB)

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(smem)),
      "l"(gmem), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}

struct ChunkMeta {
  uint32_t key;
  int32_t head;
  const char* grad;
  char* wrow;
  float* srow;
};

template <typename T, int NVEC>
__global__ void __launch_bounds__(kAsyncWarps * 32, 1)
bwd_update_async_kernel(const uint32_t* __restrict__ skeys, const int32_t* __restrict__ svals, int64_t nnz,
                        const char* __restrict__ gbase, const __grid_constant__ ShardTab tab, uint32_t invalid,
                        int opt, float lr, float eps) {
  using A = typename Acc<T>::type;
  constexpr int R = kAsyncVecs / NVEC;          // occurrences per chunk (<= 32)
  constexpr int VEC = 16 / sizeof(T);           // elements per vector
  constexpr int RPS = 32 / NVEC;                // rows processed per warp step
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint4* ring = reinterpret_cast<uint4*>(smem_raw);  // [warps][stages][2][256] x 16 B
  ChunkMeta* meta_all = reinterpret_cast<ChunkMeta*>(smem_raw + (size_t)kAsyncWarps * kAsyncStages * 2 *
                                                                    kAsyncVecs * 16);
  uint64_t* bars_all = reinterpret_cast<uint64_t*>(meta_all + (size_t)kAsyncWarps * kAsyncStages * (R + 1));
  __shared__ uint32_t s_kb[kMaxShards];
  __shared__ uint16_t s_ld[kMaxShards];
  __shared__ const char* s_wp[kMaxShards];
  __shared__ float* s_st[kMaxShards];
  for (int i = threadIdx.x; i < tab.n; i += blockDim.x) {
    s_kb[i] = tab.key_base[i];
    s_ld[i] = tab.ld[i];
    s_wp[i] = tab.weights[i];
    s_st[i] = tab.state[i];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* wring = ring + (size_t)warp * kAsyncStages * 2 * kAsyncVecs;
  ChunkMeta* wmeta = meta_all + (size_t)warp * kAsyncStages * (R + 1);
  uint64_t* wbars = bars_all + warp * kAsyncStages;
  if (lane < kAsyncStages) mbar_init1(&wbars[lane]);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  uint32_t parity_bits = 0;  // per-stage phase parity
  const int64_t nchunks = ceil_div(nnz, R);
  const int64_t wstride = (int64_t)gridDim.x * kAsyncWarps;
  const int64_t first = (int64_t)blockIdx.x * kAsyncWarps + warp;

  // keys / values of a chunk are fetched into registers one chunk ahead of the
  // resolve + copy issue, so their latency overlaps the previous chunk's work
  uint32_t rk = 0, rkp = 0;
  int32_t rgv = 0;
  int64_t rc = -1;
  auto fetch = [&](int64_t c) {
    rc = c;
    if (c < nchunks && lane <= R) {
      const int64_t pos = c * R + lane;
      rk = pos < nnz ? __ldg(skeys + pos) : 0xFFFFFFFEu;
      rkp = pos > 0 && pos <= nnz ? __ldg(skeys + pos - 1) : 0xFFFFFFFFu;
      rgv = (lane < R && pos < nnz) ? __ldg(svals + pos) : 0;
    }
  };
  // resolve the fetched chunk into stage `st` and issue its copies (one group)
  auto issue = [&](int st) {
    ChunkMeta* m = wmeta + st * (R + 1);
    const int64_t c = rc;
    if (c < nchunks) {
      const int64_t pos = c * R + lane;
      if (lane <= R) {
        const uint32_t k = rk;
        ChunkMeta mm;
        mm.key = k;
        mm.head = (lane < R && pos < nnz && k != invalid && k != rkp) ? 1 : 0;
        mm.grad = (lane < R && pos < nnz) ? gbase + ((int64_t)rgv << 4) : nullptr;
        mm.wrow = nullptr;
        mm.srow = nullptr;
        if (mm.head) {
          int lo = 0, hi = tab.n - 1;
          while (lo < hi) {
            int mid = (lo + hi + 1) >> 1;
            if (s_kb[mid] <= k) lo = mid; else hi = mid - 1;
          }
          const int64_t row = (int64_t)(k - s_kb[lo]);
          mm.wrow = const_cast<char*>(s_wp[lo]) + row * s_ld[lo] * (int64_t)sizeof(T);
          mm.srow = s_st[lo] ? s_st[lo] + row : nullptr;
        }
        m[lane] = mm;
      }
      __syncwarp();
      // one bulk (TMA) copy per row and array, issued by the row's own lane
      uint4* gbuf = wring + (size_t)st * 2 * kAsyncVecs;
      uint4* wbuf = gbuf + kAsyncVecs;
      constexpr uint32_t RB = NVEC * 16;
      uint32_t mine = 0;
      if (lane < R) {
        const ChunkMeta& mi = m[lane];
        if (mi.grad && mi.key != invalid) {
          bulk_g2s(gbuf + lane * NVEC, mi.grad, RB, &wbars[st]);
          mine += RB;
        }
        if (mi.head) {
          bulk_g2s(wbuf + lane * NVEC, mi.wrow, RB, &wbars[st]);
          mine += RB;
        }
      }
      const uint32_t total = __reduce_add_sync(0xffffffffu, mine);
      if (lane == 0) mbar_arrive_tx(&wbars[st], total);
    } else if (lane == 0) {
      mbar_arrive_tx(&wbars[st], 0);  // keep the stage's phase sequence uniform
    }
  };

  int64_t c = first;
  fetch(c);
  issue(0);
  fetch(c + wstride);
  issue(1);
  fetch(c + 2 * wstride);
  for (int st = 0; c < nchunks; c += wstride, st = (st + 1) % kAsyncStages) {
    issue((st + 2) % kAsyncStages);  // chunk c + 2*stride (keys fetched last iteration)
    fetch(c + 3 * wstride);          // keys of chunk c + 3*stride, consumed next iteration
    mbar_wait_parity(&wbars[st], (parity_bits >> st) & 1u);
    parity_bits ^= 1u << st;
    __syncwarp();
    const ChunkMeta* m = wmeta + st * (R + 1);
    const uint4* gbuf = wring + (size_t)st * 2 * kAsyncVecs;
    const uint4* wbuf = gbuf + kAsyncVecs;
    const int64_t p0 = c * R;
    const int sub = lane / NVEC, v = lane % NVEC;
#pragma unroll 1
    for (int s = 0; s < R; s += RPS) {
      const int i = s + sub;
      const ChunkMeta mi = m[i];
      A acc[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) acc[e] = A(0);
      if (mi.head) {
        Frag<T, VEC> f;
        f.r = *reinterpret_cast<const typename Frag<T, VEC>::Raw*>(&gbuf[i * NVEC + v]);
        f.add_to(acc);
        int q = i + 1;
        for (; q < R && m[q].key == mi.key; ++q) {
          Frag<T, VEC> f2;
          f2.r = *reinterpret_cast<const typename Frag<T, VEC>::Raw*>(&gbuf[q * NVEC + v]);
          f2.add_to(acc);
        }
        if (q == R) {  // the run may continue into the next chunk(s)
          for (int64_t j = p0 + R; j < nnz && __ldg(skeys + j) == mi.key; ++j) {
            A x[VEC];
            Loader<T, VEC>::load(reinterpret_cast<const T*>(gbase + ((int64_t)__ldg(svals + j) << 4)) + v * VEC, x);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[e] += x[e];
          }
        }
      }
      A step = (A)lr;
      if (opt == DMT_OPT_ROWWISE_ADAGRAD) {
        float sq = 0.f;
#pragma unroll
        for (int e = 0; e < VEC; ++e) sq += (float)(acc[e] * acc[e]);
        for (int o = NVEC >> 1; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o, NVEC);
        if (mi.head) {
          const float s_new = *mi.srow + sq / (float)(NVEC * VEC);
          step = (A)(lr / (sqrtf(s_new) + eps));
          __syncwarp(__activemask());
          if (v == 0) *mi.srow = s_new;
        }
      }
      if (mi.head) {
        Frag<T, VEC> wf;
        wf.r = *reinterpret_cast<const typename Frag<T, VEC>::Raw*>(&wbuf[i * NVEC + v]);
        A nw[VEC];
#pragma unroll
        for (int e = 0; e < VEC; ++e) nw[e] = A(0);
        wf.add_to(nw);
#pragma unroll
        for (int e = 0; e < VEC; ++e) nw[e] = nw[e] - step * acc[e];
        Loader<T, VEC>::store(reinterpret_cast<T*>(mi.wrow) + v * VEC, nw);
      }
    }
    __syncwarp();
  }
  // stages issued past the last chunk carry no copies (0-byte arrivals)
}

template <typename T, int NVEC>
int launch_async_update(const uint32_t* keys, const int32_t* vals, int64_t nnz, const char* gbase,
                        const ShardTab& tab, uint32_t invalid, int opt, float lr, float eps, cudaStream_t s) {
  constexpr int R = kAsyncVecs / NVEC;
  const size_t smem = (size_t)kAsyncWarps * kAsyncStages * 2 * kAsyncVecs * 16 +
                      (size_t)kAsyncWarps * kAsyncStages * (R + 1) * sizeof(ChunkMeta) +
                      (size_t)kAsyncWarps * kAsyncStages * 8;
  auto kern = bwd_update_async_kernel<T, NVEC>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return DMT_ERR_CUDA;
    attr = true;
  }
  const int64_t nchunks = ceil_div(nnz, R);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nchunks, kAsyncWarps),
                                                                          DMT_NUM_SMS));
  kern<<<grid, kAsyncWarps * 32, smem, s>>>(keys, vals, nnz, gbase, tab, invalid, opt, lr, eps);
  return DMT_OK;
}

// ---- bucketed backward (the default fast path) -----------------------------
// Prepare (needs only the indices; runs on a side stream under the tower
// module): every valid occurrence's sort key (shard key base + row) is
// counted into its bucket of 2^bshift consecutive keys, the counts are
// scanned, and each occurrence is scattered into its bucket as one 64-bit item
// (key << 32 | 16-byte offset of its gradient row).  Apply (needs the
// gradients): each CTA takes whole buckets, sorts a bucket's items in shared
// memory by (key, gradient row) -- a canonical order, so the update does not
// depend on the scatter's arrival order (deterministic, no float atomics) --
// compacts the run heads (one per unique row), and every thread group reduces
// one run in that order and applies SGD / row-wise Adagrad to the row once.
// Replaces the 25-bit CUB radix sort + the key -> shard -> row dependent chain
// of the earlier apply: rows of a bucket are resolved from shared memory.
constexpr int kBktThreads = 256;
constexpr int kBktCap = 2048;  // items of one bucket sorted in shared memory at once

inline int bucket_shift(int64_t nnz, int64_t key_space) {
  // widest bucket whose mean population (uniform keys) stays <= 1024 items
  int s = 4;
  const double dens = (double)std::max<int64_t>(nnz, 1) / (double)std::max<int64_t>(key_space, 1);
  while (s < 20 && dens * (double)(1ll << (s + 1)) <= 1024.0) ++s;
  return s;
}

inline int64_t bucket_count(int64_t key_space, int bshift) { return (key_space >> bshift) + 1; }

// keys of positions no bag covers (a capacity-padded step a hands the backward
// more value slots than occurrences) must sort last and be skipped: fill with
// the invalid key first
__global__ void fill_u32_kernel(uint32_t* __restrict__ p, int64_t n, uint32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void bwd_bucket_keys_kernel(const dmt_lookup_segment* __restrict__ segs,
                                       const int64_t* __restrict__ offsets, const int32_t* __restrict__ indices,
                                       uint32_t invalid, uint32_t* __restrict__ keys, int32_t* __restrict__ vals,
                                       const char* __restrict__ gbase, int es, int bshift,
                                       uint32_t* __restrict__ counts) {
  const dmt_lookup_segment& sg = segs[blockIdx.y];
  const int sub = threadIdx.x & 7;
  const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  if (b >= sg.nbags) return;
  const int64_t gb = sg.bag_begin + b;
  const int64_t beg = offsets[gb], end = offsets[gb + 1];
  const int32_t goff = (int32_t)((reinterpret_cast<const char*>(sg.out) + (size_t)(b * sg.out_ld) * es - gbase) >> 4);
  for (int64_t k = beg + sub; k < end; k += 8) {
    const int64_t r = (int64_t)__ldg(indices + k) - sg.row_begin;
    const bool in = r >= 0 && r < sg.rows;
    const uint32_t key = in ? (uint32_t)(sg.key_base + r) : invalid;
    keys[k] = key;
    vals[k] = goff;
    if (in) atomicAdd(counts + (key >> bshift), 1u);
  }
}

// exclusive scan of counts[0, n) into offs[0, n]; cursor = offs (one CTA)
__global__ void __launch_bounds__(1024) bucket_scan_kernel(const uint32_t* __restrict__ counts, int64_t n,
                                                           uint32_t* __restrict__ offs, uint32_t* __restrict__ cursor) {
  __shared__ uint32_t warp_tot[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < n; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < n ? counts[i] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t excl = carry + (wid ? warp_tot[wid - 1] : 0u) + x - v;
    if (i < n) {
      offs[i] = excl;
      cursor[i] = excl;
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) offs[n] = carry;
}

__global__ void bwd_bucket_scatter_kernel(const uint32_t* __restrict__ keys, const int32_t* __restrict__ vals,
                                          int64_t nnz, uint32_t invalid, int bshift, uint32_t* __restrict__ cursor,
                                          uint64_t* __restrict__ items) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = __ldg(keys + k);
    if (key == invalid) continue;
    const uint32_t pos = atomicAdd(cursor + (key >> bshift), 1u);
    items[pos] = ((uint64_t)key << 32) | (uint32_t)__ldg(vals + k);
  }
}

// in-place ascending bitonic sort of s[0, P), P a power of two (block-wide)
__device__ __forceinline__ void bitonic_smem(uint64_t* s, int P) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = s[i], b = s[ixj];
          if ((a > b) == ((i & k) == 0)) {
            s[i] = b;
            s[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
}

// the same over global memory (oversized buckets: skewed / hot keys), with
// the strides below kBktCap done in shared memory per chunk
__device__ void bitonic_global(uint64_t* g, int64_t P, uint64_t* s) {
  const int C = kBktCap;
  auto local_stages = [&](int64_t k, int jmax) {
    // strides jmax..1 of merge level k, chunk by chunk through shared memory
    for (int64_t c0 = 0; c0 < P; c0 += C) {
      for (int i = threadIdx.x; i < C; i += blockDim.x) s[i] = g[c0 + i];
      __syncthreads();
      for (int j = jmax; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < C; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const uint64_t a = s[i], b = s[ixj];
            if ((a > b) == (((c0 + i) & k) == 0)) {
              s[i] = b;
              s[ixj] = a;
            }
          }
        }
        __syncthreads();
      }
      for (int i = threadIdx.x; i < C; i += blockDim.x) g[c0 + i] = s[i];
      __syncthreads();
    }
  };
  for (int64_t k = 2; k <= P; k <<= 1) {
    int64_t j = k >> 1;
    for (; j >= C; j >>= 1) {
      for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
        const int64_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t a = g[i], b = g[ixj];
          if ((a > b) == ((i & k) == 0)) {
            g[i] = b;
            g[ixj] = a;
          }
        }
      }
      __syncthreads();
    }
    local_stages(k, (int)j);
  }
}

template <typename T, int VEC, int NV>
__global__ void __launch_bounds__(kBktThreads, 4)
bwd_bucket_apply_kernel(const uint64_t* __restrict__ items, const uint32_t* __restrict__ boff, int64_t nbuckets,
                        uint64_t* __restrict__ scratch, const char* __restrict__ gbase,
                        const __grid_constant__ ShardTab tab, int log2g, int opt, float lr, float eps) {
  using A = typename Acc<T>::type;
  __shared__ uint64_t s_items[kBktCap];
  __shared__ uint16_t s_run[kBktCap + 1];
  __shared__ uint32_t s_wsum[kBktThreads / 32];
  __shared__ int s_nruns;
  __shared__ uint32_t s_kb[kMaxShards];
  __shared__ uint16_t s_ld[kMaxShards], s_w[kMaxShards];
  __shared__ const char* s_wp[kMaxShards];
  __shared__ float* s_st[kMaxShards];
  for (int i = threadIdx.x; i < tab.n; i += blockDim.x) {
    s_kb[i] = tab.key_base[i];
    s_ld[i] = tab.ld[i];
    s_w[i] = tab.width[i];
    s_wp[i] = tab.weights[i];
    s_st[i] = tab.state[i];
  }
  __syncthreads();
  const int nsh = tab.n;
  const int G = 1 << log2g;
  const int t = threadIdx.x & (G - 1);
  const int gid = threadIdx.x >> log2g;
  const int ngroups = kBktThreads >> log2g;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int E = kBktCap / kBktThreads;  // window items per thread in the head scan

  for (int64_t bk = blockIdx.x; bk < nbuckets; bk += gridDim.x) {
    const int64_t beg = boff[bk];
    const int64_t n = (int64_t)boff[bk + 1] - beg;
    if (n == 0) continue;
    const uint64_t* src;  // the bucket's items, sorted
    if (n <= kBktCap) {
      int P = 2;
      while (P < n) P <<= 1;
      for (int i = threadIdx.x; i < P; i += blockDim.x) s_items[i] = i < n ? items[beg + i] : ~0ull;
      __syncthreads();
      bitonic_smem(s_items, P);
      src = nullptr;
    } else {
      int64_t P = kBktCap;
      while (P < n) P <<= 1;
      uint64_t* g = scratch + 2 * beg;  // P <= 2n: disjoint per bucket
      for (int64_t i = threadIdx.x; i < P; i += blockDim.x) g[i] = i < n ? items[beg + i] : ~0ull;
      __syncthreads();
      bitonic_global(g, P, s_items);
      src = g;
    }
    for (int64_t w0 = 0; w0 < n; w0 += kBktCap) {
      const int wn = (int)(n - w0 < kBktCap ? n - w0 : (int64_t)kBktCap);
      if (src) {
        for (int i = threadIdx.x; i < wn; i += blockDim.x) s_items[i] = src[w0 + i];
        __syncthreads();
      }
      const uint32_t prev_key = w0 > 0 ? (uint32_t)(src[w0 - 1] >> 32) : 0xFFFFFFFFu;
      // run heads of the window -> s_run[0, nruns) (block scan of head flags)
      uint32_t cnt = 0;
      bool hd[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = threadIdx.x * E + e;
        hd[e] = false;
        if (i < wn) {
          const uint32_t k = (uint32_t)(s_items[i] >> 32);
          const uint32_t kp = i ? (uint32_t)(s_items[i - 1] >> 32) : prev_key;
          hd[e] = k != kp;
        }
        cnt += hd[e];
      }
      uint32_t x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) s_wsum[wid] = x;
      __syncthreads();
      uint32_t before = x - cnt;
      for (int w = 0; w < wid; ++w) before += s_wsum[w];
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (hd[e]) s_run[before++] = (uint16_t)(threadIdx.x * E + e);
      if (threadIdx.x == kBktThreads - 1) s_nruns = (int)before;
      __syncthreads();
      const int nruns = s_nruns;
      // one run (= one unique row) per thread group; warp-uniform trip count
      // (the Adagrad reduction shuffles across the whole warp)
      const int gpw = 32 >> log2g;
      for (int rb = (gid / gpw) * gpw; rb < nruns; rb += ngroups) {
        const int r = rb + gid % gpw;
        if (r >= nruns) continue;  // whole-group uniform; Adagrad below masks by active groups
        const int i0 = s_run[r];
        const uint32_t key = (uint32_t)(s_items[i0] >> 32);
        int lo = 0, hi = nsh - 1;  // last shard with key_base <= key
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_kb[mid] <= key) lo = mid; else hi = mid - 1;
        }
        const int width = s_w[lo];
        const int64_t row = (int64_t)(key - s_kb[lo]);
        T* W = const_cast<T*>(reinterpret_cast<const T*>(s_wp[lo])) + row * s_ld[lo];
        Frag<T, VEC> w[NV], g0[NV];
        const T* gp0 = reinterpret_cast<const T*>(gbase + ((int64_t)(uint32_t)s_items[i0] << 4));
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int c = (v * G + t) * VEC;
          if (c < width) {
            w[v].load(W + c);
            g0[v].load(gp0 + c);
          } else {
            w[v].zero();
            g0[v].zero();
          }
        }
        A acc[NV][VEC];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
#pragma unroll
          for (int e = 0; e < VEC; ++e) acc[v][e] = A(0);
          g0[v].add_to(acc[v]);
        }
        // the rest of the run, in sorted order (may run past the window)
        for (int64_t j = w0 + i0 + 1; j < n; ++j) {
          const uint64_t it = (j - w0 < wn) ? s_items[j - w0] : src[j];
          if ((uint32_t)(it >> 32) != key) break;
          const T* gp = reinterpret_cast<const T*>(gbase + ((int64_t)(uint32_t)it << 4));
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            const int c = (v * G + t) * VEC;
            if (c < width) {
              A xx[VEC];
              Loader<T, VEC>::load(gp + c, xx);
#pragma unroll
              for (int e = 0; e < VEC; ++e) acc[v][e] += xx[e];
            }
          }
        }
        A step = (A)lr;
        if (opt == DMT_OPT_ROWWISE_ADAGRAD) {
          float sq = 0.f;
#pragma unroll
          for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < VEC; ++e) sq += (float)(acc[v][e] * acc[v][e]);
          const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
          for (int o = G >> 1; o > 0; o >>= 1) sq += __shfl_xor_sync(gmask, sq, o, G);
          float* st = s_st[lo] + row;
          const float s_new = *st + sq / (float)width;
          step = (A)(lr / (sqrtf(s_new) + eps));
          __syncwarp(__activemask());
          if (t == 0) *st = s_new;
        }
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          const int c = (v * G + t) * VEC;
          if (c < width) {
            A nw[VEC];
#pragma unroll
            for (int e = 0; e < VEC; ++e) nw[e] = A(0);
            w[v].add_to(nw);
#pragma unroll
            for (int e = 0; e < VEC; ++e) nw[e] = nw[e] - step * acc[v][e];
            Loader<T, VEC>::store(W + c, nw);
          }
        }
      }
      __syncthreads();  // s_items / s_run reused by the next window / bucket
    }
  }
}

// ---- hand-written LSD radix sort of (key, value) pairs -----------------------
// The prepare's sort: keys < 2^end_bit (25 bits at C2: 26 shards x 1M rows),
// values = 16-byte gradient-row offsets.  ceil(end_bit / 9) stable passes of
// <= 9-bit digits (3 at C2, vs CUB onesweep's 4 x 8 bits), each pass three
// kernels over 4096-element tiles:
//   upsweep   per-tile digit histogram (shared-memory atomics) -> counts[d][t]
//   scan      exclusive scan of counts in digit-major order (tile order within
//             a digit: what makes the pass stable across tiles)
//   downsweep stable rank inside the tile -- warp w ranks its 512-element
//             sub-tile as 4 independent 128-element streams (4 steps of 32,
//             __match_any_sync against a per-stream digit counter; the four
//             chains interleave), streams and warps combined in element
//             order -- then the tile is reordered by (digit, rank) in shared
//             memory and stored so consecutive threads write consecutive
//             slots of one digit's run.
// The order equals any stable sort's (identical to the CUB path), so the
// apply's summation order and results are unchanged.
constexpr int kRadixBits = 9;
constexpr int kRadixBins = 1 << kRadixBits;
constexpr int kRadixThreads = 256;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixItems = 16;                              // per thread
constexpr int kRadixTile = kRadixThreads * kRadixItems;      // 4096
constexpr int kRadixSub = kRadixTile / kRadixWarps;          // 512 per warp

inline int radix_passes(int end_bit) { return (end_bit + kRadixBits - 1) / kRadixBits; }
inline int radix_digit_bits(int end_bit) {
  const int np = radix_passes(end_bit);
  return (end_bit + np - 1) / np;
}

__global__ void __launch_bounds__(kRadixThreads) radix_upsweep(const uint32_t* __restrict__ keys, int64_t n,
                                                               int shift, uint32_t mask, int64_t ntiles,
                                                               uint32_t* __restrict__ counts) {
  __shared__ uint32_t hist[kRadixBins];
  for (int i = threadIdx.x; i < kRadixBins; i += kRadixThreads) hist[i] = 0;
  __syncthreads();
  const int64_t t = blockIdx.x;
  const int64_t base = t * kRadixTile;
  uint32_t k[kRadixItems];
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    const int64_t idx = base + i * kRadixThreads + threadIdx.x;
    k[i] = idx < n ? __ldg(keys + idx) : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i)
    if (k[i] != 0xFFFFFFFFu) atomicAdd(&hist[(k[i] >> shift) & mask], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d <= (int)mask; d += kRadixThreads) counts[(int64_t)d * ntiles + t] = hist[d];
}

constexpr int kRadixStreams = 4;                                  // independent rank chains per warp
constexpr int kRadixStreamLen = kRadixSub / kRadixStreams;        // 128 elements each

__global__ void __launch_bounds__(kRadixThreads, 3) radix_downsweep(
    const uint32_t* __restrict__ keys_in, const int32_t* __restrict__ vals_in, uint32_t* __restrict__ keys_out,
    int32_t* __restrict__ vals_out, int64_t n, int shift, int dbits, int64_t ntiles,
    const uint32_t* __restrict__ offsets) {
  extern __shared__ __align__(16) uint8_t radix_smem[];
  // [warp * streams + stream][digit] counts -> exclusive prefix in element order
  uint16_t* wcnt = reinterpret_cast<uint16_t*>(radix_smem);
  uint32_t* skeys = reinterpret_cast<uint32_t*>(wcnt + kRadixWarps * kRadixStreams * kRadixBins);
  int32_t* svals = reinterpret_cast<int32_t*>(skeys + kRadixTile);
  uint32_t* dstart = reinterpret_cast<uint32_t*>(svals + kRadixTile);  // tile-local start of each digit
  uint32_t* goff = dstart + kRadixBins;                                 // global start of (digit, tile)
  uint32_t* wsum = goff + kRadixBins;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t mask = (1u << dbits) - 1u;
  const int64_t t = blockIdx.x;
  const int64_t base = t * kRadixTile;
  const int64_t wbase = base + warp * kRadixSub;
  {
    uint4* z = reinterpret_cast<uint4*>(wcnt);
    constexpr int nz = kRadixWarps * kRadixStreams * kRadixBins * 2 / 16;
    for (int i = threadIdx.x; i < nz; i += kRadixThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  for (int d = threadIdx.x; d < kRadixBins; d += kRadixThreads)
    goff[d] = d <= (int)mask ? offsets[(int64_t)d * ntiles + t] : 0u;
  // item i = stream (i % S), step (i / S): element wbase + stream * 128 + step * 32 + lane
  uint32_t k[kRadixItems];
  int32_t v[kRadixItems];
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    const int64_t idx = wbase + (i % kRadixStreams) * kRadixStreamLen + (i / kRadixStreams) * 32 + lane;
    const bool ok = idx < n;
    k[i] = ok ? __ldg(keys_in + idx) : 0xFFFFFFFFu;
    v[i] = ok ? __ldg(vals_in + idx) : 0;
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
  uint16_t r[kRadixItems];
  uint16_t* myc = wcnt + warp * kRadixStreams * kRadixBins;
#pragma unroll
  for (int step = 0; step < kRadixItems / kRadixStreams; ++step) {
    uint32_t d[kRadixStreams], m[kRadixStreams], before[kRadixStreams];
    bool ok[kRadixStreams];
#pragma unroll
    for (int q = 0; q < kRadixStreams; ++q) {  // S independent chains: their latencies overlap
      const int i = step * kRadixStreams + q;
      ok[q] = k[i] != 0xFFFFFFFFu;
      d[q] = ok[q] ? (k[i] >> shift) & mask : (uint32_t)kRadixBins - 1u;
      m[q] = __match_any_sync(0xffffffffu, d[q]) & __ballot_sync(0xffffffffu, ok[q]);
      before[q] = myc[q * kRadixBins + d[q]];
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kRadixStreams; ++q) {
      const int i = step * kRadixStreams + q;
      if (ok[q]) {
        r[i] = (uint16_t)(before[q] + __popc(m[q] & lt));
        if ((m[q] & lt) == 0) myc[q * kRadixBins + d[q]] = (uint16_t)(before[q] + __popc(m[q]));
      }
    }
    __syncwarp();
  }
  __syncthreads();
  // per digit: exclusive prefix over (warp, stream) -- element order
  for (int d = threadIdx.x; d < kRadixBins; d += kRadixThreads) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps * kRadixStreams; ++w) {
      const uint32_t c = wcnt[w * kRadixBins + d];
      wcnt[w * kRadixBins + d] = (uint16_t)run;
      run += c;
    }
    dstart[d] = run;  // tile histogram for now
  }
  __syncthreads();
  {  // exclusive scan of the tile histogram over digits (2 digits per thread)
    const int d0 = threadIdx.x * 2;
    const uint32_t a = dstart[d0], b = dstart[d0 + 1];
    uint32_t x = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < kRadixWarps; ++w)
      if (w < warp) wpre += wsum[w];
    const uint32_t excl = wpre + x - (a + b);
    __syncthreads();
    dstart[d0] = excl;
    dstart[d0 + 1] = excl + a;
  }
  __syncthreads();
  // reorder the tile by (digit, rank) in shared memory ...
#pragma unroll
  for (int i = 0; i < kRadixItems; ++i) {
    if (k[i] == 0xFFFFFFFFu) continue;
    const uint32_t d = (k[i] >> shift) & mask;
    const uint32_t pos = dstart[d] + myc[(i % kRadixStreams) * kRadixBins + d] + r[i];
    skeys[pos] = k[i];
    svals[pos] = v[i];
  }
  __syncthreads();
  // ... and store it so consecutive threads write consecutive slots of a run
  const int cnt = n - base < kRadixTile ? (int)(n - base) : kRadixTile;
  for (int i = threadIdx.x; i < cnt; i += kRadixThreads) {
    const uint32_t kk = skeys[i];
    const uint32_t d = (kk >> shift) & mask;
    const int64_t dst = (int64_t)goff[d] + (i - (int64_t)dstart[d]);
    keys_out[dst] = kk;
    vals_out[dst] = svals[i];
  }
}

constexpr size_t kRadixDownSmem = (size_t)kRadixWarps * kRadixStreams * kRadixBins * 2 + (size_t)kRadixTile * 8 +
                                  (size_t)kRadixBins * 8 + kRadixWarps * 4;

inline int64_t radix_tiles(int64_t n) { return (n + kRadixTile - 1) / kRadixTile; }

// Exclusive scan of the digit-major (digit, tile) counts: tile sums, then each
// block adds the sums of the tiles before it and scans its own 4096 counts
// (two launches; replaces the CUB DeviceScan of round 1).  The count arrays
// are multiples of kRadixBins long, so whole 16-byte vectors.
constexpr int kScanItems = 4;
constexpr int kScanTile = kRadixThreads * kScanItems;  // 1024

__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v, uint32_t* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  uint32_t t = 0;
  for (int i = 0; i < kRadixWarps; ++i) t += red[i];
  return t;
}

__global__ void __launch_bounds__(kRadixThreads) scan_u32_tile_sums(const uint32_t* __restrict__ in, int64_t n,
                                                                    uint32_t* __restrict__ sums) {
  __shared__ uint32_t red[kRadixWarps];
  const int64_t i0 = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t v = 0;
  if (i0 < n) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(in + i0));
    v = x.x + x.y + x.z + x.w;
  }
  v = block_sum_u32(v, red);
  if (threadIdx.x == 0) sums[blockIdx.x] = v;
}

__global__ void __launch_bounds__(kRadixThreads) scan_u32_tiles(const uint32_t* __restrict__ in, int64_t n,
                                                                const uint32_t* __restrict__ sums,
                                                                uint32_t* __restrict__ out) {
  __shared__ uint32_t red[kRadixWarps];
  __shared__ uint32_t wsum[kRadixWarps];
  uint32_t p = 0;
  for (int i = threadIdx.x; i < (int)blockIdx.x; i += kRadixThreads) p += __ldg(sums + i);
  const uint32_t prefix = block_sum_u32(p, red);
  // thread t scans items [t * 4, t * 4 + 4) of the tile
  const int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  uint32_t x[kScanItems] = {0u, 0u, 0u, 0u};
  if (base < n) {
    const uint4 q = __ldg(reinterpret_cast<const uint4*>(in + base));
    x[0] = q.x; x[1] = q.y; x[2] = q.z; x[3] = q.w;
  }
  uint32_t tsum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) tsum += x[i];
  // exclusive scan of the thread totals: warp inclusive scan + warp offsets
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  uint32_t inc = tsum;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (l >= o) inc += y;
  }
  if (l == 31) wsum[w] = inc;
  __syncthreads();
  uint32_t woff = 0;
  for (int i = 0; i < w; ++i) woff += wsum[i];
  uint32_t run = prefix + woff + inc - tsum;
  if (base < n) {
    uint4 o;
    o.x = run; run += x[0];
    o.y = run; run += x[1];
    o.z = run; run += x[2];
    o.w = run;
    *reinterpret_cast<uint4*>(out + base) = o;
  }
}

inline size_t radix_scan_bytes(int64_t n) {
  const int64_t items = radix_tiles(std::max<int64_t>(n, 1)) * kRadixBins;
  return sizeof(uint32_t) * (size_t)((items + kScanTile - 1) / kScanTile);
}

// Sorts n pairs by the low end_bit bits of the keys; the result lands in the
// `_out` buffers when radix_passes(end_bit) is odd, else back in `_in`.
inline int radix_sort_pairs(uint32_t* keys_in, int32_t* vals_in, uint32_t* keys_out, int32_t* vals_out, int64_t n,
                            int end_bit, uint32_t* counts, uint32_t* offsets, void* scan_tmp, size_t scan_bytes,
                            cudaStream_t s) {
  if (n <= 0) return DMT_OK;
  if (n >= (int64_t(1) << 31)) return DMT_ERR_UNSUPPORTED;
  const int np = radix_passes(end_bit), db = radix_digit_bits(end_bit);
  const uint32_t mask = (1u << db) - 1u;
  const int64_t nt = radix_tiles(n);
  const int items = (int)(nt * (mask + 1));
  uint32_t *ki = keys_in, *ko = keys_out;
  int32_t *vi = vals_in, *vo = vals_out;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(radix_downsweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRadixDownSmem) !=
        cudaSuccess)
      return DMT_ERR_CUDA;
    attr = true;
  }
  for (int pass = 0; pass < np; ++pass) {
    const int shift = pass * db;
    radix_upsweep<<<(unsigned)nt, kRadixThreads, 0, s>>>(ki, n, shift, mask, nt, counts);
    DMT_CHECK_LAUNCH();
    const unsigned st = (unsigned)((items + kScanTile - 1) / kScanTile);
    if (scan_bytes < st * sizeof(uint32_t)) return DMT_ERR_DOMAIN;
    scan_u32_tile_sums<<<st, kRadixThreads, 0, s>>>(counts, items, (uint32_t*)scan_tmp);
    scan_u32_tiles<<<st, kRadixThreads, 0, s>>>(counts, items, (const uint32_t*)scan_tmp, offsets);
    radix_downsweep<<<(unsigned)nt, kRadixThreads, kRadixDownSmem, s>>>(ki, vi, ko, vo, n, shift, db, nt, offsets);
    DMT_CHECK_LAUNCH();
    std::swap(ki, ko);
    std::swap(vi, vo);
  }
  return DMT_OK;
}

struct BwdLayout {
  size_t keys_in, keys_out, vals_in, vals_out, recs, cub_temp, total;
  size_t cub_bytes;
  size_t bcounts, boffs, bcursor, items, scratch;  // bucketed path
  size_t rcounts, roffs, rscan, rscan_bytes;      // radix path
  int bshift;
  int64_t nbuckets;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline int end_bit_for(uint64_t key_space) {
  int bits = 1;
  while (bits < 32 && (1ull << bits) <= key_space) ++bits;  // must represent key_space (= invalid)
  return bits;
}

inline BwdLayout bwd_layout(int64_t nnz, int64_t key_space, int64_t nbags) {
  BwdLayout L{};
  size_t n = (size_t)(nnz > 0 ? nnz : 1);
  size_t nb = (size_t)(nbags > 0 ? nbags : 1);
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0,
                                  end_bit_for((uint64_t)key_space));
  L.cub_bytes = sort_bytes;
  size_t off = 0;
  L.keys_in = off; off = align256(off + n * 4);
  L.keys_out = off; off = align256(off + n * 4);
  L.vals_in = off; off = align256(off + n * 4);
  L.vals_out = off; off = align256(off + n * 4);
  L.recs = off; off = align256(off + nb * sizeof(BagRec));
  L.cub_temp = off; off = align256(off + L.cub_bytes);
  L.bshift = bucket_shift((int64_t)n, key_space);
  L.nbuckets = bucket_count(key_space, L.bshift);
  const size_t nbk = (size_t)L.nbuckets;
  L.bcounts = off; off = align256(off + nbk * 4);
  L.boffs = off; off = align256(off + (nbk + 1) * 4);
  L.bcursor = off; off = align256(off + nbk * 4);
  L.items = off; off = align256(off + n * 8);
  L.scratch = off; off = align256(off + 2 * n * 8 + (size_t)kBktCap * 8);
  const size_t ritems = (size_t)radix_tiles((int64_t)n) * kRadixBins;
  L.rcounts = off; off = align256(off + ritems * 4);
  L.roffs = off; off = align256(off + ritems * 4);
  L.rscan_bytes = radix_scan_bytes((int64_t)n);
  L.rscan = off; off = align256(off + L.rscan_bytes);
  L.total = off;
  return L;
}

template <typename T>
int launch_bwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* hs, int32_t n, const int64_t* offsets,
               const int32_t* indices, int64_t nnz, int64_t key_space, int32_t opt, float lr, float eps,
               void* ws, size_t ws_bytes, cudaStream_t s, int phase) {
  // phase bit 1: keys + bag records + radix sort (needs only the indices);
  // phase bit 2: the fused reduce + optimizer update (needs the gradients)
  if (nnz <= 0 || n == 0) return DMT_OK;
  if ((uint64_t)key_space >= 0xFFFFFFFFull || nnz > 0x7FFFFFFF) return DMT_ERR_UNSUPPORTED;
  int max_b = 0, max_w = 0;
  int64_t nbags = 0;
  for (int i = 0; i < n; ++i) {
    if (hs[i].nbags > max_b) max_b = hs[i].nbags;
    if (hs[i].width > max_w) max_w = hs[i].width;
    // the segments must tile bags [0, nbags) contiguously (offsets[0] == 0)
    if (hs[i].bag_begin != nbags) return DMT_ERR_PROTOCOL;
    nbags += hs[i].nbags;
    if (opt == DMT_OPT_ROWWISE_ADAGRAD && !hs[i].state) return DMT_ERR_DOMAIN;
    if (hs[i].ld > 65535 || hs[i].width > 65535) return DMT_ERR_UNSUPPORTED;
  }
  if (max_b == 0) return DMT_OK;
  // apply variants (DMT_BWD_VARIANT, read once so prepare and apply agree):
  // 7 (default) register kernel over a CUB radix sort, one occurrence per
  // group, the second row of a duplicate run prefetched (PF2), 2 CTAs / SM;
  // 5 / 6 the same at 4 / 3 CTAs / SM; 2 without PF2 (4 CTAs / SM); 1 its
  // two-occurrence form; 4 the bulk-copy staged kernel; 0 the bucketed sort + apply (hand-written bucket scatter, shared-
  // memory bitonic sort per bucket fused with the update) -- all
  // parity-tested.  The bucketed form measured slower at C2 bf16 (apply 0.83
  // vs 0.61 ms; its prepare's bucket-counter atomics 0.19 + 0.14 ms vs the CUB
  // sort), so it is not the default.
  static const int bwd_variant = [] {
    const char* e = getenv("DMT_BWD_VARIANT");
    return e ? atoi(e) : 7;
  }();
  // fast path: no mean pooling, 16-byte aligned gradient rows inside one
  // buffer (offset < 32 GB), <= kMaxShards distinct shards, vector widths
  constexpr int VEC0 = Vec16<T>::N;
  const char* gbase = nullptr;
  ShardTab tab;
  tab.n = 0;
  bool fast = true;
  for (int i = 0; i < n && fast; ++i) {
    const dmt_lookup_segment& g = hs[i];
    if (g.pooling == DMT_POOL_MEAN || (g.out_ld * (int64_t)sizeof(T)) % 16 || ((uintptr_t)g.out & 15) ||
        g.width % VEC0 || g.ld % VEC0 || ((uintptr_t)g.weights & 15))
      fast = false;
    if (!gbase || (const char*)g.out < gbase) gbase = (const char*)g.out;
  }
  if (fast) {
    for (int i = 0; i < n && fast; ++i) {
      const dmt_lookup_segment& g = hs[i];
      const int64_t span = ((const char*)g.out - gbase) + (int64_t)g.nbags * g.out_ld * (int64_t)sizeof(T);
      if (span >= (int64_t(1) << 35)) fast = false;
      bool seen = false;
      for (int j = 0; j < tab.n; ++j)
        if (tab.key_base[j] == (uint32_t)g.key_base) seen = true;
      if (!seen) {
        if (tab.n == kMaxShards) { fast = false; break; }
        int j = tab.n++;
        tab.key_base[j] = (uint32_t)g.key_base;
        tab.ld[j] = (uint16_t)g.ld;
        tab.width[j] = (uint16_t)g.width;
        tab.weights[j] = (const char*)g.weights;
        tab.state[j] = (float*)g.state;
      }
    }
    // sort the shard table by key base (insertion sort; tiny)
    for (int i = 1; i < tab.n; ++i)
      for (int j = i; j > 0 && tab.key_base[j - 1] > tab.key_base[j]; --j) {
        std::swap(tab.key_base[j - 1], tab.key_base[j]);
        std::swap(tab.ld[j - 1], tab.ld[j]);
        std::swap(tab.width[j - 1], tab.width[j]);
        std::swap(tab.weights[j - 1], tab.weights[j]);
        std::swap(tab.state[j - 1], tab.state[j]);
      }
  }
  BwdLayout L = bwd_layout(nnz, key_space, nbags);
  if (ws_bytes < L.total) return DMT_ERR_DOMAIN;
  char* w = (char*)ws;
  uint32_t* keys_in = (uint32_t*)(w + L.keys_in);
  uint32_t* keys_out = (uint32_t*)(w + L.keys_out);
  int32_t* vals_in = (int32_t*)(w + L.vals_in);
  int32_t* vals_out = (int32_t*)(w + L.vals_out);
  BagRec* recs = (BagRec*)(w + L.recs);
  const uint32_t invalid = (uint32_t)key_space;

  // sort of the prepare (DMT_BWD_SORT): 0 (default) the hand-written radix
  // sort above (3 passes of 9 / 8 / 8 bits at C2), 1 CUB onesweep (4 passes)
  static const int bwd_sort = [] {
    const char* e = getenv("DMT_BWD_SORT");
    return e && std::string(e) == "cub" ? 1 : 0;
  }();
  const int end_bit = end_bit_for((uint64_t)key_space);
  // where the sorted pairs land: CUB and odd radix pass counts -> `_out`
  const bool sorted_in_out = bwd_sort == 1 || (radix_passes(end_bit) & 1);
  const uint32_t* skeys = sorted_in_out ? keys_out : keys_in;
  const int32_t* svals = sorted_in_out ? vals_out : vals_in;
  const bool bucketed = fast && bwd_variant == 0;
  uint32_t* bcounts = (uint32_t*)(w + L.bcounts);
  uint32_t* boffs = (uint32_t*)(w + L.boffs);
  uint32_t* bcursor = (uint32_t*)(w + L.bcursor);
  uint64_t* items = (uint64_t*)(w + L.items);
  uint64_t* scratch = (uint64_t*)(w + L.scratch);
  if (phase & 1) {
    const unsigned fg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nnz, 256), DMT_NUM_SMS * 8));
    fill_u32_kernel<<<fg, 256, 0, s>>>(keys_in, nnz, invalid);
    DMT_CHECK_LAUNCH();
  }
  if ((phase & 1) && bucketed) {
    if (cudaMemsetAsync(bcounts, 0, (size_t)L.nbuckets * 4, s) != cudaSuccess) return DMT_ERR_CUDA;
    dim3 kg((unsigned)ceil_div((int64_t)max_b * 8, 256), n);
    bwd_bucket_keys_kernel<<<kg, 256, 0, s>>>(segs, offsets, indices, invalid, keys_in, vals_in, gbase,
                                              (int)sizeof(T), L.bshift, bcounts);
    DMT_CHECK_LAUNCH();
    bucket_scan_kernel<<<1, 1024, 0, s>>>(bcounts, L.nbuckets, boffs, bcursor);
    DMT_CHECK_LAUNCH();
    const unsigned sg = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nnz, 256), DMT_NUM_SMS * 8));
    bwd_bucket_scatter_kernel<<<sg, 256, 0, s>>>(keys_in, vals_in, nnz, invalid, L.bshift, bcursor, items);
    DMT_CHECK_LAUNCH();
  } else if (phase & 1) {
    dim3 kg((unsigned)ceil_div((int64_t)max_b * 8, 256), n);
    if (fast)
      bwd_keys_fast_kernel<<<kg, 256, 0, s>>>(segs, offsets, indices, invalid, keys_in, vals_in, gbase,
                                              (int)sizeof(T));
    else
      bwd_keys_kernel<<<kg, 256, 0, s>>>(segs, offsets, indices, invalid, keys_in, vals_in, recs, (int)sizeof(T));
    DMT_CHECK_LAUNCH();
    if (bwd_sort == 1) {
      size_t cub_bytes = L.cub_bytes;
      if (cub::DeviceRadixSort::SortPairs((void*)(w + L.cub_temp), cub_bytes, keys_in, keys_out, vals_in, vals_out,
                                          (int)nnz, 0, end_bit, s) != cudaSuccess)
        return DMT_ERR_CUDA;
    } else {
      const int rc = radix_sort_pairs(keys_in, vals_in, keys_out, vals_out, nnz, end_bit, (uint32_t*)(w + L.rcounts),
                                      (uint32_t*)(w + L.roffs), (void*)(w + L.rscan), L.rscan_bytes, s);
      if (rc != DMT_OK) return rc;
    }
  }
  if (!(phase & 2)) return DMT_OK;
  constexpr int VEC = Vec16<T>::N;
  if (bucketed) {
    const int nvec = (max_w + VEC0 - 1) / VEC0;
    int G = 1, log2g = 0;
    while (G * 2 < nvec && G < 32) { G <<= 1; ++log2g; }
    const int nv = (nvec + G - 1) / G;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(L.nbuckets, (int64_t)DMT_NUM_SMS * 4));
    if (nv == 1)
      bwd_bucket_apply_kernel<T, VEC0, 1><<<grid, kBktThreads, 0, s>>>(items, boffs, L.nbuckets, scratch, gbase,
                                                                       tab, log2g, opt, lr, eps);
    else if (nv == 2)
      bwd_bucket_apply_kernel<T, VEC0, 2><<<grid, kBktThreads, 0, s>>>(items, boffs, L.nbuckets, scratch, gbase,
                                                                       tab, log2g, opt, lr, eps);
    else if (nv <= 4)
      bwd_bucket_apply_kernel<T, VEC0, 4><<<grid, kBktThreads, 0, s>>>(items, boffs, L.nbuckets, scratch, gbase,
                                                                       tab, log2g, opt, lr, eps);
    else
      return DMT_ERR_UNSUPPORTED;
    DMT_CHECK_LAUNCH();
    return DMT_OK;
  }
  bool vec_ok = true;
  for (int i = 0; i < n; ++i) {
    const dmt_lookup_segment& g = hs[i];
    if (g.width % VEC || g.ld % VEC || g.out_ld % VEC || ((uintptr_t)g.weights & 15) || ((uintptr_t)g.out & 15))
      vec_ok = false;
  }
  auto grid_for = [&](int log2g) {
    const int gpb = kLookupThreads >> log2g;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ceil_div(nnz, 4), gpb), (int64_t)DMT_NUM_SMS * 12));
  };
  const int nvec_all = (max_w + VEC - 1) / VEC;
  // 4/8-byte rows: bulk-copy (TMA) staged kernel; 16-bit rows keep the
  // register-resident kernel below (measured faster for bf16 at C2)
  // tuning knob for the 16-bit apply: 0 (default) register kernel, one
  // occurrence per thread group at 4 CTAs / SM; 1 the earlier two-occurrence
  // form; 4 the bulk-copy staged kernel (all three parity-tested)
  const bool async16 = sizeof(T) == 2 && bwd_variant == 4;
  if (fast && (sizeof(T) >= 4 || async16) && nvec_all * VEC == max_w &&
      (nvec_all == 8 || nvec_all == 16 || nvec_all == 32)) {
    bool uniform_w = true;
    for (int i = 0; i < n; ++i) uniform_w = uniform_w && hs[i].width == max_w;
    if (uniform_w) {
      int rc;
      if (nvec_all == 8)
        rc = launch_async_update<T, 8>(skeys, svals, nnz, gbase, tab, invalid, opt, lr, eps, s);
      else if (nvec_all == 16)
        rc = launch_async_update<T, 16>(skeys, svals, nnz, gbase, tab, invalid, opt, lr, eps, s);
      else
        rc = launch_async_update<T, 32>(skeys, svals, nnz, gbase, tab, invalid, opt, lr, eps, s);
      if (rc != DMT_OK) return rc;
      DMT_CHECK_LAUNCH();
      return DMT_OK;
    }
  }
  if (fast) {
    // G threads per row with two 16-byte vectors each (NV = 2): twice the rows
    // per warp of the one-vector layout at the same register cost
    const int nvec = (max_w + VEC - 1) / VEC;
    int G = 1, log2g = 0;
    while (G * 2 < nvec && G < 32) { G <<= 1; ++log2g; }
    const int nv = (nvec + G - 1) / G;
    if (nv == 1)
      bwd_update_fast_kernel<T, VEC, 1, 4><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, gbase, tab, invalid, log2g, opt, lr, eps);
    else if (nv == 2 && bwd_variant == 1)  // two occurrences per group, 2 CTAs / SM
      bwd_update_fast_kernel<T, VEC, 2, 2><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, gbase, tab, invalid, log2g, opt, lr, eps);
    else if (nv == 2 && bwd_variant == 2)  // one occurrence per group, 4 CTAs / SM
      bwd_update_fast_kernel<T, VEC, 2, 1, 4><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, gbase, tab, invalid, log2g, opt, lr, eps);
    else if (nv == 2 && bwd_variant == 5)
      bwd_update_fast_kernel<T, VEC, 2, 1, 4, true><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, gbase, tab, invalid, log2g, opt, lr, eps);
    else if (nv == 2 && bwd_variant == 6)
      bwd_update_fast_kernel<T, VEC, 2, 1, 3, true><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, gbase, tab, invalid, log2g, opt, lr, eps);
    else if (nv == 2)  // default: PF2, 2 CTAs / SM.  bf16 C2 apply (tools/lookup_bench.py): 580 us
      // (variant 2, shard binary search) -> 509 (bucketed shard table) -> 505 us (+ PF2)
      bwd_update_fast_kernel<T, VEC, 2, 1, 2, true><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, gbase, tab, invalid, log2g, opt, lr, eps);
    else if (nv <= 4)
      bwd_update_fast_kernel<T, VEC, 4, 1><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, gbase, tab, invalid, log2g, opt, lr, eps);
    else
      return DMT_ERR_UNSUPPORTED;
  } else if (vec_ok) {
    const int nvec = (max_w + VEC - 1) / VEC;
    int G = 1, log2g = 0;
    while (G < nvec && G < 32) { G <<= 1; ++log2g; }
    const int nv = (nvec + G - 1) / G;
    if (nv == 1)
      bwd_update_kernel<T, VEC, 1, 4><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, recs, invalid, log2g, opt, lr, eps);
    else if (nv == 2)
      bwd_update_kernel<T, VEC, 2, 2><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, recs, invalid, log2g, opt, lr, eps);
    else if (nv <= 4)
      bwd_update_kernel<T, VEC, 4, 1><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, recs, invalid, log2g, opt, lr, eps);
    else
      return DMT_ERR_UNSUPPORTED;
  } else {
    if (max_w > 32 * 8) return DMT_ERR_UNSUPPORTED;
    int G = 1, log2g = 0;
    while (G < max_w && G < 32) { G <<= 1; ++log2g; }
    const int nv = (max_w + G - 1) / G;
    if (nv == 1)
      bwd_update_kernel<T, 1, 1, 4><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, recs, invalid, log2g, opt, lr, eps);
    else if (nv <= 4)
      bwd_update_kernel<T, 1, 4, 1><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, recs, invalid, log2g, opt, lr, eps);
    else
      bwd_update_kernel<T, 1, 8, 1><<<grid_for(log2g), kLookupThreads, 0, s>>>(
          skeys, svals, nnz, recs, invalid, log2g, opt, lr, eps);
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

}  // namespace dmt

extern "C" {

int dmt_pooled_lookup_fwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host, int32_t num_segs,
                          const int64_t* offsets, const int32_t* indices, int32_t dtype, int32_t* err,
                          dmt_stream_t stream) {
  if (num_segs < 0) return DMT_ERR_DOMAIN;
  if (num_segs == 0) return DMT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32: return dmt::launch_fwd<float>(segs, segs_host, num_segs, offsets, indices, err, s);
    case DMT_BF16: return dmt::launch_fwd<__nv_bfloat16>(segs, segs_host, num_segs, offsets, indices, err, s);
    case DMT_F64: return dmt::launch_fwd<double>(segs, segs_host, num_segs, offsets, indices, err, s);
    case DMT_F16: return dmt::launch_fwd<__half>(segs, segs_host, num_segs, offsets, indices, err, s);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

size_t dmt_pooled_lookup_bwd_workspace_size(int64_t nnz, int64_t key_space, int64_t num_bags) {
  return dmt::bwd_layout(nnz, key_space, num_bags).total;
}

static int bwd_dispatch(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host, int32_t num_segs,
                        const int64_t* offsets, const int32_t* indices, int64_t nnz, int64_t key_space,
                        int32_t dtype, int32_t optimizer, float lr, float eps, void* workspace,
                        size_t workspace_bytes, dmt_stream_t stream, int phase) {
  if (num_segs < 0 || nnz < 0) return DMT_ERR_DOMAIN;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32:
      return dmt::launch_bwd<float>(segs, segs_host, num_segs, offsets, indices, nnz, key_space, optimizer, lr,
                                    eps, workspace, workspace_bytes, s, phase);
    case DMT_BF16:
      return dmt::launch_bwd<__nv_bfloat16>(segs, segs_host, num_segs, offsets, indices, nnz, key_space,
                                            optimizer, lr, eps, workspace, workspace_bytes, s, phase);
    case DMT_F64:
      return dmt::launch_bwd<double>(segs, segs_host, num_segs, offsets, indices, nnz, key_space, optimizer, lr,
                                     eps, workspace, workspace_bytes, s, phase);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

int dmt_pooled_lookup_bwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host, int32_t num_segs,
                          const int64_t* offsets, const int32_t* indices, int64_t nnz, int64_t key_space,
                          int32_t dtype, int32_t optimizer, float lr, float eps, void* workspace,
                          size_t workspace_bytes, dmt_stream_t stream) {
  return bwd_dispatch(segs, segs_host, num_segs, offsets, indices, nnz, key_space, dtype, optimizer, lr, eps,
                      workspace, workspace_bytes, stream, 3);
}

int dmt_pooled_lookup_bwd_prepare(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host,
                                  int32_t num_segs, const int64_t* offsets, const int32_t* indices, int64_t nnz,
                                  int64_t key_space, int32_t dtype, void* workspace, size_t workspace_bytes,
                                  dmt_stream_t stream) {
  return bwd_dispatch(segs, segs_host, num_segs, offsets, indices, nnz, key_space, dtype, DMT_OPT_SGD, 0.f, 0.f,
                      workspace, workspace_bytes, stream, 1);
}

int dmt_pooled_lookup_bwd_apply(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host,
                                int32_t num_segs, int64_t nnz, int64_t key_space, int32_t dtype, int32_t optimizer,
                                float lr, float eps, void* workspace, size_t workspace_bytes, dmt_stream_t stream) {
  return bwd_dispatch(segs, segs_host, num_segs, nullptr, nullptr, nnz, key_space, dtype, optimizer, lr, eps,
                      workspace, workspace_bytes, stream, 2);
}

}  // extern "C"
