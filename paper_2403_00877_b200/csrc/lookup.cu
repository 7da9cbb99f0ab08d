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
constexpr int kUnroll = 8;

// G threads per bag (power of two <= 32), NV vectors of VEC elements per thread.
template <typename T, int VEC, int NV>
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
  for (int64_t k0 = beg; k0 < end; k0 += kUnroll) {
    Frag<T, VEC> fr[kUnroll][NV];
    bool use[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      use[u] = false;
      if (k0 + u < end) {
        int64_t r = (int64_t)__ldg(indices + k0 + u) - row_begin;
        bool in = r >= 0 && r < rows;
        if (!in && !filt) bad = 1;
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
    for (int u = 0; u < kUnroll; ++u)
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
      int64_t r = (int64_t)__ldg(indices + k) - sg.row_begin;
      if (r < 0 || r >= sg.rows) {
        if (!sg.row_filter) bad = 1;
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
    if (NV == 1)
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
// Backward: key build -> stable radix sort -> run-length encode -> per-row
// reduction in sorted (= original occurrence) order -> fused optimizer.
// ----------------------------------------------------------------------------
constexpr uint32_t kInvalidKeyOffset = 0;  // invalid key = key_space

__device__ __forceinline__ int find_seg(const dmt_lookup_segment* __restrict__ segs, int n, int64_t gb) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {  // last seg with bag_begin <= gb
    int mid = (lo + hi + 1) >> 1;
    if (segs[mid].bag_begin <= gb) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// One thread per bag of one segment: emits (key, bag) for each occurrence.
__global__ void bwd_keys_kernel(const dmt_lookup_segment* __restrict__ segs, const int64_t* __restrict__ offsets,
                                const int32_t* __restrict__ indices, int64_t base_off, uint32_t invalid,
                                uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const dmt_lookup_segment& sg = segs[blockIdx.y];
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= sg.nbags) return;
  int64_t gb = sg.bag_begin + b;
  int64_t beg = offsets[gb], end = offsets[gb + 1];
  for (int64_t k = beg; k < end; ++k) {
    int64_t r = (int64_t)indices[k] - sg.row_begin;
    bool in = r >= 0 && r < sg.rows;
    keys[k - base_off] = in ? (uint32_t)(sg.key_base + r) : invalid;
    vals[k - base_off] = (int32_t)gb;
  }
}

template <typename T, int VEC>
__global__ void __launch_bounds__(kLookupThreads)
bwd_update_kernel(const dmt_lookup_segment* __restrict__ segs, int nsegs, const int64_t* __restrict__ offsets,
                  const uint32_t* __restrict__ ukeys, const int64_t* __restrict__ run_off,
                  const int32_t* __restrict__ num_runs_p, const int32_t* __restrict__ sorted_bags,
                  uint32_t invalid, int log2g, int nv, int opt, float lr, float eps) {
  using A = typename Acc<T>::type;
  const int G = 1 << log2g;
  const int gid = threadIdx.x >> log2g, t = threadIdx.x & (G - 1);
  const int groups_per_block = kLookupThreads >> log2g;
  const int num_runs = *num_runs_p;
  // warp-uniform trip count: every lane of a warp runs the same iterations so
  // the Adagrad shuffles below never diverge.
  for (int64_t base = (int64_t)blockIdx.x * groups_per_block; base < num_runs;
       base += (int64_t)gridDim.x * groups_per_block) {
    const int64_t run = base + gid;
    bool valid = run < num_runs;
    uint32_t key = valid ? ukeys[run] : invalid;
    valid = valid && key != invalid;
    int64_t r0 = 0, r1 = 0, row = 0;
    const dmt_lookup_segment* s0 = segs;
    if (valid) {
      r0 = run_off[run];
      r1 = run_off[run + 1];
      s0 = &segs[find_seg(segs, nsegs, sorted_bags[r0])];
      row = (int64_t)key - s0->key_base;
    }
    T* __restrict__ W = const_cast<T*>(reinterpret_cast<const T*>(s0->weights)) + row * s0->ld;
    const int width = valid ? s0->width : 0;
    for (int vbase = 0; vbase < nv; vbase += 4) {
      A acc[4][VEC];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[q][e] = A(0);
      for (int64_t i = r0; i < r1; ++i) {
        int64_t gb = sorted_bags[i];
        const dmt_lookup_segment& sg = segs[find_seg(segs, nsegs, gb)];
        const T* gp = reinterpret_cast<const T*>(sg.out) + (gb - sg.bag_begin) * sg.out_ld;
        A scale = A(1);
        if (sg.pooling == DMT_POOL_MEAN) scale = A(1) / (A)(offsets[gb + 1] - offsets[gb]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int c = ((vbase + q) * G + t) * VEC;
          if (vbase + q < nv && c < width) {
            A v[VEC];
            Loader<T, VEC>::load(gp + c, v);
#pragma unroll
            for (int e = 0; e < VEC; ++e) acc[q][e] += scale * v[e];
          }
        }
      }
      if (opt == DMT_OPT_SGD) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int c = ((vbase + q) * G + t) * VEC;
          if (vbase + q < nv && c < width) {
            A w[VEC];
            Loader<T, VEC>::load(W + c, w);
#pragma unroll
            for (int e = 0; e < VEC; ++e) w[e] = w[e] - (A)lr * acc[q][e];
            Loader<T, VEC>::store(W + c, w);
          }
        }
      } else {
        // row-wise Adagrad needs mean(g^2) over the whole row: single pass
        // (host guarantees nv <= 4 for Adagrad).
        float sq = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          int c = ((vbase + q) * G + t) * VEC;
          if (vbase + q < nv && c < width)
#pragma unroll
            for (int e = 0; e < VEC; ++e) sq += (float)(acc[q][e] * acc[q][e]);
        }
        for (int o = G >> 1; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o, G);
        if (valid) {
          float* st = reinterpret_cast<float*>(s0->state) + row;
          float s_new = *st + sq / (float)width;
          float denom = sqrtf(s_new) + eps;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            int c = ((vbase + q) * G + t) * VEC;
            if (vbase + q < nv && c < width) {
              A w[VEC];
              Loader<T, VEC>::load(W + c, w);
#pragma unroll
              for (int e = 0; e < VEC; ++e) w[e] = w[e] - (A)(lr / denom) * acc[q][e];
              Loader<T, VEC>::store(W + c, w);
            }
          }
          __syncwarp((G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (threadIdx.x & 31 & ~(G - 1))));
          if (t == 0) *st = s_new;
        }
      }
    }
  }
}

struct BwdLayout {
  size_t keys_in, keys_out, vals_in, vals_out, ukeys, counts, nruns, run_off, scan, cub_temp, total;
  size_t cub_bytes;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline int end_bit_for(uint64_t key_space) {
  int bits = 1;
  while (bits < 32 && (1ull << bits) <= key_space) ++bits;  // need to represent key_space (invalid)
  return bits;
}

inline BwdLayout bwd_layout(int64_t nnz, int64_t key_space) {
  BwdLayout L{};
  size_t n = (size_t)(nnz > 0 ? nnz : 1);
  size_t sort_bytes = 0, rle_bytes = 0;
  cub::DeviceRadixSort::SortPairs((void*)nullptr, sort_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0,
                                  end_bit_for((uint64_t)key_space));
  cub::DeviceRunLengthEncode::Encode((void*)nullptr, rle_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                     (int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  L.cub_bytes = sort_bytes > rle_bytes ? sort_bytes : rle_bytes;
  size_t off = 0;
  L.keys_in = off; off = align256(off + n * 4);
  L.keys_out = off; off = align256(off + n * 4);
  L.vals_in = off; off = align256(off + n * 4);
  L.vals_out = off; off = align256(off + n * 4);
  L.ukeys = off; off = align256(off + n * 4);
  L.counts = off; off = align256(off + n * 4);
  L.nruns = off; off = align256(off + 16);
  L.run_off = off; off = align256(off + (n + 1) * 8);
  L.scan = off; off = align256(off + dmt_lengths_to_offsets_workspace_size((int64_t)n));
  L.cub_temp = off; off = align256(off + L.cub_bytes);
  L.total = off;
  return L;
}

template <typename T>
int launch_bwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* hs, int32_t n, const int64_t* offsets,
               const int32_t* indices, int64_t nnz, int64_t key_space, int32_t opt, float lr, float eps,
               void* ws, size_t ws_bytes, cudaStream_t s) {
  if (nnz <= 0) return DMT_OK;
  if ((uint64_t)key_space >= 0xFFFFFFFFull || nnz > 0x7FFFFFFF) return DMT_ERR_UNSUPPORTED;
  BwdLayout L = bwd_layout(nnz, key_space);
  if (ws_bytes < L.total) return DMT_ERR_DOMAIN;
  char* w = (char*)ws;
  uint32_t* keys_in = (uint32_t*)(w + L.keys_in);
  uint32_t* keys_out = (uint32_t*)(w + L.keys_out);
  int32_t* vals_in = (int32_t*)(w + L.vals_in);
  int32_t* vals_out = (int32_t*)(w + L.vals_out);
  uint32_t* ukeys = (uint32_t*)(w + L.ukeys);
  int32_t* counts = (int32_t*)(w + L.counts);
  int32_t* nruns = (int32_t*)(w + L.nruns);
  int64_t* run_off = (int64_t*)(w + L.run_off);
  void* scan_ws = (void*)(w + L.scan);
  void* cub_ws = (void*)(w + L.cub_temp);
  const uint32_t invalid = (uint32_t)key_space;

  // the segments must tile bags [first.bag_begin, ...) contiguously
  int max_b = 0, max_w = 0;
  for (int i = 0; i < n; ++i) {
    if (hs[i].nbags > max_b) max_b = hs[i].nbags;
    if (hs[i].width > max_w) max_w = hs[i].width;
    if (i > 0 && hs[i].bag_begin != hs[i - 1].bag_begin + hs[i - 1].nbags) return DMT_ERR_PROTOCOL;
  }
  if (max_b == 0 || n == 0) return DMT_OK;
  // base offset: offsets[first bag] -- read on device would need a sync; the
  // caller passes indices already based at the first bag's offset (= 0 in the
  // pipeline: segments cover the owner's whole received KJT).
  dim3 kg((unsigned)ceil_div(max_b, 256), n);
  bwd_keys_kernel<<<kg, 256, 0, s>>>(segs, offsets, indices, 0, invalid, keys_in, vals_in);
  DMT_CHECK_LAUNCH();
  size_t cub_bytes = L.cub_bytes;
  if (cub::DeviceRadixSort::SortPairs(cub_ws, cub_bytes, keys_in, keys_out, vals_in, vals_out, (int)nnz, 0,
                                      end_bit_for((uint64_t)key_space), s) != cudaSuccess)
    return DMT_ERR_CUDA;
  cub_bytes = L.cub_bytes;
  if (cub::DeviceRunLengthEncode::Encode(cub_ws, cub_bytes, keys_out, ukeys, counts, nruns, (int)nnz, s) !=
      cudaSuccess)
    return DMT_ERR_CUDA;
  // run offsets: exclusive scan of counts (n runs <= nnz; tail counts unused)
  int rc = dmt_lengths_to_offsets(counts, nnz, run_off, scan_ws, (dmt_stream_t)s);
  if (rc != DMT_OK) return rc;
  constexpr int VEC = Vec16<T>::N;
  bool vec_ok = true;
  for (int i = 0; i < n; ++i) {
    const dmt_lookup_segment& g = hs[i];
    if (g.width % VEC || g.ld % VEC || g.out_ld % VEC || ((uintptr_t)g.weights & 15) || ((uintptr_t)g.out & 15))
      vec_ok = false;
  }
  int grid = DMT_NUM_SMS * 8;
  if (vec_ok) {
    int nvec = (max_w + VEC - 1) / VEC;
    int G = 1, log2g = 0;
    while (G < nvec && G < 32) { G <<= 1; ++log2g; }
    int nv = (nvec + G - 1) / G;
    if (opt == DMT_OPT_ROWWISE_ADAGRAD && nv > 4) return DMT_ERR_UNSUPPORTED;
    bwd_update_kernel<T, VEC><<<grid, kLookupThreads, 0, s>>>(segs, n, offsets, ukeys, run_off, nruns, vals_out,
                                                              invalid, log2g, nv, opt, lr, eps);
  } else {
    int G = 1, log2g = 0;
    while (G < max_w && G < 32) { G <<= 1; ++log2g; }
    int nv = (max_w + G - 1) / G;
    if (opt == DMT_OPT_ROWWISE_ADAGRAD && nv > 4) return DMT_ERR_UNSUPPORTED;
    bwd_update_kernel<T, 1><<<grid, kLookupThreads, 0, s>>>(segs, n, offsets, ukeys, run_off, nruns, vals_out,
                                                            invalid, log2g, nv, opt, lr, eps);
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

size_t dmt_pooled_lookup_bwd_workspace_size(int64_t nnz, int64_t key_space, int32_t num_segs) {
  (void)num_segs;
  return dmt::bwd_layout(nnz, key_space).total;
}

int dmt_pooled_lookup_bwd(const dmt_lookup_segment* segs, const dmt_lookup_segment* segs_host, int32_t num_segs,
                          const int64_t* offsets, const int32_t* indices, int64_t nnz, int64_t key_space,
                          int32_t dtype, int32_t optimizer, float lr, float eps, void* workspace,
                          size_t workspace_bytes, dmt_stream_t stream) {
  if (num_segs < 0 || nnz < 0) return DMT_ERR_DOMAIN;
  cudaStream_t s = (cudaStream_t)stream;
  switch (dtype) {
    case DMT_F32:
      return dmt::launch_bwd<float>(segs, segs_host, num_segs, offsets, indices, nnz, key_space, optimizer, lr,
                                    eps, workspace, workspace_bytes, s);
    case DMT_BF16:
      return dmt::launch_bwd<__nv_bfloat16>(segs, segs_host, num_segs, offsets, indices, nnz, key_space,
                                            optimizer, lr, eps, workspace, workspace_bytes, s);
    case DMT_F64:
      return dmt::launch_bwd<double>(segs, segs_host, num_segs, offsets, indices, nnz, key_space, optimizer, lr,
                                     eps, workspace, workspace_bytes, s);
    default: return DMT_ERR_UNSUPPORTED;
  }
}

}  // extern "C"
