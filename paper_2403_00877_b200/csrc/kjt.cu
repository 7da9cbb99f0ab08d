// KJT plumbing: lengths -> offsets scan and step-a bucketing.
//
// Reference: step a of _distribute_and_lookup ships, for every (src, owner),
// the full bag list of each shard the owner holds, bundled in shard-id order
// (towersim/exchange.py:162-178).  On the device that is a jagged gather of
// per-feature (lengths, values) segments into per-owner send slots; the
// all-to-all that follows is NCCL (or an in-process copy) on these buffers.
#include <dlfcn.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace dmt {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;  // per thread
constexpr int kScanTile = kScanThreads * kScanItems;

// Block-wide exclusive scan of per-thread sums (int64) via warp shuffles.
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    int64_t s = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) warp_sums[lane] = s;  // inclusive
  }
  __syncthreads();
  int64_t warp_prefix = warp ? warp_sums[warp - 1] : 0;
  if (total) *total = warp_sums[(blockDim.x >> 5) - 1];
  int64_t excl = warp_prefix + x - v;
  __syncthreads();
  return excl;
}

// Pass 1: per-tile sums.
__global__ void scan_tile_sums(const int32_t* __restrict__ len, int64_t n, int64_t* __restrict__ tile_sums) {
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += len[idx];
  }
  int64_t total;
  block_exclusive_scan(s, &total);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// Pass 2: exclusive scan of tile sums (single block, loops if many tiles).
__global__ void scan_tile_prefix(int64_t* __restrict__ tile_sums, int64_t ntiles) {
  int64_t carry = 0;
  for (int64_t base = 0; base < ntiles; base += kScanThreads) {
    int64_t idx = base + threadIdx.x;
    int64_t v = idx < ntiles ? tile_sums[idx] : 0;
    int64_t total;
    int64_t ex = block_exclusive_scan(v, &total);
    if (idx < ntiles) tile_sums[idx] = carry + ex;
    carry += total;
    __syncthreads();
  }
}

// Pass 3: each tile rescans its items with the tile prefix.  Thread t owns
// kScanItems consecutive items so the scan is a plain sequential prefix.
__global__ void scan_apply(const int32_t* __restrict__ len, int64_t n, const int64_t* __restrict__ tile_prefix,
                           int64_t* __restrict__ out) {
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  int32_t v[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + i;
    v[i] = idx < n ? len[idx] : 0;
    s += v[i];
  }
  int64_t ex = block_exclusive_scan(s, nullptr) + tile_prefix[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    int64_t idx = base + i;
    if (idx < n) out[idx] = ex;
    ex += v[i];
    if (idx == n - 1) out[n] = ex;
  }
}

__global__ void zero_one(int64_t* p) { p[0] = 0; }

// Bucketize: grid.y = slot, grid.x strides over the slot's lengths + values.
__global__ void bucketize_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ offsets,
                                 const int32_t* __restrict__ values, int32_t B,
                                 const int32_t* __restrict__ slot_feature,
                                 const int64_t* __restrict__ slot_off, int32_t* __restrict__ out_lengths,
                                 int32_t* __restrict__ out_values) {
  const int s = blockIdx.y;
  const int f = slot_feature[s];
  const int64_t vbeg = offsets[(int64_t)f * B];
  const int64_t vend = offsets[(int64_t)(f + 1) * B];
  const int64_t nnz = vend - vbeg;
  const int64_t dst = slot_off[s];
  // a slot whose values exceed its room (capacity-padded step a over its
  // capacity; dmt_kjt_check_capacity flags it) ships empty bags instead:
  // lengths and values stay consistent and no write leaves the slot
  const bool over = nnz > slot_off[s + 1] - dst;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += stride)
    out_lengths[(int64_t)s * B + i] = over ? 0 : lengths[(int64_t)f * B + i];
  if (over) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride)
    out_values[dst + i] = __ldg(values + vbeg + i);
}

__global__ void slot_offsets_kernel(const int64_t* __restrict__ offsets, int32_t B, int32_t num_slots,
                                    const int32_t* __restrict__ slot_feature, int64_t* __restrict__ out) {
  // single block; num_slots is small (shards per world)
  int64_t carry = 0;
  for (int base = 0; base < num_slots; base += blockDim.x) {
    int s = base + threadIdx.x;
    int64_t v = 0;
    if (s < num_slots) {
      int f = slot_feature[s];
      v = offsets[(int64_t)(f + 1) * B] - offsets[(int64_t)f * B];
    }
    int64_t total;
    int64_t ex = block_exclusive_scan(v, &total);
    if (s < num_slots) out[s] = carry + ex;
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[num_slots] = carry;
}

// Step a over NVLink peer stores: the same bundling, but every slot goes
// straight to its owner's receive buffers (per-slot destination pointers,
// IPC-mapped for remote owners) -- the all-to-alls of lengths and values
// become one barrier.  slot_room[s] bounds the slot's values (its fixed
// capacity); a slot over it ships empty bags like bucketize_kernel.
struct SlotDst {
  int32_t* len;
  int32_t* val;
  int64_t room;
};

__global__ void bucketize_peer_kernel(const int32_t* __restrict__ lengths, const int64_t* __restrict__ offsets,
                                      const int32_t* __restrict__ values, int32_t B,
                                      const int32_t* __restrict__ slot_feature, const SlotDst* __restrict__ dst) {
  const int s = blockIdx.y;
  const int f = slot_feature[s];
  const SlotDst d = dst[s];
  const int64_t vbeg = offsets[(int64_t)f * B];
  const int64_t nnz = offsets[(int64_t)(f + 1) * B] - vbeg;
  const bool over = nnz > d.room;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < B; i += stride)
    d.len[i] = over ? 0 : lengths[(int64_t)f * B + i];
  if (over) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += stride)
    d.val[i] = __ldg(values + vbeg + i);
}

// Capacity-padded step a (ragged batches under CUDA graphs): every slot of
// the send buffer has a fixed capacity, so the step-a splits are static and
// no count exchange / host sync is needed; the owner then packs each
// (src, shard) region's actual values (count from the packed offsets of the
// received lengths) back-to-back, which is the layout the lookup reads.
__global__ void kjt_compact_kernel(const int32_t* __restrict__ src, const int64_t* __restrict__ offsets, int32_t B,
                                   int32_t nseg, const int64_t* __restrict__ seg_src_start, int32_t* __restrict__ dst) {
  for (int seg = blockIdx.x; seg < nseg; seg += gridDim.x) {
    const int64_t b0 = (int64_t)seg * B;
    const int64_t beg = offsets[b0], cnt = offsets[b0 + B] - beg;
    const int32_t* s = src + seg_src_start[seg];
    int32_t* d = dst + beg;
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) d[i] = s[i];
  }
}

// flag |= 1 if any feature's nnz exceeds its slot capacity
__global__ void kjt_check_capacity_kernel(const int64_t* __restrict__ offsets, int32_t B, int32_t F,
                                          const int64_t* __restrict__ cap, int32_t* __restrict__ flag) {
  for (int f = blockIdx.x * blockDim.x + threadIdx.x; f < F; f += gridDim.x * blockDim.x)
    if (offsets[(int64_t)(f + 1) * B] - offsets[(int64_t)f * B] > cap[f]) atomicOr(flag, 1);
}

}  // namespace dmt

extern "C" {

int dmt_kjt_compact(const int32_t* src, const int64_t* offsets, int32_t B, int32_t num_segments,
                    const int64_t* seg_src_start, int32_t* dst, dmt_stream_t stream) {
  if (B < 0 || num_segments < 0) return DMT_ERR_DOMAIN;
  if (num_segments == 0 || B == 0) return DMT_OK;
  const unsigned grid = (unsigned)std::min<int64_t>(num_segments, (int64_t)DMT_NUM_SMS * 8);
  dmt::kjt_compact_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(src, offsets, B, num_segments, seg_src_start, dst);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_kjt_check_capacity(const int64_t* offsets, int32_t B, int32_t F, const int64_t* capacity, int32_t* flag,
                           dmt_stream_t stream) {
  if (B < 0 || F < 0) return DMT_ERR_DOMAIN;
  if (F == 0) return DMT_OK;
  dmt::kjt_check_capacity_kernel<<<(unsigned)dmt::ceil_div(F, 256), 256, 0, (cudaStream_t)stream>>>(offsets, B, F,
                                                                                                   capacity, flag);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

size_t dmt_lengths_to_offsets_workspace_size(int64_t n) {
  return sizeof(int64_t) * (size_t)(dmt::ceil_div(n, dmt::kScanTile) + 1);
}

int dmt_lengths_to_offsets(const int32_t* lengths, int64_t n, int64_t* offsets, void* scratch,
                           dmt_stream_t stream) {
  if (n < 0) return DMT_ERR_DOMAIN;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    dmt::zero_one<<<1, 1, 0, s>>>(offsets);
    DMT_CHECK_LAUNCH();
    return DMT_OK;
  }
  int64_t ntiles = dmt::ceil_div(n, dmt::kScanTile);
  int64_t* tiles = (int64_t*)scratch;
  dmt::scan_tile_sums<<<(unsigned)ntiles, dmt::kScanThreads, 0, s>>>(lengths, n, tiles);
  dmt::scan_tile_prefix<<<1, dmt::kScanThreads, 0, s>>>(tiles, ntiles);
  dmt::scan_apply<<<(unsigned)ntiles, dmt::kScanThreads, 0, s>>>(lengths, n, tiles, offsets);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_kjt_bucketize(const int32_t* lengths, const int64_t* offsets, const int32_t* values, int32_t B,
                      int32_t num_slots, const int32_t* slot_feature, const int64_t* slot_value_offset,
                      int32_t* out_lengths, int32_t* out_values, dmt_stream_t stream) {
  if (B < 0 || num_slots < 0) return DMT_ERR_DOMAIN;
  if (num_slots == 0 || B == 0) return DMT_OK;
  if (num_slots > 65535) return DMT_ERR_UNSUPPORTED;
  dim3 grid(64, num_slots);
  dmt::bucketize_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(lengths, offsets, values, B, slot_feature,
                                                                 slot_value_offset, out_lengths, out_values);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_kjt_bucketize_peer(const int32_t* lengths, const int64_t* offsets, const int32_t* values, int32_t B,
                           int32_t num_slots, const int32_t* slot_feature, const void* slot_dst,
                           dmt_stream_t stream) {
  if (B < 0 || num_slots < 0) return DMT_ERR_DOMAIN;
  if (num_slots == 0 || B == 0) return DMT_OK;
  if (num_slots > 65535) return DMT_ERR_UNSUPPORTED;
  dim3 grid(64, num_slots);
  dmt::bucketize_peer_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(lengths, offsets, values, B, slot_feature,
                                                                      (const dmt::SlotDst*)slot_dst);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

int dmt_kjt_slot_offsets(const int64_t* offsets, int32_t B, int32_t num_slots, const int32_t* slot_feature,
                         int64_t* slot_value_offset, dmt_stream_t stream) {
  if (num_slots < 0 || B < 0) return DMT_ERR_DOMAIN;
  dmt::slot_offsets_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(offsets, B, num_slots, slot_feature,
                                                                  slot_value_offset);
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

const char* dmt_version(void) { return "libdmt 0.1.0 sm_100a"; }

int dmt_enable_peer_access(int peer_device) {
  int cur = 0;
  if (cudaGetDevice(&cur) != cudaSuccess) return DMT_ERR_CUDA;
  if (peer_device == cur) return DMT_OK;
  int can = 0;
  if (cudaDeviceCanAccessPeer(&can, cur, peer_device) != cudaSuccess || !can) return DMT_ERR_UNSUPPORTED;
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free status
    return DMT_OK;
  }
  if (e != cudaSuccess) {
    dmt::set_last_error(e);
    return DMT_ERR_CUDA;
  }
  return DMT_OK;
}

// Allocation base of a device pointer through the driver API, resolved at run
// time so the library does not link libcuda (CPU-only hosts load it too).
static int alloc_base(const void* ptr, uintptr_t* base) {
  typedef int (*range_fn)(unsigned long long*, size_t*, unsigned long long);
  static range_fn fn = nullptr;
  if (!fn) {
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libcuda.so.1", RTLD_NOW);
    if (!h) return DMT_ERR_UNSUPPORTED;
    fn = (range_fn)dlsym(h, "cuMemGetAddressRange_v2");
    if (!fn) return DMT_ERR_UNSUPPORTED;
  }
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (unsigned long long)(uintptr_t)ptr) != 0) return DMT_ERR_DOMAIN;
  *base = (uintptr_t)b;
  return DMT_OK;
}

int dmt_ipc_export(const void* ptr, void* handle64, int64_t* offset) {
  if (!ptr || !handle64 || !offset) return DMT_ERR_DOMAIN;
  uintptr_t base = 0;
  int st = alloc_base(ptr, &base);
  if (st != DMT_OK) return st;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
  if (e != cudaSuccess) {
    dmt::set_last_error(e);
    return DMT_ERR_CUDA;
  }
  memcpy(handle64, &h, sizeof(h));
  *offset = (int64_t)((uintptr_t)ptr - base);
  return DMT_OK;
}

int dmt_ipc_open(const void* handle64, void** base) {
  if (!handle64 || !base) return DMT_ERR_DOMAIN;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    dmt::set_last_error(e);
    return DMT_ERR_CUDA;
  }
  return DMT_OK;
}

int dmt_ipc_close(void* base) {
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) {
    dmt::set_last_error(e);
    return DMT_ERR_CUDA;
  }
  return DMT_OK;
}

static thread_local char g_last_error[256] = "no error";

const char* dmt_last_error(void) { return g_last_error; }

}  // extern "C"

namespace dmt {
void set_last_error(cudaError_t e) {
  snprintf(g_last_error, sizeof(g_last_error), "%s (%d)", cudaGetErrorString(e), (int)e);
}
}  // namespace dmt

extern "C" {

}  // extern "C"
