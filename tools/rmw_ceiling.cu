// Ceiling probe for the embedding-backward apply's access pattern: U unique
// sorted random 256-byte rows of a 26M x 128 bf16 table, read-modify-write
// (plus an L2-resident "gradient" row per update).  Varies rows in flight per
// thread group (CH) and threads per row so the achievable random-row RMW
// bandwidth on this B200 bounds what the apply kernel can reach.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rmw_ceiling tools/rmw_ceiling.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int TPR, int CH, bool GRAD, bool WRITE>
__global__ void __launch_bounds__(256) rmw(uint4* __restrict__ W, const uint32_t* __restrict__ rows, int64_t U,
                                           const uint4* __restrict__ G, int gmask) {
  constexpr int NV = 16 / TPR;  // 16-byte vectors per thread (256 B rows)
  const int t = threadIdx.x % TPR;
  const int64_t grp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / TPR;
  const int64_t ngrp = (int64_t)gridDim.x * blockDim.x / TPR;
  for (int64_t base = grp * CH; base < U; base += ngrp * CH) {
    uint32_t r[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) r[c] = base + c < U ? __ldg(rows + base + c) : 0xFFFFFFFFu;
    uint4 w[CH][NV], g[CH][NV];
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (r[c] != 0xFFFFFFFFu) {
          w[c][v] = W[(int64_t)r[c] * 16 + v * TPR + t];
          if (GRAD) g[c][v] = __ldg(G + (int64_t)((base + c) & gmask) * 16 + v * TPR + t);
        }
#pragma unroll
    for (int c = 0; c < CH; ++c)
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (r[c] != 0xFFFFFFFFu) {
          uint4 x = w[c][v];
          if (GRAD) { x.x += g[c][v].x; x.y ^= g[c][v].y; x.z += g[c][v].z; x.w ^= g[c][v].w; }
          else x.x += 1;
          if (WRITE) W[(int64_t)r[c] * 16 + v * TPR + t] = x;
          else if (x.x == 0x12345678u) W[0] = x;
        }
  }
}

template <int TPR, int CH, bool GRAD, bool WRITE>
void run(const char* name, uint4* W, const uint32_t* rows, int64_t U, const uint4* G, int minb) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, rmw<TPR, CH, GRAD, WRITE>, 256, 0);
  for (int bps : {minb, nb}) {
    if (bps > nb || bps < 1) continue;
    int grid = 148 * bps;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) rmw<TPR, CH, GRAD, WRITE><<<grid, 256>>>(W, rows, U, G, (1 << 18) - 1);
    cudaEventRecord(a);
    const int n = 10;
    for (int i = 0; i < n; ++i) rmw<TPR, CH, GRAD, WRITE><<<grid, 256>>>(W, rows, U, G, (1 << 18) - 1);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= n;
    double bytes = (double)U * 256 * (WRITE ? 2 : 1);
    printf("%-28s TPR=%2d CH=%d blocks/SM=%d (max %d): %7.1f us  %6.0f GB/s (W bytes)\n", name, TPR, CH, bps, nb,
           ms * 1e3, bytes / ms / 1e6);
  }
}

int main() {
  const int64_t rows_total = 26000000, U = 3929004;
  std::vector<uint32_t> all(rows_total);
  for (int64_t i = 0; i < rows_total; ++i) all[i] = (uint32_t)i;
  std::mt19937_64 rng(1);
  for (int64_t i = 0; i < U; ++i) std::swap(all[i], all[i + rng() % (rows_total - i)]);
  std::vector<uint32_t> sel(all.begin(), all.begin() + U);
  std::sort(sel.begin(), sel.end());
  uint4 *W, *G;
  uint32_t* rows;
  cudaMalloc(&W, rows_total * 256);
  cudaMalloc(&G, (1 << 18) * 256);
  cudaMemset(W, 0, rows_total * 256);
  cudaMemset(G, 0, (1 << 18) * 256);
  cudaMalloc(&rows, U * 4);
  cudaMemcpy(rows, sel.data(), U * 4, cudaMemcpyHostToDevice);
  run<16, 1, false, false>("read only", W, rows, U, G, 4);
  run<16, 2, false, false>("read only", W, rows, U, G, 4);
  run<16, 1, false, true>("rmw", W, rows, U, G, 4);
  run<16, 2, false, true>("rmw", W, rows, U, G, 4);
  run<16, 4, false, true>("rmw", W, rows, U, G, 4);
  run<8, 1, false, true>("rmw", W, rows, U, G, 4);
  run<8, 2, false, true>("rmw", W, rows, U, G, 4);
  run<8, 4, false, true>("rmw", W, rows, U, G, 2);
  run<16, 1, true, true>("rmw + L2 grad", W, rows, U, G, 4);
  run<16, 2, true, true>("rmw + L2 grad", W, rows, U, G, 4);
  run<16, 4, true, true>("rmw + L2 grad", W, rows, U, G, 4);
  run<8, 1, true, true>("rmw + L2 grad", W, rows, U, G, 4);
  run<8, 2, true, true>("rmw + L2 grad", W, rows, U, G, 4);
  // unsorted order
  std::shuffle(sel.begin(), sel.end(), rng);
  cudaMemcpy(rows, sel.data(), U * 4, cudaMemcpyHostToDevice);
  run<16, 2, false, true>("rmw unsorted", W, rows, U, G, 4);
  run<16, 4, false, true>("rmw unsorted", W, rows, U, G, 4);
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
