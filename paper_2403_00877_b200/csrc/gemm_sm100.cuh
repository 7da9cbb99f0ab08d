#pragma once
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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>

#include "common.cuh"

namespace dmt {
namespace gemm {

constexpr int kEpiWarps = 8;   // two warps per TMEM lane quarter, each owns half the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kBlockM = 128;
constexpr int kAtomBytes = 128;  // one SWIZZLE_128B row = BLOCK_K bytes per stage
constexpr int kUmmaKBytes = 32;  // K bytes consumed by one tcgen05.mma (16 x bf16 / 8 x tf32)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
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

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// TMA load delivered to the same shared-memory offset of every CTA in
// ``mask`` (cluster multicast), completing tx bytes on each one's mbarrier.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int KIND>  // 0 = f16/bf16, 1 = tf32
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                     uint32_t accumulate) {
  if constexpr (KIND == 0) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
}

// cta_group::2: the leader CTA issues one MMA for the pair (M = 256: each CTA
// supplies 128 rows of A and half of B's columns from its own shared memory at
// the same offsets; each CTA's TMEM receives its own 128 accumulator rows)
__device__ __forceinline__ void umma2(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                      uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// completion of the pair's MMAs -> the barrier at this offset in every CTA of mask
__device__ __forceinline__ void umma2_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// shared::cluster address of the same shared variable in CTA ``rank``
__device__ __forceinline__ uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA into this CTA's shared memory, completing tx bytes on the leader CTA's barrier
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t leader_bar, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(leader_bar)
      : "memory");
}

__device__ __forceinline__ void umma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of 32-bit TMEM -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 registers per thread -> 32 lanes x 32 columns of 32-bit TMEM.
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
      "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
      "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// SM100 shared-memory matrix descriptor, K-major, SWIZZLE_128B:
//   [0,14) start>>4  [16,30) LBO>>4 (unused for swizzled K-major)
//   [32,46) SBO>>4 = 1024 B between 8-row core groups   [46,48) version = 1
//   [61,64) layout = 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo = 16, uint32_t sbo = 1024) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Operand tile in shared memory (SWIZZLE_128B), ROWS x one 128-byte K block:
//   K-major : ROWS rows of 128 B (K contiguous); 8-row groups 1024 B apart
//             (SBO); one MMA K-step advances the start address by 32 B.
//   MN-major: ROWS/ATOM columns of ATOM = 128/es MN-elements; each column is
//             BK K-rows of 128 B (LBO = BK*128 B between columns, SBO = 1024 B
//             between 8-K-row groups); one MMA K-step = 32/es K-rows =
//             4096/es bytes.  This is how dW = G^T X and dX = G W read their
//             operands without any transpose kernel.
template <typename TIN, bool MN>
struct Operand {
  static constexpr int ES = sizeof(TIN);
  static constexpr int BK = kAtomBytes / ES;       // K elements per stage
  static constexpr int ATOM = kAtomBytes / ES;     // MN elements per 128-byte atom
  static constexpr uint32_t COL_BYTES = BK * kAtomBytes;
  __device__ static __forceinline__ uint64_t desc(uint32_t base) {
    return MN ? make_desc(base, COL_BYTES, 1024) : make_desc(base, 16, 1024);
  }
  __device__ static __forceinline__ uint64_t kstep(int kk) {
    return MN ? (uint64_t)(((uint32_t)kk * (4096u / ES)) >> 4) : (uint64_t)((kk * kUmmaKBytes) >> 4);
  }
  // CTA ``rank`` of a 2-CTA cluster loads its share of a ROWS-row tile and
  // multicasts it to both: K-major -> row half [rank*ROWS/2, +ROWS/2) (the
  // map's box has ROWS/2 rows); MN-major -> the 128-byte MN atoms c with
  // c % 2 == rank.
  template <int ROWS>
  __device__ static __forceinline__ void load_half_mc(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int k0,
                                                      int r0, int rank) {
    if constexpr (!MN) {
      tma_load_2d_mc(dst + rank * (ROWS / 2) * kAtomBytes, map, bar, k0, r0 + rank * (ROWS / 2), 0x3);
    } else {
#pragma unroll
      for (int c = 0; c < ROWS / ATOM; ++c)
        if ((c & 1) == rank) tma_load_2d_mc(dst + c * COL_BYTES, map, bar, r0 + c * ATOM, k0, 0x3);
    }
  }
  // 2-SM pair: ROWS rows starting at r0 into this CTA, tx on the leader's barrier
  template <int ROWS>
  __device__ static __forceinline__ void load_2sm(uint8_t* dst, const CUtensorMap* map, uint32_t leader_bar, int k0,
                                                  int r0) {
    if constexpr (!MN) {
      tma_load_2d_2sm(dst, map, leader_bar, k0, r0);
    } else {
#pragma unroll
      for (int c = 0; c < ROWS / ATOM; ++c) tma_load_2d_2sm(dst + c * COL_BYTES, map, leader_bar, r0 + c * ATOM, k0);
    }
  }
  template <int ROWS>
  __device__ static __forceinline__ void load(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int k0, int r0) {
    if constexpr (!MN) {
      tma_load_2d(dst, map, bar, k0, r0);
    } else {
#pragma unroll
      for (int c = 0; c < ROWS / ATOM; ++c) tma_load_2d(dst + c * COL_BYTES, map, bar, r0 + c * ATOM, k0);
    }
  }
};

// Instruction descriptor (kind::f16 / kind::tf32), both operands K-major:
//   [4,6) D fmt = 1 (f32)  [7,10) A fmt  [10,13) B fmt  [17,23) N>>3  [24,29) M>>4
//   [15] A major (1 = MN)  [16] B major (1 = MN)
__host__ __device__ constexpr uint32_t make_idesc(int ab_fmt, int m, int n, bool a_mn = false, bool b_mn = false) {
  return (1u << 4) | ((uint32_t)ab_fmt << 7) | ((uint32_t)ab_fmt << 10) | ((uint32_t)(a_mn ? 1 : 0) << 15) |
         ((uint32_t)(b_mn ? 1 : 0) << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

struct Params {
  int64_t m, n, k;
  int64_t ld_d, ld_x, rows_per_group, ld_group;
  void* d;
  const float* bias;
  const void* x0;
  const void* xl;
  void* aux;
  const void* c;
  float* aux2;
  float beta;
  float alpha;
  int scale_acc;
  int aux2_accum;
  int out_dtype;
  int in_dtype;
  int epilogue;
  int vec_store;
  int vec_x;
  int coalesced;
  int prefetch;  // bit 0: x0, 1: xl, 2: c, 3: aux2 -- L2 prefetch of the epilogue operands
  int npairs;    // DCN_FINAL: d = acc + beta*C + sum_j pg[j] * pu[j] (instead of aux2)
  const void* pg[DMT_GEMM_MAX_PAIRS];
  const void* pu[DMT_GEMM_MAX_PAIRS];
  float* colsum;  // DCN_BWD: per (128-row tile, 32-row quarter) column sums of the stored gu
  int kchunk;     // tf32: K blocks accumulated per TMEM chunk (see gemm_kernel)
  int ngroups_out;  // > 0: row m -> gout[m / rows_per_group] + (m % rows_per_group) * ld_d
  void* gout[DMT_GEMM_MAX_OUT_GROUPS];
  int ncolg;        // > 0: column n -> colg[n / colg_w] + m * colg_ld[g] + n % colg_w
  int colg_w;
  void* colg[DMT_GEMM_MAX_COL_GROUPS];
  int64_t colg_ld[DMT_GEMM_MAX_COL_GROUPS];
  int ksplit;     // split-K: units = tiles x ksplit; split s covers K blocks [s*kbs, (s+1)*kbs)
  int kbs;        //   and writes its raw fp32 accumulator at output rows + s * m (workspace)
  int tma_out;    // direct path: bit 0 = output stored by TMA (emaps.od), bit 1 = 64-column boxes (emaps.od64)
  int pf_ahead;   // staged epilogue: L2-prefetch the operands this many slabs ahead (0 = off)
  int direct;     // register-direct epilogue (no shared-memory staging); DMT_GEMM_EPI=staged turns it off
  int dbg;        // experiment only (DMT_GEMM_DBG): 1 skip epilogue work, 2 / 16 direct epilogue without
                  // stores / TMEM loads, 4 skip MMAs, 8 skip TMA loads
};

// Output row address.  The grouped layout (per-feature DLRM projection rows
// scattered into the tower output) needs a 64-bit division; plain GEMMs take
// the multiply-only branch (ncu showed the division's I2F / MUFU.RCP sequence
// among the epilogue's hottest instructions).
template <typename TO>
__device__ __forceinline__ TO* out_row(const Params& p, int64_t row) {
  TO* d = reinterpret_cast<TO*>(p.d);
  if (p.ngroups_out)  // scattered row blocks (peer step-f receive buffers)
    return reinterpret_cast<TO*>(p.gout[row / p.rows_per_group]) + (row % p.rows_per_group) * p.ld_d;
  if (p.rows_per_group > p.m) return d + row * p.ld_d;
  return d + (row / p.rows_per_group) * p.ld_group + (row % p.rows_per_group) * p.ld_d;
}

// Address of output element (row, col): the plain / grouped-row layouts, or a
// scattered column block (the dX GEMM storing shards into their owners'
// gradient buffers).  A 32-column chunk never straddles a column block.
template <typename TO>
__device__ __forceinline__ TO* out_ptr(const Params& p, int64_t row, int64_t col) {
  if (p.ncolg) {
    const int g = (int)(col / p.colg_w);
    return reinterpret_cast<TO*>(p.colg[g]) + row * p.colg_ld[g] + (col - (int64_t)g * p.colg_w);
  }
  return out_row<TO>(p, row) + col;
}

// 32 consecutive elements of one row <-> 32 fp32 registers.  The vector forms
// need 16-byte alignment; the scalar forms are predicated (tail / unaligned).
template <typename TX>
__device__ __forceinline__ void load32v(const TX* __restrict__ p, float* v) {
  if constexpr (sizeof(TX) == 4) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      float4 x = *reinterpret_cast<const float4*>(p + i);
      v[i] = x.x; v[i + 1] = x.y; v[i + 2] = x.z; v[i + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint4 x = *reinterpret_cast<const uint4*>(p + i);
      const TX* h = reinterpret_cast<const TX*>(&x);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[i + j] = to_f<TX>(h[j]);
    }
  }
}
template <typename TO>
__device__ __forceinline__ void store32v(TO* __restrict__ p, const float* v) {
  if constexpr (sizeof(TO) == 4) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  } else {
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
      uint4 x;
      TO* h = reinterpret_cast<TO*>(&x);
#pragma unroll
      for (int j = 0; j < 8; ++j) h[j] = from_f<TO>(v[i + j]);
      *reinterpret_cast<uint4*>(p + i) = x;
    }
  }
}
template <typename TX>
__device__ __forceinline__ void load32s(const TX* __restrict__ p, float* v, int n) {
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = (i < n) ? to_f<TX>(p[i]) : 0.f;
}
template <typename TO>
__device__ __forceinline__ void store32s(TO* __restrict__ p, const float* v, int n) {
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < n) p[i] = from_f<TO>(v[i]);
}

// 8 consecutive elements (16 B for 16-bit types, 32 B for fp32) <-> 8 floats.
template <typename T>
__device__ __forceinline__ void load8(const T* __restrict__ p, float* v) {
  if constexpr (sizeof(T) == 4) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
    uint4 x = *reinterpret_cast<const uint4*>(p);
    const T* h = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = to_f<T>(h[j]);
  }
}
template <typename T>
__device__ __forceinline__ void store8(T* __restrict__ p, const float* v) {
  if constexpr (sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    uint4 x;
    T* h = reinterpret_cast<T*>(&x);
#pragma unroll
    for (int j = 0; j < 8; ++j) h[j] = from_f<T>(v[j]);
    *reinterpret_cast<uint4*>(p) = x;
  }
}

// Epilogue math for 8 columns of one row (coalesced path: 4 lanes per row).
template <typename TIN, typename TO>
__device__ __forceinline__ void epi8(const Params& p, int64_t row, int64_t col, float* v) {
  if (p.epilogue == DMT_EPI_BIAS || p.epilogue == DMT_EPI_CROSS) {
    float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + col));
    float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + col + 4));
    v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
    v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
  }
  const int64_t xo = row * p.ld_x + col;
  if (p.epilogue == DMT_EPI_CROSS) {
    float a[8], b[8];
    load8<TIN>(reinterpret_cast<const TIN*>(p.x0) + xo, a);
    load8<TIN>(reinterpret_cast<const TIN*>(p.xl) + xo, b);
    if (p.aux) store8<TIN>(reinterpret_cast<TIN*>(p.aux) + xo, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = a[j] * v[j] + b[j];
  } else if (p.epilogue == DMT_EPI_ACC || p.epilogue == DMT_EPI_DCN_BWD || p.epilogue == DMT_EPI_DCN_FINAL) {
    if (p.beta != 0.f) {
      float c[8];
      load8<TO>(reinterpret_cast<const TO*>(p.c) + row * p.ld_d + col, c);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += p.beta * c[j];
    }
    if (p.epilogue == DMT_EPI_DCN_FINAL) {
      float d[8];
      load8<float>(p.aux2 + xo, d);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += d[j];
    } else if (p.epilogue == DMT_EPI_DCN_BWD) {
      float x0[8], u[8], d[8];
      load8<TIN>(reinterpret_cast<const TIN*>(p.x0) + xo, x0);
      load8<TIN>(reinterpret_cast<const TIN*>(p.xl) + xo, u);
      if (p.aux2_accum) load8<float>(p.aux2 + xo, d);
      else {
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        x0[j] *= v[j];          // gu = g * x0
        d[j] += v[j] * u[j];    // dx0 += g * u
      }
      store8<TIN>(reinterpret_cast<TIN*>(p.aux) + xo, x0);
      store8<float>(p.aux2 + xo, d);
    }
  }
  store8<TO>(out_ptr<TO>(p, row, col), v);
}

// Raw (unconverted) epilogue inputs of one 8-column row piece, so two pieces'
// loads can be in flight before either is consumed (memory-level parallelism).
template <typename TIN, typename TO>
struct EpiIn {
  using RI = typename std::conditional<sizeof(TIN) == 4, float4, uint4>::type;
  using RO = typename std::conditional<sizeof(TO) == 4, float4, uint4>::type;
  RI x0[sizeof(TIN) == 4 ? 2 : 1], u[sizeof(TIN) == 4 ? 2 : 1];
  RO c[sizeof(TO) == 4 ? 2 : 1];
  float4 d[2];
};

template <typename R, typename T, int N>
__device__ __forceinline__ void rawld(const T* p, R (&r)[N]) {
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = reinterpret_cast<const R*>(p)[i];
}
template <typename R, typename T, int N>
__device__ __forceinline__ void rawcvt(const R (&r)[N], float* v) {
  load8<T>(reinterpret_cast<const T*>(&r[0]), v);
}

template <typename TIN, typename TO, bool FEAT>
__device__ __forceinline__ void epi_load(const Params& p, int64_t row, int64_t col, EpiIn<TIN, TO>& in) {
  const int64_t xo = row * p.ld_x + col;
  const int e = p.epilogue;
  if (e == DMT_EPI_CROSS || e == DMT_EPI_DCN_BWD || e == DMT_EPI_RELU_BWD)
    rawld(reinterpret_cast<const TIN*>(p.x0) + xo, in.x0);
  if (e == DMT_EPI_CROSS || (e == DMT_EPI_DCN_BWD && p.aux2)) rawld(reinterpret_cast<const TIN*>(p.xl) + xo, in.u);
  if ((e == DMT_EPI_ACC || e == DMT_EPI_DCN_BWD || e == DMT_EPI_DCN_FINAL) && p.beta != 0.f)
    rawld(reinterpret_cast<const TO*>(p.c) + row * p.ld_d + col, in.c);
  if ((e == DMT_EPI_DCN_FINAL && !(FEAT ? p.npairs : 0)) || (e == DMT_EPI_DCN_BWD && p.aux2 && p.aux2_accum))
    rawld(p.aux2 + xo, in.d);
}

// L2 prefetch of one 8-column row piece's epilogue operands (no registers
// held): issued a few slabs ahead of the register loads in the staged path.
__device__ __forceinline__ void l2pf(const void* a) { asm volatile("prefetch.global.L2 [%0];" ::"l"(a)); }
template <typename TIN, typename TO, bool FEAT>
__device__ __forceinline__ void epi_prefetch(const Params& p, int64_t row, int64_t col) {
  const int64_t xo = row * p.ld_x + col;
  const int e = p.epilogue;
  if (e == DMT_EPI_CROSS || e == DMT_EPI_DCN_BWD || e == DMT_EPI_RELU_BWD) l2pf(reinterpret_cast<const TIN*>(p.x0) + xo);
  if (e == DMT_EPI_CROSS || (e == DMT_EPI_DCN_BWD && p.aux2)) l2pf(reinterpret_cast<const TIN*>(p.xl) + xo);
  if ((e == DMT_EPI_ACC || e == DMT_EPI_DCN_BWD || e == DMT_EPI_DCN_FINAL) && p.beta != 0.f)
    l2pf(reinterpret_cast<const TO*>(p.c) + row * p.ld_d + col);
  if ((e == DMT_EPI_DCN_FINAL && !(FEAT ? p.npairs : 0)) || (e == DMT_EPI_DCN_BWD && p.aux2 && p.aux2_accum))
    l2pf(p.aux2 + xo);
}

// dx0 = sum_l g_{l+1} * u_l straight from the saved layer tensors (DCN_FINAL).
// Out of line: its loads would otherwise raise the register pressure of every
// epilogue variant compiled into the kernel.
template <typename TIN>
__device__ __forceinline__ void pair_sum8(const Params& p, int64_t xo, float* v) {
#pragma unroll
  for (int j = 0; j < DMT_GEMM_MAX_PAIRS; ++j) {  // constant indices: no local copy of p.pg / p.pu
    if (j >= p.npairs) break;
    float g[8], u[8];
    load8<TIN>(reinterpret_cast<const TIN*>(p.pg[j]) + xo, g);
    load8<TIN>(reinterpret_cast<const TIN*>(p.pu[j]) + xo, u);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] += g[i] * u[i];
  }
}

// gu as stored (rounded to the operand type): what the dW GEMM and the bias
// gradient see
template <typename T>
__device__ __forceinline__ float stored(float x) {
  return to_f<T>(from_f<T>(x));
}

// av: when non-null, the aux output (CROSS u / DCN_BWD gu) goes there instead
// of global memory; store_out = false leaves the output in v (TMA-stored
// epilogue path).
template <typename TIN, typename TO, bool FEAT>
__device__ __forceinline__ void epi_finish(const Params& p, int64_t row, int64_t col, float* v,
                                           const EpiIn<TIN, TO>& in, float* gs, int64_t soff,
                                           float* av = nullptr, bool store_out = true) {
  const int e = p.epilogue;
  if (e == DMT_EPI_BIAS || e == DMT_EPI_CROSS || e == DMT_EPI_BIAS_RELU) {
    float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + col));
    float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + col + 4));
    v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
    v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
  }
  if (e == DMT_EPI_BIAS_RELU) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = fmaxf(v[j], 0.f);
  }
  const int64_t xo = row * p.ld_x + col;
  if (e == DMT_EPI_RELU_BWD) {
    float a[8];
    rawcvt<typename EpiIn<TIN, TO>::RI, TIN>(in.x0, a);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = a[j] > 0.f ? v[j] : 0.f;
  }
  if (e == DMT_EPI_CROSS) {
    float a[8], b[8];
    rawcvt<typename EpiIn<TIN, TO>::RI, TIN>(in.x0, a);
    rawcvt<typename EpiIn<TIN, TO>::RI, TIN>(in.u, b);
    if (av) {
#pragma unroll
      for (int j = 0; j < 8; ++j) av[j] = v[j];
    } else if (p.aux) {
      store8<TIN>(reinterpret_cast<TIN*>(p.aux) + xo, v);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = a[j] * v[j] + b[j];
  } else if (e == DMT_EPI_ACC || e == DMT_EPI_DCN_BWD || e == DMT_EPI_DCN_FINAL) {
    if (p.beta != 0.f) {
      float c[8];
      rawcvt<typename EpiIn<TIN, TO>::RO, TO>(in.c, c);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] += p.beta * c[j];
    }
    if (e == DMT_EPI_DCN_FINAL) {
      if ((FEAT ? p.npairs : 0)) {
        pair_sum8<TIN>(p, xo, v);
      } else {
        float d[8];
        rawcvt<float4, float>(in.d, d);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] += d[j];
      }
    } else if (e == DMT_EPI_DCN_BWD) {
      float x0[8];
      rawcvt<typename EpiIn<TIN, TO>::RI, TIN>(in.x0, x0);
#pragma unroll
      for (int j = 0; j < 8; ++j) x0[j] *= v[j];
      if (av) {
#pragma unroll
        for (int j = 0; j < 8; ++j) av[j] = x0[j];
      } else {
        store8<TIN>(reinterpret_cast<TIN*>(p.aux) + xo, x0);
      }
      if (gs) {
#pragma unroll
        for (int j = 0; j < 8; ++j) gs[j] = stored<TIN>(x0[j]);
      }
      if (p.aux2) {
        float u[8], d[8];
        rawcvt<typename EpiIn<TIN, TO>::RI, TIN>(in.u, u);
        if (p.aux2_accum) rawcvt<float4, float>(in.d, d);
        else {
#pragma unroll
          for (int j = 0; j < 8; ++j) d[j] = 0.f;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) d[j] += v[j] * u[j];
        store8<float>(p.aux2 + xo, d);
      }
    }
  }
  if (store_out) store8<TO>(out_ptr<TO>(p, row + soff, col), v);  // soff: split-K workspace rows
}

// ---- TMA-stored epilogue (register-direct path) ----------------------------
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(smem))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// One row (this lane's) of a 32-column chunk of 16-bit outputs into half
// `hf` of a 32 x 64 staging tile (128-byte rows: the TMA store then writes
// whole 128-byte lines).  Rows are 128 B apart, so 8 lanes can cover only 4
// distinct 16-byte bank groups per store: 2-way conflicts, accepted.
template <typename T>
__device__ __forceinline__ void stage_row64(uint8_t* buf, int lane, const float* v, int hf) {
  static_assert(sizeof(T) == 2, "16-bit outputs");
  uint4 ch[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    T* h = reinterpret_cast<T*>(&ch[c]);
#pragma unroll
    for (int e = 0; e < 8; ++e) h[e] = from_f<T>(v[c * 8 + e]);
  }
  uint4* row = reinterpret_cast<uint4*>(buf + lane * 128) + hf * 4;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int idx = (j + lane) & 3;
    uint4 x = ch[0];
#pragma unroll
    for (int c = 1; c < 4; ++c)
      if (idx == c) x = ch[c];
    row[idx] = x;
  }
}

// One row (this lane's) of a 32 x 32 output chunk into an unswizzled staging
// tile (row pitch 32 * sizeof(T)) for a TMA store.  Store j of lane r writes
// 16-byte piece (j + s_r) mod P, s_r chosen so that every 8-lane phase covers
// all 32 banks (bf16: rows 64 B apart -> s = r / 2; fp32: 128 B -> s = r).
template <typename T>
__device__ __forceinline__ void stage_row(uint8_t* buf, int lane, const float* v) {
  constexpr int P = 32 * (int)sizeof(T) / 16;  // 16-byte pieces per row
  uint4 ch[P];
#pragma unroll
  for (int c = 0; c < P; ++c) {
    constexpr int E = 16 / (int)sizeof(T);
    T* h = reinterpret_cast<T*>(&ch[c]);
#pragma unroll
    for (int e = 0; e < E; ++e) h[e] = from_f<T>(v[c * E + e]);
  }
  const int sft = sizeof(T) == 4 ? lane : (lane >> 1);
  uint4* row = reinterpret_cast<uint4*>(buf + lane * 32 * (int)sizeof(T));
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const int idx = (j + sft) & (P - 1);
    uint4 x = ch[0];
#pragma unroll
    for (int c = 1; c < P; ++c)
      if (idx == c) x = ch[c];
    row[idx] = x;
  }
}

// The epilogue operands of a tile (x0 / xl / C / dx0 blocks) do not depend on
// the accumulator: the producer prefetches them into L2 with one 2-D TMA
// prefetch per operand when it starts the tile's operand loads, one
// tile-mainloop ahead of the epilogue, so the epilogue's loads hit L2.
// (Per-row 1-D bulk prefetches were measured slower: hundreds of small TMA
// requests per tile queue in front of the operand loads.)
__device__ __forceinline__ void l2_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1)
               : "memory");
}

struct EpiMaps {
  CUtensorMap x0, xl, c, d2;
  CUtensorMap od;    // TMA store of the output (32 x 32 boxes)
  CUtensorMap od64;  // 16-bit outputs: 32 rows x 64 columns (whole 128-byte lines)
};

constexpr int kStileFloats = 32 * 33;

// Column sums of one warp's 32 x 32 staged gu chunk (lane = column, rows in
// order): the fused DCN bias gradient partial of (128-row tile, quarter q).
__device__ __forceinline__ void colsum_chunk(const Params& p, float* stile, int64_t m0, int q, int64_t col0,
                                             int lane) {
  __syncwarp();
  float acc = 0.f;
#pragma unroll 8
  for (int r = 0; r < 32; ++r) acc += stile[r * 33 + lane];
  p.colsum[((m0 / 128) * 4 + q) * p.n + col0 + lane] = acc;
  __syncwarp();
}  // per-warp padded 32x32 fp32 staging tile

// BN: tile N (64/128/256); NOPS: 1 (plain) or 3 (3xTF32); KIND: 0 f16-family, 1 tf32
// FEAT: compile in the DCN-backward extras (fused bias-gradient column sums,
// DCN_FINAL pair sums); kept out of the other variants' register budget.
// CL: CTAs per cluster along M: 1, or 2 = a cta_group::2 pair.  The pair
// computes a 256 x BN tile with one MMA stream issued by the leader CTA: each
// CTA stages its own 128 rows of A and one half of B's BN columns, so every
// operand byte is read from shared memory once for the pair (a single-CTA
// 128 x BN tile re-reads all of B per CTA: 1.5x the shared-memory operand
// traffic at BN = 256, which the epilogue's staging then competes with).
template <int BN, int NOPS, int KIND, int STAGES, typename TIN, typename TO, bool AMN, bool BMN, bool FEAT,
          int CL = 1>
__global__ void __launch_bounds__(kThreads, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
            const __grid_constant__ CUtensorMap map_a_lo, const __grid_constant__ CUtensorMap map_b_lo,
            const __grid_constant__ EpiMaps emaps, const Params p, uint32_t idesc) {
  constexpr int A_BYTES = kBlockM * kAtomBytes;
  constexpr int B_BYTES = (BN / CL) * kAtomBytes;  // this CTA's share of the B tile
  static_assert(CL == 1 || (KIND == 0 && NOPS == 1), "2-SM pairs: 16-bit operands");
  constexpr int NSETS = (NOPS == 3) ? 2 : 1;  // hi (+ lo) operand copies
  constexpr int STAGE_BYTES = NSETS * (A_BYTES + B_BYTES);
  // tf32 (fp32 parity path): two accumulators + two chunk-scratch buffers
  constexpr int ACC_BUFS = (KIND == 1) ? 4 : 2;
  constexpr uint32_t TMEM_COLS = (ACC_BUFS * BN <= 32) ? 32 : (ACC_BUFS * BN <= 64 ? 64 :
                                 (ACC_BUFS * BN <= 128 ? 128 : (ACC_BUFS * BN <= 256 ? 256 : 512)));
  static_assert(ACC_BUFS * BN <= 512, "TMEM columns");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;   // tf32 chunk scratch buffers: MMA -> epilogue
  uint64_t* sempty = sfull + 2;   //                             epilogue -> MMA
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(sempty + 2);
  float* stile_all = reinterpret_cast<float*>(smem + STAGES * STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t tiles_m = ceil_div(p.m, kBlockM), tiles_n = ceil_div(p.n, BN);
  // work unit = CL vertically adjacent tiles sharing n0 (one per cluster CTA)
  const int64_t num_units = ceil_div(tiles_m, CL) * tiles_n * p.ksplit;
  const int crank = CL > 1 ? (int)cluster_rank() : 0;
  const int64_t u_first = blockIdx.x / CL, u_step = gridDim.x / CL;
  // unit u = (tile u / ksplit, K split u % ksplit)
  auto unit_m0 = [&](int64_t u) { return (int64_t)((((u / p.ksplit) / tiles_n) * CL + crank) * kBlockM); };
  auto unit_n0 = [&](int64_t u) { return (int64_t)(((u / p.ksplit) % tiles_n) * BN); };
  const int num_kb_all = (int)ceil_div(p.k * (int64_t)sizeof(TIN), kAtomBytes);
  auto unit_kb0 = [&](int64_t u) { return (int)(u % p.ksplit) * p.kbs; };
  auto unit_kb1 = [&](int64_t u) { return min(num_kb_all, (int)(u % p.ksplit + 1) * p.kbs); };
  constexpr int K_ELEMS = kAtomBytes / sizeof(TIN);
  using OA = Operand<TIN, AMN>;
  using OB = Operand<TIN, BMN>;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // (pair: only the leader's is used; both CTAs' TMA complete on it)
      mbar_init(&empty[s], 1);  // released by the (leader's) MMA commit
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kEpiWarps * CL);  // one arrive per epilogue warp of the pair (leader's)
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CL == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CL > 1) cluster_sync_all();  // peers' barriers initialised before any multicast
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    }
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t u = u_first; u < num_units; u += u_step) {
      const int m0 = (int)unit_m0(u);
      const int n0 = (int)unit_n0(u);
      if (lane == 0 && p.prefetch) {
        if (p.prefetch & 1) l2_prefetch_2d(&emaps.x0, n0, m0);
        if (p.prefetch & 2) l2_prefetch_2d(&emaps.xl, n0, m0);
        if (p.prefetch & 4) l2_prefetch_2d(&emaps.c, n0, m0);
        if (p.prefetch & 8) l2_prefetch_2d(&emaps.d2, n0, m0);
      }
      if (lane == 0) {
        const int kb_end = unit_kb1(u);
        for (int kb = unit_kb0(u); kb < kb_end; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          if (p.dbg & 8) {  // experiment: no operand loads (MMA-only rate)
            if (crank == 0) mbar_arrive(&full[stage]);
          } else if constexpr (CL == 2) {
            // both CTAs' loads complete on the leader's barrier; the leader
            // expects the pair's bytes
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
            const uint32_t lbar = mapa_rank(&full[stage], 0);
            OA::template load_2sm<kBlockM>(sa, &map_a, lbar, kb * K_ELEMS, m0);
            OB::template load_2sm<BN / 2>(sb, &map_b, lbar, kb * K_ELEMS, n0 + crank * (BN / 2));
          } else {
            mbar_expect_tx(&full[stage], STAGE_BYTES);
            OA::template load<kBlockM>(sa, &map_a, &full[stage], kb * K_ELEMS, m0);
            OB::template load<BN>(sb, &map_b, &full[stage], kb * K_ELEMS, n0);
          }
          if (NSETS == 2 && !(p.dbg & 8)) {
            uint8_t* sa2 = sb + B_BYTES;
            uint8_t* sb2 = sa2 + A_BYTES;
            OA::template load<kBlockM>(sa2, &map_a_lo, &full[stage], kb * K_ELEMS, m0);
            OB::template load<BN>(sb2, &map_b_lo, &full[stage], kb * K_ELEMS, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && crank == 0) {  // a pair's MMAs are issued by its leader
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      int s_it = 0;  // tf32 chunk-scratch uses
      for (int64_t u = u_first; u < num_units; u += u_step, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        // tf32: the tensor core's accumulation truncates, so a long K chain
        // drifts (measured ~3e-5 max-norm relative at K = 3328, 10x fp32's).
        // Every p.kchunk K blocks start a fresh accumulation in a scratch TMEM
        // buffer; the epilogue warps fold it into the tile's accumulator with
        // round-to-nearest fp32 adds in chunk order (deterministic).
        uint32_t tmem_t = tmem_d;
        bool first = true;
        const int kb_beg = unit_kb0(u), kb_end = unit_kb1(u);
        for (int kb = kb_beg; kb < kb_end; ++kb) {
          if constexpr (KIND == 1) {
            if (kb > kb_beg && (kb - kb_beg) % p.kchunk == 0) {
              if (tmem_t != tmem_d) umma_commit(&sfull[(s_it - 1) & 1]);  // previous chunk complete
              mbar_wait(&sempty[s_it & 1], ((s_it >> 1) & 1) ^ 1);
              tc_fence_after();
              tmem_t = tmem_base + (2 + (s_it & 1)) * BN;
              ++s_it;
              first = true;
            }
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint64_t da = OA::desc(smem_u32(sa));
          const uint64_t db = OB::desc(smem_u32(sb));
#pragma unroll
          for (int kk = 0; kk < kAtomBytes / kUmmaKBytes; ++kk) {
            const uint64_t ada = OA::kstep(kk), adb = OB::kstep(kk);
            const uint32_t accum = (first && kk == 0) ? 0u : 1u;
            if (p.dbg & 4) continue;  // experiment: no MMAs (operand-feed rate)
            if constexpr (CL == 2) umma2(tmem_t, da + ada, db + adb, idesc, accum);
            else umma<KIND>(tmem_t, da + ada, db + adb, idesc, accum);
            if constexpr (NSETS == 2) {
              uint8_t* sa2 = sb + B_BYTES;
              uint8_t* sb2 = sa2 + A_BYTES;
              const uint64_t da2 = OA::desc(smem_u32(sa2));
              const uint64_t db2 = OB::desc(smem_u32(sb2));
              umma<KIND>(tmem_t, da + ada, db2 + adb, idesc, 1u);  // hi * lo
              umma<KIND>(tmem_t, da2 + ada, db + adb, idesc, 1u);  // lo * hi
            }
          }
          // smem slot reusable once these MMAs retire (in both CTAs of a pair)
          if constexpr (CL == 2) umma2_commit_mc(&empty[stage], 0x3);
          else umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          first = false;
        }
        if constexpr (KIND == 1) {
          if (tmem_t != tmem_d) umma_commit(&sfull[(s_it - 1) & 1]);
        }
        if constexpr (CL == 2) umma2_commit_mc(&tfull[acc], 0x3);  // both CTAs' accumulators complete
        else umma_commit(&tfull[acc]);  // accumulator complete
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;                       // TMEM lane quarter accessible to this warp
    const int half = (warp - 2) / 4;              // which half of the tile's columns
    constexpr int kColsPerWarp = BN / (kEpiWarps / 4);
    int it = 0;
    int e_it = 0;  // tf32 chunk-scratch uses (mirrors the MMA warp's s_it)
    for (int64_t u = u_first; u < num_units; u += u_step, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int64_t m0 = unit_m0(u);
      const int64_t n0 = unit_n0(u);
      const int64_t soff = (u % p.ksplit) * p.m;  // split-K: partial s lands at rows + s * m
      float* stile = stile_all + (warp - 2) * kStileFloats;
      if (p.dbg & 1) {  // experiment: accumulator hand-off only, no epilogue work
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
        __syncwarp();
        tc_fence_before();
        if (lane == 0) {
          if constexpr (CL == 2) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
          else mbar_arrive(&tempty[acc]);
        }
        continue;
      }
      if constexpr (KIND == 1) {
        // fold chunks 1.. of this tile into its accumulator (chunk order)
        const int nch = (unit_kb1(u) - unit_kb0(u) + p.kchunk - 1) / p.kchunk;
        const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
        for (int c = 1; c < nch; ++c, ++e_it) {
          mbar_wait(&sfull[e_it & 1], (e_it >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int col = half * kColsPerWarp; col < (half + 1) * kColsPerWarp; col += 32) {
            float v[32], w[32];
            tmem_ld32(lane_base + (uint32_t)((2 + (e_it & 1)) * BN + col), v);
            tmem_ld32(lane_base + (uint32_t)(acc * BN + col), w);
#pragma unroll
            for (int i = 0; i < 32; ++i) w[i] += v[i];
            tmem_st32(lane_base + (uint32_t)(acc * BN + col), w);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sempty[e_it & 1]);
        }
      }
      if (p.direct && p.coalesced && !(FEAT && p.colsum) && n0 + (int64_t)(half + 1) * kColsPerWarp <= p.n) {
        // Direct path for epilogues that read nothing from global memory
        // (NONE / BIAS / BIAS_RELU / ACC without C): lane = row, a 32-column
        // TMEM chunk -> registers -> a bank-staggered 32 x 32 staging tile in
        // the output type -> one TMA bulk store per chunk, and the accumulator
        // is handed back as soon as its last chunk is read.  Measured on
        // 8192 x 3328 x 3328 (tools/cublas_compare.py): 140 us with the
        // staged fp32 transposition, 132 us here; the mainloop alone (no
        // epilogue work, DMT_GEMM_DBG=1) 118 us, TMEM reads alone 119 us.
        constexpr int kChunks = kColsPerWarp / 32;
        const int64_t r = m0 + q * 32 + lane;
        const bool ok = r < p.m;
        const int64_t cbase = n0 + half * kColsPerWarp;
        const EpiIn<TIN, TO> none{};  // (load-free epilogues only)
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < kChunks; ++c) {
          float v[32];
          if (!(p.dbg & 16))
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + half * kColsPerWarp + c * 32), v);
          else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = (float)i;
          }
          if (c + 1 == kChunks) {  // accumulator fully read: hand it back before the stores
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if constexpr (CL == 2) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
              else mbar_arrive(&tempty[acc]);
            }
          }
          if (p.scale_acc) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
          }
          if (p.dbg & 2) {  // experiment: accumulator reads only
            if (v[31] == 1234.5f && v[7] == 1.f) reinterpret_cast<float*>(p.d)[0] = v[0];
            continue;
          }
          const int64_t col = cbase + c * 32;
          const bool td = p.tma_out & 1;
          if (ok) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              epi_finish<TIN, TO, FEAT>(p, r, col + 8 * j, v + 8 * j, none, nullptr, soff, nullptr, !td);
          }
          if (td && sizeof(TO) == 2 && (p.tma_out & 2) && (kChunks % 2) == 0) {
            // pairs of chunks into one 32 x 64 tile, one TMA store per pair
            uint8_t* sd = reinterpret_cast<uint8_t*>(stile);
            if ((c & 1) == 0) {
              if (lane == 0) bulk_wait_read0();
              __syncwarp();
            }
            if constexpr (sizeof(TO) == 2) stage_row64<TO>(sd, lane, v, c & 1);
            if (c & 1) {
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&emaps.od64, sd, (int)(col - 32), (int)(m0 + q * 32));
                bulk_commit();
              }
            }
          } else if (td) {
            // the previous chunk's TMA store must have read the staging tile
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
            uint8_t* sd = reinterpret_cast<uint8_t*>(stile);
            stage_row<TO>(sd, lane, v);
            fence_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&emaps.od, sd, (int)col, (int)(m0 + q * 32));
              bulk_commit();
            }
          }
        }
        continue;
      }
      if (p.coalesced && n0 + (int64_t)(half + 1) * kColsPerWarp <= p.n) {
        // Pipelined full-width path: the epilogue operands (x0 / u / C / dx0)
        // do not depend on the accumulator, so the loads of slab-pair k+1 are
        // issued before slab-pair k is finished -- and the first ones before
        // the accumulator barrier -- hiding their latency behind the MMAs.
        // slab k = 8 rows x 32 columns of this warp's chunk (k & 3) of chunk k >> 2
        constexpr int kSlabs = (kColsPerWarp / 32) * 4;
        const int c8 = (lane & 3) * 8;
        auto slab_pos = [&](int k, int64_t& r, int64_t& col) {
          col = n0 + half * kColsPerWarp + (k >> 2) * 32 + c8;
          r = m0 + q * 32 + (k & 3) * 8 + (lane >> 2);
        };
        EpiIn<TIN, TO> nx;
        {
          int64_t r, col;
          slab_pos(0, r, col);
          if (r < p.m) epi_load<TIN, TO, FEAT>(p, r, col, nx);
          for (int k = 1; k < p.pf_ahead && k < kSlabs; ++k) {
            slab_pos(k, r, col);
            if (r < p.m) epi_prefetch<TIN, TO, FEAT>(p, r, col);
          }
        }
        mbar_wait(&tfull[acc], acc_phase);
        tc_fence_after();
#pragma unroll 1
        for (int k = 0; k < kSlabs; ++k) {
          if ((k & 3) == 0) {  // stage the next 32-column chunk of the accumulator
            float v[32];
            tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) +
                          (uint32_t)(acc * BN + half * kColsPerWarp + (k >> 2) * 32), v);
            if (p.scale_acc) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 32; ++i) stile[lane * 33 + i] = v[i];
            __syncwarp();
          }
          EpiIn<TIN, TO> cur = nx;
          int64_t r, col;
          slab_pos(k, r, col);
          if (k + 1 < kSlabs) {
            int64_t rn, coln;
            slab_pos(k + 1, rn, coln);
            if (rn < p.m) epi_load<TIN, TO, FEAT>(p, rn, coln, nx);
          }
          if (p.pf_ahead && k + p.pf_ahead < kSlabs) {
            int64_t rp, colp;
            slab_pos(k + p.pf_ahead, rp, colp);
            if (rp < p.m) epi_prefetch<TIN, TO, FEAT>(p, rp, colp);
          }
          const int rl = (k & 3) * 8 + (lane >> 2);
          float a[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) a[j] = stile[rl * 33 + c8 + j];
          if (FEAT && p.colsum) {
            // stored gu back into the consumed staging slots, zero for rows >= m
            float gq[8];
            if (r < p.m) epi_finish<TIN, TO, FEAT>(p, r, col, a, cur, gq, soff);
            else {
#pragma unroll
              for (int j = 0; j < 8; ++j) gq[j] = 0.f;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) stile[rl * 33 + c8 + j] = gq[j];
            if ((k & 3) == 3) colsum_chunk(p, stile, m0, q, col - c8, lane);
          } else if (r < p.m) {
            epi_finish<TIN, TO, FEAT>(p, r, col, a, cur, nullptr, soff);
          }
        }
        __syncwarp();
        tc_fence_before();
        if (lane == 0) {
          if constexpr (CL == 2) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
          else mbar_arrive(&tempty[acc]);
        }
        continue;
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t row = m0 + q * 32 + lane;
      const bool row_ok = row < p.m;
#pragma unroll 1
      for (int c = half * kColsPerWarp; c < (half + 1) * kColsPerWarp; c += 32) {
        float v[32];
        tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c), v);
        if (p.scale_acc) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
        }
        const int64_t col = n0 + c;
        const int64_t rem = p.n - col;
        const int ncols = rem <= 0 ? 0 : (rem < 32 ? (int)rem : 32);
        if (ncols == 0) continue;  // warp-uniform
        if (ncols == 32 && p.coalesced) {
          // stage the 32x32 chunk (thread = row) through a padded smem tile,
          // then 4 lanes per row: every global access of the warp covers 8
          // rows x 64-128 contiguous bytes instead of 32 scattered rows.
#pragma unroll
          for (int i = 0; i < 32; ++i) stile[lane * 33 + i] = v[i];
          __syncwarp();
          const int c8 = (lane & 3) * 8;
#pragma unroll 1
          for (int it = 0; it < 4; it += 2) {
            // two 8-row slabs per pass: both slabs' inputs are loaded before
            // either is consumed
            const int rl0 = it * 8 + (lane >> 2), rl1 = rl0 + 8;
            const int64_t r0 = m0 + q * 32 + rl0, r1 = r0 + 8;
            EpiIn<TIN, TO> in0, in1;
            if (r0 < p.m) epi_load<TIN, TO, FEAT>(p, r0, col + c8, in0);
            if (r1 < p.m) epi_load<TIN, TO, FEAT>(p, r1, col + c8, in1);
            float a[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = stile[rl0 * 33 + c8 + j];
            float gq[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) gq[j] = 0.f;
            if (r0 < p.m) epi_finish<TIN, TO, FEAT>(p, r0, col + c8, a, in0, (FEAT && p.colsum) ? gq : nullptr, soff);
            if (FEAT && p.colsum) {
#pragma unroll
              for (int j = 0; j < 8; ++j) { stile[rl0 * 33 + c8 + j] = gq[j]; gq[j] = 0.f; }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = stile[rl1 * 33 + c8 + j];
            if (r1 < p.m) epi_finish<TIN, TO, FEAT>(p, r1, col + c8, a, in1, (FEAT && p.colsum) ? gq : nullptr, soff);
            if (FEAT && p.colsum) {
#pragma unroll
              for (int j = 0; j < 8; ++j) stile[rl1 * 33 + c8 + j] = gq[j];
            }
          }
          if (FEAT && p.colsum) colsum_chunk(p, stile, m0, q, col, lane);
          __syncwarp();
          continue;
        }
        if (!row_ok) continue;
        const bool full = ncols == 32;
        if (p.epilogue == DMT_EPI_BIAS || p.epilogue == DMT_EPI_CROSS || p.epilogue == DMT_EPI_BIAS_RELU) {
          if (full) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4 bb = __ldg(reinterpret_cast<const float4*>(p.bias + col + i));
              v[i] += bb.x; v[i + 1] += bb.y; v[i + 2] += bb.z; v[i + 3] += bb.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += (i < ncols) ? p.bias[col + i] : 0.f;
          }
        }
        if (p.epilogue == DMT_EPI_BIAS_RELU) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
        } else if (p.epilogue == DMT_EPI_RELU_BWD) {
          const TIN* mp = reinterpret_cast<const TIN*>(p.x0) + row * p.ld_x + col;
          float t[32];
          if (full && p.vec_x) load32v<TIN>(mp, t);
          else load32s<TIN>(mp, t, ncols);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = t[i] > 0.f ? v[i] : 0.f;
        }
        if (p.epilogue == DMT_EPI_CROSS) {
          const TIN* x0p = reinterpret_cast<const TIN*>(p.x0) + row * p.ld_x + col;
          const TIN* xlp = reinterpret_cast<const TIN*>(p.xl) + row * p.ld_x + col;
          TIN* auxp = p.aux ? reinterpret_cast<TIN*>(p.aux) + row * p.ld_x + col : nullptr;
          float t[32];
          if (full && p.vec_x) {
            if (auxp) store32v<TIN>(auxp, v);
            load32v<TIN>(x0p, t);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= t[i];
            load32v<TIN>(xlp, t);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += t[i];
          } else {
            if (auxp) store32s<TIN>(auxp, v, ncols);
            load32s<TIN>(x0p, t, ncols);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= t[i];
            load32s<TIN>(xlp, t, ncols);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += t[i];
          }
        } else if (p.epilogue == DMT_EPI_ACC || p.epilogue == DMT_EPI_DCN_BWD || p.epilogue == DMT_EPI_DCN_FINAL) {
          if (p.beta != 0.f) {
            const TO* cp = reinterpret_cast<const TO*>(p.c) + row * p.ld_d + col;
            float t[32];
            if (full && p.vec_store) load32v<TO>(cp, t);
            else load32s<TO>(cp, t, ncols);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += p.beta * t[i];
          }
          if (p.epilogue != DMT_EPI_ACC) {
            float* dxp = p.aux2 + row * p.ld_x + col;
            const bool vx = full && p.vec_x;
            if (p.epilogue == DMT_EPI_DCN_FINAL && (FEAT ? p.npairs : 0)) {
#pragma unroll
              for (int j = 0; j < DMT_GEMM_MAX_PAIRS; ++j) {
                if (j >= (FEAT ? p.npairs : 0)) break;
                const TIN* gp = reinterpret_cast<const TIN*>(p.pg[j]) + row * p.ld_x + col;
                const TIN* upp = reinterpret_cast<const TIN*>(p.pu[j]) + row * p.ld_x + col;
                float t[32], w[32];
                if (vx) { load32v<TIN>(gp, t); load32v<TIN>(upp, w); }
                else { load32s<TIN>(gp, t, ncols); load32s<TIN>(upp, w, ncols); }
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] += t[i] * w[i];
              }
            } else if (p.epilogue == DMT_EPI_DCN_FINAL) {
              float t[32];
              if (vx) load32v<float>(dxp, t);
              else load32s<float>(dxp, t, ncols);
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] += t[i];
            } else {
              // g = v; gu = g * x0 -> aux; dx0 (+)= g * u -> aux2
              const TIN* x0p = reinterpret_cast<const TIN*>(p.x0) + row * p.ld_x + col;
              const TIN* up = reinterpret_cast<const TIN*>(p.xl) + row * p.ld_x + col;
              TIN* gup = reinterpret_cast<TIN*>(p.aux) + row * p.ld_x + col;
              float t[32], w[32];
              if (vx) load32v<TIN>(x0p, t);
              else load32s<TIN>(x0p, t, ncols);
#pragma unroll
              for (int i = 0; i < 32; ++i) w[i] = v[i] * t[i];
              if (vx) store32v<TIN>(gup, w);
              else store32s<TIN>(gup, w, ncols);
              if (p.aux2) {  // dx0 accumulation (legacy form; NULL with the pair-sum final layer)
              if (vx) load32v<TIN>(up, t);
              else load32s<TIN>(up, t, ncols);
              if (p.aux2_accum) {
                if (vx) load32v<float>(dxp, w);
                else load32s<float>(dxp, w, ncols);
              } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) w[i] = 0.f;
              }
#pragma unroll
              for (int i = 0; i < 32; ++i) w[i] += v[i] * t[i];
              if (vx) store32v<float>(dxp, w);
              else store32s<float>(dxp, w, ncols);
              }
            }
          }
        }
        if (full && p.vec_store) store32v<TO>(out_ptr<TO>(p, row + soff, col), v);
        else store32s<TO>(out_ptr<TO>(p, row + soff, col), v, ncols);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CL == 2) mbar_arrive_cluster(mapa_rank(&tempty[acc], 0));
        else mbar_arrive(&tempty[acc]);
      }
    }
    if (p.tma_out && lane == 0) bulk_wait0();  // TMA-stored outputs complete before exit
  }

  __syncthreads();
  if constexpr (CL == 2) {
    // both CTAs done with the pair's TMEM and barriers before the dealloc /
    // exit (the peer's epilogue arrives on the leader's barriers)
    cluster_sync_all();
    if (warp == 1) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS)
                   : "memory");
    }
  } else if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
  }
}

// ---------------------------------------------------------------- host ------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// K-major operand [rows, k] (row stride ld): box {128 B of K, box_rows}.
// MN-major operand stored [k, rows] (row stride ld): box {128 B of MN, 128 B / es K-rows}.
static bool make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int64_t ld, int dtype,
                     int box_rows, bool mn = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  CUtensorMapDataType t;
  size_t es = dtype_size(dtype);
  switch (dtype) {
    case DMT_BF16: t = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16; break;
    case DMT_F16: t = CU_TENSOR_MAP_DATA_TYPE_FLOAT16; break;
    case DMT_F32: t = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; break;
    default: return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)k, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)(kAtomBytes / es), (cuuint32_t)box_rows};
  if (mn) {
    dims[0] = (cuuint64_t)rows;
    dims[1] = (cuuint64_t)k;
    box[0] = (cuuint32_t)(kAtomBytes / es);
    box[1] = (cuuint32_t)(kAtomBytes / es);
  }
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, t, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-major [rows, cols] block (row stride ld), no swizzle: box {box_cols, box_rows}
// for the L2 prefetch of epilogue operands.
static bool make_plain_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int dtype,
                           int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn || !ptr) return false;
  CUtensorMapDataType t;
  switch (dtype) {
    case DMT_BF16: t = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16; break;
    case DMT_F16: t = CU_TENSOR_MAP_DATA_TYPE_FLOAT16; break;
    case DMT_F32: t = CU_TENSOR_MAP_DATA_TYPE_FLOAT32; break;
    default: return false;
  }
  const size_t es = dtype_size(dtype);
  if (((uintptr_t)ptr % 16) || ((ld * es) % 16) || ((box_cols * es) % 16)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, t, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// tf32 accumulation chunk in 32-element K blocks (DMT_TF32_KCHUNK overrides;
// measured: tools/fp32_accuracy.py)
static int tf32_kchunk() {
  static int kc = [] {
    const char* e = getenv("DMT_TF32_KCHUNK");
    int v = e ? atoi(e) : 4;
    return v > 0 ? v : 1 << 30;
  }();
  return kc;
}

template <int BN, int NOPS, int KIND, int STAGES, typename TIN, typename TO, bool AMN, bool BMN, bool FEAT,
          int CL = 1>
static int launch(const dmt_gemm_args* a, const void* a_lo, const void* b_lo, cudaStream_t s) {
  constexpr int NSETS = (NOPS == 3) ? 2 : 1;
  constexpr int STAGE_BYTES = NSETS * (kBlockM + BN / CL) * kAtomBytes;
  constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ +
                          (size_t)kEpiWarps * kStileFloats * 4 /*epilogue staging*/;
  static_assert(SMEM <= 232448, "smem");
  CUtensorMap ma, mb, mal, mbl;
  if (!make_map(&ma, a->a, a->m, a->k, a->lda, a->in_dtype, kBlockM, AMN)) return DMT_ERR_CUDA;
  // 2-CTA clusters: a K-major B box covers the CTA's half of the tile rows
  if (!make_map(&mb, a->b, a->n, a->k, a->ldb, a->in_dtype, (CL > 1 && !BMN) ? BN / CL : BN, BMN))
    return DMT_ERR_CUDA;
  if (NSETS == 2) {
    if (!make_map(&mal, a_lo, a->m, a->k, a->lda, a->in_dtype, kBlockM, AMN)) return DMT_ERR_CUDA;
    if (!make_map(&mbl, b_lo, a->n, a->k, a->ldb, a->in_dtype, BN, BMN)) return DMT_ERR_CUDA;
  } else {
    mal = ma;
    mbl = mb;
  }
  Params p;
  p.m = a->m; p.n = a->n; p.k = a->k;
  p.ld_d = a->ld_d; p.ld_x = a->ld_x;
  p.rows_per_group = a->rows_per_group > 0 ? a->rows_per_group : a->m + 1;
  p.ld_group = a->ld_group;
  p.d = a->d; p.bias = a->bias; p.x0 = a->x0; p.xl = a->xl; p.aux = a->aux;
  p.c = a->c ? a->c : a->d;
  p.aux2 = a->aux2;
  p.npairs = a->npairs;
  for (int j = 0; j < DMT_GEMM_MAX_PAIRS; ++j) {
    p.pg[j] = j < a->npairs ? a->pair_g[j] : nullptr;
    p.pu[j] = j < a->npairs ? a->pair_u[j] : nullptr;
  }
  p.colsum = a->colsum_part;
  p.aux2_accum = (a->flags & DMT_GEMM_AUX2_ACCUM) != 0;
  p.scale_acc = (a->flags & DMT_GEMM_SCALE_ACC) != 0;
  p.alpha = a->alpha;
  p.kchunk = tf32_kchunk();
  {
    static const int dbg = [] {
      const char* e = getenv("DMT_GEMM_DBG");
      return e ? atoi(e) : 0;
    }();
    p.dbg = dbg;
    // per-lane L2 prefetch of the staged epilogue's operands two slabs ahead:
    // pays only on DCN_FINAL, whose fp32 dx0 operand doubles the bytes per
    // piece (8192 x 3328 x 3328: 151 -> 137 us; CROSS / DCN_BWD / ACC +1-5 %,
    // tools/gemm_bench.py).  DMT_EPI_PF_AHEAD=n forces n slabs (0 = off).
    static const int pfa = [] {
      const char* e = getenv("DMT_EPI_PF_AHEAD");
      return e ? atoi(e) : -1;
    }();
    p.pf_ahead = pfa >= 0 ? pfa : ((a->epilogue == DMT_EPI_DCN_FINAL && a->aux2 && a->npairs == 0) ? 2 : 0);
  }
  {
    const int num_kb = (int)ceil_div(a->k * (int64_t)sizeof(TIN), kAtomBytes);
    p.ksplit = a->ksplit > 1 ? a->ksplit : 1;
    p.kbs = (int)ceil_div(num_kb, p.ksplit);
    if constexpr (CL > 1) {
      if (p.ksplit > 1) return DMT_ERR_UNSUPPORTED;
    }
  }
  p.beta = a->beta; p.out_dtype = a->out_dtype; p.in_dtype = a->in_dtype; p.epilogue = a->epilogue;
  size_t eo = dtype_size(a->out_dtype);
  p.vec_store = ((uintptr_t)a->d % 16 == 0) && ((a->ld_d * eo) % 16 == 0) && ((a->ld_group * eo) % 16 == 0);
  p.ngroups_out = a->n_out_groups;
  p.ncolg = a->n_col_groups;
  p.colg_w = a->col_group_width > 0 ? a->col_group_width : 1;
  for (int j = 0; j < DMT_GEMM_MAX_COL_GROUPS; ++j) {
    p.colg[j] = j < a->n_col_groups ? a->col_group[j] : nullptr;
    p.colg_ld[j] = j < a->n_col_groups ? a->col_group_ld[j] : 0;
    if (j < a->n_col_groups)
      p.vec_store = p.vec_store && ((uintptr_t)a->col_group[j] % 16 == 0) && ((a->col_group_ld[j] * eo) % 16 == 0);
  }
  for (int j = 0; j < DMT_GEMM_MAX_OUT_GROUPS; ++j) {
    p.gout[j] = j < a->n_out_groups ? a->out_group[j] : nullptr;
    if (j < a->n_out_groups) p.vec_store = p.vec_store && ((uintptr_t)a->out_group[j] % 16 == 0);
  }
  size_t ei = dtype_size(a->in_dtype);
  p.vec_x = ((uintptr_t)a->x0 % 16 == 0) && ((uintptr_t)a->xl % 16 == 0) && ((uintptr_t)a->aux % 16 == 0) &&
            ((uintptr_t)a->aux2 % 16 == 0) && ((a->ld_x * ei) % 16 == 0) && ((a->ld_x * 4) % 16 == 0);
  for (int j = 0; j < a->npairs; ++j)
    p.vec_x = p.vec_x && ((uintptr_t)a->pair_g[j] % 16 == 0) && ((uintptr_t)a->pair_u[j] % 16 == 0);
  p.vec_store = p.vec_store && ((uintptr_t)p.c % 16 == 0);
  const bool needs_x = a->epilogue == DMT_EPI_CROSS || a->epilogue == DMT_EPI_DCN_BWD ||
                       a->epilogue == DMT_EPI_DCN_FINAL || a->epilogue == DMT_EPI_RELU_BWD;
  p.coalesced = p.vec_store && (!needs_x || p.vec_x);
  {
    // register-direct epilogue with TMA-stored outputs for epilogues that read
    // nothing from global memory (NONE / BIAS / BIAS_RELU / ACC with beta 0):
    // per-lane row loads of x0 / u / C are slower than the staged path's
    // coalesced ones (tools/gemm_bench.py).  DMT_GEMM_EPI=staged turns it off.
    static const bool staged = [] {
      const char* e = getenv("DMT_GEMM_EPI");
      return e && std::string(e) == "staged";
    }();
    const bool loads = needs_x || a->aux || a->aux2 ||
                       (a->beta != 0.f && (a->epilogue == DMT_EPI_ACC || a->epilogue == DMT_EPI_DCN_BWD ||
                                           a->epilogue == DMT_EPI_DCN_FINAL));
    p.direct = !staged && !loads;
  }
  // fused bias-gradient column sums: every 32-column chunk must take a
  // coalesced epilogue path (n % 32 == 0) with 16-byte partial-row stores
  if (p.colsum && (!p.coalesced || a->n % 32 || ((uintptr_t)p.colsum % 16) || a->epilogue != DMT_EPI_DCN_BWD))
    return DMT_ERR_UNSUPPORTED;
  // L2 prefetch of epilogue inputs: 16-byte aligned rows only (bulk copy rule)
  const bool plain_rows = p.rows_per_group > a->m;
  p.prefetch = 0;
  // Measured (tools/gemm_bench.py, B200): the prefetch pays only for the
  // crossnet forward on 192-wide tiles (-5 %); on the DCN-backward epilogues
  // and 256-wide tiles the extra TMA / L2 traffic costs more than the latency
  // it hides (+3..15 %), so those are left to the register-pipelined loads.
  (void)plain_rows;
  if (p.vec_x && a->epilogue == DMT_EPI_CROSS && BN <= 192) p.prefetch |= 1 | 2;
  {
    // experiment override: DMT_EPI_PREFETCH = bit mask (1 x0, 2 xl/u, 4 C, 8 dx0)
    static const int forced = [] {
      const char* e = getenv("DMT_EPI_PREFETCH");
      return e ? atoi(e) : -1;
    }();
    if (forced >= 0 && p.vec_x) {
      int m = 0;
      if (needs_x || a->epilogue == DMT_EPI_RELU_BWD) m |= forced & 1;
      if (a->epilogue == DMT_EPI_CROSS || (a->epilogue == DMT_EPI_DCN_BWD && a->aux2)) m |= forced & 2;
      if ((a->epilogue == DMT_EPI_ACC || a->epilogue == DMT_EPI_DCN_BWD || a->epilogue == DMT_EPI_DCN_FINAL) &&
          a->beta != 0.f)
        m |= forced & 4;
      if (a->aux2 && (a->epilogue == DMT_EPI_DCN_FINAL || (a->flags & DMT_GEMM_AUX2_ACCUM))) m |= forced & 8;
      p.prefetch = m;
    }
  }
  if (a->flags & DMT_GEMM_NO_PREFETCH) p.prefetch = 0;
  EpiMaps em;
  memset(&em, 0, sizeof(em));
  if (p.prefetch) {
    const int bc = BN;  // box inner dim <= 256 elements
    bool ok = true;
    if (p.prefetch & 1) ok = ok && make_plain_map(&em.x0, a->x0, a->m, a->n, a->ld_x, a->in_dtype, bc, kBlockM);
    if (p.prefetch & 2) ok = ok && make_plain_map(&em.xl, a->xl, a->m, a->n, a->ld_x, a->in_dtype, bc, kBlockM);
    if (p.prefetch & 4) ok = ok && make_plain_map(&em.c, p.c, a->m, a->n, a->ld_d, a->out_dtype, bc, kBlockM);
    if (p.prefetch & 8) ok = ok && make_plain_map(&em.d2, a->aux2, a->m, a->n, a->ld_x, DMT_F32, bc, kBlockM);
    if (!ok) p.prefetch = 0;  // a hint only: skip it when a block cannot be described
  }
  // direct-path TMA stores: plain row-major output (no grouped / scattered
  // layouts, no split-K workspace)
  p.tma_out = 0;
  if (p.direct && p.ksplit == 1 && !p.ngroups_out && !p.ncolg && p.rows_per_group > a->m && !(a->flags & DMT_GEMM_NO_TMA_STORE)) {
    if (make_plain_map(&em.od, a->d, a->m, a->n, a->ld_d, a->out_dtype, 32, 32)) p.tma_out |= 1;
    static const bool wide = [] {
      const char* e = getenv("DMT_GEMM_TMA64");
      return !e || atoi(e) != 0;
    }();
    if ((p.tma_out & 1) && wide && sizeof(TO) == 2 &&
        make_plain_map(&em.od64, a->d, a->m, a->n, a->ld_d, a->out_dtype, 64, 32))
      p.tma_out |= 2;
  }
  if (a->bias && ((uintptr_t)a->bias % 16)) return DMT_ERR_UNSUPPORTED;
  auto kern = gemm_kernel<BN, NOPS, KIND, STAGES, TIN, TO, AMN, BMN, FEAT, CL>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
    if (e != cudaSuccess) {
      set_last_error(e);
      return DMT_ERR_CUDA;
    }
    attr_set = true;
  }
  int64_t tiles = ceil_div(a->m, kBlockM) * ceil_div(a->n, BN) * p.ksplit;
  const int fmt = (KIND == 1) ? 2 : (std::is_same<TIN, __half>::value ? 0 : 1);
  uint32_t idesc = make_idesc(fmt, kBlockM * CL, BN, AMN, BMN);  // pair: M = 256
  if constexpr (CL == 1) {
    int grid = (int)std::min<int64_t>(tiles, DMT_NUM_SMS);
    kern<<<grid, kThreads, SMEM, s>>>(ma, mb, mal, mbl, em, p, idesc);
  } else {
    // persistent over co-resident clusters only (GPCs with an odd SM count
    // cannot host a full pair on every SM)
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static int max_clusters = 0;
    if (!max_clusters) {
      cfg.gridDim = dim3(DMT_NUM_SMS / CL * CL);
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) n = DMT_NUM_SMS / CL;
      max_clusters = n;
    }
    const int64_t units = ceil_div(a->m, (int64_t)kBlockM * CL) * ceil_div(a->n, (int64_t)BN);
    cfg.gridDim = dim3((unsigned)(std::min<int64_t>(units, max_clusters) * CL));
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, mal, mbl, em, p, idesc);
    if (e != cudaSuccess) {
      set_last_error(e);
      return DMT_ERR_CUDA;
    }
  }
  DMT_CHECK_LAUNCH();
  return DMT_OK;
}

// Tile width for 16-bit operands.  The persistent grid runs ceil(tiles / 148)
// waves, each as long as one tile's mainloop (~BN) plus a fixed per-tile cost
// (~kTileOverheadCols columns' worth: pipeline fill, accumulator hand-off), so
// pick the BN minimising waves * (BN + overhead).  E.g. 16384 x 1664: BN 256
// -> 7 tile columns (the last half empty) = 896 tiles = 7 waves; BN 192 -> 8
// waves of 3/4-width tiles (17 % less); dW 1664 x 1664: 91 tiles of 256 leave
// 57 SMs idle, 117 tiles of 192 are one 25 % shorter wave.
constexpr int64_t kTileOverheadCols = 32;
static int pick_bn(int64_t m, int64_t n, int flags) {
  if (flags & DMT_GEMM_BN_MASK) return 64 * ((flags & DMT_GEMM_BN_MASK) >> DMT_GEMM_BN_SHIFT);
  if (n <= 64) return 64;
  const int cand[4] = {256, 192, 128, 64};
  int best = 256;
  int64_t best_cost = INT64_MAX;
  for (int bn : cand) {
    if (bn == 64 && n > 512) continue;  // narrow tiles re-read A too often
    const int64_t tiles = ceil_div(m, kBlockM) * ceil_div(n, (int64_t)bn);
    // narrow tiles are bound by the shared-memory operand bandwidth of the
    // single-CTA MMA (A + B bytes per flop grow as BN shrinks): measured
    // ~1.2x the per-column time at BN 128 and ~1.5x at BN 64
    const int64_t eff = bn == 128 ? 154 : (bn == 64 ? 96 : bn);
    const int64_t cost = ceil_div(tiles, (int64_t)DMT_NUM_SMS) * (eff + kTileOverheadCols);
    if (cost < best_cost) {
      best_cost = cost;
      best = bn;
    }
  }
  return best;
}

template <typename TIN, typename TO, bool AMN, bool BMN, bool FEAT>
static int dispatch_n(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s) {
  if constexpr (std::is_same<TIN, float>::value) {
    if (a->n <= 64) return launch<64, 3, 1, 4, TIN, TO, AMN, BMN, FEAT>(a, alo, blo, s);
    return launch<128, 3, 1, 3, TIN, TO, AMN, BMN, FEAT>(a, alo, blo, s);
  } else {
    const int bn = pick_bn(a->m, a->n, a->flags);
    if constexpr (std::is_same<TIN, __nv_bfloat16>::value && !FEAT) {
      // cta_group::2 pairs (256 x BN tiles; each CTA holds half of B): BN 256,
      // or 192 with K-major B (an MN-major half must be whole 64-column atoms)
      // Measured (tools/gemm_bench.py, B200): pairs win on the 3328-wide T = 1
      // tower GEMMs (dW 190 -> 144-155 us, fused-SGD dW 164 -> 142, crossnet
      // 156 -> 148, DCN_BWD 183 -> 172) and are neutral or slower on the
      // 1664-wide ones, where the tile-width choice is BN 192.
      const bool pair_ok = (bn == 256 || (bn == 192 && !BMN)) && ceil_div(a->m, kBlockM) >= 2;
      const bool pair = pair_ok && !(a->flags & DMT_GEMM_SINGLE_CTA) &&
                        ((a->flags & DMT_GEMM_CLUSTER) || (bn == 256 && a->n >= 2048));
      if (pair) {
        // (6 stages fit too -- 231,680 B -- and measured no faster: the pair
        // mainloop is bound by L2 throughput, not by stage depth)
        if (bn == 256) return launch<256, 1, 0, 5, TIN, TO, AMN, BMN, FEAT, 2>(a, alo, blo, s);
        if constexpr (!BMN) return launch<192, 1, 0, 6, TIN, TO, AMN, BMN, FEAT, 2>(a, alo, blo, s);
      }
    }
    switch (bn) {
      case 64: return launch<64, 1, 0, 8, TIN, TO, AMN, BMN, FEAT>(a, alo, blo, s);
      case 128: return launch<128, 1, 0, 6, TIN, TO, AMN, BMN, FEAT>(a, alo, blo, s);
      case 192: return launch<192, 1, 0, 4, TIN, TO, AMN, BMN, FEAT>(a, alo, blo, s);
      default: return launch<256, 1, 0, 4, TIN, TO, AMN, BMN, FEAT>(a, alo, blo, s);
    }
  }
}

// One translation unit per operand-majorness combination (gemm_{kk,km,mk,mm}.cu)
// instantiates these, so the tile-width x dtype matrix compiles in parallel.
int gemm_major_kk(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s);
int gemm_major_km(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s);
int gemm_major_mk(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s);
int gemm_major_mm(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s);

// The FEAT variants exist only for the K-major A operand (the DCN dX GEMMs:
// B MN-major for 16-bit types, both K-major on the transposed fp32 path).
template <typename TIN, typename TO, bool AMN, bool BMN>
static int dispatch_f(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s) {
  const bool feat = a->npairs > 0 || a->colsum_part != nullptr;
  if constexpr (!AMN) {
    if (feat) return dispatch_n<TIN, TO, AMN, BMN, true>(a, alo, blo, s);
  } else {
    if (feat) return DMT_ERR_UNSUPPORTED;
  }
  return dispatch_n<TIN, TO, AMN, BMN, false>(a, alo, blo, s);
}

template <bool AMN, bool BMN>
static int dispatch_types(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s) {
  switch (a->in_dtype) {
    case DMT_BF16:
      switch (a->out_dtype) {
        case DMT_F32: return dispatch_f<__nv_bfloat16, float, AMN, BMN>(a, alo, blo, s);
        case DMT_BF16: return dispatch_f<__nv_bfloat16, __nv_bfloat16, AMN, BMN>(a, alo, blo, s);
        case DMT_F16: return dispatch_f<__nv_bfloat16, __half, AMN, BMN>(a, alo, blo, s);
        default: return DMT_ERR_UNSUPPORTED;
      }
    case DMT_F16:
      switch (a->out_dtype) {
        case DMT_F32: return dispatch_f<__half, float, AMN, BMN>(a, alo, blo, s);
        case DMT_BF16: return dispatch_f<__half, __nv_bfloat16, AMN, BMN>(a, alo, blo, s);
        case DMT_F16: return dispatch_f<__half, __half, AMN, BMN>(a, alo, blo, s);
        default: return DMT_ERR_UNSUPPORTED;
      }
    case DMT_F32:
      switch (a->out_dtype) {
        case DMT_F32: return dispatch_f<float, float, AMN, BMN>(a, alo, blo, s);
        case DMT_BF16: return dispatch_f<float, __nv_bfloat16, AMN, BMN>(a, alo, blo, s);
        case DMT_F16: return dispatch_f<float, __half, AMN, BMN>(a, alo, blo, s);
        default: return DMT_ERR_UNSUPPORTED;
      }
    default: return DMT_ERR_UNSUPPORTED;
  }
}

}  // namespace gemm
}  // namespace dmt

