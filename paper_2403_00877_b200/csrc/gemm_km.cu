// tcgen05 GEMM instantiations: A K-major, B MN-major (gemm_sm100.cuh)
#include "gemm_sm100.cuh"

namespace dmt {
namespace gemm {
int gemm_major_km(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s) {
  return dispatch_types<false, true>(a, alo, blo, s);
}
}  // namespace gemm
}  // namespace dmt
