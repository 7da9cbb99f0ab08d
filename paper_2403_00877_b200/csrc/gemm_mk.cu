// tcgen05 GEMM instantiations: A MN-major, B K-major (gemm_sm100.cuh)
#include "gemm_sm100.cuh"

namespace dmt {
namespace gemm {
int gemm_major_mk(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s) {
  return dispatch_types<true, false>(a, alo, blo, s);
}
}  // namespace gemm
}  // namespace dmt
