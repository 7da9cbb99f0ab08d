// tcgen05 GEMM instantiations: A MN-major, B MN-major (gemm_sm100.cuh)
#include "gemm_sm100.cuh"

namespace dmt {
namespace gemm {
int gemm_major_mm(const dmt_gemm_args* a, const void* alo, const void* blo, cudaStream_t s) {
  return dispatch_types<true, true>(a, alo, blo, s);
}
}  // namespace gemm
}  // namespace dmt
