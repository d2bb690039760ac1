// K4 CTA-pair kernel instantiations for A = F8, B = FU4 (see gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace fqg {
void gemm_pair_F8_FU4(const GemmArgs& g, const GemmPlan& p, cudaStream_t s) {
    dispatch_pair<F8, FU4>(g, p, s);
}
}  // namespace fqg
