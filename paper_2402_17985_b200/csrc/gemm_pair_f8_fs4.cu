// K4 CTA-pair kernel instantiations for A = F8, B = FS4 (see gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace fqg {
void gemm_pair_F8_FS4(const GemmArgs& g, const GemmPlan& p, cudaStream_t s) {
    dispatch_pair<F8, FS4>(g, p, s);
}
}  // namespace fqg
