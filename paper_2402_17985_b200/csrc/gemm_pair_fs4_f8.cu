// K4 CTA-pair kernel instantiations for A = FS4, B = F8 (see gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace fqg {
void gemm_pair_FS4_F8(const GemmArgs& g, const GemmPlan& p, cudaStream_t s) {
    dispatch_pair<FS4, F8>(g, p, s);
}
}  // namespace fqg
