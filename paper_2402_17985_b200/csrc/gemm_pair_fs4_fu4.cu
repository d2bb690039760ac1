// K4 CTA-pair kernel instantiations for A = FS4, B = FU4 (see gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace fqg {
void gemm_pair_FS4_FU4(const GemmArgs& g, const GemmPlan& p, cudaStream_t s) {
    dispatch_pair<FS4, FU4>(g, p, s);
}
}  // namespace fqg
