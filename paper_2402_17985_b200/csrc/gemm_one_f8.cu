// K4 single-CTA kernel instantiations for A = F8 (see gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace fqg {
void gemm_one_F8(const GemmArgs& g, int bn, cudaStream_t s) {
    const int bf = kfmt(g.b_fmt);
    if (bn == 128) {
        if (bf == F8) return dispatch_out<128, F8, F8>(g, s);
        if (bf == FS4) return dispatch_out<128, F8, FS4>(g, s);
        return dispatch_out<128, F8, FU4>(g, s);
    }
    if (bf == F8) return dispatch_out<256, F8, F8>(g, s);
    if (bf == FS4) return dispatch_out<256, F8, FS4>(g, s);
    return dispatch_out<256, F8, FU4>(g, s);
}
}  // namespace fqg
