// gemm.cu — K4 host side: the launch plan (tile shape, split-K) and the
// dispatch to the per-format kernel translation units (gemm_pair_*.cu,
// gemm_one_*.cu; the kernels themselves are in gemm_kernels.cuh).
#include "gemm_kernels.cuh"

namespace fqg {
void gemm_pair_F8_F8(const GemmArgs& g, const GemmPlan& p, cudaStream_t s);
void gemm_pair_F8_FS4(const GemmArgs& g, const GemmPlan& p, cudaStream_t s);
void gemm_pair_F8_FU4(const GemmArgs& g, const GemmPlan& p, cudaStream_t s);
void gemm_pair_FS4_F8(const GemmArgs& g, const GemmPlan& p, cudaStream_t s);
void gemm_pair_FS4_FS4(const GemmArgs& g, const GemmPlan& p, cudaStream_t s);
void gemm_pair_FS4_FU4(const GemmArgs& g, const GemmPlan& p, cudaStream_t s);
void gemm_one_F8(const GemmArgs& g, int bn, cudaStream_t s);
void gemm_one_FS4(const GemmArgs& g, int bn, cudaStream_t s);
void gemv_i8(const GemmArgs& g, const GemmPlan& p, cudaStream_t s);

namespace {
void dispatch_pair_fmt(const GemmArgs& g, const GemmPlan& p, cudaStream_t s) {
    const int af = kfmt(g.a_fmt), bf = kfmt(g.b_fmt);
    if (af == F8 && bf == F8) return gemm_pair_F8_F8(g, p, s);
    if (af == F8 && bf == FS4) return gemm_pair_F8_FS4(g, p, s);
    if (af == F8 && bf == FU4) return gemm_pair_F8_FU4(g, p, s);
    if (af == FS4 && bf == F8) return gemm_pair_FS4_F8(g, p, s);
    if (af == FS4 && bf == FS4) return gemm_pair_FS4_FS4(g, p, s);
    return gemm_pair_FS4_FU4(g, p, s);
}
}  // namespace


void make_tmap_2d_u8(CUtensorMap* map, const void* base, uint64_t inner_bytes, uint64_t rows,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_rows,
                     CUtensorMapSwizzle swz) {
    require(reinterpret_cast<uintptr_t>(base) % 16 == 0, "tma: base must be 16-byte aligned");
    require(row_stride_bytes % 16 == 0, "tma: row stride must be a multiple of 16 bytes");
    const cuuint64_t dims[2] = {inner_bytes, rows};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box_inner, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r =
        encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw Error(FQG_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
}

void gemm_i8(const GemmArgs& g, cudaStream_t stream) {
    require(g.m >= 1 && g.n >= 1 && g.kp >= 1, "gemm: empty shape");
    require(g.m < (1ll << 31) && g.n < (1ll << 31), "gemm: shape too large");
    require(g.a_fmt == FQG_I8 || g.a_fmt == FQG_I4, "gemm: operand A must be I8 or I4");
    require(g.b_fmt == FQG_I8 || g.b_fmt == FQG_I4 || g.b_fmt == FQG_I4_BIASED,
            "gemm: operand B must be I8 or I4");
    require(g.b_fmt != FQG_I4_BIASED || g.rowsum != nullptr,
            "gemm: biased int4 weights need the operand row sums");
    require(g.kp % 32 == 0, "gemm: K' must be a multiple of 32");
    // INT32 exactness: |acc| <= K' * 127 * 127 must stay below 2^31.
    require(g.kp * 127ll * 127ll < (1ll << 31), "gemm: K' too large for exact INT32 accumulation");
    int dev = 0;
    FQG_CUDA(cudaGetDevice(&dev));
    const GemmPlan p = plan_gemm(g.m, g.n, g.kp, g.a_fmt, g.b_fmt, g.variant, num_sms(dev));
    if (p.kernel == 3)
        gemv_i8(g, p, stream);
    else if (p.kernel == 2)
        dispatch_pair_fmt(g, p, stream);
    else if (kfmt(g.a_fmt) == F8)
        gemm_one_F8(g, p.tile_n, stream);
    else
        gemm_one_FS4(g, p.tile_n, stream);
}

GemmPlan plan_gemm(int64_t m, int64_t n, int64_t kp, int a_fmt, int b_fmt, int variant, int sms) {
    // variant: 0 auto, 1 single-CTA 128 x BN tiles, 2 CTA-pair kernel.
    // FQG_GEMM_VARIANT / FQG_GEMM_NB override auto (tuning experiments).
    static const int env_variant = [] {
        const char* e = std::getenv("FQG_GEMM_VARIANT");
        return e ? std::atoi(e) : 0;
    }();
    static const int nb_env = [] {
        const char* e = std::getenv("FQG_GEMM_NB");
        return e ? std::atoi(e) : 0;
    }();
    GemmPlan p{};
    int v = variant != 0 ? variant : env_variant;
    // Measured at 2048 x 4096 x 7488: pair 61 us (int8 weights) / 71 us (biased
    // int4), single-CTA 71 us (int4); a weights-in-TMEM variant (unpacked int4
    // weights as the MMA's A operand in TMEM) measured 79-87 us and was removed.
    // The pair kernel also for small M: its split-K spreads the weight stream over
    // the CTA pairs (M = 1 at 8192^2: 61 us on 32 single CTAs before).
    // Decode-size M (1-2 rows, int8 operands): the weight stream on CUDA cores (gemv.cu).
    if ((v == 0 || v == 3) && m <= 2 && a_fmt == FQG_I8 && b_fmt == FQG_I8) {
        p.kernel = 3;
        p.tile_m = 2;
        p.tile_n = 4;  // output columns per warp pass
        const int64_t groups = (n + 3) / 4;  // 4-column groups, spread over the CTAs
        p.ctas = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(groups, 4 * sms)));
        return p;
    }
    if (v == 0) v = (n > 128 && a_fmt == FQG_I8) ? 2 : 1;
    const int64_t num_kb = (kp + BK - 1) / BK;
    if (v == 2) {
        p.kernel = 2;
        // 256 x 512 tiles (NB = 2) need enough tiles to fill the CTA pairs;
        // otherwise 256 x 256 (plus split-K when even those are few).
        const int64_t t2 = ((m + 255) / 256) * ((n + 511) / 512);
        int nb = nb_env ? nb_env : (n >= 512 && t2 >= 48 ? 2 : 1);
        // Packed (int4) weights: 512 x 256 tiles (nb = 3) instead of 256 x 512, which
        // halve the expanded B tile per MAC (the int4 main loop is bound by shared-
        // memory bandwidth, gemm_kernels.cuh PairLayout).
        const bool packed_b = b_fmt == FQG_I4 || b_fmt == FQG_I4_BIASED;
        const int64_t t3 = ((m + 511) / 512) * ((n + 255) / 256);
        if (!nb_env && nb == 2 && packed_b && m >= 512 && t3 >= 48) nb = 3;
        p.tile_m = nb == 3 ? 512 : 2 * BM;
        p.tile_n = nb == 3 ? 256 : 256 * nb;
        const int64_t tiles = ((m + p.tile_m - 1) / p.tile_m) * ((n + p.tile_n - 1) / p.tile_n);
        const int64_t pairs = std::max(1, sms / 2);
        // Split-K for small M: fewer than half the pairs would have a tile.
        if (nb == 1 && 2 * tiles <= pairs && num_kb >= 8) {
            const int64_t sp = std::min<int64_t>({pairs / tiles, num_kb / 4, 8});
            if (sp >= 2) p.splits = static_cast<int>(sp);
        }
        p.ctas = static_cast<int>(2 * (p.splits >= 2 ? tiles * p.splits
                                                     : std::max<int64_t>(1, std::min(tiles, pairs))));
    } else {
        p.kernel = 1;
        p.tile_m = BM;
        p.tile_n = n <= 128 ? 128 : 256;
        const int64_t tiles = ((m + BM - 1) / BM) * ((n + p.tile_n - 1) / p.tile_n);
        p.ctas = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(tiles, sms)));
    }
    return p;
}

}  // namespace fqg

