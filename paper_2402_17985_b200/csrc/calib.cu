// calib.cu — fq::quantize_layer (pipeline.cpp:76-152, modes O1/O2) with its
// scans on the device: the calibration statistics
// (collect_channel_maxes, calibration.cpp:9-28), the weight row maxima, and the
// KL bit-width selection (select_bit_width, quantize.cpp:145-158) over the
// flattened calibration activations and the flattened weight.
//
// Exactness. Every value the reference histograms is recomputed on the device
// with the same IEEE FP64 operations: x / s_j (divide_columns, smoothing.cpp:75),
// the saturating / strict splits (split.cuh, flatten.cpp:8-15,60-74), W * s_j
// (scale_rows, smoothing.cpp:88), q = clamp(round(v / scale)) and q * scale
// (quantize.cpp:44-45, dequantize :50-56), and the bin index
// floor((v - lo) / width) (build_histogram, quantize.cpp:85-110). Maxima are
// exact; bin counts are integers. The host then forms the normalized
// distributions and the KL sums in the reference's order with the same libm,
// so the ratios and the chosen bits equal the reference's bit for bit. The
// plan stages between the scans (smoothing scales, boxplot truncation,
// build_flatten_plan) are host arithmetic on K values (host.cu).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "fqg_internal.h"
#include "gptq.h"
#include "host.h"
#include "split.cuh"

namespace fqg {
namespace {

using namespace split;

constexpr int kThreads = 256;

// Value sources: element (row, col) of the tensor the reference histograms.
struct ActSrc {  // vstack of repeat_columns(flatten_tensor(divide_columns(calib)))
    const double* x;  // [rows][k]
    int64_t ldx;
    const int32_t* amap;  // [kp] j << 12 | piece, or -1
    const double* s;
    const int32_t* cap;   // [k] plan_x capacity
    double t, rt;
    int64_t cols;         // kp
    bool strict = false;
    __device__ double operator()(int64_t row, int64_t col, bool& over) const {
        const int32_t mp = amap[col];
        if (mp < 0) return 0.0;
        const int j = mp >> 12, p = mp & 0xFFF;
        const double v = __ddiv_rn(x[row * ldx + j], s[j]);  // smoothing.cpp:75
        const Split sp = split_elem(v, t, rt, cap[j]);
        over |= sp.sat;
        return p < sp.cnt ? (sp.neg ? -t : t) : (p == sp.cnt ? (sp.neg ? -sp.rem : sp.rem) : 0.0);
    }
};
struct WgtSrc {  // flatten_rows(repeat_channels(scale_rows(W, s)), plan_w), strict
    const double* w;  // [k][n]
    int64_t n;
    const int32_t* wmap;  // [kp] j << 12 | piece, or -1
    const int32_t* wcap;  // [kp] plan_w capacity
    const double* s;
    double t, rt;
    int64_t cols;         // n
    __device__ double operator()(int64_t row, int64_t col, bool& over) const {
        const int32_t mp = wmap[row];
        if (mp < 0) return 0.0;
        const int j = mp >> 12, p = mp & 0xFFF;
        const double v = __dmul_rn(w[static_cast<int64_t>(j) * n + col], s[j]);  // smoothing.cpp:88
        const Split sp = split_elem(v, t, rt, wcap[row]);
        over |= sp.sat;
        return p < sp.cnt ? (sp.neg ? -t : t) : (p == sp.cnt ? (sp.neg ? -sp.rem : sp.rem) : 0.0);
    }
};

// Column / row absmax of a plain matrix (collect_channel_maxes, row_max_abs).
__global__ void __launch_bounds__(kThreads) k_col_absmax(const double* __restrict__ x, int64_t rows,
                                                         int64_t cols, unsigned long long* out) {
    for (int64_t c = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; c < cols;
         c += static_cast<int64_t>(gridDim.x) * kThreads) {
        double mx = 0.0;
        for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) mx = fmax(mx, fabs(x[r * cols + c]));
        atomicMax(out + c, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
}
__global__ void __launch_bounds__(kThreads) k_row_absmax(const double* __restrict__ x, int64_t cols,
                                                         unsigned long long* out) {
    __shared__ double red[kThreads / 32];
    const int64_t r = blockIdx.x;
    double mx = 0.0;
    for (int64_t c = threadIdx.x; c < cols; c += kThreads) mx = fmax(mx, fabs(x[r * cols + c]));
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kThreads / 32; ++w) mx = fmax(mx, red[w]);
        out[r] = static_cast<unsigned long long>(__double_as_longlong(mx));
    }
}

// Pass 0: max |v| over the tensor (and the strict-capacity overflow flag).
template <class Src>
__global__ void __launch_bounds__(kThreads) k_src_absmax(Src src, int64_t rows,
                                                         unsigned long long* amax,
                                                         unsigned int* overflow) {
    __shared__ double red[kThreads / 32];
    double mx = 0.0;
    bool over = false;
    const int64_t total = rows * src.cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * kThreads)
        mx = fmax(mx, fabs(src(i / src.cols, i % src.cols, over)));
    if (__any_sync(0xffffffffu, over) && (threadIdx.x & 31) == 0) atomicOr(overflow, 1u);
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kThreads / 32; ++w) mx = fmax(mx, red[w]);
        atomicMax(amax, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
}

// build_histogram's bin (quantize.cpp:99-103): floor((v - lo) / width), clamped.
__device__ __forceinline__ int bin_of(double v, double lo, double width, int bins) {
    const double u = floor(__ddiv_rn(__dsub_rn(v, lo), width));
    return u < 0.0 ? 0 : (u > static_cast<double>(bins - 1) ? bins - 1 : static_cast<int>(u));
}
// quantize_per_tensor without override (quantize.cpp:34-47) then dequantize (:50-56).
__device__ __forceinline__ double round_trip(double v, double scale, double qmax) {
    double r = round(__ddiv_rn(v, scale));
    r = r < -qmax ? -qmax : (qmax < r ? qmax : r);
    return __dmul_rn(r, scale);
}

// Pass 1: the three histograms of divergence_ratio (quantize.cpp:136-144) on the
// layout [-mx, mx]: P of the values, Q4 / Q8 of their INT4 / INT8 round trips.
template <class Src>
__global__ void __launch_bounds__(kThreads) k_src_hist(Src src, int64_t rows, double mx, int bins,
                                                       unsigned long long* __restrict__ hist) {
    extern __shared__ unsigned int sh[];  // [3][bins]
    for (int i = threadIdx.x; i < 3 * bins; i += kThreads) sh[i] = 0u;
    __syncthreads();
    const double lo = -mx, width = __ddiv_rn(__dsub_rn(mx, lo), static_cast<double>(bins));
    const double s4 = __ddiv_rn(mx, 7.0), s8 = __ddiv_rn(mx, 127.0);
    const int64_t total = rows * src.cols;
    bool over = false;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * kThreads) {
        const double v = src(i / src.cols, i % src.cols, over);
        atomicAdd(&sh[bin_of(v, lo, width, bins)], 1u);
        atomicAdd(&sh[bins + bin_of(round_trip(v, s4, 7.0), lo, width, bins)], 1u);
        atomicAdd(&sh[2 * bins + bin_of(round_trip(v, s8, 127.0), lo, width, bins)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * bins; i += kThreads)
        if (sh[i]) atomicAdd(hist + i, static_cast<unsigned long long>(sh[i]));
}

// The tensor itself, row-major (the O3 path's GEMM-like operands).
template <class Src>
__global__ void __launch_bounds__(kThreads) k_src_materialize(Src src, int64_t rows,
                                                              double* __restrict__ out) {
    bool over = false;
    const int64_t total = rows * src.cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * kThreads)
        out[i] = src(i / src.cols, i % src.cols, over);
}

int grid_for(int64_t work, int sms) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((work + kThreads - 1) / kThreads,
                                                                    8LL * sms)));
}

template <class Src>
void scan(const Src& src, int64_t rows, int bins, int sms, double* mx, bool* overflow,
          std::vector<unsigned long long>* hist) {
    unsigned long long* d = nullptr;  // [amax, overflow, 3 * bins counts]
    const size_t bytes = (2 + 3 * static_cast<size_t>(bins)) * 8;
    FQG_CUDA(cudaMalloc(&d, bytes));
    struct Free {
        void* p;
        ~Free() { cudaFree(p); }
    } fr{d};
    FQG_CUDA(cudaMemset(d, 0, bytes));
    const int grid = grid_for(rows * src.cols, sms);
    k_src_absmax<Src><<<grid, kThreads>>>(src, rows, d, reinterpret_cast<unsigned int*>(d + 1));
    FQG_CUDA(cudaGetLastError());
    unsigned long long h2[2];
    FQG_CUDA(cudaMemcpy(h2, d, 16, cudaMemcpyDeviceToHost));
    std::memcpy(mx, &h2[0], 8);
    *overflow = (h2[1] & 0xFFFFFFFFull) != 0;
    hist->assign(3 * static_cast<size_t>(bins), 0);
    if (*mx == 0.0 || hist->empty()) return;
    const size_t smem = 3 * static_cast<size_t>(bins) * 4;
    require(smem <= 200 * 1024, "calibrate: too many histogram bins");
    FQG_CUDA(cudaFuncSetAttribute(k_src_hist<Src>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    k_src_hist<Src><<<grid, kThreads, smem>>>(src, rows, *mx, bins, d + 2);
    FQG_CUDA(cudaGetLastError());
    FQG_CUDA(cudaMemcpy(hist->data(), d + 2, hist->size() * 8, cudaMemcpyDeviceToHost));
}

// build_histogram's normalization (quantize.cpp:104-110) and kl_divergence
// (:112-121), in the reference's order.
std::vector<double> normalized(const unsigned long long* counts, int bins, double total) {
    constexpr double kHistogramEps = 1e-10;  // quantize.cpp:12
    std::vector<double> p(static_cast<size_t>(bins));
    double norm = 0.0;
    for (int i = 0; i < bins; ++i) {
        p[i] = static_cast<double>(counts[i]) / total + kHistogramEps;
        norm += p[i];
    }
    for (double& v : p) v /= norm;
    return p;
}
double kl(const std::vector<double>& p, const std::vector<double>& q) {
    double d = 0.0;
    for (size_t i = 0; i < p.size(); ++i) d += p[i] * std::log(p[i] / q[i]);
    return std::max(d, 0.0);
}
// divergence_ratio (quantize.cpp:136-144): KL(P, Q4) / max(KL(P, Q8), 1e-12); 0 for a zero tensor.
double divergence_ratio(double mx, const std::vector<unsigned long long>& h, int bins, double total) {
    constexpr double kKlFloor = 1e-12;  // quantize.cpp:13
    if (mx == 0.0) return 0.0;
    const auto p = normalized(h.data(), bins, total);
    const auto q4 = normalized(h.data() + bins, bins, total);
    const auto q8 = normalized(h.data() + 2 * bins, bins, total);
    return kl(p, q4) / std::max(kl(p, q8), kKlFloor);
}

template <class T>
T* upload(const std::vector<T>& v, std::vector<void*>& keep) {
    void* p = nullptr;
    FQG_CUDA(cudaMalloc(&p, std::max<size_t>(16, v.size() * sizeof(T))));
    keep.push_back(p);
    FQG_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return static_cast<T*>(p);
}

}  // namespace
}  // namespace fqg

struct fqg_recipe_s {
    int bits = 8;
    int64_t k = 0, n = 0, block = 32;
    std::vector<double> s;
    double t_x = 0, t_w = 0, act_scale = 0, w_scale = 0, kl_act = 0, kl_w = 0;
    std::vector<int64_t> e_x, e_w;
    std::vector<int32_t> weight_q;  // O3: GPTQ weight_q [K'][N]
};

using namespace fqg;

extern "C" {

void fqg_quant_options_default(fqg_quant_options* o) {
    // pipeline.hpp:24-34 (QuantOptions)
    *o = fqg_quant_options{2, 0.5, 1.3, 1.86, 32, 2048, 1, 1, 0.01};
}

int fqg_calibrate(const double* weight, int64_t k, int64_t n, const double* calib, int64_t samples,
                  int64_t rows, const fqg_quant_options* o, int device, fqg_recipe_t* out) {
    return guard([&] {
        require(weight && calib && o && out, "calibrate: null argument");
        require(k >= 1 && n >= 1 && samples >= 1 && rows >= 1,
                "quantize_layer: empty calibration set");
        require(o->mode >= 1 && o->mode <= 3, "calibrate: mode must be O1 (1), O2 (2) or O3 (3)");
        require(o->gamma >= 0.0, "select_bit_width: gamma must be >= 0");
        require(o->bins >= 16, "build_histogram: bin_count < 16");
        int prev = -1;
        FQG_CUDA(cudaGetDevice(&prev));
        FQG_CUDA(cudaSetDevice(device));
        std::vector<void*> keep;
        struct Free {
            std::vector<void*>& v;
            int dev;
            ~Free() {
                for (void* p : v) cudaFree(p);
                if (dev >= 0) cudaSetDevice(dev);
            }
        } fr{keep, prev};
        const int sms = num_sms(device);
        const int64_t m = samples * rows;
        // the calibration samples stacked [samples * rows][k] (collect_channel_maxes
        // walks every sample row), and W [k][n]
        const double* dx = upload(std::vector<double>(calib, calib + m * k), keep);
        const double* dw = upload(std::vector<double>(weight, weight + k * n), keep);
        std::vector<unsigned long long> bits_max(static_cast<size_t>(k), 0);
        unsigned long long* dmax = upload(bits_max, keep);
        k_col_absmax<<<dim3(static_cast<unsigned>((k + kThreads - 1) / kThreads),
                            static_cast<unsigned>(std::min<int64_t>(m, 64))),
                       kThreads>>>(dx, m, k, dmax);
        FQG_CUDA(cudaGetLastError());
        std::vector<double> act_max(k), wmax(k);
        FQG_CUDA(cudaMemcpy(act_max.data(), dmax, k * 8, cudaMemcpyDeviceToHost));
        k_row_absmax<<<static_cast<unsigned>(k), kThreads>>>(dw, n, dmax);
        FQG_CUDA(cudaGetLastError());
        FQG_CUDA(cudaMemcpy(wmax.data(), dmax, k * 8, cudaMemcpyDeviceToHost));

        auto r = std::make_unique<fqg_recipe_s>();
        r->k = k;
        r->n = n;
        r->block = o->block;
        // pipeline.cpp:94-105: smoothing scales, smoothed activation maxima
        r->s.resize(k);
        if (o->smooth)
            smoothing_scales(act_max.data(), wmax.data(), k, o->alpha, r->s.data());
        else
            std::fill(r->s.begin(), r->s.end(), 1.0);
        std::vector<double> smax(k);
        for (int64_t j = 0; j < k; ++j) smax[j] = act_max[j] / r->s[j];
        // :108-109 truncation and plan_x
        r->t_x = derive_truncation(smax.data(), k, o->beta, o->clip != 0);
        const Plan px = build_plan(smax.data(), k, r->t_x, o->block);
        // :114-119 row maxima of repeat_channels(scale_rows(W, s)): max_n |W s_j| =
        // RN(max_n |W| * s_j) (rounding is monotone), copied to the plan_x slots
        std::vector<double> rmax(px.padded, 0.0);
        for (int64_t j = 0; j < k; ++j) {
            const double v = wmax[j] * r->s[j];
            rmax[j] = v;
            for (int64_t q = 0; q < px.ext[j]; ++q) rmax[k + px.off[j] + q] = v;
        }
        r->t_w = derive_truncation(rmax.data(), k + px.c_extend, o->beta, o->clip != 0);
        const Plan pw = build_plan(rmax.data(), px.padded, r->t_w, o->block);
        r->e_x = px.ext;
        r->e_w = pw.ext;
        const GatherMaps g = compile_maps(px, pw);

        // :122-132 select_bit_width on the flattened calibration activations and w_flat
        const int bins = static_cast<int>(o->bins);
        ActSrc as{dx, k, upload(g.amap, keep), upload(r->s, keep), upload(g.cap_x, keep),
                  r->t_x, 1.0 / r->t_x, g.kp};
        double mx_a = 0.0, mx_w = 0.0;
        bool over_a = false, over_w = false;
        std::vector<unsigned long long> ha, hw;
        scan(as, m, bins, sms, &mx_a, &over_a, &ha);
        WgtSrc ws{dw, n, upload(g.wmap, keep), upload(g.wcap, keep), as.s, r->t_w, 1.0 / r->t_w, n};
        scan(ws, g.kp, bins, sms, &mx_w, &over_w, &hw);
        if (over_w)
            throw Error(FQG_ERR_RUNTIME,
                        "flatten_rows: value exceeds plan capacity (plan built from different "
                        "statistics)");
        r->kl_act = divergence_ratio(mx_a, ha, bins, static_cast<double>(m * g.kp));
        r->kl_w = divergence_ratio(mx_w, hw, bins, static_cast<double>(g.kp * n));
        const int chosen = (r->kl_act < o->gamma && r->kl_w < o->gamma) ? 4 : 8;
        r->bits = o->mode == 1 ? 8 : chosen;  // :133-134 (O1 pins 8 bits)
        // :137-143 static activation scale, weight scale from the flattened maximum
        const double qmax = static_cast<double>((1 << (r->bits - 1)) - 1);
        r->act_scale = r->t_x / qmax;
        if (mx_w == 0.0) throw Error(FQG_ERR_RUNTIME, "quantize_layer: weight is all zero");
        r->w_scale = mx_w / qmax;
        if (o->mode == 3) {  // :144-147 gptq_optimize(w_flat, hessian_from_calibration(flat acts))
            require(g.kp * g.kp <= (int64_t{1} << 31), "calibrate O3: K' too large for the Hessian");
            double* xf = nullptr;
            double* wf = nullptr;
            int32_t* qd = nullptr;
            FQG_CUDA(cudaMalloc(&xf, static_cast<size_t>(m * g.kp) * 8));
            keep.push_back(xf);
            FQG_CUDA(cudaMalloc(&wf, static_cast<size_t>(g.kp * n) * 8));
            keep.push_back(wf);
            FQG_CUDA(cudaMalloc(&qd, static_cast<size_t>(g.kp * n) * 4));
            keep.push_back(qd);
            k_src_materialize<ActSrc><<<grid_for(m * g.kp, sms), kThreads>>>(as, m, xf);
            k_src_materialize<WgtSrc><<<grid_for(g.kp * n, sms), kThreads>>>(ws, g.kp, wf);
            FQG_CUDA(cudaGetLastError());
            gptq_weight_q(xf, m, static_cast<int>(g.kp), wf, n, o->damping, r->w_scale, qmax, qd);
            r->weight_q.resize(static_cast<size_t>(g.kp * n));
            FQG_CUDA(cudaMemcpy(r->weight_q.data(), qd, r->weight_q.size() * 4, cudaMemcpyDeviceToHost));
        }
        *out = r.release();
    });
}

int fqg_recipe_get(fqg_recipe_t r, fqg_layer_desc* d, double* kl_ratio_act, double* kl_ratio_w) {
    return guard([&] {
        require(r && d, "fqg_recipe_get: null argument");
        *d = fqg_layer_desc{};
        d->bits = r->bits;
        d->k = r->k;
        d->n = r->n;
        d->smooth_scales = r->s.data();
        d->t_x = r->t_x;
        d->ext_x = r->e_x.data();
        d->block_x = r->block;
        d->t_w = r->t_w;
        d->ext_w = r->e_w.data();
        d->block_w = r->block;
        d->act_scale = r->act_scale;
        d->w_scale = r->w_scale;
        d->weight_q = r->weight_q.empty() ? nullptr : r->weight_q.data();
        d->n_total = r->n;
        d->a_format = FQG_I8;
        d->b_format = r->bits == 4 ? FQG_I4 : FQG_I8;
        if (kl_ratio_act) *kl_ratio_act = r->kl_act;
        if (kl_ratio_w) *kl_ratio_w = r->kl_w;
    });
}

int fqg_recipe_free(fqg_recipe_t r) {
    return guard([&] { delete r; });
}

}  // extern "C"
