// layer.cu — the layer handle behind the C ABI: a frozen, device-resident
// recipe (fq::LayerQuantConfig, pipeline.hpp:37-49) and the forward pass that
// replaces fq::run_layer (pipeline.cpp:159-169).
//
// HBM layout per layer:
//   d_s    f64 [K]        smoothing scales (divide, smoothing.cpp:75)
//   d_cap  i32 [K]        plan_x capacity E_x + 1
//   d_amap i32 [K']       composite activation gather map (j << 12 | piece)
//   d_wq   u8  [N][ldb]   weights, K-major: int8 (ldb = K') or packed int4 (K'/2)
//   d_scale f64 [2]       {s_x, s_w}
// Per forward (stream-ordered allocations): q [M][ldq] int8 / packed int4.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "fqg_internal.h"
#include "host.h"
#include "host_pool.h"
#include "kernels.h"

namespace fqg {

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
    void alloc(size_t bytes) { FQG_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16))); }
};

}  // namespace fqg

struct fqg_layer_s {
    int device = 0;
    int bits = 8, a_fmt = FQG_I8, b_fmt = FQG_I8, scale_mode = FQG_SCALE_STATIC;
    int64_t k = 0, n = 0, c1 = 0, kp = 0, n_total = 0, n_begin = 0;
    int64_t ldb = 0;
    double t_x = 0, t_w = 0, act_scale = 0, w_scale = 0, qmax = 127;
    int64_t width_x = 0;
    int64_t n_ext2 = 0;  // channels with >= 2 plan_x extension slots
    fqg::DevBuf d_s, d_rs, d_rs32, d_cap, d_off, d_wsrc, d_amap, d_wq, d_scale;
    // K1 16-bit certificates (flatten16.cu), static scale only: [0] bf16, [1] f16
    fqg::DevBuf d_cj[2], d_pj[2], d_hot, d_hotm, d_hotg, d_wsrc16;
    int64_t nhot = 0;
};

namespace fqg {
namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        FQG_CUDA(cudaGetDevice(&prev));
        if (prev != dev) FQG_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
    }
};

template <class T>
void upload(DevBuf& b, const std::vector<T>& v) {
    b.alloc(v.size() * sizeof(T));
    FQG_CUDA(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
}

// int32 [K'][n_total] row-major (reference weight_q) -> K-major int8/int4 [n][ldb].
std::vector<uint8_t> pack_weight_q(const int32_t* wq, int64_t kp, int64_t n_total, int64_t n_begin,
                                   int64_t n, int qmax, bool pack4, int64_t ldb) {
    std::vector<uint8_t> out(static_cast<size_t>(n * ldb), 0);
    for (int64_t kq = 0; kq < kp; ++kq) {
        const int32_t* row = wq + kq * n_total + n_begin;
        for (int64_t c = 0; c < n; ++c) {
            const int32_t v = row[c];
            require(v >= -qmax && v <= qmax, "weight_q value outside [-qmax, qmax]");
            if (pack4) {
                uint8_t& b = out[c * ldb + i4_byte(kq)];
                b |= static_cast<uint8_t>(((v + 8) & 0xF) << i4_shift(kq));  // biased nibble
            } else {
                out[c * ldb + kq] = static_cast<uint8_t>(static_cast<int8_t>(v));
            }
        }
    }
    return out;
}

fqg_layer_s* create(const fqg_layer_desc& d) {
    require(d.bits == 4 || d.bits == 8, "bits must be 4 or 8");
    require(d.k >= 1 && d.n >= 1, "layer: empty shape");
    require(d.smooth_scales && d.ext_x && d.ext_w, "layer: recipe arrays are required");
    require(d.weight_q || d.weight, "layer: weight_q or weight is required");
    require(d.t_x > 0.0 && std::isfinite(d.t_x), "layer: t_x must be > 0");
    require(d.a_format == FQG_I8 || d.a_format == FQG_I4, "layer: a_format must be I8 or I4");
    require(d.b_format == FQG_I8 || d.b_format == FQG_I4, "layer: b_format must be I8 or I4");
    require(d.bits == 4 || (d.a_format == FQG_I8 && d.b_format == FQG_I8),
            "layer: packed int4 operands need bits == 4");
    require(d.scale_mode == FQG_SCALE_STATIC || d.scale_mode == FQG_SCALE_DYNAMIC,
            "layer: bad scale_mode");
    const int64_t n_total = d.n_total > 0 ? d.n_total : d.n;
    require(d.n_begin >= 0 && d.n_begin + d.n <= n_total, "layer: shard outside [0, n_total)");
    if (d.scale_mode == FQG_SCALE_STATIC)
        require(d.act_scale > 0.0 && std::isfinite(d.act_scale),
                "quantize_per_tensor: scale override must be positive");

    DeviceGuard dg(d.device);
    auto* L = new fqg_layer_s();
    try {
        L->device = d.device;
        L->bits = d.bits;
        L->a_fmt = d.a_format;
        L->b_fmt = d.b_format;
        L->scale_mode = d.scale_mode;
        L->k = d.k;
        L->n = d.n;
        L->n_total = n_total;
        L->n_begin = d.n_begin;
        L->t_x = d.t_x;
        L->t_w = d.t_w;
        L->act_scale = d.act_scale;
        L->qmax = static_cast<double>((1 << (d.bits - 1)) - 1);
        const Plan px = plan_from_ext(d.t_x, d.ext_x, d.k, d.block_x);
        const Plan pw = plan_from_ext(d.t_w, d.ext_w, px.padded, d.block_w);
        // The GEMM consumes K' in steps of 32 (tcgen05 kind::i8 K) and packs int4
        // in groups of 32; both padded widths must be 32-aligned (the reference's
        // default block, flatten.hpp:20). Checked before any packing or upload.
        if (px.padded % 32 != 0 || pw.padded % 32 != 0)
            throw Error(FQG_ERR_UNSUPPORTED,
                        "layer: plan padded widths must be multiples of 32 (block_x/block_w)");
        L->c1 = px.padded;
        L->kp = pw.padded;
        const GatherMaps g = compile_maps(px, pw);
        require(L->kp * 127ll * 127ll < (1ll << 31), "layer: K' too large for exact INT32");
        for (int64_t j = 0; j < d.k; ++j)
            require(d.smooth_scales[j] != 0.0 && std::isfinite(d.smooth_scales[j]),
                    "layer: smoothing scales must be finite and non-zero");
        upload(L->d_s, std::vector<double>(d.smooth_scales, d.smooth_scales + d.k));
        std::vector<double> rs(d.k);
        std::vector<float> rs32(d.k);
        for (int64_t j = 0; j < d.k; ++j) {
            rs[j] = 1.0 / d.smooth_scales[j];  // correctly rounded
            rs32[j] = static_cast<float>(rs[j]);
        }
        upload(L->d_rs, rs);
        upload(L->d_rs32, rs32);
        upload(L->d_cap, g.cap_x);
        upload(L->d_off, g.off_x);
        L->n_ext2 = 0;
        for (int64_t j = 0; j < d.k; ++j) L->n_ext2 += d.ext_x[j] >= 2 ? 1 : 0;
        upload(L->d_wsrc, g.wsrc);
        {  // K1 16-bit path: plan_w copy sources with padding -> the zero byte at column K'
            std::vector<int32_t> w16(g.wsrc);
            for (auto& v : w16) v = v < 0 ? static_cast<int32_t>(L->kp) : v;
            upload(L->d_wsrc16, w16);
        }
        upload(L->d_amap, g.amap);
        L->width_x = g.width_x;

        const bool pack4 = d.b_format == FQG_I4;
        L->ldb = pack4 ? L->kp / 2 : L->kp;
        L->d_wq.alloc(static_cast<size_t>(L->n * L->ldb));
        if (d.weight_q) {
            require(d.w_scale > 0.0 && std::isfinite(d.w_scale), "layer: w_scale must be > 0");
            L->w_scale = d.w_scale;
            const auto packed = pack_weight_q(d.weight_q, L->kp, n_total, d.n_begin, d.n,
                                              static_cast<int>(L->qmax), pack4, L->ldb);
            FQG_CUDA(cudaMemcpy(L->d_wq.p, packed.data(), packed.size(), cudaMemcpyHostToDevice));
        } else {
            // Offline weight tail of quantize_layer on the device (K3).
            require(d.t_w > 0.0 && std::isfinite(d.t_w), "layer: t_w must be > 0");
            DevBuf w, wmap, wcap, capw, scratch;
            const size_t wbytes = static_cast<size_t>(d.k * n_total) * sizeof(double);
            w.alloc(wbytes);
            FQG_CUDA(cudaMemcpy(w.p, d.weight, wbytes, cudaMemcpyHostToDevice));
            upload(wmap, g.wmap);
            upload(wcap, g.wcap);
            upload(capw, g.capw_src);
            scratch.alloc(16);
            FQG_CUDA(cudaMemset(scratch.p, 0, 16));
            auto* amax = scratch.as<unsigned long long>();
            auto* over = reinterpret_cast<unsigned int*>(amax + 1);
            weight_absmax(w.as<double>(), d.k, n_total, L->d_s.as<double>(), capw.as<int32_t>(),
                          d.t_w, amax, over, num_sms(d.device), 0);
            unsigned long long host[2] = {0, 0};
            FQG_CUDA(cudaMemcpy(host, scratch.p, 16, cudaMemcpyDeviceToHost));
            if (static_cast<unsigned int>(host[1]) != 0)
                throw Error(FQG_ERR_RUNTIME,
                            "flatten_rows: value exceeds plan capacity (plan built from "
                            "different statistics)");
            double wmax;
            std::memcpy(&wmax, &host[0], 8);
            if (wmax == 0.0) throw Error(FQG_ERR_RUNTIME, "quantize_layer: weight is all zero");
            L->w_scale = wmax / L->qmax;  // pipeline.cpp:139-143
            weight_quant(w.as<double>(), n_total, d.n_begin, d.n, L->d_s.as<double>(),
                         wmap.as<int32_t>(), wcap.as<int32_t>(), L->kp, d.t_w, L->w_scale,
                         L->qmax, pack4, L->d_wq.as<uint8_t>(), L->ldb, 0);
            FQG_CUDA(cudaDeviceSynchronize());
        }
        const double sc[2] = {d.scale_mode == FQG_SCALE_STATIC ? d.act_scale : 0.0, L->w_scale};
        L->d_scale.alloc(sizeof(sc));
        FQG_CUDA(cudaMemcpy(L->d_scale.p, sc, sizeof(sc), cudaMemcpyHostToDevice));
        if (d.scale_mode == FQG_SCALE_STATIC && d.k % 8 == 0) {
            for (int f = 0; f < 2; ++f) {
                L->d_cj[f].alloc(static_cast<size_t>(d.k) * sizeof(float));
                L->d_pj[f].alloc(static_cast<size_t>(d.k) * sizeof(uint16_t));
                tier1_tables(L->d_s.as<double>(), d.k, d.act_scale, d.t_x, L->qmax, f == 1,
                             L->d_cj[f].as<float>(), L->d_pj[f].as<uint16_t>(), 0);
            }
            // Hot channels: a calibrated maximum >= kHotE * T_x means most of the
            // channel's elements carry full pieces; K1 runs them through the exact
            // split on every row instead of queueing them (certificate P_j = 0xFFFF
            // keeps them off the queue).
            constexpr int64_t kHotE = 4;
            constexpr size_t kMaxHot = 128;  // flatten16.cu: 32 lanes x kHotRegs
            std::vector<int32_t> hot;
            for (int64_t j = 0; j < d.k; ++j)
                if (d.ext_x[j] >= kHotE) hot.push_back(static_cast<int32_t>(j));
            if (hot.size() > kMaxHot) {  // keep the channels with the most extension slots
                std::stable_sort(hot.begin(), hot.end(),
                                 [&](int32_t a, int32_t b) { return d.ext_x[a] > d.ext_x[b]; });
                hot.resize(kMaxHot);
                std::sort(hot.begin(), hot.end());
            }
            L->nhot = static_cast<int64_t>(hot.size());
            upload(L->d_hot, hot);
            // K1 tables for the hot channels: {j, capacity, ext_offset, RN32(1/s_j)}
            // and, per group of 8 channels, hot mask | index of its first hot channel << 8.
            std::vector<int32_t> hotm(4 * hot.size());
            std::vector<int32_t> hotg(static_cast<size_t>((d.k / 8 + 3) / 4 * 4), 0);  // 16-byte multiple
            for (size_t h = 0; h < hot.size(); ++h) {
                const int32_t j = hot[h];
                float r32 = rs32[j];
                int32_t rbits;
                std::memcpy(&rbits, &r32, 4);
                hotm[4 * h] = j;
                hotm[4 * h + 1] = g.cap_x[j];
                hotm[4 * h + 2] = g.off_x[j];
                hotm[4 * h + 3] = rbits;
                int32_t& e = hotg[j / 8];
                if ((e & 0xFF) == 0) e |= static_cast<int32_t>(h) << 8;
                e |= 1 << (j % 8);
            }
            upload(L->d_hotm, hotm);
            upload(L->d_hotg, hotg);

            std::vector<uint16_t> pj(static_cast<size_t>(d.k));
            for (int f = 0; f < 2 && !hot.empty(); ++f) {
                FQG_CUDA(cudaMemcpy(pj.data(), L->d_pj[f].p, pj.size() * 2, cudaMemcpyDeviceToHost));
                for (int32_t j : hot) pj[j] = 0xFFFF;
                FQG_CUDA(cudaMemcpy(L->d_pj[f].p, pj.data(), pj.size() * 2, cudaMemcpyHostToDevice));
            }
            FQG_CUDA(cudaDeviceSynchronize());
        }
        return L;
    } catch (...) {
        delete L;
        throw;
    }
}

int64_t ldq_of(const fqg_layer_s* L) { return L->a_fmt == FQG_I4 ? L->kp / 2 : L->kp; }

// Per-call device scratch: q operand, and in dynamic mode {s_x, s_w, amax}.
struct CallScratch {
    void* q = nullptr;
    double* scale = nullptr;
    unsigned long long* amax = nullptr;
    cudaStream_t st;
    ~CallScratch() {
        if (q) cudaFreeAsync(q, st);
        if (scale) cudaFreeAsync(scale, st);
    }
};

bool biased_b(const fqg_layer_s* L) { return L->b_fmt == FQG_I4; }

void quantize_acts(const fqg_layer_s* L, const void* x, int x_dtype, int64_t m, void* q,
                   double* scale, unsigned long long* amax, unsigned long long* sat,
                   int32_t* rowsum, cudaStream_t st) {
    FlattenArgs a{};
    a.rowsum = rowsum;
    a.x = x;
    a.x_dtype = x_dtype;
    a.ldx = L->k;
    a.m = m;
    a.k = L->k;
    a.kp = L->kp;
    a.s = L->d_s.as<double>();
    a.rs = L->d_rs.as<double>();
    a.rs32 = L->d_rs32.as<float>();
    a.cap = L->d_cap.as<int32_t>();
    a.off = L->d_off.as<int32_t>();
    a.n_ext2 = L->n_ext2;
    a.wsrc = L->d_wsrc.as<int32_t>();
    a.amap = L->d_amap.as<int32_t>();
    a.c1 = L->c1;
    a.width = L->width_x;
    a.t = L->t_x;
    a.scale = scale;
    a.amax = amax;
    a.qmax = L->qmax;
    a.pack4 = L->a_fmt == FQG_I4;
    a.q = static_cast<uint8_t*>(q);
    a.ldq = ldq_of(L);
    a.sat = sat;
    a.num_sms = num_sms(L->device);
    static const bool general_only = [] {
        const char* e = std::getenv("FQG_K1_GENERAL");
        return e != nullptr && std::atoi(e) != 0;
    }();
    const int f = x_dtype == FQG_BF16 ? 0 : (x_dtype == FQG_F16 ? 1 : -1);
    if (f >= 0 && amax == nullptr && !general_only && L->d_cj[f].p != nullptr) {
        a.cj = L->d_cj[f].as<float>();
        a.pj = L->d_pj[f].as<uint16_t>();
        a.hot = L->d_hot.as<int32_t>();
        a.hotm = L->d_hotm.as<int32_t>();
        a.hotg = L->d_hotg.as<int32_t>();
        a.nhot = L->nhot;
        a.wsrc16 = L->d_wsrc16.as<int32_t>();
        a.act_scale = L->act_scale;
    }
    flatten_quant(a, st);
}

// Int4 weights are stored biased (nibble = q + 8, FQG_I4_BIASED): the GEMM
// needs the operand row sums, from K1 or (when absent) from a rowsum pass.
void run_gemm(const fqg_layer_s* L, const void* q, const int32_t* rowsum, int64_t m, void* y,
              int y_dtype, int64_t ldy, const double* scale, const void* bias, int bias_dtype,
              cudaStream_t st) {
    int32_t* own = nullptr;
    if (biased_b(L) && rowsum == nullptr) {
        FQG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&own), static_cast<size_t>(m) * 4, st));
        operand_rowsum(static_cast<const uint8_t*>(q), ldq_of(L), m, L->kp, L->a_fmt == FQG_I4, own,
                       st);
        rowsum = own;
    }
    GemmArgs g{q, L->a_fmt, ldq_of(L), L->d_wq.p, biased_b(L) ? FQG_I4_BIASED : L->b_fmt, L->ldb,
               m, L->n, L->kp, y, y_dtype, ldy, scale, bias, bias ? bias_dtype : FQG_NONE};
    g.rowsum = rowsum;
    g.qmax_a = g.qmax_b = static_cast<int>(L->qmax);  // both operands hold bits-wide values
    try {
        gemm_i8(g, st);
    } catch (...) {
        if (own) cudaFreeAsync(own, st);
        throw;
    }
    if (own) FQG_CUDA(cudaFreeAsync(own, st));
}

void forward(const fqg_layer_s* L, const void* x, int x_dtype, int64_t m, void* y, int y_dtype,
             int64_t ldy, const void* bias, int bias_dtype, unsigned long long* sat,
             cudaStream_t st) {
    require(m >= 1, "run_layer: empty input");
    require(x != nullptr && y != nullptr, "run_layer: null buffer");
    require(ldy >= L->n, "run_layer: ldy < n");
    CallScratch cs;
    cs.st = st;
    // q operand [m][ldq], then the row sums (16-byte aligned: ldq % 16 == 0)
    const size_t qbytes = static_cast<size_t>(m * ldq_of(L));
    FQG_CUDA(cudaMallocAsync(&cs.q, qbytes + (biased_b(L) ? static_cast<size_t>(m) * 4 : 0), st));
    int32_t* rowsum =
        biased_b(L) ? reinterpret_cast<int32_t*>(static_cast<uint8_t*>(cs.q) + qbytes) : nullptr;
    const double* scale = L->d_scale.as<double>();
    double* kscale = L->d_scale.as<double>();
    if (L->scale_mode == FQG_SCALE_DYNAMIC) {
        FQG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&cs.scale), 32, st));
        cs.amax = reinterpret_cast<unsigned long long*>(cs.scale + 2);
        FQG_CUDA(cudaMemcpyAsync(cs.scale, L->d_scale.p, 16, cudaMemcpyDeviceToDevice, st));
        FQG_CUDA(cudaMemsetAsync(cs.amax, 0, 8, st));
        scale = kscale = cs.scale;
    }
    quantize_acts(L, x, x_dtype, m, cs.q, kscale, cs.amax, sat, rowsum, st);
    run_gemm(L, cs.q, rowsum, m, y, y_dtype, ldy, scale, bias, bias_dtype, st);
}

// Pinned bounce buffers per (thread, device), grown on demand.
struct Bounce {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFreeHost(p);
            p = nullptr;
            cap = 0;
            FQG_CUDA(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
            cap = bytes;
        }
        return p;
    }
};

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace
}  // namespace fqg

using namespace fqg;

extern "C" {

int fqg_layer_create(const fqg_layer_desc* desc, fqg_layer_t* out) {
    return guard([&] {
        require(desc && out, "fqg_layer_create: null argument");
        *out = create(*desc);
    });
}

int fqg_layer_destroy(fqg_layer_t layer) {
    return guard([&] {
        if (!layer) return;
        DeviceGuard dg(layer->device);
        delete layer;
    });
}

int fqg_layer_get_info(fqg_layer_t L, fqg_layer_info* i) {
    return guard([&] {
        require(L && i, "fqg_layer_get_info: null argument");
        *i = {L->bits,  L->a_fmt, L->b_fmt,  L->scale_mode, L->k,     L->n,
              L->c1,    L->kp,    L->n_total, L->n_begin,   L->t_x,   L->t_w,
              L->act_scale, L->w_scale, L->n * L->ldb};
    });
}

int fqg_layer_weight_q(fqg_layer_t L, int32_t* wq, double* w_scale) {
    return guard([&] {
        require(L != nullptr, "fqg_layer_weight_q: null layer");
        DeviceGuard dg(L->device);
        std::vector<uint8_t> packed(static_cast<size_t>(L->n * L->ldb));
        FQG_CUDA(cudaMemcpy(packed.data(), L->d_wq.p, packed.size(), cudaMemcpyDeviceToHost));
        if (wq) {
            for (int64_t c = 0; c < L->n; ++c)
                for (int64_t kq = 0; kq < L->kp; ++kq) {
                    int v;
                    if (L->b_fmt == FQG_I4) {
                        const int nib = (packed[c * L->ldb + i4_byte(kq)] >> i4_shift(kq)) & 0xF;
                        v = nib - 8;  // biased storage
                    } else {
                        v = static_cast<int8_t>(packed[c * L->ldb + kq]);
                    }
                    wq[kq * L->n + c] = v;
                }
        }
        if (w_scale) *w_scale = L->w_scale;
    });
}

int fqg_layer_forward(fqg_layer_t L, const void* x, int x_dtype, int64_t m, void* y, int y_dtype,
                      int64_t ldy, const void* bias, int bias_dtype,
                      unsigned long long* saturation_dev, void* stream) {
    return guard([&] {
        require(L != nullptr, "run_layer: null layer");
        DeviceGuard dg(L->device);
        forward(L, x, x_dtype, m, y, y_dtype, ldy, bias, bias_dtype, saturation_dev,
                static_cast<cudaStream_t>(stream));
    });
}

int fqg_layer_quantize_acts_ex(fqg_layer_t L, const void* x, int x_dtype, int64_t m, void* q,
                               int32_t* rowsum_dev, unsigned long long* saturation_dev,
                               void* stream) {
    return guard([&] {
        require(L != nullptr && x && q && m >= 1, "quantize_acts: bad argument");
        require(L->scale_mode == FQG_SCALE_STATIC,
                "quantize_acts: the split entry points take the static scale");
        DeviceGuard dg(L->device);
        quantize_acts(L, x, x_dtype, m, q, L->d_scale.as<double>(), nullptr, saturation_dev,
                      rowsum_dev, static_cast<cudaStream_t>(stream));
    });
}

int fqg_layer_quantize_acts(fqg_layer_t L, const void* x, int x_dtype, int64_t m, void* q,
                            unsigned long long* saturation_dev, void* stream) {
    return fqg_layer_quantize_acts_ex(L, x, x_dtype, m, q, nullptr, saturation_dev, stream);
}

int fqg_layer_gemm_ex(fqg_layer_t L, const void* q, const int32_t* rowsum_dev, int64_t m,
                      void* y, int y_dtype, int64_t ldy, const void* bias, int bias_dtype,
                      void* stream) {
    return guard([&] {
        require(L != nullptr && q && y && m >= 1, "layer_gemm: bad argument");
        require(ldy >= L->n, "layer_gemm: ldy < n");
        DeviceGuard dg(L->device);
        run_gemm(L, q, rowsum_dev, m, y, y_dtype, ldy, L->d_scale.as<double>(), bias, bias_dtype,
                 static_cast<cudaStream_t>(stream));
    });
}

int fqg_layer_gemm(fqg_layer_t L, const void* q, int64_t m, void* y, int y_dtype, int64_t ldy,
                   const void* bias, int bias_dtype, void* stream) {
    return fqg_layer_gemm_ex(L, q, nullptr, m, y, y_dtype, ldy, bias, bias_dtype, stream);
}

int fqg_shard_bounds(int64_t n_total, int world, int rank, int64_t* b0, int64_t* b1,
                     int64_t* width) {
    return guard([&] {
        require(n_total >= 1 && world >= 1 && rank >= 0 && rank < world,
                "shard_bounds: bad rank/world");
        int64_t per = (n_total + world - 1) / world;
        per = (per + 31) / 32 * 32;  // 32-aligned shards (the GEMM's K-major int4 groups)
        const int64_t s0 = std::min<int64_t>(n_total, static_cast<int64_t>(rank) * per);
        if (b0) *b0 = s0;
        if (b1) *b1 = std::min<int64_t>(n_total, s0 + per);
        if (width) *width = std::min<int64_t>(n_total, per);
    });
}

int fqg_layer_forward_sharded(fqg_layer_t L, const void* x, int x_dtype, int64_t m, void* gather,
                              int y_dtype, int world, int rank, const void* bias, int bias_dtype,
                              unsigned long long* saturation_dev, fqg_allgather_fn allgather,
                              void* comm, void* stream) {
    return guard([&] {
        require(L != nullptr && x && gather && m >= 1, "forward_sharded: bad argument");
        require(world >= 1 && rank >= 0 && rank < world, "forward_sharded: bad rank/world");
        require(y_dtype == FQG_F16 || y_dtype == FQG_BF16 || y_dtype == FQG_F32 ||
                    y_dtype == FQG_F64,
                "forward_sharded: output dtype must be F16/BF16/F32/F64");
        int64_t b0 = 0, b1 = 0, width = 0;
        if (fqg_shard_bounds(L->n_total, world, rank, &b0, &b1, &width) != FQG_OK)
            throw Error(FQG_ERR_INVALID, g_last_error);
        require(b0 == L->n_begin && b1 - b0 == L->n,
                "forward_sharded: the layer is not this rank's fqg_shard_bounds shard");
        DeviceGuard dg(L->device);
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        const int esz = dtype_size(y_dtype);
        uint8_t* slot = static_cast<uint8_t*>(gather) + static_cast<size_t>(rank) * m * width * esz;
        forward(L, x, x_dtype, m, slot, y_dtype, width, bias, bias_dtype, saturation_dev, st);
        if (allgather != nullptr && world > 1) {
            // ncclDataType_t: ncclFloat16 = 6, ncclFloat32 = 7, ncclFloat64 = 8, ncclBfloat16 = 9
            const int nt = y_dtype == FQG_F16 ? 6 : y_dtype == FQG_F32 ? 7 : y_dtype == FQG_F64 ? 8 : 9;
            const int rc = allgather(slot, gather, static_cast<size_t>(m * width), nt, comm, stream);
            if (rc != 0)
                throw Error(FQG_ERR_RUNTIME, "forward_sharded: allgather returned " + std::to_string(rc));
        }
    });
}

// The drop-in host call, pipelined: M is cut into row chunks that alternate
// between two streams, so the host->device copy of chunk c + 1, the kernels of
// chunk c and the device->host copy of chunk c - 1 overlap (PCIe is full
// duplex). Rows are independent under the static scale, so chunking is exact.
int fqg_layer_run_host(fqg_layer_t L, const double* x_host, int64_t m, double* y_host,
                       int64_t* saturation) {
    return guard([&] {
        require(L != nullptr && x_host && y_host, "run_layer: null argument");
        require(m >= 1, "run_layer: empty input");
        DeviceGuard dg(L->device);
        static thread_local cudaStream_t streams[64][2] = {};
        cudaStream_t* ss = streams[L->device & 63];
        for (int i = 0; i < 2; ++i)
            if (ss[i] == nullptr) FQG_CUDA(cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking));
        cudaStream_t st = ss[0];
        void *dx = nullptr, *dy = nullptr;
        unsigned long long* dsat = nullptr;
        const size_t xb = static_cast<size_t>(m * L->k) * 8, yb = static_cast<size_t>(m * L->n) * 8;
        FQG_CUDA(cudaMallocAsync(&dx, xb, st));
        FQG_CUDA(cudaMallocAsync(&dy, yb, st));
        FQG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dsat), 8, st));
        cudaEvent_t ev[2];
        FQG_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        FQG_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
        struct Free {
            void *a, *b, *c;
            cudaStream_t s0, s1;
            cudaEvent_t e0, e1;
            ~Free() {
                cudaEventRecord(e1, s1);  // stream 1's work done before the frees
                cudaStreamWaitEvent(s0, e1, 0);
                cudaFreeAsync(a, s0);
                cudaFreeAsync(b, s0);
                cudaFreeAsync(c, s0);
                cudaStreamSynchronize(s0);
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
            }
        } fr{dx, dy, dsat, ss[0], ss[1], ev[0], ev[1]};
        FQG_CUDA(cudaMemsetAsync(dsat, 0, 8, st));
        FQG_CUDA(cudaEventRecord(ev[0], st));  // allocations + zeroed counter visible to stream 1
        FQG_CUDA(cudaStreamWaitEvent(ss[1], ev[0], 0));
        // ~8 chunks of >= 128 rows (a multiple of 32 keeps the GEMM tiles full).
        // The dynamic scale is one absmax over the whole input (quantize.cpp:34-40):
        // a single chunk then, so every row sees the same s_x.
        const int64_t chunk = L->scale_mode == FQG_SCALE_DYNAMIC
                                  ? m
                                  : std::max<int64_t>(128, ((m + 7) / 8 + 31) / 32 * 32);
        // Pageable host buffers (the drop-in's fq::Matrix) are staged through
        // pinned bounce buffers, two chunk slots each way: the parallel host copy
        // of chunk c overlaps the DMA and kernels of chunks c - 1 and c - 2.
        const bool staged = !(is_pinned(x_host) && is_pinned(y_host));
        static thread_local Bounce bx[64][2], by[64][2];
        static thread_local cudaEvent_t evx[64][2] = {}, evy[64][2] = {};
        cudaEvent_t* ex = evx[L->device & 63];
        cudaEvent_t* ey = evy[L->device & 63];
        for (int i = 0; i < 2 && staged; ++i) {
            if (ex[i] == nullptr) FQG_CUDA(cudaEventCreateWithFlags(&ex[i], cudaEventDisableTiming));
            if (ey[i] == nullptr) FQG_CUDA(cudaEventCreateWithFlags(&ey[i], cudaEventDisableTiming));
        }
        const size_t cxb = static_cast<size_t>(chunk * L->k) * 8, cyb = static_cast<size_t>(chunk * L->n) * 8;
        struct Pending {
            int64_t r0 = 0, mc = 0;
            bool live = false;
        } pend[2];
        auto drain = [&](int slot) {  // chunk in y slot `slot` -> the caller's buffer
            if (!pend[slot].live) return;
            FQG_CUDA(cudaEventSynchronize(ey[slot]));
            parallel_copy(y_host + pend[slot].r0 * L->n, by[L->device & 63][slot].p,
                                 static_cast<size_t>(pend[slot].mc * L->n) * 8);
            pend[slot].live = false;
        };
        int ci = 0;
        for (int64_t r0 = 0; r0 < m; r0 += chunk, ++ci) {
            const int64_t mc = std::min(chunk, m - r0);
            const int slot = ci & 1;
            cudaStream_t s = ss[slot];
            const double* xs = x_host + r0 * L->k;
            double* dxs = static_cast<double*>(dx) + r0 * L->k;
            double* dys = static_cast<double*>(dy) + r0 * L->n;
            const size_t nxb = static_cast<size_t>(mc * L->k) * 8, nyb = static_cast<size_t>(mc * L->n) * 8;
            if (staged) {
                void* px = bx[L->device & 63][slot].get(cxb);
                by[L->device & 63][slot].get(cyb);
                if (ci >= 2) FQG_CUDA(cudaEventSynchronize(ex[slot]));  // H2D of chunk c-2 read it
                parallel_copy(px, xs, nxb);
                FQG_CUDA(cudaMemcpyAsync(dxs, px, nxb, cudaMemcpyHostToDevice, s));
                FQG_CUDA(cudaEventRecord(ex[slot], s));
            } else {
                FQG_CUDA(cudaMemcpyAsync(dxs, xs, nxb, cudaMemcpyHostToDevice, s));
            }
            forward(L, dxs, FQG_F64, mc, dys, FQG_F64, L->n, nullptr, FQG_NONE, dsat, s);
            if (staged) {
                drain(slot);  // chunk c - 2 leaves the y slot before chunk c's D2H lands
                FQG_CUDA(cudaMemcpyAsync(by[L->device & 63][slot].p, dys, nyb,
                                         cudaMemcpyDeviceToHost, s));
                FQG_CUDA(cudaEventRecord(ey[slot], s));
                pend[slot] = {r0, mc, true};
            } else {
                FQG_CUDA(cudaMemcpyAsync(y_host + r0 * L->n, dys, nyb, cudaMemcpyDeviceToHost, s));
            }
        }
        if (staged) {
            drain(ci & 1);  // the older of the two outstanding chunks first
            drain((ci + 1) & 1);
        }
        FQG_CUDA(cudaEventRecord(ev[1], ss[1]));
        FQG_CUDA(cudaStreamWaitEvent(st, ev[1], 0));
        unsigned long long sat = 0;
        FQG_CUDA(cudaMemcpyAsync(&sat, dsat, 8, cudaMemcpyDeviceToHost, st));
        FQG_CUDA(cudaStreamSynchronize(st));
        if (saturation) *saturation = static_cast<int64_t>(sat);
    });
}

}  // extern "C"
