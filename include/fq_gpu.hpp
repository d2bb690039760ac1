// fq_gpu.hpp — drop-in B200 replacement for the reference hot path, for C++
// callers of the reference library (namespace fq, /root/reference/proj/core).
//
// Include AFTER "fq/pipeline.hpp" and link libfqg.so. Provides
//
//   fq::Matrix fq::gpu::run_layer(const fq::LayerQuantConfig&, const fq::Matrix&);
//   fq::Matrix fq::gpu::run_layer(const fq::LayerQuantConfig&, const fq::Matrix&,
//                                 std::int64_t& saturation_events);
//
// with exactly the signatures, semantics and exception types of fq::run_layer
// (pipeline.hpp:83-84, pipeline.cpp:159-169): same f64 outputs bit for bit,
// same saturation count, std::invalid_argument on a channel-count mismatch,
// std::runtime_error for device failures. The quantized layer is uploaded to
// HBM on first use and cached per (thread, recipe object, weight buffer);
// fq::gpu::Layer gives explicit control of that lifetime.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "fqg.h"

namespace fq {
namespace gpu {

[[noreturn]] inline void throw_status(int rc, const char* where) {
    const std::string msg = std::string(where) + ": " + fqg_last_error();
    if (rc == FQG_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// One LayerQuantConfig resident on a device (weights packed K-major; int4
// weights stay packed in HBM for 4-bit layers).
class Layer {
   public:
    explicit Layer(const LayerQuantConfig& cfg, int device = 0) {
        fqg_layer_desc d{};
        d.bits = cfg.bits;
        d.k = cfg.plan_x.channels();
        d.n = cfg.weight_q.q.cols;
        d.smooth_scales = cfg.smooth_scales.s.data();
        d.t_x = cfg.plan_x.threshold;
        d.ext_x = cfg.plan_x.extensions.data();
        d.block_x = cfg.plan_x.block;
        d.t_w = cfg.plan_w.threshold;
        d.ext_w = cfg.plan_w.extensions.data();
        d.block_w = cfg.plan_w.block;
        d.act_scale = cfg.act_scale;
        d.weight_q = cfg.weight_q.q.data.data();
        d.w_scale = cfg.weight_q.params.scale;
        d.n_total = d.n;
        d.n_begin = 0;
        d.a_format = FQG_I8;
        d.b_format = cfg.bits == 4 ? FQG_I4 : FQG_I8;
        d.scale_mode = FQG_SCALE_STATIC;
        d.device = device;
        if (static_cast<std::int64_t>(cfg.smooth_scales.s.size()) != d.k)
            throw std::invalid_argument("run_layer: smoothing scales do not match plan_x");
        if (cfg.weight_q.q.rows != cfg.plan_w.padded_width)
            throw std::invalid_argument("run_layer: weight_q rows do not match plan_w");
        fqg_layer_t h = nullptr;
        const int rc = fqg_layer_create(&d, &h);
        if (rc != FQG_OK) throw_status(rc, "fqg_layer_create");
        h_.reset(h);
        k_ = d.k;
        n_ = d.n;
    }

    Matrix run(const Matrix& x, std::int64_t& saturation_events) const {
        if (x.cols != k_)  // pipeline.cpp:161-163
            throw std::invalid_argument("run_layer: input channel count does not match recipe");
        std::vector<double> y(static_cast<std::size_t>(x.rows * n_));
        std::int64_t sat = 0;
        const int rc = fqg_layer_run_host(h_.get(), x.data.data(), x.rows, y.data(), &sat);
        if (rc != FQG_OK) throw_status(rc, "fqg_layer_run_host");
        saturation_events = sat;
        return Matrix(x.rows, n_, std::move(y));
    }

   private:
    struct Del {
        void operator()(fqg_layer_t h) const { fqg_layer_destroy(h); }
    };
    std::unique_ptr<fqg_layer_s, Del> h_;
    std::int64_t k_ = 0, n_ = 0;
};

inline const Layer& cached_layer(const LayerQuantConfig& cfg) {
    struct Entry {
        const void* weights;
        std::size_t size;
        double act_scale;
        std::unique_ptr<Layer> layer;
    };
    thread_local std::unordered_map<const LayerQuantConfig*, Entry> cache;
    Entry& e = cache[&cfg];
    if (!e.layer || e.weights != cfg.weight_q.q.data.data() ||
        e.size != cfg.weight_q.q.data.size() || e.act_scale != cfg.act_scale) {
        e.layer = std::make_unique<Layer>(cfg);
        e.weights = cfg.weight_q.q.data.data();
        e.size = cfg.weight_q.q.data.size();
        e.act_scale = cfg.act_scale;
    }
    return *e.layer;
}

inline Matrix run_layer(const LayerQuantConfig& cfg, const Matrix& x,
                        std::int64_t& saturation_events) {
    if (x.cols != cfg.plan_x.channels())
        throw std::invalid_argument("run_layer: input channel count does not match recipe");
    return cached_layer(cfg).run(x, saturation_events);
}

inline Matrix run_layer(const LayerQuantConfig& cfg, const Matrix& x) {
    std::int64_t ignored = 0;
    return fq::gpu::run_layer(cfg, x, ignored);  // qualified: ADL would also find fq::run_layer
}

}  // namespace gpu
}  // namespace fq
