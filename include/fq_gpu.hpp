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
// HBM on first use and cached process-wide by recipe CONTENT (every field
// run_layer reads, weights included; LRU, FQG_LAYER_CACHE entries, default 4);
// fq::gpu::Layer gives explicit control of that lifetime. Host buffers may be
// pageable: the library stages them through pinned bounce buffers.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <mutex>
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

// Content key of a recipe: every field run_layer reads, the weights included
// (fqg_hash64 is parallel over 1 MiB blocks: ~1 ms per 100 MB of weight_q).
inline std::uint64_t recipe_key(const LayerQuantConfig& cfg) {
    std::uint64_t h = 0x6671676b6579ull;  // "fqgkey"
    auto add = [&h](const void* p, std::size_t n) { h = fqg_hash64(p, n, h); };
    auto add_plan = [&](const FlattenPlan& p) {
        add(&p.threshold, sizeof(p.threshold));
        add(&p.block, sizeof(p.block));
        add(p.extensions.data(), p.extensions.size() * sizeof(p.extensions[0]));
    };
    add(&cfg.bits, sizeof(cfg.bits));
    add(&cfg.act_scale, sizeof(cfg.act_scale));
    add(cfg.smooth_scales.s.data(), cfg.smooth_scales.s.size() * sizeof(double));
    add_plan(cfg.plan_x);
    add_plan(cfg.plan_w);
    add(&cfg.weight_q.params.scale, sizeof(cfg.weight_q.params.scale));
    add(&cfg.weight_q.q.rows, sizeof(cfg.weight_q.q.rows));
    add(&cfg.weight_q.q.cols, sizeof(cfg.weight_q.q.cols));
    add(cfg.weight_q.q.data.data(), cfg.weight_q.q.data.size() * sizeof(cfg.weight_q.q.data[0]));
    return h;
}

// Process-wide LRU cache of device layers keyed by recipe content (layers are
// immutable, so threads share them; capacity FQG_LAYER_CACHE, default 4).
inline std::shared_ptr<const Layer> cached_layer(const LayerQuantConfig& cfg) {
    struct Entry {
        std::uint64_t key;
        std::shared_ptr<const Layer> layer;
    };
    static std::mutex mu;
    static std::vector<Entry> lru;  // most recently used last
    static const std::size_t cap = [] {
        const char* e = std::getenv("FQG_LAYER_CACHE");
        const long v = e ? std::strtol(e, nullptr, 10) : 4;
        return static_cast<std::size_t>(v > 0 ? v : 1);
    }();
    const std::uint64_t key = recipe_key(cfg);
    {
        std::lock_guard<std::mutex> lk(mu);
        for (std::size_t i = 0; i < lru.size(); ++i)
            if (lru[i].key == key) {
                Entry e = lru[i];
                lru.erase(lru.begin() + static_cast<std::ptrdiff_t>(i));
                lru.push_back(e);
                return e.layer;
            }
    }
    auto layer = std::make_shared<const Layer>(cfg);  // outside the lock: uploads weights
    std::lock_guard<std::mutex> lk(mu);
    lru.push_back({key, layer});
    while (lru.size() > cap) lru.erase(lru.begin());
    return layer;
}

inline Matrix run_layer(const LayerQuantConfig& cfg, const Matrix& x,
                        std::int64_t& saturation_events) {
    if (x.cols != cfg.plan_x.channels())
        throw std::invalid_argument("run_layer: input channel count does not match recipe");
    return cached_layer(cfg)->run(x, saturation_events);
}

inline Matrix run_layer(const LayerQuantConfig& cfg, const Matrix& x) {
    std::int64_t ignored = 0;
    return fq::gpu::run_layer(cfg, x, ignored);  // qualified: ADL would also find fq::run_layer
}

}  // namespace gpu
}  // namespace fq
