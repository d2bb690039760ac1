// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (oracle). A C-ABI wrapper around the
// UNMODIFIED reference library (fq_core built from /root/reference/proj/core/src
// by oracle/Makefile). Nothing on the product path links or loads this file;
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it as the
// checker and as the reference CPU arm.
//
// Every entry point forwards to the reference function named in its comment;
// no arithmetic of the hot path is restated here.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fq/archive.hpp"
#include "fq/calibration.hpp"
#include "fq/flatten.hpp"
#include "fq/matrix.hpp"
#include "fq/pipeline.hpp"
#include "fq/quantize.hpp"
#include "fq/schemas.hpp"
#include "fq/smoothing.hpp"
#include "fq/synthetic.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return -2;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return -3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

fq::Matrix mat(const double* p, int64_t r, int64_t c) {
    return fq::Matrix(r, c, std::vector<double>(p, p + r * c));
}

// A FlattenPlan from its defining arrays, the way build_flatten_plan lays it
// out (flatten.cpp:17-45): ext_offset = exclusive prefix sum, padded to block.
fq::FlattenPlan plan_from(double t, const int64_t* e, int64_t k, int64_t block) {
    fq::FlattenPlan p;
    p.threshold = t;
    p.block = block;
    p.extensions.assign(e, e + k);
    p.ext_offset.resize(k);
    int64_t acc = 0;
    for (int64_t j = 0; j < k; ++j) {
        p.ext_offset[j] = acc;
        acc += e[j];
    }
    p.c_extend = acc;
    p.padded_width = (p.width() + block - 1) / block * block;
    return p;
}

}  // namespace

extern "C" {

struct fqref_layer {
    fq::LayerQuantConfig cfg;
};

struct fqref_synth_opts {
    int64_t rows, samples, in_channels, out_channels;
    double outlier_fraction, outlier_min, outlier_max, channel_spread;
    double act_tail_prob_max, act_tail_scale, weight_row_spread;
    uint64_t seed;
};

struct fqref_qopts {
    int mode;  // 1=O1 2=O2 3=O3
    double alpha, beta, gamma;
    int64_t block, bins;
    double damping;
    int smooth, clip;
};

struct fqref_layer_info {
    int bits;
    int64_t K, N, C1, Kp, cext_x, cext_w;
    double T_x, T_w, act_scale, s_w, kl_ratio_act, kl_ratio_w;
};

const char* fqref_last_error(void) { return g_err.c_str(); }

void fqref_default_synth_opts(fqref_synth_opts* o) {
    fq::SyntheticOptions d;
    *o = {d.rows, d.samples, d.in_channels, d.out_channels, d.outlier_fraction, d.outlier_min,
          d.outlier_max, d.channel_spread, d.act_tail_prob_max, d.act_tail_scale,
          d.weight_row_spread, d.seed};
}

void fqref_default_qopts(fqref_qopts* o) {
    fq::QuantOptions d;
    *o = {static_cast<int>(d.mode) + 1, d.alpha, d.beta, d.gamma, d.block, d.bins, d.damping,
          d.smooth ? 1 : 0, d.clip ? 1 : 0};
}

// fq::make_synthetic_layer (synthetic.cpp:121-159).
int fqref_synthetic_layer(const fqref_synth_opts* o, int64_t index, double* weight,
                          double* calib, double* test_input, int64_t* outlier_idx,
                          int64_t* n_outliers) {
    return guard([&] {
        fq::SyntheticOptions so;
        so.rows = o->rows;
        so.samples = o->samples;
        so.in_channels = o->in_channels;
        so.out_channels = o->out_channels;
        so.outlier_fraction = o->outlier_fraction;
        so.outlier_min = o->outlier_min;
        so.outlier_max = o->outlier_max;
        so.channel_spread = o->channel_spread;
        so.act_tail_prob_max = o->act_tail_prob_max;
        so.act_tail_scale = o->act_tail_scale;
        so.weight_row_spread = o->weight_row_spread;
        so.seed = o->seed;
        const fq::SyntheticLayer l = fq::make_synthetic_layer(so, index);
        if (weight) std::memcpy(weight, l.weight.data.data(), l.weight.data.size() * 8);
        if (calib) {
            for (size_t s = 0; s < l.calib.size(); ++s)
                std::memcpy(calib + s * l.calib[s].data.size(), l.calib[s].data.data(),
                            l.calib[s].data.size() * 8);
        }
        if (test_input)
            std::memcpy(test_input, l.test_input.data.data(), l.test_input.data.size() * 8);
        if (n_outliers) *n_outliers = static_cast<int64_t>(l.outlier_channels.size());
        if (outlier_idx)
            std::copy(l.outlier_channels.begin(), l.outlier_channels.end(), outlier_idx);
    });
}

// fq::quantize_layer (pipeline.cpp:76-152).
int fqref_quantize_layer(const double* w, int64_t k, int64_t n, const double* calib,
                         int64_t samples, int64_t rows, const fqref_qopts* o,
                         fqref_layer** out) {
    return guard([&] {
        fq::QuantOptions q;
        q.mode = static_cast<fq::QuantMode>(o->mode - 1);
        q.alpha = o->alpha;
        q.beta = o->beta;
        q.gamma = o->gamma;
        q.block = o->block;
        q.bins = o->bins;
        q.damping = o->damping;
        q.smooth = o->smooth != 0;
        q.clip = o->clip != 0;
        std::vector<fq::Matrix> cs;
        for (int64_t s = 0; s < samples; ++s) cs.push_back(mat(calib + s * rows * k, rows, k));
        auto* l = new fqref_layer{fq::quantize_layer(mat(w, k, n), cs, q)};
        *out = l;
    });
}

// An explicit recipe (LayerQuantConfig fields, pipeline.hpp:37-49) from arrays.
int fqref_layer_from_arrays(int bits, int64_t k, int64_t n, const double* s, double t_x,
                            const int64_t* e_x, int64_t block_x, double t_w,
                            const int64_t* e_w, int64_t block_w, const int32_t* wq,
                            double s_w, double act_scale, fqref_layer** out) {
    return guard([&] {
        auto* l = new fqref_layer{};
        l->cfg.bits = bits;
        l->cfg.smooth_scales.s.assign(s, s + k);
        l->cfg.plan_x = plan_from(t_x, e_x, k, block_x);
        l->cfg.plan_w = plan_from(t_w, e_w, l->cfg.plan_x.padded_width, block_w);
        l->cfg.truncation.threshold = t_x;
        l->cfg.truncation_w.threshold = t_w;
        const int64_t kp = l->cfg.plan_w.padded_width;
        l->cfg.weight_q.q = fq::IntMatrix(kp, n, std::vector<int32_t>(wq, wq + kp * n));
        l->cfg.weight_q.params = {bits, s_w};
        l->cfg.act_scale = act_scale;
        *out = l;
    });
}

void fqref_layer_free(fqref_layer* l) { delete l; }

int fqref_layer_info_get(const fqref_layer* l, fqref_layer_info* i) {
    return guard([&] {
        const auto& c = l->cfg;
        *i = {c.bits,
              c.plan_x.channels(),
              c.weight_q.q.cols,
              c.plan_x.padded_width,
              c.plan_w.padded_width,
              c.plan_x.c_extend,
              c.plan_w.c_extend,
              c.plan_x.threshold,
              c.plan_w.threshold,
              c.act_scale,
              c.weight_q.params.scale,
              c.kl_ratio_act,
              c.kl_ratio_w};
    });
}

int fqref_layer_arrays(const fqref_layer* l, double* s, int64_t* e_x, int64_t* e_w,
                       int32_t* wq) {
    return guard([&] {
        const auto& c = l->cfg;
        if (s) std::copy(c.smooth_scales.s.begin(), c.smooth_scales.s.end(), s);
        if (e_x) std::copy(c.plan_x.extensions.begin(), c.plan_x.extensions.end(), e_x);
        if (e_w) std::copy(c.plan_w.extensions.begin(), c.plan_w.extensions.end(), e_w);
        if (wq) std::copy(c.weight_q.q.data.begin(), c.weight_q.q.data.end(), wq);
    });
}

// fq::run_layer (pipeline.cpp:159-169). nthreads > 1 splits the rows into
// contiguous blocks, one unmodified run_layer call per block: bit-identical
// because the activation scale is static and rows are independent.
int fqref_run_layer(const fqref_layer* l, const double* x, int64_t m, double* y,
                    int64_t* saturation, int nthreads) {
    return guard([&] {
        const int64_t k = l->cfg.plan_x.channels();
        const int64_t n = l->cfg.weight_q.q.cols;
        if (nthreads <= 1 || m < 2) {
            int64_t sat = 0;
            const fq::Matrix out = fq::run_layer(l->cfg, mat(x, m, k), sat);
            std::memcpy(y, out.data.data(), out.data.size() * 8);
            if (saturation) *saturation = sat;
            return;
        }
        const int64_t t = std::min<int64_t>(nthreads, m);
        std::vector<int64_t> sats(t, 0);
        std::vector<std::string> errs(t);
        std::vector<std::thread> pool;
        for (int64_t b = 0; b < t; ++b) {
            pool.emplace_back([&, b] {
                const int64_t r0 = m * b / t, r1 = m * (b + 1) / t;
                try {
                    const fq::Matrix out =
                        fq::run_layer(l->cfg, mat(x + r0 * k, r1 - r0, k), sats[b]);
                    std::memcpy(y + r0 * n, out.data.data(), out.data.size() * 8);
                } catch (const std::exception& e) {
                    errs[b] = e.what();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
        int64_t total = 0;
        for (int64_t s : sats) total += s;
        if (saturation) *saturation = total;
    });
}

// The activation half of run_layer (pipeline.cpp:164-167): divide_columns ->
// flatten_tensor(saturating) -> repeat_columns -> quantize_per_tensor(static).
int fqref_quantized_acts(const fqref_layer* l, const double* x, int64_t m, int32_t* qx,
                         int64_t* saturation) {
    return guard([&] {
        const auto& c = l->cfg;
        const int64_t k = c.plan_x.channels();
        int64_t sat = 0;
        const fq::Matrix divided = fq::divide_columns(mat(x, m, k), c.smooth_scales.s);
        const fq::Matrix flat = fq::flatten_tensor(divided, c.plan_x, sat);
        const fq::Matrix rep = fq::repeat_columns(flat, c.plan_w);
        const fq::QuantizedTensor q = fq::quantize_per_tensor(rep, c.bits, c.act_scale);
        std::copy(q.q.data.begin(), q.q.data.end(), qx);
        if (saturation) *saturation = sat;
    });
}

// fq::int_matmul_raw (quantize.cpp:166-188).
int fqref_int_matmul_raw(const int32_t* qx, int64_t m, int64_t kp, int bits_x,
                         const int32_t* qw, int64_t n, int bits_w, int64_t* acc) {
    return guard([&] {
        fq::QuantizedTensor a, b;
        a.q = fq::IntMatrix(m, kp, std::vector<int32_t>(qx, qx + m * kp));
        a.params = {bits_x, 1.0};
        b.q = fq::IntMatrix(kp, n, std::vector<int32_t>(qw, qw + kp * n));
        b.params = {bits_w, 1.0};
        const auto r = fq::int_matmul_raw(a, b);
        std::copy(r.begin(), r.end(), acc);
    });
}

// fq::build_flatten_plan (flatten.cpp:17-45).
int fqref_build_flatten_plan(const double* maxes, int64_t k, double t, int64_t block,
                             int64_t* e, int64_t* off, int64_t* c_ext, int64_t* padded) {
    return guard([&] {
        const fq::FlattenPlan p =
            fq::build_flatten_plan(std::span<const double>(maxes, k), t, block);
        std::copy(p.extensions.begin(), p.extensions.end(), e);
        if (off) std::copy(p.ext_offset.begin(), p.ext_offset.end(), off);
        *c_ext = p.c_extend;
        *padded = p.padded_width;
    });
}

// fq::split_against_threshold (flatten.cpp:8-15).
void fqref_split_against_threshold(double a, double t, int64_t* count, double* rem) {
    const fq::SlotSplit s = fq::split_against_threshold(a, t);
    *count = s.count;
    *rem = s.remainder;
}

// fq::flatten_tensor strict (flatten.cpp:128-130) or saturating (:132-134).
int fqref_flatten_tensor(const double* x, int64_t rows, int64_t cols, double t,
                         const int64_t* e, int64_t block, int saturating, double* out,
                         int64_t* sat) {
    return guard([&] {
        const fq::FlattenPlan p = plan_from(t, e, cols, block);
        fq::Matrix r;
        if (saturating) {
            int64_t s = 0;
            r = fq::flatten_tensor(mat(x, rows, cols), p, s);
            if (sat) *sat = s;
        } else {
            r = fq::flatten_tensor(mat(x, rows, cols), p);
        }
        std::copy(r.data.begin(), r.data.end(), out);
    });
}

// fq::flatten_rows strict (flatten.cpp:154-156).
int fqref_flatten_rows(const double* w, int64_t rows, int64_t cols, double t, const int64_t* e,
                       int64_t block, double* out) {
    return guard([&] {
        const fq::Matrix r = fq::flatten_rows(mat(w, rows, cols), plan_from(t, e, rows, block));
        std::copy(r.data.begin(), r.data.end(), out);
    });
}

// fq::repeat_channels (flatten.cpp:136-152) / fq::repeat_columns (:158-174).
int fqref_repeat(const double* m, int64_t rows, int64_t cols, double t, const int64_t* e,
                 int64_t block, int by_columns, double* out) {
    return guard([&] {
        fq::Matrix r;
        if (by_columns)
            r = fq::repeat_columns(mat(m, rows, cols), plan_from(t, e, cols, block));
        else
            r = fq::repeat_channels(mat(m, rows, cols), plan_from(t, e, rows, block));
        std::copy(r.data.begin(), r.data.end(), out);
    });
}

// fq::quantize_per_tensor (quantize.cpp:23-48); scale == nullptr -> absmax.
int fqref_quantize_per_tensor(const double* m, int64_t rows, int64_t cols, int bits,
                              const double* scale, int32_t* q, double* scale_out) {
    return guard([&] {
        std::optional<double> ov;
        if (scale) ov = *scale;
        const fq::QuantizedTensor r = fq::quantize_per_tensor(mat(m, rows, cols), bits, ov);
        std::copy(r.q.data.begin(), r.q.data.end(), q);
        if (scale_out) *scale_out = r.params.scale;
    });
}

// fq::collect_channel_maxes (calibration.cpp:9-28), fq::derive_truncation
// (:75-90), fq::smoothing_scales (smoothing.cpp:34-66), fq::row_max_abs.
int fqref_collect_channel_maxes(const double* calib, int64_t samples, int64_t rows, int64_t k,
                                double* maxes) {
    return guard([&] {
        std::vector<fq::Matrix> cs;
        for (int64_t s = 0; s < samples; ++s) cs.push_back(mat(calib + s * rows * k, rows, k));
        const fq::ChannelStats st = fq::collect_channel_maxes(cs);
        std::copy(st.max_abs.begin(), st.max_abs.end(), maxes);
    });
}

int fqref_derive_truncation(const double* maxes, int64_t k, double beta, int clip, double* t) {
    return guard([&] {
        *t = fq::derive_truncation(std::span<const double>(maxes, k), beta, clip != 0).threshold;
    });
}

int fqref_smoothing_scales(const double* act_max, const double* w_max, int64_t k, double alpha,
                           double* s) {
    return guard([&] {
        const fq::SmoothingScales r = fq::smoothing_scales(std::span<const double>(act_max, k),
                                                           std::span<const double>(w_max, k),
                                                           alpha);
        std::copy(r.s.begin(), r.s.end(), s);
    });
}

// The on-disk contract of the reference CLI (flattenquant_cli.cpp:199-238
// cmd_quantize, :241-281 load_recipes / cmd_infer), driven through the
// reference's own schemas.cpp (recipe JSON) and archive.cpp (FQTA): `layers`
// recipes named names[i] are written as recipe.json + <qmodel> with
// "<layer>.qweight" int32 tensors, exactly as cmd_quantize writes them.
int fqref_write_model(const fqref_layer* const* layers, const char* const* names, int64_t count,
                      const char* recipe_path, const char* qmodel_path) {
    return guard([&] {
        fq::TensorArchive qmodel;
        fq::RecipeFile recipe;
        recipe.options = layers[0]->cfg.options;
        for (int64_t i = 0; i < count; ++i) {
            qmodel.add(std::string(names[i]) + ".qweight", layers[i]->cfg.weight_q.q);
            recipe.layers.push_back({names[i], layers[i]->cfg});
        }
        fq::write_archive(qmodel, qmodel_path);
        fq::save_text(recipe_path, fq::to_json(recipe));
    });
}

// An FQTA archive of f64 tensors (names[i], rows[i] x cols[i], data[i]).
int fqref_write_f64_archive(const char* path, const char* const* names, const double* const* data,
                            const int64_t* rows, const int64_t* cols, int64_t count) {
    return guard([&] {
        fq::TensorArchive a;
        for (int64_t i = 0; i < count; ++i) a.add(names[i], mat(data[i], rows[i], cols[i]));
        fq::write_archive(a, path);
    });
}

// cmd_infer (flattenquant_cli.cpp:254-281) with load_recipes (:241-252): the
// reference's own parse_recipe_json + read_archive + run_layer + write_archive.
int fqref_infer(const char* qmodel_path, const char* recipe_path, const char* input_path,
                const char* out_path, int64_t* saturated_total, int64_t* ran_out) {
    return guard([&] {
        const fq::RecipeFile recipe = fq::parse_recipe_json(fq::load_text(recipe_path));
        const fq::TensorArchive qmodel = fq::read_archive(qmodel_path);
        std::vector<std::pair<std::string, fq::LayerQuantConfig>> configs;
        for (const auto& rec : recipe.layers) {
            fq::LayerQuantConfig cfg = rec.config;
            cfg.weight_q.q = qmodel.require(rec.layer + ".qweight").int_matrix();
            configs.emplace_back(rec.layer, std::move(cfg));
        }
        const fq::TensorArchive inputs = fq::read_archive(input_path);
        fq::TensorArchive outputs;
        std::int64_t sat_total = 0, ran = 0;
        for (const auto& entry : inputs.entries) {
            const auto slash = entry.name.find('/');
            if (slash == std::string::npos || !entry.is_float()) continue;
            const std::string layer = entry.name.substr(0, slash);
            const fq::LayerQuantConfig* cfg = nullptr;
            for (const auto& c : configs)
                if (c.first == layer) cfg = &c.second;
            if (cfg == nullptr) throw std::runtime_error("no recipe for " + layer);
            std::int64_t sat = 0;
            outputs.add(entry.name, fq::run_layer(*cfg, entry.matrix(), sat));
            sat_total += sat;
            ++ran;
        }
        if (ran == 0) throw std::runtime_error("input archive has no <layer>/<name> tensors");
        fq::write_archive(outputs, out_path);
        if (saturated_total) *saturated_total = sat_total;
        if (ran_out) *ran_out = ran;
    });
}

}  // extern "C"
