// host.cu — host-side arithmetic of the hot path's boundary (no device code):
// the flatten plan (flatten.cpp:8-45), the composite gather maps compiled from
// two plans, the offline recipe stages of quantize_layer for pinned bit widths
// (calibration.cpp, smoothing.cpp, pipeline.cpp:76-138) and the deterministic
// synthetic-layer generator (synthetic.hpp:17-36, synthetic.cpp:10-92).
//
// Compiled with -ffp-contract=off on the host side: every FP64 statement is
// evaluated exactly as the reference evaluates it.
#include <algorithm>
#include <cmath>
#include <random>
#include <vector>

#include "fqg_internal.h"
#include "host.h"

namespace fqg {

SlotSplit split_against_threshold(double a, double t) {
    SlotSplit s;
    s.rem = std::fmod(a, t);  // exact
    s.count = static_cast<int64_t>(std::llround((a - s.rem) / t));
    return s;
}

Plan build_plan(const double* maxes, int64_t k, double t, int64_t block) {
    require(t > 0.0, "build_flatten_plan: threshold must be > 0");
    require(block >= 1, "build_flatten_plan: block must be >= 1");
    require(k >= 1, "build_flatten_plan: no channels");
    Plan p;
    p.threshold = t;
    p.block = block;
    p.ext.resize(k);
    p.off.resize(k);
    int64_t c = 0;
    for (int64_t j = 0; j < k; ++j) {
        const double mx = maxes[j];
        require(mx >= 0.0 && std::isfinite(mx),
                "build_flatten_plan: channel maxima must be finite and >= 0");
        p.off[j] = c;
        p.ext[j] = split_against_threshold(mx, t).count;
        c += p.ext[j];
    }
    p.c_extend = c;
    p.padded = (k + c + block - 1) / block * block;
    return p;
}

Plan plan_from_ext(double t, const int64_t* e, int64_t k, int64_t block) {
    require(k >= 1 && block >= 1, "plan: bad geometry");
    Plan p;
    p.threshold = t;
    p.block = block;
    p.ext.assign(e, e + k);
    p.off.resize(k);
    int64_t c = 0;
    for (int64_t j = 0; j < k; ++j) {
        require(e[j] >= 0, "plan: negative extension count");
        p.off[j] = c;
        c += e[j];
    }
    p.c_extend = c;
    p.padded = (k + c + block - 1) / block * block;
    return p;
}

// Owner of a column of a flattened tensor: slot j -> (j, 0), extension slot
// channels() + off[j] + q -> (j, 1 + q), alignment padding -> (-1, 0).
static void owners(const Plan& p, std::vector<int64_t>& src, std::vector<int64_t>& piece) {
    const int64_t k = static_cast<int64_t>(p.ext.size());
    src.assign(p.padded, -1);
    piece.assign(p.padded, 0);
    for (int64_t j = 0; j < k; ++j) {
        src[j] = j;
        for (int64_t q = 0; q < p.ext[j]; ++q) {
            src[k + p.off[j] + q] = j;
            piece[k + p.off[j] + q] = 1 + q;
        }
    }
}

GatherMaps compile_maps(const Plan& px, const Plan& pw) {
    const int64_t k = static_cast<int64_t>(px.ext.size());
    require(static_cast<int64_t>(pw.ext.size()) == px.padded,
            "plan_w must have plan_x.padded_width channels");
    require(k < (1 << 19), "gather map: K must be < 524288");
    std::vector<int64_t> sx, px_piece, sw, pw_piece;
    owners(px, sx, px_piece);  // flat column r  -> (j, p_x)
    owners(pw, sw, pw_piece);  // final column k' -> (r, p_w)
    GatherMaps g;
    g.kp = pw.padded;
    g.amap.assign(g.kp, -1);
    g.wmap.assign(g.kp, -1);
    g.wcap.assign(g.kp, 1);
    g.cap_x.resize(k);
    g.off_x.resize(k);
    g.capw_src.resize(k);
    g.c1 = px.padded;
    g.width_x = k + px.c_extend;
    g.wsrc.assign(g.kp - px.padded, -1);
    for (int64_t kq = px.padded; kq < g.kp; ++kq) g.wsrc[kq - px.padded] = static_cast<int32_t>(sw[kq]);
    g.ecomp.assign(k, -1);
    g.xsrc.assign(px.c_extend, 0);
    for (int64_t j = 0; j < k; ++j) {
        if (px.ext[j] == 0) continue;
        g.ecomp[j] = static_cast<int32_t>(g.n_ext++);
        for (int64_t q = 0; q < px.ext[j]; ++q)
            g.xsrc[px.off[j] + q] = static_cast<int32_t>((g.ecomp[j] << 12) | (1 + q));
    }
    for (int64_t j = 0; j < k; ++j) {
        require(px.ext[j] + 1 <= kMaxPieces, "plan_x: a channel has more than 4095 extensions");
        g.cap_x[j] = static_cast<int32_t>(px.ext[j] + 1);
        g.off_x[j] = static_cast<int32_t>(px.off[j]);
        // Every copy row of source row j carries row j's maximum, hence the
        // same plan_w extension count (repeat_channels, flatten.cpp:136-152).
        g.capw_src[j] = static_cast<int32_t>(pw.ext[j] + 1);
    }
    for (int64_t kq = 0; kq < g.kp; ++kq) {
        const int64_t r = sw[kq];
        if (r < 0) continue;             // plan_w alignment padding
        const int64_t j = sx[r];
        if (j < 0) continue;             // plan_x alignment padding row/column
        // repeat_columns (flatten.cpp:158-174): final column kq carries flat
        // column r, i.e. piece px_piece[r] of source channel j.
        g.amap[kq] = static_cast<int32_t>((j << 12) | px_piece[r]);
        // flatten_rows of repeat_channels (flatten.cpp:104-152): final row kq is
        // piece pw_piece[kq] of repeated row r, a copy of source row j.
        require(pw.ext[r] + 1 <= kMaxPieces, "plan_w: a row has more than 4095 extensions");
        g.wmap[kq] = static_cast<int32_t>((j << 12) | pw_piece[kq]);
        g.wcap[kq] = static_cast<int32_t>(pw.ext[r] + 1);
    }
    return g;
}

// calibration.cpp:30-48 — quartiles by linear interpolation of order statistics.
static double at_fraction(const std::vector<double>& sorted, double p) {
    const double pos = p * static_cast<double>(sorted.size() - 1);
    const auto lo = static_cast<size_t>(pos);
    const size_t hi = std::min(lo + 1, sorted.size() - 1);
    const double frac = pos - static_cast<double>(lo);
    return sorted[lo] + frac * (sorted[hi] - sorted[lo]);
}

double derive_truncation(const double* maxes, int64_t k, double beta, bool clip) {
    require(k >= 1, "quartiles of empty vector");
    std::vector<double> sorted(maxes, maxes + k);
    std::sort(sorted.begin(), sorted.end());
    const double q1 = at_fraction(sorted, 0.25), q3 = at_fraction(sorted, 0.75);
    const double iqr = q3 - q1;
    require(beta > 0.0, "truncation_threshold: beta must be > 0");
    const double lo = q1 - 1.5 * iqr, hi = q3 + 1.5 * iqr;  // calibration.cpp:50-58
    double sum = 0.0;
    for (int64_t j = 0; j < k; ++j) sum += clip ? std::clamp(maxes[j], lo, hi) : maxes[j];
    const double mean = sum / static_cast<double>(k);  // calibration.cpp:60-73
    if (mean <= 0.0)
        throw Error(FQG_ERR_RUNTIME, "degenerate calibration: all channel maxima are zero");
    return beta * mean;
}

void smoothing_scales(const double* act_max, const double* w_max, int64_t k, double alpha,
                      double* s) {
    require(k >= 1, "smoothing_scales: empty channel maxima");
    require(alpha >= 0.0 && alpha <= 1.0, "smoothing_scales: alpha must be in [0,1]");
    bool nza = false, nzw = false;
    for (int64_t j = 0; j < k; ++j) {
        nza |= act_max[j] != 0.0;
        nzw |= w_max[j] != 0.0;
    }
    require(nza && nzw, "smoothing_scales: all channel maxima are zero");
    double sum = 0.0;
    for (int64_t j = 0; j < k; ++j) sum += act_max[j];
    const double mu = sum / static_cast<double>(k);
    double sq = 0.0;
    for (int64_t j = 0; j < k; ++j) sq += (act_max[j] - mu) * (act_max[j] - mu);
    const double sigma = std::sqrt(sq / static_cast<double>(k));
    auto sigmoid = [](double v) { return 1.0 / (1.0 + std::exp(-v)); };
    auto norm = [&](double v) { return sigma > 0.0 ? (v - mu) / sigma : 0.0; };
    for (int64_t j = 0; j < k; ++j) {
        const double num = std::pow(sigmoid(norm(act_max[j])), alpha);
        const double den = std::pow(sigmoid(norm(w_max[j])), 1.0 - alpha);
        s[j] = num / den;
    }
}

// ---------------------------------------------------------------- synthetic
namespace {
class Rng {
   public:
    Rng(uint64_t seed, uint64_t stream) : gen_(seed ^ (0x9E3779B97F4A7C15ULL * (stream + 1))) {}
    double uniform() { return static_cast<double>(gen_() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
    double gaussian() {
        const double u1 = static_cast<double>((gen_() >> 11) + 1) * 0x1.0p-53;
        const double u2 = static_cast<double>(gen_() >> 11) * 0x1.0p-53;
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
    }
    int64_t index(int64_t n) { return static_cast<int64_t>(gen_() % static_cast<uint64_t>(n)); }

   private:
    std::mt19937_64 gen_;
};
}  // namespace

void synthetic_layer(const fqg_synth_opts& o, int64_t index, double* weight, double* calib,
                     double* test_input, int64_t test_rows) {
    require(!(o.outlier_min > o.outlier_max || o.outlier_min < 0.0),
            "synthetic: bad outlier factor range");
    Rng rng(o.seed, static_cast<uint64_t>(index));
    const int64_t kc = o.in_channels, nc = o.out_channels;
    // pick_outlier_channels (synthetic.cpp:86-103): partial Fisher-Yates.
    int64_t count = 0;
    if (o.outlier_fraction > 0.0) {
        count = std::llround(o.outlier_fraction * static_cast<double>(kc));
        count = std::clamp<int64_t>(count, 1, kc);
    }
    std::vector<int64_t> all(kc);
    for (int64_t i = 0; i < kc; ++i) all[i] = i;
    for (int64_t i = 0; i < count; ++i) {
        const int64_t j = i + rng.index(kc - i);
        std::swap(all[i], all[j]);
    }
    std::vector<int64_t> picked(all.begin(), all.begin() + count);
    std::sort(picked.begin(), picked.end());
    std::vector<double> scale(kc);
    for (auto& s : scale) s = std::exp(o.channel_spread * rng.gaussian());
    for (int64_t c : picked) scale[c] = rng.uniform(o.outlier_min, o.outlier_max);
    const double tail_prob = rng.uniform(0.0, o.act_tail_prob_max);
    for (int64_t i = 0; i < kc; ++i) {
        const double row_scale = std::exp(o.weight_row_spread * rng.gaussian());
        for (int64_t j = 0; j < nc; ++j) {
            const double v = rng.gaussian() * row_scale;
            if (weight) weight[i * nc + j] = v;
        }
    }
    auto sample = [&](double* out, int64_t rows) {
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < kc; ++j) {
                double v = rng.gaussian();
                if (rng.uniform() < tail_prob) v *= o.act_tail_scale;
                const double x = v * scale[j];
                if (out) out[i * kc + j] = x;
            }
    };
    for (int64_t s = 0; s < o.samples; ++s) sample(calib ? calib + s * o.rows * kc : nullptr, o.rows);
    sample(test_input, test_rows);
}

}  // namespace fqg

using namespace fqg;

extern "C" {

void fqg_split_against_threshold(double abs_value, double t, int64_t* count, double* rem) {
    const SlotSplit s = split_against_threshold(abs_value, t);
    *count = s.count;
    *rem = s.rem;
}

int fqg_build_flatten_plan(const double* maxes, int64_t k, double t, int64_t block, int64_t* e,
                           int64_t* off, int64_t* c_extend, int64_t* padded_width) {
    return guard([&] {
        const Plan p = build_plan(maxes, k, t, block);
        std::copy(p.ext.begin(), p.ext.end(), e);
        if (off) std::copy(p.off.begin(), p.off.end(), off);
        *c_extend = p.c_extend;
        *padded_width = p.padded;
    });
}

void fqg_collect_channel_maxes(const double* calib, int64_t rows, int64_t k, double* m) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < k; ++j) m[j] = std::max(m[j], std::abs(calib[i * k + j]));
}

int fqg_recipe_plan(const double* weight, int64_t k, int64_t n, const double* act_maxes, int bits,
                    double alpha, double beta, int64_t block, int smooth, int clip, double* s,
                    double* t_x, int64_t* e_x, int64_t* c1, double* t_w, int64_t* e_w,
                    int64_t e_w_capacity, int64_t* kp, double* act_scale) {
    return guard([&] {
        require(bits == 4 || bits == 8, "bits must be 4 or 8");
        require(k >= 1 && n >= 1, "recipe: empty layer");
        // pipeline.cpp:89-105
        std::vector<double> wmax(k, 0.0), smax(k);
        for (int64_t j = 0; j < k; ++j)
            for (int64_t c = 0; c < n; ++c) wmax[j] = std::max(wmax[j], std::abs(weight[j * n + c]));
        if (smooth)
            smoothing_scales(act_maxes, wmax.data(), k, alpha, s);
        else
            std::fill(s, s + k, 1.0);
        for (int64_t j = 0; j < k; ++j) smax[j] = act_maxes[j] / s[j];
        // :108-109
        *t_x = derive_truncation(smax.data(), k, beta, clip != 0);
        const Plan px = build_plan(smax.data(), k, *t_x, block);
        std::copy(px.ext.begin(), px.ext.end(), e_x);
        *c1 = px.padded;
        // :114-119 — row maxima of repeat_channels(scale_rows(W, s), plan_x)
        std::vector<double> ws_max(k, 0.0), rmax(px.padded, 0.0);
        for (int64_t j = 0; j < k; ++j)
            for (int64_t c = 0; c < n; ++c)
                ws_max[j] = std::max(ws_max[j], std::abs(weight[j * n + c] * s[j]));
        for (int64_t j = 0; j < k; ++j) {
            rmax[j] = ws_max[j];
            for (int64_t q = 0; q < px.ext[j]; ++q) rmax[k + px.off[j] + q] = ws_max[j];
        }
        *t_w = derive_truncation(rmax.data(), k + px.c_extend, beta, clip != 0);
        const Plan pw = build_plan(rmax.data(), px.padded, *t_w, block);
        require(e_w_capacity >= px.padded, "recipe: e_w buffer smaller than plan_x.padded_width");
        std::copy(pw.ext.begin(), pw.ext.end(), e_w);
        *kp = pw.padded;
        *act_scale = *t_x / static_cast<double>((1 << (bits - 1)) - 1);  // :138
    });
}

int fqg_gather_maps(const int64_t* ext_x, int64_t k, int64_t block_x, const int64_t* ext_w,
                    int64_t block_w, int32_t* amap, int32_t* wmap, int32_t* wcap, int64_t* kp,
                    int64_t capacity) {
    return guard([&] {
        const Plan px = plan_from_ext(1.0, ext_x, k, block_x);
        const Plan pw = plan_from_ext(1.0, ext_w, px.padded, block_w);
        const GatherMaps g = compile_maps(px, pw);
        *kp = g.kp;
        require(capacity >= g.kp, "gather_maps: output capacity smaller than K'");
        std::copy(g.amap.begin(), g.amap.end(), amap);
        std::copy(g.wmap.begin(), g.wmap.end(), wmap);
        std::copy(g.wcap.begin(), g.wcap.end(), wcap);
    });
}

void fqg_synth_default(fqg_synth_opts* o) {
    *o = {32, 8, 128, 128, 0.01, 20.0, 100.0, 0.5, 0.08, 5.0, 0.25, 42};
}

int fqg_synthetic_layer(const fqg_synth_opts* o, int64_t index, double* weight, double* calib,
                        double* test_input, int64_t test_rows) {
    return guard([&] { synthetic_layer(*o, index, weight, calib, test_input, test_rows); });
}

}  // extern "C"
