// test_drop_in.cpp — the reference's own C++ API, unmodified (fq_core from
// /root/reference/proj/core, built into oracle/_ref/libfq_ref.so), next to the
// drop-in fq::gpu::run_layer (include/fq_gpu.hpp over libfqg.so). Mirrors the
// reference's tests: pipeline outputs and saturation counts must be identical
// bit for bit (pipeline.cpp:159-169), zero input gives zero output
// (test_pipeline.cpp:107-113), and a channel mismatch throws
// std::invalid_argument (test_pipeline.cpp:115-120). Exit code 0 = all PASS.
#include <cstdio>
#include <stdexcept>
#include <string>

#include "fq/pipeline.hpp"
#include "fq/synthetic.hpp"
#include "fq_gpu.hpp"

static int failures = 0;
static void check(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what.c_str());
    if (!ok) ++failures;
}

static fq::Matrix scaled(const fq::Matrix& m, double f) {
    fq::Matrix r = m;
    for (double& v : r.data) v *= f;
    return r;
}

int main() {
    fq::SyntheticOptions so;  // the reference synthetic model: seed 42
    so.layers = 4;
    so.in_channels = 256;
    so.out_channels = 192;
    so.rows = 48;
    so.samples = 4;
    for (int mode = 0; mode < 2; ++mode) {
        fq::QuantOptions qo;
        qo.mode = mode == 0 ? fq::QuantMode::O1 : fq::QuantMode::O2;
        if (mode == 1) qo.gamma = 1e6;  // force the 4-bit choice (test_pipeline.cpp:127)
        for (std::int64_t li = 0; li < so.layers; ++li) {
            const fq::SyntheticLayer L = fq::make_synthetic_layer(so, li);
            const fq::LayerQuantConfig cfg = fq::quantize_layer(L.weight, L.calib, qo);
            const std::string tag = std::string(mode == 0 ? "O1" : "O2") + " layer" +
                                    std::to_string(li) + " bits=" + std::to_string(cfg.bits);
            for (double f : {1.0, 3.0}) {
                const fq::Matrix x = scaled(L.test_input, f);
                std::int64_t sat_ref = -1, sat = -2;
                const fq::Matrix y_ref = fq::run_layer(cfg, x, sat_ref);
                const fq::Matrix y = fq::gpu::run_layer(cfg, x, sat);
                check(y == y_ref && sat == sat_ref,
                      tag + " x*" + std::to_string(f) + ": bit-exact run_layer, saturation " +
                          std::to_string(sat) + "/" + std::to_string(sat_ref));
            }
            const fq::Matrix vs = fq::vstack(L.calib);
            check(fq::gpu::run_layer(cfg, vs) == fq::run_layer(cfg, vs),
                  tag + ": stacked calibration rows (M=" + std::to_string(vs.rows) + ")");
        }
    }
    {
        const fq::SyntheticLayer L = fq::make_synthetic_layer(so, 0);
        const fq::LayerQuantConfig cfg = fq::quantize_layer(L.weight, L.calib, fq::QuantOptions{});
        check(fq::gpu::run_layer(cfg, fq::Matrix(3, so.in_channels)) ==
                  fq::Matrix(3, so.out_channels),
              "zero input produces zero output");
        bool threw = false;
        try {
            fq::gpu::run_layer(cfg, fq::Matrix(3, so.in_channels + 1));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        check(threw, "channel-count mismatch throws std::invalid_argument");
        fq::gpu::Layer explicit_layer(cfg);
        std::int64_t s1 = 0, s2 = 0;
        check(explicit_layer.run(L.test_input, s1) == fq::run_layer(cfg, L.test_input, s2) &&
                  s1 == s2,
              "fq::gpu::Layer explicit handle");
    }
    {  // the layer cache is keyed by recipe content: an in-place edit at the same
       // address (e.g. O2 weights replaced by O3 GPTQ weights) is never served stale
        const fq::SyntheticLayer L = fq::make_synthetic_layer(so, 1);
        fq::LayerQuantConfig cfg = fq::quantize_layer(L.weight, L.calib, fq::QuantOptions{});
        const fq::Matrix y0 = fq::gpu::run_layer(cfg, L.test_input);
        const auto* addr = cfg.weight_q.q.data.data();
        for (auto& v : cfg.weight_q.q.data) v = -v;
        const fq::Matrix y1 = fq::gpu::run_layer(cfg, L.test_input);
        check(addr == cfg.weight_q.q.data.data() && y1 == fq::run_layer(cfg, L.test_input) &&
                  !(y1 == y0),
              "in-place weight edit at the same address is not served from the cache");
        cfg.act_scale *= 0.5;
        check(fq::gpu::run_layer(cfg, L.test_input) == fq::run_layer(cfg, L.test_input),
              "edited act_scale is not served from the cache");
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "ALL PASS", failures);
    return failures ? 1 : 0;
}
