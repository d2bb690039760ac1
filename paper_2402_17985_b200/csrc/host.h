// host.h — host-side plan arithmetic and gather-map compiler (host.cu).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/fqg.h"

namespace fqg {

constexpr int64_t kMaxPieces = 4095;  // piece index is stored in 12 bits of a map entry

struct SlotSplit {
    int64_t count = 0;
    double rem = 0.0;
};
SlotSplit split_against_threshold(double a, double t);

// fq::FlattenPlan (flatten.hpp:17-33) in plain vectors.
struct Plan {
    double threshold = 0.0;
    int64_t block = 32;
    std::vector<int64_t> ext, off;
    int64_t c_extend = 0;
    int64_t padded = 0;
};
Plan build_plan(const double* maxes, int64_t k, double t, int64_t block);
Plan plan_from_ext(double t, const int64_t* e, int64_t k, int64_t block);

// The composite maps over the final K' columns/rows:
//   amap[k'] = (j << 12) | p_x : activation column k' is piece p_x of channel j
//   wmap[k'] = (j << 12) | p_w : weight row k' is piece p_w of (smoothed) row j
//   -1 for alignment padding; wcap[k'] = plan_w capacity of that row.
struct GatherMaps {
    int64_t kp = 0;
    std::vector<int32_t> amap, wmap, wcap;
    std::vector<int32_t> cap_x;     // [K] plan_x capacity E_x + 1
    std::vector<int32_t> capw_src;  // [K] plan_w capacity of source row j
};
GatherMaps compile_maps(const Plan& px, const Plan& pw);

double derive_truncation(const double* maxes, int64_t k, double beta, bool clip);
void smoothing_scales(const double* act_max, const double* w_max, int64_t k, double alpha,
                      double* s);
void synthetic_layer(const fqg_synth_opts& o, int64_t index, double* weight, double* calib,
                     double* test_input, int64_t test_rows);

}  // namespace fqg
