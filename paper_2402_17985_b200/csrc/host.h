// host.h — host-side plan arithmetic and gather-map compiler (host.cu).
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/fqg.h"

namespace fqg {

constexpr int64_t kMaxPieces = 4095;  // piece index is stored in 12 bits of a map entry

// FQG_I4 packing: per group of 32 consecutive k, byte i (0..15) holds k = 32g + i
// in its low nibble and k = 32g + 16 + i in its high nibble.
inline int64_t i4_byte(int64_t k) { return (k >> 5) * 16 + (k & 15); }
inline int i4_shift(int64_t k) { return (k & 16) ? 4 : 0; }

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
    std::vector<int32_t> off_x;     // [K] plan_x ext_offset
    // Channels with extension slots get a compact index ecomp[j] (else -1);
    // plan_x extension slot K + i holds piece p of channel j: xsrc[i] = ecomp[j] << 12 | p.
    std::vector<int32_t> ecomp, xsrc;
    int64_t n_ext = 0;
    std::vector<int32_t> capw_src;  // [K] plan_w capacity of source row j
    // Final columns [C1, K') are plan_w extension copies of flattened columns:
    // wsrc[k' - C1] = r, or -1 for plan_w alignment padding.
    std::vector<int32_t> wsrc;
    int64_t c1 = 0, width_x = 0;
};
GatherMaps compile_maps(const Plan& px, const Plan& pw);

double derive_truncation(const double* maxes, int64_t k, double beta, bool clip);
void smoothing_scales(const double* act_max, const double* w_max, int64_t k, double alpha,
                      double* s);
void synthetic_layer(const fqg_synth_opts& o, int64_t index, double* weight, double* calib,
                     double* test_input, int64_t test_rows);

}  // namespace fqg
