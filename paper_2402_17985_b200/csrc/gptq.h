// gptq.h — the O3 weight path (gptq.cu), called by fqg_calibrate (calib.cu).
#pragma once
#include <cstdint>

namespace fqg {
// x_flat: device [rows][dim] flattened calibration activations; w_flat: device
// [dim][ncol] flattened weight; q_dev: device int32 [dim][ncol] (weight_q).
void gptq_weight_q(const double* x_flat, int64_t rows, int dim, const double* w_flat, int64_t ncol,
                   double damping, double s, double qmax, int32_t* q_dev);
}  // namespace fqg
