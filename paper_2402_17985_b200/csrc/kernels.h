// kernels.h — launch interfaces of the HBM-bound kernels in flatten.cu.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace fqg {

struct FlattenArgs {
    const void* x;                // [m][ldx] activations
    int x_dtype;                  // FQG_F64/F32/F16/BF16
    int64_t ldx;                  // elements
    int64_t m, k, kp;
    const double* s;              // [k] smoothing scales
    const double* rs;             // [k] RN(1 / s), for the exact FMA-corrected division
    const float* rs32;            // [k] RN32(1 / s), FP32 fast path
    const int32_t* cap;           // [k] plan_x capacity E_x + 1
    const int32_t* off;           // [k] plan_x ext_offset: piece p >= 1 of j at k + off + p - 1
    int64_t n_ext2;               // channels with >= 2 extension slots (queue sizing)
    const int32_t* wsrc;          // [kp - c1] flat column copied into final column c1 + i, or -1
    const int32_t* amap;          // [kp] (j << 12 | p) or -1 (K2 / reference map)
    int64_t c1, width;            // plan_x.padded_width, plan_x.width()
    double t;                     // plan_x threshold T_x
    double* scale;                // device; [0] = s_x (read; written in dynamic mode)
    unsigned long long* amax;     // dynamic mode: zeroed absmax cell, else nullptr
    double qmax;
    bool pack4;                   // packed int4 output
    uint8_t* q;                   // [m][ldq] bytes
    int64_t ldq;
    unsigned long long* sat;      // optional saturation accumulator
    int num_sms;
    // 16-bit fast path (flatten16.cu): per-channel certificate for this dtype
    // (k_tier1_tables), or nullptr to use the general kernel.
    const float* cj = nullptr;
    const uint16_t* pj = nullptr;
    const int32_t* hot = nullptr;  // channels always taking the exact path (pj = 0xFFFF)
    const int32_t* hotm = nullptr; // [nhot] x {j, capacity, ext_offset, RN32(1/s_j) bits}
    const int32_t* hotg = nullptr; // [k / 8] hot mask of the group | first hot index << 8
    int64_t nhot = 0;
    const int32_t* wsrc16 = nullptr;  // wsrc with padding (-1) mapped to column kp (a zero byte)
    double act_scale = 0.0;          // static s_x (host copy)
    int32_t* rowsum = nullptr;    // optional [m] sums of each final operand row
};
void flatten_quant(const FlattenArgs& a, cudaStream_t st);
// Row sums of a K1 operand [m][ldq] (int8, or signed packed int4).
void operand_rowsum(const uint8_t* q, int64_t ldq, int64_t m, int64_t kp, bool pack4,
                    int32_t* out, cudaStream_t st);

// flatten16.cu: certificate tables for bf16 (f16 = false) or f16 inputs, and
// the TMA-staged K1 (returns false when the call is outside its contract:
// dtype, dynamic scale, alignment, shared-memory size).
void tier1_tables(const double* s, int64_t k, double act_scale, double t, double qmax, bool f16,
                  float* cj, uint16_t* pj, cudaStream_t st);
bool flatten16(const FlattenArgs& a, cudaStream_t st);

void weight_absmax(const double* w, int64_t k, int64_t ncols, const double* s,
                   const int32_t* capw_src, double t_w, unsigned long long* amax,
                   unsigned int* overflow, int num_sms, cudaStream_t st);

void weight_quant(const double* w, int64_t ldw, int64_t n_begin, int64_t n, const double* s,
                  const int32_t* wmap, const int32_t* wcap, int64_t kp, double t_w, double s_w,
                  double qmax, bool pack4, uint8_t* wq, int64_t ldq, cudaStream_t st);

}  // namespace fqg
