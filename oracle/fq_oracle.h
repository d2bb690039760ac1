/* fq_oracle.h — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * FlattenQuant reference hot path (/root/reference/proj/core). Used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the checker;
 * never linked or loaded by the product (paper_2402_17985_b200/).
 *
 * Parity of this restatement is pinned (tests/test_oracle.py) against
 *   (1) the reference's own known-answer tests (test_flatten.cpp, test_quantize.cpp,
 *       test_pipeline.cpp), restated as golden vectors in tests/golden/, and
 *   (2) the unmodified reference compiled here into oracle/_ref/libfq_ref.so.
 *
 * All matrices are row-major, dims int64. Return codes: 0 ok, -2 invalid
 * argument (std::invalid_argument in the reference), -3 runtime error
 * (std::runtime_error in the reference).
 */
#ifndef FQ_ORACLE_H
#define FQ_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* flatten.cpp:8-15 */
void fqo_split_against_threshold(double abs_value, double t, int64_t* count, double* rem);
/* flatten.cpp:17-45 ; off may be NULL */
int fqo_build_flatten_plan(const double* maxes, int64_t k, double t, int64_t block, int64_t* e,
                           int64_t* off, int64_t* c_ext, int64_t* padded);
/* smoothing.cpp:68-79 */
void fqo_divide_columns(const double* x, int64_t rows, int64_t cols, const double* s,
                        double* out);
/* smoothing.cpp:81-92 */
void fqo_scale_rows(const double* w, int64_t rows, int64_t cols, const double* s, double* out);
/* flatten.cpp:76-102 (strict: -3 on capacity overflow; else counts into *sat) */
int fqo_flatten_columns(const double* x, int64_t rows, int64_t cols, double t, const int64_t* e,
                        int64_t block, int strict, double* out, int64_t* sat);
/* flatten.cpp:104-124 */
int fqo_flatten_rows(const double* w, int64_t rows, int64_t cols, double t, const int64_t* e,
                     int64_t block, int strict, double* out);
/* flatten.cpp:136-152 */
void fqo_repeat_channels(const double* w, int64_t rows, int64_t cols, const int64_t* e,
                         int64_t block, double* out);
/* flatten.cpp:158-174 */
void fqo_repeat_columns(const double* x, int64_t rows, int64_t cols, const int64_t* e,
                        int64_t block, double* out);
/* plan geometry shared by the four functions above: padded = ceil_block(k + sum e) */
int64_t fqo_padded_width(const int64_t* e, int64_t k, int64_t block);
/* matrix.cpp:71-75 */
double fqo_max_abs(const double* m, int64_t n);
/* quantize.cpp:23-48 ; scale <= 0 means "no override" (absmax scale) */
int fqo_quantize_per_tensor(const double* m, int64_t n, int bits, double scale_override,
                            int32_t* q, double* scale_out);
/* quantize.cpp:160-164 */
int fqo_accumulator_bound_ok(int64_t qmax_x, int64_t qmax_w, int64_t inner);
/* quantize.cpp:166-188 (int64 accumulators, i-k-j, zero skip) */
int fqo_int_matmul_raw(const int32_t* qx, int64_t m, int64_t kp, int bits_x, const int32_t* qw,
                       int64_t n, int bits_w, int64_t* acc);
/* quantize.cpp:190-198 */
void fqo_int_matmul_dequant(const int64_t* acc, int64_t count, double s_x, double s_w,
                            double* y);

/* calibration.cpp:9-28 */
void fqo_collect_channel_maxes(const double* calib, int64_t samples, int64_t rows, int64_t k,
                               double* maxes);
/* calibration.cpp:30-48 / :50-58 / :60-73 / :75-90 */
int fqo_derive_truncation(const double* maxes, int64_t k, double beta, int clip, double* t);
/* smoothing.cpp:34-66 */
int fqo_smoothing_scales(const double* act_max, const double* w_max, int64_t k, double alpha,
                         double* s);

/* A frozen recipe (pipeline.hpp:37-49), flattened to arrays. */
typedef struct fqo_layer {
    int bits;
    int64_t k, n;
    double* s;        /* [k]   smoothing scales */
    double t_x, t_w;
    int64_t* e_x;     /* [k]   plan_x extensions */
    int64_t* e_w;     /* [c1]  plan_w extensions */
    int64_t c1, kp, block;
    int32_t* wq;      /* [kp*n] weight_q, row-major K'xN */
    double s_w, act_scale;
} fqo_layer;

/* pipeline.cpp:76-152 for modes O1/O2 with the bit width pinned by the caller
 * (select_bit_width's KL choice is out of the hot-path scope). */
int fqo_quantize_layer_pinned(const double* w, int64_t k, int64_t n, const double* calib,
                              int64_t samples, int64_t rows, int bits, double alpha,
                              double beta, int64_t block, int smooth, int clip, fqo_layer* out);
void fqo_layer_free(fqo_layer* l);

/* pipeline.cpp:164-167, the activation half of run_layer: qx M*K' int32 */
int fqo_quantize_acts(const fqo_layer* l, const double* x, int64_t m, int32_t* qx, int64_t* sat);

/* pipeline.cpp:159-169 (qx/acc optional debug outputs: M*K' int32, M*N int64) */
int fqo_run_layer(const fqo_layer* l, const double* x, int64_t m, double* y, int64_t* sat,
                  int32_t* qx_out, int64_t* acc_out);

#ifdef __cplusplus
}
#endif
#endif
