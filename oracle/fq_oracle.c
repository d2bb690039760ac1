/* fq_oracle.c — TEST INFRASTRUCTURE ONLY (see fq_oracle.h).
 *
 * A literal, single-threaded restatement of the reference hot path in C11.
 * Each function follows the reference statement order so that every FP64
 * operation (IEEE divide, fmod, llround, round, clamp) is evaluated on the same
 * operands in the same order; compile with -ffp-contract=off (oracle/Makefile).
 * File:line citations are into /root/reference/proj/core/src/.
 */
#include "fq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OK 0
#define EINVAL_ -2
#define ERUNTIME -3

/* flatten.cpp:8-15 — fmod is exact; count = llround((a - rem) / T). */
void fqo_split_against_threshold(double abs_value, double t, int64_t* count, double* rem) {
    const double r = fmod(abs_value, t);
    *rem = r;
    *count = (int64_t)llround((abs_value - r) / t);
}

int64_t fqo_padded_width(const int64_t* e, int64_t k, int64_t block) {
    int64_t w = k;
    for (int64_t j = 0; j < k; ++j) w += e[j];
    return (w + block - 1) / block * block; /* flatten.cpp:42-43 */
}

/* flatten.cpp:17-45 */
int fqo_build_flatten_plan(const double* maxes, int64_t k, double t, int64_t block, int64_t* e,
                           int64_t* off, int64_t* c_ext, int64_t* padded) {
    if (t <= 0.0) return EINVAL_;
    if (block < 1) return EINVAL_;
    if (k <= 0) return EINVAL_;
    int64_t c = 0;
    for (int64_t j = 0; j < k; ++j) {
        const double mx = maxes[j];
        if (mx < 0.0 || !isfinite(mx)) return EINVAL_;
        if (off) off[j] = c;
        int64_t cnt;
        double rem;
        fqo_split_against_threshold(mx, t, &cnt, &rem);
        e[j] = cnt;
        c += cnt;
    }
    *c_ext = c;
    *padded = (k + c + block - 1) / block * block;
    return OK;
}

/* smoothing.cpp:68-79 — X'[i,j] = X[i,j] / s_j (division, not reciprocal). */
void fqo_divide_columns(const double* x, int64_t rows, int64_t cols, const double* s,
                        double* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = x[i * cols + j] / s[j];
}

/* smoothing.cpp:81-92 — W'[i,j] = W[i,j] * s_i. */
void fqo_scale_rows(const double* w, int64_t rows, int64_t cols, const double* s, double* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = w[i * cols + j] * s[i];
}

/* flatten.cpp:60-74 — returns 1 when the element saturates. Slot p of the
 * ordered list [j, ext...] receives the value through out[idx[p]]. */
static int split_into_slots(double x, double t, int64_t capacity, double* out,
                            const int64_t* slot_index) {
    const double sign = x < 0.0 ? -1.0 : 1.0;
    int64_t count;
    double rem;
    fqo_split_against_threshold(fabs(x), t, &count, &rem);
    int saturated = 0;
    if (count > capacity || (count == capacity && rem > 0.0)) {
        count = capacity;
        rem = 0.0;
        saturated = 1;
    }
    for (int64_t p = 0; p < count; ++p) out[slot_index[p]] = sign * t;
    if (count < capacity) out[slot_index[count]] = sign * rem;
    return saturated;
}

static void prefix(const int64_t* e, int64_t k, int64_t* off) {
    int64_t c = 0;
    for (int64_t j = 0; j < k; ++j) {
        off[j] = c;
        c += e[j];
    }
}

/* flatten.cpp:76-102 (columns are channels) */
int fqo_flatten_columns(const double* x, int64_t rows, int64_t cols, double t, const int64_t* e,
                        int64_t block, int strict, double* out, int64_t* sat) {
    const int64_t pw = fqo_padded_width(e, cols, block);
    int64_t* off = malloc(sizeof(int64_t) * (size_t)cols);
    int64_t emax = 0;
    for (int64_t j = 0; j < cols; ++j) emax = e[j] > emax ? e[j] : emax;
    int64_t* idx = malloc(sizeof(int64_t) * (size_t)(emax + 1));
    prefix(e, cols, off);
    memset(out, 0, sizeof(double) * (size_t)(rows * pw));
    int64_t saturated = 0;
    int rc = OK;
    for (int64_t i = 0; i < rows && rc == OK; ++i) {
        for (int64_t j = 0; j < cols; ++j) {
            const int64_t first = cols + off[j];
            idx[0] = i * pw + j;
            for (int64_t p = 1; p <= e[j]; ++p) idx[p] = i * pw + first + p - 1;
            if (split_into_slots(x[i * cols + j], t, e[j] + 1, out, idx)) {
                if (strict) {
                    rc = ERUNTIME;
                    break;
                }
                ++saturated;
            }
        }
    }
    if (sat) *sat = saturated;
    free(off);
    free(idx);
    return rc;
}

/* flatten.cpp:104-124 (rows are channels) */
int fqo_flatten_rows(const double* w, int64_t rows, int64_t cols, double t, const int64_t* e,
                     int64_t block, int strict, double* out) {
    const int64_t pw = fqo_padded_width(e, rows, block);
    int64_t* off = malloc(sizeof(int64_t) * (size_t)rows);
    int64_t emax = 0;
    for (int64_t j = 0; j < rows; ++j) emax = e[j] > emax ? e[j] : emax;
    int64_t* idx = malloc(sizeof(int64_t) * (size_t)(emax + 1));
    prefix(e, rows, off);
    memset(out, 0, sizeof(double) * (size_t)(pw * cols));
    int rc = OK;
    for (int64_t j = 0; j < rows && rc == OK; ++j) {
        const int64_t first = rows + off[j];
        for (int64_t c = 0; c < cols; ++c) {
            idx[0] = j * cols + c;
            for (int64_t p = 1; p <= e[j]; ++p) idx[p] = (first + p - 1) * cols + c;
            if (split_into_slots(w[j * cols + c], t, e[j] + 1, out, idx) && strict) {
                rc = ERUNTIME;
                break;
            }
        }
    }
    free(off);
    free(idx);
    return rc;
}

/* flatten.cpp:136-152 — row j copied into every slot of slot_of(j). */
void fqo_repeat_channels(const double* w, int64_t rows, int64_t cols, const int64_t* e,
                         int64_t block, double* out) {
    const int64_t pw = fqo_padded_width(e, rows, block);
    int64_t* off = malloc(sizeof(int64_t) * (size_t)rows);
    prefix(e, rows, off);
    memset(out, 0, sizeof(double) * (size_t)(pw * cols));
    for (int64_t j = 0; j < rows; ++j) {
        const int64_t first = rows + off[j];
        for (int64_t c = 0; c < cols; ++c) {
            const double v = w[j * cols + c];
            out[j * cols + c] = v;
            for (int64_t p = 0; p < e[j]; ++p) out[(first + p) * cols + c] = v;
        }
    }
    free(off);
}

/* flatten.cpp:158-174 — column j copied into every slot of slot_of(j). */
void fqo_repeat_columns(const double* x, int64_t rows, int64_t cols, const int64_t* e,
                        int64_t block, double* out) {
    const int64_t pw = fqo_padded_width(e, cols, block);
    int64_t* off = malloc(sizeof(int64_t) * (size_t)cols);
    prefix(e, cols, off);
    memset(out, 0, sizeof(double) * (size_t)(rows * pw));
    for (int64_t i = 0; i < rows; ++i) {
        for (int64_t j = 0; j < cols; ++j) {
            const double v = x[i * cols + j];
            out[i * pw + j] = v;
            const int64_t first = cols + off[j];
            for (int64_t p = 0; p < e[j]; ++p) out[i * pw + first + p] = v;
        }
    }
    free(off);
}

/* matrix.cpp:71-75 */
double fqo_max_abs(const double* m, int64_t n) {
    double mx = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double a = fabs(m[i]);
        mx = mx < a ? a : mx; /* std::max(mx, |v|) */
    }
    return mx;
}

/* quantize.cpp:23-48 — q = clamp(round(v / s), -qmax, qmax), round half away. */
int fqo_quantize_per_tensor(const double* m, int64_t n, int bits, double scale_override,
                            int32_t* q, double* scale_out) {
    if (bits != 4 && bits != 8) return EINVAL_;
    const double qmax = (double)((1 << (bits - 1)) - 1);
    double s;
    if (scale_override > 0.0) {
        if (!isfinite(scale_override)) return EINVAL_;
        s = scale_override;
    } else if (scale_override < 0.0 || scale_override == 0.0) {
        /* caller encodes "no override" as 0 or negative */
        const double mx = fqo_max_abs(m, n);
        if (mx == 0.0) return ERUNTIME; /* "degenerate scale" */
        s = mx / qmax;
    } else {
        return EINVAL_;
    }
    for (int64_t i = 0; i < n; ++i) {
        const double r = round(m[i] / s);
        const double c = r < -qmax ? -qmax : (qmax < r ? qmax : r); /* std::clamp */
        q[i] = (int32_t)c;
    }
    if (scale_out) *scale_out = s;
    return OK;
}

/* quantize.cpp:160-164 */
int fqo_accumulator_bound_ok(int64_t qmax_x, int64_t qmax_w, int64_t inner) {
    if (qmax_x <= 0 || qmax_w <= 0 || inner <= 0) return 0;
    return inner <= INT64_MAX / (qmax_x * qmax_w);
}

/* quantize.cpp:166-188 */
int fqo_int_matmul_raw(const int32_t* qx, int64_t m, int64_t kp, int bits_x, const int32_t* qw,
                       int64_t n, int bits_w, int64_t* acc) {
    const int64_t qmx = (1 << (bits_x - 1)) - 1, qmw = (1 << (bits_w - 1)) - 1;
    if (!fqo_accumulator_bound_ok(qmx, qmw, kp)) return EINVAL_;
    memset(acc, 0, sizeof(int64_t) * (size_t)(m * n));
    for (int64_t i = 0; i < m; ++i) {
        for (int64_t k = 0; k < kp; ++k) {
            const int64_t a = qx[i * kp + k];
            if (a == 0) continue;
            const int32_t* b = qw + k * n;
            int64_t* c = acc + i * n;
            for (int64_t j = 0; j < n; ++j) c[j] += a * (int64_t)b[j];
        }
    }
    return OK;
}

/* quantize.cpp:190-198 — the product s_x*s_w is formed once in FP64. */
void fqo_int_matmul_dequant(const int64_t* acc, int64_t count, double s_x, double s_w,
                            double* y) {
    const double s = s_x * s_w;
    for (int64_t i = 0; i < count; ++i) y[i] = (double)acc[i] * s;
}

/* calibration.cpp:9-28 */
void fqo_collect_channel_maxes(const double* calib, int64_t samples, int64_t rows, int64_t k,
                               double* maxes) {
    for (int64_t j = 0; j < k; ++j) maxes[j] = 0.0;
    for (int64_t s = 0; s < samples; ++s)
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < k; ++j) {
                const double a = fabs(calib[(s * rows + i) * k + j]);
                maxes[j] = maxes[j] < a ? a : maxes[j];
            }
}

static int cmp_double(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x > y) - (x < y);
}

/* calibration.cpp:30-48 — linear interpolation between order statistics. */
static double at_fraction(const double* sorted, int64_t n, double p) {
    const double pos = p * (double)(n - 1);
    const int64_t lo = (int64_t)pos;
    const int64_t hi = lo + 1 < n - 1 ? lo + 1 : n - 1;
    const double frac = pos - (double)lo;
    return sorted[lo] + frac * (sorted[hi] - sorted[lo]);
}

/* calibration.cpp:75-90 (clip: :50-58, threshold: :60-73) */
int fqo_derive_truncation(const double* maxes, int64_t k, double beta, int clip, double* t) {
    if (k <= 0) return EINVAL_;
    double* sorted = malloc(sizeof(double) * (size_t)k);
    memcpy(sorted, maxes, sizeof(double) * (size_t)k);
    qsort(sorted, (size_t)k, sizeof(double), cmp_double);
    const double q1 = at_fraction(sorted, k, 0.25);
    const double q3 = at_fraction(sorted, k, 0.75);
    const double iqr = q3 - q1;
    free(sorted);
    if (beta <= 0.0) return EINVAL_;
    const double lo = q1 - 1.5 * iqr, hi = q3 + 1.5 * iqr;
    double sum = 0.0;
    for (int64_t j = 0; j < k; ++j) {
        double v = maxes[j];
        if (clip) v = v < lo ? lo : (hi < v ? hi : v); /* std::clamp */
        sum += v;
    }
    const double mean = sum / (double)k;
    if (mean <= 0.0) return ERUNTIME;
    *t = beta * mean;
    return OK;
}

static double sigmoid(double x) { return 1.0 / (1.0 + exp(-x)); }

/* smoothing.cpp:34-66 (mu/sigma of the ACTIVATION maxima for both sigmoids) */
int fqo_smoothing_scales(const double* act_max, const double* w_max, int64_t k, double alpha,
                         double* s) {
    if (k <= 0) return EINVAL_;
    if (alpha < 0.0 || alpha > 1.0) return EINVAL_;
    int nz_a = 0, nz_w = 0;
    for (int64_t j = 0; j < k; ++j) {
        nz_a |= act_max[j] != 0.0;
        nz_w |= w_max[j] != 0.0;
    }
    if (!nz_a || !nz_w) return EINVAL_;
    double sum = 0.0;
    for (int64_t j = 0; j < k; ++j) sum += act_max[j];
    const double mu = sum / (double)k;
    double sq = 0.0;
    for (int64_t j = 0; j < k; ++j) sq += (act_max[j] - mu) * (act_max[j] - mu);
    const double sigma = sqrt(sq / (double)k);
    for (int64_t j = 0; j < k; ++j) {
        const double na = sigma > 0.0 ? (act_max[j] - mu) / sigma : 0.0;
        const double nw = sigma > 0.0 ? (w_max[j] - mu) / sigma : 0.0;
        const double num = pow(sigmoid(na), alpha);
        const double den = pow(sigmoid(nw), 1.0 - alpha);
        s[j] = num / den;
    }
    return OK;
}

void fqo_layer_free(fqo_layer* l) {
    free(l->s);
    free(l->e_x);
    free(l->e_w);
    free(l->wq);
    memset(l, 0, sizeof(*l));
}

/* pipeline.cpp:76-152, O1/O2 with caller-pinned bits (no GPTQ, no KL). */
int fqo_quantize_layer_pinned(const double* w, int64_t k, int64_t n, const double* calib,
                              int64_t samples, int64_t rows, int bits, double alpha,
                              double beta, int64_t block, int smooth, int clip, fqo_layer* out) {
    int rc;
    if (samples < 1) return EINVAL_;
    if (bits != 4 && bits != 8) return EINVAL_;
    memset(out, 0, sizeof(*out));
    out->bits = bits;
    out->k = k;
    out->n = n;
    out->block = block;
    double* act_max = malloc(sizeof(double) * (size_t)k);
    double* w_max = malloc(sizeof(double) * (size_t)k);
    out->s = malloc(sizeof(double) * (size_t)k);
    fqo_collect_channel_maxes(calib, samples, rows, k, act_max); /* :89 */
    for (int64_t j = 0; j < k; ++j) {                              /* :90 row_max_abs */
        double mx = 0.0;
        for (int64_t c = 0; c < n; ++c) {
            const double a = fabs(w[j * n + c]);
            mx = mx < a ? a : mx;
        }
        w_max[j] = mx;
    }
    if (smooth) {
        rc = fqo_smoothing_scales(act_max, w_max, k, alpha, out->s); /* :94-95 */
        if (rc) goto fail;
    } else {
        for (int64_t j = 0; j < k; ++j) out->s[j] = 1.0;
    }
    double* w_s = malloc(sizeof(double) * (size_t)(k * n));
    fqo_scale_rows(w, k, n, out->s, w_s); /* :100 */
    for (int64_t j = 0; j < k; ++j) act_max[j] = act_max[j] / out->s[j]; /* :102-105 */
    rc = fqo_derive_truncation(act_max, k, beta, clip, &out->t_x);     /* :108 */
    if (rc) {
        free(w_s);
        goto fail;
    }
    out->e_x = malloc(sizeof(int64_t) * (size_t)k);
    int64_t cext;
    rc = fqo_build_flatten_plan(act_max, k, out->t_x, block, out->e_x, NULL, &cext, &out->c1);
    if (rc) {
        free(w_s);
        goto fail;
    }
    /* :114-120 weight side */
    double* w_rep = malloc(sizeof(double) * (size_t)(out->c1 * n));
    fqo_repeat_channels(w_s, k, n, out->e_x, block, w_rep);
    free(w_s);
    double* rmax = malloc(sizeof(double) * (size_t)out->c1);
    for (int64_t r = 0; r < out->c1; ++r) {
        double mx = 0.0;
        for (int64_t c = 0; c < n; ++c) {
            const double a = fabs(w_rep[r * n + c]);
            mx = mx < a ? a : mx;
        }
        rmax[r] = mx;
    }
    rc = fqo_derive_truncation(rmax, k + cext, beta, clip, &out->t_w); /* real (unpadded) rows */
    if (!rc) {
        out->e_w = malloc(sizeof(int64_t) * (size_t)out->c1);
        int64_t cext_w;
        rc = fqo_build_flatten_plan(rmax, out->c1, out->t_w, block, out->e_w, NULL, &cext_w,
                                    &out->kp);
    }
    free(rmax);
    if (rc) {
        free(w_rep);
        goto fail;
    }
    double* w_flat = malloc(sizeof(double) * (size_t)(out->kp * n));
    rc = fqo_flatten_rows(w_rep, out->c1, n, out->t_w, out->e_w, block, 1, w_flat);
    free(w_rep);
    if (rc) {
        free(w_flat);
        goto fail;
    }
    const double qmax = (double)((1 << (bits - 1)) - 1);
    out->act_scale = out->t_x / qmax; /* :138 */
    const double wmax = fqo_max_abs(w_flat, out->kp * n);
    if (wmax == 0.0) {
        free(w_flat);
        rc = ERUNTIME;
        goto fail;
    }
    out->s_w = wmax / qmax; /* :139-143 */
    out->wq = malloc(sizeof(int32_t) * (size_t)(out->kp * n));
    rc = fqo_quantize_per_tensor(w_flat, out->kp * n, bits, out->s_w, out->wq, NULL); /* :149 */
    free(w_flat);
    if (rc) goto fail;
    free(act_max);
    free(w_max);
    return OK;
fail:
    free(act_max);
    free(w_max);
    fqo_layer_free(out);
    return rc;
}

/* pipeline.cpp:159-169 */
/* The activation half of run_layer (pipeline.cpp:164-167): divide_columns ->
 * flatten_tensor (saturating) -> repeat_columns -> quantize_per_tensor with the
 * static act_scale. qx: M*K' int32. */
int fqo_quantize_acts(const fqo_layer* l, const double* x, int64_t m, int32_t* qx, int64_t* sat) {
    const int64_t k = l->k, c1 = l->c1, kp = l->kp;
    int rc;
    double* divided = malloc(sizeof(double) * (size_t)(m * k));
    fqo_divide_columns(x, m, k, l->s, divided);
    double* flat = malloc(sizeof(double) * (size_t)(m * c1));
    int64_t s = 0;
    rc = fqo_flatten_columns(divided, m, k, l->t_x, l->e_x, l->block, 0, flat, &s);
    free(divided);
    double* rep = malloc(sizeof(double) * (size_t)(m * kp));
    fqo_repeat_columns(flat, m, c1, l->e_w, l->block, rep);
    free(flat);
    rc = rc ? rc : fqo_quantize_per_tensor(rep, m * kp, l->bits, l->act_scale, qx, NULL);
    free(rep);
    if (sat) *sat = s;
    return rc;
}

int fqo_run_layer(const fqo_layer* l, const double* x, int64_t m, double* y, int64_t* sat,
                  int32_t* qx_out, int64_t* acc_out) {
    const int64_t kp = l->kp, n = l->n;
    int32_t* qx = qx_out ? qx_out : malloc(sizeof(int32_t) * (size_t)(m * kp));
    int64_t s = 0;
    int rc = fqo_quantize_acts(l, x, m, qx, &s);
    int64_t* acc = acc_out ? acc_out : malloc(sizeof(int64_t) * (size_t)(m * n));
    rc = rc ? rc : fqo_int_matmul_raw(qx, m, kp, l->bits, l->wq, n, l->bits, acc);
    if (!rc) fqo_int_matmul_dequant(acc, m * n, l->act_scale, l->s_w, y);
    if (sat) *sat = s;
    if (!qx_out) free(qx);
    if (!acc_out) free(acc);
    return rc;
}
