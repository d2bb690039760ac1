// gptq.cu — the O3 offline weight path of fq::quantize_layer on the device
// (SURVEY.md §8f row 4): hessian_from_calibration (gptq.cpp:73-104),
// inverse_upper_factor (Cholesky, inverse of the lower factor, H^-1 and its
// Cholesky factor; gptq.cpp:14-70) and gptq_optimize (gptq.cpp:106-161).
//
// Exactness. The reference is sequential FP64 code; every output element is a
// fixed sequence of IEEE operations over an index in ascending order (the
// Hessian's sum over calibration rows, each Cholesky entry's sum over k < j,
// each inverse entry's sum over k in [j, i), each H^-1 entry's sum over k >=
// max(i, j), each weight's error updates over the block's columns). The device
// keeps every such sequence inside one thread, in the same order and with the
// same roundings (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn / __dsqrt_rn, no
// contraction), and parallelizes only across independent elements; the
// sequential dependencies (Cholesky columns, GPTQ columns) become kernel
// launches in order. The result, weight_q, equals the reference bit for bit.
#include <algorithm>
#include <cmath>
#include <vector>

#include "fqg_internal.h"
#include "gptq.h"

namespace fqg {
namespace {

constexpr int kT = 256;

unsigned blocks_for(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, (n + kT - 1) / kT)); }

// H[i][j] = sum_r 2 * x[r][i] * x[r][j] over rows with x[r][i] != 0 (gptq.cpp:88-96).
// 16 x 16 output tile per block, rows staged through shared memory; each thread
// owns one H entry and adds in ascending row order.
__global__ void __launch_bounds__(256) k_hessian(const double* __restrict__ x, int64_t rows, int dim,
                                                 double* __restrict__ h) {
    __shared__ double xi_s[32][16], xj_s[32][16];
    const int ti = threadIdx.x >> 4, tj = threadIdx.x & 15;
    const int i = blockIdx.y * 16 + ti, j = blockIdx.x * 16 + tj;
    double acc = 0.0;
    for (int64_t r0 = 0; r0 < rows; r0 += 32) {
        for (int e = threadIdx.x; e < 32 * 16; e += 256) {
            const int rr = e >> 4, cc = e & 15;
            const int64_t r = r0 + rr;
            const int gi = blockIdx.y * 16 + cc, gj = blockIdx.x * 16 + cc;
            xi_s[rr][cc] = (r < rows && gi < dim) ? x[r * dim + gi] : 0.0;
            xj_s[rr][cc] = (r < rows && gj < dim) ? x[r * dim + gj] : 0.0;
        }
        __syncthreads();
        const int nr = static_cast<int>(rows - r0 < 32 ? rows - r0 : 32);
        for (int rr = 0; rr < nr; ++rr) {
            const double xi = xi_s[rr][ti];
            if (xi == 0.0) continue;
            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(2.0, xi), xj_s[rr][tj]));
        }
        __syncthreads();
    }
    if (i < dim && j < dim) h[static_cast<int64_t>(i) * dim + j] = acc;
}

// One column j of cholesky_lower (gptq.cpp:14-31) in place: every thread forms
// the pivot d (the same sequence, redundantly) and its own entry below it.
__global__ void __launch_bounds__(kT) k_chol_col(double* __restrict__ a, int n, int j,
                                                 int* __restrict__ bad) {
    const int i = j + blockIdx.x * kT + threadIdx.x;
    const double* aj = a + static_cast<int64_t>(j) * n;
    double d = aj[j];
    for (int k = 0; k < j; ++k) d = __dsub_rn(d, __dmul_rn(aj[k], aj[k]));
    if (!(d > 0.0)) {
        if (i == j) *bad = 1;
        return;
    }
    const double pivot = __dsqrt_rn(d);
    if (i == j) {
        a[static_cast<int64_t>(j) * n + j] = pivot;
    } else if (i < n) {
        double* ai = a + static_cast<int64_t>(i) * n;
        double s = ai[j];
        for (int k = 0; k < j; ++k) s = __dsub_rn(s, __dmul_rn(ai[k], aj[k]));
        ai[j] = __ddiv_rn(s, pivot);
    }
    // the upper part of column j is zeroed (gptq.cpp:29)
    for (int u = blockIdx.x * kT + threadIdx.x; u < j; u += gridDim.x * kT)
        a[static_cast<int64_t>(u) * n + j] = 0.0;
}

// invert_lower (gptq.cpp:34-45): thread j owns column j of inv(L) (stored
// transposed, invT[j][i] = inv[i][j]) and runs its forward substitution.
__global__ void __launch_bounds__(kT) k_invert_lower(const double* __restrict__ l, int n,
                                                     double* __restrict__ invT) {
    const int j = blockIdx.x * kT + threadIdx.x;
    if (j >= n) return;
    double* col = invT + static_cast<int64_t>(j) * n;
    for (int i = 0; i < j; ++i) col[i] = 0.0;
    col[j] = __ddiv_rn(1.0, l[static_cast<int64_t>(j) * n + j]);
    for (int i = j + 1; i < n; ++i) {
        const double* li = l + static_cast<int64_t>(i) * n;
        double s = 0.0;
        for (int k = j; k < i; ++k) s = __dadd_rn(s, __dmul_rn(li[k], col[k]));
        col[i] = __ddiv_rn(-s, li[i]);
    }
}

// H^-1 = linv^T linv (gptq.cpp:54-64): entry (i, j), i <= j, sums k from j up.
__global__ void __launch_bounds__(kT) k_hinv(const double* __restrict__ invT, int n,
                                             double* __restrict__ hinv) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
    if (e >= static_cast<int64_t>(n) * n) return;
    const int i = static_cast<int>(e / n), j = static_cast<int>(e % n);
    if (i > j) return;
    const double* ci = invT + static_cast<int64_t>(i) * n;  // linv[k][i] = invT[i][k]
    const double* cj = invT + static_cast<int64_t>(j) * n;
    double s = 0.0;
    for (int k = j; k < n; ++k) s = __dadd_rn(s, __dmul_rn(ci[k], cj[k]));
    hinv[static_cast<int64_t>(i) * n + j] = s;
    hinv[static_cast<int64_t>(j) * n + i] = s;
}

__global__ void k_transpose(const double* __restrict__ a, int n, double* __restrict__ t) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
    if (e >= static_cast<int64_t>(n) * n) return;
    const int64_t i = e / n, j = e % n;
    t[j * n + i] = a[i * n + j];
}

// gptq_optimize, column j (gptq.cpp:129-135): q and the scaled error of row j.
__global__ void k_gptq_quant_row(const double* __restrict__ work, int64_t ncol, int j,
                                 const double* __restrict__ u, int kdim, double s, double qmax,
                                 int32_t* __restrict__ q, double* __restrict__ err_row) {
    const int64_t c = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
    if (c >= ncol) return;
    const double d = u[static_cast<int64_t>(j) * kdim + j];
    const double w = work[static_cast<int64_t>(j) * ncol + c];
    double r = round(__ddiv_rn(w, s));
    r = r < -qmax ? -qmax : (qmax < r ? qmax : r);
    q[static_cast<int64_t>(j) * ncol + c] = static_cast<int32_t>(r);
    err_row[c] = __ddiv_rn(__dsub_rn(w, __dmul_rn(r, s)), d);
}

// Propagation of the errors of block rows [j0, j1) into rows [k0, k1)
// (gptq.cpp:137-153): work[k][c] -= u[j][k] * err[j][c] for j ascending, skipping
// zero factors; each thread owns one (k, c).
__global__ void k_gptq_update(double* __restrict__ work, int64_t ncol, int k0, int k1, int j0,
                              int j1, int b0, const double* __restrict__ u, int kdim,
                              const double* __restrict__ err) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(kT) + threadIdx.x;
    const int64_t rows = k1 - k0;
    if (e >= rows * ncol) return;
    const int k = k0 + static_cast<int>(e / ncol);
    const int64_t c = e % ncol;
    double w = work[static_cast<int64_t>(k) * ncol + c];
    for (int j = j0; j < j1; ++j) {
        const double ujk = u[static_cast<int64_t>(j) * kdim + k];
        if (ujk == 0.0) continue;
        w = __dsub_rn(w, __dmul_rn(ujk, err[static_cast<int64_t>(j - b0) * ncol + c]));
    }
    work[static_cast<int64_t>(k) * ncol + c] = w;
}

void cholesky_lower(double* a, int n, int* bad) {
    for (int j = 0; j < n; ++j) {
        k_chol_col<<<blocks_for(n - j), kT>>>(a, n, j, bad);
        FQG_CUDA(cudaGetLastError());
    }
}

}  // namespace

void gptq_weight_q(const double* x_flat, int64_t rows, int dim, const double* w_flat, int64_t ncol,
                   double damping, double s, double qmax, int32_t* q_dev) {
    require(damping > 0.0, "hessian_from_calibration: damping must be > 0");
    require(s > 0.0, "gptq_optimize: per-tensor scale must be > 0");
    const size_t nn = static_cast<size_t>(dim) * dim;
    double *h = nullptr, *inv = nullptr, *work = nullptr, *err = nullptr, *u = nullptr;
    int* bad = nullptr;
    constexpr int kUpdateBlock = 128;  // gptq.cpp:11
    const int block = dim < kUpdateBlock ? dim : kUpdateBlock;
    FQG_CUDA(cudaMalloc(&h, nn * 8));
    struct Free {
        std::vector<void*> p;
        ~Free() {
            for (void* q : p) cudaFree(q);
        }
    } fr{{h}};
    FQG_CUDA(cudaMalloc(&inv, nn * 8));
    fr.p.push_back(inv);
    FQG_CUDA(cudaMalloc(&u, nn * 8));
    fr.p.push_back(u);
    FQG_CUDA(cudaMalloc(&work, static_cast<size_t>(dim) * ncol * 8));
    fr.p.push_back(work);
    FQG_CUDA(cudaMalloc(&err, static_cast<size_t>(block) * ncol * 8));
    fr.p.push_back(err);
    FQG_CUDA(cudaMalloc(&bad, 4));
    fr.p.push_back(bad);
    FQG_CUDA(cudaMemset(bad, 0, 4));

    // hessian_from_calibration: H, then the damping of the diagonal (gptq.cpp:97-103)
    k_hessian<<<dim3((dim + 15) / 16, (dim + 15) / 16), 256>>>(x_flat, rows, dim, h);
    FQG_CUDA(cudaGetLastError());
    std::vector<double> diag(static_cast<size_t>(dim));
    FQG_CUDA(cudaMemcpy2D(diag.data(), 8, h, static_cast<size_t>(dim + 1) * 8, 8, dim,
                          cudaMemcpyDeviceToHost));
    double diag_mean = 0.0;
    for (int i = 0; i < dim; ++i) diag_mean += diag[i];
    diag_mean /= static_cast<double>(dim);
    for (int i = 0; i < dim; ++i) diag[i] += damping * diag_mean;
    FQG_CUDA(cudaMemcpy2D(h, static_cast<size_t>(dim + 1) * 8, diag.data(), 8, 8, dim,
                          cudaMemcpyHostToDevice));

    // inverse_upper_factor (gptq.cpp:49-70)
    cholesky_lower(h, dim, bad);                                   // h := L
    k_invert_lower<<<blocks_for(dim), kT>>>(h, dim, inv);          // inv := inv(L)^T
    FQG_CUDA(cudaGetLastError());
    k_hinv<<<blocks_for(static_cast<int64_t>(dim) * dim), kT>>>(inv, dim, h);  // h := H^-1
    FQG_CUDA(cudaGetLastError());
    cholesky_lower(h, dim, bad);                                   // h := L2
    k_transpose<<<blocks_for(static_cast<int64_t>(dim) * dim), kT>>>(h, dim, u);  // u := L2^T
    FQG_CUDA(cudaGetLastError());
    int hbad = 0;
    FQG_CUDA(cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost));
    if (hbad) throw Error(FQG_ERR_RUNTIME, "ill-conditioned Hessian, increase damping");

    // gptq_optimize (gptq.cpp:119-160)
    FQG_CUDA(cudaMemcpy(work, w_flat, static_cast<size_t>(dim) * ncol * 8, cudaMemcpyDeviceToDevice));
    for (int b0 = 0; b0 < dim; b0 += block) {
        const int b1 = std::min(b0 + block, dim);
        for (int j = b0; j < b1; ++j) {
            k_gptq_quant_row<<<blocks_for(ncol), kT>>>(work, ncol, j, u, dim, s, qmax, q_dev,
                                                       err + static_cast<int64_t>(j - b0) * ncol);
            FQG_CUDA(cudaGetLastError());
            if (j + 1 < b1) {
                k_gptq_update<<<blocks_for(static_cast<int64_t>(b1 - j - 1) * ncol), kT>>>(
                    work, ncol, j + 1, b1, j, j + 1, b0, u, dim, err);
                FQG_CUDA(cudaGetLastError());
            }
        }
        if (b1 < dim) {
            k_gptq_update<<<blocks_for(static_cast<int64_t>(dim - b1) * ncol), kT>>>(
                work, ncol, b1, dim, b0, b1, b0, u, dim, err);
            FQG_CUDA(cudaGetLastError());
        }
    }
    FQG_CUDA(cudaDeviceSynchronize());
}

}  // namespace fqg
