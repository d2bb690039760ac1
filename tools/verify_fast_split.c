/* Brute-force check that the fast exact arithmetic used by K1/K3 equals the
 * reference's IEEE operations (flatten.cpp:8-15, smoothing.cpp:75,
 * quantize.cpp:44):
 *   div:   q = fma(fma(-q0, s, x), r, q0), q0 = x*r, r = RN(1/s)   == x / s
 *   split: n0 = floor(a * rT); rem = fma(-n0, T, a) (+-1 correction)
 *          == (llround((a - fmod(a,T)) / T), fmod(a, T))
 * gcc -O2 -ffp-contract=off -march=x86-64-v3 verify_fast_split.c -lm */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t s_ = 88172645463325252ull;
static uint64_t rnd(void) { s_ ^= s_ << 13; s_ ^= s_ >> 7; s_ ^= s_ << 17; return s_; }
static double u01(void) { return (double)(rnd() >> 11) * 0x1.0p-53; }
static double bf16_round(double v) {
    float f = (float)v; uint32_t b; memcpy(&b, &f, 4);
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000u; memcpy(&f, &b, 4); return (double)f;
}


static double fast_div(double x, double s, double r) {
    const double q0 = x * r;
    const double e = fma(-q0, s, x);
    return fma(e, r, q0);
}
static void fast_split(double a, double t, double rt, long long cap, long long* n, double* rem) {
    double t0 = a * rt;
    if (t0 >= (double)(cap + 2)) { *n = cap + 2; *rem = 1.0; return; } /* saturated */
    double n0 = floor(t0);
    double r = fma(-n0, t, a);
    if (r < 0.0) { n0 -= 1.0; r = fma(-n0, t, a); }
    else if (r >= t) { n0 += 1.0; r = fma(-n0, t, a); }
    *n = (long long)n0; *rem = r;
}

int main(int argc, char** argv) {
    long long iters = argc > 1 ? atoll(argv[1]) : 100000000ll;
    if (argc > 2) s_ ^= (uint64_t)atoll(argv[2]) * 0x9E3779B97F4A7C15ull;
    long long bad_div = 0, bad_split = 0, bad_q = 0;
    for (long long it = 0; it < iters; ++it) {
        /* smoothing scale: lognormal-ish in [1e-3, 1e3]; x: bf16 values with outliers */
        double s = exp((u01() - 0.5) * 14.0);
        if ((it & 1023) == 0) s = 1.0 + (double)(rnd() % 7) * 0x1p-52;       /* near 1 */
        double x = bf16_round((u01() - 0.5) * exp((u01() - 0.3) * 12.0));
        if ((it & 7) == 0) x = (u01() - 0.5) * exp((u01() - 0.3) * 12.0);     /* f64 inputs */
        const double r = 1.0 / s;
        const double v = x / s, vf = fast_div(x, s, r);
        if (v != vf) { if (bad_div++ < 5) printf("div  x=%a s=%a ieee=%a fast=%a\n", x, s, v, vf); }
        /* split against a threshold drawn near v's magnitude, incl. exact multiples */
        const double a = fabs(v);
        double t = a / (1.0 + u01() * 40.0) + 1e-300;
        if ((it & 15) == 0) t = a / (double)(1 + rnd() % 50);                 /* exact-ish fits */
        if (t <= 0.0 || !isfinite(t)) continue;
        const long long cap = 1 + (long long)(rnd() % 200);
        const double rem_ref = fmod(a, t);
        const long long n_ref = llround((a - rem_ref) / t);
        long long n; double rem;
        fast_split(a, t, 1.0 / t, cap, &n, &rem);
        const int sat_ref = n_ref > cap || (n_ref == cap && rem_ref > 0.0);
        const int sat = n > cap || (n == cap && rem > 0.0);
        if (sat != sat_ref || (!sat && (n != n_ref || rem != rem_ref))) {
            if (bad_split++ < 5) printf("split a=%a t=%a ref=(%lld,%a) fast=(%lld,%a)\n", a, t, n_ref, rem_ref, n, rem);
        }
        /* remainder quantization: round(rem / s_x) vs fast_div */
        const double sx = t / 127.0;
        const double q_ref = round(rem_ref / sx), q = round(fast_div(rem_ref, sx, 1.0 / sx));
        if (q != q_ref) { if (bad_q++ < 5) printf("quant rem=%a sx=%a\n", rem_ref, sx); }
    }
    printf("iters=%lld bad_div=%lld bad_split=%lld bad_quant=%lld\n", iters, bad_div, bad_split, bad_q);
    return (bad_div || bad_split || bad_q) ? 1 : 0;
}
