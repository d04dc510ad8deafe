// cvk_complex.h -- complex FP64 scalar arithmetic shared by host and device.
//
// The reference computes with std::complex<double> under g++ -O2 on x86-64:
// no FMA contraction, multiply as (ac - bd, ad + bc), division through
// libgcc's __divdc3 (SURVEY.md Appendix B "Numerics of the host oracle").
// Everything here reproduces those roundings exactly; the library is built
// with nvcc --fmad=false / g++ -ffp-contract=off so no product is fused.
// tests/test_complex_div.py checks cvk_cdiv against libgcc bit for bit.
#pragma once

#if defined(__CUDACC__)
#define CVK_HD __host__ __device__ __forceinline__
#else
#define CVK_HD inline
#include <cmath>
#endif

#include <float.h>

#if !defined(__CUDACC__)
struct cvk_double2_host {
    double x, y;
};
typedef cvk_double2_host cvk_c;
#else
typedef double2 cvk_c;
#endif

CVK_HD cvk_c cvk_make(double re, double im) {
    cvk_c r;
    r.x = re;
    r.y = im;
    return r;
}

CVK_HD cvk_c cvk_add(cvk_c a, cvk_c b) { return cvk_make(a.x + b.x, a.y + b.y); }
CVK_HD cvk_c cvk_sub(cvk_c a, cvk_c b) { return cvk_make(a.x - b.x, a.y - b.y); }
CVK_HD cvk_c cvk_neg(cvk_c a) { return cvk_make(-a.x, -a.y); }
CVK_HD cvk_c cvk_conj(cvk_c a) { return cvk_make(a.x, -a.y); }

// (ac - bd, ad + bc), the libstdc++/GCC inline expansion (no NaN rescue).
CVK_HD cvk_c cvk_mul(cvk_c a, cvk_c b) {
    const double ac = a.x * b.x, bd = a.y * b.y, ad = a.x * b.y, bc = a.y * b.x;
    return cvk_make(ac - bd, ad + bc);
}

// conj(a) * b exactly as std::conj(x) * y is rounded in dot_hermitian.
CVK_HD cvk_c cvk_cmul(cvk_c a, cvk_c b) { return cvk_mul(cvk_conj(a), b); }

// real * complex: GCC scales both parts (no promotion to complex).
CVK_HD cvk_c cvk_scale(double s, cvk_c a) { return cvk_make(s * a.x, s * a.y); }
// complex / real: both parts divided.
CVK_HD cvk_c cvk_divr(cvk_c a, double s) { return cvk_make(a.x / s, a.y / s); }

// std::norm: re^2 + im^2.
CVK_HD double cvk_norm(cvk_c a) { return a.x * a.x + a.y * a.y; }

CVK_HD double cvk_fabs(double v) { return v < 0 ? -v : v; }

// libgcc __divdc3 (GCC >= 12 algorithm: Smith's method with scaling guards
// for huge / tiny operands).  The final NaN-recovery block of libgcc only
// fires for inf/NaN operands, which the solvers never produce, and is omitted.
CVK_HD cvk_c cvk_cdiv(cvk_c num, cvk_c den) {
    double a = num.x, b = num.y, c = den.x, d = den.y;
    const double RBIG = DBL_MAX / 2.0;
    const double RMIN = DBL_MIN;
    const double RMIN2 = DBL_EPSILON;
    const double RMINSCAL = 1.0 / DBL_EPSILON;
    const double RMAX2 = RBIG * RMIN2;
    double ratio, denom, x, y;
    if (cvk_fabs(c) < cvk_fabs(d)) {
        if (cvk_fabs(d) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (cvk_fabs(d) < RMIN2) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        } else if (((cvk_fabs(a) < RMIN) && (cvk_fabs(b) < RMAX2) && (cvk_fabs(d) < RMAX2)) ||
                   ((cvk_fabs(b) < RMIN) && (cvk_fabs(a) < RMAX2) && (cvk_fabs(d) < RMAX2))) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        }
        ratio = c / d;
        denom = (c * ratio) + d;
        if (cvk_fabs(ratio) > RMIN) {
            x = ((a * ratio) + b) / denom;
            y = ((b * ratio) - a) / denom;
        } else {
            x = ((c * (a / d)) + b) / denom;
            y = ((c * (b / d)) - a) / denom;
        }
    } else {
        if (cvk_fabs(c) >= RBIG) { a = a / 2; b = b / 2; c = c / 2; d = d / 2; }
        if (cvk_fabs(c) < RMIN2) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        } else if (((cvk_fabs(a) < RMIN) && (cvk_fabs(b) < RMAX2) && (cvk_fabs(c) < RMAX2)) ||
                   ((cvk_fabs(b) < RMIN) && (cvk_fabs(a) < RMAX2) && (cvk_fabs(c) < RMAX2))) {
            a = a * RMINSCAL; b = b * RMINSCAL; c = c * RMINSCAL; d = d * RMINSCAL;
        }
        ratio = d / c;
        denom = (d * ratio) + c;
        if (cvk_fabs(ratio) > RMIN) {
            x = ((b * ratio) + a) / denom;
            y = (b - (a * ratio)) / denom;
        } else {
            x = (a + (d * (b / c))) / denom;
            y = (b - (d * (a / c))) / denom;
        }
    }
    return cvk_make(x, y);
}

// std::abs(std::complex<double>) is cabs == hypot; used only for the
// breakdown thresholds (krylov.cpp:83,99,117,...).
CVK_HD double cvk_abs(cvk_c a) {
#if defined(__CUDA_ARCH__)
    return hypot(a.x, a.y);
#else
    return std::hypot(a.x, a.y);
#endif
}
