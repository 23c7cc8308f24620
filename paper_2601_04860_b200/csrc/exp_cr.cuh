// exp_cr.cuh -- correctly rounded exp(x) on [-700, 0] in double-double.
//
// Host + device (included by render.cu, fuse.cu and by the CPU test
// tests/test_exp_cr.py, which pins it against a 40-digit decimal exp and
// against the C library's exp).  Compile without FMA contraction; the
// explicit fma() calls are exact products.
#pragma once

#include <math.h>

#ifdef __CUDACC__
#define DIVAS_HD __host__ __device__ __forceinline__
#else
#define DIVAS_HD static
#endif

namespace divas {

// ---- correctly rounded exp on [-700, 0] (double-double evaluation) --------
// The reference's exp calls (the marcher's alpha = 1 - exp(-sigma dt), the
// fusion's thick depth weight exp(-alpha1 r r)) go to the C library's exp
// (glibc: error <= 0.511 ulp by its implementation's analysis), so whenever
// the exact value is farther than 0.011 ulp from a rounding midpoint glibc
// returns the correctly rounded double.  exp_cr evaluates exp(x) to ~2^-61
// relative (Cody-Waite reduction by ln2 in three parts, degree-17 Taylor: the
// tail in double, the leading four steps in double-double), returns the
// correctly rounded double and, when the exact value is within 0.02 ulp of a midpoint
// (`ambiguous`), the other neighbour the reference might have produced.
struct DD {
    double h, l;
};
DIVAS_HD DD dd_fast(double a, double b) {   // |a| >= |b|
    const double s = a + b;
    return DD{s, b - (s - a)};
}
DIVAS_HD DD dd_two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return DD{s, (a - (s - bb)) + (b - bb)};
}
DIVAS_HD DD dd_add(DD a, DD b) {
    const DD s = dd_two_sum(a.h, b.h);
    return dd_fast(s.h, s.l + (a.l + b.l));
}
DIVAS_HD DD dd_mul(DD a, DD b) {
    const double p = a.h * b.h;
    const double e = fma(a.h, b.h, -p) + (a.h * b.l + a.l * b.h);
    return dd_fast(p, e);
}

DIVAS_HD double exp_cr(double x, bool &ambiguous, double &alt) {
    const double L1 = 0x1.62e42ff000000p-1, L2 = -0x1.718432a1b0e26p-35,
                 L3 = -0x1.9ff0342542fc3p-90;     // ln2 = L1 + L2 + L3, L1 32 bits
    const double k = rint(x * 0x1.71547652b82fep+0);
    const double r1 = x - k * L1;                  // exact (k L1 exact, Sterbenz)
    const double p = k * L2;
    const double pe = fma(k, L2, -p);
    DD r = dd_two_sum(r1, -p);
    r = dd_fast(r.h, r.l - pe - k * L3);           // |r| <= ln2 / 2
    // exp(r) = 1 + r (1 + r (1/2 + r (1/6 + r q))), q = sum_{n>=4} r^(n-4) / n!
    // to n = 17 (truncation < 2^-70).  q in double: its error (< 2u q) enters
    // scaled by r^4 <= 0.0145, i.e. < 2^-62 of the result (0.002 ulp); the
    // last four steps in double-double.
    const double c[14] = {0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10,
                          0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19,
                          0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29,
                          0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41,
                          0x1.ae7f3e733b81fp-45, 0x1.952c77030ad4ap-49};
    double q = c[13];
#pragma unroll
    for (int n = 12; n >= 0; --n) q = q * r.h + c[n];
    DD s = dd_add(dd_mul(r, DD{q, 0.0}), DD{0x1.5555555555555p-3, 0x1.5555555555555p-57});
    s = dd_add(dd_mul(r, s), DD{0.5, 0.0});
    s = dd_add(dd_mul(r, s), DD{1.0, 0.0});
    s = dd_add(dd_mul(r, s), DD{1.0, 0.0});
    const int ki = (int)k;
    DD e = dd_fast(ldexp(s.h, ki), ldexp(s.l, ki));
    const double up = nextafter(e.h, 1e300), dn = nextafter(e.h, 0.0);
    const double side = e.l >= 0.0 ? up - e.h : e.h - dn;
    ambiguous = fabs(e.l) > 0.48 * side;
    alt = e.l >= 0.0 ? up : dn;
    return e.h;
}

// exp(x) as the reference's C library returns it, up to the rare ambiguous
// case above (then the correctly rounded value): exp_cr on [-700, 0] (normal
// results), the CUDA exp elsewhere (x > 0 does not occur on the path; below
// -700 the result is < 1e-304).
DIVAS_HD double exp_ref(double x) {
    if (x >= -700.0 && x <= 0.0) {
        bool amb;
        double alt;
        return exp_cr(x, amb, alt);
    }
    return exp(x);
}

}  // namespace divas
