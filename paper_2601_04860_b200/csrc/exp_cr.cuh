// exp_cr.cuh -- correctly rounded exp(x) on [-38, 0] in double-double.
//
// Host + device (included by render.cu and by the CPU test
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

// ---- correctly rounded exp on [-38, 0] (double-double evaluation) ---------
// The reference's alpha = 1 - exp(-sigma dt) calls the C library's exp
// (glibc: error <= 0.511 ulp by its implementation's analysis), so whenever
// the exact value is farther than 0.011 ulp from a rounding midpoint glibc
// returns the correctly rounded double.  exp_cr evaluates exp(x) to ~2^-90
// relative (Cody-Waite reduction by ln2 in three parts, x / 2^8, degree-9
// Taylor in double-double, eight squarings), returns the correctly rounded
// double and, when the exact value is within 0.02 ulp of a midpoint
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
    // 1/n!, n = 0..9, as double-doubles
    const double ch[10] = {1.0, 1.0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
                           0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13,
                           0x1.a01a01a01a01ap-16, 0x1.71de3a556c734p-19};
    const double cl[10] = {0.0, 0.0, 0.0, 0x1.5555555555555p-57, 0x1.5555555555555p-59,
                           0x1.1111111111111p-63, -0x1.f49f49f49f49fp-65, 0x1.a01a01a01a01ap-73,
                           0x1.a01a01a01a01ap-76, -0x1.c154f8ddc6c00p-73};
    const double L1 = 0x1.62e42ff000000p-1, L2 = -0x1.718432a1b0e26p-35,
                 L3 = -0x1.9ff0342542fc3p-90;     // ln2 = L1 + L2 + L3, L1 32 bits
    const double k = rint(x * 0x1.71547652b82fep+0);
    const double r1 = x - k * L1;                  // exact (k L1 exact, Sterbenz)
    const double p = k * L2;
    const double pe = fma(k, L2, -p);
    DD r = dd_two_sum(r1, -p);
    r = dd_fast(r.h, r.l - pe - k * L3);
    r.h *= 0x1p-8;
    r.l *= 0x1p-8;
    DD s{ch[9], cl[9]};
#pragma unroll
    for (int n = 8; n >= 0; --n) s = dd_add(dd_mul(s, r), DD{ch[n], cl[n]});
#pragma unroll
    for (int i = 0; i < 8; ++i) s = dd_mul(s, s);
    const int ki = (int)k;
    DD e = dd_fast(ldexp(s.h, ki), ldexp(s.l, ki));
    const double up = nextafter(e.h, 1e300), dn = nextafter(e.h, 0.0);
    const double side = e.l >= 0.0 ? up - e.h : e.h - dn;
    ambiguous = fabs(e.l) > 0.48 * side;
    alt = e.l >= 0.0 ? up : dn;
    return e.h;
}

}  // namespace divas
