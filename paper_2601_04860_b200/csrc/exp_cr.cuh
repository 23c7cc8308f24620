// exp_cr.cuh -- glibc's exp restated bit for bit (exp_glibc, what every
// kernel uses), and a correctly rounded exp on [-700, 0] in double-double
// (exp_cr, kept as an independent check in tests/test_exp_cr.py).
//
// Host + device (included by render.cu, fuse.cu and by the CPU test
// tests/test_exp_cr.py, which pins it against a 40-digit decimal exp and
// against the C library's exp).  Compile without FMA contraction; the
// explicit fma() calls are exact products.
#pragma once

#include <math.h>
#include <string.h>

#include "exp_table.cuh"

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

// ---- glibc's exp, bit for bit --------------------------------------------
// The reference's exp calls go to the C library: glibc 2.39 on x86-64, whose
// ifunc picks the FMA build of the optimized-routines algorithm (e_exp.c):
// exp(x) = 2^(k/128) exp(r), x = k ln2/128 + r, a degree-5 polynomial for
// exp(r) - 1 and the table 2^(k/128) ~ scale (1 + tail) (exp_table.cuh,
// generated from the definition by tools/gen_exp_table.py).  The FMA build
// contracts exactly these operations (read from its object code and checked
// against libm on 2e7 random arguments, tests/test_exp_cr.py): kd = fma(x,
// InvLn2N, Shift), the two reduction steps, both inner polynomial pairs, the
// two r^2 / r^4 terms and the final scale + scale * tmp (its out-of-range
// tail, specialcase(), is not contracted).  Restated with
// explicit fma() (this header is compiled without contraction), the result
// is glibc's for every argument: no correctly-rounded approximation and no
// "ambiguous" cases.
#ifdef __CUDACC__
static __device__ const unsigned long long kExpTabDev[256] = {DIVAS_EXP_TABLE_VALUES};
#endif
static const unsigned long long kExpTabHost[256] = {DIVAS_EXP_TABLE_VALUES};

DIVAS_HD unsigned long long exp_tab(int i) {
#ifdef __CUDA_ARCH__
    return __ldg(kExpTabDev + i);
#else
    return kExpTabHost[i];
#endif
}

DIVAS_HD unsigned long long dbits(double x) {
#ifdef __CUDA_ARCH__
    return (unsigned long long)__double_as_longlong(x);
#else
    unsigned long long u;
    memcpy(&u, &x, 8);
    return u;
#endif
}

DIVAS_HD double bitsd(unsigned long long u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}

// specialcase() of e_exp.c: |x| in [512, 1024) (scale's exponent out of range)
DIVAS_HD double exp_glibc_special(double tmp, unsigned long long sbits, unsigned long long ki) {
    if ((ki & 0x80000000ull) == 0) {                    // k > 0
        sbits -= 1009ull << 52;
        const double scale = bitsd(sbits);
        return 0x1p1009 * fma(scale, tmp, scale);
    }
    sbits += 1022ull << 52;                            // k < 0: subnormal results
    const double scale = bitsd(sbits);
    double y = scale + scale * tmp;
    if (y < 1.0) {
        double lo = scale - y + scale * tmp;
        const double hi = 1.0 + y;
        lo = 1.0 - hi + y + lo;
        y = (hi + lo) - 1.0;
        if (y == 0.0) y = 0.0;
    }
    return 0x1p-1022 * y;
}

DIVAS_HD double exp_glibc(double x) {
    const double InvLn2N = 0x1.71547652b82fep7, NegLn2hiN = -0x1.62e42fefa0000p-8,
                 NegLn2loN = -0x1.cf79abc9e3b3ap-47, Shift = 0x1.8p52;
    const double C2 = 0x1.ffffffffffdbdp-2, C3 = 0x1.555555555543cp-3,
                 C4 = 0x1.55555cf172b91p-5, C5 = 0x1.1111167a4d017p-7;
    unsigned abstop = (unsigned)(dbits(x) >> 52) & 0x7ffu;
    const unsigned t54 = 0x3c9u, t512 = 0x408u, t1024 = 0x409u;   // top12 of 2^-54, 512, 1024
    if (abstop - t54 >= t512 - t54) {
        if (abstop - t54 >= 0x80000000u) return 1.0 + x;            // |x| < 2^-54
        if (abstop >= t1024) {
            if (dbits(x) == 0xfff0000000000000ull) return 0.0;       // -inf
            if (abstop >= 0x7ffu) return 1.0 + x;                    // inf, NaN
            return (dbits(x) >> 63) ? 0.0 : bitsd(0x7ff0000000000000ull);
        }
        abstop = 0;                                                  // large |x| below
    }
    const double kd0 = fma(x, InvLn2N, Shift);
    const unsigned long long ki = dbits(kd0);
    const double kd = kd0 - Shift;
    double r = fma(kd, NegLn2hiN, x);
    r = fma(kd, NegLn2loN, r);
    const int idx = 2 * (int)(ki % 128);
    const unsigned long long top = ki << 45;
    const double tail = bitsd(exp_tab(idx));
    const unsigned long long sbits = exp_tab(idx + 1) + top;
    const double A = fma(r, C3, C2);
    const double t0 = tail + r;
    const double r2 = r * r;
    const double B = fma(r, C5, C4);
    const double t1 = fma(A, r2, t0);
    const double tmp = fma(r2 * r2, B, t1);
    if (abstop == 0) return exp_glibc_special(tmp, sbits, ki);
    const double scale = bitsd(sbits);
    return fma(scale, tmp, scale);
}

// exp(x) exactly as the reference's C library returns it.
DIVAS_HD double exp_ref(double x) { return exp_glibc(x); }

}  // namespace divas
