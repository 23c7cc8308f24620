// common.cuh -- shared device helpers for the DivAS sm_100a kernels.
//
// Every translation unit is compiled with -fmad=false: the reference's numba
// kernels emit no FMA, so neither may we.  Double
// division and sqrt keep nvcc's IEEE round-to-nearest defaults (no fast-math).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/divas_b200.h"

#include <cstdlib>
#include <utility>

namespace divas {

constexpr int kCamStride = DIVAS_CAM_STRIDE;

// Programmatic dependent launch (sm_90+): a kernel of the step's chains is
// launched with programmatic stream serialization (launch_pdl), so its blocks
// are scheduled while the previous kernel's last blocks drain; every such
// kernel starts with griddep_wait(), which returns once the previous grid has
// completed and its writes are visible -- nothing is read or written before.
// Without the launch attribute griddepcontrol.wait is a no-op.
#ifndef DIVAS_PDL_EARLY
#define DIVAS_PDL_EARLY 1
#endif
__device__ __forceinline__ void griddep_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // this block is running: once every block of the grid is, the next kernel
    // of the stream may start placing its blocks in the slots our tail frees
    // (they then wait in griddep_wait for this grid to complete)
    if (DIVAS_PDL_EARLY) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

inline bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("DIVAS_PDL");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on != 0;
}

// kernel<<<grid, block, smem, s>>>(args...) with the programmatic-serialization
// attribute (kernel must begin with griddep_wait())
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// numba's int(math.floor(x)) on x86-64 lowers to cvttsd2si: values outside
// int64 (and NaN) become INT64_MIN.  CUDA's cvt saturates instead, so restate.
__device__ __forceinline__ long long nb_floor_int(double x) {
    double f = floor(x);
    if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0))
        return (long long)0x8000000000000000ULL;
    return (long long)f;
}

// Order-preserving float <-> uint32 key (for atomicMin/atomicMax of f32).
__device__ __forceinline__ uint32_t f32_key(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_f32(uint32_t k) {
    uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
    return __uint_as_float(b);
}

// refine_mask per pixel (segmenter.py:141-152): valid pixels get
// clip(f64(m) * (1 - (z - lo) / (hi - lo)), 0, 1) (zhat = 0 for a constant
// map), invalid ones 0; then round to f32.
__device__ __forceinline__ float refine_px(float m, float z, int32_t n, bool any, double lo,
                                           double span) {
    double o = 0.0;
    if (any && n > 0) {
        const double zh = span > 0.0 ? ((double)z - lo) / span : 0.0;
        o = (double)m * (1.0 - zh);
    }
    if (o < 0.0) o = 0.0;   // np.clip keeps NaN, so do these compares
    if (o > 1.0) o = 1.0;
    return __double2float_rn(o);
}

// The same value without the f64 division on almost every pixel: zhat from
// the view's reciprocal rspan = RN(1 / span), then the f32 rounding of the
// clipped product is CERTIFIED.  For 0 <= z - lo <= span and |m| <= M the
// approximate product is within 7.1 * 2^-53 * max(1, M) of the reference's
// (three roundings of zhat, two of 1 - zhat, two of the product); when no f32
// rounding boundary lies within E = 2^-48 * max(1, |m|) of it (4x slack) the
// f32 result is the reference's.  Otherwise -- and for zero, subnormal or
// out-of-range values -- refine_px's exact chain runs.
__device__ __forceinline__ float refine_px_fast(float m, float z, int32_t n, bool any, double lo,
                                                double span, double rspan) {
    if (!(any && n > 0)) return 0.0f;                       // o = 0 -> clip -> +0
    if (!(span > 0.0)) return refine_px(m, z, n, any, lo, span);
    const double a = (double)z - lo;
    if (!(a >= 0.0 && a < span)) return refine_px(m, z, n, any, lo, span);
    // 0 <= zhat <= 1 here, so m * (1 - zhat) is m * (a non-negative number):
    // a zero mask gives a zero of m's sign, which the clip keeps
    if (m == 0.0f) return m;
    double c = (double)m * (1.0 - a * rspan);
    if (c < 0.0) c = 0.0;
    if (c > 1.0) c = 1.0;
    const float f = __double2float_rn(c);
#ifndef DIVAS_REFINE_ICERT
#define DIVAS_REFINE_ICERT 1
#endif
    if (DIVAS_REFINE_ICERT && fabsf(m) <= 1.0f) {
        // the same certificate in integer arithmetic (E = 2^-48 for |m| <= 1):
        // for c in [2^e, 2^(e+1)), e >= -22, the only f32 rounding midpoint of
        // c's f32 interval sits where the low 29 significand bits L equal
        // 2^28, and one f64 ulp is 2^(e-52), so c +- E stays on one side of
        // every midpoint iff |L - 2^28| > 2^(4-e) (the binade edges are f32
        // values, >= 2^(e-25) from any midpoint)
        const unsigned long long bits = (unsigned long long)__double_as_longlong(c);
        const int e = (int)((bits >> 52) & 0x7ffu) - 1023;
        const int L = (int)((uint32_t)bits & 0x1fffffffu) - (1 << 28);
        if (e >= -22 && e <= 0 && abs(L) > (1 << (4 - e))) return f;
        return refine_px(m, z, n, any, lo, span);
    }
    if (f > 1.17549435e-38f && f < 3.0e38f) {
        const double E = 3.552713678800501e-15 * fmax(1.0, fabs((double)m));   // 2^-48 max(1, |m|)
        const double fd = (double)f;
        const double up = (double)__int_as_float(__float_as_int(f) + 1);
        const double dn = (double)__int_as_float(__float_as_int(f) - 1);
        if (c + E < 0.5 * (fd + up) && c - E > 0.5 * (fd + dn)) return f;
    }
    return refine_px(m, z, n, any, lo, span);
}

void set_error(const char *fmt, ...);
int check_launch(const char *what);

}  // namespace divas
