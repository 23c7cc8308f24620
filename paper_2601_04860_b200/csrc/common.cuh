// common.cuh -- shared device helpers for the DivAS sm_100a kernels.
//
// Every translation unit is compiled with -fmad=false: the reference's numba
// kernels emit no FMA, so neither may we.  Double
// division and sqrt keep nvcc's IEEE round-to-nearest defaults (no fast-math).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/divas_b200.h"

namespace divas {

constexpr int kCamStride = DIVAS_CAM_STRIDE;

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

void set_error(const char *fmt, ...);
int check_launch(const char *what);

}  // namespace divas
