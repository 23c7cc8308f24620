// bands.cuh -- per-view 8x8-tile depth bands for exact thin-path rejection.
//
// (The bands also cover pixels with m == 0.5: band_px.)
// A footprint pixel p supports a thin candidate at depth x_d iff
//   mask_p > 0.5 && n_p > 0 && |fl(x_d - D_p)| <= tau(n_p)          (fusion.py:361-367)
// which implies  D_p - tau(1 + 2^-52) <= x_d <= D_p + tau(1 + 2^-52).  A tile's
// band is the hull of those intervals over its eligible pixels, widened by a
// 1e-12 relative margin that dominates every rounding involved.  A supporting
// pixel's interval lies inside its own tile's band, so if x_d lies outside the
// band of EVERY tile that can contain the footprint box, support is exactly 0,
// p_cov = 0 and (for thin_percent_cover > 0) t = 0 < thin_accept: the pair
// cannot vote and needs neither corner projections nor a scan.
#pragma once

#include "common.cuh"

namespace divas {

#ifndef DIVAS_BAND_TILE
#define DIVAS_BAND_TILE 8
#endif
constexpr int kBandTile = DIVAS_BAND_TILE;        // 8 or 4
// band test: boxes touching more tiles than this are not tested (scanned)
constexpr int kBandMaxTiles = kBandTile == 8 ? 16 : 36;
// per-view refine keys: z min, z max (order-preserving f32 keys), n min, n max
// over the valid pixels (n > 0)
constexpr int kKeys = 4;

struct BandParams {
    double gamma, beta, bmax, dx;
    int hm, wm, ntx, nty;
};

// Per-pixel scan records, two 8-byte planes per view (16 B/px in all):
//   A = {refined mask, d_exp, or NaN when the pixel cannot support a thin
//        candidate (mask <= 0.5 or n == 0)}; the mask's sign bit flags a
//        supporting pixel whose tau differs from the view's base tau(n_min)
//        (readers take |mask|: refined masks are >= 0)
//   B = {tau_d(n) as f32, n_samples bits},
//        written only at supporting pixels (elsewhere A's NaN decides)
// A view whose supporting pixels all share one tau is scanned from plane A
// alone (8 bytes per pixel) with that tau from the view's tau-range entry;
// one where few supporting pixels differ from the base tau is also scanned
// from A alone, with the base tau, and an item that meets a flagged pixel is
// recounted exactly; other views read B as well.
// View v's records start at v * 2 * hm * wm float2: A plane, then B plane.
constexpr float kIneligible = -1e30f;

// Bands: per view nty * ntx tile entries, then two 16-byte entries: the
// view's {min, max} key (order-preserving u32, as the z keys) of tau32 over
// the supporting pixels the pass saw, the count of flagged and of supporting
// pixels; then {base tau32 bits (NaN: none), min and max n_samples over the
// supporting pixels, base n (0: none)}.  A supporting pixel is flagged when
// its f64 tau differs from the base tau(n_min) (exact, not by the f32 key).
__host__ __device__ inline int64_t band_view_stride(int nty, int ntx) {
    return (int64_t)nty * ntx + 2;
}

__device__ __forceinline__ uint32_t tau_key(float t) {   // t >= 0: order-preserving
    return __float_as_uint(t);
}

// tau-range entries of views [0, nv) of a band buffer: {UINT_MAX, 0} (empty)
static __global__ void band_init(double2 *__restrict__ bands, int nv, int nty, int ntx) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v < nv) {
        uint32_t *e = reinterpret_cast<uint32_t *>(bands + v * band_view_stride(nty, ntx) +
                                                   (int64_t)nty * ntx);
        e[0] = 0xffffffffu;
        e[1] = 0u;
        e[2] = 0u;                                   // flagged supporting pixels
        e[3] = 0u;                                   // supporting pixels
        e[4] = 0x7fc00000u;                          // base tau: none yet
        e[5] = 0xffffffffu;                          // n range of the supporting pixels
        e[6] = 0u;
        e[7] = 0u;                                   // base n: none yet
    }
}

// A pixel widens its tile's band when m >= 0.5 and n > 0 (thin support needs
// m > 0.5, the thick gate m >= mask_thr = 0.5: the band covers both, so a
// tile whose band misses x_d can neither support a thin candidate nor hold a
// thick centre pixel that passes the depth test, tau_depth <= tau_thin);
// returns the pixel's tau as f32 when it can support (m > 0.5), else
// kIneligible.
__device__ __forceinline__ float band_px(float m, int32_t n, float d, const BandParams &B,
                                         double &lo, double &hi, double &t64) {
    if (m >= 0.5f && n > 0) {
        double b = B.beta * (double)n;
        if (b > B.bmax) b = B.bmax;
        const double t = (2.0 * B.gamma + b) * B.dx;
        const double D = (double)d;
        const double mg = 1e-12 * (fabs(D) + t);
        lo = fmin(lo, D - t - mg);
        hi = fmax(hi, D + t + mg);
        t64 = t;
        return m > 0.5f ? (float)t : kIneligible;
    }
    return kIneligible;
}
__device__ __forceinline__ float band_px(float m, int32_t n, float d, const BandParams &B,
                                         double &lo, double &hi) {
    double t64;
    return band_px(m, n, d, B, lo, hi, t64);
}

// One thread per VEC-pixel column chunk and 8 rows; TPW = 8 / VEC threads form
// a tile row and combine with shuffles.  REFINE: also produce the refined mask
// from the raw one (segmenter.py:141-152) and band on the refined values.
#ifndef DIVAS_BAND_MINB
#define DIVAS_BAND_MINB 5
#endif
template <int VEC, bool REFINE>
__global__ void __launch_bounds__(256, DIVAS_BAND_MINB)
band_pass(BandParams B, const float *__restrict__ mask, const float *__restrict__ z,
          const int32_t *__restrict__ nsamp, const float *__restrict__ dexp,
          float *__restrict__ refined, const uint32_t *__restrict__ minmax,
          double2 *__restrict__ bands, float2 *__restrict__ records, int nv,
          const int4 *__restrict__ roi = nullptr) {
    constexpr int TPW = kBandTile / VEC;
    const int v = nv - 1 - (int)blockIdx.z;          // reverse view order: L2 reuse of z / n
    const int64_t plane = (int64_t)B.hm * B.wm;
    const int64_t off = (int64_t)v * plane;
    float2 *__restrict__ recA = records + 2 * off;   // this view's A plane
    float2 *__restrict__ recB = recA + plane;        // and B plane
    uint32_t tmin = 0xffffffffu, tmax = 0u;          // tau keys of the supporting pixels
    // plane B is needed only when the view's supporting pixels can differ in
    // tau: with the n range known (refine keys), one tau(n) for all -> skip it
    bool write_b = true;
    float base = __int_as_float(0x7fc00000);         // tau(n_min); NaN without keys
    double base64 = __longlong_as_double(0x7ff8000000000000LL);   // the same in f64
    if (minmax) {
        const uint32_t n0 = minmax[kKeys * v + 2], n1 = minmax[kKeys * v + 3];
        double l0 = 0.0, h0 = 0.0, t1 = 0.0;
        write_b = n0 <= n1 && band_px(1.0f, (int32_t)n0, 0.0f, B, l0, h0) !=
                                  band_px(1.0f, (int32_t)n1, 0.0f, B, l0, h0);
        if (n0 <= n1) base = band_px(1.0f, (int32_t)n0, 0.0f, B, l0, h0, t1);
        if (n0 <= n1) base64 = t1;
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
            uint32_t *e = reinterpret_cast<uint32_t *>(bands + (int64_t)v * band_view_stride(B.nty, B.ntx) +
                                                       (int64_t)B.nty * B.ntx);
            e[4] = __float_as_uint(base);
            e[7] = n0 <= n1 ? n0 : 0u;
        }
    }
    uint32_t nlo = 0xffffffffu, nhi = 0u;            // n range of the supporting pixels
    uint32_t cnt = 0;              // supporting pixels (low 16 bits), flagged ones (high)
    // ROI (optional): the view's tile-aligned window {x0, y0, x1, y1}; the
    // grid covers the largest window, blocks past this view's window idle
    int rx0 = 0, rx1 = B.wm - 1, ty = (int)blockIdx.y;
    if (roi) {
        const int4 w = roi[v];
        rx0 = w.x;
        rx1 = min(w.z, B.wm - 1);
        ty += w.y / kBandTile;
        if (ty * kBandTile > min(w.w, B.hm - 1)) return;
    }
    const int chunk = blockIdx.x * blockDim.x + threadIdx.x;
    const int x0 = rx0 + chunk * VEC;
    const bool active = x0 <= rx1 && x0 < B.wm;
    bool any = false;
    double lo_ref = 0.0, span = 0.0;
    if (REFINE) {
        const uint32_t kmin = minmax[kKeys * v], kmax = minmax[kKeys * v + 1];
        any = kmin <= kmax;
        lo_ref = any ? (double)key_f32(kmin) : 0.0;
        const double hi_ref = any ? (double)key_f32(kmax) : 0.0;
        span = hi_ref - lo_ref;
    }
    double lo = __longlong_as_double(0x7ff0000000000000LL);   // +inf
    double hi = -lo;
    if (active) {
        for (int r = 0; r < kBandTile; ++r) {
            const int row = ty * kBandTile + r;
            if (row >= B.hm) break;
            const int64_t p = off + (int64_t)row * B.wm + x0;
            float m[VEC], d[VEC];
            int32_t n[VEC];
            if (VEC == 4) {
                const float4 mm = __ldg(reinterpret_cast<const float4 *>(mask + p));
                const int4 nn = __ldg(reinterpret_cast<const int4 *>(nsamp + p));
                const float4 dd = __ldg(reinterpret_cast<const float4 *>(dexp + p));
                m[0] = mm.x; m[1] = mm.y; m[2] = mm.z; m[3] = mm.w;
                n[0] = nn.x; n[1] = nn.y; n[2] = nn.z; n[3] = nn.w;
                d[0] = dd.x; d[1] = dd.y; d[2] = dd.z; d[3] = dd.w;
                if (REFINE) {
                    const float4 zz = __ldg(reinterpret_cast<const float4 *>(z + p));
                    const float zv[4] = {zz.x, zz.y, zz.z, zz.w};
                    for (int k = 0; k < 4; ++k) m[k] = refine_px(m[k], zv[k], n[k], any, lo_ref, span);
                    if (refined)
                        __stcs(reinterpret_cast<float4 *>(refined + p), make_float4(m[0], m[1], m[2], m[3]));
                }
            } else {
                m[0] = __ldg(mask + p);
                n[0] = __ldg(nsamp + p);
                d[0] = __ldg(dexp + p);
                if (REFINE) {
                    m[0] = refine_px(m[0], __ldg(z + p), n[0], any, lo_ref, span);
                    if (refined) refined[p] = m[0];
                }
            }
            const int64_t q = p - off;                 // pixel within the view
            float2 a[VEC], b[VEC];
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                double t64 = 0.0;
                const float t32 = band_px(m[k], n[k], d[k], B, lo, hi, t64);
                const bool sup = t32 >= 0.0f;
                // every pixel flags when base is NaN (no refine keys): then the
                // flag path is never chosen (nflag = nsup)
                const bool flag = sup && !(t64 == base64);
                cnt += sup ? (flag ? 0x10001u : 1u) : 0u;
                a[k] = make_float2(flag ? -m[k] : m[k], sup ? d[k] : __int_as_float(0x7fc00000));
                b[k] = make_float2(t32, __int_as_float(n[k]));
                if (sup) {
                    tmin = min(tmin, tau_key(t32));
                    tmax = max(tmax, tau_key(t32));
                    nlo = min(nlo, (uint32_t)n[k]);
                    nhi = max(nhi, (uint32_t)n[k]);
                }
            }
            if (VEC == 4) {
                float4 *a4 = reinterpret_cast<float4 *>(recA + q);
                a4[0] = make_float4(a[0].x, a[0].y, a[1 % VEC].x, a[1 % VEC].y);
                a4[1] = make_float4(a[2 % VEC].x, a[2 % VEC].y, a[3 % VEC].x, a[3 % VEC].y);
                // B is read only where A holds a depth (a supporting pixel;
                // elsewhere A's NaN decides), so only those entries are written
                if (write_b) {
#pragma unroll
                    for (int k = 0; k < VEC; ++k)
                        if (a[k].y == a[k].y) recB[q + k] = b[k];
                }
            } else {
                recA[q] = a[0];
                if (write_b && a[0].y == a[0].y) recB[q] = b[0];
            }
        }
    }
#pragma unroll
    for (int o = 1; o < TPW; o <<= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    double2 *bv = bands + (int64_t)v * band_view_stride(B.nty, B.ntx);
    if (active && (threadIdx.x % TPW) == 0) {
        const int tx = x0 / kBandTile;
        bv[(int64_t)ty * B.ntx + tx] = make_double2(lo, hi);
    }
    // the view's tau range and flag counts: warp-reduce, atomics per warp
    // (warps without a supporting pixel -- most of them -- skip it all)
    // (a warp sees at most 32 x 8 x VEC <= 1024 pixels: the halves do not carry)
    if (__any_sync(0xffffffffu, cnt != 0)) {
        for (int o = 16; o > 0; o >>= 1) {
            tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
            tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
            nlo = min(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
            nhi = max(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if ((threadIdx.x & 31) == 0) {
            uint32_t *e = reinterpret_cast<uint32_t *>(bv + (int64_t)B.nty * B.ntx);
            atomicMin(e, tmin);
            atomicMax(e + 1, tmax);
            atomicAdd(e + 2, cnt >> 16);
            atomicAdd(e + 3, cnt & 0xffffu);
            atomicMin(e + 5, nlo);
            atomicMax(e + 6, nhi);
        }
    }
}

inline BandParams band_params(const double *pv, double dx, int hm, int wm) {
    BandParams B;
    B.gamma = pv[0]; B.beta = pv[1]; B.bmax = pv[2]; B.dx = dx;
    B.hm = hm; B.wm = wm;
    B.ntx = (wm + kBandTile - 1) / kBandTile;
    B.nty = (hm + kBandTile - 1) / kBandTile;
    return B;
}

inline size_t band_bytes(int nv, int hm, int wm) {
    return (size_t)nv * band_view_stride((hm + kBandTile - 1) / kBandTile,
                                         (wm + kBandTile - 1) / kBandTile) * sizeof(double2);
}

inline size_t record_bytes(int nv, int hm, int wm) {
    return (size_t)nv * hm * wm * 2 * sizeof(float2);
}

static inline void launch_band_init(double2 *bands, const BandParams &B, int nv, cudaStream_t s) {
    band_init<<<(nv + 255) / 256, 256, 0, s>>>(bands, nv, B.nty, B.ntx);
}

}  // namespace divas
