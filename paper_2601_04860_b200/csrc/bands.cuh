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

// L2 cache-policy helpers (sm_80+): a fractional evict-last policy and
// 16-byte stores carrying it
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void st_evict_last(float4 *p, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                 ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

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
    griddep_wait();                     // PDL: after the previous kernel completes
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
// band_px with the tile hull in f32 and directed rounding (band_pass2): the
// interval [D - tau(1 + 2^-52), D + tau(1 + 2^-52)] that can hold a
// supporting x_d lies inside [RD(D - T), RU(D + T)], T = one f32 ulp above
// RU(tau) -- a hull wider than the f64 one by about an f32 ulp, which the
// band tests only ever read as a conservative bound.
__device__ __forceinline__ float band_px32(float m, int32_t n, float d, const BandParams &B,
                                           float &lo, float &hi, double &t64) {
    if (m >= 0.5f && n > 0) {
        double b = B.beta * (double)n;
        if (b > B.bmax) b = B.bmax;
        const double t = (2.0 * B.gamma + b) * B.dx;
        const float T = __int_as_float(__float_as_int(__double2float_ru(t)) + 1);
        lo = fminf(lo, __fsub_rd(d, T));
        hi = fmaxf(hi, __fadd_ru(d, T));
        t64 = t;
        return m > 0.5f ? __double2float_rn(t) : kIneligible;
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

// Row-split variant of band_pass<4, *> (128-bit loads only): a thread owns a
// 4-pixel chunk of TWO rows and issues all eight of its 16-byte loads (mask,
// n, d_exp, z of both rows) before any arithmetic, so four times as many
// threads keep loads in flight as in band_pass (8 rows per thread, one row of
// loads at a time).  Lane = 8 * rq + c: rows 2 rq, 2 rq + 1 of the 8-row tile
// band, chunk c of the warp's 32 pixels; a tile (8 x 8) is the 8 lanes
// {c, c ^ 1} x rq, combined with three shuffles.  Same outputs as band_pass.
#ifndef DIVAS_BAND_WARPS
#define DIVAS_BAND_WARPS 4
#endif
constexpr int kBand2Warps = DIVAS_BAND_WARPS;
#ifndef DIVAS_BAND_ROWS
#define DIVAS_BAND_ROWS 4
#endif
constexpr int kBand2Rows = DIVAS_BAND_ROWS;   // 8-row tile bands per block (grid-stride in y)
#ifndef DIVAS_BAND_RPT
#define DIVAS_BAND_RPT 1
#endif
constexpr int kBandRpt = DIVAS_BAND_RPT;   // rows of the 8-row band per thread (1 or 2)
constexpr int kBandCpw = 4 * kBandRpt;     // 4-pixel chunks per warp row
template <bool REFINE>
__global__ void __launch_bounds__(32 * kBand2Warps)
band_pass2(BandParams B, const float *__restrict__ mask, const float *__restrict__ z,
           const int32_t *__restrict__ nsamp, const float *__restrict__ dexp,
           float *__restrict__ refined, const uint32_t *__restrict__ minmax,
           double2 *__restrict__ bands, float2 *__restrict__ records, int nv,
           const int4 *__restrict__ roi = nullptr) {
    griddep_wait();                     // PDL: after the previous kernel completes
    static_assert(kBandTile == 8, "row-split band pass assumes 8x8 tiles");
    const int v = nv - 1 - (int)blockIdx.z;          // reverse view order: L2 reuse of z / n
    const uint64_t pol = l2_policy_evict_last();
    // the view's window and keys in one round trip (no dependent prologue loads)
    const int4 w = roi ? __ldg(roi + v) : make_int4(0, 0, B.wm - 1, B.hm - 1);
    const uint4 keys = minmax ? __ldg(reinterpret_cast<const uint4 *>(minmax) + v)
                              : make_uint4(0xffffffffu, 0u, 0xffffffffu, 0u);
    const int64_t plane = (int64_t)B.hm * B.wm;
    const int64_t off = (int64_t)v * plane;
    float2 *__restrict__ recA = records + 2 * off;
    float2 *__restrict__ recB = recA + plane;
    bool write_b = true;
    float base = __int_as_float(0x7fc00000);
    double base64 = __longlong_as_double(0x7ff8000000000000LL);
    if (minmax) {
        const uint32_t n0 = keys.z, n1 = keys.w;
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
    const int rx0 = w.x, rx1 = min(w.z, B.wm - 1);
    const int ty_first = w.y / kBandTile, ty_last = min(w.w, B.hm - 1) / kBandTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rq = lane / kBandCpw, c = lane % kBandCpw;
    const int chunk = ((int)blockIdx.x * kBand2Warps + warp) * kBandCpw + c;
    const int x0 = rx0 + chunk * 4;
    const bool active = x0 <= rx1 && x0 < B.wm;
    bool any = false;
    double lo_ref = 0.0, span = 0.0, rspan = 0.0;
    if (REFINE) {
        const uint32_t kmin = keys.x, kmax = keys.y;
        any = kmin <= kmax;
        lo_ref = any ? (double)key_f32(kmin) : 0.0;
        const double hi_ref = any ? (double)key_f32(kmax) : 0.0;
        span = hi_ref - lo_ref;
        rspan = span > 0.0 ? 1.0 / span : 0.0;
    }
    uint32_t tmin = 0xffffffffu, tmax = 0u, nlo = 0xffffffffu, nhi = 0u, cnt = 0;
    double2 *bv = bands + (int64_t)v * band_view_stride(B.nty, B.ntx);
    // this block's tile bands: ty_first + blockIdx.y * kBand2Rows + i
    float4 mm[2], dd[2], zz[2];
    int4 nn[2];
    bool ok0 = false, ok1 = false;
    auto load = [&](int ty) {
        const int row0 = ty * kBandTile + kBandRpt * rq;
        ok0 = active && ty <= ty_last && row0 < B.hm;
        ok1 = kBandRpt > 1 && active && ty <= ty_last && row0 + 1 < B.hm;
#pragma unroll
        for (int r = 0; r < kBandRpt; ++r) {
            const bool okr = r ? ok1 : ok0;
            const int64_t p = off + (int64_t)(row0 + r) * B.wm + x0;
            mm[r] = okr ? __ldg(reinterpret_cast<const float4 *>(mask + p)) : make_float4(0.f, 0.f, 0.f, 0.f);
            nn[r] = okr ? __ldg(reinterpret_cast<const int4 *>(nsamp + p)) : make_int4(0, 0, 0, 0);
            dd[r] = okr ? __ldg(reinterpret_cast<const float4 *>(dexp + p)) : make_float4(0.f, 0.f, 0.f, 0.f);
            zz[r] = (REFINE && okr) ? __ldg(reinterpret_cast<const float4 *>(z + p))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    };
    const int tyb = ty_first + (int)blockIdx.y * kBand2Rows;
    if (tyb > ty_last) return;
    load(tyb);
#pragma unroll 1
    for (int i = 0; i < kBand2Rows; ++i) {
        const int ty = tyb + i;
        if (ty > ty_last) break;
        const int row0 = ty * kBandTile + kBandRpt * rq;
        const bool c0 = ok0, c1 = ok1;
        float4 cm[2] = {mm[0], mm[1]}, cd[2] = {dd[0], dd[1]}, cz[2] = {zz[0], zz[1]};
        int4 cn[2] = {nn[0], nn[1]};
        if (i + 1 < kBand2Rows) load(ty + 1);        // next band's loads in flight meanwhile
        float lo = __int_as_float(0x7f800000);      // +inf
        float hi = -lo;
#pragma unroll
        for (int r = 0; r < kBandRpt; ++r) {
            if (!(r ? c1 : c0)) continue;
            const int64_t p = off + (int64_t)(row0 + r) * B.wm + x0;
            float m[4] = {cm[r].x, cm[r].y, cm[r].z, cm[r].w};
            const int32_t n[4] = {cn[r].x, cn[r].y, cn[r].z, cn[r].w};
            const float d[4] = {cd[r].x, cd[r].y, cd[r].z, cd[r].w};
            if (REFINE) {
                const float zv[4] = {cz[r].x, cz[r].y, cz[r].z, cz[r].w};
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    m[k] = refine_px_fast(m[k], zv[k], n[k], any, lo_ref, span, rspan);
                if (refined)
                    __stcs(reinterpret_cast<float4 *>(refined + p), make_float4(m[0], m[1], m[2], m[3]));
            }
            const int64_t q = p - off;
            float2 a[4], b[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                double t64 = 0.0;
                const float t32 = band_px32(m[k], n[k], d[k], B, lo, hi, t64);
                const bool sup = t32 >= 0.0f;
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
            float4 *a4 = reinterpret_cast<float4 *>(recA + q);
#ifndef DIVAS_REC_EVICT_LAST
#define DIVAS_REC_EVICT_LAST 1
#endif
            if (DIVAS_REC_EVICT_LAST) {
                // the pair kernel reads these next: keep them in L2 (evict-last
                // policy) against the streams running beside this pass
                st_evict_last(a4, make_float4(a[0].x, a[0].y, a[1].x, a[1].y), pol);
                st_evict_last(a4 + 1, make_float4(a[2].x, a[2].y, a[3].x, a[3].y), pol);
            } else {
                a4[0] = make_float4(a[0].x, a[0].y, a[1].x, a[1].y);
                a4[1] = make_float4(a[2].x, a[2].y, a[3].x, a[3].y);
            }
            if (write_b) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (a[k].y == a[k].y) recB[q + k] = b[k];
            }
        }
        // the 8 lanes of a tile: chunk pair (xor 1) x row pairs (xor 8, 16)
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
#pragma unroll
        for (int o = kBandCpw; o < 32; o <<= 1) {          // the tile's other row groups
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (active && rq == 0 && (c & 1) == 0)
            bv[(int64_t)ty * B.ntx + x0 / kBandTile] = make_double2((double)lo, (double)hi);
    }
    if (__any_sync(0xffffffffu, cnt != 0)) {
        for (int o = 16; o > 0; o >>= 1) {
            tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
            tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
            nlo = min(nlo, __shfl_xor_sync(0xffffffffu, nlo, o));
            nhi = max(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if (lane == 0) {
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
    launch_pdl(band_init, dim3((nv + 255) / 256), dim3(256), 0, s, bands, nv, B.nty, B.ntx);
}

}  // namespace divas
