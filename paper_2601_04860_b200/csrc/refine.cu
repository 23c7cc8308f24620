// refine.cu -- kernel (a): depth-weighted confidence refinement (paper Eq. 2).
//
// Reference: segmenter.refine_mask (/root/reference/pkg/src/divas/segmenter.py:129-152)
//   valid = n_samples > 0; lo, hi = min, max of z over valid pixels (f64);
//   zhat = (z - lo) / (hi - lo)  (0 if hi - lo <= 0);
//   out = clip(f64(mask) * (1 - zhat), 0, 1) on valid pixels, 0 elsewhere; -> f32 RNE.
//
// Two launches over all views at once, 128-bit loads:
//   1. refine_minmax: per-view min/max of z over valid pixels.  min/max are
//      exact in any order, so blocks reduce in registers + warp shuffles and
//      publish one order-preserving-key atomicMin/atomicMax per block.
//   2. refine_apply: the elementwise pass, visiting views in reverse order so
//      the z / n_samples tiles the reduction read last are still L2-resident.
// HBM bytes per pixel: 8 (reduction) + 16 (apply) minus the L2 hits.
#include "bands.cuh"
#include "tma.cuh"

#include <algorithm>
#include <cstdlib>

namespace divas {

constexpr int kRefineThreads = 256;

// refine_init and band_init in one launch (one kernel boundary less on the
// refine chain): ws may be null (keys supplied by the caller)
__global__ void refine_band_init(uint32_t *ws, double2 *__restrict__ bands, int nv, int nty,
                                 int ntx) {
    griddep_wait();                     // PDL: after the previous kernel completes
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nv) return;
    if (ws) {
        ws[kKeys * v] = 0xffffffffu;
        ws[kKeys * v + 1] = 0u;
        ws[kKeys * v + 2] = 0xffffffffu;
        ws[kKeys * v + 3] = 0u;
    }
    uint32_t *e = reinterpret_cast<uint32_t *>(bands + v * band_view_stride(nty, ntx) +
                                               (int64_t)nty * ntx);
    e[0] = 0xffffffffu;
    e[1] = 0u;
    e[2] = 0u;
    e[3] = 0u;
    e[4] = 0x7fc00000u;
    e[5] = 0xffffffffu;
    e[6] = 0u;
    e[7] = 0u;
}

__global__ void refine_init(uint32_t *ws, int nv) {
    griddep_wait();                     // PDL: after the previous kernel completes
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nv) {
        ws[kKeys * i] = 0xffffffffu;      // z min key
        ws[kKeys * i + 1] = 0u;           // z max key
        ws[kKeys * i + 2] = 0xffffffffu;  // n min over valid pixels
        ws[kKeys * i + 3] = 0u;           // n max
    }
}

__device__ __forceinline__ void block_minmax_publish(uint32_t kmin, uint32_t kmax, uint32_t *slot) {
    __shared__ uint32_t s_min[kRefineThreads / 32], s_max[kRefineThreads / 32];
    for (int o = 16; o > 0; o >>= 1) {
        kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) { s_min[warp] = kmin; s_max[warp] = kmax; }
    __syncthreads();
    if (warp == 0) {
        kmin = lane < kRefineThreads / 32 ? s_min[lane] : 0xffffffffu;
        kmax = lane < kRefineThreads / 32 ? s_max[lane] : 0u;
        for (int o = 16; o > 0; o >>= 1) {
            kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
            kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
        }
        if (lane == 0 && kmin <= kmax) {
            atomicMin(slot, kmin);
            atomicMax(slot + 1, kmax);
        }
    }
}

// grid = (blocks_per_view, nv); VEC = 4 (float4/int4) or 1 (scalar fallback)
template <int VEC>
__global__ void __launch_bounds__(kRefineThreads)
refine_minmax(const float *__restrict__ z, const int32_t *__restrict__ n, int64_t plane,
              uint32_t *__restrict__ ws) {
    griddep_wait();                     // PDL: after the previous kernel completes
    const int v = blockIdx.y;
    const float *zv = z + (int64_t)v * plane;
    const int32_t *nvp = n + (int64_t)v * plane;
    uint32_t kmin = 0xffffffffu, kmax = 0u, nmin = 0xffffffffu, nmax = 0u;
    const int64_t nvec = plane / VEC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (VEC == 4) {
            const float4 zz = __ldg(reinterpret_cast<const float4 *>(zv) + i);
            const int4 nn = __ldg(reinterpret_cast<const int4 *>(nvp) + i);
            // n > 0 pixels: z keys, and the n range (as unsigned: n > 0)
            if (nn.x > 0) { uint32_t k = f32_key(zz.x); kmin = min(kmin, k); kmax = max(kmax, k); }
            if (nn.y > 0) { uint32_t k = f32_key(zz.y); kmin = min(kmin, k); kmax = max(kmax, k); }
            if (nn.z > 0) { uint32_t k = f32_key(zz.z); kmin = min(kmin, k); kmax = max(kmax, k); }
            if (nn.w > 0) { uint32_t k = f32_key(zz.w); kmin = min(kmin, k); kmax = max(kmax, k); }
            // invalid pixels (n <= 0) map to the neutral elements
            nmin = min(nmin, min(min(nn.x > 0 ? (uint32_t)nn.x : 0xffffffffu,
                                     nn.y > 0 ? (uint32_t)nn.y : 0xffffffffu),
                                 min(nn.z > 0 ? (uint32_t)nn.z : 0xffffffffu,
                                     nn.w > 0 ? (uint32_t)nn.w : 0xffffffffu)));
            nmax = max(nmax, (uint32_t)max(max(nn.x, nn.y), max(max(nn.z, nn.w), 0)));
        } else {
            const int32_t nk = __ldg(nvp + i);
            if (nk > 0) {
                uint32_t k = f32_key(__ldg(zv + i));
                kmin = min(kmin, k);
                kmax = max(kmax, k);
                nmin = min(nmin, (uint32_t)nk);
                nmax = max(nmax, (uint32_t)nk);
            }
        }
    }
    block_minmax_publish(kmin, kmax, ws + kKeys * v);
    __syncthreads();                                   // the publish reuses shared memory
    block_minmax_publish(nmin, nmax, ws + kKeys * v + 2);
}

// refine_minmax through the TMA engine: each block streams its run of the
// view's z and n_samples planes through kTmaStages shared-memory stages of
// kTmaTile elements (1-D cp.async.bulk, one elected thread issues, mbarrier
// completion), so the loads need no registers and kTmaStages - 1 tiles stay
// in flight while the block reduces the current one.  Same keys as
// refine_minmax<4> (min / max are exact in any order).  Needs plane % 4 == 0
// and 16-byte aligned planes.
#ifndef DIVAS_TMA_TILE
#define DIVAS_TMA_TILE 1024
#endif
#ifndef DIVAS_TMA_STAGES
#define DIVAS_TMA_STAGES 4
#endif
#ifndef DIVAS_TMA_BPS
#define DIVAS_TMA_BPS 12
#endif
constexpr int kTmaTile = DIVAS_TMA_TILE;   // elements per plane per stage
constexpr int kTmaStages = DIVAS_TMA_STAGES;
__global__ void __launch_bounds__(kRefineThreads)
refine_minmax_tma(const float *__restrict__ z, const int32_t *__restrict__ n, int64_t plane,
                  uint32_t *__restrict__ ws) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *sz = reinterpret_cast<float *>(smem);
    int32_t *sn = reinterpret_cast<int32_t *>(smem + (size_t)kTmaStages * kTmaTile * 4);
    __shared__ __align__(8) uint64_t full[kTmaStages];
    const int v = blockIdx.y;
    const float *zv = z + (int64_t)v * plane;
    const int32_t *nvp = n + (int64_t)v * plane;
    // this block's contiguous run of whole tiles (the last may be partial)
    const int64_t ntiles_v = (plane + kTmaTile - 1) / kTmaTile;
    const int64_t per = (ntiles_v + gridDim.x - 1) / gridDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * per;
    const int64_t t1 = min(ntiles_v, t0 + per);
    uint32_t kmin = 0xffffffffu, kmax = 0u, nmin = 0xffffffffu, nmax = 0u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kTmaStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int64_t t) {                     // thread 0 only
        const int s = (int)(t % kTmaStages);
        const int64_t e0 = t * kTmaTile;
        const uint32_t cnt = (uint32_t)min((int64_t)kTmaTile, plane - e0);
        mbar_arrive_expect_tx(&full[s], 8u * cnt);
        tma_load_1d(sz + (size_t)s * kTmaTile, zv + e0, 4u * cnt, &full[s]);
        tma_load_1d(sn + (size_t)s * kTmaTile, nvp + e0, 4u * cnt, &full[s]);
    };
    if (threadIdx.x == 0)
        for (int64_t t = t0; t < min(t1, t0 + kTmaStages); ++t) issue(t);
    for (int64_t t = t0; t < t1; ++t) {
        const int s = (int)(t % kTmaStages);
        mbar_wait(&full[s], (uint32_t)(((t - t0) / kTmaStages) & 1));
        const int64_t e0 = t * kTmaTile;
        const int cnt = (int)min((int64_t)kTmaTile, plane - e0);
        const float4 *z4 = reinterpret_cast<const float4 *>(sz + (size_t)s * kTmaTile);
        const int4 *n4 = reinterpret_cast<const int4 *>(sn + (size_t)s * kTmaTile);
        for (int i = threadIdx.x; i < cnt / 4; i += blockDim.x) {
            const float4 zz = z4[i];
            const int4 nn = n4[i];
            if (nn.x > 0) { uint32_t k = f32_key(zz.x); kmin = min(kmin, k); kmax = max(kmax, k); }
            if (nn.y > 0) { uint32_t k = f32_key(zz.y); kmin = min(kmin, k); kmax = max(kmax, k); }
            if (nn.z > 0) { uint32_t k = f32_key(zz.z); kmin = min(kmin, k); kmax = max(kmax, k); }
            if (nn.w > 0) { uint32_t k = f32_key(zz.w); kmin = min(kmin, k); kmax = max(kmax, k); }
            nmin = min(nmin, min(min(nn.x > 0 ? (uint32_t)nn.x : 0xffffffffu,
                                     nn.y > 0 ? (uint32_t)nn.y : 0xffffffffu),
                                 min(nn.z > 0 ? (uint32_t)nn.z : 0xffffffffu,
                                     nn.w > 0 ? (uint32_t)nn.w : 0xffffffffu)));
            nmax = max(nmax, (uint32_t)max(max(nn.x, nn.y), max(max(nn.z, nn.w), 0)));
        }
        __syncthreads();                              // stage s consumed by every thread
        if (threadIdx.x == 0 && t + kTmaStages < t1) {
            // order those generic-proxy reads before the bulk copy's writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(t + kTmaStages);
        }
    }
    block_minmax_publish(kmin, kmax, ws + kKeys * v);
    __syncthreads();
    block_minmax_publish(nmin, nmax, ws + kKeys * v + 2);
}

// band_pass2<true> with its plane loads moved to the TMA engine: a block's
// 64-px strip of each 8-row tile band is brought into shared memory by 32
// one-dimensional bulk copies (warp 0: one lane per (plane, row), completion
// on an mbarrier), two stages deep, so the next band streams in while the
// current one is computed and the threads issue no global loads or address
// arithmetic for the planes.  Rows are staged from the strip start rounded
// down to 16 bytes (68 floats per staged row: the rounding slack, and rows
// land in different banks); the arithmetic, records and bands are
// band_pass2's, so the outputs are identical.  Needs wm % 4 == 0 and
// 16-byte aligned planes (the launcher checks; band_pass2 otherwise).
constexpr int kTmaStrip = kBand2Warps * kBandCpw * 4;    // pixels per block strip
constexpr int kTmaRowF = kTmaStrip + 4;                   // staged row, in floats
constexpr int kTmaBandStages = 2;
constexpr size_t kTmaBandSmem = (size_t)kTmaBandStages * 4 * kBandTile * kTmaRowF * 4;
__global__ void __launch_bounds__(32 * kBand2Warps)
band_pass_tma(BandParams B, const float *__restrict__ mask, const float *__restrict__ z,
              const int32_t *__restrict__ nsamp, const float *__restrict__ dexp,
              float *__restrict__ refined, const uint32_t *__restrict__ minmax,
              double2 *__restrict__ bands, float2 *__restrict__ records, int nv,
              const int4 *__restrict__ roi) {
    static_assert(kBandTile == 8 && kBandRpt == 1, "TMA band pass: 8x8 tiles, one row per thread");
    extern __shared__ __align__(128) float bsm[];              // [stage][plane][row][kTmaRowF]
    __shared__ __align__(8) uint64_t s_bar[kTmaBandStages];
    const int v = nv - 1 - (int)blockIdx.z;
    const uint64_t pol = l2_policy_evict_last();
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
    const int strip = rx0 + (int)blockIdx.x * kTmaStrip;           // block's first pixel
    const int sx0 = strip & ~3;                                     // staged from here
    const int sofs = strip - sx0;                                   // 0..3, block-uniform
    const int cl = warp * kBandCpw + c;                             // chunk within the strip
    const int x0 = strip + cl * 4;
    const bool active = x0 <= rx1 && x0 < B.wm;
    bool any = false;
    double lo_ref = 0.0, span = 0.0, rspan = 0.0;
    {
        const uint32_t kmin = keys.x, kmax = keys.y;
        any = kmin <= kmax;
        lo_ref = any ? (double)key_f32(kmin) : 0.0;
        const double hi_ref = any ? (double)key_f32(kmax) : 0.0;
        span = hi_ref - lo_ref;
        rspan = span > 0.0 ? 1.0 / span : 0.0;
    }
    uint32_t tmin = 0xffffffffu, tmax = 0u, nlo = 0xffffffffu, nhi = 0u, cnt = 0;
    double2 *bv = bands + (int64_t)v * band_view_stride(B.nty, B.ntx);
    const int tyb = ty_first + (int)blockIdx.y * kBand2Rows;
    if (tyb > ty_last || strip > rx1 || strip >= B.wm) return;      // block-uniform
    if (threadIdx.x == 0) {
        for (int s2 = 0; s2 < kTmaBandStages; ++s2) mbar_init(&s_bar[s2], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int len = min(kTmaRowF, B.wm - sx0);                      // floats per staged row
    const float *const planes[4] = {mask, z, reinterpret_cast<const float *>(nsamp), dexp};
    // warp 0: one (plane, row) bulk copy per lane into stage st for tile band ty
    auto issue = [&](int ty, int st) {
        const int pl = lane >> 3, r = lane & 7;
        const int row = ty * kBandTile + r;
        const bool ok = ty <= ty_last && row < B.hm;
        const uint32_t bytes = ok ? (uint32_t)len * 4u : 0u;
        const uint32_t total = __reduce_add_sync(0xffffffffu, bytes);
        if (lane == 0) mbar_arrive_expect_tx(&s_bar[st], total);
        __syncwarp();
        if (ok)
            tma_load_1d(bsm + (((size_t)st * 4 + pl) * kBandTile + r) * kTmaRowF,
                        planes[pl] + off + (int64_t)row * B.wm + sx0, bytes, &s_bar[st]);
    };
    if (warp == 0) {
        issue(tyb, 0);
        if (kBand2Rows > 1) issue(tyb + 1, 1);
    }
#pragma unroll 1
    for (int i = 0; i < kBand2Rows; ++i) {
        const int ty = tyb + i;
        if (ty > ty_last) break;
        const int st = i % kTmaBandStages;
        mbar_wait(&s_bar[st], (uint32_t)((i / kTmaBandStages) & 1));
        const int row0 = ty * kBandTile + rq;
        const bool c0 = active && row0 < B.hm;
        float lo = __int_as_float(0x7f800000);      // +inf
        float hi = -lo;
        if (c0) {
            const float *sp = bsm + ((size_t)st * 4 * kBandTile + rq) * kTmaRowF + sofs + cl * 4;
            const size_t ps = (size_t)kBandTile * kTmaRowF;          // plane stride
            float m[4], zv[4], d[4];
            int32_t n[4];
            if (sofs == 0) {
                const float4 m4 = *reinterpret_cast<const float4 *>(sp);
                const float4 z4 = *reinterpret_cast<const float4 *>(sp + ps);
                const float4 n4 = *reinterpret_cast<const float4 *>(sp + 2 * ps);
                const float4 d4 = *reinterpret_cast<const float4 *>(sp + 3 * ps);
                m[0] = m4.x; m[1] = m4.y; m[2] = m4.z; m[3] = m4.w;
                zv[0] = z4.x; zv[1] = z4.y; zv[2] = z4.z; zv[3] = z4.w;
                n[0] = __float_as_int(n4.x); n[1] = __float_as_int(n4.y);
                n[2] = __float_as_int(n4.z); n[3] = __float_as_int(n4.w);
                d[0] = d4.x; d[1] = d4.y; d[2] = d4.z; d[3] = d4.w;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    m[k] = sp[k];
                    zv[k] = sp[ps + k];
                    n[k] = __float_as_int(sp[2 * ps + k]);
                    d[k] = sp[3 * ps + k];
                }
            }
            const int64_t p = off + (int64_t)row0 * B.wm + x0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                m[k] = refine_px_fast(m[k], zv[k], n[k], any, lo_ref, span, rspan);
            if (refined)
                __stcs(reinterpret_cast<float4 *>(refined + p), make_float4(m[0], m[1], m[2], m[3]));
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
            st_evict_last(a4, make_float4(a[0].x, a[0].y, a[1].x, a[1].y), pol);
            st_evict_last(a4 + 1, make_float4(a[2].x, a[2].y, a[3].x, a[3].y), pol);
            if (write_b) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (a[k].y == a[k].y) recB[q + k] = b[k];
            }
        }
        // the 8 lanes of a tile: chunk pair (xor 1) x row groups (xor 4, 8, 16)
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
#pragma unroll
        for (int o = kBandCpw; o < 32; o <<= 1) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (active && rq == 0 && (c & 1) == 0)
            bv[(int64_t)ty * B.ntx + x0 / kBandTile] = make_double2((double)lo, (double)hi);
        if (i + kTmaBandStages < kBand2Rows) {
            __syncthreads();                          // every thread is done with stage st
            if (warp == 0) {
                // order those generic-proxy reads before the bulk copy's writes
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(ty + kTmaBandStages, st);
            }
        }
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

static int blocks_per_view(int64_t plane, int nv);

static void launch_minmax(const float *z, const int32_t *n, int64_t plane, int nv, uint32_t *ws,
                          cudaStream_t s) {
    // The TMA pipeline is selected at run time with DIVAS_TMA=1 (measured on
    // C3: 40.1 us against 39.2 us for refine_minmax<4>'s 128-bit loads, which
    // already stream at ~5 TB/s; tests/test_gpu_tma.py keeps it exact).
    static int use_tma = -1;
    if (use_tma < 0) {
        const char *e = getenv("DIVAS_TMA");
        use_tma = (e && e[0] == '1') ? 1 : 0;
    }
    const size_t smem = (size_t)kTmaStages * kTmaTile * 8;
    static unsigned long long attr_set = 0;        // bit per device ordinal < 64
    if (use_tma && plane % 4 == 0 && ((((uintptr_t)z) | ((uintptr_t)n)) & 15) == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        const unsigned long long bit = 1ull << (dev & 63);
        if (!(__atomic_load_n(&attr_set, __ATOMIC_RELAXED) & bit)) {
            cudaFuncSetAttribute(refine_minmax_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
            __atomic_fetch_or(&attr_set, bit, __ATOMIC_RELAXED);
        }
        // blocks per view: enough for ~3 resident blocks per SM over all views
        const int64_t ntiles = (plane + kTmaTile - 1) / kTmaTile;
        int64_t b = std::max<int64_t>(1, std::min<int64_t>(ntiles, (148 * DIVAS_TMA_BPS + nv - 1) / nv));
        dim3 grid((unsigned)b, (unsigned)nv);
        refine_minmax_tma<<<grid, kRefineThreads, smem, s>>>(z, n, plane, ws);
    } else {
        dim3 grid(blocks_per_view(plane, nv), nv);
        if (plane % 4 == 0 && ((((uintptr_t)z) | ((uintptr_t)n)) & 15) == 0)
            launch_pdl(refine_minmax<4>, grid, dim3(kRefineThreads), 0, s, z, n, plane, ws);
        else
            refine_minmax<1><<<grid, kRefineThreads, 0, s>>>(z, n, plane, ws);
    }
}

template <int VEC>
__global__ void __launch_bounds__(kRefineThreads)
refine_apply(const float *__restrict__ mask, const float *__restrict__ z,
             const int32_t *__restrict__ n, float *__restrict__ out, int64_t plane,
             const uint32_t *__restrict__ ws) {
    griddep_wait();                     // PDL: after the previous kernel completes
    const int v = gridDim.y - 1 - blockIdx.y;   // reverse view order: L2 reuse
    const uint32_t kmin = ws[kKeys * v], kmax = ws[kKeys * v + 1];
    const bool any = kmin <= kmax;
    const double lo = any ? (double)key_f32(kmin) : 0.0;
    const double hi = any ? (double)key_f32(kmax) : 0.0;
    const double span = hi - lo;
    const double rspan = span > 0.0 ? 1.0 / span : 0.0;
    const int64_t off = (int64_t)v * plane;
    const int64_t nvec = plane / VEC;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (VEC == 4) {
            const float4 m = __ldg(reinterpret_cast<const float4 *>(mask + off) + i);
            const float4 zz = __ldg(reinterpret_cast<const float4 *>(z + off) + i);
            const int4 nn = __ldg(reinterpret_cast<const int4 *>(n + off) + i);
            float4 o;
            o.x = refine_px_fast(m.x, zz.x, nn.x, any, lo, span, rspan);
            o.y = refine_px_fast(m.y, zz.y, nn.y, any, lo, span, rspan);
            o.z = refine_px_fast(m.z, zz.z, nn.z, any, lo, span, rspan);
            o.w = refine_px_fast(m.w, zz.w, nn.w, any, lo, span, rspan);
            __stcs(reinterpret_cast<float4 *>(out + off) + i, o);
        } else {
            out[off + i] = refine_px_fast(mask[off + i], z[off + i], n[off + i], any, lo, span, rspan);
        }
    }
}

static int blocks_per_view(int64_t plane, int nv) {
    int64_t b = (plane / 4 + 4 * kRefineThreads - 1) / (4 * kRefineThreads);
    int64_t cap = 4096 / (nv > 0 ? nv : 1);
    if (cap < 1) cap = 1;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace divas

using namespace divas;

extern "C" size_t divas_refine_workspace_size(int32_t nv) {
    return (size_t)(nv > 0 ? nv : 1) * kKeys * sizeof(uint32_t);
}

extern "C" int divas_refine(int32_t nv, int64_t hm, int64_t wm, const float *mask,
                            const float *z_surface, const int32_t *n_samples, float *out,
                            void *workspace, size_t workspace_bytes, void *stream) {
    if (nv <= 0 || hm <= 0 || wm <= 0) { set_error("divas_refine: empty view set"); return DIVAS_EINVAL; }
    if (nv > 65535) { set_error("divas_refine: too many views (%d)", nv); return DIVAS_EINVAL; }
    if (!mask || !z_surface || !n_samples || !out || !workspace) {
        set_error("divas_refine: null pointer");
        return DIVAS_EINVAL;
    }
    if (workspace_bytes < divas_refine_workspace_size(nv)) {
        set_error("divas_refine: workspace too small");
        return DIVAS_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *ws = (uint32_t *)workspace;
    const int64_t plane = hm * wm;
    const bool vec = (plane % 4 == 0) &&
                     ((((uintptr_t)mask) | ((uintptr_t)z_surface) | ((uintptr_t)n_samples) |
                       ((uintptr_t)out)) & 15) == 0;
    refine_init<<<(nv + 255) / 256, 256, 0, s>>>(ws, nv);
    dim3 grid(blocks_per_view(plane, nv), nv);
    launch_minmax(z_surface, n_samples, plane, nv, ws, s);
    if (vec) {
        launch_pdl(refine_apply<4>, grid, dim3(kRefineThreads), 0, s, mask, z_surface, n_samples,
                   out, plane, (const uint32_t *)ws);
    } else {
        refine_apply<1><<<grid, kRefineThreads, 0, s>>>(mask, z_surface, n_samples, out, plane, ws);
    }
    return check_launch("divas_refine");
}

static int refine_bands_impl(int32_t nv, int64_t hm, int64_t wm, const float *mask,
                             const float *z_surface, const int32_t *n_samples, const float *dexp,
                             float *out, const double *pv, double dx_vox, void *records,
                             void *bands, void *workspace, size_t workspace_bytes,
                             const int32_t *roi, int32_t roi_w, int32_t roi_h,
                             const uint32_t *keys, void *stream) {
    if (nv <= 0 || hm <= 0 || wm <= 0) { set_error("divas_refine_bands: empty view set"); return DIVAS_EINVAL; }
    if (nv > 65535 || hm > 0x7fffffff / 2 || wm > 0x7fffffff / 2) {
        set_error("divas_refine_bands: plane too large");
        return DIVAS_EINVAL;
    }
    if (!mask || !z_surface || !n_samples || !dexp || !pv || !records || !bands || !workspace) {
        set_error("divas_refine_bands: null pointer");
        return DIVAS_EINVAL;
    }
    if (workspace_bytes < divas_refine_workspace_size(nv)) {
        set_error("divas_refine_bands: workspace too small");
        return DIVAS_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    uint32_t *ws = (uint32_t *)workspace;
    const int64_t plane = hm * wm;
    const bool vec = (wm % 4 == 0) &&
                     ((((uintptr_t)mask) | ((uintptr_t)z_surface) | ((uintptr_t)n_samples) |
                       ((uintptr_t)out) | ((uintptr_t)dexp) | ((uintptr_t)records)) & 15) == 0;
    // keys: the views' z min / max computed elsewhere (divas_refine_minmax,
    // e.g. by another rank); else computed here
    const uint32_t *mm = keys ? keys : ws;
    dim3 grid(blocks_per_view(plane, nv), nv);
    const BandParams B = band_params(pv, dx_vox, (int)hm, (int)wm);
    launch_pdl(refine_band_init, dim3((nv + 255) / 256), dim3(256), 0, s, keys ? nullptr : ws,
               (double2 *)bands, nv, B.nty, B.ntx);
    // grid extent: the whole plane, or the largest window (+ one tile of slack
    // for a window start that is not tile aligned in the caller's numbers)
    const int64_t gw = roi ? std::min<int64_t>(wm, (int64_t)roi_w + kBandTile) : wm;
    const int64_t gty = roi ? std::min<int64_t>(B.nty, (roi_h + kBandTile - 1) / kBandTile + 1)
                            : B.nty;
    const int4 *r4 = reinterpret_cast<const int4 *>(roi);
    if (vec) {
        if (!keys) launch_minmax(z_surface, n_samples, plane, nv, ws, s);
        // threads per block: enough 4-pixel chunks for the (window) width, in
        // warps, so narrow windows do not idle half of every block
        const int64_t chunks = gw / 4;
#ifndef DIVAS_BAND_ROWSPLIT
#define DIVAS_BAND_ROWSPLIT 1
#endif
        if (DIVAS_BAND_ROWSPLIT && kBandTile == 8) {
            // row-split pass: 8 chunks per warp, kBand2Warps warps per block
            const int64_t per = kBandCpw * kBand2Warps;
            dim3 bg((unsigned)((chunks + per - 1) / per),
                    (unsigned)((gty + kBand2Rows - 1) / kBand2Rows), (unsigned)nv);
            // TMA staging is opt-in (DIVAS_BAND_TMA=1): measured on C3 85 us
            // against 77 us for band_pass2, which is issue-bound, not
            // load-latency-bound (tests/test_gpu_tma.py keeps it exact)
            static int use_tma = -1;
            if (use_tma < 0) {
                const char *e = getenv("DIVAS_BAND_TMA");
                use_tma = (e && e[0] == '1') ? 1 : 0;
            }
            const bool tma_ok = use_tma && wm % 4 == 0 &&
                                ((((uintptr_t)mask) | ((uintptr_t)z_surface) |
                                  ((uintptr_t)n_samples) | ((uintptr_t)dexp)) & 15) == 0;
            if (tma_ok) {
                static unsigned long long attr_set = 0;   // bit per device ordinal < 64
                int dev = 0;
                cudaGetDevice(&dev);
                const unsigned long long bit = 1ull << (dev & 63);
                if (!(__atomic_load_n(&attr_set, __ATOMIC_RELAXED) & bit)) {
                    cudaFuncSetAttribute(band_pass_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kTmaBandSmem);
                    __atomic_fetch_or(&attr_set, bit, __ATOMIC_RELAXED);
                }
                band_pass_tma<<<bg, 32 * kBand2Warps, kTmaBandSmem, s>>>(
                    B, mask, z_surface, n_samples, dexp, out, mm, (double2 *)bands,
                    (float2 *)records, nv, r4);
            } else {
                launch_pdl(band_pass2<true>, bg, dim3(32 * kBand2Warps), 0, s, B, mask,
                           z_surface, n_samples, dexp, out, mm, (double2 *)bands,
                           (float2 *)records, nv, r4);
            }
        } else {
            const int bt = (int)std::min<int64_t>(256, std::max<int64_t>(32, (chunks + 31) / 32 * 32));
            dim3 bg((unsigned)((chunks + bt - 1) / bt), (unsigned)gty, (unsigned)nv);
            band_pass<4, true><<<bg, bt, 0, s>>>(B, mask, z_surface, n_samples, dexp, out, mm,
                                                 (double2 *)bands, (float2 *)records, nv, r4);
        }
    } else {
        if (!keys) launch_minmax(z_surface, n_samples, plane, nv, ws, s);
        dim3 bg((unsigned)((gw + 255) / 256), (unsigned)gty, (unsigned)nv);
        band_pass<1, true><<<bg, 256, 0, s>>>(B, mask, z_surface, n_samples, dexp, out, mm,
                                              (double2 *)bands, (float2 *)records, nv, r4);
    }
    return check_launch("divas_refine_bands");
}

extern "C" int divas_refine_bands(int32_t nv, int64_t hm, int64_t wm, const float *mask,
                                  const float *z_surface, const int32_t *n_samples,
                                  const float *dexp, float *out, const double *pv, double dx_vox,
                                  void *records, void *bands, void *workspace,
                                  size_t workspace_bytes, void *stream) {
    return refine_bands_impl(nv, hm, wm, mask, z_surface, n_samples, dexp, out, pv, dx_vox,
                             records, bands, workspace, workspace_bytes, nullptr, 0, 0, nullptr,
                             stream);
}

extern "C" int divas_refine_minmax(int32_t nv, int64_t hm, int64_t wm, const float *z_surface,
                                   const int32_t *n_samples, uint32_t *keys, void *stream) {
    if (nv <= 0 || hm <= 0 || wm <= 0 || !z_surface || !n_samples || !keys) {
        set_error("divas_refine_minmax: bad arguments");
        return DIVAS_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t plane = hm * wm;
    refine_init<<<(nv + 255) / 256, 256, 0, s>>>(keys, nv);
    launch_minmax(z_surface, n_samples, plane, nv, keys, s);
    return check_launch("divas_refine_minmax");
}

extern "C" int divas_refine_bands_keys(int32_t nv, int64_t hm, int64_t wm, const float *mask,
                                       const float *z_surface, const int32_t *n_samples,
                                       const float *dexp, float *out, const double *pv,
                                       double dx_vox, void *records, void *bands,
                                       const uint32_t *keys, void *workspace,
                                       size_t workspace_bytes, const int32_t *roi, int32_t roi_w,
                                       int32_t roi_h, void *stream) {
    if (!keys) { set_error("divas_refine_bands_keys: null keys"); return DIVAS_EINVAL; }
    if (roi && (roi_w < 1 || roi_h < 1)) {
        set_error("divas_refine_bands_keys: empty window");
        return DIVAS_EINVAL;
    }
    return refine_bands_impl(nv, hm, wm, mask, z_surface, n_samples, dexp, out, pv, dx_vox,
                             records, bands, workspace, workspace_bytes, roi, roi_w, roi_h, keys,
                             stream);
}

extern "C" int divas_refine_bands_roi(int32_t nv, int64_t hm, int64_t wm, const float *mask,
                                      const float *z_surface, const int32_t *n_samples,
                                      const float *dexp, float *out, const double *pv,
                                      double dx_vox, void *records, void *bands, void *workspace,
                                      size_t workspace_bytes, const int32_t *roi, int32_t roi_w,
                                      int32_t roi_h, void *stream) {
    if (!roi || roi_w < 1 || roi_h < 1) {
        set_error("divas_refine_bands_roi: empty window");
        return DIVAS_EINVAL;
    }
    return refine_bands_impl(nv, hm, wm, mask, z_surface, n_samples, dexp, out, pv, dx_vox,
                             records, bands, workspace, workspace_bytes, roi, roi_w, roi_h,
                             nullptr, stream);
}

extern "C" size_t divas_records_size(int32_t nv, int64_t hm, int64_t wm) {
    return (size_t)(nv > 0 ? nv : 0) * (size_t)(hm > 0 ? hm : 0) * (size_t)(wm > 0 ? wm : 0) *
           sizeof(float4);
}

extern "C" size_t divas_bands_size(int32_t nv, int64_t hm, int64_t wm) {
    return band_bytes(nv, (int)hm, (int)wm);
}

// ---------------------------------------------------------------------------
// Bounding box of the pixels whose mask is >= thr, per view: the upload
// window of d_min / d_max / d_exp in refine_and_fuse.  Those maps are read
// by the fusion only at pixels whose refined mask reaches mask_thr (thick
// centres) or exceeds 0.5 (thin support) -- refined <= raw, so raw >= thr
// with thr <= both -- and at the 4-neighbours of thick centres (gradient).
// ---------------------------------------------------------------------------
namespace divas {

__global__ void bbox_init(int32_t *bbox, int nv) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nv) {
        bbox[4 * i] = 0x7fffffff;
        bbox[4 * i + 1] = 0x7fffffff;
        bbox[4 * i + 2] = -1;
        bbox[4 * i + 3] = -1;
    }
}

// grid (blocks_per_view, nv); one pixel per thread per iteration
__global__ void __launch_bounds__(kRefineThreads)
mask_bbox(const float *__restrict__ masks, int64_t hm, int64_t wm, float thr,
          int32_t *__restrict__ bbox) {
    const int v = blockIdx.y;
    const int64_t plane = hm * wm;
    const float *m = masks + (int64_t)v * plane;
    int x0 = 0x7fffffff, y0 = 0x7fffffff, x1 = -1, y1 = -1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < plane;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (__ldg(m + i) >= thr) {
            const int y = (int)(i / wm), x = (int)(i - (int64_t)y * wm);
            x0 = min(x0, x); x1 = max(x1, x);
            y0 = min(y0, y); y1 = max(y1, y);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o));
        y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
        x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o));
        y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
    }
    if ((threadIdx.x & 31) == 0 && x1 >= 0) {
        atomicMin(bbox + 4 * v, x0);
        atomicMin(bbox + 4 * v + 1, y0);
        atomicMax(bbox + 4 * v + 2, x1);
        atomicMax(bbox + 4 * v + 3, y1);
    }
}

}  // namespace divas

extern "C" int divas_mask_bbox(int32_t nv, int64_t hm, int64_t wm, const float *masks, float thr,
                               int32_t *bbox, void *stream) {
    if (nv <= 0 || hm <= 0 || wm <= 0 || !masks || !bbox) {
        set_error("divas_mask_bbox: bad arguments");
        return DIVAS_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    bbox_init<<<(nv + 255) / 256, 256, 0, s>>>(bbox, nv);
    dim3 grid(blocks_per_view(hm * wm, nv), nv);
    mask_bbox<<<grid, kRefineThreads, 0, s>>>(masks, hm, wm, thr, bbox);
    return check_launch("divas_mask_bbox");
}
