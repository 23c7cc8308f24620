// overlay.cu -- 2D back-projection of the fused grid onto one view.
//
// Reference: fusion._overlay_kernel / project_grid_overlay
// (/root/reference/pkg/src/divas/fusion.py:771-865).  One thread per pixel:
// the ray through the pixel centre marches [d_min - dx, d_max + dx] on valid
// pixels (the grid-box slab otherwise) at half-voxel steps and reports a hit
// on the first voxel with p >= threshold.  Same f64 evaluation order, no FMA.
#include <algorithm>

#include "common.cuh"

namespace divas {

// numba int(x) for f64 x: truncation; out of range -> INT64_MIN (cvttsd2si)
__device__ __forceinline__ long long nb_trunc_int(double x) {
    const double f = trunc(x);
    if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0))
        return (long long)0x8000000000000000ULL;
    return (long long)f;
}

struct OverlayConst {
    double r[9], p[3], fx, fy, cx, cy;
    int h, w;
    int64_t g;
    double o[3], dx, bc[3], bh[3], thr, step;
    int unbounded;
};

__global__ void overlay_kernel(OverlayConst C, const float *__restrict__ dmin,
                               const float *__restrict__ dmax,
                               const int32_t *__restrict__ nsamp,
                               const double *__restrict__ probs, uint8_t *__restrict__ out) {
    const int64_t npix = (int64_t)C.h * C.w;
    for (int64_t pi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pi < npix;
         pi += (int64_t)gridDim.x * blockDim.x) {
        const int iy = (int)(pi / C.w);
        const int ix = (int)(pi - (int64_t)iy * C.w);
        const double xc = ((double)ix + 0.5 - C.cx) / C.fx;
        const double yc = (C.cy - ((double)iy + 0.5)) / C.fy;
        double ddx = C.r[0] * xc + C.r[1] * yc - C.r[2];
        double ddy = C.r[3] * xc + C.r[4] * yc - C.r[5];
        double ddz = C.r[6] * xc + C.r[7] * yc - C.r[8];
        const double norm = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
        ddx /= norm;
        ddy /= norm;
        ddz /= norm;
        double t0, t1;
        if (nsamp[pi] > 0) {
            t0 = (double)dmin[pi] - C.dx;
            if (t0 < 0.0) t0 = 0.0;
            t1 = (double)dmax[pi] + C.dx;
        } else {
            t0 = 0.0;
            t1 = 1e30;
            for (int ax = 0; ax < 3; ++ax) {
                const double o = C.p[ax];
                const double d = ax == 0 ? ddx : (ax == 1 ? ddy : ddz);
                const double lo = C.o[ax];
                const double hi = C.o[ax] + (double)C.g * C.dx;
                if (fabs(d) < 1e-12) {
                    if (o < lo || o > hi) { t1 = -1.0; break; }
                } else {
                    double ta = (lo - o) / d;
                    double tb = (hi - o) / d;
                    if (ta > tb) { const double tmp = ta; ta = tb; tb = tmp; }
                    if (ta > t0) t0 = ta;
                    if (tb < t1) t1 = tb;
                }
            }
            if (t1 < t0) { out[pi] = 0; continue; }
        }
        uint8_t hit = 0;
        const long long n = nb_trunc_int((t1 - t0) / C.step) + 1;
        for (long long i = 0; i < n + 1; ++i) {
            double t = t0 + (double)i * C.step;
            if (t > t1) t = t1;
            double px = C.p[0] + ddx * t;
            double py = C.p[1] + ddy * t;
            double pz = C.p[2] + ddz * t;
            if (C.unbounded != 0) {
                const double nx = (px - C.bc[0]) / C.bh[0];
                const double ny = (py - C.bc[1]) / C.bh[1];
                const double nz = (pz - C.bc[2]) / C.bh[2];
                const double r = sqrt(nx * nx + ny * ny + nz * nz);
                if (r > 1.0) {
                    const double s = (2.0 - 1.0 / r) / r;
                    px = C.bc[0] + nx * s * C.bh[0];
                    py = C.bc[1] + ny * s * C.bh[1];
                    pz = C.bc[2] + nz * s * C.bh[2];
                }
            }
            const long long gx = nb_floor_int((px - C.o[0]) / C.dx);
            const long long gy = nb_floor_int((py - C.o[1]) / C.dx);
            const long long gz = nb_floor_int((pz - C.o[2]) / C.dx);
            if (0 <= gx && gx < C.g && 0 <= gy && gy < C.g && 0 <= gz && gz < C.g) {
                if (probs[(gx * C.g + gy) * C.g + gz] >= C.thr) { hit = 1; break; }
            }
            if (t >= t1) break;
        }
        out[pi] = hit;
    }
}

}  // namespace divas

using namespace divas;

extern "C" int divas_overlay(const double *cam, int32_t h, int32_t w, const float *dmin,
                             const float *dmax, const int32_t *nsamp, const double *probs,
                             int64_t g, const double origin[3], double dx_vox, const double bc[3],
                             const double bh[3], int32_t unbounded, double thr, uint8_t *out,
                             void *stream) {
    if (!cam || !dmin || !dmax || !nsamp || !probs || !out || !origin || !bc || !bh) {
        set_error("divas_overlay: null pointer");
        return DIVAS_EINVAL;
    }
    if (h < 1 || w < 1 || g < 1) { set_error("divas_overlay: empty"); return DIVAS_EINVAL; }
    OverlayConst C;
    for (int i = 0; i < 9; ++i) C.r[i] = cam[i];
    for (int i = 0; i < 3; ++i) {
        C.p[i] = cam[9 + i];
        C.o[i] = origin[i];
        C.bc[i] = bc[i];
        C.bh[i] = bh[i];
    }
    C.fx = cam[12]; C.fy = cam[13]; C.cx = cam[14]; C.cy = cam[15];
    C.h = h; C.w = w; C.g = g; C.dx = dx_vox; C.thr = thr;
    C.step = 0.5 * dx_vox;
    C.unbounded = unbounded;
    const int64_t npix = (int64_t)h * w;
    const int64_t blocks = std::min<int64_t>((npix + 127) / 128, 148 * 64);
    overlay_kernel<<<(unsigned)blocks, 128, 0, (cudaStream_t)stream>>>(C, dmin, dmax, nsamp,
                                                                       probs, out);
    return check_launch("divas_overlay");
}
