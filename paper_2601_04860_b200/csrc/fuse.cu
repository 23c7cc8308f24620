// fuse.cu -- kernel (b): multi-view voxel fusion.
//
// Reference: fusion._fuse_kernel -> _voxel_views (/root/reference/pkg/src/divas/
// fusion.py:493-509, :410-490) with its helpers _project_px (:170-184),
// _pixel_index (:187-192), _grad_at (:195-229, padded-plane semantics of
// _gradient_maps :684-689), _contract_pt (:243-254), _thick_pair (:257-303),
// _thin_pair (:306-370) and the value-sorted sums (:373-407).
//
// Pipeline (both launches on the caller's stream, no host sync):
//   fuse_gate    dense stream over the slab [lo, hi): 16-byte rho loads, 32-byte
//                zero stores of p (and optional votes / occupancy), and a
//                warp-aggregated append of every voxel that clears the exact
//                density gate  rho >= rho_thr || (enable_thin && rho >= rho_thin)
//                to a work list.  Below both gates no pair can vote, so p = 0
//                exactly ("exact shortcuts").
//   fuse_sparse  persistent grid (SM count x occupancy) walking the work list,
//                one voxel per thread, all views per thread.  Camera records
//                are staged once per CTA in shared memory (broadcast reads).
//                Contributions are inserted into per-thread sorted scratch so
//                the sums run in the reference's value-sorted order: results
//                are bit-identical under view permutation, as the reference's.
//
// Arithmetic: IEEE f64 in the reference's evaluation order, no FMA (this TU is
// compiled with -fmad=false), binary32 exactly at the 8 numba f32 sites.
#include <algorithm>

#include "common.cuh"

namespace divas {

struct FuseConst {
    int64_t g, lo, hi;
    double origin0, origin1, origin2, dx;
    int nv, hm, wm;
    double gamma, beta, bmax, lam, rho_thr, rho_thin, thin_pct, alpha1, thin_accept, eps,
        mask_thr, thin_floor, kappa;
    int enable_thin;
    double bc0, bc1, bc2, bh0, bh1, bh2;
    int unbounded;
    double occ_thr;
};

struct FuseOut {
    double *probs;
    int32_t *n_thick, *n_thin;
    double *sw, *smw, *st;
    uint8_t *occ;
};

struct FuseMaps {
    const float *masks, *dmins, *dmaxs, *dexps;
    const int32_t *nsamps;
};

// ---------------------------------------------------------------------------
// dense gate pass
// ---------------------------------------------------------------------------
constexpr int kGateThreads = 256;

__device__ __forceinline__ bool density_gate(float rho, const FuseConst &C) {
    const double r = (double)rho;
    return r >= C.rho_thr || (C.enable_thin && r >= C.rho_thin);
}

// Each thread owns 4 consecutive voxels (one float4 of rho).  The loop walks
// warp-uniform strides so all 32 lanes reach the shuffles together.
__global__ void __launch_bounds__(kGateThreads)
fuse_gate(const float *__restrict__ dens, FuseConst C, FuseOut O, uint32_t *__restrict__ work,
          unsigned long long *__restrict__ count) {
    const int lane = threadIdx.x & 31;
    const int64_t n = C.hi - C.lo;
    const int64_t nquads = (n + 3) / 4;
    const bool aligned = (C.lo & 3) == 0;
    const uint8_t occ0 = (0.0 >= C.occ_thr) ? 1 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t wbase = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); wbase < nquads;
         wbase += stride) {
        const int64_t q = wbase + lane;
        const int64_t base = C.lo + 4 * q;
        float r[4];
        int k4 = 0;
        if (q < nquads) {
            { const int64_t left = C.hi - base; k4 = left < 4 ? (int)left : 4; }
            if (aligned && k4 == 4) {
                const float4 v = __ldg(reinterpret_cast<const float4 *>(dens + base));
                r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
            } else {
                for (int k = 0; k < 4; ++k) r[k] = k < k4 ? __ldg(dens + base + k) : 0.f;
            }
            if (aligned && k4 == 4) {
                const double2 z2 = make_double2(0.0, 0.0);
                __stcs(reinterpret_cast<double2 *>(O.probs + base), z2);
                __stcs(reinterpret_cast<double2 *>(O.probs + base) + 1, z2);
                if (O.n_thick) *reinterpret_cast<int4 *>(O.n_thick + base) = make_int4(0, 0, 0, 0);
                if (O.n_thin) *reinterpret_cast<int4 *>(O.n_thin + base) = make_int4(0, 0, 0, 0);
                if (O.sw) {
                    reinterpret_cast<double2 *>(O.sw + base)[0] = z2;
                    reinterpret_cast<double2 *>(O.sw + base)[1] = z2;
                }
                if (O.smw) {
                    reinterpret_cast<double2 *>(O.smw + base)[0] = z2;
                    reinterpret_cast<double2 *>(O.smw + base)[1] = z2;
                }
                if (O.st) {
                    reinterpret_cast<double2 *>(O.st + base)[0] = z2;
                    reinterpret_cast<double2 *>(O.st + base)[1] = z2;
                }
                if (O.occ) *reinterpret_cast<uchar4 *>(O.occ + base) = make_uchar4(occ0, occ0, occ0, occ0);
            } else {
                for (int k = 0; k < k4; ++k) {
                    O.probs[base + k] = 0.0;
                    if (O.n_thick) O.n_thick[base + k] = 0;
                    if (O.n_thin) O.n_thin[base + k] = 0;
                    if (O.sw) O.sw[base + k] = 0.0;
                    if (O.smw) O.smw[base + k] = 0.0;
                    if (O.st) O.st[base + k] = 0.0;
                    if (O.occ) O.occ[base + k] = occ0;
                }
            }
        }
        unsigned bits = 0;
        for (int k = 0; k < k4; ++k)
            if (density_gate(r[k], C)) bits |= 1u << k;
        const int cnt = __popc(bits);
        int incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total == 0) continue;
        unsigned long long slot = 0;
        if (lane == 31) slot = atomicAdd(count, (unsigned long long)total);
        slot = __shfl_sync(0xffffffffu, slot, 31) + (unsigned long long)(incl - cnt);
        while (bits) {
            const int k = __ffs(bits) - 1;
            bits &= bits - 1;
            work[slot++] = (uint32_t)(base + k);
        }
    }
}

// ---------------------------------------------------------------------------
// per-pair arithmetic (exact restatement of the reference helpers)
// ---------------------------------------------------------------------------
struct Cam {
    const double *r;   // r[9] row-major: r[row*3 + col]
    double p0, p1, p2, fx, fy, cx, cy, w, h;
};

__device__ __forceinline__ Cam load_cam(const double *s, int v) {
    const double *c = s + v * kCamStride;
    Cam k;
    k.r = c;
    k.p0 = c[9]; k.p1 = c[10]; k.p2 = c[11];
    k.fx = c[12]; k.fy = c[13]; k.cx = c[14]; k.cy = c[15]; k.w = c[16]; k.h = c[17];
    return k;
}

// _project_px (fusion.py:170-184); returns in_front, writes u, v, d
__device__ __forceinline__ bool project_px(const Cam &k, double px, double py, double pz,
                                           double &u, double &v, double &d) {
    const double relx = px - k.p0;
    const double rely = py - k.p1;
    const double relz = pz - k.p2;
    const double zc = k.r[2] * relx + k.r[5] * rely + k.r[8] * relz;
    d = -zc;
    if (d <= 0.0) { u = -1.0; v = -1.0; return false; }
    const double xc = k.r[0] * relx + k.r[3] * rely + k.r[6] * relz;
    const double yc = k.r[1] * relx + k.r[4] * rely + k.r[7] * relz;
    u = (k.fx * (xc / d) + k.cx) / k.w;
    v = (k.cy - k.fy * (yc / d)) / k.h;
    return true;
}

// _pixel_index (fusion.py:187-192)
__device__ __forceinline__ long long pixel_index(double u, long long n) {
    long long i = nb_floor_int(u * (double)n);
    if (i > n - 1) i = n - 1;
    return i;
}

// _grad_at over the padded (hm, wm) plane (fusion.py:195-229, :684-689)
__device__ __forceinline__ double grad_at(const float *__restrict__ dexp,
                                          const float *__restrict__ dmin,
                                          const float *__restrict__ dmax, int hm, int wm, int ix,
                                          int iy, double eps, double kappa) {
    const int64_t c = (int64_t)iy * wm + ix;
    const float center = __ldg(dexp + c);
    const float r32 = __ldg(dmax + c) - __ldg(dmin + c);            // f32 site
    const double rng = (double)r32 + eps;
    double gmax = 0.0, s;
    if (ix > 0) {
        s = (double)fabsf(__ldg(dexp + c - 1) - center) / rng;      // f32 site
        if (s > gmax) gmax = s;
    }
    if (ix < wm - 1) {
        s = (double)fabsf(__ldg(dexp + c + 1) - center) / rng;
        if (s > gmax) gmax = s;
    }
    if (iy > 0) {
        s = (double)fabsf(__ldg(dexp + c - wm) - center) / rng;
        if (s > gmax) gmax = s;
    }
    if (iy < hm - 1) {
        s = (double)fabsf(__ldg(dexp + c + wm) - center) / rng;
        if (s > gmax) gmax = s;
    }
    double g = 1.0 / (1.0 + kappa * gmax);
    const double hi = 1.0 - eps;
    if (g > hi) g = hi;
    if (g < 0.0) g = 0.0;
    return g;
}

// _thick_pair (fusion.py:257-303); returns ok, writes the depth weight
__device__ __forceinline__ bool thick_pair(const FuseConst &C, const Cam &k, double xc0,
                                           double xc1, double xc2, double u, double v,
                                           double x_d, float dmin, float dmax, float dexp,
                                           int32_t nsamp, double g, double &wd) {
    const double *R = k.r;
    const double rx = (u * k.w - k.cx) / k.fx;
    const double ry = (k.cy - v * k.h) / k.fy;
    double ddx = R[0] * rx + R[1] * ry - R[2];
    double ddy = R[3] * rx + R[4] * ry - R[5];
    double ddz = R[6] * rx + R[7] * ry - R[8];
    const double norm = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    ddx /= norm;
    ddy /= norm;
    ddz /= norm;
    const double t_proj = ((xc0 - k.p0) * ddx + (xc1 - k.p1) * ddy + (xc2 - k.p2) * ddz);
    double t_c = t_proj;
    if (t_c < (double)dmin) t_c = (double)dmin;
    else if (t_c > (double)dmax) t_c = (double)dmax;
    double pcx = k.p0 + ddx * t_c;
    double pcy = k.p1 + ddy * t_c;
    double pcz = k.p2 + ddz * t_c;
    if (C.unbounded != 0) {   // _contract_pt (fusion.py:243-254)
        const double nx = (pcx - C.bc0) / C.bh0;
        const double ny = (pcy - C.bc1) / C.bh1;
        const double nz = (pcz - C.bc2) / C.bh2;
        const double r = sqrt(nx * nx + ny * ny + nz * nz);
        if (r > 1.0) {
            const double s = (2.0 - 1.0 / r) / r;
            pcx = C.bc0 + nx * s * C.bh0;
            pcy = C.bc1 + ny * s * C.bh1;
            pcz = C.bc2 + nz * s * C.bh2;
        }
    }
    const double dx = xc0 - pcx;
    const double dy = xc1 - pcy;
    const double dz = xc2 - pcz;
    const double delta = sqrt(dx * dx + dy * dy + dz * dz);
    const float span = dmax - dmin;                                   // f32 site
    const double tau_sp = C.dx * g + C.lam * (double)span;
    double b = C.beta * (double)nsamp;
    if (b > C.bmax) b = C.bmax;
    const double tau_dp = (C.gamma + b) * C.dx;
    const bool ok = (delta <= tau_sp) && (fabs(x_d - (double)dexp) <= tau_dp);
    const float msum = dmin + dmax;                                   // f32 site
    const double mu = 0.5 * (double)msum;
    double hd = 0.5 * (double)span;                                   // f32 site
    if (hd < C.eps) hd = C.eps;
    const double r = fabs(t_c - mu) / hd;
    wd = exp(-C.alpha1 * r * r);
    return ok;
}

// _thin_pair (fusion.py:306-370); returns ok_footprint, writes npix and t
__device__ __forceinline__ bool thin_pair(const FuseConst &C, const Cam &k, double xc0,
                                          double xc1, double xc2, double x_d,
                                          const float *__restrict__ mask,
                                          const float *__restrict__ dexp,
                                          const int32_t *__restrict__ nsamp, long long &npix_out,
                                          double &t_out) {
    const double half = 0.5 * C.dx;
    double umin = 1e30, umax = -1e30, vmin = 1e30, vmax = -1e30;
#pragma unroll 1
    for (int j = 0; j < 8; ++j) {
        const double sx = ((j & 1) == 0) ? -1.0 : 1.0;
        const double sy = ((j & 2) == 0) ? -1.0 : 1.0;
        const double sz = ((j & 4) == 0) ? -1.0 : 1.0;
        double cu, cv, cd;
        if (!project_px(k, xc0 + sx * half, xc1 + sy * half, xc2 + sz * half, cu, cv, cd))
            return false;
        if (cu < umin) umin = cu;
        if (cu > umax) umax = cu;
        if (cv < vmin) vmin = cv;
        if (cv > vmax) vmax = cv;
    }
    const long long wi = (long long)k.w;
    const long long hi = (long long)k.h;
    long long xs = nb_floor_int(umin * k.w);
    long long xe = nb_floor_int(umax * k.w);
    long long ys = nb_floor_int(vmin * k.h);
    long long ye = nb_floor_int(vmax * k.h);
    if (xe < 0 || xs > wi - 1 || ye < 0 || ys > hi - 1) return false;
    if (xs < 0) xs = 0;
    if (ys < 0) ys = 0;
    if (xe > wi - 1) xe = wi - 1;
    if (ye > hi - 1) ye = hi - 1;
    long long support = 0, npix = 0;
    double m_max = 0.0;
    const double tau_base = 2.0 * C.gamma;
    for (long long yy = ys; yy <= ye; ++yy) {
        const int64_t row = yy * (int64_t)C.wm;
        for (long long xx = xs; xx <= xe; ++xx) {
            npix += 1;
            const double mv = (double)__ldg(mask + row + xx);
            if (mv > m_max) m_max = mv;
            if (mv > 0.5) {
                const int32_t ns = __ldg(nsamp + row + xx);
                if (ns > 0) {
                    double b = C.beta * (double)ns;
                    if (b > C.bmax) b = C.bmax;
                    const double tau_d = (tau_base + b) * C.dx;
                    if (fabs(x_d - (double)__ldg(dexp + row + xx)) <= tau_d) support += 1;
                }
            }
        }
    }
    const double p_cov = (double)support / (double)npix;
    npix_out = npix;
    t_out = (p_cov >= C.thin_pct) ? m_max : p_cov;
    return true;
}

// ---------------------------------------------------------------------------
// sparse pass: one gated voxel per thread
// ---------------------------------------------------------------------------
constexpr int kFuseThreads = 128;

template <int MAXV>
__global__ void __launch_bounds__(kFuseThreads)
fuse_sparse(FuseConst C, const double *__restrict__ cams, const float *__restrict__ dens,
            FuseMaps M, FuseOut O, const uint32_t *__restrict__ work,
            const unsigned long long *__restrict__ count) {
    extern __shared__ double s_cam[];
    for (int i = threadIdx.x; i < C.nv * kCamStride; i += blockDim.x) s_cam[i] = cams[i];
    __syncthreads();
    const unsigned long long n = *count;
    const int64_t plane = (int64_t)C.hm * C.wm;
    const int64_t gg = C.g * C.g;
    double tw[MAXV], tmw[MAXV], tt[MAXV];
    for (unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (unsigned long long)gridDim.x * blockDim.x) {
        const int64_t vi = (int64_t)work[t];
        const int64_t ix = vi / gg;
        const int64_t rem = vi - ix * gg;
        const int64_t iy = rem / C.g;
        const int64_t iz = rem - iy * C.g;
        const double rho = (double)__ldg(dens + vi);
        const double xc0 = C.origin0 + ((double)ix + 0.5) * C.dx;
        const double xc1 = C.origin1 + ((double)iy + 0.5) * C.dx;
        const double xc2 = C.origin2 + ((double)iz + 0.5) * C.dx;
        int n_thick = 0, n_thin = 0;
        for (int view = 0; view < C.nv; ++view) {
            const Cam k = load_cam(s_cam, view);
            double u, v, x_d;
            if (!project_px(k, xc0, xc1, xc2, u, v, x_d)) continue;
            if (u < 0.0 || u >= 1.0 || v < 0.0 || v >= 1.0) continue;
            const long long px = pixel_index(u, (long long)k.w);
            const long long py = pixel_index(v, (long long)k.h);
            const int64_t vplane = (int64_t)view * plane;
            const int64_t pix = vplane + py * (int64_t)C.wm + px;
            const int32_t ns = __ldg(M.nsamps + pix);
            if (ns <= 0) continue;                       // valids[view, py, px] == 0
            const float m = __ldg(M.masks + pix);
            bool routed_thick = false;
            if ((double)m >= C.mask_thr && rho >= C.rho_thr) {
                const double g = grad_at(M.dexps + vplane, M.dmins + vplane, M.dmaxs + vplane,
                                         C.hm, C.wm, (int)px, (int)py, C.eps, C.kappa);
                double wd;
                if (thick_pair(C, k, xc0, xc1, xc2, u, v, x_d, __ldg(M.dmins + pix),
                               __ldg(M.dmaxs + pix), __ldg(M.dexps + pix), ns, g, wd)) {
                    // stable sorted insert by (w, m*w): same order as the
                    // reference's insertion sort (fusion.py:389-407)
                    const double km = (double)m * wd;
                    int j = n_thick - 1;
                    while (j >= 0 && (tw[j] > wd || (tw[j] == wd && tmw[j] > km))) {
                        tw[j + 1] = tw[j];
                        tmw[j + 1] = tmw[j];
                        --j;
                    }
                    tw[j + 1] = wd;
                    tmw[j + 1] = km;
                    ++n_thick;
                    routed_thick = true;
                }
            }
            if (!routed_thick && C.enable_thin) {
                const double fmax = k.fx > k.fy ? k.fx : k.fy;
                if ((double)m > C.thin_floor && rho >= C.rho_thin && x_d > 0.0 &&
                    C.dx * fmax / x_d >= 1.0) {
                    long long npix;
                    double t_s;
                    if (thin_pair(C, k, xc0, xc1, xc2, x_d, M.masks + vplane, M.dexps + vplane,
                                  M.nsamps + vplane, npix, t_s) &&
                        npix > 0 && t_s >= C.thin_accept) {
                        int j = n_thin - 1;
                        while (j >= 0 && tt[j] > t_s) { tt[j + 1] = tt[j]; --j; }
                        tt[j + 1] = t_s;
                        ++n_thin;
                    }
                }
            }
        }
        double sw = 0.0, smw = 0.0, st = 0.0;
        for (int i = 0; i < n_thick; ++i) { sw += tw[i]; smw += tmw[i]; }
        for (int i = 0; i < n_thin; ++i) st += tt[i];
        const double denom = sw + (double)n_thin;
        const double p = (denom > C.eps) ? (smw + st) / denom : 0.0;
        O.probs[vi] = p;
        if (O.n_thick) O.n_thick[vi] = n_thick;
        if (O.n_thin) O.n_thin[vi] = n_thin;
        if (O.sw) O.sw[vi] = sw;
        if (O.smw) O.smw[vi] = smw;
        if (O.st) O.st[vi] = st;
        if (O.occ) O.occ[vi] = (p >= C.occ_thr) ? 1 : 0;
    }
}

// ---------------------------------------------------------------------------
// f64 gradient maps (export for parity tests; fuse computes g on the fly)
// ---------------------------------------------------------------------------
__global__ void gradient_maps_kernel(int nv, int hm, int wm, const float *__restrict__ dexps,
                                     const float *__restrict__ dmins,
                                     const float *__restrict__ dmaxs,
                                     const int32_t *__restrict__ nsamps, double eps, double kappa,
                                     double *__restrict__ out) {
    const int64_t plane = (int64_t)hm * wm;
    const int64_t total = plane * nv;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = i / plane;
        const int64_t r = i - v * plane;
        const int iy = (int)(r / wm), ix = (int)(r - (int64_t)iy * wm);
        out[i] = nsamps[i] > 0 ? grad_at(dexps + v * plane, dmins + v * plane, dmaxs + v * plane,
                                         hm, wm, ix, iy, eps, kappa)
                               : 0.0;
    }
}

template <int MAXV>
static int launch_sparse(const FuseConst &C, const double *cams, const float *dens,
                         const FuseMaps &M, const FuseOut &O, const uint32_t *work,
                         const unsigned long long *count, cudaStream_t s) {
    const size_t smem = (size_t)C.nv * kCamStride * sizeof(double);
    static int blocks_per_sm = 0, n_sm = 0;   // device properties only
    if (blocks_per_sm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(fuse_sparse<MAXV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fuse_sparse<MAXV>, kFuseThreads, smem);
        blocks_per_sm = b > 0 ? b : 1;
    }
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fuse_sparse<MAXV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    fuse_sparse<MAXV><<<n_sm * blocks_per_sm, kFuseThreads, smem, s>>>(C, cams, dens, M, O, work,
                                                                        count);
    return check_launch("divas_fuse(sparse)");
}

}  // namespace divas

using namespace divas;

extern "C" size_t divas_fuse_workspace_size(int64_t n_vox, int32_t nv) {
    (void)nv;
    return 256 + (size_t)(n_vox > 0 ? n_vox : 0) * sizeof(uint32_t);
}

extern "C" const int64_t *divas_fuse_gated_count(const void *workspace) {
    return (const int64_t *)workspace;
}

extern "C" int divas_fuse(const divas_fuse_args *a, void *workspace, size_t workspace_bytes,
                          void *stream) {
    if (!a) { set_error("divas_fuse: null args"); return DIVAS_EINVAL; }
    if (a->g < 1) { set_error("divas_fuse: bad grid resolution"); return DIVAS_EINVAL; }
    const int64_t nvox = a->g * a->g * a->g;
    if (a->vox_lo < 0 || a->vox_hi > nvox || a->vox_lo > a->vox_hi) {
        set_error("divas_fuse: voxel range [%lld, %lld) outside [0, %lld)", (long long)a->vox_lo,
                  (long long)a->vox_hi, (long long)nvox);
        return DIVAS_EINVAL;
    }
    if (nvox > 0xffffffffLL) { set_error("divas_fuse: grid too large for 32-bit work list"); return DIVAS_EINVAL; }
    if (a->nv < 1 || a->nv > 1024) { set_error("divas_fuse: view count %d outside [1, 1024]", a->nv); return DIVAS_EINVAL; }
    if (a->hm < 1 || a->wm < 1) { set_error("divas_fuse: empty planes"); return DIVAS_EINVAL; }
    if (!a->density || !a->cams || !a->masks || !a->dmins || !a->dmaxs || !a->dexps ||
        !a->nsamps || !a->probs || !workspace) {
        set_error("divas_fuse: null pointer");
        return DIVAS_EINVAL;
    }
    const int64_t n = a->vox_hi - a->vox_lo;
    if (workspace_bytes < divas_fuse_workspace_size(n, a->nv)) {
        set_error("divas_fuse: workspace too small");
        return DIVAS_EWORKSPACE;
    }
    if (n == 0) return DIVAS_OK;
    cudaStream_t s = (cudaStream_t)stream;
    FuseConst C;
    C.g = a->g; C.lo = a->vox_lo; C.hi = a->vox_hi;
    C.origin0 = a->origin[0]; C.origin1 = a->origin[1]; C.origin2 = a->origin[2];
    C.dx = a->dx_vox;
    C.nv = a->nv; C.hm = a->hm; C.wm = a->wm;
    const double *pv = a->pv;
    C.gamma = pv[0]; C.beta = pv[1]; C.bmax = pv[2]; C.lam = pv[3]; C.rho_thr = pv[4];
    C.rho_thin = pv[5]; C.thin_pct = pv[6]; C.alpha1 = pv[7]; C.thin_accept = pv[8];
    C.eps = pv[9]; C.mask_thr = pv[10]; C.thin_floor = pv[11]; C.kappa = pv[12];
    C.enable_thin = pv[13] != 0.0;
    C.bc0 = a->bc[0]; C.bc1 = a->bc[1]; C.bc2 = a->bc[2];
    C.bh0 = a->bh[0]; C.bh1 = a->bh[1]; C.bh2 = a->bh[2];
    C.unbounded = a->unbounded;
    C.occ_thr = a->occ_thr;
    FuseOut O{a->probs, a->n_thick, a->n_thin, a->sw, a->smw, a->st, a->occ};
    FuseMaps M{a->masks, a->dmins, a->dmaxs, a->dexps, a->nsamps};
    unsigned long long *count = (unsigned long long *)workspace;
    uint32_t *work = (uint32_t *)((char *)workspace + 256);
    if (cudaMemsetAsync(count, 0, sizeof(unsigned long long), s) != cudaSuccess)
        return check_launch("divas_fuse(memset)");
    {
        static int n_sm = 0;
        if (n_sm == 0) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        }
        const int64_t nquads = (n + 3) / 4;
        int64_t blocks = (nquads + kGateThreads - 1) / kGateThreads;
        blocks = std::min<int64_t>(blocks, (int64_t)n_sm * 16);
        fuse_gate<<<(unsigned)std::max<int64_t>(blocks, 1), kGateThreads, 0, s>>>(a->density, C, O,
                                                                                 work, count);
        int rc = check_launch("divas_fuse(gate)");
        if (rc) return rc;
    }
    if (a->nv <= 32) return launch_sparse<32>(C, a->cams, a->density, M, O, work, count, s);
    if (a->nv <= 64) return launch_sparse<64>(C, a->cams, a->density, M, O, work, count, s);
    if (a->nv <= 128) return launch_sparse<128>(C, a->cams, a->density, M, O, work, count, s);
    if (a->nv <= 256) return launch_sparse<256>(C, a->cams, a->density, M, O, work, count, s);
    return launch_sparse<1024>(C, a->cams, a->density, M, O, work, count, s);
}

extern "C" int divas_gradient_maps(int32_t nv, int32_t hm, int32_t wm, const float *dexps,
                                   const float *dmins, const float *dmaxs, const int32_t *nsamps,
                                   double eps, double kappa, double *out, void *stream) {
    if (nv < 1 || hm < 1 || wm < 1) { set_error("divas_gradient_maps: empty"); return DIVAS_EINVAL; }
    if (!dexps || !dmins || !dmaxs || !nsamps || !out) {
        set_error("divas_gradient_maps: null pointer");
        return DIVAS_EINVAL;
    }
    const int64_t total = (int64_t)nv * hm * wm;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 32);
    gradient_maps_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        nv, hm, wm, dexps, dmins, dmaxs, nsamps, eps, kappa, out);
    return check_launch("divas_gradient_maps");
}
