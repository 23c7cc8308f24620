// render.cu -- fixture producers on the device: the volumetric ray marcher
// (render_view / march_ray) and the density bake (bake_density_grid).
//
// Reference: /root/reference/pkg/src/divas/render.py:96-292 (numba) and
// scene.py:69-105, :194-201, geometry.py:140-147, :242-256 (numpy).
// these make the fusion's inputs; at C5 the CPU
// render of the 128 views takes minutes, one launch here.
//
// Arithmetic: the reference's f64 evaluation order, no FMA contraction
// (-fmad=false), except the two sites where numpy goes through BLAS (see
// np_density): there the fused chains OpenBLAS computes are restated with
// explicit fma().  The only operation whose bits could differ from the
// reference could be exp inside the marcher's alpha = 1 - exp(-sigma * dt):
// it is glibc's exp restated bit for bit (exp_glibc, exp_cr.cuh), so alpha is
// the reference's.  The marcher still carries the machinery of an absolute
// bound on how far each running quantity can be from the reference's (an
// earlier correctly-rounded exp could differ in the last bit near rounding
// midpoints) and flags a pixel `unsure` when a decision lies within that
// bound; with the exact exp every bound is 0 and no pixel is flagged.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "exp_cr.cuh"

namespace divas {

constexpr int kMaxPrims = DIVAS_MAX_PRIMS;
constexpr double kU = 1.1102230246251565e-16;     // 2^-53

// rounding slack of one IEEE op whose inputs may differ by E_in between the
// reference and here: none when they are identical
__device__ __forceinline__ double rs(double Ein, double res) {
    return Ein > 0.0 ? 2.0 * kU * fabs(res) : 0.0;
}

struct SceneConst {
    int n;
    uint8_t kind[kMaxPrims];
    double par[kMaxPrims][7];
    double dens[kMaxPrims], soft[kMaxPrims];
    double col[kMaxPrims][3];
    double bg[3];
    // per primitive: an axis-aligned box outside which its density is
    // exactly 0 (inflated by the soft edge and a rounding margin); empty
    // (lo > hi) for a zero-density primitive
    double lo[kMaxPrims][3], hi[kMaxPrims][3];
};

struct MarchConst {
    int n_steps;
    double near_, far_, tau_cw, min_w;
};

// _prim_density (render.py:96-157): max density over primitives, first wins
// ties; returns the argmax index in *bi (-1 when empty space)
//
// Only primitives whose step range [k0, k1] holds step k are evaluated: the
// others are outside their zero-density box at this sample, so their d is
// exactly 0 and `d > best` (best >= 0) never selects them -- the result is
// the full loop's.
__device__ __forceinline__ double prim_density(const SceneConst &S, double px, double py,
                                               double pz, int &bi, const int *k0,
                                               const int *k1, int k) {
    double best = 0.0;
    bi = -1;
    for (int i = 0; i < S.n; ++i) {
        if (k < k0[i] || k > k1[i]) continue;
        const double *P = S.par[i];
        double sd;
        const int kind = S.kind[i];
        if (kind == 0) {
            const double dx = px - P[0], dy = py - P[1], dz = pz - P[2];
            const double dist = sqrt(dx * dx + dy * dy + dz * dz);
            sd = dist - P[3];
            if (P[4] > 0.0) {
                const double sd2 = P[4] - dist;
                if (sd2 > sd) sd = sd2;
            }
        } else if (kind == 1) {
            const double qx = fabs(px - P[0]) - P[3];
            const double qy = fabs(py - P[1]) - P[4];
            const double qz = fabs(pz - P[2]) - P[5];
            const double ox = qx > 0.0 ? qx : 0.0, oy = qy > 0.0 ? qy : 0.0,
                         oz = qz > 0.0 ? qz : 0.0;
            const double outside = sqrt(ox * ox + oy * oy + oz * oz);
            double mx = qx > qy ? qx : qy;
            if (qz > mx) mx = qz;
            sd = outside + (mx < 0.0 ? mx : 0.0);
        } else {
            const double ax = P[0], ay = P[1], az = P[2];
            const double abx = P[3] - ax, aby = P[4] - ay, abz = P[5] - az;
            const double denom = abx * abx + aby * aby + abz * abz;
            double t = 0.0;
            if (denom > 0.0) {
                t = ((px - ax) * abx + (py - ay) * aby + (pz - az) * abz) / denom;
                if (t < 0.0) t = 0.0;
                else if (t > 1.0) t = 1.0;
            }
            const double dx = px - (ax + t * abx), dy = py - (ay + t * aby),
                         dz = pz - (az + t * abz);
            sd = sqrt(dx * dx + dy * dy + dz * dz) - P[6];
        }
        double fall;
        if (S.soft[i] > 0.0) {
            fall = 1.0 - sd / S.soft[i];
            if (fall < 0.0) fall = 0.0;
            else if (fall > 1.0) fall = 1.0;
        } else {
            fall = sd <= 0.0 ? 1.0 : 0.0;
        }
        const double d = S.dens[i] * fall;
        if (d > best) {
            best = d;
            bi = i;
        }
    }
    return best;
}

struct MarchOut {
    double c[3], dmin, dmax, dexp, zpk;
    double Ec[3], Edexp;       // bounds of |ours - reference| for the float results
    int count;
    bool valid, unsure;
};

// _march (render.py:160-218) with the error bookkeeping described above.
// |e - e_ref| <= 4u e (two libraries within 1 ulp each); every other op is the
// same IEEE op on inputs within the tracked bounds, so its result moves by at
// most (input bound propagated) + 2u |result| (one rounding on each side).
__device__ __forceinline__ void march(const SceneConst &S, const MarchConst &R, double ox,
                                      double oy, double oz, double dx, double dy, double dz,
                                      MarchOut &o) {
    const double dt = (R.far_ - R.near_) / (double)R.n_steps;
    double T = 1.0, cum = 0.0, d_min = 0.0, d_max = 0.0, last_hit = 0.0;
    double w_peak = 0.0, z_peak = 0.0, wsum = 0.0, wt = 0.0;
    double cr = 0.0, cg = 0.0, cb = 0.0;
    double ET = 0.0, Ecum = 0.0, Ewsum = 0.0, Ewt = 0.0, Ewpk = 0.0;
    double Er = 0.0, Eg = 0.0, Eb = 0.0;
    // unsure_peak: the argmax sample (z_surface) is uncertain; it only
    // matters when the ray ends valid (invalid rays report z = 0)
    bool have_min = false, stopped = false, unsure = false, unsure_peak = false;
    int count = 0;
    // Steps at which a primitive can be nonzero: the ray's parameter interval
    // through the primitive's zero-density box, widened by one step each way
    // (the box already carries a margin far above the rounding of o + d t).
    int k0[kMaxPrims], k1[kMaxPrims];
    const double o3[3] = {ox, oy, oz}, d3[3] = {dx, dy, dz};
    for (int i = 0; i < S.n; ++i) {
        double t0 = -1e300, t1 = 1e300;
        for (int j = 0; j < 3; ++j) {
            const double lo = S.lo[i][j], hi = S.hi[i][j];
            if (d3[j] == 0.0) {
                if (o3[j] < lo || o3[j] > hi) { t0 = 1e300; t1 = -1e300; }
            } else {
                double ta = (lo - o3[j]) / d3[j], tb = (hi - o3[j]) / d3[j];
                if (ta > tb) { const double x = ta; ta = tb; tb = x; }
                t0 = fmax(t0, ta);
                t1 = fmin(t1, tb);
            }
        }
        int a = 1 << 30, b = -1;
        if (t0 <= t1) {
            const double fa = floor((t0 - R.near_) / dt - 0.5) - 1.0;
            const double fb = ceil((t1 - R.near_) / dt - 0.5) + 1.0;
            if (fb >= 0.0 && fa <= (double)(R.n_steps - 1)) {
                a = fa < 0.0 ? 0 : (int)fa;
                b = fb > (double)(R.n_steps - 1) ? R.n_steps - 1 : (int)fb;
            }
        }
        k0[i] = a;
        k1[i] = b;
    }
    for (int k = 0; k < R.n_steps; ++k) {
        // A step where no primitive can be nonzero has sigma = 0, so w = 0 and
        // T, cum and every sum are unchanged: it repeats the previous step's
        // decisions and is skipped (step 0 always runs: with a negative
        // min_weight it sets d_min even at zero weight).
        if (k > 0) {
            bool act = false;
            int next = R.n_steps;
            for (int i = 0; i < S.n; ++i) {
                act |= (k >= k0[i] && k <= k1[i]);
                if (k0[i] > k && k0[i] < next) next = k0[i];
            }
            if (!act) {
                k = next - 1;
                continue;
            }
        }
        const double t = R.near_ + ((double)k + 0.5) * dt;
        int pi;
        const double sigma = prim_density(S, ox + dx * t, oy + dy * t, oz + dz * t, pi, k0, k1, k);
        double a = 0.0, Ea = 0.0;
        if (sigma > 0.0) {
            const double x = -sigma * dt;
            if (x < -38.0) {
                a = 1.0;          // exp(x) < 2^-54: 1 - exp(x) rounds to 1 for any exp
            } else {
                a = 1.0 - exp_glibc(x);   // the C library's exp, bit for bit: Ea = 0
            }
            if (ET + Ea > 0.0 && T < 1e-280) unsure = true;   // subnormal: no rel. bound
        }
        if (!(sigma > 0.0)) {      // w = 0: nothing moves (decisions as before)
            if (!have_min && cum > R.min_w) {
                if (Ecum > 0.0 && fabs(cum - R.min_w) <= Ecum) unsure = true;
                have_min = true;
                d_min = t;
            }
            if (cum >= R.tau_cw) {
                d_max = t;
                stopped = true;
                break;
            }
            continue;
        }
        const double w = T * a;
        const double Ew = ET * a + T * Ea + rs(ET + Ea, w);
        if (w > 0.0) {
            count += 1;
            last_hit = t;
            wsum += w;
            Ewsum += Ew + rs(Ewsum + Ew, wsum);
            const double wtt = w * t;
            const double Ewtt = Ew * t + rs(Ew, wtt);
            wt += wtt;
            Ewt += Ewtt + rs(Ewt + Ewtt, wt);
            if (Ew + Ewpk > 0.0 && fabs(w - w_peak) <= Ew + Ewpk) unsure_peak = true;
            if (w > w_peak) {
                w_peak = w;
                Ewpk = Ew;
                z_peak = t;
            }
            const double *col = S.col[pi];
            const double c0 = w * col[0], c1 = w * col[1], c2 = w * col[2];
            const double E0 = Ew * fabs(col[0]) + rs(Ew, c0), E1 = Ew * fabs(col[1]) + rs(Ew, c1),
                         E2 = Ew * fabs(col[2]) + rs(Ew, c2);
            cr += c0;
            cg += c1;
            cb += c2;
            Er += E0 + rs(Er + E0, cr);
            Eg += E1 + rs(Eg + E1, cg);
            Eb += E2 + rs(Eb + E2, cb);
        }
        cum += w;
        Ecum += Ew + rs(Ecum + Ew, cum);
        const double om = 1.0 - a;
        const double Eom = Ea + rs(Ea, om);
        const double Tn = T * om;
        ET = ET * om + T * Eom + rs(ET + Eom, Tn);
        T = Tn;
        if (!have_min) {
            if (Ecum > 0.0 && fabs(cum - R.min_w) <= Ecum) unsure = true;
            if (cum > R.min_w) {
                have_min = true;
                d_min = t;
            }
        }
        if (Ecum > 0.0 && fabs(cum - R.tau_cw) <= Ecum) unsure = true;
        if (cum >= R.tau_cw) {
            d_max = t;
            stopped = true;
            break;
        }
    }
    if (!stopped) d_max = last_hit;
    const double rem = 1.0 - cum;
    const double b0 = rem * S.bg[0], b1 = rem * S.bg[1], b2 = rem * S.bg[2];
    cr += b0;
    cg += b1;
    cb += b2;
    const double Erem = Ecum + rs(Ecum, rem);
    const double Eb0 = Erem * fabs(S.bg[0]) + rs(Erem, b0),
                 Eb1 = Erem * fabs(S.bg[1]) + rs(Erem, b1),
                 Eb2 = Erem * fabs(S.bg[2]) + rs(Erem, b2);
    o.Ec[0] = Er + Eb0 + rs(Er + Eb0, cr);
    o.Ec[1] = Eg + Eb1 + rs(Eg + Eb1, cg);
    o.Ec[2] = Eb + Eb2 + rs(Eb + Eb2, cb);
    o.c[0] = cr;
    o.c[1] = cg;
    o.c[2] = cb;
    o.valid = have_min;
    o.count = count;
    o.Edexp = 0.0;
    if (!have_min) {
        o.dmin = o.dmax = o.dexp = o.zpk = 0.0;
        o.count = 0;
    } else {
        double de = wt / wsum;
        double Ede = 0.0;
        if (Ewt + Ewsum > 0.0) {
            if (wsum > 2.0 * Ewsum) Ede = 2.0 * (Ewt + fabs(de) * Ewsum) / wsum + 2.0 * kU * fabs(de);
            else unsure = true;
        }
        // the clamp is 1-Lipschitz: the clamped value keeps the bound Ede
        if (de < d_min) de = d_min;
        else if (de > d_max) de = d_max;
        unsure |= unsure_peak;
        o.dmin = d_min;
        o.dmax = d_max;
        o.dexp = de;
        o.Edexp = Ede;
        o.zpk = z_peak;
    }
    o.unsure = unsure;
}

// true when v and every value within E of it round to the same f32
__device__ __forceinline__ bool f32_stable(double v, double E) {
    return E == 0.0 || __double2float_rn(v - E) == __double2float_rn(v + E);
}

// _render (render.py:221-254): one thread per pixel of view blockIdx.y, the
// ray through the pixel centre; outputs [view][h][w] (rgb [view][h][w][3])
__global__ void __launch_bounds__(128)
render_kernel(SceneConst S, MarchConst R, const double *__restrict__ cams, int h, int w,
              float *__restrict__ rgb, float *__restrict__ dmin, float *__restrict__ dmax,
              float *__restrict__ dexp, int32_t *__restrict__ nsamp,
              float *__restrict__ zsurf, uint8_t *__restrict__ unsure) {
    const int64_t npix = (int64_t)h * w;
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npix) return;
    const int view = blockIdx.y;
    const double *c = cams + (int64_t)view * kCamStride;
    const int iy = (int)(p / w), ix = (int)(p - (int64_t)iy * w);
    const double fx = __ldg(c + 12), fy = __ldg(c + 13), cx = __ldg(c + 14), cy = __ldg(c + 15);
    const double xc = ((double)ix + 0.5 - cx) / fx;
    const double yc = (cy - ((double)iy + 0.5)) / fy;
    double dxw = __ldg(c + 0) * xc + __ldg(c + 1) * yc - __ldg(c + 2);
    double dyw = __ldg(c + 3) * xc + __ldg(c + 4) * yc - __ldg(c + 5);
    double dzw = __ldg(c + 6) * xc + __ldg(c + 7) * yc - __ldg(c + 8);
    const double norm = sqrt(dxw * dxw + dyw * dyw + dzw * dzw);
    dxw /= norm;
    dyw /= norm;
    dzw /= norm;
    MarchOut o;
    march(S, R, __ldg(c + 9), __ldg(c + 10), __ldg(c + 11), dxw, dyw, dzw, o);
    const int64_t q = (int64_t)view * npix + p;
    bool u = o.unsure;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        rgb[3 * q + j] = __double2float_rn(o.c[j]);
        u |= !f32_stable(o.c[j], o.Ec[j]);
    }
    u |= !f32_stable(o.dexp, o.Edexp);
    dmin[q] = __double2float_rn(o.dmin);
    dmax[q] = __double2float_rn(o.dmax);
    dexp[q] = __double2float_rn(o.dexp);
    nsamp[q] = o.count;
    zsurf[q] = __double2float_rn(o.zpk);
    if (unsure) unsure[q] = u ? 1 : 0;
}

// march_ray (render.py:257-267) on explicit unit rays [n][6]: out [n][8] f64
// (r, g, b, d_min, d_max, d_exp, n_samples, z_surface), err [n][4] the bounds
// on r, g, b, d_exp (d_min, d_max, z and n are exact unless unsure)
__global__ void __launch_bounds__(128)
march_kernel(SceneConst S, MarchConst R, int64_t n, const double *__restrict__ rays,
             double *__restrict__ out, double *__restrict__ err, uint8_t *__restrict__ unsure) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double *r = rays + 6 * i;
    MarchOut o;
    march(S, R, r[0], r[1], r[2], r[3], r[4], r[5], o);
    double *d = out + 8 * i;
    d[0] = o.c[0]; d[1] = o.c[1]; d[2] = o.c[2];
    d[3] = o.dmin; d[4] = o.dmax; d[5] = o.dexp; d[6] = (double)o.count; d[7] = o.zpk;
    if (err) {
        err[4 * i + 0] = o.Ec[0]; err[4 * i + 1] = o.Ec[1]; err[4 * i + 2] = o.Ec[2];
        err[4 * i + 3] = o.Edexp;
    }
    if (unsure) unsure[i] = o.unsure ? 1 : 0;
}

// ScenePrimitive.density_at (scene.py:69-105) as NUMPY evaluates it: the
// last-axis norm sums squares left to right; `ab @ ab` (1-D, BLAS ddot) and
// `points @ ab` (BLAS dgemv) are the fused chains OpenBLAS computes on the
// machine that produced the golden vectors (oracle/divas_oracle_render.c)
__device__ __forceinline__ double np_density(const SceneConst &S, int i, double px, double py,
                                             double pz) {
    const double *P = S.par[i];
    double sd;
    const int kind = S.kind[i];
    if (kind == 0) {
        const double dx = px - P[0], dy = py - P[1], dz = pz - P[2];
        const double dist = sqrt(dx * dx + dy * dy + dz * dz);
        sd = dist - P[3];
        if (P[4] > 0.0) {
            const double s2 = P[4] - dist;
            sd = s2 > sd ? s2 : sd;
        }
    } else if (kind == 1) {
        const double qx = fabs(px - P[0]) - P[3];
        const double qy = fabs(py - P[1]) - P[4];
        const double qz = fabs(pz - P[2]) - P[5];
        const double ox = qx > 0.0 ? qx : 0.0, oy = qy > 0.0 ? qy : 0.0, oz = qz > 0.0 ? qz : 0.0;
        const double outside = sqrt(ox * ox + oy * oy + oz * oz);
        double mx = qx;
        if (qy > mx) mx = qy;
        if (qz > mx) mx = qz;
        sd = outside + (mx < 0.0 ? mx : 0.0);
    } else {
        const double abx = P[3] - P[0], aby = P[4] - P[1], abz = P[5] - P[2];
        const double denom = fma(abz, abz, fma(aby, aby, abx * abx));
        double t = 0.0;
        if (denom > 0.0) {
            const double rx = px - P[0], ry = py - P[1], rz = pz - P[2];
            t = fma(rz, abz, fma(rx, abx, ry * aby)) / denom;
            t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
        }
        const double dx = px - (P[0] + t * abx), dy = py - (P[1] + t * aby),
                     dz = pz - (P[2] + t * abz);
        sd = sqrt(dx * dx + dy * dy + dz * dz) - P[6];
    }
    double fall;
    if (S.soft[i] > 0.0) {
        fall = 1.0 - sd / S.soft[i];
        fall = fall < 0.0 ? 0.0 : (fall > 1.0 ? 1.0 : fall);
    } else {
        fall = sd <= 0.0 ? 1.0 : 0.0;
    }
    return S.dens[i] * fall;
}

struct BakeConst {
    int64_t g;
    int gshift;
    double o[3], dx, bc[3], bh[3];
    int unbounded;
};

// bake_density_grid (scene.py:194-201): voxel centres (geometry.py:140-147),
// contracted when unbounded (geometry.py:242-256), max density over
// primitives, rounded to f32.  One thread per voxel, [ix, iy, iz] C order.
__global__ void __launch_bounds__(256)
bake_kernel(SceneConst S, BakeConst B, float *__restrict__ out) {
    const int64_t n = B.g * B.g * B.g;
    for (int64_t vi = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; vi < n;
         vi += (int64_t)gridDim.x * blockDim.x) {
        int64_t ix, iy, iz;
        if (B.gshift >= 0) {
            const int64_t m = B.g - 1;
            ix = vi >> (2 * B.gshift);
            iy = (vi >> B.gshift) & m;
            iz = vi & m;
        } else {
            ix = vi / (B.g * B.g);
            iy = (vi / B.g) % B.g;
            iz = vi % B.g;
        }
        double p[3] = {B.o[0] + ((double)ix + 0.5) * B.dx, B.o[1] + ((double)iy + 0.5) * B.dx,
                       B.o[2] + ((double)iz + 0.5) * B.dx};
        if (B.unbounded) {
            double q[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) q[k] = (p[k] - B.bc[k]) / B.bh[k];
            const double r = sqrt(fma(q[2], q[2], fma(q[1], q[1], q[0] * q[0])));
            if (!(r <= 1.0)) {
                const double s = 2.0 - 1.0 / r;
#pragma unroll
                for (int k = 0; k < 3; ++k) p[k] = B.bc[k] + (s * (q[k] / r)) * B.bh[k];
            }
        }
        // outside a primitive's zero-density box its d is exactly 0, which
        // never raises np.maximum's running max (>= 0): skip it
        double best = 0.0;
        for (int i = 0; i < S.n; ++i) {
            if (p[0] < S.lo[i][0] || p[0] > S.hi[i][0] || p[1] < S.lo[i][1] ||
                p[1] > S.hi[i][1] || p[2] < S.lo[i][2] || p[2] > S.hi[i][2])
                continue;
            const double d = np_density(S, i, p[0], p[1], p[2]);
            if (d > best) best = d;
        }
        out[vi] = __double2float_rn(best);
    }
}

static int make_scene(const divas_scene *sc, SceneConst &S, const char *who) {
    if (!sc) { set_error("%s: null scene", who); return DIVAS_EINVAL; }
    if (sc->n_prims < 0 || sc->n_prims > kMaxPrims) {
        set_error("%s: %d primitives (supported: 0..%d)", who, sc->n_prims, kMaxPrims);
        return DIVAS_EINVAL;
    }
    if (sc->n_prims > 0 && (!sc->kinds || !sc->params || !sc->density || !sc->colors ||
                            !sc->soft)) {
        set_error("%s: null scene array", who);
        return DIVAS_EINVAL;
    }
    S.n = sc->n_prims;
    for (int i = 0; i < S.n; ++i) {
        if (sc->kinds[i] > 2) {
            set_error("%s: primitive %d has unknown kind %d", who, i, (int)sc->kinds[i]);
            return DIVAS_EINVAL;
        }
        S.kind[i] = sc->kinds[i];
        for (int j = 0; j < 7; ++j) S.par[i][j] = sc->params[7 * i + j];
        S.dens[i] = sc->density[i];
        S.soft[i] = sc->soft[i];
        for (int j = 0; j < 3; ++j) S.col[i][j] = sc->colors[3 * i + j];
        // zero-density box: outside it every computed sd exceeds the soft
        // edge (sphere: |p - c| >= |p_j - c_j|; box: sd >= q_j; capsule: the
        // segment lies in its endpoints' box), so fall, hence d, is 0
        const double *P = S.par[i];
        const double sw = S.soft[i];
        double lo[3], hi[3];
        for (int j = 0; j < 3; ++j) {
            if (S.kind[i] == 0) { lo[j] = P[j] - (P[3] + sw); hi[j] = P[j] + (P[3] + sw); }
            else if (S.kind[i] == 1) { lo[j] = P[j] - (P[3 + j] + sw); hi[j] = P[j] + (P[3 + j] + sw); }
            else {
                lo[j] = std::min(P[j], P[3 + j]) - (P[6] + sw);
                hi[j] = std::max(P[j], P[3 + j]) + (P[6] + sw);
            }
            const double m = 1e-9 * (1.0 + fabs(lo[j]) + fabs(hi[j]));
            lo[j] -= m;
            hi[j] += m;
        }
        const bool finite = std::isfinite(lo[0]) && std::isfinite(lo[1]) && std::isfinite(lo[2]) &&
                            std::isfinite(hi[0]) && std::isfinite(hi[1]) && std::isfinite(hi[2]);
        for (int j = 0; j < 3; ++j) {
            if (!(S.dens[i] > 0.0)) { S.lo[i][j] = 1.0; S.hi[i][j] = -1.0; }   // never nonzero
            else if (!finite) { S.lo[i][j] = -1e300; S.hi[i][j] = 1e300; }   // always evaluate
            else { S.lo[i][j] = lo[j]; S.hi[i][j] = hi[j]; }
        }
    }
    for (int j = 0; j < 3; ++j) S.bg[j] = sc->background[j];
    return DIVAS_OK;
}

static int make_march(const divas_render_cfg *cfg, MarchConst &R, const char *who) {
    if (!cfg) { set_error("%s: null config", who); return DIVAS_EINVAL; }
    if (cfg->samples_per_ray < 1 || !(cfg->near_ < cfg->far_) ||
        !(cfg->tau_cw > 0.0 && cfg->tau_cw <= 1.0)) {
        set_error("%s: invalid render config", who);   // RenderConfig.__post_init__
        return DIVAS_EINVAL;
    }
    R.n_steps = cfg->samples_per_ray;
    R.near_ = cfg->near_;
    R.far_ = cfg->far_;
    R.tau_cw = cfg->tau_cw;
    R.min_w = cfg->min_weight;
    return DIVAS_OK;
}

}  // namespace divas

using namespace divas;

extern "C" int divas_render(const divas_scene *scene, const divas_render_cfg *cfg, int32_t nv,
                            const double *cams, int32_t h, int32_t w, float *rgb, float *d_min,
                            float *d_max, float *d_exp, int32_t *n_samples, float *z_surface,
                            uint8_t *unsure, void *stream) {
    SceneConst S;
    MarchConst R;
    int rc = make_scene(scene, S, "divas_render");
    if (rc) return rc;
    if ((rc = make_march(cfg, R, "divas_render"))) return rc;
    if (nv < 0 || h < 1 || w < 1) { set_error("divas_render: bad sizes"); return DIVAS_EINVAL; }
    if (nv == 0) return DIVAS_OK;
    if (!cams || !rgb || !d_min || !d_max || !d_exp || !n_samples || !z_surface) {
        set_error("divas_render: null pointer");
        return DIVAS_EINVAL;
    }
    const int64_t npix = (int64_t)h * w;
    if (nv > 65535) { set_error("divas_render: too many views per call"); return DIVAS_EINVAL; }
    const dim3 grid((unsigned)((npix + 127) / 128), (unsigned)nv);
    render_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(S, R, cams, h, w, rgb, d_min, d_max,
                                                          d_exp, n_samples, z_surface, unsure);
    return check_launch("divas_render");
}

extern "C" int divas_march_rays(const divas_scene *scene, const divas_render_cfg *cfg, int64_t n,
                                const double *rays, double *out, double *err, uint8_t *unsure,
                                void *stream) {
    SceneConst S;
    MarchConst R;
    int rc = make_scene(scene, S, "divas_march_rays");
    if (rc) return rc;
    if ((rc = make_march(cfg, R, "divas_march_rays"))) return rc;
    if (n < 0) { set_error("divas_march_rays: negative count"); return DIVAS_EINVAL; }
    if (n == 0) return DIVAS_OK;
    if (!rays || !out) { set_error("divas_march_rays: null pointer"); return DIVAS_EINVAL; }
    march_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(S, R, n, rays,
                                                                               out, err, unsure);
    return check_launch("divas_march_rays");
}

extern "C" int divas_bake_density(const divas_scene *scene, int64_t g, const double origin[3],
                                  double dx_vox, int32_t unbounded, const double bc[3],
                                  const double bh[3], float *out, void *stream) {
    SceneConst S;
    int rc = make_scene(scene, S, "divas_bake_density");
    if (rc) return rc;
    if (g < 1 || !origin || !out || (unbounded && (!bc || !bh))) {
        set_error("divas_bake_density: bad arguments");
        return DIVAS_EINVAL;
    }
    BakeConst B;
    B.g = g;
    B.gshift = -1;
    for (int s = 0; s < 31; ++s)
        if ((int64_t)1 << s == g) B.gshift = s;
    B.dx = dx_vox;
    B.unbounded = unbounded ? 1 : 0;
    for (int k = 0; k < 3; ++k) {
        B.o[k] = origin[k];
        B.bc[k] = unbounded ? bc[k] : 0.0;
        B.bh[k] = unbounded ? bh[k] : 1.0;
    }
    const int64_t n = g * g * g;
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, 148 * 32);
    bake_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(S, B, out);
    return check_launch("divas_bake_density");
}
