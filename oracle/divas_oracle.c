/*
 * divas_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's hot path, used as the checker for
 * the CUDA implementation (tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg only).  Nothing in the product package
 * paper_2601_04860_b200/ links, loads or calls this file.
 *
 * Reference algorithm (all paths relative to /root/reference/pkg/src/divas/):
 *   refine_mask          segmenter.py:129-152
 *   _grad_at / _gradient_map / _gradient_maps
 *                        fusion.py:195-240, :684-689  (padded (Hmax,Wmax) semantics)
 *   _project_px          fusion.py:170-184
 *   _pixel_index         fusion.py:187-192
 *   _contract_pt         fusion.py:243-254
 *   _thick_pair          fusion.py:257-303
 *   _thin_pair           fusion.py:306-370
 *   _sorted_sum(_pairs)  fusion.py:373-407
 *   _voxel_views         fusion.py:410-490
 *   _fuse_kernel         fusion.py:493-509
 *
 * Arithmetic contract: IEEE binary64 evaluated left to
 * right as the numba source parenthesises it, NO FMA contraction (build with
 * -ffp-contract=off), and binary32 arithmetic exactly at the eight sites where
 * numba types `f32 - f32` / `f32 + f32` as float32.  Threshold compares widen
 * the f32 operand to f64.  `int(floor(x))` follows numba on x86-64
 * (cvttsd2si: out-of-range or NaN -> INT64_MIN).
 *
 * The oracle is pinned against golden vectors produced by the reference
 * itself (tests/golden/make_golden.py writes the tests/golden npz fixtures).
 *
 * Extra outputs beyond the reference (for the parity gates): per-voxel integer
 * votes n_thick / n_thin and the sorted sums sw, smw, st.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <stdatomic.h>
#include <unistd.h>

#define ORACLE_API __attribute__((visibility("default")))

/* numba int(math.floor(x)) on x86-64 -> cvttsd2si semantics */
static inline int64_t nb_floor_int(double x)
{
    double f = floor(x);
    if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0))
        return INT64_MIN;
    return (int64_t)f;
}

/* ------------------------------------------------------------------------- */
/* refine_mask  (segmenter.py:141-152)                                        */
/* ------------------------------------------------------------------------- */
ORACLE_API int oracle_refine(int64_t h, int64_t w, const float *mask,
                             const float *z, const int32_t *nsamp, float *out)
{
    int64_t n = h * w;
    int any = 0;
    double lo = 0.0, hi = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (nsamp[i] > 0) {
            double zi = (double)z[i];
            if (!any) { lo = zi; hi = zi; any = 1; }
            else {
                if (zi < lo) lo = zi;
                if (zi > hi) hi = zi;
            }
        }
    }
    double span = hi - lo;
    for (int64_t i = 0; i < n; ++i) {
        double o = 0.0;
        if (any && nsamp[i] > 0) {
            double zh = (span > 0) ? ((double)z[i] - lo) / span : 0.0;
            o = (double)mask[i] * (1.0 - zh);
        }
        /* np.clip(out, 0, 1) then astype(float32) */
        if (o < 0.0) o = 0.0;
        if (o > 1.0) o = 1.0;
        out[i] = (float)o;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* depth-gradient factor (fusion.py:195-240) on a (h, w) map                   */
/* ------------------------------------------------------------------------- */
static double grad_at(const float *dexp, const float *dmin, const float *dmax,
                      int64_t h, int64_t w, int64_t ix, int64_t iy,
                      double eps, double kappa)
{
    float center = dexp[iy * w + ix];
    float r32 = dmax[iy * w + ix] - dmin[iy * w + ix];      /* f32 site */
    double rng = (double)r32 + eps;
    double gmax = 0.0, s;
    if (ix > 0) {
        s = (double)fabsf(dexp[iy * w + ix - 1] - center) / rng;  /* f32 site */
        if (s > gmax) gmax = s;
    }
    if (ix < w - 1) {
        s = (double)fabsf(dexp[iy * w + ix + 1] - center) / rng;
        if (s > gmax) gmax = s;
    }
    if (iy > 0) {
        s = (double)fabsf(dexp[(iy - 1) * w + ix] - center) / rng;
        if (s > gmax) gmax = s;
    }
    if (iy < h - 1) {
        s = (double)fabsf(dexp[(iy + 1) * w + ix] - center) / rng;
        if (s > gmax) gmax = s;
    }
    double g = 1.0 / (1.0 + kappa * gmax);
    double hi = 1.0 - eps;
    if (g > hi) g = hi;
    if (g < 0.0) g = 0.0;
    return g;
}

ORACLE_API int oracle_gradient_maps(int64_t nv, int64_t h, int64_t w,
                                    const float *dexps, const float *dmins,
                                    const float *dmaxs, const uint8_t *valids,
                                    double eps, double kappa, double *out)
{
    for (int64_t v = 0; v < nv; ++v) {
        const int64_t off = v * h * w;
        for (int64_t iy = 0; iy < h; ++iy)
            for (int64_t ix = 0; ix < w; ++ix)
                out[off + iy * w + ix] = valids[off + iy * w + ix]
                    ? grad_at(dexps + off, dmins + off, dmaxs + off, h, w, ix, iy, eps, kappa)
                    : 0.0;
    }
    return 0;
}

/* ------------------------------------------------------------------------- */
/* fusion                                                                     */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t g;                 /* grid resolution G */
    const double *origin;      /* [3] min corner */
    double dx_vox;             /* voxel size */
    const float *density;      /* [G^3] rho, [ix,iy,iz] C-order */
    int64_t nv, hm, wm;        /* views, padded height / width */
    const double *rots;        /* [nv,3,3] world_from_camera rotation */
    const double *poss;        /* [nv,3] */
    const double *intr;        /* [nv,6] fx fy cx cy w h */
    const float *masks, *dmins, *dmaxs, *dexps;   /* [nv,hm,wm] */
    const int32_t *nsamps;     /* [nv,hm,wm] */
    const uint8_t *valids;     /* [nv,hm,wm] */
    const double *gmaps;       /* [nv,hm,wm] precomputed g */
    const double *pv;          /* [14] FusionParams.as_vector() */
    const double *bc, *bh;     /* [3] bounds centre / half */
    int64_t unbounded;
    int64_t vox_lo, vox_hi;    /* flat voxel range to evaluate */
    int64_t early_out;         /* 1: skip voxels below both density gates (exact) */
    int64_t nthreads;          /* 0: one worker per online CPU */
    double *out;               /* [G^3] p */
    int32_t *n_thick, *n_thin; /* [G^3] or NULL */
    double *sw, *smw, *st;     /* [G^3] or NULL */
} oracle_fuse_args;

typedef struct { double u, v, d; int in_front; } proj_t;

static inline proj_t project_px(const double *rot, const double *pos,
                                double fx, double fy, double cx, double cy,
                                double w, double h, double px, double py, double pz)
{
    proj_t r;
    double relx = px - pos[0];
    double rely = py - pos[1];
    double relz = pz - pos[2];
    double zc = rot[0 * 3 + 2] * relx + rot[1 * 3 + 2] * rely + rot[2 * 3 + 2] * relz;
    double d = -zc;
    r.d = d;
    if (d <= 0.0) { r.u = -1.0; r.v = -1.0; r.in_front = 0; return r; }
    double xc = rot[0 * 3 + 0] * relx + rot[1 * 3 + 0] * rely + rot[2 * 3 + 0] * relz;
    double yc = rot[0 * 3 + 1] * relx + rot[1 * 3 + 1] * rely + rot[2 * 3 + 1] * relz;
    r.u = (fx * (xc / d) + cx) / w;
    r.v = (cy - fy * (yc / d)) / h;
    r.in_front = 1;
    return r;
}

static inline int64_t pixel_index(double u, int64_t n)
{
    int64_t i = nb_floor_int(u * (double)n);
    if (i > n - 1) i = n - 1;
    return i;
}

/* _thick_pair: returns ok; writes the depth weight */
static int thick_pair(double xc0, double xc1, double xc2, const double *rot,
                      const double *pos, double fx, double fy, double cx, double cy,
                      double w, double h, double u, double v, double x_d,
                      float dmin, float dmax, float dexp, int32_t nsamp, double g,
                      double dx_vox, double gamma, double beta, double bmax,
                      double lam, double alpha1, double eps, const double *bc,
                      const double *bh, int64_t unbounded, double *wd_out)
{
    double rx = (u * w - cx) / fx;
    double ry = (cy - v * h) / fy;
    double ddx = rot[0] * rx + rot[1] * ry - rot[2];
    double ddy = rot[3] * rx + rot[4] * ry - rot[5];
    double ddz = rot[6] * rx + rot[7] * ry - rot[8];
    double norm = sqrt(ddx * ddx + ddy * ddy + ddz * ddz);
    ddx /= norm;
    ddy /= norm;
    ddz /= norm;
    double t_proj = ((xc0 - pos[0]) * ddx + (xc1 - pos[1]) * ddy + (xc2 - pos[2]) * ddz);
    double t_c = t_proj;
    if (t_c < (double)dmin) t_c = (double)dmin;
    else if (t_c > (double)dmax) t_c = (double)dmax;
    double pcx = pos[0] + ddx * t_c;
    double pcy = pos[1] + ddy * t_c;
    double pcz = pos[2] + ddz * t_c;
    if (unbounded != 0) {
        double nx = (pcx - bc[0]) / bh[0];
        double ny = (pcy - bc[1]) / bh[1];
        double nz = (pcz - bc[2]) / bh[2];
        double r = sqrt(nx * nx + ny * ny + nz * nz);
        if (r > 1.0) {
            double s = (2.0 - 1.0 / r) / r;
            pcx = bc[0] + nx * s * bh[0];
            pcy = bc[1] + ny * s * bh[1];
            pcz = bc[2] + nz * s * bh[2];
        }
    }
    double dx = xc0 - pcx;
    double dy = xc1 - pcy;
    double dz = xc2 - pcz;
    double delta = sqrt(dx * dx + dy * dy + dz * dz);
    float span = dmax - dmin;                               /* f32 site */
    double tau_sp = dx_vox * g + lam * (double)span;
    double b = beta * (double)nsamp;
    if (b > bmax) b = bmax;
    double tau_dp = (gamma + b) * dx_vox;
    int ok = (delta <= tau_sp) && (fabs(x_d - (double)dexp) <= tau_dp);
    float msum = dmin + dmax;                               /* f32 site */
    double mu = 0.5 * (double)msum;
    double hd = 0.5 * (double)span;                         /* f32 site (same op) */
    if (hd < eps) hd = eps;
    double r = fabs(t_c - mu) / hd;
    *wd_out = exp(-alpha1 * r * r);
    return ok;
}

/* _thin_pair: returns ok_footprint; writes npix and t */
static int thin_pair(double xc0, double xc1, double xc2, const double *rot,
                     const double *pos, double fx, double fy, double cx, double cy,
                     double w, double h, double x_d, const float *mask,
                     const float *dexp, const int32_t *nsamp, const uint8_t *valid,
                     int64_t wm, double dx_vox, double gamma, double beta,
                     double bmax, double thin_pct, int64_t *npix_out, double *t_out)
{
    double half = 0.5 * dx_vox;
    double umin = 1e30, umax = -1e30, vmin = 1e30, vmax = -1e30;
    for (int j = 0; j < 8; ++j) {
        double sx = ((j & 1) == 0) ? -1.0 : 1.0;
        double sy = ((j & 2) == 0) ? -1.0 : 1.0;
        double sz = ((j & 4) == 0) ? -1.0 : 1.0;
        proj_t c = project_px(rot, pos, fx, fy, cx, cy, w, h,
                              xc0 + sx * half, xc1 + sy * half, xc2 + sz * half);
        if (!c.in_front) return 0;
        if (c.u < umin) umin = c.u;
        if (c.u > umax) umax = c.u;
        if (c.v < vmin) vmin = c.v;
        if (c.v > vmax) vmax = c.v;
    }
    int64_t wi = (int64_t)w;
    int64_t hi = (int64_t)h;
    int64_t xs = nb_floor_int(umin * w);
    int64_t xe = nb_floor_int(umax * w);
    int64_t ys = nb_floor_int(vmin * h);
    int64_t ye = nb_floor_int(vmax * h);
    if (xe < 0 || xs > wi - 1 || ye < 0 || ys > hi - 1) return 0;
    if (xs < 0) xs = 0;
    if (ys < 0) ys = 0;
    if (xe > wi - 1) xe = wi - 1;
    if (ye > hi - 1) ye = hi - 1;
    int64_t support = 0, npix = 0;
    double m_max = 0.0;
    for (int64_t yy = ys; yy <= ye; ++yy) {
        for (int64_t xx = xs; xx <= xe; ++xx) {
            npix += 1;
            double mv = (double)mask[yy * wm + xx];
            if (mv > m_max) m_max = mv;
            if (mv > 0.5 && valid[yy * wm + xx] != 0) {
                double b = beta * (double)nsamp[yy * wm + xx];
                if (b > bmax) b = bmax;
                double tau_d = (2.0 * gamma + b) * dx_vox;
                if (fabs(x_d - (double)dexp[yy * wm + xx]) <= tau_d) support += 1;
            }
        }
    }
    double p_cov = (double)support / (double)npix;
    *npix_out = npix;
    *t_out = (p_cov >= thin_pct) ? m_max : p_cov;
    return 1;
}

static double sorted_sum(double *values, int64_t n)
{
    for (int64_t i = 1; i < n; ++i) {
        double key = values[i];
        int64_t j = i - 1;
        while (j >= 0 && values[j] > key) { values[j + 1] = values[j]; --j; }
        values[j + 1] = key;
    }
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += values[i];
    return s;
}

static void sorted_sum_pairs(double *w, double *mw, int64_t n, double *sw, double *sm)
{
    for (int64_t i = 1; i < n; ++i) {
        double kw = w[i], km = mw[i];
        int64_t j = i - 1;
        while (j >= 0 && (w[j] > kw || (w[j] == kw && mw[j] > km))) {
            w[j + 1] = w[j];
            mw[j + 1] = mw[j];
            --j;
        }
        w[j + 1] = kw;
        mw[j + 1] = km;
    }
    double a = 0.0, b = 0.0;
    for (int64_t i = 0; i < n; ++i) { a += w[i]; b += mw[i]; }
    *sw = a;
    *sm = b;
}

static void voxel_views(const oracle_fuse_args *A, int64_t vi,
                        double *tw, double *tmw, double *tt)
{
    const double *pv = A->pv;
    const double gamma = pv[0], beta = pv[1], bmax = pv[2], lam = pv[3];
    const double rho_thr = pv[4], rho_thin = pv[5], thin_pct = pv[6];
    const double alpha1 = pv[7], thin_accept = pv[8], eps = pv[9];
    const double mask_thr = pv[10], thin_floor = pv[11];
    const int enable_thin = pv[13] != 0.0;
    const int64_t g = A->g, gg = g * g;
    const int64_t ix = vi / gg;
    const int64_t rem = vi - ix * gg;
    const int64_t iy = rem / g;
    const int64_t iz = rem - iy * g;
    const double dx_vox = A->dx_vox;
    const double rho = (double)A->density[vi];
    double p = 0.0, sw = 0.0, smw = 0.0, st = 0.0;
    int64_t n_thick = 0, n_thin = 0;

    if (A->early_out && rho < rho_thr && (rho < rho_thin || !enable_thin))
        goto store;   /* exact: no pair can pass either density gate */
    {
    const double xc0 = A->origin[0] + ((double)ix + 0.5) * dx_vox;
    const double xc1 = A->origin[1] + ((double)iy + 0.5) * dx_vox;
    const double xc2 = A->origin[2] + ((double)iz + 0.5) * dx_vox;
    const int64_t plane = A->hm * A->wm;
    for (int64_t view = 0; view < A->nv; ++view) {
        const double *in = A->intr + view * 6;
        const double fx = in[0], fy = in[1], cx = in[2], cy = in[3], w = in[4], h = in[5];
        const double *rot = A->rots + view * 9;
        const double *pos = A->poss + view * 3;
        proj_t pr = project_px(rot, pos, fx, fy, cx, cy, w, h, xc0, xc1, xc2);
        if (!pr.in_front || pr.u < 0.0 || pr.u >= 1.0 || pr.v < 0.0 || pr.v >= 1.0)
            continue;
        const double x_d = pr.d;
        const int64_t px = pixel_index(pr.u, (int64_t)w);
        const int64_t py = pixel_index(pr.v, (int64_t)h);
        const int64_t pix = view * plane + py * A->wm + px;
        if (A->valids[pix] == 0) continue;
        const float m = A->masks[pix];
        int routed_thick = 0;
        if ((double)m >= mask_thr && rho >= rho_thr) {
            double wd;
            int ok = thick_pair(xc0, xc1, xc2, rot, pos, fx, fy, cx, cy, w, h,
                                pr.u, pr.v, x_d, A->dmins[pix], A->dmaxs[pix],
                                A->dexps[pix], A->nsamps[pix], A->gmaps[pix], dx_vox,
                                gamma, beta, bmax, lam, alpha1, eps, A->bc, A->bh,
                                A->unbounded, &wd);
            if (ok) {
                tw[n_thick] = wd;
                tmw[n_thick] = (double)m * wd;
                n_thick += 1;
                routed_thick = 1;
            }
        }
        if (!routed_thick && enable_thin) {
            const double fmax = fx > fy ? fx : fy;
            if ((double)m > thin_floor && rho >= rho_thin && x_d > 0.0
                    && dx_vox * fmax / x_d >= 1.0) {
                int64_t npix;
                double t;
                int okf = thin_pair(xc0, xc1, xc2, rot, pos, fx, fy, cx, cy, w, h,
                                    x_d, A->masks + view * plane, A->dexps + view * plane,
                                    A->nsamps + view * plane, A->valids + view * plane,
                                    A->wm, dx_vox, gamma, beta, bmax, thin_pct,
                                    &npix, &t);
                if (okf && npix > 0 && t >= thin_accept) {
                    tt[n_thin] = t;
                    n_thin += 1;
                }
            }
        }
    }
    sorted_sum_pairs(tw, tmw, n_thick, &sw, &smw);
    st = sorted_sum(tt, n_thin);
    double denom = sw + (double)n_thin;
    p = (denom > eps) ? (smw + st) / denom : 0.0;
    }
store:
    A->out[vi] = p;
    if (A->n_thick) A->n_thick[vi] = (int32_t)n_thick;
    if (A->n_thin) A->n_thin[vi] = (int32_t)n_thin;
    if (A->sw) A->sw[vi] = sw;
    if (A->smw) A->smw[vi] = smw;
    if (A->st) A->st[vi] = st;
}

typedef struct {
    const oracle_fuse_args *A;
    _Atomic int64_t *next;
} worker_ctx;

#define ORACLE_CHUNK 256

static void *fuse_worker(void *arg)
{
    worker_ctx *c = (worker_ctx *)arg;
    const oracle_fuse_args *A = c->A;
    const int64_t nv = A->nv > 0 ? A->nv : 1;
    double *scratch = (double *)malloc(sizeof(double) * 3 * (size_t)nv);
    double *tw = scratch, *tmw = scratch + nv, *tt = scratch + 2 * nv;
    for (;;) {
        int64_t s = atomic_fetch_add(c->next, ORACLE_CHUNK);
        if (s >= A->vox_hi) break;
        int64_t e = s + ORACLE_CHUNK < A->vox_hi ? s + ORACLE_CHUNK : A->vox_hi;
        for (int64_t vi = s; vi < e; ++vi)
            voxel_views(A, vi, tw, tmw, tt);
    }
    free(scratch);
    return NULL;
}

ORACLE_API int oracle_max_threads(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

/* Voxel-owned accumulation: results are independent of the thread count,
 * exactly as the reference's prange over voxel chunks (fusion.py:17-20). */
ORACLE_API int oracle_fuse(const oracle_fuse_args *A)
{
    int nt = A->nthreads > 0 ? (int)A->nthreads : oracle_max_threads();
    if (nt > 1024) nt = 1024;
    _Atomic int64_t next = A->vox_lo;
    worker_ctx ctx = { A, &next };
    if (nt == 1) { fuse_worker(&ctx); return 0; }
    pthread_t th[1024];
    int started = 0;
    for (int i = 0; i < nt; ++i) {
        if (pthread_create(&th[i], NULL, fuse_worker, &ctx) != 0) break;
        ++started;
    }
    if (started == 0) fuse_worker(&ctx);
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    return 0;
}
