/* divas_oracle_render.c -- CPU oracle for the fixture producers (TEST
 * INFRASTRUCTURE ONLY; see oracle/__init__.py).
 *
 * Restates, op for op in IEEE binary64 without contraction:
 *   _prim_density  /root/reference/pkg/src/divas/render.py:96-157
 *   _march         render.py:160-218
 *   _render        render.py:221-254 (ray through each pixel centre)
 *   bake_density_grid scene.py:194-201 with ScenePrimitive.signed_distance /
 *                  density_at (scene.py:69-105), VoxelGrid.centers
 *                  (geometry.py:140-147) and contract (geometry.py:242-256).
 *
 * The bake restates NUMPY's evaluation, not numba's: np.linalg.norm over the
 * last axis sums the squares left to right; a 1-D `x @ x` / `np.linalg.norm`
 * of a 3-vector goes through BLAS ddot, and `points @ ab` through dgemv.  On
 * the machine that produced the golden vectors (OpenBLAS 0.3.30
 * DYNAMIC_ARCH, AVX-512 host) those are the fused chains
 * fma(x2,y2, fma(x1,y1, x0*y0)) (ddot) and fma(p2,a2, fma(p0,a0, p1*a1))
 * (dgemv), measured bit for bit over 2e4 random vectors each; they enter
 * only the capsule's segment parameter and the unbounded contraction.
 * exp is the C library's, which is also what numba's math.exp calls.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
    int64_t n;
    const uint8_t *kinds;      /* 0 sphere, 1 box, 2 capsule */
    const double *params;      /* [n][7] */
    const double *dens;        /* [n] */
    const double *cols;        /* [n][3] */
    const double *soft;        /* [n] */
    const double *bg;          /* [3] */
} oracle_scene;

typedef struct {
    int64_t n_steps;
    double near_, far_, tau_cw, min_w;
} oracle_render_cfg;

/* render.py:96-157 */
static double prim_density(const oracle_scene *S, double px, double py, double pz, int64_t *bi)
{
    double best = 0.0;
    int64_t best_i = -1;
    for (int64_t i = 0; i < S->n; ++i) {
        const double *P = S->params + 7 * i;
        double sd;
        if (S->kinds[i] == 0) {
            const double dx = px - P[0], dy = py - P[1], dz = pz - P[2];
            const double dist = sqrt(dx * dx + dy * dy + dz * dz);
            sd = dist - P[3];
            if (P[4] > 0.0) {
                const double sd2 = P[4] - dist;
                if (sd2 > sd) sd = sd2;
            }
        } else if (S->kinds[i] == 1) {
            const double qx = fabs(px - P[0]) - P[3];
            const double qy = fabs(py - P[1]) - P[4];
            const double qz = fabs(pz - P[2]) - P[5];
            const double ox = qx > 0.0 ? qx : 0.0, oy = qy > 0.0 ? qy : 0.0, oz = qz > 0.0 ? qz : 0.0;
            const double outside = sqrt(ox * ox + oy * oy + oz * oz);
            double mx = qx > qy ? qx : qy;
            if (qz > mx) mx = qz;
            const double inside = mx < 0.0 ? mx : 0.0;
            sd = outside + inside;
        } else {
            const double ax = P[0], ay = P[1], az = P[2];
            const double abx = P[3] - ax, aby = P[4] - ay, abz = P[5] - az;
            const double denom = abx * abx + aby * aby + abz * abz;
            double t;
            if (denom > 0.0) {
                t = ((px - ax) * abx + (py - ay) * aby + (pz - az) * abz) / denom;
                if (t < 0.0) t = 0.0;
                else if (t > 1.0) t = 1.0;
            } else {
                t = 0.0;
            }
            const double cx = ax + t * abx, cy = ay + t * aby, cz = az + t * abz;
            const double dx = px - cx, dy = py - cy, dz = pz - cz;
            sd = sqrt(dx * dx + dy * dy + dz * dz) - P[6];
        }
        double fall;
        if (S->soft[i] > 0.0) {
            fall = 1.0 - sd / S->soft[i];
            if (fall < 0.0) fall = 0.0;
            else if (fall > 1.0) fall = 1.0;
        } else {
            fall = sd <= 0.0 ? 1.0 : 0.0;
        }
        const double d = S->dens[i] * fall;
        if (d > best) {
            best = d;
            best_i = i;
        }
    }
    *bi = best_i;
    return best;
}

/* render.py:160-218; out = r, g, b, d_min, d_max, d_exp, n_samples, z_surface */
void oracle_march(const oracle_scene *S, const oracle_render_cfg *R, const double *ray,
                  double *out)
{
    const double ox = ray[0], oy = ray[1], oz = ray[2];
    const double dx = ray[3], dy = ray[4], dz = ray[5];
    const double dt = (R->far_ - R->near_) / (double)R->n_steps;
    double T = 1.0, cum = 0.0, d_min = 0.0, d_max = 0.0, last_hit = 0.0;
    double w_peak = 0.0, z_peak = 0.0, wsum = 0.0, wt = 0.0, cr = 0.0, cg = 0.0, cb = 0.0;
    int have_min = 0, stopped = 0;
    int64_t count = 0;
    for (int64_t k = 0; k < R->n_steps; ++k) {
        const double t = R->near_ + ((double)k + 0.5) * dt;
        int64_t pi;
        const double sigma = prim_density(S, ox + dx * t, oy + dy * t, oz + dz * t, &pi);
        const double a = sigma > 0.0 ? 1.0 - exp(-sigma * dt) : 0.0;
        const double w = T * a;
        if (w > 0.0) {
            count += 1;
            last_hit = t;
            wsum += w;
            wt += w * t;
            if (w > w_peak) {
                w_peak = w;
                z_peak = t;
            }
            cr += w * S->cols[3 * pi + 0];
            cg += w * S->cols[3 * pi + 1];
            cb += w * S->cols[3 * pi + 2];
        }
        cum += w;
        T *= (1.0 - a);
        if (!have_min && cum > R->min_w) {
            have_min = 1;
            d_min = t;
        }
        if (cum >= R->tau_cw) {
            d_max = t;
            stopped = 1;
            break;
        }
    }
    if (!stopped) d_max = last_hit;
    cr += (1.0 - cum) * S->bg[0];
    cg += (1.0 - cum) * S->bg[1];
    cb += (1.0 - cum) * S->bg[2];
    out[0] = cr; out[1] = cg; out[2] = cb;
    if (!have_min) {
        out[3] = out[4] = out[5] = out[7] = 0.0;
        out[6] = 0.0;
        return;
    }
    double d_exp = wt / wsum;
    if (d_exp < d_min) d_exp = d_min;
    else if (d_exp > d_max) d_exp = d_max;
    out[3] = d_min; out[4] = d_max; out[5] = d_exp; out[6] = (double)count; out[7] = z_peak;
}

typedef struct {
    const oracle_scene *S;
    const oracle_render_cfg *R;
    const double *rot, *pos, *intr;   /* rot row-major [3][3]; intr fx fy cx cy w h */
    float *rgb, *dmin, *dmax, *dexp, *zs;
    int32_t *ns;
    int64_t p0, p1;
} render_job;

static void *render_worker(void *arg)
{
    const render_job *J = (const render_job *)arg;
    const double *r = J->rot;
    const double fx = J->intr[0], fy = J->intr[1], cx = J->intr[2], cy = J->intr[3];
    const int64_t width = (int64_t)J->intr[4];
    for (int64_t p = J->p0; p < J->p1; ++p) {
        const int64_t iy = p / width, ix = p - iy * width;
        /* render.py:226-235 */
        const double xc = ((double)ix + 0.5 - cx) / fx;
        const double yc = (cy - ((double)iy + 0.5)) / fy;
        double dxw = r[0] * xc + r[1] * yc - r[2];
        double dyw = r[3] * xc + r[4] * yc - r[5];
        double dzw = r[6] * xc + r[7] * yc - r[8];
        const double norm = sqrt(dxw * dxw + dyw * dyw + dzw * dzw);
        dxw /= norm;
        dyw /= norm;
        dzw /= norm;
        const double ray[6] = {J->pos[0], J->pos[1], J->pos[2], dxw, dyw, dzw};
        double o[8];
        oracle_march(J->S, J->R, ray, o);
        J->rgb[3 * p + 0] = (float)o[0];
        J->rgb[3 * p + 1] = (float)o[1];
        J->rgb[3 * p + 2] = (float)o[2];
        J->dmin[p] = (float)o[3];
        J->dmax[p] = (float)o[4];
        J->dexp[p] = (float)o[5];
        J->ns[p] = (int32_t)o[6];
        J->zs[p] = (float)o[7];
    }
    return NULL;
}

/* render.py:221-254 over all pixels of one camera */
void oracle_render(const oracle_scene *S, const oracle_render_cfg *R, const double *rot,
                   const double *pos, const double *intr, float *rgb, float *dmin, float *dmax,
                   float *dexp, int32_t *ns, float *zs, int64_t nthreads)
{
    const int64_t npix = (int64_t)intr[4] * (int64_t)intr[5];
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    render_job jobs[256];
    for (int64_t t = 0; t < nthreads; ++t) {
        jobs[t] = (render_job){S, R, rot, pos, intr, rgb, dmin, dmax, dexp, zs, ns,
                               npix * t / nthreads, npix * (t + 1) / nthreads};
        pthread_create(&th[t], NULL, render_worker, &jobs[t]);
    }
    for (int64_t t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ScenePrimitive.density_at (scene.py:69-105) in numpy's evaluation order */
static double np_density_at(const oracle_scene *S, int64_t i, double px, double py, double pz)
{
    const double *P = S->params + 7 * i;
    double sd;
    if (S->kinds[i] == 0) {
        const double dx = px - P[0], dy = py - P[1], dz = pz - P[2];
        const double dist = sqrt(dx * dx + dy * dy + dz * dz);
        sd = dist - P[3];
        if (P[4] > 0.0) {
            const double s2 = P[4] - dist;
            sd = s2 > sd ? s2 : sd;                         /* np.maximum */
        }
    } else if (S->kinds[i] == 1) {
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
        const double denom = fma(abz, abz, fma(aby, aby, abx * abx));       /* ddot */
        double t = 0.0;
        if (denom > 0.0) {
            const double rx = px - P[0], ry = py - P[1], rz = pz - P[2];
            t = fma(rz, abz, fma(rx, abx, ry * aby)) / denom;               /* dgemv */
            t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);                        /* np.clip */
        }
        const double dx = px - (P[0] + t * abx), dy = py - (P[1] + t * aby),
                     dz = pz - (P[2] + t * abz);
        sd = sqrt(dx * dx + dy * dy + dz * dz) - P[6];
    }
    double fall;
    if (S->soft[i] > 0.0) {
        fall = 1.0 - sd / S->soft[i];
        fall = fall < 0.0 ? 0.0 : (fall > 1.0 ? 1.0 : fall);
    } else {
        fall = sd <= 0.0 ? 1.0 : 0.0;
    }
    return S->dens[i] * fall;
}

typedef struct {
    const oracle_scene *S;
    int64_t g;
    const double *origin;
    double dx;
    int64_t unbounded;
    const double *bc, *bh;
    float *out;
    int64_t v0, v1;
} bake_job;

static void *bake_worker(void *arg)
{
    const bake_job *J = (const bake_job *)arg;
    const int64_t g = J->g;
    for (int64_t vi = J->v0; vi < J->v1; ++vi) {
        const int64_t ix = vi / (g * g), iy = (vi / g) % g, iz = vi % g;
        double p[3] = {J->origin[0] + ((double)ix + 0.5) * J->dx,
                       J->origin[1] + ((double)iy + 0.5) * J->dx,
                       J->origin[2] + ((double)iz + 0.5) * J->dx};
        if (J->unbounded) {                                     /* geometry.py:242-256 */
            double n[3];
            for (int k = 0; k < 3; ++k) n[k] = (p[k] - J->bc[k]) / J->bh[k];
            const double r = sqrt(fma(n[2], n[2], fma(n[1], n[1], n[0] * n[0])));
            if (!(r <= 1.0)) {
                const double s = 2.0 - 1.0 / r;
                for (int k = 0; k < 3; ++k) p[k] = J->bc[k] + (s * (n[k] / r)) * J->bh[k];
            }
        }
        double best = 0.0;                                      /* scene.py:186-191 */
        for (int64_t i = 0; i < J->S->n; ++i) {
            const double d = np_density_at(J->S, i, p[0], p[1], p[2]);
            if (d > best) best = d;
        }
        J->out[vi] = (float)best;
    }
    return NULL;
}

/* scene.py:194-201 */
void oracle_bake(const oracle_scene *S, int64_t g, const double *origin, double dx,
                 int64_t unbounded, const double *bc, const double *bh, float *out,
                 int64_t nthreads)
{
    const int64_t n = g * g * g;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    bake_job jobs[256];
    for (int64_t t = 0; t < nthreads; ++t) {
        jobs[t] = (bake_job){S, g, origin, dx, unbounded, bc, bh, out,
                             n * t / nthreads, n * (t + 1) / nthreads};
        pthread_create(&th[t], NULL, bake_worker, &jobs[t]);
    }
    for (int64_t t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}
