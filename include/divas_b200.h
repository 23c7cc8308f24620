/*
 * divas_b200.h -- C ABI of the B200-native DivAS fusion hot path.
 *
 * One shared library, libdivas_b200.so (sm_100a), built from
 * paper_2601_04860_b200/csrc/.  Plain pointers and sizes only: every array
 * argument is a DEVICE pointer (CUDA global memory, C-contiguous, 16-byte
 * aligned unless stated), `stream` is a cudaStream_t passed as void*, and the
 * caller owns every buffer ("Ownership").  The library
 * keeps no mutable global state: all scratch lives in a caller-provided
 * workspace, so calls are re-entrant across threads and streams.
 *
 * Every entry point returns 0 on success or a nonzero DIVAS_E* code; the
 * message of the calling thread's last failure is divas_last_error().
 * Kernels are enqueued asynchronously on `stream`; nothing synchronises.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/divas/):
 *   divas_refine         <- segmenter.refine_mask            segmenter.py:129-152
 *   divas_fuse           <- fusion._gradient_maps + fusion._fuse_kernel
 *                           (the numba operator that fusion.fuse calls)
 *                                                           fusion.py:684-689, :493-509, :720-723
 *   divas_gradient_maps  <- fusion._gradient_maps            fusion.py:684-689
 *   divas_threshold      <- `ogrid.probs >= threshold` + np.argwhere
 *                                                           ablation.py:109
 *   divas_overlay        <- fusion._overlay_kernel           fusion.py:771-843
 *   divas_vgrid_payload  <- io.write_vgrid's transpose        io.py:59-69
 *   divas_pair_trace     <- fusion.thick_check / thin_check   fusion.py:549-646
 *   divas_render         <- render._render (render_view)      render.py:221-292
 *   divas_march_rays     <- render._march (march_ray)         render.py:160-218, :257-267
 *   divas_bake_density   <- scene.bake_density_grid           scene.py:194-201
 */
#ifndef DIVAS_B200_H
#define DIVAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DIVAS_ABI_VERSION 11

/* error codes */
#define DIVAS_OK          0
#define DIVAS_EINVAL      1   /* bad argument (shape, size, null pointer)   */
#define DIVAS_ECUDA       2   /* CUDA launch / runtime failure              */
#define DIVAS_EWORKSPACE  3   /* workspace too small                        */

/* Per-view camera record, DIVAS_CAM_STRIDE doubles per view, in device
 * memory:  r[9] (world_from_camera[:3,:3] row-major; columns are the camera
 * axes in world, geometry.py:61-64), pos[3] (world_from_camera[:3,3]),
 * fx, fy, cx, cy, width, height  (fusion.py:671-673, :444-451). */
#define DIVAS_CAM_STRIDE 18

/* FusionParams.as_vector() layout (fusion.py:80-87). */
#define DIVAS_NPARAM 14

/* Views are stored as padded SoA planes [nv][hm][wm] exactly as
 * fusion._pack_views builds them (fusion.py:653-681): (hm, wm) is the largest
 * view, smaller views sit in the top-left corner, padding is zero.  The valid
 * flag is derived as n_samples > 0 (render.py:67-69). */

/* ---------------------------------------------------------------------- */
/* Refinement: out = clip(mask * (1 - zhat), 0, 1) on valid pixels, 0 else, */
/* zhat min-max normalised over each view's valid pixels (Eq. 2).           */
/* ---------------------------------------------------------------------- */
size_t divas_refine_workspace_size(int32_t nv);
int divas_refine(int32_t nv, int64_t hm, int64_t wm,
                 const float *mask, const float *z_surface, const int32_t *n_samples,
                 float *out, void *workspace, size_t workspace_bytes, void *stream);

/* Refinement fused with the fusion's per-view "aux" data, in one pass:
 *   out      [nv][hm][wm] f32 refined masks as divas_refine (may be NULL);
 *   records  per view two [hm][wm] float2 planes (divas_records_size bytes):
 *            A = {refined mask, d_exp or NaN where the pixel cannot support a
 *            thin candidate}; the mask's sign bit flags a supporting pixel
 *            whose tau_d differs from the view's base tau_d(n_min) (readers
 *            take |mask|); B = {tau_d(n) as f32, n_samples bits}, written
 *            only at supporting pixels;
 *   bands    per view [ceil(hm/8)][ceil(wm/8)] {lo, hi} f64 per 8x8 tile (the
 *            depth interval in which a thin candidate can find support) and
 *            two more 16-byte entries: {min, max} order-preserving u32 keys
 *            of tau_d over the view's supporting pixels, the counts of
 *            flagged and of supporting pixels; {base tau_d f32 bits, 0, 0,
 *            0} (divas_bands_size).
 * pv = FusionParams.as_vector() and dx_vox (the tolerances depend on them).
 * Views are independent: view k's slices start at k * divas_records_size(1,..)
 * / k * divas_bands_size(1,..) bytes, so a single view can be (re)built in
 * place with nv = 1 and offset pointers. */
size_t divas_records_size(int32_t nv, int64_t hm, int64_t wm);
size_t divas_bands_size(int32_t nv, int64_t hm, int64_t wm);
int divas_refine_bands(int32_t nv, int64_t hm, int64_t wm,
                       const float *mask, const float *z_surface, const int32_t *n_samples,
                       const float *dexp, float *out, const double *pv, double dx_vox,
                       void *records, void *bands, void *workspace, size_t workspace_bytes,
                       void *stream);
/* As divas_refine_bands, but records and bands are built only inside one
 * window per view: roi = DEVICE int32 [nv][4] {x0, y0, x1, y1} (inclusive
 * pixel bounds, x0 and y0 multiples of 8), roi_w / roi_h = the largest
 * window's width / height (grid size).  The per-view min/max of z still
 * covers the whole view (the refinement is exactly the full one inside the
 * window); `out`, records and bands outside the windows are left untouched.
 * Used with the projection of a slab's gated voxels: the fusion of that slab
 * reads no pixel outside it (sharding.slab_view_rois). */
/* The per-view refine keys on their own: keys [nv][4] u32 = z min, z max
 * (order-preserving f32 keys) and n min, n max over the valid pixels (an
 * empty view has min > max).  Lets the
 * views' min/max passes be split across ranks and the keys exchanged; then
 * divas_refine_bands_keys builds the records from them (roi may be NULL). */
int divas_refine_minmax(int32_t nv, int64_t hm, int64_t wm, const float *z_surface,
                        const int32_t *n_samples, uint32_t *keys, void *stream);
int divas_refine_bands_keys(int32_t nv, int64_t hm, int64_t wm,
                            const float *mask, const float *z_surface, const int32_t *n_samples,
                            const float *dexp, float *out, const double *pv, double dx_vox,
                            void *records, void *bands, const uint32_t *keys, void *workspace,
                            size_t workspace_bytes, const int32_t *roi, int32_t roi_w,
                            int32_t roi_h, void *stream);
int divas_refine_bands_roi(int32_t nv, int64_t hm, int64_t wm,
                           const float *mask, const float *z_surface, const int32_t *n_samples,
                           const float *dexp, float *out, const double *pv, double dx_vox,
                           void *records, void *bands, void *workspace, size_t workspace_bytes,
                           const int32_t *roi, int32_t roi_w, int32_t roi_h, void *stream);

/* ---------------------------------------------------------------------- */
/* Fusion                                                                   */
/* ---------------------------------------------------------------------- */
/* `mode` of divas_fuse_args: 0 (DIVAS_FUSE_FULL) or an OR of steps.        */
#define DIVAS_STEP_GATE        1  /* zero the outputs on [lo, hi), build the
                                     gated-voxel list                          */
#define DIVAS_STEP_CLEAR_ALL   2  /* zero every contribution bit              */
#define DIVAS_STEP_CLEAR_VIEWS 4  /* zero the bits of views [view_lo, view_hi) */
#define DIVAS_STEP_PAIRS       8  /* evaluate views [view_lo, view_hi)          */
#define DIVAS_STEP_REDUCE     16  /* value-sorted sums over all nv views -> p  */
#define DIVAS_STEP_ZERO       32  /* only the zero fill of the outputs on
                                     [lo, hi) (p, votes, sums, occupancy, peer
                                     buffers): with GATE_KEEP below, the dense
                                     fill can run on another stream, e.g.
                                     beside the compute-bound PAIRS step      */
#define DIVAS_STEP_GATE_KEEP  64  /* with GATE: build the gated-voxel list but
                                     leave the outputs untouched (a ZERO step
                                     must precede REDUCE)                     */
#define DIVAS_FUSE_FULL        0  /* = GATE | CLEAR_ALL | PAIRS(all) | REDUCE  */
#define DIVAS_FUSE_INCREMENTAL (DIVAS_STEP_CLEAR_VIEWS | DIVAS_STEP_PAIRS | DIVAS_STEP_REDUCE)
/* Steps without GATE reuse the gated list, and steps without PAIRS the
 * contributions, that earlier calls left in the same workspace (same density,
 * range, params and output buffers).  Between calls the caller may edit the
 * workspace regions (divas_fuse_ws_regions), e.g. to exchange contributions
 * between ranks that evaluated different views (views-sharding). */

typedef struct divas_fuse_args {
    int64_t g;                   /* grid resolution G (voxels per axis)       */
    double origin[3];            /* grid min corner (VoxelGrid.origin)        */
    double dx_vox;               /* VoxelGrid.voxel_size()                    */
    const float *density;        /* [G^3] rho, [ix,iy,iz] C-order             */
    int32_t nv;                  /* number of views (>= 1)                    */
    int32_t hm, wm;              /* padded plane height / width               */
    const double *cams;          /* [nv][DIVAS_CAM_STRIDE]                    */
    const float *masks;          /* [nv][hm][wm] refined confidences (read only
                                    when records == NULL)                     */
    const float *dmins, *dmaxs, *dexps;   /* [nv][hm][wm]                     */
    const int32_t *nsamps;       /* [nv][hm][wm]                              */
    double pv[DIVAS_NPARAM];     /* FusionParams.as_vector()                  */
    double bc[3], bh[3];         /* SceneBounds centre / half (fusion.py:542) */
    int32_t unbounded;           /* spherical contraction on/off              */
    int64_t vox_lo, vox_hi;      /* flat voxel range [lo, hi) to fuse (a slab) */
    double *probs;               /* [G^3] out, written on [lo, hi); may be
                                    page-locked host memory (unified addressing:
                                    the kernels write it directly).  NULL is
                                    allowed in calls without REDUCE: GATE then
                                    leaves the (caller-zeroed) output alone.   */
    int32_t *n_thick, *n_thin;   /* [G^3] integer votes, or NULL              */
    double *sw, *smw, *st;       /* [G^3] sorted sums, or NULL                */
    uint8_t *occ;                /* [G^3] fused threshold p >= occ_thr, or NULL */
    double occ_thr;
    int64_t max_gated;           /* slot capacity: upper bound on voxels that pass
                                    the density gate in [lo, hi); <= 0 means
                                    hi - lo (always safe).  divas_gate_count
                                    gives the exact figure for a density grid. */
    const void *records;         /* scan records / bands of divas_refine_bands   */
    const void *bands;           /* for these views, pv and dx_vox; NULL: built
                                    in the workspace from masks/n/d_exp         */
    int32_t nv_cap;              /* views the workspace holds (>= nv; <= 0: nv) */
    int32_t mode;                /* DIVAS_FUSE_FULL or DIVAS_STEP_* flags       */
    int32_t view_lo, view_hi;    /* views evaluated by PAIRS / cleared by
                                    CLEAR_VIEWS (ignored by FULL)              */
    uint8_t *const *occ_peers;   /* device array of n_peers device pointers, or
                                    NULL: [G^3] occupancy buffers (one per rank,
                                    e.g. NVLink peer mappings of symmetric
                                    memory).  The fused occupancy of [lo, hi)
                                    is stored into EVERY listed buffer at the
                                    same offsets -- the slab all-gather fused
                                    into the gate (zeros) and reduce (p >=
                                    occ_thr) stores.  Independent of `occ`.    */
    int32_t n_peers;
    uint64_t *fallbacks;         /* NULL, or device [DIVAS_NFALLBACK] counters:
                                    how often each certified shortcut could
                                    not decide and the reference's exact chain
                                    ran (DIVAS_FB_*; accumulated, never reset) */
} divas_fuse_args;

/* Fallback counters of divas_fuse_args.fallbacks (exact-chain evaluations). */
#define DIVAS_FB_CENTRE      0   /* centre pixel / frustum: exact u, v chain     */
#define DIVAS_FB_THICK       1   /* thick spatial test: exact _thick_pair chain  */
#define DIVAS_FB_THICK_T     2   /* thick weight: exact t_proj for the clamp     */
#define DIVAS_FB_CORNERS     3   /* thin footprint: exact 8-corner chain         */
#define DIVAS_FB_RECOUNT     4   /* thin support: f64 recount of the footprint   */
#define DIVAS_FB_THIN_GATE   5   /* thin gate dx * max(fx, fy) / x_d >= 1 in f64 */
#define DIVAS_FB_BAND_WIDE   6   /* band test skipped: box wider than its tiles  */
#define DIVAS_FB_TILE_SKIP   7   /* (not a fallback) pair tiles rejected whole by
                                    the tile-level band test                    */
#define DIVAS_FB_THIN_SORT   8   /* reduction: a voxel's thin sum needed the
                                    value sort (its view-order sum was not
                                    certified exact in every order)             */
#define DIVAS_NFALLBACK      9

/* Workspace bytes for divas_fuse with slot capacity `max_gated`, `nv_cap`
 * views of padded size hm x wm (~ max_gated * (4 + nv_cap * 24.25) bytes for
 * the [view][slot] contributions, plus records and bands when the caller does
 * not supply them). */
size_t divas_fuse_workspace_size(int64_t max_gated, int32_t nv_cap, int32_t hm, int32_t wm);
/* The same with internal_aux = 0 for callers that always pass records/bands
 * (divas_refine_bands output): the record / band regions are then not
 * reserved (C3: ~390 MB less).  divas_fuse sizes its layout by whether
 * args->records is NULL. */
size_t divas_fuse_workspace_size_ext(int64_t max_gated, int32_t nv_cap, int32_t hm, int32_t wm,
                                     int32_t internal_aux);
int divas_fuse(const divas_fuse_args *args, void *workspace, size_t workspace_bytes,
               void *stream);

/* Count the voxels of [vox_lo, vox_hi) that pass the exact density gate
 * rho >= pv[4] || (pv[13] != 0 && rho >= pv[5]); only args->g, vox_lo, vox_hi,
 * density and pv are read.  The count lands in divas_fuse_gated_count(ws)
 * (workspace >= 256 bytes). */
int divas_gate_count(const divas_fuse_args *args, void *workspace, void *stream);

/* Device pointers into a divas_fuse workspace: the gated-voxel count of the
 * last call (int64) and its overflow flag (int32, nonzero when the count
 * exceeded max_gated -- voxels past the capacity were then left at p = 0). */
const int64_t *divas_fuse_gated_count(const void *workspace);
const int32_t *divas_fuse_overflow(const void *workspace);

/* Byte offsets of the workspace regions for (max_gated, nv_cap, hm, wm,
 * internal_aux as in divas_fuse_workspace_size_ext):
 * out[0] gated-voxel list (u32 [cap]), out[1] thick bits, out[2] thin bits
 * (u32 [ceil(nv_cap/32)][cap] each), out[3] w, out[4] m*w, out[5] t
 * (f64 [nv_cap][cap] each), out[6] total size. */
void divas_fuse_ws_regions(int64_t max_gated, int32_t nv_cap, int32_t hm, int32_t wm,
                           int32_t internal_aux, size_t out[7]);

/* The f64 depth-gradient maps of fusion._gradient_maps on the padded planes
 * (divas_fuse computes g on the fly; this export is for parity tests and for
 * fusion.depth_gradient).  valid_only != 0: invalid pixels get 0 as in
 * _gradient_map (fusion.py:232-240); 0: _grad_at at every pixel. */
int divas_gradient_maps(int32_t nv, int32_t hm, int32_t wm, const float *dexps,
                        const float *dmins, const float *dmaxs, const int32_t *nsamps,
                        double eps, double kappa, int32_t valid_only, double *out, void *stream);

/* ---------------------------------------------------------------------- */
/* Per-pair decision trace: the reference's public per-pair operations      */
/* thick_check / thin_check (fusion.py:549-646), which _fuse_traced          */
/* (fusion.py:727-764) and fuse(trace_path=...) are built on.  Their        */
/* arithmetic differs from the fused kernel's exactly where the reference's */
/* does: _thick_pair receives Python floats (f64 at the d_min/d_max sites)  */
/* and the gradient uses each view's true-size neighbourhood.  One record   */
/* per query (point, rho, view), evaluated on the device.                   */
/* ---------------------------------------------------------------------- */
#define DIVAS_STAGE_FRUSTUM      0
#define DIVAS_STAGE_NO_SURFACE   1
#define DIVAS_STAGE_MASK_GATE    2
#define DIVAS_STAGE_DENSITY_GATE 3
#define DIVAS_STAGE_SPATIAL      4
#define DIVAS_STAGE_DEPTH        5
#define DIVAS_STAGE_PASSED       6

typedef struct divas_pair_record {
    int32_t stage;               /* thick_check stage (DIVAS_STAGE_*)         */
    int32_t thin_candidate;      /* thin_check candidate flag                 */
    double m, delta, g, tau_spatial, tau_depth, t_proj, t_clamped, x_d, mu_d, h_d, r, w_depth;
    int64_t x_start, x_end, y_start, y_end, support_count, n_pixels;
    double p_covered, m_max, t;
} divas_pair_record;

typedef struct divas_trace_args {
    int32_t nv, hm, wm;          /* padded planes; true sizes from cams      */
    const double *cams;          /* [nv][DIVAS_CAM_STRIDE]                    */
    const float *masks, *dmins, *dmaxs, *dexps;
    const int32_t *nsamps;       /* [nv][hm][wm]                              */
    double pv[DIVAS_NPARAM];
    double bc[3], bh[3];
    int32_t unbounded;
    double dx_vox;               /* voxel_size (the cube edge of thin_check)  */
    int64_t n;                   /* queries                                   */
    const double *points;        /* [n][3] voxel centres (world)              */
    const double *rho;           /* [n] densities                             */
    const int32_t *views;        /* [n] view index per query                  */
    divas_pair_record *out;      /* [n]                                       */
} divas_trace_args;

int divas_pair_trace(const divas_trace_args *args, void *stream);

/* ---------------------------------------------------------------------- */
/* Threshold / extract: occ[i] = p[i] >= thr;  idx = C-order indices of the */
/* set voxels (np.argwhere order), written as (ix,iy,iz) int64 triples when */
/* g > 0 (needs n == g^3) or as flat int64 indices when g == 0.  *count     */
/* (device int64) receives the number of set voxels.  occ / idx may be NULL.*/
/* ---------------------------------------------------------------------- */
size_t divas_threshold_workspace_size(int64_t n);
int divas_threshold(const double *p, int64_t n, double thr, int64_t g,
                    uint8_t *occ, int64_t *idx, int64_t *count,
                    void *workspace, size_t workspace_bytes, void *stream);

/* .vgrid payload (io.write_vgrid, io.py:59-69): out[iz][iy][ix] =       */
/* (float)p[ix][iy][iz] -- the file's x-fastest float32 order.              */
int divas_vgrid_payload(const double *p, int64_t g, float *out, void *stream);

/* ---------------------------------------------------------------------- */
/* Overlay: binary mask of pixels whose ray meets a voxel with p >= thr     */
/* (project_grid_overlay).  HOST arrays: cam (one DIVAS_CAM_STRIDE record), */
/* origin, bc, bh.  DEVICE arrays: dmin/dmax/nsamp [h][w] planes of the     */
/* view, probs [G^3], out [h][w] uint8.                                     */
/* ---------------------------------------------------------------------- */
int divas_overlay(const double *cam, int32_t h, int32_t w, const float *dmin,
                  const float *dmax, const int32_t *nsamp, const double *probs,
                  int64_t g, const double origin[3], double dx_vox,
                  const double bc[3], const double bh[3], int32_t unbounded,
                  double thr, uint8_t *out, void *stream);

/* ---------------------------------------------------------------------- */
/* Fixture producers: the volumetric ray       */
/* marcher and the density bake.  The scene is HOST memory (it is copied    */
/* into the launch); cams / rays / outputs are DEVICE memory.               */
/* ---------------------------------------------------------------------- */
#define DIVAS_MAX_PRIMS 128

typedef struct {                /* SceneModel.packed() (scene.py:126-151)   */
    int32_t n_prims;            /* 0 .. DIVAS_MAX_PRIMS                     */
    const uint8_t *kinds;       /* [n] 0 sphere, 1 box, 2 capsule           */
    const double *params;       /* [n][7] (packed() layout)                 */
    const double *density;      /* [n]                                      */
    const double *colors;       /* [n][3]                                   */
    const double *soft;         /* [n] soft-edge widths                     */
    double background[3];
} divas_scene;

typedef struct {                /* RenderConfig (render.py:37-50)           */
    int32_t samples_per_ray;
    double near_, far_, tau_cw, min_weight;
} divas_render_cfg;

/* render_view for nv cameras of one size: outputs [nv][h][w] (rgb
 * [nv][h][w][3]).  unsure (nullable, [nv][h][w]) flags the pixels whose
 * bits could differ from the reference's because CUDA's exp and the C
 * library's differ in the last place and that difference could cross a
 * decision or an f32 rounding boundary (a certified bound, see render.cu);
 * every other pixel is bit-identical to render_view's. */
int divas_render(const divas_scene *scene, const divas_render_cfg *cfg, int32_t nv,
                 const double *cams, int32_t h, int32_t w, float *rgb, float *d_min,
                 float *d_max, float *d_exp, int32_t *n_samples, float *z_surface,
                 uint8_t *unsure, void *stream);

/* march_ray on n unit rays [n][6] (origin, direction): out [n][8] f64 =
 * r, g, b, d_min, d_max, d_exp, n_samples, z_surface; err (nullable) [n][4] =
 * bounds of |out - reference| for r, g, b, d_exp; unsure (nullable) [n] as
 * above (d_min, d_max, z_surface, n_samples exact when 0). */
int divas_march_rays(const divas_scene *scene, const divas_render_cfg *cfg, int64_t n,
                     const double *rays, double *out, double *err, uint8_t *unsure,
                     void *stream);

/* bake_density_grid: out [G^3] f32, [ix,iy,iz], voxel centres
 * origin + (i + 0.5) * dx_vox, contracted (geometry.contract) when
 * unbounded with bounds centre bc / half extent bh (HOST arrays). */
int divas_bake_density(const divas_scene *scene, int64_t g, const double origin[3],
                       double dx_vox, int32_t unbounded, const double bc[3], const double bh[3],
                       float *out, void *stream);

/* ---------------------------------------------------------------------- */
const char *divas_last_error(void);

/* Per view, the bounding box {x0, y0, x1, y1} (DEVICE int32 [nv][4]; empty:
 * x1 = -1) of the pixels of DEVICE masks [nv][hm][wm] with mask >= thr: the
 * upload window of the depth maps in refine_and_fuse (they are read only at
 * pixels whose refined mask -- at most the raw one -- clears the thick or thin
 * mask threshold, and at the 4-neighbours of those). */
int divas_mask_bbox(int32_t nv, int64_t hm, int64_t wm, const float *masks, float thr,
                    int32_t *bbox, void *stream);

/* Host -> device copy of a pitched sub-rectangle (cudaMemcpy2DAsync): the
 * windowed upload of view planes in refine_and_fuse. */
int divas_copy2d_h2d(void *dst, size_t dpitch, const void *src, size_t spitch,
                     size_t width_bytes, size_t height, void *stream);

/* One sub-rectangle of a batched window upload (divas_gather2d_h2d): `rows`
 * rows of `width_bytes` bytes from page-locked host memory src (row pitch
 * spitch) to device memory dst (row pitch dpitch). */
typedef struct divas_copy2d {
    const void *src;
    void *dst;
    int64_t spitch, dpitch, width_bytes, rows;
} divas_copy2d;

/* Every rectangle of jobs[0 .. n) read by the SMs straight from page-locked
 * host memory (mapped through unified addressing) in one launch: short-row
 * windows move at the link rate instead of the copy engine's per-row rate.
 * Each src must be page-locked (cudaHostAlloc / cudaHostRegister);
 * DIVAS_EINVAL otherwise.  Same result as one divas_copy2d_h2d per job. */
int divas_gather2d_h2d(const divas_copy2d *jobs, int32_t n, void *stream);

/* Store `bytes` of device memory src into every buffer of a DEVICE table of
 * n_peers pointers (symmetric-memory peer mappings), at `offset`: one rank's
 * block of an all-gather as NVLink stores in one launch (the caller then runs
 * a device barrier). */
int divas_peer_put(const void *src, size_t bytes, uint8_t *const *peers, int32_t n_peers,
                   size_t offset, void *stream);
int divas_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DIVAS_B200_H */
