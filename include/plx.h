/*
 * plx.h -- C ABI of the B200 (sm_100a) Plenoxels optimisation hot path.
 *
 * This is the drop-in boundary: every entry point replaces one L0 kernel call
 * of the reference package `plenoxel` (pkg/src/plenoxel/_kernels.py, "K"),
 * or one numpy structure op (grid.py, "G"), at the seam where the reference's
 * L1 wrappers call into numba.  Conventions follow the
 * reference's:
 *   - the caller owns and allocates every buffer (outputs, gradients, scratch);
 *     entry points never allocate persistent state -- with ONE exception:
 *     plx_train_step creates, on its first call per device, a side stream, a
 *     high-priority stream and four events (TV runs beside the backward) and
 *     keeps them for the process; plx_release_streams() destroys them;
 *   - kernels never fail on data; argument validation returns PLX_EINVAL;
 *   - all pointers are DEVICE pointers unless stated; work is enqueued on
 *     `stream` (a cudaStream_t, NULL = legacy default stream) and is
 *     asynchronous -- nothing here synchronises the host.
 *
 * Storage differs from the reference in precision and layout: the grid's
 * data are float32 in two arrays, `density` [rows] (sigma) and `table`
 * [rows x 28] (SH channel-major in columns 1..27, column 0 padding), so the
 * sigma gathers of the march touch a compact 4 B/row array instead of 112-
 * byte rows; the gradient buffer and RMSProp state are float32 (rows x 28,
 * column 0 = sigma).  Row arrays (table, grad, v) have a pitch of PLX_STRIDE
 * = 32 floats: every row is one 128-byte cache line, so row gathers and
 * read-modify-writes never straddle lines or write partial sectors.  Arithmetic is float64 except the colour dot products.
 * Rays are float64 (N x 3).  The touched-row set of GradientBuffer (G:25-68:
 * touched_mask + insertion-ordered touched_ids + count) is kept as the byte
 * mask alone; the count is produced by plx_opt_step / plx_count_touched.
 */
#ifndef PLX_H
#define PLX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PLX_ROW 28     /* columns of a row: sigma (or padding) + 27 SH        */
#define PLX_STRIDE 32  /* row pitch in floats: 128-byte rows, one cache line;
                          columns 28..31 are padding (never read as data)  */

enum {
    PLX_OK = 0,
    PLX_EINVAL = 1,   /* bad argument (reference: ValueError) */
    PLX_ECUDA = 2,    /* launch / runtime error */
};

/* Sparse grid: replaces the (links, table, lo, hi, scale, dmax) argument
 * group of render_forward / render_backward / max_weight_accum / tv_grid
 * (K:174-177, K:242-248, K:415-416, K:457-459) and SparseGrid (G:71-92). */
typedef struct {
    const int32_t *links;  /* [Dx*Dy*Dz] C-order (z fastest), -1 = empty     */
    float *table;          /* [rows*PLX_STRIDE] SH rows: columns 1..27 = the
                              reference table's SH columns; column 0 is
                              padding (16-byte rows), never read          */
    float *density;        /* [rows] sigma = the reference table column 0  */
    int64_t dims[3];       /* Dx, Dy, Dz (each >= 2)                         */
    int64_t rows;
    double lo[3], hi[3];   /* aabb_min / aabb_max                            */
    double scale[3];       /* lattice_scale = (D-1)/extent   (G:137-139)     */
    double dmax[3];        /* D-1                            (R:132)         */
    const uint32_t *cell_occ; /* optional: 1 bit per trilinear base cell,
                                 set iff any of its 8 corners is occupied
                                 (plx_build_cell_occ); NULL = test the links */
    float *sigma_lat;      /* optional [Dx*Dy*Dz] lattice-indexed mirror of
                              density: the sigma of the row at each lattice
                              point, NaN where empty (plx_build_sigma_lat).
                              The march then reads the 8 corner sigmas in
                              ONE gather level (no links, no rows) and loads
                              links only for the samples it keeps.  The
                              optimisers keep it current (need row_cell);
                              rebuild after editing density or links.  For
                              an identity-linked dense grid it may simply
                              alias `density` (then nothing is maintained). */
    const int32_t *row_cell; /* [rows] lattice point of each row (inverse of
                              links, plx_build_row_cell); required with
                              sigma_lat by the optimisers                 */
    uint32_t *brick_dead;  /* optional, with a sigma_lat that is not density:
                              1 bit per brick of 8^3 base cells (bricks
                              ((Dx-2)/8+1) x ((Dy-2)/8+1) x ((Dz-2)/8+1),
                              z fastest), set iff every cell of the brick
                              has no occupied corner or 8 occupied corners
                              with sigma < 0 -- no position inside can be
                              composited (K:211, K:293), so the march skips
                              its sigma gathers.  plx_build_brick_dead
                              sets it; the optimisers clear the bricks
                              around every row whose sigma becomes >= 0;
                              rebuild after editing density or links. */
} plx_grid;

/* GradientBuffer (G:25-68): data + touched mask, and optionally the
 * touched-id list + count (touched_ids / _count).  When tids/tcnt are set,
 * plx_opt_step compacts the mask into them and updates the list (two-phase);
 * when both are NULL it sweeps the mask in place. */
typedef struct {
    float *grad;           /* [rows*PLX_STRIDE] */
    uint8_t *tmask;        /* [rows]    */
    int32_t *tids;         /* [rows] scratch, or NULL (order unspecified)  */
    int64_t *tcnt;         /* [1] length of tids after plx_opt_step, or NULL */
} plx_grad;

/* RenderOptions (R:27-42) resolved to kernel scalars (R:63-64, R:132-139). */
typedef struct {
    double step;           /* step_frac * min(voxel_size)                    */
    double stop_thresh;
    double bg[3];
    int32_t nearest;       /* interp == "nearest"                            */
    int32_t absolute;      /* formula == "absolute"                          */
    int64_t *stats;        /* optional device int64[4], ACCUMULATED by the
                              march kernels: {march positions evaluated (up
                              to the early stop), samples composited, 32-
                              position chunks, rays}; NULL = off          */
} plx_render_opts;

/* A camera ray pool: replaces the reference's host-built
 * ray arrays (camera.py:91-134 generate_rays / to_ndc, camera.py:292-314
 * all_rays; 96 B of float64 per ray) by the views' camera records and the
 * float32 ground-truth colours (12 B per ray).  Kernels regenerate a ray
 * from its pool row, bit-identical to the reference's arrays.  Pool row p is
 * global pixel pixel[p] (or p when pixel == NULL) = view * W*H + y * W + x,
 * row-major pixels as all_rays orders them. */
#define PLX_CAM 16   /* doubles per camera record */
typedef struct {
    const double *cams;      /* [n_views][PLX_CAM]: c2w[:3,:4] row-major (12),
                                focal, width, height, near (camera.py:27-48) */
    const float *rgb;        /* [rows][3] gt colours (the image float32
                                values, camera.py:193), or NULL           */
    const int64_t *pixel;    /* optional [rows] global pixel id per pool row
                                (forward-facing pools drop invalid rays)   */
    int64_t n_views, width, height;
    int32_t ndc;             /* forward-facing: march rays warped to NDC
                                (camera.py:103-134); SH uses the world dir */
    int32_t reserved;
    double scale;            /* origin pre-scale (360 scenes, T:375-377), 1 */
} plx_cameras;

/* A ray batch.  If idx != NULL ray r of the batch is pool row idx[r] of
 * origins/dirs/viewdirs/target (device-resident ray pool);
 * outputs are always indexed by batch position r.  With cams != NULL the
 * pool is that camera pool instead: origins/dirs/viewdirs are ignored and
 * target defaults to cams->rgb (used when target == NULL). */
typedef struct {
    const double *origins;   /* [*,3]                                        */
    const double *dirs;      /* [*,3] march directions                       */
    const double *viewdirs;  /* [*,3] SH directions (unit)                   */
    const double *target;    /* [*,3] gt rgb (mse_mode) or dL/dC; may be NULL */
    const double *jitter;    /* [n] start offsets in steps, or NULL (= 0)    */
    const int64_t *idx;      /* [n] pool indices, or NULL                    */
    int64_t n;
    const plx_cameras *cams; /* HOST pointer to a camera pool, or NULL      */
} plx_rays;

/* Materialise pool rows idx[0..n) (or rows 0..n-1 when idx == NULL) of a
 * camera pool as float64 (n,3) arrays: march origins / directions, view
 * directions and gt colours (any output may be NULL) -- all_rays
 * (camera.py:292-314) on the device. */
int plx_generate_rays(const plx_cameras *cams, const int64_t *idx, int64_t n, double *origins,
                      double *dirs, double *viewdirs, double *rgb, void *stream);
/* to_ndc (camera.py:103-134) of n device rays in place, for the camera
 * record `cam` (HOST double[PLX_CAM]); valid[n] (uint8, may be NULL) =
 * |d_z| > 1e-10. */
int plx_to_ndc(const double *cam, double *origins, double *dirs, uint8_t *valid, int64_t n,
               void *stream);

/* Image metrics of evaluate (T:309-347): losses.psnr / losses.ssim
 * (losses.py:110-165) of one view on the device.  a, b: (h, w, c) float64;
 * window: HOST double[11], the normalised Gaussian of losses.py:124-128.
 * out_sums (device double[2], ACCUMULATED) += {sum of (a-b)^2 over all
 * values, sum of the SSIM map over the valid interior [5:-5, 5:-5] of every
 * channel}; psnr = -10 log10(out[0] / (h w c)), ssim = out[1] / ((h-10)
 * (w-10) c).  scratch: plx_image_metrics_scratch_bytes(h, w, c) bytes.
 * window == NULL: only the squared-error sum (psnr alone, any image size). */
int64_t plx_image_metrics_scratch_bytes(int64_t h, int64_t w, int64_t c);
int plx_image_metrics(const double *a, const double *b, int64_t h, int64_t w, int64_t c,
                      const double *window, double k1, double k2, double *out_sums,
                      void *scratch, int64_t scratch_bytes, void *stream);

/* render_forward (K:173-238) via render_rays (R:114-140).
 * out_trans / out_wsum may be NULL. */
int plx_render_fwd(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o,
                   double *out_rgb, double *out_trans, double *out_wsum, void *stream);

/* render_backward (K:241-411) via fused_mse_backward (R:253-279, mse_mode=1,
 * up_scale = 2/n_total) and render_rays_backward (R:205-239, mse_mode=0,
 * target = upstream dL/dC).  Gradients are ADDED into gb->grad with f32
 * reductions (red.global.add.f32: the hardware flushes subnormal operands
 * and results to zero, so contributions below 1.18e-38 in magnitude are
 * dropped -- the reference's f64 accumulator keeps them; K:581 then skips
 * only exact zeros); every occupied stencil row of every recorded sample is marked
 * in gb->tmask.  out_sums (device double[2]) is ACCUMULATED with
 * {mse_sum, cauchy_sum}; out_rgb may be NULL.  `scratch` is a device
 * workspace of at least plx_render_scratch_bytes(g, o, rays->n) bytes (it
 * replaces the reference's per-call s_* scratch arrays, R:277-278). */
int64_t plx_render_scratch_bytes(const plx_grid *g, const plx_render_opts *o, int64_t n_rays);
int plx_render_fused_bwd(const plx_grid *g, const plx_rays *rays,
                         const plx_render_opts *o, int32_t mse_mode, double up_scale,
                         double lam_cauchy, plx_grad *gb, double *out_rgb,
                         double *out_sums, void *scratch, int64_t scratch_bytes,
                         void *stream);

/* max_weight_accum (K:414-453) via SparseGrid.max_weight_accumulate
 * (G:287-302).  out_w [rows] float64 is max-updated in place (caller zeroes). */
int plx_max_weight(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o,
                   double *out_w, void *stream);

/* tv_grid (K:456-569) via tv_loss (L:50-77).  Cells are either the explicit
 * list `cells` [count] (flat C-order ids) or, when cells == NULL, the wrapped
 * contiguous run start, start+1, ... (mod ncell) of sample_tv_cells
 * (L:41-47).  out_sums (device double[2]) is ACCUMULATED with the raw
 * {sigma_sum, sh_sum}. */
int plx_tv(const plx_grid *g, const int64_t *cells, int64_t start, int64_t count,
           double fac_x, double fac_y, double fac_z, double eps, double f_sigma,
           double f_sh, int32_t wrap_x, int32_t wrap_y, int32_t wrap_z,
           int32_t with_grad, plx_grad *gb, double *out_sums, void *stream);

/* opt_step (K:572-590) via optim.step (O:81-97), fused with clear_grad
 * (K:593-600) when clear != 0.  Visits rows whose tmask is set; entries with
 * g == 0 keep their stale state.  out_count (device int64, may be NULL)
 * receives the number of touched rows (GradientBuffer.n_touched).
 * guard (device double[5], may be NULL) moves the trainer's divergence check
 * (T:473-480) onto the device: guard[0..3] = the step's loss sums {mse,
 * cauchy, tv_sigma, tv_sh}, guard[4] = sticky halt flag; if any sum is
 * non-finite or guard[4] != 0, nothing is updated or cleared and guard[4]
 * is set to 1, so the host can check asynchronously. */
int plx_opt_step(plx_grid *g, float *v, plx_grad *gb, double lr_sigma, double lr_sh,
                 double beta, double eps, int32_t rmsprop, int32_t clear,
                 double *guard, int64_t *out_count, void *stream);

/* clear_grad (K:593-600) alone (GradientBuffer.clear, G:62-64): zero the
 * touched rows of gb->grad and reset gb->tmask.  out_count as above. */
int plx_clear_grad(plx_grad *gb, int64_t rows, int64_t *out_count, void *stream);

/* ---- data-parallel exchange (no reference counterpart: the
 * reference is single-process, K:267 "for ri in range(nray)").  Rays shard
 * across ranks, the grid is replicated, and the per-step gradient exchange +
 * update replaces T:483-486 (optim.step + grads.clear) on every rank. ---- */

/* Ordered (ascending) list of the set bytes of tmask[rows] -> ids[*count]
 * (device), e.g. the union of the ranks' touched rows after an all_reduce
 * MAX of the masks.  scratch: plx_scan_scratch_bytes(rows) bytes. */
int plx_touched_list(const uint8_t *tmask, int64_t rows, int32_t *ids, int64_t *count,
                     void *scratch, void *stream);
/* dst[j] = src row ids[j] for j < *count (device): rows of PLX_STRIDE floats
 * packed at a 28-float pitch (the all-reduce moves no padding); cap bounds
 * the launch (rows). */
int plx_pack_rows(const float *src, const int32_t *ids, const int64_t *count, int64_t cap,
                  float *dst, void *stream);
/* opt_step over the rows ids[0..*count): gradients from gpack[j] (packed,
 * e.g. all-reduced) or, if gpack == NULL, from gb->grad rows; clear != 0
 * zeroes gb->grad and gb->tmask of the listed rows.  guard / out_count as in
 * plx_opt_step. */
int plx_opt_step_list(plx_grid *g, float *v, plx_grad *gb, const int32_t *ids,
                      const int64_t *count, const float *gpack, double lr_sigma, double lr_sh,
                      double beta, double eps, int32_t rmsprop, int32_t clear, double *guard,
                      int64_t *out_count, void *stream);

/* The ranks' buffers as seen from this process (own ones local, the others
 * CUDA-IPC-mapped peer memory over NVLink). */
#define PLX_MAX_PEERS 8
typedef struct {
    int32_t n, rank;
    int64_t rows;
    float *grad[PLX_MAX_PEERS];        /* rows x PLX_STRIDE each */
    uint8_t *tmask[PLX_MAX_PEERS];
    float *table[PLX_MAX_PEERS];       /* SH rows (column 0 unused) */
    float *density[PLX_MAX_PEERS];
    float *sigma_lat[PLX_MAX_PEERS];   /* lattice sigma mirrors, may be NULL */
} plx_dp_peers;
/* Fused reduce + update + broadcast over peer memory: rank `rank` owns the
 * 128-row-aligned slice [rows*rank/n, rows*(rank+1)/n); for every row of it
 * touched on ANY rank it sums the n gradient rows (rank order), applies the
 * update with its own RMSProp state v, and stores the new sigma / SH row
 * (and lattice sigma) into all n grids.  Gradients and masks are NOT cleared
 * (each rank clears its own with plx_clear_grad after all ranks finished:
 * the caller orders the ranks with a collective before and after).
 * out_count (local) accumulates the slice's union count. */
int plx_dp_owner_update(const plx_dp_peers *p, float *v, const int32_t *row_cell,
                        double lr_sigma, double lr_sh, double beta, double eps, int32_t rmsprop,
                        double *guard, int64_t *out_count, void *stream);
/* CUDA IPC of a device buffer that may sit inside a larger allocation. */
int plx_ipc_export(const void *ptr, uint8_t handle[64], int64_t *offset);
int plx_ipc_import(const uint8_t handle[64], int64_t offset, void **base_out, void **ptr_out);
int plx_ipc_close(void *base);

/* GradientBuffer.n_touched (G:42-44): out_count (device int64) = popcount. */
int plx_count_touched(const uint8_t *tmask, int64_t rows, int64_t *out_count,
                      void *stream);

/* Structure ops (G:228-285).  Both are two-phase because the new row count
 * must reach the host to size the new table (as numpy does):
 *   1. *_mark   -> flags[ncell_new] (uint8)
 *   2. plx_scan_ids(flags) -> new_links (int32, -1 where flag==0) + count
 *   3. *_apply  -> new table (+ kept ids for prune)
 * plx_scan_scratch_bytes(n) sizes the scan workspace. */
int plx_prune_mark(const plx_grid *g, const double *weights, double threshold,
                   uint8_t *deemed_scratch /* 2 * ncell bytes */, uint8_t *flags,
                   void *stream);
int plx_prune_apply(const plx_grid *g, const int32_t *new_links, int64_t *kept_old,
                    float *new_table, float *new_density, void *stream);
int plx_upsample_mark(const plx_grid *g, const int64_t new_dims[3], uint8_t *flags,
                      void *stream);
int plx_upsample_apply(const plx_grid *g, const int64_t new_dims[3],
                       const int32_t *new_links, float *new_table, float *new_density,
                       void *stream);
int64_t plx_scan_scratch_bytes(int64_t n);
int plx_scan_ids(const uint8_t *flags, int64_t n, int32_t *ids, int64_t *count,
                 void *scratch, void *stream);

/* SparseGrid.sample (G:182-200) at n world points pts (n,3) float64 inside
 * the AABB (the caller checks, G:147-151): out (n,28) float64 = the
 * interpolated (sigma, 27 SH) over occupied stencil corners, sigma clamped
 * at 0.  nearest: the nearest lattice point (G:158-163). */
int plx_grid_sample(const plx_grid *g, const double *pts, int64_t n, int32_t nearest,
                    double *out, void *stream);
/* SparseGrid.sample_backward (G:202-223): upstream (n,28) float64 dL/d(sigma,
 * SH); w_q * upstream added to every occupied stencil row of each point
 * (f32 atomics; the row is marked touched), the sigma entry dropped where the
 * interpolated sigma is negative. */
int plx_grid_sample_backward(const plx_grid *g, const double *pts, const double *upstream,
                             int64_t n, int32_t nearest, plx_grad *gb, void *stream);

/* Empty-space skipping helper: cell_occ bit (i,j,k) for every trilinear base
 * cell (i<Dx-1, j<Dy-1, k<Dz-1; stored over the full Dx*Dy*Dz index space)
 * = any of the 8 corner links >= 0.  Must be rebuilt after prune/upsample. */
int64_t plx_cell_occ_words(const int64_t dims[3]);
int plx_build_cell_occ(const plx_grid *g, uint32_t *cell_occ, void *stream);
/* Dead-brick bitmask (plx_grid.brick_dead) from sigma_lat: words needed,
 * and the build (g->sigma_lat required). */
int64_t plx_brick_words(const int64_t dims[3]);
int plx_build_brick_dead(const plx_grid *g, uint32_t *brick_dead, void *stream);
/* sigma_lat ([Dx*Dy*Dz] floats) and row_cell ([rows] int32). */
int plx_build_sigma_lat(const plx_grid *g, float *sigma_lat, void *stream);
int plx_build_row_cell(const plx_grid *g, int32_t *row_cell, void *stream);

/* One training step (T:441-486) as one call: zero sums[0..3], fused
 * render + backward (mse_mode, up_scale), TV on the (start, count) run when
 * tv_count > 0, and -- when update != 0 (single GPU; on N ranks the
 * exchange runs in between and the update is separate) -- plx_opt_step with
 * the fused clear and sums as the divergence guard.  events[0..3] (optional
 * cudaEvent_t) are recorded before the render, after the render, after TV
 * and after the update. */
typedef struct {
    plx_rays rays;
    plx_render_opts opts;
    double up_scale, lam_cauchy;
    void *scratch;
    int64_t scratch_bytes;
    int64_t tv_start, tv_count;
    double tv_fac[3], tv_eps, tv_f_sigma, tv_f_sh;
    int32_t update, rmsprop;
    float *v;
    double lr_sigma, lr_sh, beta, eps;
    double *sums;          /* device double[5]: 4 loss sums + sticky halt */
    int64_t *count;        /* device int64: n_touched (may be NULL)       */
    void *events[4];
    /* optional device copies of the per-step scalars (tv_start; lr_sigma,
     * lr_sh): when set the kernels read them at run time, so the call can be
     * captured in a CUDA graph once and replayed with new values */
    const int64_t *dev_tv_start;
    const double *dev_lr;
    /* optional device int64 added to rays.idx by the kernels: the batch as a
     * moving slice of a fixed index buffer, so a captured graph replays any
     * batch of the same size */
    const int64_t *dev_idx_off;
    /* optional pinned HOST memory read / written by the step's kernels (so
     * a captured step has no memcpy nodes): host_params (4 int64) is copied
     * to dev_params by the step's first kernel; the loss sums (4 doubles)
     * are written to host_sums by the update's compaction kernel */
    const int64_t *host_params;
    int64_t *dev_params;
    double *host_sums;
} plx_step_args;
int plx_train_step(plx_grid *g, plx_grad *gb, const plx_step_args *a, void *stream);
/* Destroy the per-device streams / events plx_train_step created (call with
 * no step in flight, e.g. at shutdown). */
int plx_release_streams(void);

/* ---- Multi-sphere-image background (unbounded 360 scenes) ----------------
 * Reference: msi.py (MsiBackground, BgGradientBuffer, render_rays_with_
 * background, bg_tv_loss), _kernels.py K:603-977 (render_backward_360,
 * tv_bg), optim.py O:100-107 (step_table).  All background data is f64. */
typedef struct {
    const double *data;    /* [L][H][W][4] (sigma, r, g, b), device          */
    const double *radii;   /* [L] increasing (msi.layer_radii; last may be inf) */
    int64_t L, H, W;       /* 2 <= L <= 257, H >= 2, W >= 1                   */
} plx_msi;
typedef struct {
    double *grad;          /* [L*H*W][4] f64 accumulator                     */
    uint8_t *tmask;        /* [L*H*W] touched texels                         */
    int32_t *tids;         /* [L*H*W] compacted list (plx_msi_opt_step)      */
    int64_t *tcnt;         /* device int64                                    */
} plx_msi_grad;
/* Scratch for plx_msi_render: with gradients the foreground runs through the
 * bounded backward (plx_render_fused_bwd's records, in waves) plus a
 * background stage; forward only needs a ray counter.  -1 on bad arguments. */
int64_t plx_msi_scratch_bytes(const plx_grid *g, const plx_msi *bg, const plx_render_opts *o,
                              int64_t n_rays);
/* msi.render_rays_with_background (msi.py:130-183 -> K:661-881): rays.
 * origins / dirs (world; the SH basis uses dirs) and rays.target (gt for
 * mse_mode, else the upstream dL/drgb); opts: step, stop_thresh, nearest.
 * gb == NULL: forward only.  out_sums (device double[3], accumulated):
 * {mse, cauchy_raw, beta_raw}; out_rgb (N,3), out_tfg / out_trans (N). */
int plx_msi_render(const plx_grid *g, const plx_msi *bg, const plx_rays *rays,
                   const plx_render_opts *o, int32_t mse_mode, double up_scale,
                   double lam_cauchy, double lam_beta, double beta_eps, plx_grad *gb,
                   plx_msi_grad *bgb, double *out_rgb, double *out_tfg, double *out_trans,
                   double *out_sums, void *scratch, int64_t scratch_bytes, void *stream);
/* msi.bg_tv_loss raw sums (K:884-977): cells (device int64, or NULL for the
 * run start..start+count wrapping mod L*H*W); bgb NULL = value only;
 * out_sums (device double[2], accumulated): {sigma, rgb}. */
int plx_msi_tv(const plx_msi *bg, const int64_t *cells, int64_t start, int64_t count,
               double eps, double f_sigma, double f_rgb, plx_msi_grad *bgb, double *out_sums,
               void *stream);
/* optim.step_table on the background (O:100-107, K:572-590) over the
 * texels marked in bgb->tmask, then (clear) the clear of K:593-600.
 * table = bg->data viewed as [L*H*W][4]; v likewise (RMSProp). */
int plx_msi_opt_step(double *table, double *v, plx_msi_grad *bgb, int64_t n_texels,
                     double lr_sigma, double lr_rgb, double beta, double eps, int32_t rmsprop,
                     int32_t clear, int64_t *out_count, void *stream);

/* Library identification / self-check. */
const char *plx_version(void);
int plx_device_check(void);   /* 0 iff a CUDA device with cc >= 10.0 is present */

#ifdef __cplusplus
}
#endif
#endif /* PLX_H */
