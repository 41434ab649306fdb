// plx_internal.h -- entry points shared between the library's translation
// units (not part of the C ABI in include/plx.h): the native step
// (plx_step.cu) calls the render, TV and update with device-resident
// per-step scalars and the prologue's zeroed counters.
#pragma once
#include <stdint.h>

#include "../../include/plx.h"

namespace plx {
// The 360 backward's background stage (plx_msi_render with gradients):
// render_fused_bwd_impl runs msi_bg_kernel between the colour and scatter
// kernels and the bounded kernels leave rgb / mse to it.
struct MsiHook {
    const double *data, *radii;   // background [L][H][W][4], radii [L]
    int64_t L, H, W;
    double lam_beta, beta_eps;
    double *out_tfg, *out_trans;  // (N)
    double *bg_grad;              // [L*H*W][4]
    uint8_t *bg_tmask;
};
// plx_render_fused_bwd plus: idx_off = optional device int64 added to
// rays->idx; counters_ready = the scratch's 3 counters were zeroed by the
// caller (first wave only); after_march = optional cudaEvent_t recorded once
// the first wave's march kernel is enqueued.
int render_fused_bwd_impl(const plx_grid *g, const plx_rays *rays, const int64_t *idx_off,
                          const plx_render_opts *o, int32_t mse_mode, double up_scale,
                          double lam_cauchy, plx_grad *gb, double *out_rgb, double *out_sums,
                          void *scratch, int64_t scratch_bytes, void *stream,
                          int counters_ready, void *after_march = nullptr,
                          const MsiHook *msi = nullptr);
// plx_opt_step plus: lr_dev = optional device {lr_sigma, lr_sh};
// tcnt_ready = gb->tcnt was zeroed by the caller; host_sums = optional
// pinned host double[4] that receives the guard's loss sums.
int opt_step_impl(plx_grid *g, float *v, plx_grad *gb, double lr_sigma, double lr_sh,
                  const double *lr_dev, double beta, double eps, int32_t rmsprop, int32_t clear,
                  double *guard, int64_t *out_count, void *stream, int tcnt_ready,
                  double *host_sums);
// plx_tv_loss plus start_dev = optional device run start; short_blocks = one
// 32-cell iteration per block (a background TV on a low-priority stream).
int tv_impl(const plx_grid *g, const int64_t *cells, int64_t start, const int64_t *start_dev,
            int64_t count, double fac_x, double fac_y, double fac_z, double eps, double f_sigma,
            double f_sh, int32_t wrap_x, int32_t wrap_y, int32_t wrap_z, int32_t with_grad,
            plx_grad *gb, double *out_sums, void *stream, int short_blocks = 0);
// Byte mask -> compact int32 list of its nonzero rows (tile compaction of the
// update, order within 8192-row tiles), optionally clearing the mask.
int compact_mask_impl(uint8_t *tmask, int64_t rows, int32_t *tids, int64_t *tcnt, int clear,
                      void *stream);
}  // namespace plx
