// plx_msi.cu -- multi-sphere-image background for unbounded 360 scenes
// (reference K:603-977 render_backward_360 / tv_bg, msi.py, O:100-107
// step_table).  Concentric equirectangular layers of f64 (sigma, r, g, b)
// texels beyond the foreground grid; a ray samples the grid exactly as the
// bounded render does, then the layers once per sphere crossing past the
// grid's exit, composited over black.
//
// Forward only (eval): msi_fwd_kernel here, one warp per ray.  With
// gradients the foreground runs through the bounded kernels of
// plx_render.cu (march / colour / scatter, whose work is spread over
// 32-sample segments of all rays) and msi_bg_kernel adds the background
// stage between colour and scatter (plx_render.cu).
//
// Device layout: background f64 [L][H][W][4]; its gradient f64 [L*H*W][4]
// with a byte mask (the reference's BgGradientBuffer); the grid side reuses
// plx_grid / plx_grad.
#include <cuda_runtime.h>

#include "plx_common.cuh"
#include "plx_internal.h"
#include "plx_msi.cuh"

namespace plx {
namespace {

constexpr int kMsiThreads = 128;
constexpr int kMsiWarps = kMsiThreads / 32;

struct MsiRays {
    const double *origins, *dirs, *target;
    int64_t n;
};

struct MsiOpts {
    double step, stop;
    int mse_mode;
    double up_scale, lam_beta, beta_eps;
};

struct MsiOut {
    double *rgb, *tfg, *trans, *sums;   // sums: {mse, cauchy_raw (0 without gradients), beta_raw}
};

// Forward render (K:661-833 without the reverse sweep), one warp per ray
// (rays from a device counter).  Foreground: 32 march positions per step as
// in the bounded render (f64 positions, stencil and sigma; f32 colour),
// composited with the warp product scan.  Background: the sphere crossings
// (lane = layer) compacted in layer order into shared memory, then sampled
// and composited 32 at a time.
template <bool NEAREST>
__global__ void __launch_bounds__(kMsiThreads)
    msi_fwd_kernel(DGrid G, MsiDev B, MsiRays R, MsiOpts O, MsiOut out, int *counter) {
    __shared__ double xs_t_all[kMsiWarps][kMaxCross];
    __shared__ int xs_l_all[kMsiWarps][kMaxCross];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *xs_t = xs_t_all[warp];
    int *xs_l = xs_l_all[warp];
    const unsigned lt = (1u << lane) - 1u;
    double mse_part = 0.0, beta_part = 0.0;
    for (;;) {
        int rr = 0;
        if (lane == 0) rr = atomicAdd(counter, 1);
        const int64_t ray = __shfl_sync(PLX_FULL_MASK, rr, 0);
        if (ray >= R.n) break;
        RayMarch rm;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            rm.o[a] = __ldg(R.origins + 3 * ray + a);
            rm.d[a] = __ldg(R.dirs + 3 * ray + a);
        }
        double basis[9];
        sh_basis9(rm.d[0], rm.d[1], rm.d[2], basis);   // K:699: raw ray dirs
        float bf[9];
#pragma unroll
        for (int b = 0; b < 9; ++b) bf[b] = (float)basis[b];
        double t0a, t1a;
        ray_aabb(rm.o, rm.d, G.lo, G.hi, t0a, t1a);
        ray_march_setup(rm, G, O.step, 0.0);
        double T = 1.0, A = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
        bool stopped = false;
        // ---- foreground (K:707-746) ----
        for (int64_t base = 0; base < rm.nsamp && !stopped; base += 32) {
            const int64_t si = base + lane;
            bool incl = false;
            double att = 1.0, sig = 0.0, t = 0.0, dlt = 0.0, g[3], fd[3];
            int32_t rows[8];
            int ijk[3];
            bool rows_ok = true;
            if (si < rm.nsamp) {
                sample_coords(rm, G, O.step, si, t, dlt, g);
                if (sigma_at<NEAREST>(G, g, fd, ijk, rows, sig, rows_ok)) {
                    incl = sig >= 0.0;
                    if (incl) att = exp(-sig * dlt);
                }
            }
            if (!__any_sync(PLX_FULL_MASK, incl)) continue;
            double Ti, wi;
            composite_chunk<false>(incl, att, lane, O.stop, T, A, Ti, wi, stopped);
            if (incl) {
                if (!rows_ok) load_rows<NEAREST>(G, ijk, rows);
                float c[3];
                colour_at_f32<NEAREST>(G, rows, fd, bf, c);
                if (c[0] > 0.f) c0 += wi * (double)c[0];
                if (c[1] > 0.f) c1 += wi * (double)c[1];
                if (c[2] > 0.f) c2 += wi * (double)c[2];
            }
        }
        const double tfg = T;
        // ---- background: one sample per sphere crossing (K:751-803) ----
        if (T >= O.stop) {
            const double t_exit = t1a > 0.0 ? t1a : 0.0;
            const double bdot = rm.o[0] * rm.d[0] + rm.o[1] * rm.d[1] + rm.o[2] * rm.d[2];
            const double c0n = rm.o[0] * rm.o[0] + rm.o[1] * rm.o[1] + rm.o[2] * rm.o[2];
            int nx = 0;
            for (int l0 = 0; l0 < B.L - 1; l0 += 32) {
                const int l = l0 + lane;
                bool hit = false;
                double tl = 0.0;
                if (l < B.L - 1) {
                    const double rad = __ldg(B.radii + l);
                    const double disc = bdot * bdot - c0n + rad * rad;
                    if (disc > 0.0) {
                        tl = -bdot + sqrt(disc);
                        hit = !(tl < t_exit);
                    }
                }
                const unsigned hm = __ballot_sync(PLX_FULL_MASK, hit);
                if (hit) {
                    const int q = nx + __popc(hm & lt);
                    xs_t[q] = tl;
                    xs_l[q] = l;
                }
                nx += __popc(hm);
            }
            __syncwarp();
            for (int q0 = 0; q0 < nx && !stopped; q0 += 32) {
                const int q = q0 + lane;
                bool incl = false;
                double att = 1.0, dlt = 0.0, o4[4] = {0.0, 0.0, 0.0, 0.0};
                if (q < nx) {
                    if (q + 1 < nx) dlt = xs_t[q + 1] - xs_t[q];
                    else if (q >= 1) dlt = xs_t[q] - xs_t[q - 1];
                    else dlt = 1.0;
                    const double t = xs_t[q];
                    int idx4[4];
                    double w4[4];
                    bg_stencil(B.H, B.W, rm.o[0] + t * rm.d[0], rm.o[1] + t * rm.d[1],
                               rm.o[2] + t * rm.d[2], idx4, w4);
                    bg_fetch(B, xs_l[q], idx4, w4, o4);
                    incl = o4[0] >= 0.0;
                    if (incl) att = exp(-o4[0] * dlt);
                }
                if (!__any_sync(PLX_FULL_MASK, incl)) continue;
                double Ti, wi;
                composite_chunk<false>(incl, att, lane, O.stop, T, A, Ti, wi, stopped);
                if (incl) {
                    if (o4[1] > 0.0) c0 += wi * o4[1];
                    if (o4[2] > 0.0) c1 += wi * o4[2];
                    if (o4[3] > 0.0) c2 += wi * o4[3];
                }
            }
            __syncwarp();
        }
        const double cr = warp_sum(c0), cg = warp_sum(c1), cb = warp_sum(c2);
        if (lane == 0) {
            out.rgb[3 * ray] = cr;
            out.rgb[3 * ray + 1] = cg;
            out.rgb[3 * ray + 2] = cb;
            out.tfg[ray] = tfg;
            out.trans[ray] = T;
            if (O.mse_mode) {   // K:808-814
                const double e0 = cr - __ldg(R.target + 3 * ray),
                             e1 = cg - __ldg(R.target + 3 * ray + 1),
                             e2 = cb - __ldg(R.target + 3 * ray + 2);
                mse_part += e0 * e0 + e1 * e1 + e2 * e2;
            }
            double tc = tfg;   // K:822-828
            if (tc < O.beta_eps) tc = O.beta_eps;
            if (tc > 1.0 - O.beta_eps) tc = 1.0 - O.beta_eps;
            if (O.lam_beta > 0.0) beta_part += log(tc) + log(1.0 - tc);
        }
    }
    if (lane == 0) {
        if (mse_part != 0.0) atomicAdd(out.sums + 0, mse_part);
        if (beta_part != 0.0) atomicAdd(out.sums + 2, beta_part);
    }
}

// K:884-977 (tv_bg): one thread per texel, its four neighbour sectors (self,
// l+1, j+1, i+1 with the phi wrap) loaded together, then the per-channel
// terms of the reference; f64.
__device__ __forceinline__ void ld_texel(const double *D, int64_t f, double (&o)[4]) {
    const double2 *p = reinterpret_cast<const double2 *>(D + 4 * f);
    const double2 a = __ldg(p), b = __ldg(p + 1);
    o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
}

__global__ void __launch_bounds__(256) msi_tv_kernel(MsiDev B, const int64_t *cells,
                                                     int64_t start, int64_t count, double eps,
                                                     double f_sigma, double f_rgb, double *grad,
                                                     uint8_t *tmask, double *sums) {
    const int64_t n = (int64_t)B.L * B.H * B.W;
    const double fl = (double)B.L / 256.0, fh = (double)B.H / 256.0, fw = (double)B.W / 256.0;
    const double e2 = eps * eps;
    const int64_t HW = (int64_t)B.H * B.W;
    double s_sig = 0.0, s_rgb = 0.0;
    for (int64_t ci = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ci < count;
         ci += (int64_t)gridDim.x * blockDim.x) {
        int64_t cid = cells ? cells[ci] : start + ci;
        if (!cells && cid >= n) cid %= n;
        const int64_t l = cid / HW, rem = cid - l * HW;
        const int64_t j = rem / B.W, i = rem - j * B.W;
        const bool hl = l + 1 < B.L, hj = j + 1 < B.H;
        const int64_t iw = i + 1 < B.W ? i + 1 : 0;
        const int64_t f0 = cid, fL = cid + HW, fJ = cid + B.W, fI = l * HW + j * B.W + iw;
        double v0[4], vl[4], vj[4], vi[4];
        ld_texel(B.data, f0, v0);
        ld_texel(B.data, fI, vi);
        if (hl) ld_texel(B.data, fL, vl);
        else { vl[0] = 0.0; vl[1] = v0[1]; vl[2] = v0[2]; vl[3] = v0[3]; }
        if (hj) ld_texel(B.data, fJ, vj);
        else { vj[0] = 0.0; vj[1] = v0[1]; vj[2] = v0[2]; vj[3] = v0[3]; }
        bool mark_l = false, mark_j = false, mark_i = false, mark_0 = false;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const double da = (vl[c] - v0[c]) * fl, db = (vj[c] - v0[c]) * fh,
                         dc = (vi[c] - v0[c]) * fw;
            const double val = sqrt(da * da + db * db + dc * dc + e2);
            if (c == 0) s_sig += val; else s_rgb += val;
            if (!grad || !(val > 0.0)) continue;
            const double inv = (c == 0 ? f_sigma : f_rgb) / val;
            double g0 = 0.0;
            if (hl) {
                mark_l = true;
                atomicAdd(grad + 4 * fL + c, da * fl * inv);
                g0 -= da * fl * inv;
            } else if (c == 0) {
                g0 -= da * fl * inv;
            }
            if (hj) {
                mark_j = true;
                atomicAdd(grad + 4 * fJ + c, db * fh * inv);
                g0 -= db * fh * inv;
            } else if (c == 0) {
                g0 -= db * fh * inv;
            }
            mark_i = true;
            atomicAdd(grad + 4 * fI + c, dc * fw * inv);
            g0 -= dc * fw * inv;
            if (g0 != 0.0) {
                mark_0 = true;
                atomicAdd(grad + 4 * f0 + c, g0);
            }
        }
        if (mark_l) tmask[fL] = 1;
        if (mark_j) tmask[fJ] = 1;
        if (mark_i) tmask[fI] = 1;
        if (mark_0) tmask[f0] = 1;
    }
    s_sig = warp_sum(s_sig);
    s_rgb = warp_sum(s_rgb);
    if ((threadIdx.x & 31) == 0) {
        if (s_sig != 0.0) atomicAdd(sums, s_sig);
        if (s_rgb != 0.0) atomicAdd(sums + 1, s_rgb);
    }
}

// O:100-107 / K:572-590 on the f64 background table over the compacted
// touched list (sorted within each 8192-texel tile), then the clear of
// K:593-600: one thread per texel, its three 32-B sectors (grad, v, table)
// loaded together.  The background's touched texels are scattered over GBs
// of f64 state, so this is a random-sector RMW; a (texel, channel) thread map
// chained the loads behind the grad clear's store and ran 4-6x slower
// (scripts/probes/texel_rmw.cu), and a mask sweep in address order (lane = 4
// texels) serialised the touched texels per lane and was slower still.
#ifndef MSI_OPT_U
#define MSI_OPT_U 2
#endif
__device__ __forceinline__ double rms_apply(double &t, double &vv, double g, double lr,
                                            double beta, double eps, int rmsprop) {
    if (g == 0.0) return t;
    if (rmsprop) {
        vv = beta * vv + (1.0 - beta) * g * g;
        t -= lr * g / (sqrt(vv) + eps);
    } else {
        t -= lr * g;
    }
    return t;
}

__global__ void __launch_bounds__(256) msi_opt_kernel(double *__restrict__ table,
                                                      double *__restrict__ v,
                                                      double *__restrict__ grad,
                                                      const int32_t *__restrict__ tids,
                                                      const int64_t *tcnt, double lr_first,
                                                      double lr_rest, double beta, double eps,
                                                      int rmsprop, int clear) {
    // MSI_OPT_U texels per thread per pass, all their sector loads issued
    // before any use (the kernel is bound by the latency of its scattered
    // sectors): 1 -> 2 took the update from 776 to 466 us on 3 M texels
    const int64_t n = *tcnt;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t0 < n; t0 += MSI_OPT_U * stride) {
        int64_t r[MSI_OPT_U];
        double2 g[MSI_OPT_U][2], tb[MSI_OPT_U][2], vv[MSI_OPT_U][2];
#pragma unroll
        for (int u = 0; u < MSI_OPT_U; ++u) {
            const int64_t t = t0 + u * stride;
            r[u] = t < n ? (int64_t)tids[t] : -1;
        }
#pragma unroll
        for (int u = 0; u < MSI_OPT_U; ++u) {
            if (r[u] < 0) continue;
            const double2 *gp = reinterpret_cast<const double2 *>(grad + 4 * r[u]);
            const double2 *tp = reinterpret_cast<const double2 *>(table + 4 * r[u]);
            g[u][0] = gp[0];
            g[u][1] = gp[1];
            tb[u][0] = tp[0];
            tb[u][1] = tp[1];
            vv[u][0] = vv[u][1] = make_double2(0.0, 0.0);
            if (rmsprop) {
                const double2 *vp = reinterpret_cast<const double2 *>(v + 4 * r[u]);
                vv[u][0] = vp[0];
                vv[u][1] = vp[1];
            }
        }
#pragma unroll
        for (int u = 0; u < MSI_OPT_U; ++u) {
            if (r[u] < 0) continue;
            if (clear) {
                double2 *gp = reinterpret_cast<double2 *>(grad + 4 * r[u]);
                gp[0] = make_double2(0.0, 0.0);
                gp[1] = gp[0];
            }
            rms_apply(tb[u][0].x, vv[u][0].x, g[u][0].x, lr_first, beta, eps, rmsprop);
            rms_apply(tb[u][0].y, vv[u][0].y, g[u][0].y, lr_rest, beta, eps, rmsprop);
            rms_apply(tb[u][1].x, vv[u][1].x, g[u][1].x, lr_rest, beta, eps, rmsprop);
            rms_apply(tb[u][1].y, vv[u][1].y, g[u][1].y, lr_rest, beta, eps, rmsprop);
            double2 *tp = reinterpret_cast<double2 *>(table + 4 * r[u]);
            tp[0] = tb[u][0];
            tp[1] = tb[u][1];
            if (rmsprop) {
                double2 *vp = reinterpret_cast<double2 *>(v + 4 * r[u]);
                vp[0] = vv[u][0];
                vp[1] = vv[u][1];
            }
        }
    }
}

constexpr int64_t kFwdScratch = 256;   // the forward kernel's ray counter

int num_sms_msi() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int msi_status() { return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA; }

}  // namespace
}  // namespace plx

using namespace plx;

extern "C" int64_t plx_msi_scratch_bytes(const plx_grid *g, const plx_msi *bg,
                                         const plx_render_opts *o, int64_t n_rays) {
    if (!g || !bg || !o || o->step <= 0.0 || n_rays < 0) return -1;
    // forward: msi_render_kernel's records; backward: the bounded render's
    const int64_t fwd = kFwdScratch;
    const int64_t bwd = plx_render_scratch_bytes(g, o, n_rays);
    if (bwd < 0) return -1;
    return fwd > bwd ? fwd : bwd;
}

extern "C" int plx_msi_render(const plx_grid *g, const plx_msi *bg, const plx_rays *rays,
                              const plx_render_opts *o, int32_t mse_mode, double up_scale,
                              double lam_cauchy, double lam_beta, double beta_eps, plx_grad *gb,
                              plx_msi_grad *bgb, double *out_rgb, double *out_tfg,
                              double *out_trans, double *out_sums, void *scratch,
                              int64_t scratch_bytes, void *stream) {
    if (!g || !bg || !rays || !o || !out_sums) return PLX_EINVAL;
    if (rays->n > 0 && (!out_rgb || !out_tfg || !out_trans || !scratch)) return PLX_EINVAL;
    if (!bg->data || !bg->radii || bg->L < 2 || bg->H < 2 || bg->W < 1 || bg->L - 1 > kMaxCross)
        return PLX_EINVAL;
    if (rays->n < 0 || o->step <= 0.0) return PLX_EINVAL;
    if (rays->cams) return PLX_EINVAL;   // array rays only (plx_generate_rays materialises a pool)
    if (rays->n > 0 && (!rays->origins || !rays->dirs || !rays->target)) return PLX_EINVAL;
    if (gb && (!gb->grad || !gb->tmask || !bgb || !bgb->grad || !bgb->tmask)) return PLX_EINVAL;
    if (rays->n == 0) return PLX_OK;
    if (gb) {
        // backward: the foreground through the bounded kernels (march,
        // colour, scatter) with the background stage (msi_bg_kernel) between
        // colour and scatter; the SH basis uses the raw ray dirs (K:699)
        plx_rays r = *rays;
        r.viewdirs = rays->dirs;
        r.jitter = nullptr;
        plx_render_opts o2 = *o;
        o2.absolute = 0;   // K:661-881 composites with the relative formula
        MsiHook h{bg->data, bg->radii, bg->L, bg->H, bg->W, lam_beta, beta_eps,
                  out_tfg, out_trans, bgb->grad, bgb->tmask};
        return plx::render_fused_bwd_impl(g, &r, nullptr, &o2, mse_mode, up_scale, lam_cauchy,
                                          gb, out_rgb, out_sums, scratch, scratch_bytes, stream,
                                          0, nullptr, &h);
    }
    if (scratch_bytes < kFwdScratch) return PLX_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    DGrid G = make_dgrid(*g);
    MsiDev B{bg->data, bg->radii, (int)bg->L, (int)bg->H, (int)bg->W};
    MsiOpts O{o->step, o->stop_thresh, mse_mode, up_scale, lam_beta, beta_eps};
    int *counter = reinterpret_cast<int *>(scratch);
    MsiRays R{rays->origins, rays->dirs, rays->target, rays->n};
    MsiOut out{out_rgb, out_tfg, out_trans, out_sums};
    if (cudaMemsetAsync(counter, 0, sizeof(int), s) != cudaSuccess) return PLX_ECUDA;
    int64_t nb = (rays->n + kMsiWarps - 1) / kMsiWarps;
    if (nb > (int64_t)num_sms_msi() * 8) nb = (int64_t)num_sms_msi() * 8;
    if (o->nearest)
        msi_fwd_kernel<true><<<(unsigned)nb, kMsiThreads, 0, s>>>(G, B, R, O, out, counter);
    else
        msi_fwd_kernel<false><<<(unsigned)nb, kMsiThreads, 0, s>>>(G, B, R, O, out, counter);
    return msi_status();
}

extern "C" int plx_msi_tv(const plx_msi *bg, const int64_t *cells, int64_t start, int64_t count,
                          double eps, double f_sigma, double f_rgb, plx_msi_grad *bgb,
                          double *out_sums, void *stream) {
    if (!bg || !bg->data || !out_sums || count < 0 || bg->L < 1 || bg->H < 1 || bg->W < 1)
        return PLX_EINVAL;
    if (bgb && (!bgb->grad || !bgb->tmask)) return PLX_EINVAL;
    if (count == 0) return PLX_OK;
    MsiDev B{bg->data, bg->radii, (int)bg->L, (int)bg->H, (int)bg->W};
    int64_t nb = (count + 255) / 256;
    if (nb > (int64_t)num_sms_msi() * 8) nb = (int64_t)num_sms_msi() * 8;
    msi_tv_kernel<<<(unsigned)nb, 256, 0, (cudaStream_t)stream>>>(
        B, cells, start, count, eps, f_sigma, f_rgb, bgb ? bgb->grad : nullptr,
        bgb ? bgb->tmask : nullptr, out_sums);
    return msi_status();
}

extern "C" int plx_msi_opt_step(double *table, double *v, plx_msi_grad *bgb, int64_t n_texels,
                                double lr_sigma, double lr_rgb, double beta, double eps,
                                int32_t rmsprop, int32_t clear, int64_t *out_count,
                                void *stream) {
    if (!table || !bgb || !bgb->grad || !bgb->tmask || !bgb->tids || !bgb->tcnt ||
        (rmsprop && !v) || n_texels < 0)
        return PLX_EINVAL;
    if (n_texels == 0) return PLX_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (n_texels > INT32_MAX) return PLX_EINVAL;
    const int rc = plx::compact_mask_impl(bgb->tmask, n_texels, bgb->tids, bgb->tcnt, clear,
                                          stream);
    if (rc != PLX_OK) return rc;
    int64_t nb = (n_texels + 255) / 256;
    if (nb > (int64_t)num_sms_msi() * 8) nb = (int64_t)num_sms_msi() * 8;
    msi_opt_kernel<<<(unsigned)nb, 256, 0, s>>>(table, v, bgb->grad, bgb->tids, bgb->tcnt,
                                                lr_sigma, lr_rgb, beta, eps, rmsprop, clear);
    if (out_count && cudaMemcpyAsync(out_count, bgb->tcnt, sizeof(int64_t),
                                     cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return PLX_ECUDA;
    return msi_status();
}
