// plx_msi.cu -- multi-sphere-image background for unbounded 360 scenes
// (reference K:603-977 render_backward_360 / tv_bg, msi.py, O:100-107
// step_table).  Concentric equirectangular layers of f64 (sigma, r, g, b)
// texels beyond the foreground grid; a ray samples the grid exactly as the
// bounded render does, then the layers once per sphere crossing past the
// grid's exit, composited over black; the backward sweeps the concatenated
// samples in reverse.
//
// Device layout: background f64 [L][H][W][4]; its gradient f64 [L*H*W][4]
// with a byte mask (the reference's BgGradientBuffer); the grid side reuses
// plx_grid / plx_grad.  Per-ray records (t, delta, sigma, T, w, colour,
// layer) live in a caller-provided scratch, one block of `cap` records per
// ray, processed in waves that fit the scratch.
#include <cuda_runtime.h>

#include "plx_common.cuh"
#include "plx_internal.h"

namespace plx {
namespace {

constexpr int kMsiThreads = 128;
constexpr int kMsiWarps = kMsiThreads / 32;
constexpr int kMaxCross = 256;   // sphere crossings per ray (layers - 1)

struct MsiDev {
    const double *data;   // [L][H][W][4]
    const double *radii;  // [L]
    int L, H, W;
};

struct MsiRays {
    const double *origins, *dirs, *target;
    int64_t n;
};

struct MsiOpts {
    double step, stop;
    int mse_mode;
    double up_scale, lam_cauchy, lam_beta, beta_eps;
};

struct MsiOut {
    double *rgb, *tfg, *trans, *sums;   // sums: {mse, cauchy_raw, beta_raw}
    float *grad;                        // grid gradient rows (pitch PLX_STRIDE), or null
    uint8_t *tmask;
    double *bg_grad;                    // [L*H*W][4]
    uint8_t *bg_tmask;
};

struct MsiRec {
    int *counter;
    int64_t cap;
    double *t, *dlt, *sig, *T, *w;
    double4 *c;   // colour (pre-clamp), .w unused
    int *lay;     // -1 foreground, else the layer
};

// K:606-645 (_bg_stencil): bilinear texel stencil within one layer at the
// sphere angles of p; texel centres at half texels, phi wraps, theta clamps.
__device__ __forceinline__ void bg_stencil(int H, int W, double px, double py, double pz,
                                           int *idx4, double *w4) {
    const double pi = 3.141592653589793;
    const double r = sqrt(px * px + py * py + pz * pz);
    const double phi = atan2(py, px);
    double ct = pz / r;
    if (ct > 1.0) ct = 1.0;
    if (ct < -1.0) ct = -1.0;
    const double theta = acos(ct);
    double u = (phi + pi) / (2.0 * pi) * (double)W - 0.5;
    u = u - floor(u / (double)W) * (double)W;
    double vv = theta / pi * (double)H - 0.5;
    if (vv < 0.0) vv = 0.0;
    if (vv > (double)H - 1.0) vv = (double)H - 1.0;
    int i0 = (int)u;
    if (i0 > W - 1) i0 = W - 1;
    const double fu = u - (double)i0;
    int i1 = i0 + 1;
    if (i1 >= W) i1 = 0;
    int j0 = (int)vv;
    if (j0 > H - 2) j0 = H - 2;
    const double fv = vv - (double)j0;
    idx4[0] = j0 * W + i0;
    idx4[1] = j0 * W + i1;
    idx4[2] = (j0 + 1) * W + i0;
    idx4[3] = (j0 + 1) * W + i1;
    w4[0] = (1.0 - fu) * (1.0 - fv);
    w4[1] = fu * (1.0 - fv);
    w4[2] = (1.0 - fu) * fv;
    w4[3] = fu * fv;
}

// K:648-658 (_bg_fetch): texel-major accumulation of the 4 channels.
__device__ __forceinline__ void bg_fetch(const MsiDev &B, int layer, const int *idx4,
                                         const double *w4, double *out4) {
    out4[0] = out4[1] = out4[2] = out4[3] = 0.0;
    const double4 *base = reinterpret_cast<const double4 *>(B.data) + (int64_t)layer * B.H * B.W;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const double2 *tp = reinterpret_cast<const double2 *>(base + idx4[q]);
        const double2 ta = __ldg(tp), tb = __ldg(tp + 1);
        const double4 tx = make_double4(ta.x, ta.y, tb.x, tb.y);
        out4[0] += w4[q] * tx.x;
        out4[1] += w4[q] * tx.y;
        out4[2] += w4[q] * tx.z;
        out4[3] += w4[q] * tx.w;
    }
}

// Grid rows + trilinear fractions of the position at lattice coordinates g
// (the stencil of K:84-123 recomputed for the scatter, as K:818-821 does).
template <bool NEAREST>
__device__ __forceinline__ void stencil_rows(const DGrid &G, const double *g, int32_t *rows,
                                             double *f) {
    int ijk[3];
    if (NEAREST) {
        int64_t i = (int64_t)(g[0] + 0.5), j = (int64_t)(g[1] + 0.5), k = (int64_t)(g[2] + 0.5);
        if (i > G.Dx - 1) i = G.Dx - 1;
        if (j > G.Dy - 1) j = G.Dy - 1;
        if (k > G.Dz - 1) k = G.Dz - 1;
        ijk[0] = (int)i;
        ijk[1] = (int)j;
        ijk[2] = (int)k;
    } else {
        int64_t i0 = (int64_t)g[0], j0 = (int64_t)g[1], k0 = (int64_t)g[2];
        if (i0 > G.Dx - 2) i0 = G.Dx - 2;
        if (j0 > G.Dy - 2) j0 = G.Dy - 2;
        if (k0 > G.Dz - 2) k0 = G.Dz - 2;
        ijk[0] = (int)i0;
        ijk[1] = (int)j0;
        ijk[2] = (int)k0;
        f[0] = g[0] - (double)i0;
        f[1] = g[1] - (double)j0;
        f[2] = g[2] - (double)k0;
    }
    load_rows<NEAREST>(G, ijk, rows);
}

// One warp per ray (rays from a device counter).  Foreground: 32 march
// positions per step as in the bounded backward (f64 positions, stencil and
// sigma; f32 colour), composited with the warp product scan.  Background:
// the sphere crossings (lane = layer) compacted in layer order into shared
// memory, then sampled and composited 32 at a time.  Backward: records in
// reverse chunks, the suffix sums S_i = sum_{j>i} w_j ReLU(c_j) per chunk by
// a warp scan plus the carry (K:780-800), the grid scatter with red.v4 and
// the texel scatter with f64 atomics.
#ifndef MSI_MINB
#define MSI_MINB 4
#endif
template <bool NEAREST>
__global__ void __launch_bounds__(kMsiThreads, MSI_MINB)
    msi_render_kernel(DGrid G, MsiDev B, MsiRays R, MsiOpts O, MsiOut out, MsiRec S) {
    __shared__ double xs_t_all[kMsiWarps][kMaxCross];
    __shared__ int xs_l_all[kMsiWarps][kMaxCross];
    // backward staging of the foreground scatter: per fg sample (dense slot)
    // and corner, the row and (w gsig, w gc_r, w gc_g, w gc_b) in f64
    constexpr int NQS = NEAREST ? 1 : 8;
    __shared__ int32_t st_row_all[kMsiWarps][32 * NQS];
    __shared__ double4 st_val_all[kMsiWarps][32 * NQS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t *st_row = st_row_all[warp];
    double4 *st_val = st_val_all[warp];
    // this lane's float4 of a 28-float row in the cooperative scatter
    const int su = lane % 7, spair = lane / 7;
    double *xs_t = xs_t_all[warp];
    int *xs_l = xs_l_all[warp];
    const unsigned lt = (1u << lane) - 1u;
    const bool with_grad = out.grad != nullptr;
    double mse_part = 0.0, cau_part = 0.0, beta_part = 0.0;
    for (;;) {
        int rr = 0;
        if (lane == 0) rr = atomicAdd(S.counter, 1);
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
        // coefficient e = 4 su + j of the row: 0 sigma, 1-9 R, 10-18 G, 19-27 B
        double sb[4];
        int sk[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int e = 4 * su + j;
            sk[j] = e == 0 ? 0 : 1 + (e - 1) / 9;
            const int bi = e == 0 ? 0 : (e - 1) % 9;
            double bv = basis[0];
#pragma unroll
            for (int b = 1; b < 9; ++b)
                if (bi == b) bv = basis[b];
            sb[j] = bv;
        }
        double t0a, t1a;
        ray_aabb(rm.o, rm.d, G.lo, G.hi, t0a, t1a);
        ray_march_setup(rm, G, O.step, 0.0);
        const int64_t rb = ray * S.cap;
        double T = 1.0, A = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
        int m = 0;
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
            const unsigned msk = __ballot_sync(PLX_FULL_MASK, incl);
            if (incl) {
                if (!rows_ok) load_rows<NEAREST>(G, ijk, rows);
                float c[3];
                colour_at_f32<NEAREST>(G, rows, fd, bf, c);
                const int64_t k = rb + m + __popc(msk & lt);
                S.t[k] = t;
                S.dlt[k] = dlt;
                S.sig[k] = sig;
                S.T[k] = Ti;
                S.w[k] = wi;
                S.c[k] = make_double4(c[0], c[1], c[2], 0.0);
                S.lay[k] = -1;
                if (c[0] > 0.f) c0 += wi * (double)c[0];
                if (c[1] > 0.f) c1 += wi * (double)c[1];
                if (c[2] > 0.f) c2 += wi * (double)c[2];
            }
            m += __popc(msk);
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
                double att = 1.0, sig = 0.0, t = 0.0, dlt = 0.0, o4[4] = {0.0, 0.0, 0.0, 0.0};
                int lay = 0;
                if (q < nx) {
                    if (q + 1 < nx) dlt = xs_t[q + 1] - xs_t[q];
                    else if (q >= 1) dlt = xs_t[q] - xs_t[q - 1];
                    else dlt = 1.0;
                    t = xs_t[q];
                    lay = xs_l[q];
                    int idx4[4];
                    double w4[4];
                    bg_stencil(B.H, B.W, rm.o[0] + t * rm.d[0], rm.o[1] + t * rm.d[1],
                               rm.o[2] + t * rm.d[2], idx4, w4);
                    bg_fetch(B, lay, idx4, w4, o4);
                    sig = o4[0];
                    incl = sig >= 0.0;
                    if (incl) att = exp(-sig * dlt);
                }
                if (!__any_sync(PLX_FULL_MASK, incl)) continue;
                double Ti, wi;
                composite_chunk<false>(incl, att, lane, O.stop, T, A, Ti, wi, stopped);
                const unsigned msk = __ballot_sync(PLX_FULL_MASK, incl);
                if (incl) {
                    const int64_t k = rb + m + __popc(msk & lt);
                    S.t[k] = t;
                    S.dlt[k] = dlt;
                    S.sig[k] = sig;
                    S.T[k] = Ti;
                    S.w[k] = wi;
                    S.c[k] = make_double4(o4[1], o4[2], o4[3], 0.0);
                    S.lay[k] = lay;
                    if (o4[1] > 0.0) c0 += wi * o4[1];
                    if (o4[2] > 0.0) c1 += wi * o4[2];
                    if (o4[3] > 0.0) c2 += wi * o4[3];
                }
                m += __popc(msk);
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
        }
        // ---- upstream, beta regulariser (K:808-833) ----
        double up0, up1, up2;
        if (O.mse_mode) {
            const double e0 = cr - __ldg(R.target + 3 * ray), e1 = cg - __ldg(R.target + 3 * ray + 1),
                         e2 = cb - __ldg(R.target + 3 * ray + 2);
            if (lane == 0) mse_part += e0 * e0 + e1 * e1 + e2 * e2;
            up0 = O.up_scale * e0;
            up1 = O.up_scale * e1;
            up2 = O.up_scale * e2;
        } else {
            up0 = __ldg(R.target + 3 * ray);
            up1 = __ldg(R.target + 3 * ray + 1);
            up2 = __ldg(R.target + 3 * ray + 2);
        }
        double tc = tfg;
        if (tc < O.beta_eps) tc = O.beta_eps;
        if (tc > 1.0 - O.beta_eps) tc = 1.0 - O.beta_eps;
        if (O.lam_beta > 0.0 && lane == 0) beta_part += log(tc) + log(1.0 - tc);
        double bup = 0.0;
        if (O.lam_beta > 0.0 && O.beta_eps < tfg && tfg < 1.0 - O.beta_eps)
            bup = O.lam_beta * (1.0 / tc - 1.0 / (1.0 - tc));
        if (!with_grad) continue;
        // ---- reverse sweep + scatter (K:835-881) ----
        double sf0 = 0.0, sf1 = 0.0, sf2 = 0.0;   // suffix carry over later chunks
        for (int cb0 = ((m - 1) >> 5) << 5; cb0 >= 0; cb0 -= 32) {
            const int idx = cb0 + lane;
            const bool valid = idx < m;
            const int64_t k = rb + idx;
            double sig = 0.0, dlt = 0.0, Ti = 0.0, w = 0.0, t = 0.0;
            double4 c = make_double4(0.0, 0.0, 0.0, 0.0);
            int lay = -1;
            if (valid) {
                sig = S.sig[k];
                dlt = S.dlt[k];
                Ti = S.T[k];
                w = S.w[k];
                t = S.t[k];
                c = S.c[k];
                lay = S.lay[k];
            }
            const double cc0 = c.x > 0.0 ? c.x : 0.0, cc1 = c.y > 0.0 ? c.y : 0.0,
                         cc2 = c.z > 0.0 ? c.z : 0.0;
            const double y0 = valid ? w * cc0 : 0.0, y1 = valid ? w * cc1 : 0.0,
                         y2 = valid ? w * cc2 : 0.0;
            // S_i = carry + sum over later lanes of this chunk
            const double i0 = warp_scan_add(y0, lane), i1 = warp_scan_add(y1, lane),
                         i2 = warp_scan_add(y2, lane);
            const double tot0 = __shfl_sync(PLX_FULL_MASK, i0, 31),
                         tot1 = __shfl_sync(PLX_FULL_MASK, i1, 31),
                         tot2 = __shfl_sync(PLX_FULL_MASK, i2, 31);
            const double s0 = sf0 + (tot0 - i0), s1 = sf1 + (tot1 - i1), s2 = sf2 + (tot2 - i2);
            sf0 += tot0;
            sf1 += tot1;
            sf2 += tot2;
            const bool fg = valid && lay < 0;
            const unsigned fgm = __ballot_sync(PLX_FULL_MASK, fg);
            if (valid) {
                const double att = exp(-sig * dlt);
                double gsig = dlt * (up0 * (Ti * att * cc0 - s0) + up1 * (Ti * att * cc1 - s1) +
                                     up2 * (Ti * att * cc2 - s2));
                if (fg) {
                    if (O.lam_cauchy > 0.0) {
                        cau_part += log(1.0 + 2.0 * sig * sig);
                        gsig += O.lam_cauchy * 4.0 * sig / (1.0 + 2.0 * sig * sig);
                    }
                    if (bup != 0.0) gsig += bup * (-dlt * tfg);
                    const double gc0 = c.x > 0.0 ? up0 * w : 0.0,
                                 gc1 = c.y > 0.0 ? up1 * w : 0.0,
                                 gc2 = c.z > 0.0 ? up2 * w : 0.0;
                    double g[3], f[3] = {0.0, 0.0, 0.0};
#pragma unroll
                    for (int a = 0; a < 3; ++a)
                        g[a] = clamp_coord(rm.o[a] + t * rm.d[a], G.lo[a], G.scale[a],
                                           G.dmax[a]);
                    int32_t rows[8];
                    stencil_rows<NEAREST>(G, g, rows, f);
                    const int slot = __popc(fgm & lt) * NQS;
#pragma unroll
                    for (int q = 0; q < NQS; ++q) {
                        const int32_t r = rows[q];
                        st_row[slot + q] = r;
                        if (r < 0) continue;
                        const double wq = stencil_w<NEAREST>(f, q);
                        out.tmask[r] = 1;
                        st_val[slot + q] = make_double4(wq * gsig, wq * gc0, wq * gc1, wq * gc2);
                    }
                } else {
                    int idx4[4];
                    double w4[4];
                    bg_stencil(B.H, B.W, rm.o[0] + t * rm.d[0], rm.o[1] + t * rm.d[1],
                               rm.o[2] + t * rm.d[2], idx4, w4);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int64_t flat = (int64_t)lay * B.H * B.W + idx4[q];
                        const double wq = w4[q];
                        out.bg_tmask[flat] = 1;
                        double *gb = out.bg_grad + 4 * flat;
                        atomicAdd(gb, wq * gsig);
                        if (c.x > 0.0) atomicAdd(gb + 1, wq * up0 * w);
                        if (c.y > 0.0) atomicAdd(gb + 2, wq * up1 * w);
                        if (c.z > 0.0) atomicAdd(gb + 3, wq * up2 * w);
                    }
                }
            }
            __syncwarp();
            // warp-cooperative scatter: 4 (sample, corner) rows per pass, lane
            // = one float4 of a row, so each red.v4 instruction covers whole
            // 112-B rows instead of 32 scattered 16-B pieces
            const int npairs = __popc(fgm) * NQS;
            if (lane < 28) {
                for (int pidx = spair; pidx < npairs; pidx += 4) {
                    const int32_t r = st_row[pidx];
                    if (r < 0) continue;
                    const double4 sv = st_val[pidx];
                    float v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double a = sk[j] == 0 ? sv.x : sk[j] == 1 ? sv.y : sk[j] == 2 ? sv.z : sv.w;
                        v[j] = sk[j] == 0 ? (float)a : (float)(a * sb[j]);
                    }
                    if (v[0] != 0.f || v[1] != 0.f || v[2] != 0.f || v[3] != 0.f)
                        red_add_v4(out.grad + (int64_t)r * PLX_STRIDE + 4 * su, v[0], v[1], v[2],
                                   v[3]);
                }
            }
            __syncwarp();
        }
    }
    mse_part = warp_sum(mse_part);
    cau_part = warp_sum(cau_part);
    beta_part = warp_sum(beta_part);
    if (lane == 0) {
        if (mse_part != 0.0) atomicAdd(out.sums + 0, mse_part);
        if (cau_part != 0.0) atomicAdd(out.sums + 1, cau_part);
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

constexpr int64_t kRecBytes = 5 * 8 + 32 + 4;   // t, delta, sigma, T, w; colour; layer
constexpr int64_t kRecHeader = 256 + 64;          // counter + alignment slack

struct MsiLayout {
    int64_t cap, wave, bytes;
};

MsiLayout msi_layout(const plx_grid *g, const plx_msi *bg, const plx_render_opts *o,
                     int64_t n_rays) {
    MsiLayout L{};
    double ext2 = 0.0;
    for (int a = 0; a < 3; ++a) ext2 += (g->hi[a] - g->lo[a]) * (g->hi[a] - g->lo[a]);
    // R:67-69 + layers + 2 (msi.py:162)
    L.cap = (int64_t)ceil(sqrt(ext2) / o->step) + 4 + bg->L + 2;
    const int64_t per_ray = L.cap * kRecBytes;
    const int64_t budget = (int64_t)4 << 30;
    L.wave = n_rays;
    if (L.wave * per_ray > budget) L.wave = budget / per_ray > 0 ? budget / per_ray : 1;
    L.bytes = kRecHeader + L.wave * per_ray;
    return L;
}

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
    return msi_layout(g, bg, o, n_rays).bytes;
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
    const MsiLayout L = msi_layout(g, bg, o, rays->n);
    if (scratch_bytes < kRecHeader + L.cap * kRecBytes) return PLX_EINVAL;
    int64_t wave = (scratch_bytes - kRecHeader) / (L.cap * kRecBytes);
    if (wave > rays->n) wave = rays->n;
    cudaStream_t s = (cudaStream_t)stream;
    DGrid G = make_dgrid(*g);
    MsiDev B{bg->data, bg->radii, (int)bg->L, (int)bg->H, (int)bg->W};
    MsiOpts O{o->step, o->stop_thresh, mse_mode, up_scale, lam_cauchy, lam_beta, beta_eps};
    char *base = reinterpret_cast<char *>(scratch);
    MsiRec S;
    S.counter = reinterpret_cast<int *>(base);
    S.cap = L.cap;
    char *p = base + 256;
    const int64_t nrec = wave * L.cap;
    S.t = reinterpret_cast<double *>(p);
    S.dlt = S.t + nrec;
    S.sig = S.dlt + nrec;
    S.T = S.sig + nrec;
    S.w = S.T + nrec;
    uintptr_t pc = reinterpret_cast<uintptr_t>(S.w + nrec);
    pc = (pc + 31) & ~(uintptr_t)31;   // double4 needs 32-byte alignment
    S.c = reinterpret_cast<double4 *>(pc);
    S.lay = reinterpret_cast<int *>(S.c + nrec);
    for (int64_t w0 = 0; w0 < rays->n; w0 += wave) {
        const int64_t nw = rays->n - w0 < wave ? rays->n - w0 : wave;
        MsiRays R{rays->origins + 3 * w0, rays->dirs + 3 * w0, rays->target + 3 * w0, nw};
        MsiOut out{out_rgb + 3 * w0, out_tfg + w0, out_trans + w0, out_sums,
                   gb ? gb->grad : nullptr, gb ? gb->tmask : nullptr,
                   gb ? bgb->grad : nullptr, gb ? bgb->tmask : nullptr};
        if (cudaMemsetAsync(S.counter, 0, sizeof(int), s) != cudaSuccess) return PLX_ECUDA;
        int64_t nb = (nw + kMsiWarps - 1) / kMsiWarps;
        if (nb > (int64_t)num_sms_msi() * 8) nb = (int64_t)num_sms_msi() * 8;
        if (o->nearest)
            msi_render_kernel<true><<<(unsigned)nb, kMsiThreads, 0, s>>>(G, B, R, O, out, S);
        else
            msi_render_kernel<false><<<(unsigned)nb, kMsiThreads, 0, s>>>(G, B, R, O, out, S);
    }
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
