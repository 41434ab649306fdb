// plx_render.cu -- ray-march kernels for sm_100a: forward render, the fused
// forward + MSE + backward scatter, and the max-weight accumulation.
//
// Reference: pkg/src/plenoxel/_kernels.py render_forward (K:173-238),
// render_backward (K:241-411), max_weight_accum (K:414-453).
//
// Parallel decomposition (B200-first, not a translation of the sequential
// loop): one warp per ray, one lane per march position.  A ray is walked in
// chunks of 32 consecutive positions: every lane evaluates its own sample
// (stencil through `links`, float64 trilinear sigma and SH colour from f32
// rows gathered as float4), then the chunk is composited with warp scans
// (product scan of exp(-sigma*delta) for "relative", sum scan of alpha for
// "absolute"), early termination is a ballot on T < stop_thresh (T is
// monotone, so the first such lane is the reference's break point).
//
// The backward replays the march a second time instead of storing per-sample
// records: the reference's reverse suffix sum S_i = sum_{j>i} w_j c_j + T bg
// equals (rgb - prefix_i) and is formed in float64, where the cancellation is
// harmless (|error| ~ 1e-16 |rgb|).  Gradients are scattered with vector
// f32 reductions (red.global.add.v4.f32, 7 per stencil row).
#include "plx_common.cuh"

namespace plx {

enum Mode { FWD = 0, BWD = 1, MAXW = 2 };

struct RayArgs {
    const double *__restrict__ origins;
    const double *__restrict__ dirs;
    const double *__restrict__ viewdirs;
    const double *__restrict__ target;
    const double *__restrict__ jitter;
    const int64_t *__restrict__ idx;
    int64_t n;
};

struct KOpts {
    double step, stop, bg[3];
};

struct Outs {
    double *rgb, *trans, *wsum;   // FWD / BWD(rgb)
    double *sums;                 // BWD: {mse, cauchy}
    double *maxw;                 // MAXW
    float *grad;
    uint8_t *tmask;
    int mse_mode;
    double up_scale, lam_cauchy;
};

// One march position evaluated by one lane.
struct Sample {
    int32_t rows[8];
    double ws[8];
    double sig, att, dlt;
    double c[3];   // pre-clamp colour (K:305)
    bool incl;
};

// Evaluate position si (K:286-305): stencil, sigma, and for included samples
// the colour.  FWD/MAXW include sigma > 0, BWD sigma >= 0 (K:211 vs K:293).
template <int MODE, bool NEAREST>
__device__ __forceinline__ void eval_sample(const DGrid &G, const RayMarch &rm, double step,
                                            int64_t si, const double *basis, Sample &s) {
    s.incl = false;
    if (si >= rm.nsamp) return;
    double t, g[3];
    sample_coords(rm, G, step, si, t, s.dlt, g);
    bool occ;
    constexpr int NQ = NEAREST ? 1 : 8;
    stencil<NEAREST>(G, g, s.rows, s.ws, occ);
    if (!occ) return;
    // _sigma_at (K:126-135): float64 sum over occupied corners in order.
    double sig = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        int32_t r = s.rows[q];
        if (r >= 0) sig += s.ws[q] * (double)__ldg(G.table + (int64_t)r * PLX_ROW);
    }
    s.sig = sig;
    if (MODE == BWD ? !(sig >= 0.0) : !(sig > 0.0)) return;
    s.incl = true;
    s.att = exp(-sig * s.dlt);
    if (MODE == MAXW) return;
    // _color_at (K:138-152): per corner the 3 SH dots, then weight.
    double c0 = 0.0, c1 = 0.0, c2 = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        int32_t r = s.rows[q];
        if (r < 0) continue;
        const float4 *row = reinterpret_cast<const float4 *>(G.table + (int64_t)r * PLX_ROW);
        float4 v0 = __ldg(row + 0), v1 = __ldg(row + 1), v2 = __ldg(row + 2), v3 = __ldg(row + 3);
        float4 v4 = __ldg(row + 4), v5 = __ldg(row + 5), v6 = __ldg(row + 6);
        // row layout: [sig, R0..R8, G0..G8, B0..B8]
        double a0 = 0.0, a1 = 0.0, a2 = 0.0;
        a0 += basis[0] * (double)v0.y;
        a0 += basis[1] * (double)v0.z;
        a0 += basis[2] * (double)v0.w;
        a0 += basis[3] * (double)v1.x;
        a0 += basis[4] * (double)v1.y;
        a0 += basis[5] * (double)v1.z;
        a0 += basis[6] * (double)v1.w;
        a0 += basis[7] * (double)v2.x;
        a0 += basis[8] * (double)v2.y;
        a1 += basis[0] * (double)v2.z;
        a1 += basis[1] * (double)v2.w;
        a1 += basis[2] * (double)v3.x;
        a1 += basis[3] * (double)v3.y;
        a1 += basis[4] * (double)v3.z;
        a1 += basis[5] * (double)v3.w;
        a1 += basis[6] * (double)v4.x;
        a1 += basis[7] * (double)v4.y;
        a1 += basis[8] * (double)v4.z;
        a2 += basis[0] * (double)v4.w;
        a2 += basis[1] * (double)v5.x;
        a2 += basis[2] * (double)v5.y;
        a2 += basis[3] * (double)v5.z;
        a2 += basis[4] * (double)v5.w;
        a2 += basis[5] * (double)v6.x;
        a2 += basis[6] * (double)v6.y;
        a2 += basis[7] * (double)v6.z;
        a2 += basis[8] * (double)v6.w;
        double w = s.ws[q];
        c0 += w * a0;
        c1 += w * a1;
        c2 += w * a2;
    }
    s.c[0] = c0;
    s.c[1] = c1;
    s.c[2] = c2;
}

// Composite one chunk (K:213-233).  In: carry (T for relative, asum for
// absolute), incl flags.  Out: per-lane T_i and w_i (valid on included
// lanes; included lanes past the early stop are dropped), updated carry,
// `stopped` (warp-uniform).
template <bool ABS>
__device__ __forceinline__ void composite_chunk(Sample &s, int lane, double stop,
                                                double &Tcarry, double &Acarry, double &Ti,
                                                double &wi, bool &stopped) {
    double Tn;
    if (!ABS) {
        double a = s.incl ? s.att : 1.0;
        double pinc = warp_scan_mul(a, lane);
        double pexc = __shfl_up_sync(PLX_FULL_MASK, pinc, 1);
        if (lane == 0) pexc = 1.0;
        Ti = Tcarry * pexc;
        Tn = Tcarry * pinc;
    } else {
        double v = s.incl ? 1.0 - s.att : 0.0;
        double sinc = warp_scan_add(v, lane);
        double sexc = __shfl_up_sync(PLX_FULL_MASK, sinc, 1);
        if (lane == 0) sexc = 0.0;
        double before = Acarry + sexc;
        Ti = 1.0 - before;
        if (Ti < 0.0) Ti = 0.0;
        Tn = 1.0 - (before + v);
        if (Tn < 0.0) Tn = 0.0;
        Acarry = before + v;   // lane-local; broadcast below
    }
    wi = Ti - Tn;
    unsigned stopm = __ballot_sync(PLX_FULL_MASK, s.incl && Tn < stop);
    int last = 31;
    if (stopm) {
        last = __ffs(stopm) - 1;
        stopped = true;
        if (lane > last) s.incl = false;
    }
    Tcarry = __shfl_sync(PLX_FULL_MASK, Tn, last);
    if (ABS) Acarry = __shfl_sync(PLX_FULL_MASK, Acarry, last);
}

__device__ __forceinline__ double relu(double x) { return x > 0.0 ? x : 0.0; }

template <int MODE, bool ABS, bool NEAREST>
__global__ void __launch_bounds__(256) march_kernel(DGrid G, RayArgs R, KOpts O, Outs out) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t ray = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    __shared__ double red_mse[8], red_cau[8];
    double mse_part = 0.0, cau_part = 0.0;

    if (ray < R.n) {
        const int64_t src = R.idx ? R.idx[ray] : ray;
        RayMarch rm;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            rm.o[a] = __ldg(R.origins + 3 * src + a);
            rm.d[a] = __ldg(R.dirs + 3 * src + a);
        }
        double basis[9];
        if (MODE != MAXW)
            sh_basis9(__ldg(R.viewdirs + 3 * src), __ldg(R.viewdirs + 3 * src + 1),
                      __ldg(R.viewdirs + 3 * src + 2), basis);
        const double jit = (MODE != MAXW && R.jitter) ? R.jitter[ray] : 0.0;
        ray_march_setup(rm, G, O.step, jit);

        // ---------------- pass 1: forward ----------------
        double T = 1.0, A = 0.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, wsum = 0.0;
        double Q0 = 0.0, Q1 = 0.0, Q2 = 0.0;   // absolute backward: sum c(bn - bi)
        bool stopped = false;
        for (int64_t base = 0; base < rm.nsamp && !stopped; base += 32) {
            Sample s;
            eval_sample<MODE, NEAREST>(G, rm, O.step, base + lane, basis, s);
            if (!__any_sync(PLX_FULL_MASK, s.incl)) continue;
            double Ti, wi;
            composite_chunk<(MODE == MAXW ? false : ABS)>(s, lane, O.stop, T, A, Ti, wi, stopped);
            if (MODE == MAXW) {
                if (s.incl) {
                    double w = Ti * (1.0 - s.att);   // K:446
                    constexpr int NQ = NEAREST ? 1 : 8;
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        int32_t r = s.rows[q];
                        if (r >= 0)
                            atomicMax(reinterpret_cast<unsigned long long *>(out.maxw) + r,
                                      (unsigned long long)__double_as_longlong(w));
                    }
                }
                continue;
            }
            double x0 = 0.0, x1 = 0.0, x2 = 0.0, xw = 0.0;
            if (s.incl) {
                x0 = wi * relu(s.c[0]);
                x1 = wi * relu(s.c[1]);
                x2 = wi * relu(s.c[2]);
                xw = wi;
                if (MODE == BWD && ABS) {
                    double bn = (Ti - wi) > 0.0 ? 1.0 : 0.0, bi = Ti > 0.0 ? 1.0 : 0.0;
                    Q0 += relu(s.c[0]) * (bn - bi);
                    Q1 += relu(s.c[1]) * (bn - bi);
                    Q2 += relu(s.c[2]) * (bn - bi);
                }
            }
            C0 += warp_sum(x0);
            C1 += warp_sum(x1);
            C2 += warp_sum(x2);
            if (MODE == FWD) wsum += warp_sum(xw);
        }
        if (MODE == MAXW) goto done;
        {
            const double rgb0 = C0 + T * O.bg[0], rgb1 = C1 + T * O.bg[1], rgb2 = C2 + T * O.bg[2];
            if (lane == 0 && out.rgb) {
                out.rgb[3 * ray + 0] = rgb0;
                out.rgb[3 * ray + 1] = rgb1;
                out.rgb[3 * ray + 2] = rgb2;
            }
            if (MODE == FWD) {
                if (lane == 0) {
                    if (out.trans) out.trans[ray] = T;
                    if (out.wsum) out.wsum[ray] = wsum;
                }
                goto done;
            }
            // ---------------- upstream (K:330-341) ----------------
            double up0, up1, up2;
            if (out.mse_mode) {
                const double e0 = rgb0 - __ldg(R.target + 3 * src + 0);
                const double e1 = rgb1 - __ldg(R.target + 3 * src + 1);
                const double e2 = rgb2 - __ldg(R.target + 3 * src + 2);
                mse_part = e0 * e0 + e1 * e1 + e2 * e2;
                up0 = out.up_scale * e0;
                up1 = out.up_scale * e1;
                up2 = out.up_scale * e2;
            } else {
                up0 = __ldg(R.target + 3 * src + 0);
                up1 = __ldg(R.target + 3 * src + 1);
                up2 = __ldg(R.target + 3 * src + 2);
            }
            if (ABS) {   // sum over all lanes of the per-lane Q partials
                Q0 = warp_sum(Q0);
                Q1 = warp_sum(Q1);
                Q2 = warp_sum(Q2);
            }
            // sf before processing sample i in the reference's reverse sweep:
            //   relative: T bg + sum_{j>i} w_j c_j = rgb - P_i      (K:351-353, 381-383)
            //   absolute: -bg [T>0] + sum_{j>i} c_j (bn_j - bi_j)   (K:346-349, 374-376)
            const double bend = T > 0.0 ? 1.0 : 0.0;
            double P0 = 0.0, P1 = 0.0, P2 = 0.0;   // running prefix (carry)
            double T2 = 1.0, A2 = 0.0;
            bool stopped2 = false;
            for (int64_t base = 0; base < rm.nsamp && !stopped2; base += 32) {
                Sample s;
                eval_sample<MODE, NEAREST>(G, rm, O.step, base + lane, basis, s);
                if (!__any_sync(PLX_FULL_MASK, s.incl)) continue;
                double Ti, wi;
                composite_chunk<ABS>(s, lane, O.stop, T2, A2, Ti, wi, stopped2);
                const double cc0 = relu(s.c[0]), cc1 = relu(s.c[1]), cc2 = relu(s.c[2]);
                double gsig = 0.0;
                if (!ABS) {
                    double y0 = s.incl ? wi * cc0 : 0.0, y1 = s.incl ? wi * cc1 : 0.0,
                           y2 = s.incl ? wi * cc2 : 0.0;
                    double i0 = P0 + warp_scan_add(y0, lane), i1 = P1 + warp_scan_add(y1, lane),
                           i2 = P2 + warp_scan_add(y2, lane);
                    P0 = __shfl_sync(PLX_FULL_MASK, i0, 31);
                    P1 = __shfl_sync(PLX_FULL_MASK, i1, 31);
                    P2 = __shfl_sync(PLX_FULL_MASK, i2, 31);
                    const double sf0 = rgb0 - i0, sf1 = rgb1 - i1, sf2 = rgb2 - i2;
                    gsig = s.dlt * (up0 * (Ti * s.att * cc0 - sf0) + up1 * (Ti * s.att * cc1 - sf1) +
                                    up2 * (Ti * s.att * cc2 - sf2));
                } else {
                    const double Tn = Ti - wi;
                    const double bn = Tn > 0.0 ? 1.0 : 0.0, bi = Ti > 0.0 ? 1.0 : 0.0;
                    double y0 = s.incl ? cc0 * (bn - bi) : 0.0, y1 = s.incl ? cc1 * (bn - bi) : 0.0,
                           y2 = s.incl ? cc2 * (bn - bi) : 0.0;
                    double i0 = P0 + warp_scan_add(y0, lane), i1 = P1 + warp_scan_add(y1, lane),
                           i2 = P2 + warp_scan_add(y2, lane);
                    P0 = __shfl_sync(PLX_FULL_MASK, i0, 31);
                    P1 = __shfl_sync(PLX_FULL_MASK, i1, 31);
                    P2 = __shfl_sync(PLX_FULL_MASK, i2, 31);
                    const double sf0 = -O.bg[0] * bend + (Q0 - i0);
                    const double sf1 = -O.bg[1] * bend + (Q1 - i1);
                    const double sf2 = -O.bg[2] * bend + (Q2 - i2);
                    const double galpha =
                        (up0 * (cc0 * bn + sf0) + up1 * (cc1 * bn + sf1) + up2 * (cc2 * bn + sf2));
                    gsig = galpha * s.dlt * s.att;
                }
                if (!s.incl) continue;
                if (out.lam_cauchy > 0.0) {   // K:384-386
                    cau_part += log(1.0 + 2.0 * s.sig * s.sig);
                    gsig += out.lam_cauchy * 4.0 * s.sig / (1.0 + 2.0 * s.sig * s.sig);
                }
                const double gc0 = s.c[0] > 0.0 ? up0 * wi : 0.0;   // K:387-389
                const double gc1 = s.c[1] > 0.0 ? up1 * wi : 0.0;
                const double gc2 = s.c[2] > 0.0 ? up2 * wi : 0.0;
                const bool any_c = gc0 != 0.0 || gc1 != 0.0 || gc2 != 0.0;
                constexpr int NQ = NEAREST ? 1 : 8;
#pragma unroll
                for (int q = 0; q < NQ; ++q) {   // K:395-410
                    const int32_t r = s.rows[q];
                    if (r < 0) continue;
                    const double wq = s.ws[q];
                    out.tmask[r] = 1;
                    float *gr = out.grad + (int64_t)r * PLX_ROW;
                    const float gs = (float)(wq * gsig);
                    if (!any_c) {
                        red_add_f32(gr, gs);
                        continue;
                    }
                    const double k0 = wq * gc0, k1 = wq * gc1, k2 = wq * gc2;
                    float v[PLX_ROW];
                    v[0] = gs;
#pragma unroll
                    for (int b = 0; b < 9; ++b) {
                        v[1 + b] = (float)(k0 * basis[b]);
                        v[10 + b] = (float)(k1 * basis[b]);
                        v[19 + b] = (float)(k2 * basis[b]);
                    }
#pragma unroll
                    for (int m = 0; m < 7; ++m)
                        red_add_v4(gr + 4 * m, v[4 * m], v[4 * m + 1], v[4 * m + 2], v[4 * m + 3]);
                }
            }
        }
    }
done:
    if (MODE == BWD) {
        mse_part = warp_sum(mse_part);   // lanes hold identical mse_part; take lane 0's
        cau_part = warp_sum(cau_part);
        if (lane == 0) {
            red_mse[warp] = mse_part / 32.0;
            red_cau[warp] = cau_part;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, b = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                a += red_mse[w];
                b += red_cau[w];
            }
            if (a != 0.0) atomicAdd(out.sums + 0, a);
            if (b != 0.0) atomicAdd(out.sums + 1, b);
        }
    }
}

}  // namespace plx

using namespace plx;

namespace {

constexpr int kThreads = 256;

bool grid_ok(const plx_grid *g) {
    return g && g->links && g->dims[0] >= 2 && g->dims[1] >= 2 && g->dims[2] >= 2 &&
           (g->rows == 0 || g->table) &&
           g->dims[0] * g->dims[1] * g->dims[2] < (int64_t)1 << 31;
}

template <int MODE>
int launch_march(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o, Outs out,
                 void *stream) {
    if (!grid_ok(g) || !rays || !o || rays->n < 0 || !rays->origins || !rays->dirs) return PLX_EINVAL;
    if (MODE != MAXW && !rays->viewdirs) return PLX_EINVAL;
    if (MODE == BWD && (!rays->target || !out.grad || !out.tmask || !out.sums)) return PLX_EINVAL;
    if (!(o->step > 0.0)) return PLX_EINVAL;
    if (rays->n == 0) return PLX_OK;
    DGrid G = make_dgrid(*g);
    RayArgs R{rays->origins, rays->dirs, rays->viewdirs, rays->target, rays->jitter, rays->idx,
              rays->n};
    KOpts K{o->step, o->stop_thresh, {o->bg[0], o->bg[1], o->bg[2]}};
    const int warps = kThreads / 32;
    dim3 grid((unsigned)((rays->n + warps - 1) / warps));
    cudaStream_t s = (cudaStream_t)stream;
    const bool ABSF = MODE != MAXW && o->absolute;
    if (o->nearest) {
        if (ABSF) march_kernel<MODE, true, true><<<grid, kThreads, 0, s>>>(G, R, K, out);
        else march_kernel<MODE, false, true><<<grid, kThreads, 0, s>>>(G, R, K, out);
    } else {
        if (ABSF) march_kernel<MODE, true, false><<<grid, kThreads, 0, s>>>(G, R, K, out);
        else march_kernel<MODE, false, false><<<grid, kThreads, 0, s>>>(G, R, K, out);
    }
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}

}  // namespace

extern "C" int plx_render_fwd(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o,
                              double *out_rgb, double *out_trans, double *out_wsum, void *stream) {
    if (!out_rgb) return PLX_EINVAL;
    Outs out{};
    out.rgb = out_rgb;
    out.trans = out_trans;
    out.wsum = out_wsum;
    return launch_march<FWD>(g, rays, o, out, stream);
}

extern "C" int plx_render_fused_bwd(const plx_grid *g, const plx_rays *rays,
                                    const plx_render_opts *o, int32_t mse_mode, double up_scale,
                                    double lam_cauchy, plx_grad *gb, double *out_rgb,
                                    double *out_sums, void *stream) {
    if (!gb) return PLX_EINVAL;
    Outs out{};
    out.rgb = out_rgb;
    out.sums = out_sums;
    out.grad = gb->grad;
    out.tmask = gb->tmask;
    out.mse_mode = mse_mode;
    out.up_scale = up_scale;
    out.lam_cauchy = lam_cauchy;
    return launch_march<BWD>(g, rays, o, out, stream);
}

extern "C" int plx_max_weight(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o,
                              double *out_w, void *stream) {
    if (!out_w) return PLX_EINVAL;
    Outs out{};
    out.maxw = out_w;
    return launch_march<MAXW>(g, rays, o, out, stream);
}
