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
#include <stdlib.h>

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
    double f[3];   // fractional lattice offsets; weights via stencil_w
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
    stencil<NEAREST>(G, g, s.rows, s.f, occ);
    if (!occ) return;
    // _sigma_at (K:126-135): float64 sum over occupied corners in order.
    double sig = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        int32_t r = s.rows[q];
        if (r >= 0) sig += stencil_w<NEAREST>(s.f, q) * (double)__ldg(G.table + (int64_t)r * PLX_ROW);
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
        const double w = stencil_w<NEAREST>(s.f, q);
        c0 += w * a0;
        c1 += w * a1;
        c2 += w * a2;
    }
    s.c[0] = c0;
    s.c[1] = c1;
    s.c[2] = c2;
}

// Composite one chunk (K:213-233).  In: carry (T for relative, asum for
// absolute), incl flags and att per lane.  Out: per-lane T_i and w_i (valid
// on included lanes; included lanes past the early stop are dropped),
// updated carry, `stopped` (warp-uniform).  Deterministic: pass 2 replays it
// on the recorded (att, incl) and reproduces pass 1 bit-for-bit.
template <bool ABS>
__device__ __forceinline__ void composite_chunk(bool &incl, double att, int lane, double stop,
                                                double &Tcarry, double &Acarry, double &Ti,
                                                double &wi, bool &stopped) {
    double Tn;
    if (!ABS) {
        double a = incl ? att : 1.0;
        double pinc = warp_scan_mul(a, lane);
        double pexc = __shfl_up_sync(PLX_FULL_MASK, pinc, 1);
        if (lane == 0) pexc = 1.0;
        Ti = Tcarry * pexc;
        Tn = Tcarry * pinc;
    } else {
        double v = incl ? 1.0 - att : 0.0;
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
    unsigned stopm = __ballot_sync(PLX_FULL_MASK, incl && Tn < stop);
    int last = 31;
    if (stopm) {
        last = __ffs(stopm) - 1;
        stopped = true;
        if (lane > last) incl = false;
    }
    Tcarry = __shfl_sync(PLX_FULL_MASK, Tn, last);
    if (ABS) Acarry = __shfl_sync(PLX_FULL_MASK, Acarry, last);
}

__device__ __forceinline__ double relu(double x) { return x > 0.0 ? x : 0.0; }

// Per-warp-slot scratch of the backward: pass 1 records, per included
// sample, {att, c0, c1, c2} (+ sigma when the Cauchy term is on) and, per
// chunk, {first position, included-lane mask}; pass 2 replays the
// compositing from these records instead of re-gathering the grid.
struct Scratch {
    int *counter;      // dynamic ray scheduler (zeroed by the launcher)
    double4 *rec;      // [slots][nrec]
    double *rec_sig;   // [slots][nrec]
    uint2 *meta;       // [slots][nchunk]
    int64_t nrec, nchunk;
};

// Packed lattice cell (i, j, k) -> one 64-bit key (21 bits per axis).
__device__ __forceinline__ long long pack_cell(int64_t i, int64_t j, int64_t k) {
    return (long long)((i << 42) | (j << 21) | k);
}

// Per-sample scatter payload staged in shared memory by the lane-parallel
// phase of pass 2 and consumed in sample order by the accumulator below.
struct SmemSample {
    long long key;      // packed stencil cell (or lattice point for nearest)
    float f[4];         // fx, fy, fz, -
    float g[4];         // dL/dsigma, dL/dc_R, dL/dc_G, dL/dc_B  (K:384-389)
    int32_t rows[8];    // stencil rows (K:84-123), -1 = empty
};

// Lane-distributed accumulator of the backward scatter.  The gradient of
// a stencil row factorises as
//   d table[r, 0]          = sum_s w_q(s) dL/dsigma(s)
//   d table[r, 1+9ch+b]    = basis_b * sum_s w_q(s) dL/dc_ch(s)
// (basis_b is per ray), so a cell needs only 8 corners x 4 scalars = 32
// accumulators: lane L holds corner q = L/4, component k = L%4.  A sample
// costs one FMA per lane.  When the ray steps into a face/edge/corner-
// adjacent cell the shared corners are shifted between lanes (one shuffle)
// instead of flushed; a flushed corner becomes one coalesced 28-lane
// reduction on its 112-byte gradient row (lane c = column c).
template <bool NEAREST>
struct LaneAcc {
    float acc;          // this lane's (corner, component) partial sum
    int32_t row;        // row of this lane's corner, -1 = empty / none
    long long cell;     // packed current cell, -1 = none
    int q, k;           // lane's corner and component
    int kcol;           // source component of column `lane` at flush time
    float col_basis;    // basis factor of column `lane` (1 for sigma)

    __device__ __forceinline__ void init(int lane, const double *basis) {
        acc = 0.f;
        row = -1;
        cell = -1;
        q = lane >> 2;
        k = lane & 3;
        kcol = lane == 0 ? 0 : (lane < PLX_ROW ? 1 + (lane - 1) / 9 : 0);
        col_basis = lane == 0 ? 1.f : 0.f;
        if (lane >= 1 && lane < PLX_ROW) {
            const int b = (lane - 1) % 9;
#pragma unroll
            for (int bb = 0; bb < 9; ++bb)
                if (bb == b) col_basis = (float)basis[bb];
        }
    }
    __device__ __forceinline__ void flush_corner(int qq, float *grad, uint8_t *tmask, int lane) {
        const int32_t r = __shfl_sync(PLX_FULL_MASK, row, 4 * qq);
        const float a = __shfl_sync(PLX_FULL_MASK, acc, 4 * qq + kcol);
        if (r >= 0) {
            if (lane < PLX_ROW) red_add_f32(grad + (int64_t)r * PLX_ROW + lane, a * col_basis);
            if (lane == 0) tmask[r] = 1;
        }
    }
    __device__ __forceinline__ void flush_all(float *grad, uint8_t *tmask, int lane) {
#pragma unroll
        for (int qq = 0; qq < (NEAREST ? 1 : 8); ++qq) flush_corner(qq, grad, tmask, lane);
        acc = 0.f;
        row = -1;
        cell = -1;
    }
    // corner bit `bit` (4 = x, 2 = y, 1 = z) moves by delta = +-1
    __device__ __forceinline__ void shift(int bit, int delta, float *grad, uint8_t *tmask,
                                          int lane) {
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
            const bool leaving = delta > 0 ? !(qq & bit) : (qq & bit);
            if (leaving) flush_corner(qq, grad, tmask, lane);
        }
        const int off = 4 * bit;
        if (delta > 0) {   // hi corners become lo, new hi corners start empty
            const float a = __shfl_down_sync(PLX_FULL_MASK, acc, off);
            const int32_t r = __shfl_down_sync(PLX_FULL_MASK, row, off);
            acc = (q & bit) ? 0.f : a;
            row = (q & bit) ? -1 : r;
        } else {
            const float a = __shfl_up_sync(PLX_FULL_MASK, acc, off);
            const int32_t r = __shfl_up_sync(PLX_FULL_MASK, row, off);
            acc = (q & bit) ? a : 0.f;
            row = (q & bit) ? r : -1;
        }
    }
    __device__ __forceinline__ void move_to(long long nc, const SmemSample &smp, float *grad,
                                            uint8_t *tmask, int lane) {
        if (NEAREST) {
            flush_corner(0, grad, tmask, lane);
            acc = 0.f;
        } else if (cell >= 0) {
            const long long di = (nc >> 42) - (cell >> 42);
            const long long dj = ((nc >> 21) & 0x1fffff) - ((cell >> 21) & 0x1fffff);
            const long long dk = (nc & 0x1fffff) - (cell & 0x1fffff);
            if (di >= -1 && di <= 1 && dj >= -1 && dj <= 1 && dk >= -1 && dk <= 1) {
                if (di) shift(4, (int)di, grad, tmask, lane);
                if (dj) shift(2, (int)dj, grad, tmask, lane);
                if (dk) shift(1, (int)dk, grad, tmask, lane);
            } else {
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) flush_corner(qq, grad, tmask, lane);
                acc = 0.f;
            }
        }
        cell = nc;
        row = smp.rows[NEAREST ? 0 : q];
    }
    __device__ __forceinline__ void add(const SmemSample &smp) {
        const float gk = smp.g[k];
        if (NEAREST) {
            acc += q == 0 ? gk : 0.f;
        } else {
            const float wx = (q & 4) ? smp.f[0] : 1.f - smp.f[0];
            const float wy = (q & 2) ? smp.f[1] : 1.f - smp.f[1];
            const float wz = (q & 1) ? smp.f[2] : 1.f - smp.f[2];
            acc += wx * wy * wz * gk;
        }
    }
};

template <int MODE, bool ABS, bool NEAREST, int MINB>
__global__ void __launch_bounds__(256, MINB)
    march_kernel(DGrid G, RayArgs R, KOpts O, Outs out, Scratch S) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t slot = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const int64_t nslots = (int64_t)gridDim.x * (blockDim.x >> 5);
    double mse_part = 0.0, cau_part = 0.0;
    const unsigned lt_mask = (1u << lane) - 1u;
    int64_t ray = slot;
    __shared__ SmemSample smem_all[MODE == BWD ? 8 : 1][32];
    SmemSample *sm = smem_all[MODE == BWD ? warp : 0];

    for (;;) {
        if (MODE == BWD) {   // dynamic scheduling: rays differ widely in length
            int r = 0;
            if (lane == 0) r = atomicAdd(S.counter, 1);
            ray = __shfl_sync(PLX_FULL_MASK, r, 0);
        }
        if (ray >= R.n) break;
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
        int64_t nch = 0, nrec = 0;              // recorded chunks / samples
        double4 *rec = S.rec + slot * S.nrec;
        double *rec_sig = S.rec_sig + slot * S.nrec;
        uint2 *meta = S.meta + slot * S.nchunk;
        bool stopped = false;
        for (int64_t base = 0; base < rm.nsamp && !stopped; base += 32) {
            Sample s;
            eval_sample<MODE, NEAREST>(G, rm, O.step, base + lane, basis, s);
            if (!__any_sync(PLX_FULL_MASK, s.incl)) continue;
            double Ti, wi;
            composite_chunk<(MODE == MAXW ? false : ABS)>(s.incl, s.att, lane, O.stop, T, A, Ti,
                                                           wi, stopped);
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
            if (MODE == BWD) {   // record the chunk for pass 2
                const unsigned m = __ballot_sync(PLX_FULL_MASK, s.incl);
                if (lane == 0) meta[nch] = make_uint2((unsigned)base, m);
                if (s.incl) {
                    const int64_t k = nrec + __popc(m & lt_mask);
                    rec[k] = make_double4(s.att, s.c[0], s.c[1], s.c[2]);
                    if (out.lam_cauchy > 0.0) rec_sig[k] = s.sig;
                }
                ++nch;
                nrec += __popc(m);
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
        if (MODE == MAXW) {
            ray += nslots;
            continue;
        }
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
            ray += nslots;
            continue;
        }
        // ---------------- upstream (K:330-341) ----------------
        double up0, up1, up2;
        if (out.mse_mode) {
            const double e0 = rgb0 - __ldg(R.target + 3 * src + 0);
            const double e1 = rgb1 - __ldg(R.target + 3 * src + 1);
            const double e2 = rgb2 - __ldg(R.target + 3 * src + 2);
            if (lane == 0) mse_part += e0 * e0 + e1 * e1 + e2 * e2;
            up0 = out.up_scale * e0;
            up1 = out.up_scale * e1;
            up2 = out.up_scale * e2;
        } else {
            up0 = __ldg(R.target + 3 * src + 0);
            up1 = __ldg(R.target + 3 * src + 1);
            up2 = __ldg(R.target + 3 * src + 2);
        }
        if (ABS) {
            Q0 = warp_sum(Q0);
            Q1 = warp_sum(Q1);
            Q2 = warp_sum(Q2);
        }
        // ---------------- pass 2: replay + transposed scatter ----------------
        // sf before sample i in the reference's reverse sweep:
        //   relative: T bg + sum_{j>i} w_j c_j = rgb - P_i      (K:351-353, 381-383)
        //   absolute: -bg [T>0] + sum_{j>i} c_j (bn_j - bi_j)   (K:346-349, 374-376)
        const double bend = T > 0.0 ? 1.0 : 0.0;
        LaneAcc<NEAREST> ra;
        ra.init(lane, basis);
        double P0 = 0.0, P1 = 0.0, P2 = 0.0;
        double T2 = 1.0, A2 = 0.0;
        bool stopped2 = false;
        int64_t k0 = 0;
        for (int64_t c = 0; c < nch; ++c) {
            const uint2 mt = meta[c];
            const unsigned mask = mt.y;
            const int64_t si = (int64_t)mt.x + lane;
            bool incl = (mask >> lane) & 1u;
            double att = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, sig = 0.0;
            if (incl) {
                const int64_t k = k0 + __popc(mask & lt_mask);
                const double4 r4 = rec[k];
                att = r4.x;
                c0 = r4.y;
                c1 = r4.z;
                c2 = r4.w;
                if (out.lam_cauchy > 0.0) sig = rec_sig[k];
            }
            k0 += __popc(mask);
            double Ti, wi;
            composite_chunk<ABS>(incl, att, lane, O.stop, T2, A2, Ti, wi, stopped2);
            const double cc0 = relu(c0), cc1 = relu(c1), cc2 = relu(c2);
            double t, dlt, g[3];
            sample_coords(rm, G, O.step, si, t, dlt, g);
            double gsig;
            if (!ABS) {
                double y0 = incl ? wi * cc0 : 0.0, y1 = incl ? wi * cc1 : 0.0,
                       y2 = incl ? wi * cc2 : 0.0;
                double i0 = P0 + warp_scan_add(y0, lane), i1 = P1 + warp_scan_add(y1, lane),
                       i2 = P2 + warp_scan_add(y2, lane);
                P0 = __shfl_sync(PLX_FULL_MASK, i0, 31);
                P1 = __shfl_sync(PLX_FULL_MASK, i1, 31);
                P2 = __shfl_sync(PLX_FULL_MASK, i2, 31);
                const double sf0 = rgb0 - i0, sf1 = rgb1 - i1, sf2 = rgb2 - i2;
                gsig = dlt * (up0 * (Ti * att * cc0 - sf0) + up1 * (Ti * att * cc1 - sf1) +
                              up2 * (Ti * att * cc2 - sf2));
            } else {
                const double Tn = Ti - wi;
                const double bn = Tn > 0.0 ? 1.0 : 0.0, bi = Ti > 0.0 ? 1.0 : 0.0;
                double y0 = incl ? cc0 * (bn - bi) : 0.0, y1 = incl ? cc1 * (bn - bi) : 0.0,
                       y2 = incl ? cc2 * (bn - bi) : 0.0;
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
                gsig = galpha * dlt * att;
            }
            if (incl && out.lam_cauchy > 0.0) {   // K:384-386
                cau_part += log(1.0 + 2.0 * sig * sig);
                gsig += out.lam_cauchy * 4.0 * sig / (1.0 + 2.0 * sig * sig);
            }
            // per-sample scatter payload (K:387-410), staged for the in-order accumulator
            if (incl) {
                SmemSample &me = sm[lane];
                me.g[0] = (float)gsig;
                me.g[1] = c0 > 0.0 ? (float)(up0 * wi) : 0.f;
                me.g[2] = c1 > 0.0 ? (float)(up1 * wi) : 0.f;
                me.g[3] = c2 > 0.0 ? (float)(up2 * wi) : 0.f;
                if (NEAREST) {
                    int64_t i = (int64_t)(g[0] + 0.5), j = (int64_t)(g[1] + 0.5), k = (int64_t)(g[2] + 0.5);
                    if (i > G.Dx - 1) i = G.Dx - 1;
                    if (j > G.Dy - 1) j = G.Dy - 1;
                    if (k > G.Dz - 1) k = G.Dz - 1;
                    me.key = pack_cell(i, j, k);
                    me.rows[0] = __ldg(G.links + flat(G, i, j, k));
                } else {
                    int64_t i0 = (int64_t)g[0], j0 = (int64_t)g[1], kk0 = (int64_t)g[2];
                    if (i0 > G.Dx - 2) i0 = G.Dx - 2;
                    if (j0 > G.Dy - 2) j0 = G.Dy - 2;
                    if (kk0 > G.Dz - 2) kk0 = G.Dz - 2;
                    me.key = pack_cell(i0, j0, kk0);
                    me.f[0] = (float)(g[0] - (double)i0);
                    me.f[1] = (float)(g[1] - (double)j0);
                    me.f[2] = (float)(g[2] - (double)kk0);
                    const int32_t *base = G.links + flat(G, i0, j0, kk0);
                    const int64_t sy = G.Dz, sx = (int64_t)G.Dy * G.Dz;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        me.rows[q] = __ldg(base + ((q >> 2) & 1) * sx + ((q >> 1) & 1) * sy + (q & 1));
                }
            }
            __syncwarp();
            unsigned m = mask;   // already truncated at the early stop in pass 1
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                const SmemSample &smp = sm[j];
                const long long key = smp.key;
                if (key != ra.cell) ra.move_to(key, smp, out.grad, out.tmask, lane);
                ra.add(smp);
            }
            __syncwarp();
        }
        ra.flush_all(out.grad, out.tmask, lane);
        ray += nslots;
    }
    if (MODE == BWD) {   // one pair of f64 atomics per warp (no block barrier)
        cau_part = warp_sum(cau_part);
        if (lane == 0) {
            if (mse_part != 0.0) atomicAdd(out.sums + 0, mse_part);
            if (cau_part != 0.0) atomicAdd(out.sums + 1, cau_part);
        }
    }
}

}  // namespace plx

using namespace plx;

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

bool grid_ok(const plx_grid *g) {
    return g && g->links && g->dims[0] >= 2 && g->dims[1] >= 2 && g->dims[2] >= 2 &&
           (g->rows == 0 || g->table) && g->dims[0] < (1 << 21) && g->dims[1] < (1 << 21) &&
           g->dims[2] < (1 << 21) && g->dims[0] * g->dims[1] * g->dims[2] < (int64_t)1 << 31;
}

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// Minimum resident blocks per SM the backward is compiled for (register
// budget 128 vs 80 per thread); PLX_BWD_MINB=2|3 selects (default 2).
int bwd_minb() {
    static int m = 0;
    if (!m) {
        const char *e = getenv("PLX_BWD_MINB");
        m = (e && atoi(e) == 3) ? 3 : 2;
    }
    return m;
}

template <int MODE, bool ABS, bool NEAREST, int MINB>
int blocks_per_sm() {
    static int nb = 0;
    if (!nb) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, march_kernel<MODE, ABS, NEAREST, MINB>,
                                                      kThreads, 0);
        if (nb <= 0) nb = 1;
    }
    return nb;
}

template <int MINB>
int bwd_blocks_per_sm_t(const plx_render_opts *o) {
    if (o->nearest)
        return o->absolute ? blocks_per_sm<BWD, true, true, MINB>()
                           : blocks_per_sm<BWD, false, true, MINB>();
    return o->absolute ? blocks_per_sm<BWD, true, false, MINB>()
                       : blocks_per_sm<BWD, false, false, MINB>();
}

int bwd_blocks_per_sm(const plx_render_opts *o) {
    return bwd_minb() == 3 ? bwd_blocks_per_sm_t<3>(o) : bwd_blocks_per_sm_t<2>(o);
}

template <int MODE, int MINB>
void launch_variant(const plx_render_opts *o, bool ABSF, dim3 grid, cudaStream_t s, DGrid G,
                    RayArgs R, KOpts K, Outs out, Scratch S) {
    if (o->nearest) {
        if (ABSF) march_kernel<MODE, true, true, MINB><<<grid, kThreads, 0, s>>>(G, R, K, out, S);
        else march_kernel<MODE, false, true, MINB><<<grid, kThreads, 0, s>>>(G, R, K, out, S);
    } else {
        if (ABSF) march_kernel<MODE, true, false, MINB><<<grid, kThreads, 0, s>>>(G, R, K, out, S);
        else march_kernel<MODE, false, false, MINB><<<grid, kThreads, 0, s>>>(G, R, K, out, S);
    }
}

// Capacity of one warp slot: every march position of the longest chord (R:67-69).
int64_t max_records(const plx_grid *g, double step) {
    double d2 = 0.0;
    for (int a = 0; a < 3; ++a) d2 += (g->hi[a] - g->lo[a]) * (g->hi[a] - g->lo[a]);
    return (int64_t)ceil(sqrt(d2) / step) + 4;
}

struct ScratchLayout {
    int64_t slots, nrec, nchunk, bytes, off_rec, off_sig, off_meta;
};

ScratchLayout layout(const plx_grid *g, const plx_render_opts *o, int64_t n_rays) {
    ScratchLayout L;
    int64_t blocks = (int64_t)num_sms() * bwd_blocks_per_sm(o);
    const int64_t need = (n_rays + kWarps - 1) / kWarps;
    if (n_rays > 0 && need < blocks) blocks = need;
    L.slots = blocks * kWarps;
    L.nrec = max_records(g, o->step);
    L.nchunk = L.nrec / 32 + 2;
    L.off_rec = 256;
    L.off_sig = L.off_rec + L.slots * L.nrec * (int64_t)sizeof(double4);
    L.off_meta = L.off_sig + L.slots * L.nrec * (int64_t)sizeof(double);
    L.bytes = L.off_meta + L.slots * L.nchunk * (int64_t)sizeof(uint2);
    return L;
}

template <int MODE>
int launch_march(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o, Outs out,
                 void *scratch, int64_t scratch_bytes, void *stream) {
    if (!grid_ok(g) || !rays || !o || rays->n < 0 || !rays->origins || !rays->dirs) return PLX_EINVAL;
    if (rays->n >= (int64_t)1 << 31) return PLX_EINVAL;
    if (MODE != MAXW && !rays->viewdirs) return PLX_EINVAL;
    if (MODE == BWD && (!rays->target || !out.grad || !out.tmask || !out.sums || !scratch))
        return PLX_EINVAL;
    if (!(o->step > 0.0)) return PLX_EINVAL;
    if (rays->n == 0) return PLX_OK;
    DGrid G = make_dgrid(*g);
    RayArgs R{rays->origins, rays->dirs, rays->viewdirs, rays->target, rays->jitter, rays->idx,
              rays->n};
    KOpts K{o->step, o->stop_thresh, {o->bg[0], o->bg[1], o->bg[2]}};
    cudaStream_t s = (cudaStream_t)stream;
    Scratch S{};
    int64_t blocks;
    if (MODE == BWD) {
        const ScratchLayout L = layout(g, o, rays->n);
        if (scratch_bytes < L.bytes) return PLX_EINVAL;
        char *base = reinterpret_cast<char *>(scratch);
        S.counter = reinterpret_cast<int *>(base);
        S.rec = reinterpret_cast<double4 *>(base + L.off_rec);
        S.rec_sig = reinterpret_cast<double *>(base + L.off_sig);
        S.meta = reinterpret_cast<uint2 *>(base + L.off_meta);
        S.nrec = L.nrec;
        S.nchunk = L.nchunk;
        blocks = L.slots / kWarps;
        if (cudaMemsetAsync(S.counter, 0, sizeof(int), s) != cudaSuccess) return PLX_ECUDA;
    } else {   // static grid-stride over rays, occupancy-sized grid
        blocks = (rays->n + kWarps - 1) / kWarps;
        const int64_t cap = (int64_t)num_sms() * 4;
        if (blocks > cap) blocks = cap;
    }
    const bool ABSF = MODE != MAXW && o->absolute;
    dim3 grid((unsigned)blocks);
    if (MODE == BWD && bwd_minb() == 2) launch_variant<MODE, 2>(o, ABSF, grid, s, G, R, K, out, S);
    else launch_variant<MODE, 3>(o, ABSF, grid, s, G, R, K, out, S);
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
    return launch_march<FWD>(g, rays, o, out, nullptr, 0, stream);
}

extern "C" int64_t plx_render_scratch_bytes(const plx_grid *g, const plx_render_opts *o,
                                            int64_t n_rays) {
    if (!grid_ok(g) || !o || !(o->step > 0.0)) return -1;
    return layout(g, o, n_rays).bytes;
}

extern "C" int plx_render_fused_bwd(const plx_grid *g, const plx_rays *rays,
                                    const plx_render_opts *o, int32_t mse_mode, double up_scale,
                                    double lam_cauchy, plx_grad *gb, double *out_rgb,
                                    double *out_sums, void *scratch, int64_t scratch_bytes,
                                    void *stream) {
    if (!gb) return PLX_EINVAL;
    Outs out{};
    out.rgb = out_rgb;
    out.sums = out_sums;
    out.grad = gb->grad;
    out.tmask = gb->tmask;
    out.mse_mode = mse_mode;
    out.up_scale = up_scale;
    out.lam_cauchy = lam_cauchy;
    return launch_march<BWD>(g, rays, o, out, scratch, scratch_bytes, stream);
}

extern "C" int plx_max_weight(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o,
                              double *out_w, void *stream) {
    if (!out_w) return PLX_EINVAL;
    Outs out{};
    out.maxw = out_w;
    return launch_march<MAXW>(g, rays, o, out, nullptr, 0, stream);
}
