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
    unsigned long long *stats;   // optional {positions, samples, chunks, rays}
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
    float c[3];    // pre-clamp colour (K:305)
    bool incl;
};

// Evaluate position si (K:286-305): stencil, sigma, and for included samples
// the colour.  FWD/MAXW include sigma > 0, BWD sigma >= 0 (K:211 vs K:293).
// Positions, stencil rows/weights, sigma and exp(-sigma delta) are float64
// in the reference's operation order (bit-exact on f32 grids: the sample
// set, the early stop and the touched rows match the reference exactly).
// The colour dot products (8 corners x 27 SH x basis) are float32 FMAs: the
// tolerance is 1e-4 on RGB and they are ~3e-7 from float64, while float64
// here cost a third of the kernel's instructions (f32->f64 converts, and
// DMUL+DADD pairs under -fmad=false).
template <int MODE, bool NEAREST>
__device__ __forceinline__ void eval_sample(const DGrid &G, const RayMarch &rm, double step,
                                            int64_t si, const float *bf, Sample &s) {
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
        if (r >= 0) sig += stencil_w<NEAREST>(s.f, q) * (double)__ldg(G.density + r);
    }
    s.sig = sig;
    if (MODE == BWD ? !(sig >= 0.0) : !(sig > 0.0)) return;
    s.incl = true;
    s.att = exp(-sig * s.dlt);
    if (MODE == MAXW) return;
    // _color_at (K:138-152): per corner the 3 SH dots, then weight.
    float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        int32_t r = s.rows[q];
        if (r < 0) continue;
        const float4 *row = reinterpret_cast<const float4 *>(G.table + (int64_t)r * PLX_ROW);
        float4 v0 = __ldg(row + 0), v1 = __ldg(row + 1), v2 = __ldg(row + 2), v3 = __ldg(row + 3);
        float4 v4 = __ldg(row + 4), v5 = __ldg(row + 5), v6 = __ldg(row + 6);
        // row layout: [sig, R0..R8, G0..G8, B0..B8]
        float a0 = bf[0] * v0.y, a1 = bf[0] * v2.z, a2 = bf[0] * v4.w;
        a0 = __fmaf_rn(bf[1], v0.z, a0);
        a1 = __fmaf_rn(bf[1], v2.w, a1);
        a2 = __fmaf_rn(bf[1], v5.x, a2);
        a0 = __fmaf_rn(bf[2], v0.w, a0);
        a1 = __fmaf_rn(bf[2], v3.x, a1);
        a2 = __fmaf_rn(bf[2], v5.y, a2);
        a0 = __fmaf_rn(bf[3], v1.x, a0);
        a1 = __fmaf_rn(bf[3], v3.y, a1);
        a2 = __fmaf_rn(bf[3], v5.z, a2);
        a0 = __fmaf_rn(bf[4], v1.y, a0);
        a1 = __fmaf_rn(bf[4], v3.z, a1);
        a2 = __fmaf_rn(bf[4], v5.w, a2);
        a0 = __fmaf_rn(bf[5], v1.z, a0);
        a1 = __fmaf_rn(bf[5], v3.w, a1);
        a2 = __fmaf_rn(bf[5], v6.x, a2);
        a0 = __fmaf_rn(bf[6], v1.w, a0);
        a1 = __fmaf_rn(bf[6], v4.x, a1);
        a2 = __fmaf_rn(bf[6], v6.y, a2);
        a0 = __fmaf_rn(bf[7], v2.x, a0);
        a1 = __fmaf_rn(bf[7], v4.y, a1);
        a2 = __fmaf_rn(bf[7], v6.z, a2);
        a0 = __fmaf_rn(bf[8], v2.y, a0);
        a1 = __fmaf_rn(bf[8], v4.z, a1);
        a2 = __fmaf_rn(bf[8], v6.w, a2);
        const float w = (float)stencil_w<NEAREST>(s.f, q);
        c0 = __fmaf_rn(w, a0, c0);
        c1 = __fmaf_rn(w, a1, c1);
        c2 = __fmaf_rn(w, a2, c2);
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
// sample, att (f64) and {c0, c1, c2} (f32), 24 B (+ sigma when the Cauchy
// term is on) and, per
// chunk, {first position, included-lane mask}; pass 2 replays the
// compositing from these records instead of re-gathering the grid.
struct Scratch {
    int *counter;      // dynamic ray scheduler (zeroed by the launcher)
    double *rec_att;   // [slots][nrec]  exp(-sigma delta), float64 (replayed bit-exactly)
    float4 *rec_c;     // [slots][nrec]  pre-clamp colour (f32, as computed)
    double *rec_sig;   // [slots][nrec]
    uint2 *meta;       // [slots][nchunk]
    int64_t nrec, nchunk;
};

// Per-warp shared staging of one chunk's scatter payload (pass 2).  The
// lane-parallel phase writes, per included sample j: its stencil rows, its
// move code relative to the previous included sample, and val[L][j] = the
// contribution w_e(j) * g_k(j) destined for accumulator lane L (corner e =
// (L/4) ^ flip_j, component k = L%4).  The serial phase then only adds
// val[lane][j] and handles moves.  Row pitch 33 keeps both the transposed
// writes and the per-sample reads bank-conflict free.
struct SmemChunk {
    float val[32][33];
    int32_t rows[32][8];
    int mv[32];
};

// Move code of a sample relative to the previous included one (warp-
// uniform when read back): 0 = same cell; bit 7 = far jump or first sample
// (flush everything); else bit 6 | (di+1)<<4 | (dj+1)<<2 | (dk+1).
constexpr int MV_FAR = 128, MV_ADJ = 64;

__device__ __forceinline__ int axis_bits(int mv) {
    if (!(mv & MV_ADJ)) return 0;
    return (((mv >> 4) & 3) != 1 ? 4 : 0) | (((mv >> 2) & 3) != 1 ? 2 : 0) | ((mv & 3) != 1 ? 1 : 0);
}

// Lane-distributed accumulator of the backward scatter.  The gradient of
// a stencil row factorises as
//   d table[r, 0]          = sum_s w_q(s) dL/dsigma(s)
//   d table[r, 1+9ch+b]    = basis_b * sum_s w_q(s) dL/dc_ch(s)
// (basis_b is per ray), so a cell needs only 8 corners x 4 scalars = 32
// accumulators: lane L holds component k = L%4 of the corner e = (L/4) ^
// flip.  A ray visits the 8 cells around a lattice point in one contiguous
// run (they form a convex box), so a corner's accumulator lives from the
// move that brings it in to the move that takes it out.  On a face crossing
// along axis `bit` the 4 leaving corners are flushed and `flip ^= bit`
// relabels the lanes: the staying corners keep their lanes and values, the
// flushed lanes become the incoming corners -- no data moves between lanes.
// A flush is one warp instruction for the 4 leaving 112-byte gradient rows:
// lanes 0..27 = 4 corners x 7 column quads, each lane expands its quad from
// (at most two) components times the ray's basis into one
// red.global.add.v4.f32.
template <bool NEAREST>
struct LaneAcc {
    float acc;          // this lane's partial sum
    int32_t row;        // row of this lane's corner, -1 = empty / none
    int q, k;           // physical corner slot and component
    int flip;           // warp-uniform corner relabelling (xor on q)
    int quad;           // flush role: column quad lane%7 of corner slot lane/7
    int klo, khi;       // components feeding columns 4*quad .. 4*quad+3
    unsigned hisel;     // bit j: column 4*quad+j takes the khi component
    float cb[4];        // basis factor of each of the 4 columns (1 for sigma)

    __device__ __forceinline__ static int col_comp(int c) { return c == 0 ? 0 : 1 + (c - 1) / 9; }

    __device__ __forceinline__ void init(int lane, const float *bf) {
        acc = 0.f;
        row = -1;
        flip = 0;
        q = lane >> 2;
        k = lane & 3;
        quad = lane % 7;
        klo = col_comp(4 * quad);
        khi = col_comp(4 * quad + 3);
        hisel = 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = 4 * quad + j;
            if (col_comp(c) != klo) hisel |= 1u << j;
            float f = 1.f;
            if (c > 0) {
                const int b = (c - 1) % 9;
#pragma unroll
                for (int bb = 0; bb < 9; ++bb)
                    if (bb == b) f = bf[bb];
            }
            cb[j] = f;
        }
    }
    // Flush the 4 corners whose effective `bit` equals `side` (NEAREST:
    // corner 0 only) and reset their lanes.
    __device__ __forceinline__ void flush4(int bit, int side, float *grad, uint8_t *tmask,
                                           int lane) {
        int qq = 0;
        if (!NEAREST) {
            const int s = (lane / 7) & 3;
            qq = (((s & ~(bit - 1)) << 1) | (s & (bit - 1)) | (side ? bit : 0)) ^ flip;
        }
        const int32_t r = __shfl_sync(PLX_FULL_MASK, row, 4 * qq);
        const float alo = __shfl_sync(PLX_FULL_MASK, acc, 4 * qq + klo);
        const float ahi = __shfl_sync(PLX_FULL_MASK, acc, 4 * qq + khi);
        const bool mine = NEAREST ? (lane < 7) : (lane < 28);
        if (mine && r >= 0) {
            const float v0 = ((hisel & 1u) ? ahi : alo) * cb[0];
            const float v1 = ((hisel & 2u) ? ahi : alo) * cb[1];
            const float v2 = ((hisel & 4u) ? ahi : alo) * cb[2];
            const float v3 = ((hisel & 8u) ? ahi : alo) * cb[3];
            if (quad == 0) tmask[r] = 1;
            if (v0 != 0.f || v1 != 0.f || v2 != 0.f || v3 != 0.f)
                red_add_v4(grad + (int64_t)r * PLX_ROW + 4 * quad, v0, v1, v2, v3);
        }
        if (NEAREST || (((q ^ flip) & bit) != 0) == (side != 0)) {
            acc = 0.f;
            row = -1;
        }
    }
    __device__ __forceinline__ void flush_all(float *grad, uint8_t *tmask, int lane) {
        flush4(4, 0, grad, tmask, lane);
        if (!NEAREST) flush4(4, 1, grad, tmask, lane);
    }
    __device__ __forceinline__ void move(int mv, const SmemChunk &sc, int j, float *grad,
                                         uint8_t *tmask, int lane) {
        if (NEAREST || (mv & MV_FAR)) {
            flush_all(grad, tmask, lane);
        } else {
            const int di = ((mv >> 4) & 3) - 1, dj = ((mv >> 2) & 3) - 1, dk = (mv & 3) - 1;
            if (di) {
                flush4(4, di < 0, grad, tmask, lane);
                flip ^= 4;
            }
            if (dj) {
                flush4(2, dj < 0, grad, tmask, lane);
                flip ^= 2;
            }
            if (dk) {
                flush4(1, dk < 0, grad, tmask, lane);
                flip ^= 1;
            }
        }
        row = sc.rows[j][NEAREST ? 0 : (q ^ flip)];
    }
};

template <int MODE, bool ABS, bool NEAREST, int MINB>
__global__ void __launch_bounds__(128, MINB)
    march_kernel(DGrid G, RayArgs R, KOpts O, Outs out, Scratch S) {
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int64_t slot = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    const int64_t nslots = (int64_t)gridDim.x * (blockDim.x >> 5);
    double mse_part = 0.0, cau_part = 0.0;
    unsigned st_pos = 0, st_samp = 0, st_chunks = 0, st_rays = 0;   // warp-uniform
    const unsigned lt_mask = (1u << lane) - 1u;
    int64_t ray = slot;
    __shared__ SmemChunk smem_all[MODE == BWD ? 4 : 1];
    SmemChunk &sc = smem_all[MODE == BWD ? warp : 0];

    for (;;) {
        if (MODE == BWD) {   // dynamic scheduling: rays differ widely in length
            int r = 0;
            if (lane == 0) r = atomicAdd(S.counter, 1);
            ray = __shfl_sync(PLX_FULL_MASK, r, 0);
        }
        if (ray >= R.n) break;
        ++st_rays;
        const int64_t src = R.idx ? R.idx[ray] : ray;
        RayMarch rm;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            rm.o[a] = __ldg(R.origins + 3 * src + a);
            rm.d[a] = __ldg(R.dirs + 3 * src + a);
        }
        float bf[9];   // SH basis (K:27-37) in float64, used as f32 by the colour FMAs
        if (MODE != MAXW) {
            double basis[9];
            sh_basis9(__ldg(R.viewdirs + 3 * src), __ldg(R.viewdirs + 3 * src + 1),
                      __ldg(R.viewdirs + 3 * src + 2), basis);
#pragma unroll
            for (int b = 0; b < 9; ++b) bf[b] = (float)basis[b];
        }
        const double jit = (MODE != MAXW && R.jitter) ? R.jitter[ray] : 0.0;
        ray_march_setup(rm, G, O.step, jit);

        // ---------------- pass 1: forward ----------------
        double T = 1.0, A = 0.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, wsum = 0.0;
        double Q0 = 0.0, Q1 = 0.0, Q2 = 0.0;   // absolute backward: sum c(bn - bi)
        int64_t nch = 0, nrec = 0;              // recorded chunks / samples
        double *rec_att = S.rec_att + slot * S.nrec;
        float4 *rec_c = S.rec_c + slot * S.nrec;
        double *rec_sig = S.rec_sig + slot * S.nrec;
        uint2 *meta = S.meta + slot * S.nchunk;
        bool stopped = false;
        for (int64_t base = 0; base < rm.nsamp && !stopped; base += 32) {
            Sample s;
            eval_sample<MODE, NEAREST>(G, rm, O.step, base + lane, bf, s);
            const int npos = (int)min((int64_t)32, rm.nsamp - base);
            if (!__any_sync(PLX_FULL_MASK, s.incl)) {
                st_pos += npos;
                st_chunks += 1;
                continue;
            }
            double Ti, wi;
            composite_chunk<(MODE == MAXW ? false : ABS)>(s.incl, s.att, lane, O.stop, T, A, Ti,
                                                           wi, stopped);
            {   // positions up to the early stop, samples that contribute
                const unsigned im = __ballot_sync(PLX_FULL_MASK, s.incl);
                st_pos += stopped ? 32 - __clz(im) : npos;
                st_samp += __popc(im);
                st_chunks += 1;
            }
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
            const double cr0 = relu((double)s.c[0]), cr1 = relu((double)s.c[1]),
                         cr2 = relu((double)s.c[2]);
            if (MODE == BWD) {   // record the chunk for pass 2
                const unsigned m = __ballot_sync(PLX_FULL_MASK, s.incl);
                if (lane == 0) meta[nch] = make_uint2((unsigned)base, m);
                if (s.incl) {
                    const int64_t k = nrec + __popc(m & lt_mask);
                    rec_att[k] = s.att;
                    rec_c[k] = make_float4(s.c[0], s.c[1], s.c[2], 0.f);
                    if (out.lam_cauchy > 0.0) rec_sig[k] = s.sig;
                }
                ++nch;
                nrec += __popc(m);
            }
            double x0 = 0.0, x1 = 0.0, x2 = 0.0, xw = 0.0;
            if (s.incl) {
                x0 = wi * cr0;
                x1 = wi * cr1;
                x2 = wi * cr2;
                xw = wi;
                if (MODE == BWD && ABS) {
                    double bn = (Ti - wi) > 0.0 ? 1.0 : 0.0, bi = Ti > 0.0 ? 1.0 : 0.0;
                    Q0 += cr0 * (bn - bi);
                    Q1 += cr1 * (bn - bi);
                    Q2 += cr2 * (bn - bi);
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
        ra.init(lane, bf);
        double P0 = 0.0, P1 = 0.0, P2 = 0.0;
        double T2 = 1.0, A2 = 0.0;
        bool stopped2 = false;
        int64_t k0 = 0;
        // carried across chunks: last included sample's cell and the flip
        int pci = 0, pcj = 0, pck = 0;
        bool pvalid = false;
        int cflip = 0;
        for (int64_t c = 0; c < nch; ++c) {
            const uint2 mt = meta[c];
            const unsigned mask = mt.y;
            const int64_t si = (int64_t)mt.x + lane;
            bool incl = (mask >> lane) & 1u;
            double att = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, sig = 0.0;
            if (incl) {
                const int64_t k = k0 + __popc(mask & lt_mask);
                att = rec_att[k];
                const float4 c4 = rec_c[k];
                c0 = c4.x;
                c1 = c4.y;
                c2 = c4.z;
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
            // ---- lane-parallel staging of the scatter payload (K:387-410) ----
            // mask is already truncated at the early stop (pass 1)
            int ci = 0, cj = 0, ck = 0;
            float f0 = 0.f, f1 = 0.f, f2 = 0.f;
            if (incl) {
                if (NEAREST) {
                    int64_t i = (int64_t)(g[0] + 0.5), j = (int64_t)(g[1] + 0.5), k = (int64_t)(g[2] + 0.5);
                    if (i > G.Dx - 1) i = G.Dx - 1;
                    if (j > G.Dy - 1) j = G.Dy - 1;
                    if (k > G.Dz - 1) k = G.Dz - 1;
                    ci = (int)i;
                    cj = (int)j;
                    ck = (int)k;
                    sc.rows[lane][0] = __ldg(G.links + flat(G, i, j, k));
                } else {
                    int64_t i0 = (int64_t)g[0], j0 = (int64_t)g[1], kk0 = (int64_t)g[2];
                    if (i0 > G.Dx - 2) i0 = G.Dx - 2;
                    if (j0 > G.Dy - 2) j0 = G.Dy - 2;
                    if (kk0 > G.Dz - 2) kk0 = G.Dz - 2;
                    ci = (int)i0;
                    cj = (int)j0;
                    ck = (int)kk0;
                    f0 = (float)(g[0] - (double)i0);
                    f1 = (float)(g[1] - (double)j0);
                    f2 = (float)(g[2] - (double)kk0);
                    const int32_t *lb = G.links + flat(G, i0, j0, kk0);
                    const int64_t sy = G.Dz, sx = (int64_t)G.Dy * G.Dz;
                    int4 ra4, rb4;
                    ra4.x = __ldg(lb);
                    ra4.y = __ldg(lb + 1);
                    ra4.z = __ldg(lb + sy);
                    ra4.w = __ldg(lb + sy + 1);
                    rb4.x = __ldg(lb + sx);
                    rb4.y = __ldg(lb + sx + 1);
                    rb4.z = __ldg(lb + sx + sy);
                    rb4.w = __ldg(lb + sx + sy + 1);
                    *reinterpret_cast<int4 *>(&sc.rows[lane][0]) = ra4;
                    *reinterpret_cast<int4 *>(&sc.rows[lane][4]) = rb4;
                }
            }
            // move code vs the previous included sample (this chunk or carried)
            const unsigned below = mask & lt_mask;
            const int pl = below ? 31 - __clz(below) : lane;
            const int qi = __shfl_sync(PLX_FULL_MASK, ci, pl);
            const int qj = __shfl_sync(PLX_FULL_MASK, cj, pl);
            const int qk = __shfl_sync(PLX_FULL_MASK, ck, pl);
            int mv = 0;
            if (incl) {
                const bool hasp = below != 0u || pvalid;
                const int pi = below ? qi : pci, pj = below ? qj : pcj, pk = below ? qk : pck;
                if (!hasp) {
                    mv = MV_FAR;
                } else {
                    const int di = ci - pi, dj = cj - pj, dk = ck - pk;
                    if (di | dj | dk) {
                        const bool adj = !NEAREST && di >= -1 && di <= 1 && dj >= -1 && dj <= 1 &&
                                         dk >= -1 && dk <= 1;
                        mv = adj ? (MV_ADJ | ((di + 1) << 4) | ((dj + 1) << 2) | (dk + 1)) : MV_FAR;
                    }
                }
                sc.mv[lane] = mv;
            }
            // flip in effect when sample `lane` is added: carried ^ prefix xor
            int fx = incl ? axis_bits(mv) : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(PLX_FULL_MASK, fx, off);
                if (lane >= off) fx ^= y;
            }
            const int fl = cflip ^ fx;
            if (incl) {
                const float gk[4] = {(float)gsig, c0 > 0.0 ? (float)(up0 * wi) : 0.f,
                                     c1 > 0.0 ? (float)(up1 * wi) : 0.f,
                                     c2 > 0.0 ? (float)(up2 * wi) : 0.f};
                if (NEAREST) {
#pragma unroll
                    for (int L = 0; L < 32; ++L) sc.val[L][lane] = L < 4 ? gk[L] : 0.f;
                } else {
                    float wq[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        wq[e] = ((e & 4) ? f0 : 1.f - f0) * ((e & 2) ? f1 : 1.f - f1) *
                                ((e & 1) ? f2 : 1.f - f2);
#pragma unroll
                    for (int L = 0; L < 32; ++L) {
                        // lane L's corner is (L/4) ^ fl; select among the 8 weights
                        const int e = (L >> 2) ^ fl;
                        float w = wq[0];
#pragma unroll
                        for (int ee = 1; ee < 8; ++ee) w = e == ee ? wq[ee] : w;
                        sc.val[L][lane] = w * gk[L & 3];
                    }
                }
            }
            // carry to the next chunk
            const int hl = 31 - __clz(mask);   // mask != 0 for recorded chunks
            cflip = __shfl_sync(PLX_FULL_MASK, fl, hl);
            pci = __shfl_sync(PLX_FULL_MASK, ci, hl);
            pcj = __shfl_sync(PLX_FULL_MASK, cj, hl);
            pck = __shfl_sync(PLX_FULL_MASK, ck, hl);
            pvalid = true;
            __syncwarp();
            // ---- serial, in sample order: moves (flushes) + one add ----
            unsigned m = mask;
            while (m) {
                const int j = __ffs(m) - 1;
                m &= m - 1;
                const int mvj = sc.mv[j];
                if (mvj) ra.move(mvj, sc, j, out.grad, out.tmask, lane);
                ra.acc += sc.val[lane][j];
            }
            __syncwarp();
        }
        ra.flush_all(out.grad, out.tmask, lane);
        ray += nslots;
    }
    if (O.stats && lane == 0) {
        atomicAdd(O.stats + 0, (unsigned long long)st_pos);
        atomicAdd(O.stats + 1, (unsigned long long)st_samp);
        atomicAdd(O.stats + 2, (unsigned long long)st_chunks);
        atomicAdd(O.stats + 3, (unsigned long long)st_rays);
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

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;

bool grid_ok(const plx_grid *g) {
    return g && g->links && g->dims[0] >= 2 && g->dims[1] >= 2 && g->dims[2] >= 2 &&
           (g->rows == 0 || (g->table && g->density)) && g->dims[0] < (1 << 21) && g->dims[1] < (1 << 21) &&
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

// Minimum resident 128-thread blocks per SM the backward is compiled for:
// 4 / 5 / 6 = register budget 128 / 96 / 80 per thread (16 / 20 / 24
// warps per SM); PLX_BWD_MINB selects, default 4.
int bwd_minb() {
    static int m = 0;
    if (!m) {
        const char *e = getenv("PLX_BWD_MINB");
        const int v = e ? atoi(e) : 0;
        m = (v == 5 || v == 6) ? v : 4;
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
    switch (bwd_minb()) {
        case 5: return bwd_blocks_per_sm_t<5>(o);
        case 6: return bwd_blocks_per_sm_t<6>(o);
        default: return bwd_blocks_per_sm_t<4>(o);
    }
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
    int64_t slots, nrec, nchunk, bytes, off_att, off_c, off_sig, off_meta;
};

ScratchLayout layout(const plx_grid *g, const plx_render_opts *o, int64_t n_rays) {
    ScratchLayout L;
    int64_t blocks = (int64_t)num_sms() * bwd_blocks_per_sm(o);
    const int64_t need = (n_rays + kWarps - 1) / kWarps;
    if (n_rays > 0 && need < blocks) blocks = need;
    L.slots = blocks * kWarps;
    L.nrec = max_records(g, o->step);
    L.nchunk = L.nrec / 32 + 2;
    L.off_att = 256;
    L.off_c = L.off_att + L.slots * L.nrec * (int64_t)sizeof(double);
    L.off_c = (L.off_c + 15) & ~(int64_t)15;
    L.off_sig = L.off_c + L.slots * L.nrec * (int64_t)sizeof(float4);
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
    KOpts K{o->step, o->stop_thresh, {o->bg[0], o->bg[1], o->bg[2]},
            reinterpret_cast<unsigned long long *>(o->stats)};
    cudaStream_t s = (cudaStream_t)stream;
    Scratch S{};
    int64_t blocks;
    if (MODE == BWD) {
        const ScratchLayout L = layout(g, o, rays->n);
        if (scratch_bytes < L.bytes) return PLX_EINVAL;
        char *base = reinterpret_cast<char *>(scratch);
        S.counter = reinterpret_cast<int *>(base);
        S.rec_att = reinterpret_cast<double *>(base + L.off_att);
        S.rec_c = reinterpret_cast<float4 *>(base + L.off_c);
        S.rec_sig = reinterpret_cast<double *>(base + L.off_sig);
        S.meta = reinterpret_cast<uint2 *>(base + L.off_meta);
        S.nrec = L.nrec;
        S.nchunk = L.nchunk;
        blocks = L.slots / kWarps;
        if (cudaMemsetAsync(S.counter, 0, sizeof(int), s) != cudaSuccess) return PLX_ECUDA;
    } else {   // static grid-stride over rays, occupancy-sized grid
        blocks = (rays->n + kWarps - 1) / kWarps;
        const int64_t cap = (int64_t)num_sms() * 8;
        if (blocks > cap) blocks = cap;
    }
    const bool ABSF = MODE != MAXW && o->absolute;
    dim3 grid((unsigned)blocks);
    if (MODE != BWD) launch_variant<MODE, 6>(o, ABSF, grid, s, G, R, K, out, S);
    else if (bwd_minb() == 5) launch_variant<MODE, 5>(o, ABSF, grid, s, G, R, K, out, S);
    else if (bwd_minb() == 6) launch_variant<MODE, 6>(o, ABSF, grid, s, G, R, K, out, S);
    else launch_variant<MODE, 4>(o, ABSF, grid, s, G, R, K, out, S);
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
