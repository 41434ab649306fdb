// plx_render.cu -- ray-march kernels for sm_100a: forward render, the fused
// forward + MSE + backward scatter, and the max-weight accumulation.
//
// Reference: pkg/src/plenoxel/_kernels.py render_forward (K:173-238),
// render_backward (K:241-411), max_weight_accum (K:414-453).
//
// Parallel decomposition (B200-first, not a translation of the sequential
// loop): one warp per ray.  The march is walked in chunks of 32 consecutive
// positions, one lane per position: stencil through `links`, float64
// trilinear sigma from the density array, then the chunk is composited with
// warp scans (product scan of exp(-sigma*delta) for "relative", sum scan of
// alpha for "absolute"); early termination is a ballot on T < stop_thresh
// (T is monotone, so the first such lane is the reference's break point).
//
// The fused backward (bwd_kernel) runs three phases per ray:
//   A  sigma march + compositing over positions; each composited sample is
//      appended to the warp's record list {att, T, w, cell, f, rows};
//   B  colour over the DENSE sample list (32 samples per iteration, every
//      lane busy): 8 SH rows gathered as float4, f32 FMAs, rgb = sum w c+;
//   C  the reverse sweep over the dense list: suffix S_i = rgb - prefix_i
//      (float64, |error| ~ 1e-16 |rgb|), dL/dsigma and dL/dc, and the
//      lane-distributed scatter accumulator (LaneAcc) that reduces each
//      touched gradient row once per ray visit with red.global.add.v4.f32.
// Only ~1/8 of march positions are composited samples on the training
// grids, so B and C iterate over samples, not positions.
#include <stdlib.h>

#include "plx_camera.cuh"
#include "plx_common.cuh"
#include "plx_internal.h"
#include "plx_msi.cuh"

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
    const int64_t *idx_off;   // optional device offset added to idx (graph replay)
    CamPool C;                // camera pool (C.cams != nullptr): rays generated
    int64_t base;             // pool row of batch ray 0 when idx == nullptr
};

// Pool row of batch ray `ray`.
__device__ __forceinline__ int64_t ray_src(const RayArgs &R, int64_t ray) {
    return R.idx ? R.idx[ray] : R.base + ray;
}

// March origin / direction of pool row src: the arrays, or the camera pool
// (camera.py:91-134, 292-314 on the device, plx_camera.cuh).
__device__ __forceinline__ void ray_od(const RayArgs &R, int64_t src, double *o, double *d) {
    if (R.C.cams) {
        cam_march_ray(R.C, src, o, d);
        return;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        o[a] = __ldg(R.origins + 3 * src + a);
        d[a] = __ldg(R.dirs + 3 * src + a);
    }
}

// March origin / direction and the unit view (SH) direction of pool row src
// in one go (the camera ray is generated once).
__device__ __forceinline__ void ray_od_vd(const RayArgs &R, int64_t src, double *o, double *d,
                                          double *v) {
    if (R.C.cams) {
        const double *cam = cam_pixel_ray(R.C, src, o, v);
#pragma unroll
        for (int a = 0; a < 3; ++a) d[a] = v[a];
        if (R.C.scale != 1.0) {
#pragma unroll
            for (int a = 0; a < 3; ++a) o[a] = o[a] * R.C.scale;
        }
        if (R.C.ndc) cam_to_ndc(cam, o, d);
        return;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        o[a] = __ldg(R.origins + 3 * src + a);
        d[a] = __ldg(R.dirs + 3 * src + a);
        v[a] = __ldg(R.viewdirs + 3 * src + a);
    }
}

// Unit view (SH) direction of pool row src.
__device__ __forceinline__ void ray_vd(const RayArgs &R, int64_t src, double *v) {
    if (R.C.cams) {
        cam_view_dir(R.C, src, v);
        return;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) v[a] = __ldg(R.viewdirs + 3 * src + a);
}

// Target (gt colour, or the upstream dL/dC) of pool row src, channel c.
__device__ __forceinline__ double ray_tgt(const RayArgs &R, int64_t src, int c) {
    if (R.C.cams && !R.target) return (double)__ldg(R.C.rgb + 3 * src + c);
    return __ldg(R.target + 3 * src + c);
}

// Stencil rows of a recorded cell on an identity-linked grid (row = lattice
// point): computed, so the march does not store them and the colour and
// scatter kernels do not load them.
template <bool NEAREST>
__device__ __forceinline__ void identity_rows(const DGrid &G, int4 cl, int32_t *rows);

// idx + *idx_off: the batch as a device-resident slice of a fixed buffer
__device__ __forceinline__ const int64_t *ray_index(const RayArgs &R) {
    return (R.idx && R.idx_off) ? R.idx + *R.idx_off : R.idx;
}

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
    int bgmode;   // 360 backward: msi_bg_kernel owns rgb / mse and the background terms
};

// One march position evaluated by one lane.
struct Sample {
    int32_t rows[8];
    double f[3];   // fractional lattice offsets; weights via stencil_w
    double sig, att, dlt;
    float c[3];    // pre-clamp colour (K:305)
    bool incl;
};

// Evaluate position si for the forward render / max-weight (K:200-229):
// stencil, sigma, and for included samples (sigma > 0, K:211) the colour.
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
    int ijk[3];
    bool rows_ok;
    double sig;
    if (!sigma_at<NEAREST>(G, g, s.f, ijk, s.rows, sig, rows_ok)) return;
    s.sig = sig;
    if (!(sig > 0.0)) return;   // K:211 (render_forward / max_weight_accum)
    s.incl = true;
    s.att = exp(-sig * s.dlt);
    if (!rows_ok) load_rows<NEAREST>(G, ijk, s.rows);
    if (MODE == MAXW) return;
    colour_at_f32<NEAREST>(G, s.rows, s.f, bf, s.c);
}

__device__ __forceinline__ double relu(double x) { return x > 0.0 ? x : 0.0; }

// Record list of the backward (SoA; capacity cap per ray = every march
// position of the longest chord, R:67-69; a batch is processed in waves of
// rays so that the records fit a fixed budget).  The march kernel appends
// one record per composited sample; the colour kernel adds the colour and
// per-segment sums; the scatter kernel consumes them.  These replace the
// reference's per-call s_t / s_dlt / s_sig / s_T / s_w / s_cpre scratch
// (K:259-264, R:277-278).
struct Scratch {
    int *counter;      // ray scheduler of the march kernel (zeroed per wave);
                       // counter[2]: colour segment scheduler
    int64_t cap;       // records per ray
    int nseg_max;      // segments (32 records) per ray
    int *ns;           // [rays] composited samples
    int *seg_first;    // [rays] first segment of the ray (its segments are contiguous)
    int *seg_ray;      // [segments] ray of each segment
    int *nseg_total;   // segments allocated so far (zeroed per wave)
    double *ray_d;     // [rays][3] {T after the march, delta and index of the last position}
    float4 *basis;     // [rays][3] the ray's 9 SH basis values (K:27-37, f32) + 3 pad
    double *att;       // exp(-sigma delta)                    [rays][cap]
    double *T;         // transmittance before the sample
    double *w;         // compositing weight
    float4 *c;         // pre-clamp colour (colour kernel)
    int4 *cell;        // {i, j, k, position index}
    float4 *f;         // fractional offsets in the cell
    int4 *rows;        // 8 stencil rows                       [rays][cap][2]
    double *sig;       // sigma (Cauchy term only)
    double *seg_sum;   // [segments][6] {sum w c+ (RGB), sum c+ (bn - bi) (RGB)}
    double *rgb_add;   // 360 mode: [rays][3] background colour T_fg C_bg (replaces T bg)
    double *bup;       // 360 mode: [rays] beta-regulariser upstream (K:827-833)
    // spatial processing order of the segments (seg_order_*): ord[q] =
    // {segment, ray} of the q-th segment the colour / scatter kernels take;
    // nullptr = allocation order
    int2 *ord;
    int *seg_key;      // [segments] spatial bucket of each segment
    int *bucket;       // [kBuckets] counts, then (scan) cursors; zeroed by the march
    // packed records (pack != 0): the sample's cell (i | j << pk_sy | k <<
    // pk_sz) and its last-position flag (bit 31) ride in the unused 4th float
    // of f, and the 16-byte cell array is neither written nor read
    int pack, pk_sy, pk_sz;
};

// The record's cell {i, j, k, w} -- w = the position index (unpacked) or the
// last-position flag (packed) -- and its fractional offsets.
__device__ __forceinline__ void load_cell_f(const Scratch &S, int64_t k, bool with_f, int4 &cl,
                                            float4 &f4) {
    if (S.pack) {
        f4 = S.f[k];
        const uint32_t u = __float_as_uint(f4.w);
        const uint32_t my = (1u << (S.pk_sz - S.pk_sy)) - 1u, mz = (1u << (31 - S.pk_sz)) - 1u;
        cl = make_int4((int)(u & ((1u << S.pk_sy) - 1u)), (int)((u >> S.pk_sy) & my),
                       (int)((u >> S.pk_sz) & mz), (int)(u >> 31));
    } else {
        cl = S.cell[k];
        if (with_f) f4 = S.f[k];
    }
}

// Whether a record is the ray's last march position (K:200-205 delta).
__device__ __forceinline__ bool rec_is_last(const Scratch &S, const int4 &cl, double last_si) {
    return S.pack ? cl.w != 0 : (double)cl.w == last_si;
}

// The ray's colour total sum_w w c+ from its segment sums, in the order every
// consumer of the sums uses (short rays: in segment order per lane; long
// rays: lane-strided partial sums + a warp reduction), so all of them see
// bit-identical totals.
__device__ __forceinline__ void ray_colour_totals(const Scratch &S, int64_t s0, int64_t s1,
                                                  int lane, double &C0, double &C1, double &C2) {
    C0 = C1 = C2 = 0.0;
    const bool few = s1 - s0 <= 4;
    for (int64_t t = few ? s0 : s0 + lane; t < s1; t += few ? 1 : 32) {
        const double *p = S.seg_sum + 6 * t;
        C0 += p[0];
        C1 += p[1];
        C2 += p[2];
    }
    if (!few) {
        C0 = warp_sum(C0);
        C1 = warp_sum(C1);
        C2 = warp_sum(C2);
    }
}

// The q-th segment of the processing order (allocation order, or the spatial
// order of seg_place_kernel for large waves) and its ray.
__device__ __forceinline__ void seg_at(const Scratch &S, int64_t q, int64_t &sg, int &ray) {
    if (S.ord) {
        const int2 e = S.ord[q];
        sg = e.x;
        ray = e.y;
    } else {
        sg = q;
        ray = S.seg_ray[q];
    }
}

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
// DIAG (diagnostic builds, -DPLX_DIAG only; profiles/r2b_diag.md): 1 = no
// reductions, 2 = reductions into an L2-resident 8 MB window.
template <bool NEAREST, int DIAG = 0>
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
            if (DIAG == 1) {
                if (v0 == 1.2345e-30f) red_add_v4(grad + 4 * quad, v0, v1, v2, v3);
            } else if (DIAG == 2) {
                if (v0 != 0.f || v1 != 0.f || v2 != 0.f || v3 != 0.f)
                    red_add_v4(grad + (int64_t)(r & 0xffff) * PLX_STRIDE + 4 * quad, v0, v1, v2, v3);
            } else {
                if (quad == 0) tmask[r] = 1;
                if (v0 != 0.f || v1 != 0.f || v2 != 0.f || v3 != 0.f)
                    red_add_v4(grad + (int64_t)r * PLX_STRIDE + 4 * quad, v0, v1, v2, v3);
            }
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

// Dead-brick probe stride of the march (positions between probes).
#ifndef PLX_LOOK
#define PLX_LOOK 8
#endif
constexpr int kLook = PLX_LOOK;

// Empty-space skip of the march (sparse grids with a dead-brick mask),
// called after a chunk that composited nothing: returns the next chunk
// start (32-aligned with base).
__device__ __forceinline__ int64_t skip_dead_chunks(const DGrid &G, const RayMarch &rm, double step,
                                                    int64_t base, int lane) {
    // Empty space: lane l probes position base + l*kLook.  Every
    // lattice coordinate is monotone along the ray, so the
    // positions between two consecutive probes lie in the box of
    // the probes' bricks; when all bricks of that box are dead
    // (same brick, a face neighbour, or an edge neighbour plus
    // its two corner bricks) so is every position between: the
    // leading run of such intervals is skipped without sample
    // math or gathers (exact).
    const int64_t sp = base + (int64_t)lane * kLook;
    int bx = -1, by = 0, bz = 0;
    bool dead = false;
    if (sp < rm.nsamp) {
        double tt, dd, gg[3];
        sample_coords(rm, G, step, sp, tt, dd, gg);
        brick_xyz(G, gg, bx, by, bz);
        dead = brick_is_dead(G, (bx * G.By + by) * G.Bz + bz);
    }
    // the interval to the next probe is certainly dead when both
    // ends are dead and the bricks between (per-axis monotone:
    // inside the box of the two) are: same brick, a face
    // neighbour, or an edge neighbour whose two corner bricks
    // are dead too
    const int nx = __shfl_down_sync(PLX_FULL_MASK, bx, 1);
    const int ny = __shfl_down_sync(PLX_FULL_MASK, by, 1);
    const int nz = __shfl_down_sync(PLX_FULL_MASK, bz, 1);
    const unsigned dm = __ballot_sync(PLX_FULL_MASK, dead);
    bool cert = lane < 31 && dead && ((dm >> (lane + 1)) & 1u);
    if (cert) {
        const int ax = nx - bx, ay = ny - by, az = nz - bz;
        const int nd = (ax != 0) + (ay != 0) + (az != 0);
        if (ax < -1 || ax > 1 || ay < -1 || ay > 1 || az < -1 || az > 1 || nd == 3) {
            cert = false;
        } else if (nd == 2) {
            // the ray passes through one of the two other bricks
            // of the 2x2 box: b with the first differing axis
            // moved, or with the second one moved
            const int f = ax ? 0 : 1, sc = az ? 2 : 1;
            const int c1x = f == 0 ? nx : bx, c1y = f == 1 ? ny : by;
            const int c2y = sc == 1 ? ny : by, c2z = sc == 2 ? nz : bz;
            cert = brick_is_dead(G, (c1x * G.By + c1y) * G.Bz + bz) &&
                   brick_is_dead(G, (bx * G.By + c2y) * G.Bz + c2z);
        }
    }
    const unsigned cd = __ballot_sync(PLX_FULL_MASK, cert);
    const int nskip = __ffs(~cd) - 1;   // leading certain-dead intervals
    // whole chunks only: chunks keep their 32-aligned positions,
    // so the compositing scans (and their rounding) are those of
    // the march without skipping -- results are bit-identical
    return base + (int64_t)(nskip * kLook / 32) * 32;
}

// Forward render / max-weight: one pass over the positions (K:173-238,
// K:414-453).  Static grid-stride over rays.
template <int MODE, bool ABS, bool NEAREST>
__global__ void __launch_bounds__(128, 6)
    march_kernel(DGrid G, RayArgs R, KOpts O, Outs out) {
    const int lane = threadIdx.x & 31;
    const int64_t slot = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t nslots = (int64_t)gridDim.x * (blockDim.x >> 5);
    unsigned st_pos = 0, st_samp = 0, st_chunks = 0, st_rays = 0;   // warp-uniform
    for (int64_t ray = slot; ray < R.n; ray += nslots) {
        ++st_rays;
        const int64_t src = ray_src(R, ray);
        RayMarch rm;
        ray_od(R, src, rm.o, rm.d);
        float bf[9];
        if (MODE == FWD) {
            double basis[9], vd[3];
            ray_vd(R, src, vd);
            sh_basis9(vd[0], vd[1], vd[2], basis);
#pragma unroll
            for (int b = 0; b < 9; ++b) bf[b] = (float)basis[b];
        }
        const double jit = (MODE == FWD && R.jitter) ? R.jitter[ray] : 0.0;
        ray_march_setup(rm, G, O.step, jit);
        double T = 1.0, A = 0.0, C0 = 0.0, C1 = 0.0, C2 = 0.0, wsum = 0.0;
        bool stopped = false, idle = true;
        for (int64_t base = 0; base < rm.nsamp && !stopped; base += 32) {
            if (!NEAREST && G.brick_dead && idle) base = skip_dead_chunks(G, rm, O.step, base, lane);
            Sample s;
            eval_sample<MODE, NEAREST>(G, rm, O.step, base + lane, bf, s);
            const int npos = (int)min((int64_t)32, rm.nsamp - base);
            st_chunks += 1;
            idle = !__any_sync(PLX_FULL_MASK, s.incl);
            if (idle) {
                st_pos += npos;
                continue;
            }
            double Ti, wi;
            composite_chunk<(MODE == MAXW ? false : ABS)>(s.incl, s.att, lane, O.stop, T, A, Ti,
                                                           wi, stopped);
            const unsigned im = __ballot_sync(PLX_FULL_MASK, s.incl);
            st_pos += stopped ? 32 - __clz(im) : npos;
            st_samp += __popc(im);
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
            if (s.incl) {   // K:224-229: only the positive part is accumulated
                x0 = wi * relu((double)s.c[0]);
                x1 = wi * relu((double)s.c[1]);
                x2 = wi * relu((double)s.c[2]);
                xw = wi;
            }
            C0 += warp_sum(x0);
            C1 += warp_sum(x1);
            C2 += warp_sum(x2);
            wsum += warp_sum(xw);
        }
        if (MODE == FWD && lane == 0) {   // K:234-238
            out.rgb[3 * ray + 0] = C0 + T * O.bg[0];
            out.rgb[3 * ray + 1] = C1 + T * O.bg[1];
            out.rgb[3 * ray + 2] = C2 + T * O.bg[2];
            if (out.trans) out.trans[ray] = T;
            if (out.wsum) out.wsum[ray] = wsum;
        }
    }
    if (O.stats && lane == 0) {
        atomicAdd(O.stats + 0, (unsigned long long)st_pos);
        atomicAdd(O.stats + 1, (unsigned long long)st_samp);
        atomicAdd(O.stats + 2, (unsigned long long)st_chunks);
        atomicAdd(O.stats + 3, (unsigned long long)st_rays);
    }
}

// ---------------------------------------------------------------------------
// The fused forward + MSE + backward (K:241-411) as three kernels:
//   march_bwd_kernel   one warp per ray (dynamic scheduling): the sigma march
//                      and compositing over positions; every composited
//                      sample is appended to the ray's record list.
//   colour_kernel      one warp per 32-record segment of any ray: colours of
//                      the samples (8 SH rows x 7 float4, f32 FMAs) and the
//                      segment's sums sum w c+ (and the absolute form's
//                      sum c+ (bn - bi)).
//   scatter_kernel     one warp per segment: rgb / upstream from the ray's
//                      segment sums, the reverse-sweep suffix from the sums
//                      of the segments before it, dL/dsigma and dL/dc, and
//                      the lane-distributed scatter accumulator (flushed at
//                      the segment's end).
// The colour and scatter work -- ~24 us per 32 samples of dependent gathers
// and in-order flushes -- is thus spread over all warps instead of being
// serialised on the warp that marched a long ray (the single-kernel version
// ran its last half with fewer than half of its warps active).
// The march kernel allocates each ray's segments (contiguous, one atomic per
// ray) and finishes the rays that composited nothing.

#ifdef PLX_TIMELINE
__device__ unsigned long long g_timeline[2 * 8192];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// ---------------------------------------------------------------------------
// Spatial order of the segments, for large waves.  A wave touches each SH /
// gradient row from several rays at unrelated times; once the wave's row
// working set exceeds L2, the colour kernel's row gathers and the scatter's
// red.add row fills mostly miss L2 when segments are taken in allocation
// (ray) order.  Processing segments bucketed by the 3-D location of their
// first sample (a 16^3 Morton grid over the lattice) keeps the segments in
// flight spatially compact, so rows shared by crossing rays are gathered /
// reduced while still in L2.  Counting sort, three small kernels between the
// march and the colour kernel; the order within a bucket is arbitrary
// (results do not depend on it beyond f32 atomic order).  Measured (C5
// 512^3, 32 GiB waves): 2^20 rays 36.6 -> 40.4 M rays/s, 2^18 30.9 -> 33.4,
// 2^16 +2 %, equal at 2^15; at C2 (5000 rays, rays share few rows) the sort
// costs 12 us for no kernel gain, so waves below kSegOrderMinRays skip it.
// 8^3-cell buckets and keying on the middle sample measured the same.
constexpr int kBucketBits = 4;
constexpr int kBuckets = 1 << (3 * kBucketBits);
constexpr int64_t kSegOrderMinRays = 49152;

__device__ __forceinline__ int spread3(int v) {
    int r = 0;
#pragma unroll
    for (int b = 0; b < kBucketBits; ++b) r |= ((v >> b) & 1) << (3 * b);
    return r;
}

// Segments are keyed and counted in tiles of kSegTile per block: the counts
// go through a shared histogram first, so a bucket that many segments share
// (the occupied regions) takes one global atomic per tile instead of one per
// segment (the per-segment atomics serialised on the hot buckets).
constexpr int kSegTile = 2048;

__global__ void __launch_bounds__(256) seg_key_kernel(Scratch S, int shx, int shy, int shz) {
    __shared__ int hist[kBuckets];
    const int64_t nseg = *S.nseg_total;
    for (int64_t t0 = (int64_t)blockIdx.x * kSegTile; t0 < nseg; t0 += (int64_t)gridDim.x * kSegTile) {
        for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t sg = t0 + threadIdx.x; sg < nseg && sg < t0 + kSegTile; sg += blockDim.x) {
            const int ray = S.seg_ray[sg];
            const int64_t j0 = (sg - S.seg_first[ray]) * 32;
            int4 c;
            float4 fd;
            load_cell_f(S, (int64_t)ray * S.cap + j0, false, c, fd);
            const int key =
                (spread3(c.x >> shx) << 2) | (spread3(c.y >> shy) << 1) | spread3(c.z >> shz);
            S.seg_key[sg] = key;
            atomicAdd(hist + key, 1);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
            if (hist[i]) atomicAdd(S.bucket + i, hist[i]);
        __syncthreads();
    }
}

// exclusive scan of the kBuckets counts in place (one block of 1024 threads)
__global__ void __launch_bounds__(1024) seg_scan_kernel(Scratch S) {
    constexpr int PER = kBuckets / 1024;
    __shared__ int warp_tot[32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    int v[PER], sum = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        v[i] = S.bucket[PER * t + i];
        sum += v[i];
    }
    int x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(PLX_FULL_MASK, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
        int y = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int z = __shfl_up_sync(PLX_FULL_MASK, y, o);
            if (lane >= o) y += z;
        }
        warp_tot[lane] = y;
    }
    __syncthreads();
    int excl = x - sum + (w ? warp_tot[w - 1] : 0);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        S.bucket[PER * t + i] = excl;
        excl += v[i];
    }
}

// Places the segments of a tile: ranks within the tile from a shared
// histogram, one global atomic per (tile, bucket) reserves the tile's range
// of the bucket, then every segment writes its slot.
__global__ void __launch_bounds__(256) seg_place_kernel(Scratch S) {
    __shared__ int hist[kBuckets];
    constexpr int PER = kSegTile / 256;
    const int64_t nseg = *S.nseg_total;
    for (int64_t t0 = (int64_t)blockIdx.x * kSegTile; t0 < nseg; t0 += (int64_t)gridDim.x * kSegTile) {
        for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        int key[PER], rank[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int64_t sg = t0 + threadIdx.x + (int64_t)u * 256;
            key[u] = -1;
            if (sg < nseg) {
                key[u] = S.seg_key[sg];
                rank[u] = atomicAdd(hist + key[u], 1);
            }
        }
        __syncthreads();
        for (int i = threadIdx.x; i < kBuckets; i += blockDim.x)
            if (hist[i]) hist[i] = atomicAdd(S.bucket + i, hist[i]);
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int64_t sg = t0 + threadIdx.x + (int64_t)u * 256;
            if (key[u] >= 0) S.ord[hist[key[u]] + rank[u]] = make_int2((int)sg, S.seg_ray[sg]);
        }
        __syncthreads();
    }
}

template <bool ABS, bool NEAREST, int MINB>
__global__ void __launch_bounds__(128, MINB)
    march_bwd_kernel(DGrid G, RayArgs R, KOpts O, Outs out, Scratch S) {
    R.idx = ray_index(R);
    const int lane = threadIdx.x & 31;
    double mse_part = 0.0;
    const int64_t slot = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    unsigned st_pos = 0, st_samp = 0, st_chunks = 0, st_rays = 0;   // warp-uniform
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool cauchy = S.sig != nullptr;
    if (S.bucket && blockIdx.x == 0)   // counts of seg_key_kernel (runs after this kernel)
        for (int i = threadIdx.x; i < kBuckets; i += blockDim.x) S.bucket[i] = 0;
#ifdef PLX_TIMELINE
    const unsigned long long t_start = gtimer();
#endif
    for (;;) {
        int rr = 0;   // dynamic scheduling: rays differ widely in length
        if (lane == 0) rr = atomicAdd(S.counter, 1);
        const int64_t ray = __shfl_sync(PLX_FULL_MASK, rr, 0);
        if (ray >= R.n) break;
        ++st_rays;
        const int64_t src = ray_src(R, ray);
        RayMarch rm;
        {
            // the ray's SH basis (K:27-37, f64 -> f32 for the colour FMAs),
            // stored once for the colour and scatter kernels
            double vd[3], basis[9];
            ray_od_vd(R, src, rm.o, rm.d, vd);
            sh_basis9(vd[0], vd[1], vd[2], basis);
            float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int k = 0; k < 3; ++k)   // static indices: basis stays in registers
                if (lane == k)
                    b4 = make_float4((float)basis[3 * k], (float)basis[3 * k + 1],
                                     (float)basis[3 * k + 2], 0.f);
            if (lane < 3) S.basis[3 * ray + lane] = b4;
        }
        const double jit = R.jitter ? R.jitter[ray] : 0.0;
        ray_march_setup(rm, G, O.step, jit);
        const int64_t rb = ray * S.cap;   // this ray's record block
        double T = 1.0, A = 0.0;
        int ns = 0;
        bool stopped = false;
        bool idle = true;   // the previous chunk composited nothing
        for (int64_t base = 0; base < rm.nsamp && !stopped; base += 32) {
            if (!NEAREST && G.brick_dead && idle) base = skip_dead_chunks(G, rm, O.step, base, lane);
            const int64_t si = base + lane;
            bool incl = false;
            double att = 1.0, sig = 0.0, t, dlt, g[3], fd[3];
            int32_t rows[8];
            int ijk[3];
            bool rows_ok = true;
            if (si < rm.nsamp) {
                sample_coords(rm, G, O.step, si, t, dlt, g);
                // _sigma_at (K:126-135), float64, reference order
                if (sigma_at<NEAREST>(G, g, fd, ijk, rows, sig, rows_ok)) {
                    incl = sig >= 0.0;   // K:293: recorded unless sigma < 0
                    if (incl) att = exp(-sig * dlt);
                }
            }
            const int npos = (int)min((int64_t)32, rm.nsamp - base);
            st_chunks += 1;
            idle = !__any_sync(PLX_FULL_MASK, incl);
            if (idle) {
                st_pos += npos;
                continue;
            }
            double Ti, wi;
            composite_chunk<ABS>(incl, att, lane, O.stop, T, A, Ti, wi, stopped);
            const unsigned m = __ballot_sync(PLX_FULL_MASK, incl);
            st_pos += stopped ? 32 - __clz(m) : npos;
            st_samp += __popc(m);
            if (incl) {
                const int64_t k = rb + ns + __popc(m & lt_mask);
                S.att[k] = att;
                S.T[k] = Ti;
                S.w[k] = wi;
                if (S.pack) {
                    const uint32_t u = (uint32_t)ijk[0] | ((uint32_t)ijk[1] << S.pk_sy) |
                                       ((uint32_t)ijk[2] << S.pk_sz) |
                                       (si == rm.nsamp - 1 ? 0x80000000u : 0u);
                    S.f[k] = NEAREST ? make_float4(0.f, 0.f, 0.f, __uint_as_float(u))
                                     : make_float4((float)fd[0], (float)fd[1], (float)fd[2],
                                                   __uint_as_float(u));
                } else {
                    S.cell[k] = make_int4(ijk[0], ijk[1], ijk[2], (int)si);
                    if (!NEAREST) S.f[k] = make_float4((float)fd[0], (float)fd[1], (float)fd[2], 0.f);
                }
                if (!G.identity) {   // identity grids: rows follow from the cell
                    if (!rows_ok) load_rows<NEAREST>(G, ijk, rows);
                    if (!NEAREST) {
                        S.rows[2 * k] = make_int4(rows[0], rows[1], rows[2], rows[3]);
                        S.rows[2 * k + 1] = make_int4(rows[4], rows[5], rows[6], rows[7]);
                    } else {
                        S.rows[2 * k] = make_int4(rows[0], -1, -1, -1);
                    }
                }
                if (cauchy) S.sig[k] = sig;
            }
            ns += __popc(m);
        }
        // segments of 32 records, contiguous per ray, handed to the colour
        // and scatter kernels through seg_ray
        const int nseg = (ns + 31) >> 5;
        int sbase = 0;
        if (lane == 0) {
            S.ns[ray] = ns;
            S.ray_d[3 * ray] = T;
            S.ray_d[3 * ray + 1] = rm.L - O.step * (double)(rm.nsamp - 1);   // K:200-205
            S.ray_d[3 * ray + 2] = (double)(rm.nsamp - 1);
            if (nseg) sbase = atomicAdd(S.nseg_total, nseg);
            S.seg_first[ray] = sbase;
            if (ns == 0 && !out.bgmode) {   // nothing composited: rgb = T bg (K:324-341), no gradient
                const double c0 = T * O.bg[0], c1 = T * O.bg[1], c2 = T * O.bg[2];
                if (out.rgb) {
                    out.rgb[3 * ray] = c0;
                    out.rgb[3 * ray + 1] = c1;
                    out.rgb[3 * ray + 2] = c2;
                }
                if (out.mse_mode) {
                    const double e0 = c0 - ray_tgt(R, src, 0), e1 = c1 - ray_tgt(R, src, 1),
                                 e2 = c2 - ray_tgt(R, src, 2);
                    mse_part += e0 * e0 + e1 * e1 + e2 * e2;
                }
            }
        }
        sbase = __shfl_sync(PLX_FULL_MASK, sbase, 0);
        for (int k = lane; k < nseg; k += 32) S.seg_ray[sbase + k] = (int)ray;
    }
#ifdef PLX_TIMELINE
    if (lane == 0 && slot < 8192) {
        g_timeline[2 * slot] = t_start;
        g_timeline[2 * slot + 1] = gtimer();
    }
#endif
    if (O.stats && lane == 0) {
        atomicAdd(O.stats + 0, (unsigned long long)st_pos);
        atomicAdd(O.stats + 1, (unsigned long long)st_samp);
        atomicAdd(O.stats + 2, (unsigned long long)st_chunks);
        atomicAdd(O.stats + 3, (unsigned long long)st_rays);
    }
    if (lane == 0 && mse_part != 0.0) atomicAdd(out.sums + 0, mse_part);
}

// The ray's basis as stored by the march kernel.
__device__ __forceinline__ void ray_basis_rec(const Scratch &S, int64_t ray, float *bf) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float4 b = S.basis[3 * ray + k];
        bf[3 * k] = b.x;
        bf[3 * k + 1] = b.y;
        bf[3 * k + 2] = b.z;
    }
}


template <bool NEAREST>
__device__ __forceinline__ void identity_rows(const DGrid &G, int4 cl, int32_t *rows) {
    const int ijk[3] = {cl.x, cl.y, cl.z};
    load_rows<NEAREST>(G, ijk, rows);   // identity fast path: no loads
}

// Per-warp shared staging of the colour kernel: the rows of the segment's
// distinct cells and their basis dot products d = (basis . SH_R, . SH_G,
// . SH_B) (_color_at, K:138-152, factorised: colour = sum_q w_q d_q).
struct SmemColour {
    int32_t rows[32][8];    // distinct cells' stencil rows (corner order)
    int4 cell[32];          // distinct cells' lattice coordinates
    uint16_t uidx[32][8];   // (cell, corner) -> slot in d (kZeroSlot: empty corner)
    int32_t urow[256];      // the segment's distinct rows, in load order
    float4 d[257];          // d per distinct row; d[kZeroSlot] = 0
};
constexpr int kZeroSlot = 256;

// Lattice corners shared with an earlier distinct cell of the segment.  A
// ray's samples are monotone along it, so the cells containing a lattice
// point P form ONE contiguous run of the distinct-cell sequence, at most 4
// long (the ray crosses each of the 3 planes through P once).  Corner q
// (offset (q>>2, q>>1, q)&1) of cell L is corner q + ob of cell L-b iff
// off(q) + (c_L - c_{L-b}) is in {0,1}^3 -- an 8-bit mask per axis.
__device__ __forceinline__ unsigned shared_corner_mask(int4 c, int4 p, int &ob) {
    const int dx = c.x - p.x, dy = c.y - p.y, dz = c.z - p.z;
    const unsigned mx = dx == 0 ? 0xffu : dx == 1 ? 0x0fu : dx == -1 ? 0xf0u : 0u;
    const unsigned my = dy == 0 ? 0xffu : dy == 1 ? 0x33u : dy == -1 ? 0xccu : 0u;
    const unsigned mz = dz == 0 ? 0xffu : dz == 1 ? 0x55u : dz == -1 ? 0xaau : 0u;
    ob = 4 * dx + 2 * dy + dz;
    return mx & my & mz;
}

// Colours of one 32-record segment per warp.  Consecutive samples share
// cells (two per voxel at half-voxel steps), so the 8 rows of each DISTINCT
// cell are loaded once, cooperatively and coalesced: 8 lanes per row (7
// float4 + an idle lane), 4 rows per warp instruction -- 4 cache lines per
// instruction instead of up to 32 when every lane gathered its own sample's
// rows (that version ran at 70 % of the L1 throughput limit).  Each row's 3
// dot products are reduced over its 8 lanes and staged in shared memory;
// every lane then forms its sample's colour from 8 staged d's.
// DIAG 1 (diagnostic builds only): every row load from an L2-resident window.
template <bool ABS, bool NEAREST, int MINB, int DIAG = 0>
__global__ void __launch_bounds__(128, MINB)
    colour_kernel(DGrid G, RayArgs R, Scratch S) {
    R.idx = ray_index(R);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const unsigned le_mask = lane == 31 ? 0xffffffffu : (2u << lane) - 1u;
    __shared__ SmemColour smem_all[4];
    SmemColour &sm = smem_all[warp];
    const int part = lane & 7, sub = lane >> 3;   // row-load role: column quad, row slot
    const int64_t nseg = *S.nseg_total;
    // first segment static (one per warp), the rest claimed dynamically
    // (segment costs vary with their distinct cells); the next index is
    // claimed when a segment starts, so the atomic's latency hides behind
    // the segment's work.  Measured: all-static 66 / 16.4 us (early /
    // step 2000), all-dynamic 61 / 17.6, all-dynamic claiming ahead 63 / 24.6,
    // static-first claiming ahead 62.7 / 17.1.
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    // The next segment's descriptor (ray, first segment, samples, source
    // row) is prefetched in two dependent levels while this segment's rows
    // load and reduce, so the per-segment chain seg_ray -> ray fields ->
    // records -> rows pays one round trip less per level.
    int64_t nx_q = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    int64_t nx_sg = 0;
    int nx_ray = 0;
    if (nx_q < nseg) seg_at(S, nx_q, nx_sg, nx_ray);
    int nx_first = 0, nx_ns = 0;
    int64_t nx_src = 0;
    auto fetch2 = [&](int r_) {
        nx_first = S.seg_first[r_];
        nx_ns = S.ns[r_];
        nx_src = ray_src(R, r_);
    };
    if (nx_q < nseg) fetch2(nx_ray);
    int claim = 0;
    for (;;) {
        if (nx_q >= nseg) break;
        const int64_t sg = nx_sg;
        if (lane == 0) claim = atomicAdd(S.counter + 2, 1);
        const int64_t ray = nx_ray;
        const int64_t src = nx_src;
        const int j = (int)(sg - nx_first) * 32 + lane;
        const bool valid = j < nx_ns;
        float bf[9];
        ray_basis_rec(S, ray, bf);
        // this lane's 4 columns 4*part .. 4*part+3 span at most two colour
        // channels: cA feeds the first (chA), cB the second.  Per row the
        // part-0 lane then gathers R = a0+a1+a2, G = b2+a3+a4, B = b4+a5+a6.
        float cA[4], cB[4];
        {
            const int chA = part < 7 ? ((part == 0 ? 1 : 4 * part) - 1) / 9 : -1;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = 4 * part + e;   // column 0 = sigma padding; 28..31 pitch padding
                float coef = 0.f;
                int ch = -1;
                if (part < 7 && c >= 1) {
                    ch = (c - 1) / 9;
                    const int b = (c - 1) % 9;
#pragma unroll
                    for (int bb = 0; bb < 9; ++bb)
                        if (bb == b) coef = bf[bb];
                }
                cA[e] = ch >= 0 && ch == chA ? coef : 0.f;
                cB[e] = ch >= 0 && ch != chA ? coef : 0.f;
            }
        }
        const int64_t k = ray * S.cap + j;
        int4 cl = make_int4(0, 0, 0, 0);
        float4 f4 = make_float4(0.f, 0.f, 0.f, 0.f);
        int32_t rows[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
        if (valid) {
            load_cell_f(S, k, !NEAREST, cl, f4);
            if (G.identity) {
                identity_rows<NEAREST>(G, cl, rows);
            } else {
                const int4 ra = S.rows[2 * k];
                rows[0] = ra.x;
                if (!NEAREST) {
                    const int4 rb = S.rows[2 * k + 1];
                    rows[1] = ra.y;
                    rows[2] = ra.z;
                    rows[3] = ra.w;
                    rows[4] = rb.x;
                    rows[5] = rb.y;
                    rows[6] = rb.z;
                    rows[7] = rb.w;
                }
            }
        }
        // distinct cells of the segment (samples are in march order)
        const int pi = __shfl_up_sync(PLX_FULL_MASK, cl.x, 1);
        const int pj = __shfl_up_sync(PLX_FULL_MASK, cl.y, 1);
        const int pk = __shfl_up_sync(PLX_FULL_MASK, cl.z, 1);
        const bool fresh = valid && (lane == 0 || cl.x != pi || cl.y != pj || cl.z != pk);
        const unsigned fm = __ballot_sync(PLX_FULL_MASK, fresh);
        const int ci = __popc(fm & le_mask) - 1;   // this sample's distinct-cell index
        const int ncell = __popc(fm);
        if (fresh) {
#pragma unroll
            for (int q = 0; q < 8; ++q) sm.rows[ci][q] = rows[q];
            sm.cell[ci] = cl;
        }
        __syncwarp();
        // distinct rows: lane L < ncell owns cell L's corners not shared
        // with cells L-1..L-3 (shared_corner_mask); owned corners get
        // consecutive slots (warp scan), shared ones the slot of their owner
        int nrow;
        if (NEAREST) {
            nrow = ncell;
            if (lane < ncell) {
                const int32_t r = sm.rows[lane][0];
                sm.urow[lane] = r;
                sm.uidx[lane][0] = r >= 0 ? (uint16_t)lane : (uint16_t)kZeroSlot;
            }
        } else {
            unsigned m[4] = {0u, 0u, 0u, 0u}, rv = 0u;
            int ob[4] = {0, 0, 0, 0};
            if (lane < ncell) {
                const int4 c = sm.cell[lane];
#pragma unroll
                for (int b = 1; b <= 3; ++b) {   // runs are contiguous: nest the masks
                    if (lane - b >= 0) {
                        m[b] = shared_corner_mask(c, sm.cell[lane - b], ob[b]);
                        if (b > 1) m[b] &= m[b - 1];
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) rv |= (sm.rows[lane][q] >= 0 ? 1u : 0u) << q;
            }
            const unsigned own = lane < ncell ? (~m[1] & rv & 0xffu) : 0u;
            const int cnt = __popc(own);
            int incl = cnt;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int y = __shfl_up_sync(PLX_FULL_MASK, incl, off);
                if (lane >= off) incl += y;
            }
            nrow = __shfl_sync(PLX_FULL_MASK, incl, 31);
            if (lane < ncell) {
                int u = incl - cnt;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if ((own >> q) & 1u) {
                        sm.uidx[lane][q] = (uint16_t)u;
                        sm.urow[u] = sm.rows[lane][q];
                        ++u;
                    } else if (!((rv >> q) & 1u)) {
                        sm.uidx[lane][q] = (uint16_t)kZeroSlot;
                    }
                }
            }
            __syncwarp();
            if (lane < ncell) {
                const unsigned sh = m[1] & rv;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if ((sh >> q) & 1u) {
                        const int b = ((m[3] >> q) & 1u) ? 3 : ((m[2] >> q) & 1u) ? 2 : 1;
                        const int o = b == 3 ? ob[3] : b == 2 ? ob[2] : ob[1];
                        sm.uidx[lane][q] = sm.uidx[lane - b][q + o];
                    }
                }
            }
        }
        if (lane == 0) sm.d[kZeroSlot] = make_float4(0.f, 0.f, 0.f, 0.f);
        __syncwarp();
        // the distinct rows: 16 rows per pass (4 per warp instruction),
        // coalesced float4 loads; the next pass's loads are issued before
        // this pass is reduced (software pipeline)
        auto load_pass = [&](int r0, float4 *v) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int rr = r0 + 4 * u + sub;
                const int32_t row =
                    rr < nrow ? (DIAG == 1 ? (sm.urow[rr] & 0xffff) : sm.urow[rr]) : -1;
                v[u] = (row >= 0 && part < 7)
                           ? __ldg(reinterpret_cast<const float4 *>(G.table + (int64_t)row * PLX_STRIDE) + part)
                           : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        };
        float4 vc[4], vn[4];
        load_pass(0, vc);
        nx_q = nw + __shfl_sync(PLX_FULL_MASK, claim, 0);
        if (nx_q < nseg) seg_at(S, nx_q, nx_sg, nx_ray);
        for (int r0 = 0; r0 < nrow; r0 += 16) {
            if (r0 + 16 < nrow) load_pass(r0 + 16, vn);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float x[4] = {vc[u].x, vc[u].y, vc[u].z, vc[u].w};
                float pa = 0.f, pb = 0.f;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    pa = __fmaf_rn(x[e], cA[e], pa);
                    pb = __fmaf_rn(x[e], cB[e], pb);
                }
                // gather the row's channel sums at its part-0 lane
                const float a1 = __shfl_down_sync(PLX_FULL_MASK, pa, 1);
                const float a2 = __shfl_down_sync(PLX_FULL_MASK, pa, 2);
                const float b2 = __shfl_down_sync(PLX_FULL_MASK, pb, 2);
                const float a3 = __shfl_down_sync(PLX_FULL_MASK, pa, 3);
                const float a4 = __shfl_down_sync(PLX_FULL_MASK, pa, 4);
                const float b4 = __shfl_down_sync(PLX_FULL_MASK, pb, 4);
                const float a5 = __shfl_down_sync(PLX_FULL_MASK, pa, 5);
                const float a6 = __shfl_down_sync(PLX_FULL_MASK, pa, 6);
                const float pR = (pa + a1) + a2, pG = (b2 + a3) + a4, pB = (b4 + a5) + a6;
                const int rr = r0 + 4 * u + sub;
                if (part == 0 && rr < nrow) sm.d[rr] = make_float4(pR, pG, pB, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) vc[u] = vn[u];
        }
        if (nx_q < nseg) fetch2(nx_ray);
        __syncwarp();
        double x0 = 0.0, x1 = 0.0, x2 = 0.0, q0 = 0.0, q1 = 0.0, q2 = 0.0;
        if (valid) {
            float c0 = 0.f, c1 = 0.f, c2 = 0.f;
            constexpr int NQ = NEAREST ? 1 : 8;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const float4 d = sm.d[sm.uidx[ci][q]];
                float w = 1.f;
                if (!NEAREST)
                    w = ((q & 4) ? f4.x : 1.f - f4.x) * ((q & 2) ? f4.y : 1.f - f4.y) *
                        ((q & 1) ? f4.z : 1.f - f4.z);
                c0 = __fmaf_rn(w, d.x, c0);
                c1 = __fmaf_rn(w, d.y, c1);
                c2 = __fmaf_rn(w, d.z, c2);
            }
            S.c[k] = make_float4(c0, c1, c2, 0.f);
            const double wi = S.w[k];
            const double cr0 = relu((double)c0), cr1 = relu((double)c1), cr2 = relu((double)c2);
            x0 = wi * cr0;   // K:224-229: only the positive part is accumulated
            x1 = wi * cr1;
            x2 = wi * cr2;
            if (ABS) {
                const double Ti = S.T[k];
                const double bn = (Ti - wi) > 0.0 ? 1.0 : 0.0, bi = Ti > 0.0 ? 1.0 : 0.0;
                q0 = cr0 * (bn - bi);
                q1 = cr1 * (bn - bi);
                q2 = cr2 * (bn - bi);
            }
        }
        x0 = warp_sum(x0);
        x1 = warp_sum(x1);
        x2 = warp_sum(x2);
        if (ABS) {
            q0 = warp_sum(q0);
            q1 = warp_sum(q1);
            q2 = warp_sum(q2);
        }
        if (lane == 0) {
            double *o = S.seg_sum + 6 * sg;
            o[0] = x0;
            o[1] = x1;
            o[2] = x2;
            o[3] = q0;
            o[4] = q1;
            o[5] = q2;
        }
        __syncwarp();
    }
}

template <bool ABS, bool NEAREST, int MINB, int DIAG = 0>
__global__ void __launch_bounds__(128, MINB)
    scatter_kernel(DGrid G, RayArgs R, KOpts O, Outs out, Scratch S) {
    R.idx = ray_index(R);
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    const bool cauchy = S.sig != nullptr;
    __shared__ SmemChunk smem_all[4];
    SmemChunk &sc = smem_all[warp];
    double mse_part = 0.0, cau_part = 0.0;
    const int64_t nseg = *S.nseg_total;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    // static interleave: a ray's consecutive segments go to the warps of one
    // block at the same time (shared rows in one L1); dynamic scheduling
    // measured 93 -> 129 us
    // The next segment's descriptor is prefetched in two dependent levels
    // (seg_ray, then the ray's fields) during this segment, and this
    // segment's records are loaded before its prefix sums are reduced.
    int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    int64_t nx_sg = 0;
    int nx_ray = 0;
    if (q < nseg) seg_at(S, q, nx_sg, nx_ray);
    int nx_first = 0, nx_ns = 0;
    int64_t nx_src = 0;
    auto fetch2 = [&](int r_) {
        nx_first = S.seg_first[r_];
        nx_ns = S.ns[r_];
        nx_src = ray_src(R, r_);
    };
    if (q < nseg) fetch2(nx_ray);
    for (; q < nseg; q += nw) {
        const int64_t sg = nx_sg;
        const int64_t ray = nx_ray;
        const int64_t src = nx_src;
        const int ns_r = nx_ns;
        const int64_t s0 = nx_first, s1 = s0 + ((ns_r + 31) >> 5);
        const int64_t qn = q + nw;
        if (qn < nseg) seg_at(S, qn, nx_sg, nx_ray);
        const int j = (int)(sg - s0) * 32 + lane;
        const bool incl = j < ns_r;
        const unsigned mask = __ballot_sync(PLX_FULL_MASK, incl);
        double att = 1.0, Ti = 0.0, wi = 0.0, sig = 0.0;
        float4 c4 = make_float4(0.f, 0.f, 0.f, 0.f), f4 = c4;
        int4 cl = make_int4(0, 0, 0, 0);
        if (incl) {
            const int64_t k = ray * S.cap + j;
            att = S.att[k];
            Ti = S.T[k];
            wi = S.w[k];
            c4 = S.c[k];
            load_cell_f(S, k, !NEAREST, cl, f4);
            if (G.identity) {
                int32_t r8[8];
                identity_rows<NEAREST>(G, cl, r8);
                if (!NEAREST) {
                    *reinterpret_cast<int4 *>(&sc.rows[lane][0]) = make_int4(r8[0], r8[1], r8[2], r8[3]);
                    *reinterpret_cast<int4 *>(&sc.rows[lane][4]) = make_int4(r8[4], r8[5], r8[6], r8[7]);
                } else {
                    sc.rows[lane][0] = r8[0];
                }
            } else if (!NEAREST) {
                *reinterpret_cast<int4 *>(&sc.rows[lane][0]) = S.rows[2 * k];
                *reinterpret_cast<int4 *>(&sc.rows[lane][4]) = S.rows[2 * k + 1];
            } else {
                sc.rows[lane][0] = S.rows[2 * k].x;
            }
            if (cauchy) sig = S.sig[k];
        }
        // ray totals and the prefix of the segments before this one
        double C0 = 0.0, C1 = 0.0, C2 = 0.0, Q0 = 0.0, Q1 = 0.0, Q2 = 0.0;
        double B0 = 0.0, B1 = 0.0, B2 = 0.0;
        // short rays (<= 4 segments: nearly all of them) -- every lane sums
        // the few segment sums itself in segment order (broadcast loads, no
        // shuffles); long rays -- lane-strided partial sums + warp reduction.
        // The path depends only on the ray, so all of a ray's segments see
        // bit-identical totals.
        const bool few = s1 - s0 <= 4;
        for (int64_t t = few ? s0 : s0 + lane; t < s1; t += few ? 1 : 32) {
            const double *p = S.seg_sum + 6 * t;
            C0 += p[0];
            C1 += p[1];
            C2 += p[2];
            if (ABS) {
                Q0 += p[3];
                Q1 += p[4];
                Q2 += p[5];
            }
            if (t < sg) {   // before this segment: P (relative) / Q prefix (absolute)
                B0 += ABS ? p[3] : p[0];
                B1 += ABS ? p[4] : p[1];
                B2 += ABS ? p[5] : p[2];
            }
        }
        if (!few) {
            C0 = warp_sum(C0);
            C1 = warp_sum(C1);
            C2 = warp_sum(C2);
            if (ABS) {
                Q0 = warp_sum(Q0);
                Q1 = warp_sum(Q1);
                Q2 = warp_sum(Q2);
            }
            B0 = warp_sum(B0);
            B1 = warp_sum(B1);
            B2 = warp_sum(B2);
        }
        double P0 = B0, P1 = B1, P2 = B2;
        const double Tfin = S.ray_d[3 * ray], dlt_last = S.ray_d[3 * ray + 1],
                     last_si = S.ray_d[3 * ray + 2];
        // rgb = C + T bg (K:234-238); 360: C + the background's T_fg C_bg
        const double X0 = S.rgb_add ? S.rgb_add[3 * ray] : Tfin * O.bg[0];
        const double X1 = S.rgb_add ? S.rgb_add[3 * ray + 1] : Tfin * O.bg[1];
        const double X2 = S.rgb_add ? S.rgb_add[3 * ray + 2] : Tfin * O.bg[2];
        const double rgb0 = C0 + X0, rgb1 = C1 + X1, rgb2 = C2 + X2;
        const bool first = sg == s0 && !out.bgmode;
        if (first && lane == 0 && out.rgb) {
            out.rgb[3 * ray + 0] = rgb0;
            out.rgb[3 * ray + 1] = rgb1;
            out.rgb[3 * ray + 2] = rgb2;
        }
        // ---------------- upstream (K:330-341) ----------------
        double up0, up1, up2;
        if (out.mse_mode) {
            const double e0 = rgb0 - ray_tgt(R, src, 0);
            const double e1 = rgb1 - ray_tgt(R, src, 1);
            const double e2 = rgb2 - ray_tgt(R, src, 2);
            if (first && lane == 0) mse_part += e0 * e0 + e1 * e1 + e2 * e2;
            up0 = out.up_scale * e0;
            up1 = out.up_scale * e1;
            up2 = out.up_scale * e2;
        } else {
            up0 = ray_tgt(R, src, 0);
            up1 = ray_tgt(R, src, 1);
            up2 = ray_tgt(R, src, 2);
        }
        // ---------------- reverse sweep + scatter (K:343-410) ----------------
        // sf before sample i in the reference's reverse sweep:
        //   relative: T bg + sum_{j>i} w_j c_j = rgb - P_i      (K:351-353, 381-383)
        //   absolute: -bg [T>0] + sum_{j>i} c_j (bn_j - bi_j)   (K:346-349, 374-376)
        const double bend = Tfin > 0.0 ? 1.0 : 0.0;
        float bf[9];
        ray_basis_rec(S, ray, bf);
        LaneAcc<NEAREST, DIAG> ra;
        ra.init(lane, bf);
        if (qn < nseg) fetch2(nx_ray);
        // delta of this sample (K:200-205): step, except at the last position
        const double dl = rec_is_last(S, cl, last_si) ? dlt_last : O.step;
        const double cc0 = relu((double)c4.x), cc1 = relu((double)c4.y),
                     cc2 = relu((double)c4.z);
        double gsig;
        if (!ABS) {
            const double y0 = incl ? wi * cc0 : 0.0, y1 = incl ? wi * cc1 : 0.0,
                         y2 = incl ? wi * cc2 : 0.0;
            const double i0 = P0 + warp_scan_add(y0, lane), i1 = P1 + warp_scan_add(y1, lane),
                         i2 = P2 + warp_scan_add(y2, lane);
            const double sf0 = rgb0 - i0, sf1 = rgb1 - i1, sf2 = rgb2 - i2;
            gsig = dl * (up0 * (Ti * att * cc0 - sf0) + up1 * (Ti * att * cc1 - sf1) +
                         up2 * (Ti * att * cc2 - sf2));
        } else {
            const double Tn = Ti - wi;
            const double bn = Tn > 0.0 ? 1.0 : 0.0, bi = Ti > 0.0 ? 1.0 : 0.0;
            const double y0 = incl ? cc0 * (bn - bi) : 0.0, y1 = incl ? cc1 * (bn - bi) : 0.0,
                         y2 = incl ? cc2 * (bn - bi) : 0.0;
            const double i0 = P0 + warp_scan_add(y0, lane), i1 = P1 + warp_scan_add(y1, lane),
                         i2 = P2 + warp_scan_add(y2, lane);
            const double sf0 = -O.bg[0] * bend + (Q0 - i0);
            const double sf1 = -O.bg[1] * bend + (Q1 - i1);
            const double sf2 = -O.bg[2] * bend + (Q2 - i2);
            const double galpha =
                (up0 * (cc0 * bn + sf0) + up1 * (cc1 * bn + sf1) + up2 * (cc2 * bn + sf2));
            gsig = galpha * dl * att;
        }
        if (incl && cauchy) {   // K:384-386
            cau_part += log(1.0 + 2.0 * sig * sig);
            gsig += out.lam_cauchy * 4.0 * sig / (1.0 + 2.0 * sig * sig);
        }
        if (S.bup) {   // 360: the beta regulariser on the foreground transmittance (K:858-859)
            const double bup = S.bup[ray];
            if (bup != 0.0) gsig += bup * (-dl * Tfin);
        }
        // ---- lane-parallel staging of the scatter payload (K:387-410) ----
        const unsigned below = mask & lt_mask;
        const int pl = below ? lane - 1 : lane;   // the list is dense
        const int qi = __shfl_sync(PLX_FULL_MASK, cl.x, pl);
        const int qj = __shfl_sync(PLX_FULL_MASK, cl.y, pl);
        const int qk = __shfl_sync(PLX_FULL_MASK, cl.z, pl);
        int mv = 0;
        if (incl) {
            if (!below) {
                mv = MV_FAR;   // segment start: nothing carried
            } else {
                const int di = cl.x - qi, dj = cl.y - qj, dk = cl.z - qk;
                if (di | dj | dk) {
                    const bool adj = !NEAREST && di >= -1 && di <= 1 && dj >= -1 && dj <= 1 &&
                                     dk >= -1 && dk <= 1;
                    mv = adj ? (MV_ADJ | ((di + 1) << 4) | ((dj + 1) << 2) | (dk + 1)) : MV_FAR;
                }
            }
            sc.mv[lane] = mv;
        }
        // flip in effect when sample `lane` is added: prefix xor of the moves
        int fx = incl ? axis_bits(mv) : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int y = __shfl_up_sync(PLX_FULL_MASK, fx, off);
            if (lane >= off) fx ^= y;
        }
        const int fl = fx;
        if (incl) {
            const float gk[4] = {(float)gsig, c4.x > 0.f ? (float)(up0 * wi) : 0.f,
                                 c4.y > 0.f ? (float)(up1 * wi) : 0.f,
                                 c4.z > 0.f ? (float)(up2 * wi) : 0.f};
            if (NEAREST) {
#pragma unroll
                for (int L = 0; L < 32; ++L) sc.val[L][lane] = L < 4 ? gk[L] : 0.f;
            } else {
                // corner e = q ^ fl of physical slot q: xor-ing a bit of the
                // corner index swaps (1 - f, f) on that axis
                const float lx = (fl & 4) ? f4.x : 1.f - f4.x, hx = (fl & 4) ? 1.f - f4.x : f4.x;
                const float ly = (fl & 2) ? f4.y : 1.f - f4.y, hy = (fl & 2) ? 1.f - f4.y : f4.y;
                const float lz = (fl & 1) ? f4.z : 1.f - f4.z, hz = (fl & 1) ? 1.f - f4.z : f4.z;
#pragma unroll
                for (int qs = 0; qs < 8; ++qs) {
                    const float w = ((qs & 4) ? hx : lx) * ((qs & 2) ? hy : ly) *
                                    ((qs & 1) ? hz : lz);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) sc.val[4 * qs + kk][lane] = w * gk[kk];
                }
            }
        }
        __syncwarp();
        // ---- serial, in sample order: moves (flushes) + one add ----
        const int n = __popc(mask);
        for (int jj = 0; jj < n; ++jj) {
            const int mvj = sc.mv[jj];
            if (mvj) ra.move(mvj, sc, jj, out.grad, out.tmask, lane);
            ra.acc += sc.val[lane][jj];
        }
        ra.flush_all(out.grad, out.tmask, lane);
        __syncwarp();
    }
    cau_part = warp_sum(cau_part);   // one pair of f64 atomics per warp
    if (lane == 0) {
        if (mse_part != 0.0) atomicAdd(out.sums + 0, mse_part);
        if (cau_part != 0.0) atomicAdd(out.sums + 1, cau_part);
    }
}

// ---------------------------------------------------------------------------
// msi_bg_kernel -- the background stage of the 360 backward (K:749-833 and
// the background half of K:835-881).  The foreground runs through the
// bounded kernels (march_bwd_kernel, colour_kernel, scatter_kernel in
// bgmode); between colour and scatter this kernel, one warp per ray, takes
// the ray's foreground colour total and T_fg, samples the sphere layers past
// the grid's exit (lane = layer, compacted in layer order), composites them
// from T_fg over black, writes rgb / T_fg / T and the mse and beta sums, and
// leaves the scatter two per-ray scalars: the background colour (the
// foreground samples' reverse-sweep suffix rgb - P_i then includes it) and
// the beta upstream.  The background samples' own reverse sweep and texel
// scatter (f64 atomics) follow here: they come after every foreground
// sample, so their suffix sums are background-only.
struct MsiBgArgs {
    MsiDev B;
    double lam_beta, beta_eps;
    double *tfg, *trans;     // (N) outputs
    double *bg_grad;         // [L*H*W][4]
    uint8_t *bg_tmask;
};

// Per-warp shared records of the background samples (dynamic shared memory,
// L-1 crossings per warp).
struct BgRecs {
    double *t, *sig, *dlt, *T, *w, *c0, *c1, *c2;
    int *lay;   // layer, or -1: not composited (sigma < 0 or past the stop)
};

__global__ void __launch_bounds__(128) msi_bg_kernel(DGrid G, RayArgs R, KOpts O, Outs out,
                                                     Scratch S, MsiBgArgs M) {
    extern __shared__ double bg_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nc = M.B.L - 1;   // crossings per ray at most
    BgRecs rec;
    {
        double *base = bg_smem + (int64_t)warp * nc * 9;
        rec.t = base;
        rec.sig = base + nc;
        rec.dlt = base + 2 * nc;
        rec.T = base + 3 * nc;
        rec.w = base + 4 * nc;
        rec.c0 = base + 5 * nc;
        rec.c1 = base + 6 * nc;
        rec.c2 = base + 7 * nc;
        rec.lay = reinterpret_cast<int *>(base + 8 * nc);
    }
    const unsigned lt = (1u << lane) - 1u;
    double mse_part = 0.0, beta_part = 0.0;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t ray = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; ray < R.n; ray += nwarps) {
        double o[3], d[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            o[a] = __ldg(R.origins + 3 * ray + a);
            d[a] = __ldg(R.dirs + 3 * ray + a);
        }
        double Cf0 = 0.0, Cf1 = 0.0, Cf2 = 0.0;
        const int ns = S.ns[ray];
        if (ns > 0) {
            const int64_t s0 = S.seg_first[ray];
            ray_colour_totals(S, s0, s0 + ((ns + 31) >> 5), lane, Cf0, Cf1, Cf2);
        }
        const double tfg = S.ray_d[3 * ray];
        double T = tfg, A = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
        int nx = 0;
        if (T >= O.stop) {   // K:749-803
            double t0a, t1a;
            ray_aabb(o, d, G.lo, G.hi, t0a, t1a);
            const double t_exit = t1a > 0.0 ? t1a : 0.0;
            const double bdot = o[0] * d[0] + o[1] * d[1] + o[2] * d[2];
            const double c0n = o[0] * o[0] + o[1] * o[1] + o[2] * o[2];
            for (int l0 = 0; l0 < nc; l0 += 32) {
                const int l = l0 + lane;
                bool hit = false;
                double tl = 0.0;
                if (l < nc) {
                    const double rad = __ldg(M.B.radii + l);
                    const double disc = bdot * bdot - c0n + rad * rad;
                    if (disc > 0.0) {
                        tl = -bdot + sqrt(disc);
                        hit = !(tl < t_exit);
                    }
                }
                const unsigned hm = __ballot_sync(PLX_FULL_MASK, hit);
                if (hit) {
                    const int q = nx + __popc(hm & lt);
                    rec.t[q] = tl;
                    rec.lay[q] = l;
                }
                nx += __popc(hm);
            }
            __syncwarp();
            bool stopped = false;
            for (int q0 = 0; q0 < nx; q0 += 32) {
                const int q = q0 + lane;
                bool incl = false;
                double att = 1.0, sig = 0.0, dlt = 0.0, o4[4] = {0.0, 0.0, 0.0, 0.0};
                if (q < nx && !stopped) {
                    if (q + 1 < nx) dlt = rec.t[q + 1] - rec.t[q];
                    else if (q >= 1) dlt = rec.t[q] - rec.t[q - 1];
                    else dlt = 1.0;
                    const double t = rec.t[q];
                    int idx4[4];
                    double w4[4];
                    bg_stencil(M.B.H, M.B.W, o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2],
                               idx4, w4);
                    bg_fetch(M.B, rec.lay[q], idx4, w4, o4);
                    sig = o4[0];
                    incl = sig >= 0.0;
                    if (incl) att = exp(-sig * dlt);
                }
                double Ti = 0.0, wi = 0.0;
                if (__any_sync(PLX_FULL_MASK, incl))
                    composite_chunk<false>(incl, att, lane, O.stop, T, A, Ti, wi, stopped);
                if (q < nx) {
                    rec.sig[q] = sig;
                    rec.dlt[q] = dlt;
                    rec.T[q] = Ti;
                    rec.w[q] = wi;
                    rec.c0[q] = o4[1];
                    rec.c1[q] = o4[2];
                    rec.c2[q] = o4[3];
                    if (!incl) rec.lay[q] = -1;
                }
                if (incl) {
                    if (o4[1] > 0.0) b0 += wi * o4[1];
                    if (o4[2] > 0.0) b1 += wi * o4[2];
                    if (o4[3] > 0.0) b2 += wi * o4[3];
                }
            }
            __syncwarp();
        }
        const double Cb0 = warp_sum(b0), Cb1 = warp_sum(b1), Cb2 = warp_sum(b2);
        const double cr = Cf0 + Cb0, cg = Cf1 + Cb1, cb = Cf2 + Cb2;
        if (lane == 0) {
            if (out.rgb) {
                out.rgb[3 * ray] = cr;
                out.rgb[3 * ray + 1] = cg;
                out.rgb[3 * ray + 2] = cb;
            }
            M.tfg[ray] = tfg;
            M.trans[ray] = T;
            S.rgb_add[3 * ray] = Cb0;
            S.rgb_add[3 * ray + 1] = Cb1;
            S.rgb_add[3 * ray + 2] = Cb2;
        }
        // upstream, beta regulariser (K:808-833)
        double up0, up1, up2;
        if (out.mse_mode) {
            const double e0 = cr - ray_tgt(R, ray, 0), e1 = cg - ray_tgt(R, ray, 1),
                         e2 = cb - ray_tgt(R, ray, 2);
            if (lane == 0) mse_part += e0 * e0 + e1 * e1 + e2 * e2;
            up0 = out.up_scale * e0;
            up1 = out.up_scale * e1;
            up2 = out.up_scale * e2;
        } else {
            up0 = ray_tgt(R, ray, 0);
            up1 = ray_tgt(R, ray, 1);
            up2 = ray_tgt(R, ray, 2);
        }
        double tc = tfg;
        if (tc < M.beta_eps) tc = M.beta_eps;
        if (tc > 1.0 - M.beta_eps) tc = 1.0 - M.beta_eps;
        if (M.lam_beta > 0.0 && lane == 0) beta_part += log(tc) + log(1.0 - tc);
        double bup = 0.0;
        if (M.lam_beta > 0.0 && M.beta_eps < tfg && tfg < 1.0 - M.beta_eps)
            bup = M.lam_beta * (1.0 / tc - 1.0 / (1.0 - tc));
        if (lane == 0) S.bup[ray] = bup;
        // background reverse sweep + texel scatter (K:835-881, lay >= 0)
        double sf0 = 0.0, sf1 = 0.0, sf2 = 0.0;
        for (int q0 = ((nx - 1) >> 5) << 5; q0 >= 0; q0 -= 32) {
            const int q = q0 + lane;
            const bool valid = q < nx && rec.lay[q] >= 0;
            double sig = 0.0, dlt = 0.0, Ti = 0.0, w = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
            if (valid) {
                sig = rec.sig[q];
                dlt = rec.dlt[q];
                Ti = rec.T[q];
                w = rec.w[q];
                c0 = rec.c0[q];
                c1 = rec.c1[q];
                c2 = rec.c2[q];
            }
            const double cc0 = c0 > 0.0 ? c0 : 0.0, cc1 = c1 > 0.0 ? c1 : 0.0,
                         cc2 = c2 > 0.0 ? c2 : 0.0;
            const double y0 = valid ? w * cc0 : 0.0, y1 = valid ? w * cc1 : 0.0,
                         y2 = valid ? w * cc2 : 0.0;
            const double i0 = warp_scan_add(y0, lane), i1 = warp_scan_add(y1, lane),
                         i2 = warp_scan_add(y2, lane);
            const double tot0 = __shfl_sync(PLX_FULL_MASK, i0, 31),
                         tot1 = __shfl_sync(PLX_FULL_MASK, i1, 31),
                         tot2 = __shfl_sync(PLX_FULL_MASK, i2, 31);
            const double s0 = sf0 + (tot0 - i0), s1 = sf1 + (tot1 - i1), s2 = sf2 + (tot2 - i2);
            sf0 += tot0;
            sf1 += tot1;
            sf2 += tot2;
            if (valid) {
                const double att = exp(-sig * dlt);
                const double gsig = dlt * (up0 * (Ti * att * cc0 - s0) + up1 * (Ti * att * cc1 - s1) +
                                           up2 * (Ti * att * cc2 - s2));
                const double t = rec.t[q];
                const int lay = rec.lay[q];
                int idx4[4];
                double w4[4];
                bg_stencil(M.B.H, M.B.W, o[0] + t * d[0], o[1] + t * d[1], o[2] + t * d[2], idx4,
                           w4);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int64_t flat = (int64_t)lay * M.B.H * M.B.W + idx4[k];
                    const double wq = w4[k];
                    M.bg_tmask[flat] = 1;
                    double *gb = M.bg_grad + 4 * flat;
                    atomicAdd(gb, wq * gsig);
                    if (c0 > 0.0) atomicAdd(gb + 1, wq * up0 * w);
                    if (c1 > 0.0) atomicAdd(gb + 2, wq * up1 * w);
                    if (c2 > 0.0) atomicAdd(gb + 3, wq * up2 * w);
                }
            }
        }
        __syncwarp();
    }
    mse_part = warp_sum(mse_part);
    beta_part = warp_sum(beta_part);
    if (lane == 0) {
        if (mse_part != 0.0) atomicAdd(out.sums + 0, mse_part);
        if (beta_part != 0.0) atomicAdd(out.sums + 2, beta_part);
    }
}
}  // namespace plx

using namespace plx;

namespace {

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;

bool grid_ok(const plx_grid *g) {
    return g && g->links && g->dims[0] >= 2 && g->dims[1] >= 2 && g->dims[2] >= 2 &&
           (g->rows == 0 || (g->table && g->density)) && g->dims[0] < (1 << 21) &&
           g->dims[1] < (1 << 21) && g->dims[2] < (1 << 21) &&
           g->dims[0] * g->dims[1] * g->dims[2] < (int64_t)1 << 31;
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

// Kernel variants over (absolute, nearest).
#define PLX_DISPATCH(o, KERNEL, MINB, GRID, ...)                                           \
    do {                                                                                  \
        if ((o)->nearest) {                                                               \
            if ((o)->absolute) KERNEL<true, true, MINB><<<GRID, kThreads, 0, s>>>(__VA_ARGS__); \
            else KERNEL<false, true, MINB><<<GRID, kThreads, 0, s>>>(__VA_ARGS__);         \
        } else {                                                                          \
            if ((o)->absolute) KERNEL<true, false, MINB><<<GRID, kThreads, 0, s>>>(__VA_ARGS__); \
            else KERNEL<false, false, MINB><<<GRID, kThreads, 0, s>>>(__VA_ARGS__);        \
        }                                                                                 \
    } while (0)

template <bool ABS, bool NEAREST, int MINB>
int march_blocks_per_sm() {
    static int nb = 0;
    if (!nb) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, march_bwd_kernel<ABS, NEAREST, MINB>,
                                                      kThreads, 0);
        if (nb <= 0) nb = 1;
    }
    return nb;
}

#ifndef PLX_COLOUR_MINB
#define PLX_COLOUR_MINB 6
#endif
#ifndef PLX_SCATTER_MINB
#define PLX_SCATTER_MINB 5
#endif
#ifndef PLX_MARCH_MINB
#define PLX_MARCH_MINB 6
#endif
constexpr int kMarchMinB = PLX_MARCH_MINB, kColourMinB = PLX_COLOUR_MINB, kScatterMinB = PLX_SCATTER_MINB;

// Resident blocks per SM of any kernel instantiation (cached per kernel).
template <typename KernelT>
int resident_blocks(KernelT *k) {
    static int nb = 0;
    if (!nb) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, kThreads, 0);
        if (nb <= 0) nb = 1;
    }
    return nb;
}

int march_blocks(const plx_render_opts *o) {
    if (o->nearest)
        return o->absolute ? march_blocks_per_sm<true, true, kMarchMinB>()
                           : march_blocks_per_sm<false, true, kMarchMinB>();
    return o->absolute ? march_blocks_per_sm<true, false, kMarchMinB>()
                       : march_blocks_per_sm<false, false, kMarchMinB>();
}

template <int MODE>
void launch_fwd(const plx_render_opts *o, bool ABSF, dim3 grid, cudaStream_t s, DGrid G,
                RayArgs R, KOpts K, Outs out) {
    if (o->nearest) {
        if (ABSF) march_kernel<MODE, true, true><<<grid, kThreads, 0, s>>>(G, R, K, out);
        else march_kernel<MODE, false, true><<<grid, kThreads, 0, s>>>(G, R, K, out);
    } else {
        if (ABSF) march_kernel<MODE, true, false><<<grid, kThreads, 0, s>>>(G, R, K, out);
        else march_kernel<MODE, false, false><<<grid, kThreads, 0, s>>>(G, R, K, out);
    }
}

// Capacity of one warp slot: every march position of the longest chord (R:67-69).
int64_t max_records(const plx_grid *g, double step) {
    double d2 = 0.0;
    for (int a = 0; a < 3; ++a) d2 += (g->hi[a] - g->lo[a]) * (g->hi[a] - g->lo[a]);
    return (int64_t)ceil(sqrt(d2) / step) + 4;
}

// Records are kept for every march position of the longest chord of every
// ray of a wave; a batch larger than the budget runs in waves.
// Record budget per wave: 64 GiB of a 180 GB B200 (C5 sweep, 2^18..2^20
// rays: 8 GiB waves 29.4 / 32.8 / 35.0 M rays/s, 32 GiB 30.4 / 33.7 / 36.0;
// with the segment order and dead bricks 32 GiB 36.6 / 41.4 / 44.9, 64 GiB
// 37.5 / 42.3 / 45.6, 96 GiB the same as 64).  Only batches that need it
// allocate it (the scratch is sized for min(batch, wave)).
#ifndef PLX_RECORD_GIB
#define PLX_RECORD_GIB 64
#endif
constexpr int64_t kRecordBudget = (int64_t)PLX_RECORD_GIB << 30;   // bytes of records per wave
constexpr int64_t kRecordBytes = 112;                 // att, T, w, c, cell, f, rows, sig

struct ScratchLayout {
    int64_t wave, cap, bytes;
    int nseg_max;
    int64_t off_ns, off_segfirst, off_segray, off_rayd, off_basis, off_att, off_T, off_w, off_c, off_cell, off_f, off_rows,
        off_sig, off_segsum, off_rgbadd, off_bup, off_segkey, off_ord, off_bucket;
};

// Record budget per wave; PLX_RECORD_MB overrides it (tests force
// multi-wave batches at small sizes).
int64_t record_budget() {
    static int64_t v = -1;
    if (v < 0) {
        const char *e = getenv("PLX_RECORD_MB");
        v = (e && atoll(e) > 0) ? atoll(e) << 20 : kRecordBudget;
    }
    return v;
}

ScratchLayout layout(const plx_grid *g, const plx_render_opts *o, int64_t n_rays) {
    ScratchLayout L;
    L.cap = max_records(g, o->step);
    L.nseg_max = (int)((L.cap + 31) / 32);
    int64_t wave = record_budget() / (L.cap * kRecordBytes);
    if (wave < 1024) wave = 1024;
    if (n_rays > 0 && n_rays < wave) wave = n_rays;
    // equal waves: a fixed-size wave left a small last wave (2^18 rays at
    // 512^3: six waves of 43 K rays + one of 2.9 K) whose launches ran the
    // kernels mostly as tails
    if (n_rays > wave) {
        const int64_t nw = (n_rays + wave - 1) / wave;
        wave = (n_rays + nw - 1) / nw;
    }
    L.wave = wave;
    const int64_t n = wave * L.cap;
    int64_t off = 256;
    auto take = [&](int64_t bytes) {
        const int64_t at = off;
        off = (off + bytes + 255) & ~(int64_t)255;
        return at;
    };
    L.off_ns = take(wave * 4);
    L.off_segfirst = take(wave * 4);
    L.off_segray = take(wave * L.nseg_max * 4);
    L.off_rayd = take(wave * 24);
    L.off_basis = take(wave * 48);
    L.off_att = take(n * 8);
    L.off_T = take(n * 8);
    L.off_w = take(n * 8);
    L.off_c = take(n * 16);
    L.off_cell = take(n * 16);
    L.off_f = take(n * 16);
    L.off_rows = take(n * 32);
    L.off_sig = take(n * 8);
    L.off_segsum = take(wave * L.nseg_max * 48);
    L.off_rgbadd = take(wave * 24);
    L.off_bup = take(wave * 8);
    L.off_segkey = take(wave * L.nseg_max * 4);
    L.off_ord = take(wave * L.nseg_max * 8);
    L.off_bucket = take(kBuckets * 4);
    L.bytes = off;
    return L;
}

int check_rays(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o, bool views) {
    if (!grid_ok(g) || !rays || !o || rays->n < 0) return PLX_EINVAL;
    if (rays->n >= (int64_t)1 << 31) return PLX_EINVAL;
    if (rays->cams) {
        const plx_cameras *c = rays->cams;
        if (!c->cams || c->n_views < 1 || c->width < 1 || c->height < 1) return PLX_EINVAL;
        return (o->step > 0.0) ? PLX_OK : PLX_EINVAL;
    }
    // an empty batch is a no-op: its (zero-length) buffers may be null
    if (rays->n > 0 && (!rays->origins || !rays->dirs || (views && !rays->viewdirs)))
        return PLX_EINVAL;
    if (!(o->step > 0.0)) return PLX_EINVAL;
    return PLX_OK;
}

template <int MODE>
int launch_march(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o, Outs out,
                 void *stream) {
    const int rc = check_rays(g, rays, o, MODE == FWD);
    if (rc != PLX_OK) return rc;
    if (rays->n == 0) return PLX_OK;
    DGrid G = make_dgrid(*g);
    RayArgs R{rays->origins, rays->dirs, rays->viewdirs, rays->target, rays->jitter, rays->idx,
              rays->n, nullptr, make_campool(rays->cams), 0};
    KOpts K{o->step, o->stop_thresh, {o->bg[0], o->bg[1], o->bg[2]},
            reinterpret_cast<unsigned long long *>(o->stats)};
    int64_t blocks = (rays->n + kWarps - 1) / kWarps;   // static grid-stride over rays
    const int64_t cap = (int64_t)num_sms() * 12;
    if (blocks > cap) blocks = cap;
    launch_fwd<MODE>(o, MODE == FWD && o->absolute, dim3((unsigned)blocks), (cudaStream_t)stream,
                     G, R, K, out);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}

}  // namespace

extern "C" int plx_render_fwd(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o,
                              double *out_rgb, double *out_trans, double *out_wsum, void *stream) {
    if (!out_rgb && rays && rays->n > 0) return PLX_EINVAL;
    Outs out{};
    out.rgb = out_rgb;
    out.trans = out_trans;
    out.wsum = out_wsum;
    return launch_march<FWD>(g, rays, o, out, stream);
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
    return plx::render_fused_bwd_impl(g, rays, nullptr, o, mse_mode, up_scale, lam_cauchy, gb,
                                      out_rgb, out_sums, scratch, scratch_bytes, stream, 0);
}

// idx_off: optional device int64 added to rays->idx by the kernels (the
// native step's graph replays with the batch as a moving slice of a fixed
// permutation buffer).
int plx::render_fused_bwd_impl(const plx_grid *g, const plx_rays *rays, const int64_t *idx_off,
                               const plx_render_opts *o, int32_t mse_mode, double up_scale,
                               double lam_cauchy, plx_grad *gb, double *out_rgb,
                               double *out_sums, void *scratch, int64_t scratch_bytes,
                               void *stream, int counters_ready, void *after_march,
                               const MsiHook *msi) {
    if (!gb || !gb->grad || !gb->tmask || !out_sums) return PLX_EINVAL;
    const int rc = check_rays(g, rays, o, true);
    if (rc != PLX_OK) return rc;
    if (rays->n == 0) return PLX_OK;
    if ((!rays->target && !(rays->cams && rays->cams->rgb && mse_mode)) || !scratch)
        return PLX_EINVAL;
    const ScratchLayout L = layout(g, o, rays->n);
    if (scratch_bytes < L.bytes) return PLX_EINVAL;
    DGrid G = make_dgrid(*g);
    KOpts K{o->step, o->stop_thresh, {o->bg[0], o->bg[1], o->bg[2]},
            reinterpret_cast<unsigned long long *>(o->stats)};
    char *base = reinterpret_cast<char *>(scratch);
    Scratch S;
    S.counter = reinterpret_cast<int *>(base);
    S.cap = L.cap;
    S.nseg_max = L.nseg_max;
    S.nseg_total = reinterpret_cast<int *>(base) + 1;
    S.ns = reinterpret_cast<int *>(base + L.off_ns);
    S.seg_first = reinterpret_cast<int *>(base + L.off_segfirst);
    S.seg_ray = reinterpret_cast<int *>(base + L.off_segray);
    S.ray_d = reinterpret_cast<double *>(base + L.off_rayd);
    S.basis = reinterpret_cast<float4 *>(base + L.off_basis);
    S.att = reinterpret_cast<double *>(base + L.off_att);
    S.T = reinterpret_cast<double *>(base + L.off_T);
    S.w = reinterpret_cast<double *>(base + L.off_w);
    S.c = reinterpret_cast<float4 *>(base + L.off_c);
    S.cell = reinterpret_cast<int4 *>(base + L.off_cell);
    {   // packed cell records when i, j, k and a flag fit 32 bits (PLX_PACK=0: off)
        static const bool pack_env = [] {
            const char *e = getenv("PLX_PACK");
            return !(e && e[0] == '0');
        }();
        int b[3];
        for (int a = 0; a < 3; ++a) {
            b[a] = 0;
            while (((g->dims[a] - 1) >> b[a]) > 0) ++b[a];
        }
        S.pack = pack_env && b[0] + b[1] + b[2] <= 31;
        S.pk_sy = b[0];
        S.pk_sz = b[0] + b[1];
    }
    S.f = reinterpret_cast<float4 *>(base + L.off_f);
    S.rows = reinterpret_cast<int4 *>(base + L.off_rows);
    S.sig = lam_cauchy > 0.0 ? reinterpret_cast<double *>(base + L.off_sig) : nullptr;
    S.seg_sum = reinterpret_cast<double *>(base + L.off_segsum);
    S.rgb_add = msi ? reinterpret_cast<double *>(base + L.off_rgbadd) : nullptr;
    S.bup = msi ? reinterpret_cast<double *>(base + L.off_bup) : nullptr;
    // PLX_SEG_ORDER=0 / 1 forces the spatial segment order off / on (tests,
    // A/B); by default waves of at least kSegOrderMinRays rays use it
    static const int order_env = [] {
        const char *e = getenv("PLX_SEG_ORDER");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    S.seg_key = reinterpret_cast<int *>(base + L.off_segkey);
    int shift[3];
    for (int a = 0; a < 3; ++a) {   // 16 buckets per axis over the base cells
        int bits = 0;
        while (((g->dims[a] - 2) >> bits) > 0) ++bits;
        shift[a] = bits > kBucketBits ? bits - kBucketBits : 0;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int sms = num_sms();
    for (int64_t w0 = 0; w0 < rays->n; w0 += L.wave) {
        const int64_t nw = rays->n - w0 < L.wave ? rays->n - w0 : L.wave;
        RayArgs R{rays->origins, rays->dirs, rays->viewdirs, rays->target,
                  rays->jitter ? rays->jitter + w0 : nullptr, rays->idx ? rays->idx + w0 : nullptr,
                  nw, rays->idx ? idx_off : nullptr, make_campool(rays->cams), 0};
        if (!rays->idx && rays->cams) {
            R.base = w0;   // camera pool rows w0 + r
        } else if (!rays->idx) {   // implicit indices: offset the arrays instead
            R.origins += 3 * w0;
            R.dirs += 3 * w0;
            R.viewdirs += 3 * w0;
            R.target += 3 * w0;
        }
        const bool ordered = order_env >= 0 ? order_env == 1 : nw >= kSegOrderMinRays;
        S.ord = ordered ? reinterpret_cast<int2 *>(base + L.off_ord) : nullptr;
        S.bucket = ordered ? reinterpret_cast<int *>(base + L.off_bucket) : nullptr;
        Outs out{};
        out.rgb = out_rgb ? out_rgb + 3 * w0 : nullptr;
        out.sums = out_sums;
        out.grad = gb->grad;
        out.tmask = gb->tmask;
        out.mse_mode = mse_mode;
        out.up_scale = up_scale;
        out.lam_cauchy = lam_cauchy;
        out.bgmode = msi != nullptr;
        // ray counter, segment counter, colour scheduler (zeroed by the
        // native step's prologue kernel for the first wave)
        if (!(counters_ready && w0 == 0) &&
            cudaMemsetAsync(S.counter, 0, 3 * sizeof(int), s) != cudaSuccess)
            return PLX_ECUDA;
        int64_t mb = (int64_t)sms * march_blocks(o);
        if (mb > (nw + kWarps - 1) / kWarps) mb = (nw + kWarps - 1) / kWarps;
        PLX_DISPATCH(o, march_bwd_kernel, kMarchMinB, dim3((unsigned)mb), G, R, K, out, S);
        if (after_march && w0 == 0 &&
            cudaEventRecord((cudaEvent_t)after_march, s) != cudaSuccess)
            return PLX_ECUDA;
        // segment kernels: exactly one resident wave, grid-stride over the
        // segments (8 blocks per SM at 5-6 resident left a partial second
        // wave that started only after the first had done its share)
        int cb, sb;
        if (o->nearest) {
            cb = o->absolute ? resident_blocks(colour_kernel<true, true, kColourMinB>)
                             : resident_blocks(colour_kernel<false, true, kColourMinB>);
            sb = o->absolute ? resident_blocks(scatter_kernel<true, true, kScatterMinB>)
                             : resident_blocks(scatter_kernel<false, true, kScatterMinB>);
        } else {
            cb = o->absolute ? resident_blocks(colour_kernel<true, false, kColourMinB>)
                             : resident_blocks(colour_kernel<false, false, kColourMinB>);
            sb = o->absolute ? resident_blocks(scatter_kernel<true, false, kScatterMinB>)
                             : resident_blocks(scatter_kernel<false, false, kScatterMinB>);
        }
        if (S.ord) {
            seg_key_kernel<<<sms * 2, 256, 0, s>>>(S, shift[0], shift[1], shift[2]);
            seg_scan_kernel<<<1, 1024, 0, s>>>(S);
            seg_place_kernel<<<sms * 2, 256, 0, s>>>(S);
        }
#ifdef PLX_DIAG
        // diagnostic builds (profiles/r2b_diag.md): PLX_DIAG_MODE bit 1 / 2 /
        // 4 launches the colour (L2-resident rows) / scatter (no reductions)
        // / scatter (L2-resident reductions) variant BEFORE the real kernel;
        // its outputs are overwritten or go to a private buffer
        if (!o->nearest && !o->absolute && !msi) {
            static const int diag = getenv("PLX_DIAG_MODE") ? atoi(getenv("PLX_DIAG_MODE")) : 0;
            static float *dgrad = nullptr;
            static double *dsums = nullptr;
            if (diag && !dgrad) {
                cudaMalloc(&dgrad, (size_t)65536 * PLX_STRIDE * sizeof(float));
                cudaMalloc(&dsums, 64);
            }
            Outs dout = out;
            dout.rgb = nullptr;
            dout.sums = dsums;
            dout.grad = dgrad;
            if (diag & 1) {
                colour_kernel<false, false, kColourMinB, 1><<<sms * cb, kThreads, 0, s>>>(G, R, S);
                cudaMemsetAsync(S.counter + 2, 0, sizeof(int), s);   // colour scheduler
            }
            PLX_DISPATCH(o, colour_kernel, kColourMinB, dim3((unsigned)(sms * cb)), G, R, S);
            if (diag & 2)
                scatter_kernel<false, false, kScatterMinB, 1><<<sms * sb, kThreads, 0, s>>>(G, R, K, dout, S);
            if (diag & 4)
                scatter_kernel<false, false, kScatterMinB, 2><<<sms * sb, kThreads, 0, s>>>(G, R, K, dout, S);
        } else
#endif
        PLX_DISPATCH(o, colour_kernel, kColourMinB, dim3((unsigned)(sms * cb)), G, R, S);
        if (msi) {   // 360: the background stage between colour and scatter
            MsiBgArgs M{{msi->data, msi->radii, (int)msi->L, (int)msi->H, (int)msi->W},
                        msi->lam_beta, msi->beta_eps, msi->out_tfg + w0, msi->out_trans + w0,
                        msi->bg_grad, msi->bg_tmask};
            const size_t smem = (size_t)kWarps * (msi->L - 1) * 9 * sizeof(double);
            static bool smem_set = false;
            if (!smem_set) {   // up to kMaxCross crossings per warp (74 KB per block)
                cudaFuncSetAttribute(msi_bg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kWarps * kMaxCross * 9 * (int)sizeof(double));
                smem_set = true;
            }
            int64_t nb = (nw + kWarps - 1) / kWarps;
            if (nb > (int64_t)sms * 8) nb = (int64_t)sms * 8;
            msi_bg_kernel<<<(unsigned)nb, kThreads, smem, s>>>(G, R, K, out, S, M);
        }
        PLX_DISPATCH(o, scatter_kernel, kScatterMinB, dim3((unsigned)(sms * sb)), G, R, K, out, S);
    }
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}

#ifdef PLX_TIMELINE
extern "C" int plx_debug_timeline(unsigned long long *host, int n) {
    return cudaMemcpyFromSymbol(host, g_timeline, sizeof(unsigned long long) * 2 * n) == cudaSuccess
               ? PLX_OK : PLX_ECUDA;
}
#endif

extern "C" int plx_max_weight(const plx_grid *g, const plx_rays *rays, const plx_render_opts *o,
                              double *out_w, void *stream) {
    if (!out_w) return PLX_EINVAL;
    Outs out{};
    out.maxw = out_w;
    return launch_march<MAXW>(g, rays, o, out, stream);
}

// all_rays (camera.py:292-314) of pool rows on the device: one thread per ray.
__global__ void generate_rays_kernel(CamPool C, const int64_t *idx, int64_t n, double *o,
                                     double *d, double *v, double *rgb) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = idx ? idx[r] : r;
        double oo[3], dd[3];
        if (o || d) {
            cam_march_ray(C, src, oo, dd);
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                if (o) o[3 * r + a] = oo[a];
                if (d) d[3 * r + a] = dd[a];
            }
        }
        if (v) {
            cam_view_dir(C, src, dd);
#pragma unroll
            for (int a = 0; a < 3; ++a) v[3 * r + a] = dd[a];
        }
        if (rgb) {
#pragma unroll
            for (int a = 0; a < 3; ++a) rgb[3 * r + a] = (double)C.rgb[3 * src + a];
        }
    }
}

extern "C" int plx_generate_rays(const plx_cameras *cams, const int64_t *idx, int64_t n,
                                 double *origins, double *dirs, double *viewdirs, double *rgb,
                                 void *stream) {
    if (!cams || !cams->cams || n < 0 || cams->width < 1 || cams->height < 1) return PLX_EINVAL;
    if (rgb && !cams->rgb) return PLX_EINVAL;
    if (n == 0) return PLX_OK;
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    generate_rays_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        make_campool(cams), idx, n, origins, dirs, viewdirs, rgb);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}

namespace {
struct CamRecord {
    double v[PLX_CAM];
};
__global__ void to_ndc_kernel(CamRecord cam, double *o, double *d, uint8_t *valid, int64_t n) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
        const bool ok = cam_to_ndc(cam.v, o + 3 * r, d + 3 * r);
        if (valid) valid[r] = ok ? 1 : 0;
    }
}
}  // namespace

extern "C" int plx_to_ndc(const double *cam, double *origins, double *dirs, uint8_t *valid,
                          int64_t n, void *stream) {
    if (!cam || n < 0 || (n > 0 && (!origins || !dirs))) return PLX_EINVAL;
    if (n == 0) return PLX_OK;
    CamRecord c;
    for (int k = 0; k < PLX_CAM; ++k) c.v[k] = cam[k];
    int64_t blocks = (n + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (blocks > cap) blocks = cap;
    to_ndc_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(c, origins, dirs, valid, n);
    return cudaPeekAtLastError() == cudaSuccess ? PLX_OK : PLX_ECUDA;
}
