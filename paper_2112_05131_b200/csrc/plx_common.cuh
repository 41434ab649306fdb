// plx_common.cuh -- device-side helpers shared by the sm_100a kernels.
//
// Arithmetic follows the reference kernels (pkg/src/plenoxel/_kernels.py,
// "K") operation by operation in float64; translation units that include this
// header are compiled with -fmad=false so no a*b+c is contracted into an FMA
// (numba compiles the reference without fast-math, i.e. without contraction).
// With f32-representable table values this reproduces the reference's sample
// positions, stencil rows/weights, opacities and pre-clamp colours bit-for-bit.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/plx.h"

#define PLX_FULL_MASK 0xffffffffu

namespace plx {

// Kernel-side copy of plx_grid (passed by value).
// Empty-space bricks: kBrick^3 trilinear base cells.
constexpr int kBrick = 8;

struct DGrid {
    const int32_t *__restrict__ links;
    const float *__restrict__ table;     // SH rows (column 0 unused)
    const float *__restrict__ density;   // sigma per row
    const uint32_t *__restrict__ cell_occ;
    const float *sigma_lat;              // lattice-indexed sigma mirror, NaN = empty (mutable)
    bool identity;                       // links[c] == c for every point (dense grid)
    // optional dead-brick bitmask over 8^3-cell bricks (plx_build_brick_dead):
    // bit set = no position inside can be composited; Bx, By, Bz bricks per axis
    const uint32_t *brick_dead;
    int32_t Bx, By, Bz;
    int32_t Dx, Dy, Dz;
    double lo[3], hi[3], scale[3], dmax[3];
};

inline DGrid make_dgrid(const plx_grid &g) {
    DGrid d;
    d.links = g.links;
    d.table = g.table;
    d.density = g.density;
    d.cell_occ = g.cell_occ;
    d.sigma_lat = g.sigma_lat;
    // the caller aliases the sigma mirror to density exactly when the grid is
    // identity-linked (SparseGrid.lattice_sigma)
    d.identity = g.sigma_lat != nullptr && g.sigma_lat == g.density;
    // the mask is kept only beside a separate sigma mirror (sparse grids)
    d.brick_dead = (g.sigma_lat && !d.identity) ? g.brick_dead : nullptr;
    d.Bx = (int32_t)((g.dims[0] - 2) / kBrick + 1);
    d.By = (int32_t)((g.dims[1] - 2) / kBrick + 1);
    d.Bz = (int32_t)((g.dims[2] - 2) / kBrick + 1);
    d.Dx = (int32_t)g.dims[0];
    d.Dy = (int32_t)g.dims[1];
    d.Dz = (int32_t)g.dims[2];
    for (int a = 0; a < 3; ++a) {
        d.lo[a] = g.lo[a];
        d.hi[a] = g.hi[a];
        d.scale[a] = g.scale[a];
        d.dmax[a] = g.dmax[a];
    }
    return d;
}

// sh.py:18-22
constexpr double SH_C0 = 0.28209479177387814;
constexpr double SH_C1 = 0.4886025119029199;
constexpr double SH_C2_0 = 1.0925484305920792;
constexpr double SH_C2_2 = 0.31539156525252005;
constexpr double SH_C2_4 = 0.5462742152960396;

// K:27-37
__device__ __forceinline__ void sh_basis9(double x, double y, double z, double *b) {
    b[0] = SH_C0;
    b[1] = -SH_C1 * y;
    b[2] = SH_C1 * z;
    b[3] = -SH_C1 * x;
    b[4] = SH_C2_0 * x * y;
    b[5] = -SH_C2_0 * y * z;
    b[6] = SH_C2_2 * (2.0 * z * z - x * x - y * y);
    b[7] = -SH_C2_0 * x * z;
    b[8] = SH_C2_4 * (x * x - y * y);
}

// K:40-81.  Returns (t0, t1); miss iff t1 <= t0.
__device__ __forceinline__ void ray_aabb(const double *o, const double *d, const double *lo,
                                         const double *hi, double &t0_out, double &t1_out) {
    double t0 = 0.0, t1 = __longlong_as_double(0x7ff0000000000000ULL);  // +inf
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (fabs(d[a]) < 1e-15) {
            if (o[a] < lo[a] || o[a] > hi[a]) {
                t0_out = 1.0;
                t1_out = 0.0;
                return;
            }
        } else {
            double ta = (lo[a] - o[a]) / d[a];
            double tb = (hi[a] - o[a]) / d[a];
            if (ta > tb) {
                double tmp = ta;
                ta = tb;
                tb = tmp;
            }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
    }
    t0_out = t0;
    t1_out = t1;
}

// K:163-170
__device__ __forceinline__ double clamp_coord(double p, double lo, double scale, double dmax) {
    double g = (p - lo) * scale;
    if (g < 0.0) g = 0.0;
    if (g > dmax) g = dmax;
    return g;
}

// Flat C-order lattice index; 32-bit (plx_grid dims are checked to hold
// fewer than 2^31 points), as are the coordinates and corner offsets below:
// 64-bit index math was an eighth of the march's instructions.
__device__ __forceinline__ int32_t flat(const DGrid &G, int32_t i, int32_t j, int32_t k) {
    return (i * G.Dy + j) * G.Dz + k;
}

// Per-ray march parameters (K:189-205).
struct RayMarch {
    double o[3], d[3];
    double t0, L;
    int64_t nsamp;   // 0 on a miss
};

__device__ __forceinline__ void ray_march_setup(RayMarch &rm, const DGrid &G, double step,
                                                double jitter) {
    double t1;
    ray_aabb(rm.o, rm.d, G.lo, G.hi, rm.t0, t1);
    rm.t0 = rm.t0 + jitter * step;
    rm.L = t1 - rm.t0;
    rm.nsamp = 0;
    if (rm.L > 0.0) {
        int64_t n = (int64_t)ceil(rm.L / step - 1e-9);
        rm.nsamp = n < 1 ? 1 : n;
    }
}

// Lattice coordinates of sample si (K:203-208): t, delta, g.
__device__ __forceinline__ void sample_coords(const RayMarch &rm, const DGrid &G, double step,
                                              int64_t si, double &t, double &dlt, double *g) {
    t = rm.t0 + (double)(int32_t)si * step;   // si < nsamp <= the record capacity
    dlt = si < rm.nsamp - 1 ? step : rm.L - step * (double)(rm.nsamp - 1);
#pragma unroll
    for (int a = 0; a < 3; ++a) g[a] = clamp_coord(rm.o[a] + t * rm.d[a], G.lo[a], G.scale[a], G.dmax[a]);
}

// Stencil (K:84-123): rows[8] (-1 = empty), the fractional offsets f[3] and
// the base cell (trilinear) or lattice point (nearest) ijk[3]; the corner
// weight is stencil_w(f, q) (recomputed instead of stored, to save
// registers; same float64 products as K:115-121).  Returns 1 or 8.
template <bool NEAREST>
__device__ __forceinline__ int stencil(const DGrid &G, const double *g, int32_t *rows, double *f,
                                       bool &any_occ, int *ijk) {
    if (NEAREST) {
        int32_t i = (int32_t)(g[0] + 0.5), j = (int32_t)(g[1] + 0.5), k = (int32_t)(g[2] + 0.5);
        if (i > G.Dx - 1) i = G.Dx - 1;
        if (j > G.Dy - 1) j = G.Dy - 1;
        if (k > G.Dz - 1) k = G.Dz - 1;
        ijk[0] = i;
        ijk[1] = j;
        ijk[2] = k;
        rows[0] = __ldg(G.links + flat(G, i, j, k));
        any_occ = rows[0] >= 0;
        return 1;
    }
    int32_t i0 = (int32_t)g[0], j0 = (int32_t)g[1], k0 = (int32_t)g[2];
    if (i0 > G.Dx - 2) i0 = G.Dx - 2;
    if (j0 > G.Dy - 2) j0 = G.Dy - 2;
    if (k0 > G.Dz - 2) k0 = G.Dz - 2;
    ijk[0] = i0;
    ijk[1] = j0;
    ijk[2] = k0;
    if (G.cell_occ) {
        const int32_t c = flat(G, i0, j0, k0);
        if (!((__ldg(G.cell_occ + (c >> 5)) >> (c & 31)) & 1u)) {
            any_occ = false;
            return 8;
        }
    }
    f[0] = g[0] - (double)i0;
    f[1] = g[1] - (double)j0;
    f[2] = g[2] - (double)k0;
    const int32_t *base = G.links + flat(G, i0, j0, k0);
    const int32_t sy = G.Dz, sx = G.Dy * G.Dz;
    bool occ = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const int32_t r = __ldg(base + ((q >> 2) & 1) * sx + ((q >> 1) & 1) * sy + (q & 1));
        rows[q] = r;
        occ |= r >= 0;
    }
    any_occ = occ;
    return 8;
}

// Stencil rows of a base cell / lattice point (K:84-123), -1 = empty.
template <bool NEAREST>
__device__ __forceinline__ void load_rows(const DGrid &G, const int *ijk, int32_t *rows) {
    const int32_t c = flat(G, ijk[0], ijk[1], ijk[2]);
    if (G.identity) {   // dense identity-linked grid: row = lattice point
        const int32_t sy = G.Dz, sx = G.Dy * G.Dz;
        rows[0] = (int32_t)c;
        if (!NEAREST) {
#pragma unroll
            for (int q = 1; q < 8; ++q)
                rows[q] = (int32_t)(c + ((q >> 2) & 1) * sx + ((q >> 1) & 1) * sy + (q & 1));
        }
        return;
    }
    const int32_t *base = G.links + c;
    if (NEAREST) {
        rows[0] = __ldg(base);
        return;
    }
    const int32_t sy = G.Dz, sx = G.Dy * G.Dz;
#pragma unroll
    for (int q = 0; q < 8; ++q) rows[q] = __ldg(base + ((q >> 2) & 1) * sx + ((q >> 1) & 1) * sy + (q & 1));
}

// Trilinear corner weight (K:114-121): corner q = (di, dj, dk) = bits (4, 2, 1).
template <bool NEAREST>
__device__ __forceinline__ double stencil_w(const double *f, int q) {
    if (NEAREST) return 1.0;
    const double wx = (q & 4) ? f[0] : 1.0 - f[0];
    const double wy = (q & 2) ? f[1] : 1.0 - f[1];
    const double wz = (q & 1) ? f[2] : 1.0 - f[2];
    return wx * wy * wz;
}

// ---- warp collectives (f64) ----------------------------------------------
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(PLX_FULL_MASK, x, off);
    return x;
}

__device__ __forceinline__ double warp_scan_add(double x, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        double y = __shfl_up_sync(PLX_FULL_MASK, x, off);
        if (lane >= off) x = y + x;
    }
    return x;
}

__device__ __forceinline__ double warp_scan_mul(double x, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        double y = __shfl_up_sync(PLX_FULL_MASK, x, off);
        if (lane >= off) x = y * x;
    }
    return x;
}

// Vectorised fire-and-forget f32 reduction (sm_90+ PTX; SASS REDG.E.ADD.F32x4).
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

__device__ __forceinline__ void red_add_v4(float *addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}

__device__ __forceinline__ void red_add_f32(float *addr, float a) {
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(addr), "f"(a) : "memory");
}

}  // namespace plx

namespace plx {

// _color_at (K:138-152) in f32 FMAs: per corner the 3 SH dots with the
// basis, then the corner weight; c = pre-clamp colour (empty rows skipped).
template <bool NEAREST>
__device__ __forceinline__ void colour_at_f32(const DGrid &G, const int32_t *rows, const double *f,
                                              const float *bf, float *c) {
    constexpr int NQ = NEAREST ? 1 : 8;
    float c0 = 0.f, c1 = 0.f, c2 = 0.f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        int32_t r = rows[q];
        if (r < 0) continue;
        const float4 *row = reinterpret_cast<const float4 *>(G.table + (int64_t)r * PLX_STRIDE);
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
        const float w = (float)stencil_w<NEAREST>(f, q);
        c0 = __fmaf_rn(w, a0, c0);
        c1 = __fmaf_rn(w, a1, c1);
        c2 = __fmaf_rn(w, a2, c2);
    }
    c[0] = c0;
    c[1] = c1;
    c[2] = c2;
}

// _sigma_at (K:126-135) of the stencil at lattice coordinates g: float64 sum
// over occupied corners in corner order; occ = any corner occupied.  With the
// lattice-indexed mirror G.sigma_lat (NaN = empty point) the corner values
// are ONE gather level -- no links, no rows -- and an empty corner simply
// adds nothing, exactly as the reference skips it.  rows[] is filled only on
// the links path (rows_ok = true); otherwise the caller loads it with
// load_rows() for the samples it keeps.
template <bool NEAREST>
__device__ __forceinline__ bool sigma_at(const DGrid &G, const double *g, double *f, int *ijk,
                                         int32_t *rows, double &sig, bool &rows_ok) {
    sig = 0.0;
    rows_ok = false;
    bool occ = false;
    if (!G.sigma_lat) {
        stencil<NEAREST>(G, g, rows, f, occ, ijk);
        rows_ok = true;
        if (!occ) return false;
        constexpr int NQ = NEAREST ? 1 : 8;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            if (rows[q] >= 0) sig += stencil_w<NEAREST>(f, q) * (double)__ldg(G.density + rows[q]);
        return true;
    }
    if (NEAREST) {
        int32_t i = (int32_t)(g[0] + 0.5), j = (int32_t)(g[1] + 0.5), k = (int32_t)(g[2] + 0.5);
        if (i > G.Dx - 1) i = G.Dx - 1;
        if (j > G.Dy - 1) j = G.Dy - 1;
        if (k > G.Dz - 1) k = G.Dz - 1;
        ijk[0] = i;
        ijk[1] = j;
        ijk[2] = k;
        const float s = G.sigma_lat[flat(G, i, j, k)];
        if (s != s) return false;
        sig = stencil_w<NEAREST>(f, 0) * (double)s;
        return true;
    }
    int32_t i0 = (int32_t)g[0], j0 = (int32_t)g[1], k0 = (int32_t)g[2];
    if (i0 > G.Dx - 2) i0 = G.Dx - 2;
    if (j0 > G.Dy - 2) j0 = G.Dy - 2;
    if (k0 > G.Dz - 2) k0 = G.Dz - 2;
    ijk[0] = i0;
    ijk[1] = j0;
    ijk[2] = k0;
    if (G.brick_dead) {   // a dead brick: no position inside can be composited
        const int32_t b = (((unsigned)i0 / kBrick) * G.By + (unsigned)j0 / kBrick) * G.Bz +
                          (unsigned)k0 / kBrick;
        if ((__ldg(G.brick_dead + (b >> 5)) >> (b & 31)) & 1u) return false;
    }
    const int32_t c = flat(G, i0, j0, k0);
    // with a brick mask the occupancy bit only adds a dependent load before
    // the sigma gathers (an all-empty cell exits below just the same):
    // C5 2^20 44.1 -> 44.9 M rays/s without it
    if (G.cell_occ && !G.brick_dead && !((__ldg(G.cell_occ + (c >> 5)) >> (c & 31)) & 1u)) return false;
    f[0] = g[0] - (double)i0;
    f[1] = g[1] - (double)j0;
    f[2] = g[2] - (double)k0;
    const float *base = G.sigma_lat + c;
    const int32_t sy = G.Dz, sx = G.Dy * G.Dz;
    float s[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) s[q] = base[((q >> 2) & 1) * sx + ((q >> 1) & 1) * sy + (q & 1)];
    // All 8 corners occupied with sigma < 0 (NaN compares false): every term
    // w_q sigma_q is <= 0 and the largest weight is >= 1/8, so the f64 sum is
    // strictly negative and the caller drops the sample (K:293) -- the
    // weights need not be formed.  Most march positions take this exit.
    if (s[0] < 0.f && s[1] < 0.f && s[2] < 0.f && s[3] < 0.f && s[4] < 0.f && s[5] < 0.f &&
        s[6] < 0.f && s[7] < 0.f) {
        sig = -1.0;
        return true;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        if (s[q] != s[q]) continue;   // empty corner (K:131: skipped)
        occ = true;
        sig += stencil_w<NEAREST>(f, q) * (double)s[q];
    }
    return occ;
}

// Brick of the base cell at lattice coordinates g (sigma_at's clamped cell).
__device__ __forceinline__ int32_t brick_of(const DGrid &G, const double *g) {
    int32_t i0 = (int32_t)g[0], j0 = (int32_t)g[1], k0 = (int32_t)g[2];
    if (i0 > G.Dx - 2) i0 = G.Dx - 2;
    if (j0 > G.Dy - 2) j0 = G.Dy - 2;
    if (k0 > G.Dz - 2) k0 = G.Dz - 2;
    return (((unsigned)i0 / kBrick) * G.By + (unsigned)j0 / kBrick) * G.Bz + (unsigned)k0 / kBrick;
}

__device__ __forceinline__ void brick_xyz(const DGrid &G, const double *g, int &bx, int &by,
                                          int &bz) {
    int32_t i0 = (int32_t)g[0], j0 = (int32_t)g[1], k0 = (int32_t)g[2];
    if (i0 > G.Dx - 2) i0 = G.Dx - 2;
    if (j0 > G.Dy - 2) j0 = G.Dy - 2;
    if (k0 > G.Dz - 2) k0 = G.Dz - 2;
    bx = (int)((unsigned)i0 / kBrick);
    by = (int)((unsigned)j0 / kBrick);
    bz = (int)((unsigned)k0 / kBrick);
}

__device__ __forceinline__ bool brick_is_dead(const DGrid &G, int32_t b) {
    return (__ldg(G.brick_dead + (b >> 5)) >> (b & 31)) & 1u;
}

// The sigma of lattice point c became >= 0: no brick whose cells have c as a
// corner is dead any more (the mask stays a conservative under-approximation
// between rebuilds).  Bits are tested before the atomic: most are clear.
__device__ __forceinline__ void brick_revive(uint32_t *bits, int32_t c, int32_t Dx, int32_t Dy,
                                             int32_t Dz) {
    const int32_t x = c / (Dy * Dz), y = (c / Dz) % Dy, z = c % Dz;
    const int32_t By = (Dy - 2) / kBrick + 1, Bz = (Dz - 2) / kBrick + 1;
    int32_t bx[2], by[2], bz[2];
    // cells x-1 and x (those that exist) have the point as a corner
    bx[0] = (x > 0 ? x - 1 : 0) / kBrick;
    bx[1] = (x < Dx - 1 ? x : Dx - 2) / kBrick;
    by[0] = (y > 0 ? y - 1 : 0) / kBrick;
    by[1] = (y < Dy - 1 ? y : Dy - 2) / kBrick;
    bz[0] = (z > 0 ? z - 1 : 0) / kBrick;
    bz[1] = (z < Dz - 1 ? z : Dz - 2) / kBrick;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if ((a && bx[1] == bx[0]) || (b && by[1] == by[0]) || (e && bz[1] == bz[0])) continue;
                const int32_t k = (bx[a] * By + by[b]) * Bz + bz[e];
                const uint32_t m = 1u << (k & 31);
                if (bits[k >> 5] & m) atomicAnd(bits + (k >> 5), ~m);
            }
}

}  // namespace plx
